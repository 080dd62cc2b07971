#!/bin/bash
# The non-ncu part of tools/profile_round.sh (bench lines of every workload, reference arm, whole-grid
# bench, slab cost, fix-up phase times, checked build, parity evidence).  Usage: bash tools/profile_rest.sh <tag>
set -u
TAG=${1:-rNN}
OUT=gpurun_out
mkdir -p $OUT
python bench.py --impl reference > $OUT/bench_ref_$TAG.log 2>&1; echo "ref=$?"
python bench.py --init random --no-cpu > $OUT/bench_cfg4_random_$TAG.log 2>&1; echo "bench_random=$?"
python tools/wholegrid_bench.py --out $OUT/wholegrid_bench_$TAG.json > $OUT/wholegrid_$TAG.log 2>&1; echo "wholegrid=$?"
for w in cfg2 cfg3 cfg5 cfg4dense; do
  python bench.py --workload $w --no-cpu > $OUT/bench_${w}_$TAG.log 2>&1; echo "bench_$w=$?"
done
[ -f variants/phases.so ] && FDTD_LIB=variants/phases.so python tools/phase_times.py --out $OUT/phases_$TAG.txt \
    > /dev/null 2>&1; echo "phases=$?"
python tools/slab_overhead.py --out $OUT/slab_overhead_$TAG.json > $OUT/slab_$TAG.log 2>&1; echo "slab=$?"
timeout 1200 python tools/checked_run.py --out $OUT/checked_$TAG.json > $OUT/checked_$TAG.log 2>&1; echo "checked=$?"
timeout 1500 python -m pytest tests -m gpu -q -s -k "fullsize or crops or cluster or per_instance or nonfinite" \
    > $OUT/parity_evidence_$TAG.log 2>&1; echo "evidence=$?"
