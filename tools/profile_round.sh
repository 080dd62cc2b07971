#!/bin/bash
# Round profiling recipe (run under gpurun from the repo root): bench lines of every workload, the
# ncu launch list of a short bench run, one `ncu --set full` capture each of the sweep and the
# fix-up, the Sec. VI-A replay on the large-model path, the row-slab decomposition cost, the checked
# build runs and the fix-up phase times.  Usage: bash tools/profile_round.sh <tag>   (gpurun_out/)
set -u
TAG=${1:-rNN}
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/bench_full_$TAG.log 2>&1; echo "bench=$?"
python bench.py --impl reference > $OUT/bench_ref_$TAG.log 2>&1; echo "ref=$?"
python bench.py --init random --no-cpu > $OUT/bench_cfg4_random_$TAG.log 2>&1; echo "bench_random=$?"
python tools/wholegrid_bench.py --out $OUT/wholegrid_bench_$TAG.json > $OUT/wholegrid_$TAG.log 2>&1; echo "wholegrid=$?"
for w in cfg2 cfg3 cfg5 cfg4dense; do
  python bench.py --workload $w --no-cpu > $OUT/bench_${w}_$TAG.log 2>&1; echo "bench_$w=$?"
done
SHORT="python bench.py --steps 8 --warmup 4 --no-cpu --no-e2e"
$SHORT > $OUT/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $SHORT \
    > $OUT/ncu_launches_$TAG.log 2>&1; echo "launches=$?"
ncu --set full --clock-control none --import-source on -k regex:sweepk -s 1 -c 1 -o $OUT/sweep_$TAG $SHORT \
    > $OUT/ncu_sweep_$TAG.log 2>&1; echo "ncu_sweep=$?"
ncu --set full --clock-control none --import-source on -k regex:postk -s 1 -c 1 -o $OUT/post_$TAG $SHORT \
    > $OUT/ncu_post_$TAG.log 2>&1; echo "ncu_post=$?"
[ -f variants/phases.so ] && FDTD_LIB=variants/phases.so python tools/phase_times.py --out $OUT/phases_$TAG.txt \
    > /dev/null 2>&1; echo "phases=$?"
python tests/replays/cavity_replay.py --out $OUT/cavity_replay_$TAG.json > $OUT/cavity_$TAG.log 2>&1; echo "cavity=$?"
python tests/replays/cavity_replay.py --literal --out $OUT/cavity_replay_literal_$TAG.json > $OUT/cavity_lit_$TAG.log 2>&1
echo "cavity_literal=$?"
python tools/slab_overhead.py --out $OUT/slab_overhead_$TAG.json > $OUT/slab_$TAG.log 2>&1; echo "slab=$?"
timeout 1200 python tools/checked_run.py --out $OUT/checked_$TAG.json > $OUT/checked_$TAG.log 2>&1; echo "checked=$?"
timeout 1500 python -m pytest tests -m gpu -q -s -k "fullsize or crops or cluster or per_instance or nonfinite" \
    > $OUT/parity_evidence_$TAG.log 2>&1; echo "evidence=$?"
# NEXT-3: the GPU ROM builder's multigrid-PCG kernel on config 5's largest model (MG=1)
[ "${MG:-0}" = 1 ] || exit 0
python tools/rom_build_bench.py --cases cfg5 --out $OUT/rom_build_plain_$TAG.json > $OUT/rom_build_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mg_pcg -s 3 -c 1 -o $OUT/mgpcg_$TAG \
    python tools/rom_build_bench.py --cases cfg5 --out $OUT/rom_build_ncu_$TAG.json > $OUT/ncu_mgpcg_$TAG.log 2>&1
echo "ncu_mgpcg=$?"
