#!/bin/bash
# Round profiling recipe (run under gpurun from the repo root): full bench line, the ncu launch
# list of a short bench run, and one `ncu --set full` capture each of the sweep and the fix-up.
# Usage: bash tools/profile_round.sh <tag>      (outputs in gpurun_out/)
set -u
TAG=${1:-rNN}
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/bench_full_$TAG.log 2>&1; echo "bench=$?"
SHORT="python bench.py --steps 8 --warmup 4 --no-cpu --no-e2e"
$SHORT > $OUT/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $SHORT \
    > $OUT/ncu_launches_$TAG.log 2>&1; echo "launches=$?"
$SHORT > $OUT/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweepk -s 1 -c 1 -o $OUT/sweep_$TAG $SHORT \
    > $OUT/ncu_sweep_$TAG.log 2>&1; echo "ncu_sweep=$?"
$SHORT > $OUT/plain3_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:postk -s 1 -c 1 -o $OUT/post_$TAG $SHORT \
    > $OUT/ncu_post_$TAG.log 2>&1; echo "ncu_post=$?"
# NEXT-3: the GPU ROM builder's multigrid-PCG kernel on config 5's largest model (MG=1)
[ "${MG:-0}" = 1 ] || exit 0
python tools/rom_build_bench.py --cases cfg5 --out $OUT/rom_build_plain_$TAG.json > $OUT/rom_build_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mg_pcg -s 3 -c 1 -o $OUT/mgpcg_$TAG \
    python tools/rom_build_bench.py --cases cfg5 --out $OUT/rom_build_ncu_$TAG.json > $OUT/ncu_mgpcg_$TAG.log 2>&1
echo "ncu_mgpcg=$?"
