python -m pytest tests -m gpu -q -x -k "parity or boundary or slabs or pml or fullsize" > gpurun_out/r2_gputests5.log 2>&1; echo tests=$?
python bench.py --steps 40 --warmup 8 --no-cpu > gpurun_out/r2_bench5.log 2>&1; echo bench=$?
python bench.py --steps 40 --warmup 8 --no-cpu --no-e2e --workload cfg5 > gpurun_out/r2_bench5_cfg5.log 2>&1; echo bench5=$?
SHORT="python bench.py --steps 8 --warmup 4 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:postk -s 1 -c 1 -o gpurun_out/post_r02d $SHORT > gpurun_out/ncu_post_r02d.log 2>&1; echo ncu=$?
