python -m pytest tests -m gpu -q -x -s -k "parity or boundary or slabs or pml" > gpurun_out/r2_gputests4.log 2>&1; echo tests=$?
python bench.py --steps 40 --warmup 8 --no-cpu > gpurun_out/r2_bench4.log 2>&1; echo bench=$?
SHORT="python bench.py --steps 8 --warmup 4 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:postk -s 1 -c 1 -o gpurun_out/post_r02c $SHORT > gpurun_out/ncu_post_r02c.log 2>&1; echo ncu=$?
