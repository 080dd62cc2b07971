timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests15.log 2>&1; echo tests=$?
B="python bench.py --steps 80 --warmup 8 --no-cpu --no-e2e"
$B > gpurun_out/r2_b15_cfg4.log 2>&1; echo cfg4=$?
$B --workload cfg4dense > gpurun_out/r2_b15_cfg4dense.log 2>&1; echo dense=$?
FDTD_K=1 $B --workload cfg4dense > gpurun_out/r2_b15_cfg4dense_k1.log 2>&1; echo densek1=$?
