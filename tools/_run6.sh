python -m pytest tests -m gpu -q -x -k "parity or boundary or slabs" > gpurun_out/r2_gputests6.log 2>&1; echo tests=$?
B="python bench.py --steps 40 --warmup 8 --no-cpu --no-e2e"
$B > gpurun_out/r2_b6_a.log 2>&1; echo a=$?
FDTD_POST_THREADS=256 FDTD_ROM_BATCH=4 $B > gpurun_out/r2_b6_b.log 2>&1; echo b=$?
FDTD_POST_THREADS=384 FDTD_ROM_BATCH=8 $B > gpurun_out/r2_b6_c.log 2>&1; echo c=$?
$B --workload cfg5 > gpurun_out/r2_b6_d.log 2>&1; echo d=$?
FDTD_POST_THREADS=256 FDTD_ROM_BATCH=4 $B --workload cfg5 > gpurun_out/r2_b6_e.log 2>&1; echo e=$?
