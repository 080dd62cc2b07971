python -m pytest tests -m gpu -q -x -k "cluster or dense" > gpurun_out/r2_gputests10a.log 2>&1; echo clusters=$?
python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests10.log 2>&1; echo tests=$?
B="python bench.py --steps 80 --warmup 8 --no-cpu --no-e2e"
$B > gpurun_out/r2_b10_cfg4.log 2>&1; echo cfg4=$?
$B --workload cfg4dense > gpurun_out/r2_b10_cfg4dense.log 2>&1; echo dense=$?
python tools/checked_run.py > gpurun_out/r2_checked10.log 2>&1; echo checked=$?
