timeout 900 python -m pytest tests -m gpu -q -x -k "parity or cluster or slabs or pml" > gpurun_out/r2_t26.log 2>&1; echo t=$?; tail -1 gpurun_out/r2_t26.log
B="python bench.py --steps 120 --warmup 8 --no-cpu --no-e2e"
for v in tma notma tma notma; do
  if [ $v = notma ]; then E="FDTD_NO_TMA=1"; else E=""; fi
  env $E $B > gpurun_out/r2_b26.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_b26.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],4))"; done
$B --workload cfg5 > gpurun_out/r2_b26.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_b26.log').read().strip().splitlines()[-1]); r=d['roofline']; print('tma cfg5', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],4))"
FDTD_LIB=variants/phases.so python tools/phase_times.py --out gpurun_out/phases_tma.txt > /dev/null 2>&1
timeout 600 python tools/checked_run.py --out gpurun_out/checked_tma.json > gpurun_out/checked_tma.log 2>&1; echo checked=$?
