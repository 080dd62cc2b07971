B="python bench.py --steps 200 --warmup 8 --no-cpu --no-e2e --workload cfg2"
for cfg in "FDTD_CHUNK=64" "FDTD_CHUNK=96" "FDTD_CHUNK=128" "FDTD_CHUNK=192" "FDTD_CHUNK=256" "FDTD_CHUNK=128 FDTD_WARPS=2"; do
  env $cfg $B > gpurun_out/r2_b24.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/r2_b24.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],4), round(r['post_ms_per_launch'],4), d['ms_per_step'])"
done
