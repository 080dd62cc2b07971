B="python bench.py --steps 80 --warmup 8 --no-cpu --no-e2e"
for cfg in "FDTD_CHUNK=256" "FDTD_CHUNK=512" "FDTD_CHUNK=1024" "FDTD_CHUNK=128" "FDTD_WARPS=8" "FDTD_WARPS=2" "FDTD_CHUNK=512 FDTD_WARPS=8"; do
  env $cfg $B > gpurun_out/r2_b19.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/r2_b19.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],3), d['clocks']['sm_mhz'])"
done
