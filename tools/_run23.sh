B="python bench.py --steps 120 --warmup 8 --no-cpu --no-e2e"
for v in eslow efast eslow efast; do FDTD_LIB=variants/$v.so $B > gpurun_out/r2_b23.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_b23.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],3), d['clocks']['sm_mhz'])"; done
FDTD_LIB=variants/efast.so $B --no-energy > gpurun_out/r2_b23.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_b23.log').read().strip().splitlines()[-1]); r=d['roofline']; print('noenergy', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],3))"
FDTD_LIB=variants/efast.so timeout 900 python -m pytest tests -m gpu -q -x -k "parity or slabs or pml or boundary" > gpurun_out/r2_t23.log 2>&1; echo t=$?; tail -2 gpurun_out/r2_t23.log
