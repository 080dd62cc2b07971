B="python bench.py --steps 120 --warmup 8 --no-cpu --no-e2e"
for v in nom2pre m2pre nom2pre m2pre; do FDTD_LIB=variants/$v.so $B > gpurun_out/r2_b25.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_b25.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],4))"; done
FDTD_LIB=variants/m2pre.so $B --workload cfg5 > gpurun_out/r2_b25.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_b25.log').read().strip().splitlines()[-1]); r=d['roofline']; print('m2pre cfg5', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],4))"
FDTD_LIB=variants/phases.so python tools/phase_times.py --out gpurun_out/phases_m2pre.txt > /dev/null 2>&1
FDTD_LIB=variants/m2pre.so timeout 900 python -m pytest tests -m gpu -q -x -k "parity or cluster or slabs" > gpurun_out/r2_t25.log 2>&1; echo t=$?; tail -1 gpurun_out/r2_t25.log
