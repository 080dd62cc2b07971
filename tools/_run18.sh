FDTD_LIB=variants/phasesldg.so python tools/phase_times.py --out gpurun_out/phases_ldg.txt > /dev/null 2>&1; echo p=$?
B="python bench.py --steps 80 --warmup 8 --no-cpu --no-e2e"
for v in base ldg base ldg; do FDTD_LIB=variants/$v.so $B > gpurun_out/r2_b18_$v.log 2>&1; echo $v=$?; python -c "
import json; d=json.loads(open('gpurun_out/r2_b18_$v.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],3))"; done
FDTD_LIB=variants/ldg.so timeout 600 python -m pytest tests -m gpu -q -x -k "parity or cluster or slabs" > gpurun_out/r2_t18.log 2>&1; echo t=$?
