B="python bench.py --steps 80 --warmup 8 --no-cpu --no-e2e"
for w in cfg4 cfg5; do $B --workload $w > gpurun_out/r2_b20_$w.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_b20_$w.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$w', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],3))"; done
FDTD_ROM_BATCH=8 $B > gpurun_out/r2_b20_b8.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_b20_b8.log').read().strip().splitlines()[-1]); r=d['roofline']; print('B8', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],3))"
python tools/slab_overhead.py --out gpurun_out/r02_slab_overhead.json > gpurun_out/r02_slab.log 2>&1; echo slab=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or slabs or cluster" > gpurun_out/r2_t20.log 2>&1; echo t=$?
