#!/bin/bash
# Fix-up launch shape experiments (FDTD_POST_THREADS x FDTD_ROM_BATCH) on the bench workloads and the
# 8-slab emulation.  usage: bash tools/fixup_knobs.sh
run() {  # threads batch workload
  local B=""; [ "$2" != 0 ] && B="FDTD_ROM_BATCH=$2"
  r=$(env FDTD_POST_THREADS=$1 $B python bench.py --workload $3 --no-cpu --no-e2e --steps 120 --warmup 10 2>/dev/null | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.1f G sweep %.4f post %.4f' % (d['value']/1e9, d['roofline']['sweep_ms_per_launch'], d['roofline']['post_ms_per_launch']))")
  echo "$3 threads=$1 batch=$2 $r"
}
for tb in "512 0" "256 0" "256 4" "256 3" "256 2" "384 5" "128 2" "512 4"; do run $tb cfg3; done
for tb in "512 0" "256 0" "256 4" "384 5"; do run $tb cfg4; done
for tb in "512 0" "256 0" "256 2" "256 3" "512 2"; do
  set -- $tb
  B=""; [ "$2" != 0 ] && B="FDTD_ROM_BATCH=$2"
  env FDTD_POST_THREADS=$1 $B python tools/slab_overhead.py --slabs 1,8 --steps 48 --out gpurun_out/slab_t$1_b$2.json > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/slab_t$1_b$2.json'));print('slabs threads=$1 batch=$2', [(r['slabs'], round(r['cell_updates_per_s']/1e9,1), round(r['per_pass_sum_over_slabs_ms']['fixup'],3)) for r in d['rows']])"
done
