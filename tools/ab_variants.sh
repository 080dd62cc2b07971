#!/bin/bash
# A/B of library variants (variants/<name>.so) on bench workloads, interleaved reps.
# usage: bash tools/ab_variants.sh "<variants>" "<workloads>" <reps> [steps]
V=$1; W=$2; R=${3:-3}; ST=${4:-200}
for rep in $(seq $R); do for w in $W; do for v in $V; do
  r=$(FDTD_LIB=variants/$v.so python bench.py --workload $w --no-cpu --no-e2e --steps $ST --warmup 10 2>/dev/null | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.1f G sweep %.4f post %.4f clk %s %s' % (d['value']/1e9, d['roofline']['sweep_ms_per_launch'], d['roofline']['post_ms_per_launch'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons')))")
  echo "rep=$rep $w $v $r"
done; done; done
