mkdir -p gpurun_out
for w in cfg2 cfg3; do for ch in 32 64 128 256; do for wp in 4 8; do
 r=$(FDTD_CHUNK=$ch FDTD_WARPS=$wp python bench.py --workload $w --no-cpu --no-e2e --steps 400 --warmup 20 2>/dev/null | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.1f G sweep %.4f post %.4f' % (d['value']/1e9, d['roofline']['sweep_ms_per_launch'], d['roofline']['post_ms_per_launch']))")
 echo "$w chunk=$ch warps=$wp $r"
done; done; done
for ch in 256 512 1024; do for wp in 4 8; do
 r=$(FDTD_CHUNK=$ch FDTD_WARPS=$wp python bench.py --workload cfg4 --no-cpu --no-e2e --steps 100 --warmup 8 2>/dev/null | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.1f G sweep %.4f post %.4f' % (d['value']/1e9, d['roofline']['sweep_ms_per_launch'], d['roofline']['post_ms_per_launch']))")
 echo "cfg4 chunk=$ch warps=$wp $r"
done; done
