set -u
run() {
  local v=$1; shift
  env "$@" python bench.py --steps 40 --warmup 4 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['value']/1e9,1), round(r['sweep_ms_per_launch'],3), round(r['post_ms_per_launch'],3))"
}
for ch in 128 256 512 1024; do for w in 2 4; do run ch${ch}_w$w FDTD_CHUNK=$ch FDTD_WARPS=$w; done; done
