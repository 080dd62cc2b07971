timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_t21.log 2>&1; echo t=$?
FDTD_POST_THREADS=256 FDTD_ROM_BATCH=2 python tools/slab_overhead.py --slabs 8 --out gpurun_out/r02_slab8_b2t256.json > gpurun_out/r02_slab8a.log 2>&1; echo a=$?
FDTD_ROM_BATCH=2 python tools/slab_overhead.py --slabs 8 --out gpurun_out/r02_slab8_b2.json > gpurun_out/r02_slab8b.log 2>&1; echo b=$?
FDTD_POST_THREADS=256 FDTD_ROM_BATCH=4 python tools/slab_overhead.py --slabs 8 --out gpurun_out/r02_slab8_b4t256.json > gpurun_out/r02_slab8c.log 2>&1; echo c=$?
