python -m pytest tests -m gpu -q -x -k "big_rom" > gpurun_out/r2_gputests8a.log 2>&1; echo big=$?
python tests/replays/cavity_replay.py --steps 20000 --check 500 --out gpurun_out/cavity_big.json > gpurun_out/cavity_big.log 2>&1; echo cav=$?
FDTD_BIG_Q=0 python tests/replays/cavity_replay.py --steps 4000 --check 200 --out gpurun_out/cavity_batch.json > gpurun_out/cavity_batch.log 2>&1; echo cavb=$?
python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests8.log 2>&1; echo tests=$?
B="python bench.py --steps 80 --warmup 8 --no-cpu --no-e2e"
for v in head v0; do FDTD_LIB=variants/$v.so $B > gpurun_out/r2_b8_$v.log 2>&1; echo $v=$?; done
$B > gpurun_out/r2_b8_cur.log 2>&1; echo cur=$?
