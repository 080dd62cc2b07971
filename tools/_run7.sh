B="python bench.py --steps 80 --warmup 8 --no-cpu --no-e2e"
for v in v0 schur4 nopf tpw1 tpw2; do
  FDTD_LIB=variants/$v.so $B > gpurun_out/r2_b7_$v.log 2>&1; echo $v=$?
done
for v in v0 tpw1; do
  FDTD_LIB=variants/$v.so $B --workload cfg5 > gpurun_out/r2_b7_${v}_cfg5.log 2>&1; echo $v=$?
done
