B="python bench.py --steps 80 --warmup 8 --no-cpu --no-e2e"
for v in head a64tpw3 a64tpw1 a64tpw2 a64unr8 head; do FDTD_LIB=variants/$v.so $B > gpurun_out/r2_b9_$v.log 2>&1; echo $v=$?; done
for v in head a64tpw3 a64tpw1; do FDTD_LIB=variants/$v.so $B --workload cfg5 > gpurun_out/r2_b9_${v}_cfg5.log 2>&1; echo $v=$?; done
