for q in 600 64; do for prec in 64 32; do
CUDA_LAUNCH_BLOCKING=1 FDTD_LIB=paper_1609_07114_b200/libfdtdrom_check.so timeout 120 python tools/_diag_big.py $prec $q > gpurun_out/diag_big_${prec}_$q.log 2>&1; echo $prec $q $?
done; done
