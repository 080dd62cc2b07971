timeout 60 python tools/_diag_hang.py 1 cfg3crop > gpurun_out/diag_normal.log 2>&1; echo normal=$?
FDTD_LIB=paper_1609_07114_b200/libfdtdrom_check.so timeout 60 python tools/_diag_hang.py 1 cfg3crop > gpurun_out/diag_check.log 2>&1; echo check=$?
FDTD_LIB=paper_1609_07114_b200/libfdtdrom_check.so timeout 60 python tools/_diag_hang.py 4 cfg3crop > gpurun_out/diag_check4.log 2>&1; echo check4=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "cluster or dense or k_step" > gpurun_out/r2_gputests11a.log 2>&1; echo clusters=$?
