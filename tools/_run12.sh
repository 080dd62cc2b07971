timeout 60 python tools/_diag_hang.py 1 cfg3crop > gpurun_out/diag_normal.log 2>&1; echo normal=$?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests12.log 2>&1; echo tests=$?
timeout 1200 python tools/checked_run.py > gpurun_out/r2_checked12.log 2>&1; echo checked=$?
