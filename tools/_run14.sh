bash tools/_run13.sh
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests14.log 2>&1; echo tests=$?
