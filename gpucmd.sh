mkdir -p gpurun_out
( timeout 900 python tests/diag_fullsolve.py 2048 EH+Rot; timeout 900 python tests/diag_fullsolve.py 2048 HH+Rot ) > gpurun_out/fullsolve.log 2>&1
