timeout 600 python tests/diag_components.py 2048 > gpurun_out/comp.log 2>&1
