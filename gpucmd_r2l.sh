mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_behaviour.py tests/test_dist.py -m gpu -q > gpurun_out/pytest_k.log 2>&1; echo exit=$? >> gpurun_out/pytest_k.log
MS_COMBINE=0 timeout 600 python tests/diag_components.py > gpurun_out/comp_cb0.log 2>&1
MS_COMBINE=1 timeout 600 python tests/diag_components.py > gpurun_out/comp_cb1.log 2>&1
