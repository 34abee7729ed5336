mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_dist.py tests/test_gpu_behaviour.py -q > gpurun_out/pytest_dist.log 2>&1; echo exit=$? >> gpurun_out/pytest_dist.log
