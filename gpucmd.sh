timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 600 python tests/diag_components.py 2048 > gpurun_out/comp.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
