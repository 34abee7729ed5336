timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --local-solver dense --steps 1 --warmup 1 --maxit 50 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_dense.log 2>&1; echo exit=$? >> gpurun_out/bench_dense.log
