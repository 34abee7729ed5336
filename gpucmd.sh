timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --maxit 100 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4.log 2>&1; echo exit=$? >> gpurun_out/bench_c4.log
timeout 600 python bench.py --steps 1 --warmup 1 --maxit 100 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
