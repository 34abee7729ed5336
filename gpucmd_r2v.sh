mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_dist.py -m gpu -q > gpurun_out/pytest_k.log 2>&1; echo exit=$? >> gpurun_out/pytest_k.log
timeout 1500 python -m pytest tests/test_gpu_bounds.py -m gpu -q > gpurun_out/pytest_b.log 2>&1; echo exit=$? >> gpurun_out/pytest_b.log
timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/w_cfg2.log 2>&1
timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/w_strip.log 2>&1
timeout 600 python bench.py --config 3 --ny 512 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/w_w4.log 2>&1
timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > gpurun_out/w_cfg3.log 2>&1
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/w_cfg1.log 2>&1
