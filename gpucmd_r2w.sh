mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "unit_diagonal or twisted or one_copy or bitwise" > gpurun_out/pytest_k.log 2>&1; echo exit=$? >> gpurun_out/pytest_k.log
timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/p_cfg2.log 2>&1
MS_L1_CH=16 timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/p_strip16.log 2>&1
MS_L1_CH=16 MS_L1_TWIST=0 timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/p_strip16_plain.log 2>&1
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/p_cfg1.log 2>&1
