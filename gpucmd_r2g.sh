# unit-diagonal level-1 factors: correctness + A/B timing (config 2, 8-GPU strip, config 3)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "unit_diagonal or twisted or one_copy" > gpurun_out/pytest_unit.log 2>&1; echo exit=$? >> gpurun_out/pytest_unit.log
for u in 0 1; do
MS_L1_UNIT=$u timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/unit${u}_cfg2.log 2>&1
MS_L1_UNIT=$u MS_L1_TWIST=0 timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/unit${u}_cfg2_plain.log 2>&1
MS_L1_UNIT=$u timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/unit${u}_strip.log 2>&1
MS_L1_UNIT=$u timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/unit${u}_cfg3.log 2>&1
done
