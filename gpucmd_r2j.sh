mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_krylov_seams.py -m gpu -q > gpurun_out/pytest_seams.log 2>&1; echo exit=$? >> gpurun_out/pytest_seams.log
MS_L1_UNIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "unit_diagonal or twisted or one_copy" > gpurun_out/pytest_unit.log 2>&1; echo exit=$? >> gpurun_out/pytest_unit.log
for u in 0 1; do
MS_L1_UNIT=$u timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/rt_unit${u}_cfg2.log 2>&1
MS_L1_UNIT=$u timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/rt_unit${u}_strip.log 2>&1
MS_L1_UNIT=$u timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/rt_unit${u}_cfg3.log 2>&1
done
MS_L1_UNIT=1 MS_L1_NST=6 timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/rt_unit1_cfg2_nst6.log 2>&1
MS_L1_UNIT=1 MS_L1_NST=2 timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/rt_unit1_cfg2_nst2.log 2>&1
