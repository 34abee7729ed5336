# runtime ring depth (pick_nst) + unit factors: tests, A/B benches, ncu source capture of the twisted kernel at config 2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_krylov_seams.py -m gpu -q > gpurun_out/pytest_seams.log 2>&1; echo exit=$? >> gpurun_out/pytest_seams.log
MS_L1_UNIT=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/pytest_parity_unit1.log 2>&1; echo exit=$? >> gpurun_out/pytest_parity_unit1.log
for u in 0 1; do
MS_L1_UNIT=$u timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/rt_unit${u}_cfg2.log 2>&1
MS_L1_UNIT=$u timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/rt_unit${u}_strip.log 2>&1
MS_L1_UNIT=$u timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/rt_unit${u}_cfg3.log 2>&1
done
MS_L1_UNIT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l1_solve_twist -s 20 -c 1 -o gpurun_out/r02_twist_cfg2 python bench.py --config 2 --eta 1e2 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ncu_twist.log 2>&1
