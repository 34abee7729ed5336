# round-2 validation: smoke, parity suite with the measured bands, level-1 profile at config 2
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -m gpu -q -x -k "not bench_multi" > gpurun_out/pytest_parity.log 2>&1; echo exit=$? >> gpurun_out/pytest_parity.log
timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg2.log 2>&1; echo exit=$? >> gpurun_out/bench_cfg2.log
timeout 600 ncu --set full --import-source on -k regex:k_l1_solve_ring -c 1 -o gpurun_out/l1_cfg2 python bench.py --config 2 --eta 1e2 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --maxit 16 --e2e-steps 1 > gpurun_out/ncu_l1_cfg2.log 2>&1; echo exit=$? >> gpurun_out/ncu_l1_cfg2.log
