mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/pytest_parity.log 2>&1; echo exit=$? >> gpurun_out/pytest_parity.log
timeout 900 python tests/diag_parity_variants.py > gpurun_out/diag_variants.log 2>&1
for c in 1 2; do MS_L1_COPIES=$c timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/ab_cfg3_copies$c.log 2>&1; done
timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg2.log 2>&1
MS_L1_TWIST=0 timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg2_tw0.log 2>&1
timeout 600 python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg5.log 2>&1
