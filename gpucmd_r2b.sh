mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "twisted or level1 or dense_spd or coarse_apply or config1" > gpurun_out/pytest_twist.log 2>&1; echo exit=$? >> gpurun_out/pytest_twist.log
for tw in 0 1; do MS_L1_TWIST=$tw timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg2_tw$tw.log 2>&1; echo exit=$? >> gpurun_out/bench_cfg2_tw$tw.log; done
for tw in 0 1; do MS_L1_TWIST=$tw timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --maxit 200 > gpurun_out/bench_cfg3_tw$tw.log 2>&1; echo exit=$? >> gpurun_out/bench_cfg3_tw$tw.log; done
