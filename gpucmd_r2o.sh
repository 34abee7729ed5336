mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_dist.py tests/test_gpu_behaviour.py -m gpu -q > gpurun_out/pytest_k.log 2>&1; echo exit=$? >> gpurun_out/pytest_k.log
timeout 1500 python -m pytest tests/test_gpu_bounds.py -m gpu -q -k "plain or twisted or no-table or strip or mbb or multi_rank" > gpurun_out/pytest_b.log 2>&1; echo exit=$? >> gpurun_out/pytest_b.log
for c in 0 1; do
MS_CHI_DEDUP=$c timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/chi${c}_cfg3.log 2>&1
done
MS_CHI_DEDUP=1 timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/chi1_cfg4.log 2>&1
