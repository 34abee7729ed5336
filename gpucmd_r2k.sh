mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_behaviour.py -m gpu -q -x > gpurun_out/pytest_k.log 2>&1; echo exit=$? >> gpurun_out/pytest_k.log
for c in 0 1 2; do
MS_COMBINE=$c timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/cb${c}_cfg3.log 2>&1
done
MS_COMBINE=1 timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/cb1_cfg4.log 2>&1
