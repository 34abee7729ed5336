mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_dist.py -m gpu -q > gpurun_out/pytest_k.log 2>&1; echo exit=$? >> gpurun_out/pytest_k.log
MS_SYMV=0 timeout 600 python tests/diag_components.py > gpurun_out/comp_sy0.log 2>&1
MS_SYMV=1 timeout 600 python tests/diag_components.py > gpurun_out/comp_sy1.log 2>&1
for c in 0 1; do
MS_SYMV=$c timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/sy${c}_cfg3.log 2>&1
done
MS_SYMV=1 timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/sy1_cfg4.log 2>&1
