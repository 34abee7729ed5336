mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bitwise_identical or plain_cg or operator" > gpurun_out/pytest_mv.log 2>&1; echo exit=$? >> gpurun_out/pytest_mv.log
for m in 0 1; do
MS_MATVEC=$m timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/mv${m}_cfg3.log 2>&1
done
MS_MATVEC=1 timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/mv1_cfg2.log 2>&1
