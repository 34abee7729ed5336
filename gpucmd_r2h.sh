# duck-typed pcg_solve seams + level-1 ring depth variants (compile-time MS_TMA_NST) in the latency-bound regimes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_krylov_seams.py tests/test_gpu_behaviour.py -m gpu -q -x > gpurun_out/pytest_seams.log 2>&1; echo exit=$? >> gpurun_out/pytest_seams.log
for n in 3 4 6; do
L=build/var/libmsgpu_nst$n.so
MSGPU_LIB=$L MS_L1_UNIT=1 timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/nst${n}_cfg2.log 2>&1
MSGPU_LIB=$L MS_L1_UNIT=1 timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/nst${n}_strip.log 2>&1
MSGPU_LIB=$L MS_L1_UNIT=1 MS_L1_TWIST=0 timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/nst${n}_strip_plain.log 2>&1
done
