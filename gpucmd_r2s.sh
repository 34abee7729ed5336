mkdir -p gpurun_out
for m in 4 5 6; do
MSGPU_LIB=build/var/libmsgpu_cr$m.so timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/crm${m}_cfg3.log 2>&1
done
MSGPU_LIB=build/var/libmsgpu_cr4.so MS_RESTRICT_NU=1 timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/crm_nu1_cfg3.log 2>&1
