mkdir -p gpurun_out
L=build/var/libmsgpu_ch16.so
for n in 2 3 4; do
MSGPU_LIB=$L MS_L1_NST=$n timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ch16_nst${n}_cfg2.log 2>&1
done
MSGPU_LIB=$L MS_L1_NST=2 timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ch16_nst2_strip.log 2>&1
MSGPU_LIB=$L timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ch16_auto_strip.log 2>&1
