mkdir -p gpurun_out
L=build/var/libmsgpu_ch32.so
for n in 2 3; do
MSGPU_LIB=$L MS_L1_NST=$n timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ch32_nst${n}_cfg2.log 2>&1
done
MSGPU_LIB=$L MS_L1_NST=2 timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ch32_nst2_strip.log 2>&1
MSGPU_LIB=build/var/libmsgpu_ch16.so MS_L1_NST=2 MS_L1_TWIST=0 timeout 600 python bench.py --config 3 --ny 512 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ch16_plain_w4.log 2>&1
MS_L1_TWIST=0 timeout 600 python bench.py --config 3 --ny 512 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ch08_plain_w4.log 2>&1
