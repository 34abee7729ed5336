mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
for tw in 0 1; do MS_L1_TWIST=$tw timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg2_tw$tw.log 2>&1; echo exit=$? >> gpurun_out/bench_cfg2_tw$tw.log; done
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg3.log 2>&1; echo exit=$? >> gpurun_out/bench_cfg3.log
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg5.log 2>&1; echo exit=$? >> gpurun_out/bench_cfg5.log
