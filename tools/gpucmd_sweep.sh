# Bench sweep over the BASELINE configs on the final build (run from the repo root on the GPU box).
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share"
timeout 600 $B --config 1 --steps 5 > gpurun_out/sweep_cfg1.log 2>&1
for e in 1e2 1e4 1e6 1e8; do timeout 600 $B --config 2 --eta $e > gpurun_out/sweep_cfg2_$e.log 2>&1; done
timeout 900 $B --config 3 --variant HH+Rot > gpurun_out/sweep_cfg3_hhrot.log 2>&1
timeout 600 $B --config 3 --ny 256 > gpurun_out/sweep_strip.log 2>&1
timeout 900 $B --config 4 > gpurun_out/sweep_cfg4.log 2>&1
timeout 900 python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/sweep_cfg5.log 2>&1
timeout 900 python tests/diag_fullsolve.py 2048 EH+Rot > gpurun_out/fullsolve_ehrot.log 2>&1
cat gpurun_out/sweep_*.log | grep '^{' > gpurun_out/r02c_bench_sweep.jsonl
