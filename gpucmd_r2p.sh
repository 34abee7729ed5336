mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_combine2|k_cell_restrict|k_matvec" -s 60 -c 3 -o /tmp/small python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ncu_small2.log 2>&1
ncu -i /tmp/small.ncu-rep --page source --csv > gpurun_out/small_source.csv 2>/dev/null
ncu -i /tmp/small.ncu-rep --page raw --csv > gpurun_out/small_raw.csv 2>/dev/null
