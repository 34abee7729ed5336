# Round validation + profiles (run on the GPU box from the repo root: gpurun -- bash tools/gpucmd_validate_and_profile.sh):
# smoke, full GPU suite, default bench, config sweep, launch list, ncu --set full pages (csv only: .ncu-rep stay in /tmp)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 3000 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
timeout 600 python bench.py --config 2 --eta 1e2 --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg2.log 2>&1
timeout 600 python bench.py --config 3 --ny 256 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-share > gpurun_out/bench_strip.log 2>&1
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg4.log 2>&1
timeout 900 python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_cfg5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_matvec|k_cell_restrict|k_l1_solve|k_restrict_reduce|k_symv|k_combine|k_trsv" -s 700 -c 140 --csv --log-file gpurun_out/r02b_launches_iter_config3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l1_solve_ring -s 30 -c 1 -f -o /tmp/r02b_l1_ring_cfg3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ncu_l1.log 2>&1
ncu -i /tmp/r02b_l1_ring_cfg3.ncu-rep --page raw --csv > gpurun_out/r02b_l1_ring_cfg3_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"k_symv_bulk|k_symv_reduce|k_combine2|k_matvec|k_cell_restrict" -s 120 -c 5 -f -o /tmp/r02b_small_cfg3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ncu_small.log 2>&1
ncu -i /tmp/r02b_small_cfg3.ncu-rep --page raw --csv > gpurun_out/r02b_small_cfg3_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l1_solve_twist -s 20 -c 1 -f -o /tmp/r02b_twist_cfg2 python bench.py --config 2 --eta 1e2 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-share --e2e-steps 0 > gpurun_out/ncu_twist.log 2>&1
ncu -i /tmp/r02b_twist_cfg2.ncu-rep --page raw --csv > gpurun_out/r02b_l1_twist_cfg2_raw.csv 2>/dev/null
ncu -i /tmp/r02b_twist_cfg2.ncu-rep --page source --csv > gpurun_out/r02b_l1_twist_cfg2_source.csv 2>/dev/null
ls -la gpurun_out > gpurun_out/ls.log
