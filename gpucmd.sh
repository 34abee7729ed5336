CMD="python bench.py --steps 1 --warmup 1 --maxit 24 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_matvec|k_cell_restrict|k_l1_solve|k_restrict_reduce|k_symv|k_combine" -c 120 --csv --log-file gpurun_out/launches_r01b.csv $CMD > gpurun_out/ncu_a.log 2>&1
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_l1_solve|k_cell_restrict|k_combine|k_matvec|k_symv_tiles" -s 10 -c 5 -o gpurun_out/prof_r01b $CMD > gpurun_out/ncu_b.log 2>&1
CMD2="python bench.py --local-solver dense --steps 1 --warmup 1 --maxit 8 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD2 > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"k_l1_dense_apply" -s 2 -c 1 -o gpurun_out/prof_dense $CMD2 > gpurun_out/ncu_c.log 2>&1
echo done > gpurun_out/ncu_done.log
