mkdir -p gpurun_out
for rep in 1 2; do
for lib in new lb64; do
  if [ $lib = lb64 ]; then export MSGPU_LIB=$PWD/build/var/libmsgpu_lb64.so; else unset MSGPU_LIB; fi
  timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/ab_cfg3_${lib}_$rep.log 2>&1
done; done
unset MSGPU_LIB
for tw in 0 1; do MS_L1_TWIST=$tw timeout 600 python bench.py --config 5 --steps 6 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/ab_cfg5_tw$tw.log 2>&1; done
