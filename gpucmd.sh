mkdir -p gpurun_out; O=gpurun_out/ab12.log; : > $O
for v in prev t64 t128 prev t64 t128; do
  export MSGPU_LIB=$PWD/build/libmsgpu_$v.so
  echo "== bench $v" >> $O
  timeout 300 python bench.py --maxit 400 --e2e-steps 0 --no-cpu-baseline --no-parity --steps 3 --warmup 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); k=d['roofline']['kernel_ms_per_launch']; print('%.4g'%d['value'], '%.4f'%(d['ms_per_step']/d['config']['iterations_per_step']), {a:round(b*1000,1) for a,b in k.items()}, d['clocks']['sm_mhz'])
" >> $O
done
