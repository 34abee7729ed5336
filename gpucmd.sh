mkdir -p gpurun_out; O=gpurun_out/ab10.log; : > $O
for v in prev new; do
  case $v in prev) export MSGPU_LIB=$PWD/build/libmsgpu_prev.so;; new) unset MSGPU_LIB;; esac
  echo "== $v" >> $O
  timeout 600 python tests/diag_build.py 2>&1 | grep -v Warn >> $O
  timeout 900 python bench.py --config 5 --steps 20 --no-cpu-baseline 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); c=d['config']; print('config5', '%.4g'%d['value'], 'ms/step %.1f'%d['ms_per_step'], 'build/step %.3f'%c['build_s_per_step'], 'solve/step %.3f'%c['solve_s_per_step'], sum(c['iterations']))" >> $O
done
unset MSGPU_LIB
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
