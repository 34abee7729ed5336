mkdir -p gpurun_out; O=gpurun_out/ab13.log; : > $O
for v in prev new prev new; do
  case $v in prev) export MSGPU_LIB=$PWD/build/libmsgpu_prev.so;; new) unset MSGPU_LIB;; esac
  echo "== $v" >> $O
  timeout 300 python tests/diag_bitid.py 5 256 300 >> $O 2>&1
  timeout 600 python tests/diag_build.py 2>&1 | grep -v Warn >> $O
done
