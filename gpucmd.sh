mkdir -p gpurun_out
( echo "== prev"; MSGPU_LIB=$PWD/build/libmsgpu_prev.so timeout 600 python tests/diag_dist_bitid.py; echo "== new"; timeout 600 python tests/diag_dist_bitid.py ) > gpurun_out/dist_bitid.log 2>&1
