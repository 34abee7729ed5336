mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2006_13387_b200 import configs, pcg_solve
from paper_2006_13387_b200.solve import setup_spec
import scipy.sparse as sp
spec = configs.config1(seed=0, n=32, H=8, delta=2)
for tag in ("EH+Rot", "HH+Rot"):
    mesh, op, pre = setup_spec(spec, tag)
    x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=300)
    print(tag, rep.iterations, rep.converged)
A = sp.diags(np.linspace(1, 9, 40)).tocsr()
x, rep = pcg_solve(A, np.ones(40), lambda r: r / A.diagonal(), tol=1e-10)
print("generic", rep.iterations)
PY
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 3 python /tmp/san_case.py > gpurun_out/san_memcheck.log 2>&1; echo exit=$? >> gpurun_out/san_memcheck.log
MS_L1_TWIST=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 3 python /tmp/san_case.py > gpurun_out/san_memcheck_twist.log 2>&1; echo exit=$? >> gpurun_out/san_memcheck_twist.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 3 python /tmp/san_case.py > gpurun_out/san_racecheck.log 2>&1; echo exit=$? >> gpurun_out/san_racecheck.log
