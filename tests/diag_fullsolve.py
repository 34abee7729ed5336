"""Diagnostic (not collected): config 3 solved to rtol 1e-8 (time to solution)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2006_13387_b200 import configs, pcg_solve
from paper_2006_13387_b200.solve import setup_spec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
tag = sys.argv[2] if len(sys.argv) > 2 else "EH+Rot"
spec = configs.config3(seed=0, n=n)
t0 = time.perf_counter()
mesh, op, pre = setup_spec(spec, tag)
torch.cuda.synchronize()
tb = time.perf_counter() - t0
b = spec.rhs()
x, rep = pcg_solve(op, b, pre, tol=1e-8, maxit=100000, record=False)
tr = np.linalg.norm(b - op @ x) / np.linalg.norm(b)
print(f"n={n} {tag} build {tb:.2f} s, iterations {rep.iterations}, converged {rep.converged}, "
      f"solve {rep.timings['solve']:.2f} s, true residual {tr:.3e}")
