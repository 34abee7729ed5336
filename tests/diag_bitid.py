"""Diagnostic (not collected): hash of a PCG solve's x and residual history, for
bit-identity A/B between kernel variants selected by env knobs.
usage: python tests/diag_bitid.py <config:3|1|5> <n> <maxit>"""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2006_13387_b200 import configs, pcg_solve
from paper_2006_13387_b200.solve import setup_spec

cfg, n, maxit = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
spec = {1: lambda: configs.config1(seed=0, n=n), 3: lambda: configs.config3(seed=0, n=n),
        5: lambda: configs.config5(seed=0, n=n)}[cfg]()
mesh, op, pre = setup_spec(spec)
x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=maxit)
h = hashlib.sha1(np.ascontiguousarray(x).tobytes() + np.asarray(rep.residuals).tobytes()).hexdigest()[:16]
print(f"cfg{cfg} n={n} iters={rep.iterations} res={rep.residuals[-1]:.6e} hash={h}")
