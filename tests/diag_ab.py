"""Diagnostic (not collected): sign/size of the PCG alpha/beta histories (config 3)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2006_13387_b200 import configs, pcg_solve
from paper_2006_13387_b200.solve import setup_spec

for n in [int(a) for a in sys.argv[1:]]:
    spec = configs.config3(seed=0, n=n)
    mesh, op, pre = setup_spec(spec)
    x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-10, maxit=2000)
    a, b = np.array(rep.alphas), np.array(rep.betas)
    print(n, "iters", rep.iterations, "min alpha", a.min(), "min beta", b.min(), "n neg beta", int((b < 0).sum()),
          "cond", rep.cond_estimate, "res", rep.residuals[-1])
