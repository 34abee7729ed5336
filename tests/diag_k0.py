"""Diagnostic (not collected): conditioning of K0 for config 3 and the
summation-order sensitivity of the explicit-inverse coarse solve."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2006_13387_b200 import configs, pcg_solve
from paper_2006_13387_b200.solve import setup_spec

for n in [int(a) for a in sys.argv[1:]]:
    spec = configs.config3(seed=0, n=n)
    mesh, op, pre = setup_spec(spec)
    K0 = pre.coarse_matrix()
    w = np.linalg.eigvalsh(K0)
    X = np.linalg.inv(K0)
    X = 0.5 * (X + X.T)
    # residual after a few PCG iterations, restricted by the GPU coarse apply path
    rng = np.random.default_rng(0)
    for its in (0, 5, 20):
        if its == 0:
            r = rng.standard_normal(op.n_free)
        else:
            x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-14, maxit=its, record=False)
            r = spec.rhs() - op @ x
        # f0 = R0 r through the GPU: apply_coarse gives R0^T K0^-1 R0 r; use K0 only for cond stats
        f0 = K0 @ rng.standard_normal(K0.shape[0]) if its == 0 else None
        if f0 is None:
            continue
        h = K0.shape[0] // 2
        y_full = X @ f0
        y_split = X[:, :h] @ f0[:h] + X[:, h:] @ f0[h:]
        print(n, "N_c", K0.shape[0], "eig min/max", w[0], w[-1], "cond", w[-1] / w[0],
              "split rel diff", np.linalg.norm(y_full - y_split) / np.linalg.norm(y_full))
