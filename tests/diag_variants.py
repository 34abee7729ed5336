"""Diagnostic (not collected): time-to-solution of the GPU variants on
config 3 at a few sizes.  Run on the GPU box:
    python tests/diag_variants.py 256 512 1024
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2006_13387_b200 import configs, pcg_solve
from paper_2006_13387_b200.solve import setup_spec

for n in [int(a) for a in sys.argv[1:]] or [256]:
    spec = configs.config3(seed=0, n=n, H=32 if n >= 512 else 16)
    for tag in ("EH+Rot", "HH+Rot", "EH+Rot;Rand"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mesh, op, pre = setup_spec(spec, tag)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        b = torch.tensor(spec.rhs(), device="cuda")
        pcg_solve(op, b, pre, tol=1e-8, maxit=20, record=False)
        _, rep = pcg_solve(op, b, pre, tol=1e-8, maxit=40000, record=False)
        print(json.dumps({"n": n, "variant": tag, "build_s": tb, "coarse_dim": pre.coarse_dim,
                          "iters": rep.iterations, "converged": rep.converged,
                          "solve_s": rep.timings["solve"],
                          "ms_per_iter": 1e3 * rep.timings["solve"] / max(rep.iterations, 1)}), flush=True)
        del pre, op
