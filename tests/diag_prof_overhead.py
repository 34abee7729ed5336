"""Diagnostic (not collected): per-iteration time with and without the
per-kernel profiling events (config 3)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2006_13387_b200 import _lib, configs, pcg_solve
from paper_2006_13387_b200.solve import setup_spec

spec = configs.config3(seed=0)
mesh, op, pre = setup_spec(spec)
b = torch.tensor(spec.rhs(), device="cuda")
lib = _lib.load()
for prof in (0, 1, 0, 1):
    lib.ms_ctx_set_profiling(op._ctx.handle, prof)
    pcg_solve(op, b, pre, tol=1e-8, maxit=200, record=False)
    ts = []
    for _ in range(3):
        _, rep = pcg_solve(op, b, pre, tol=1e-8, maxit=400, record=False)
        ts.append(rep.timings["solve"] / rep.iterations * 1e3)
    print("profiling", prof, "ms/iter", [round(t, 4) for t in ts])
