"""Diagnostic (not collected, CPU): how much the oracle's PCG iteration count
moves when only its coarse solve is switched from cho_solve to the explicit
symmetric K0^-1 that the GPU path applies (config-3 recipe at 128^2, the
reference fixture's inputs).  Measured: 2362 -> 2314."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from oracle import mselast_oracle as O
from paper_2006_13387_b200 import configs

g = dict(np.load(Path(__file__).parent / "golden" / "ref_config3_n128.npz"))
spec = configs.ProblemSpec(
    name="golden", nx=int(g["nx"]), ny=int(g["ny"]), E=g["E"], E_min=float(g["E"].min()), E_max=1.0,
    constrained_dofs=g["constrained_dofs"], heat_dirichlet_nodes=g["heat_dirichlet_nodes"],
    load_full=g["load_full"], H=int(g["H"]), delta=int(g["delta"]), nu=float(g["nu"]))
prob = O.problem_from_spec(spec)
P = O.build_two_level(prob, H=spec.H, delta=spec.delta, level1_mode="blocks")
_, rep = O.pcg(prob.op.matrix, prob.b, P, tol=1e-8, maxit=20000)
C = P.coarse
Kinv = np.linalg.inv(C.K0)
Kinv = 0.5 * (Kinv + Kinv.T)
C.apply = lambda r: C.R0.T @ (Kinv @ (C.R0 @ r))
_, rep2 = O.pcg(prob.op.matrix, prob.b, P, tol=1e-8, maxit=20000)
print(f"reference fixture {int(g['iters'])} (jitter {g['jitter_iters']}); oracle cho_solve {rep.iterations}; "
      f"oracle explicit K0^-1 {rep2.iterations}; cond(K0) {np.linalg.cond(C.K0):.2e}")
