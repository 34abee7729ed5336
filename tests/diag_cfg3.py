"""Diagnostics for the config-3 recipe at reduced sizes (GPU)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_2006_13387_b200 import configs, pcg_solve, build_preconditioner, EigOptions
from paper_2006_13387_b200.solve import setup_spec

for n in [int(a) for a in sys.argv[1:]]:
    spec = configs.config3(seed=0, n=n)
    mesh, op, pre = setup_spec(spec)
    b = spec.rhs()
    rng = np.random.default_rng(0)
    v, w = rng.standard_normal(op.n_free), rng.standard_normal(op.n_free)
    s1, s2 = v @ pre.apply(w), w @ pre.apply(v)
    c1, c2 = v @ pre.apply_coarse(w), w @ pre.apply_coarse(v)
    pos = min(x @ pre.apply(x) for x in (v, w))
    t = time.time()
    x, rep = pcg_solve(op, b, pre, tol=1e-8, maxit=20000)
    tr = np.linalg.norm(b - op @ x) / np.linalg.norm(b)
    out = dict(n=n, N_c=pre.coarse_dim, hist=np.bincount(pre.mode_counts).tolist(), passes=pre.info["max_eig_passes"],
               sym=abs(s1 - s2) / abs(s1), csym=abs(c1 - c2) / abs(c1), pos=pos, iters=rep.iterations,
               conv=rep.converged, rec_res=rep.residuals[-1], true_res=tr, cond=rep.cond_estimate,
               hist_res=[rep.residuals[i] for i in range(0, len(rep.residuals), max(1, len(rep.residuals) // 12))],
               t=time.time() - t)
    print(json.dumps(out), flush=True)
