"""Diagnostic (not collected): two ranks on one GPU (gloo host callbacks)
against the one-rank path on config 3 at a given size.
    python tests/diag_dist.py 256 [maxit]"""
import os
import sys
from pathlib import Path

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from test_dist import _free_port, _init  # noqa: E402


def worker(rank, world, port, q, n, maxit):
    sys.path.insert(0, str(ROOT))
    _init(rank, world, port)
    try:
        from paper_2006_13387_b200 import configs, dist as D, pcg_solve
        from paper_2006_13387_b200.solve import setup_spec

        D.init_host_callbacks(0)
        spec = configs.config3(seed=0, n=n)
        mesh, op, pre = setup_spec(spec)
        r = np.random.default_rng(1).standard_normal(op.n_free)
        z = pre.apply(r)
        zc = pre.apply_coarse(r)
        av = op @ r
        x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=maxit, record=False)
        # the preconditioner on PCG-like residuals (r_k of the one-rank run, from the parent)
        rk = np.load(os.environ["DIAG_RK"])
        zk = [pre.apply(v) for v in rk]
        zck = [pre.apply_coarse(v) for v in rk]
        q.put((rank, z, zc, x, rep.iterations, pre.coarse_dim, av, zk, zck))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    from paper_2006_13387_b200 import configs, pcg_solve
    from paper_2006_13387_b200.solve import setup_spec

    spec = configs.config3(seed=0, n=n)
    mesh, op, pre = setup_spec(spec)
    rks, zks, zcks = [], [], []
    for its in (5, 20, 100, 400):
        xk, _ = pcg_solve(op, spec.rhs(), pre, tol=1e-14, maxit=its, record=False)
        v = spec.rhs() - op @ xk
        rks.append(v)
        zks.append(pre.apply(v))
        zcks.append(pre.apply_coarse(v))
    os.environ["DIAG_RK"] = "/tmp/diag_rk.npy"
    np.save("/tmp/diag_rk.npy", np.array(rks))
    del pre, op
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q, n, maxit)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((v[0], v[1:]) for v in (q.get(timeout=1200) for _ in range(2)))
    for p in procs:
        p.join()
    mesh, op, pre = setup_spec(spec)
    r = np.random.default_rng(1).standard_normal(op.n_free)
    z1, zc1 = pre.apply(r), pre.apply_coarse(r)
    x1, rep1 = pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=maxit, record=False)
    av1 = op @ r
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    for k in (0, 1):
        z, zc, x, it, nc, av, zk, zck = res[k]
        print("rank", k, "N_c", nc, pre.coarse_dim, "z", rel(z, z1), "zc", rel(zc, zc1), "Av", rel(av, av1),
              "x", rel(x, x1), "iters", it, rep1.iterations)
        print("   z on r_k (k=5,20,100,400):", [rel(a, b) for a, b in zip(zk, zks)])
        print("   coarse z on r_k:", [rel(a, b) for a, b in zip(zck, zcks)])
