"""Diagnostic (not collected): two ranks on one GPU (gloo host callbacks),
hash of x and the residual history, for bit-identity A/B of the multi-rank
iteration between library builds (MSGPU_LIB=...).  usage: python tests/diag_dist_bitid.py"""
import hashlib
import os
import socket
import sys
from pathlib import Path

import multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def worker(rank, world, port, q, tag):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import numpy as np
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2006_13387_b200 import configs, dist as D, pcg_solve
    from paper_2006_13387_b200.solve import setup_spec

    D.init_host_callbacks(0)
    spec = configs.config1(seed=0, n=64, H=16, delta=2)
    mesh, op, pre = setup_spec(spec, tag)
    x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=5000)
    h = hashlib.sha1(np.ascontiguousarray(x).tobytes() + np.asarray(rep.residuals).tobytes()).hexdigest()[:16]
    q.put((rank, rep.iterations, h))
    dist.destroy_process_group()


if __name__ == "__main__":
    for tag in ("EH+Rot", "HH+Rot"):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=worker, args=(r, 2, port, q, tag)) for r in range(2)]
        for p in ps:
            p.start()
        out = sorted(q.get(timeout=600) for _ in range(2))
        for p in ps:
            p.join(timeout=120)
        print(tag, out, flush=True)
