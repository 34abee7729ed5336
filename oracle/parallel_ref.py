"""The oracle's EH+Rot PCG at a FULL BASELINE size on all host cores -- TEST /
BASELINE INFRASTRUCTURE.

Only ``bench.py --impl reference`` (the CPU reference arm) uses this module;
the CUDA product path never imports it.  It runs the reference's algorithm
(``oracle/mselast_oracle.py``, the restatement pinned to the unmodified
reference) on the same configuration the GPU bench measures, spread over
worker processes so the host's cores are used:

* CSR assembly (assembly.py:185-220) in the main process;
* the neighbourhood heat eigenproblems (spectral.py:63-100) in a fork pool,
  solved by the oracle's ARPACK path (``lowest_eigenpairs_arpack``; dense
  ?sygvx would take ~7 s per 4,225-node pencil) -- then the coarse basis,
  K0 = R0 A R0^T and its Cholesky factor (coarse.py:58-168) in the main
  process (threaded BLAS);
* level 1 (schwarz.py:97-109): every worker owns a contiguous run of the
  delta-blocks (a strip of subdomain rows), factors them with SuperLU and
  solves them into its slice of a shared buffer; the main process then adds
  the local solutions in the reference's subdomain order (z[idx] +=
  solve(r[idx]), schwarz.py:80-81), so the sum is the sequential loop's bit
  for bit;
* the operator ``A @ p`` (krylov.py:114) by row blocks of the same CSR matrix
  (each row's dot product unchanged);
* PCG itself (krylov.py:81-134) in the main process.

Vectors cross processes through anonymous shared memory (mmap, inherited
by fork); commands go over pipes.
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os
import time

import numpy as np
import scipy.sparse.linalg as spla

from . import mselast_oracle as O

_EIG = None


def _shared(n):
    buf = mmap.mmap(-1, max(8, 8 * int(n)))
    return np.frombuffer(buf, dtype=np.float64, count=int(n))


def _eig_task(k):
    mesh, E, omegas, dirichlet = _EIG
    K, M, _ = O.local_heat_problem(mesh, E, omegas[k], dirichlet)
    return O.lowest_eigenpairs_arpack(K, M, min(7, K.n_free))


def _worker(conn, A, rows, l1_specs, offs, p, q, r, ysh):
    """Serve 'mv' (q[rows] = A[rows] p) and 'l1' (the owned subdomains'
    solves into their slices of ysh) until 'quit'."""
    Arow = A[rows[0]:rows[1]]
    solvers = [(idx, o, spla.splu(A[idx][:, idx].tocsc()).solve) for idx, o in zip(l1_specs, offs)]
    conn.send("ready")
    while True:
        cmd = conn.recv()
        if cmd == "mv":
            q[rows[0]:rows[1]] = Arow @ p
        elif cmd == "l1":
            for idx, o, solve in solvers:
                ysh[o:o + idx.size] = solve(r[idx])
        elif cmd == "quit":
            conn.send("bye")
            return
        conn.send("done")


class ParallelReference:
    """EH+Rot two-level preconditioner + operator of one BASELINE spec on
    `procs` processes.  ``matvec(p)`` and ``apply(r)`` have the oracle's
    semantics; ``info`` carries the build split."""

    def __init__(self, spec, procs=None):
        global _EIG
        procs = procs or len(os.sched_getaffinity(0))
        self.procs = procs
        t0 = time.perf_counter()
        prob = O.problem_from_spec(spec)
        self.prob = prob
        mesh, op = prob.mesh, prob.op
        n = op.n_free
        t_asm = time.perf_counter() - t0
        # coarse space: eigensolves in a pool, basis rows / K0 / factor here
        t0 = time.perf_counter()
        part = O.Partition(mesh, mesh.nx // spec.H, mesh.ny // spec.H)
        _EIG = (mesh, prob.E, part.omegas, prob.heat_dirichlet_nodes)
        with mp.get_context("fork").Pool(procs) as pool:
            eig = pool.map(_eig_task, range(len(part.omegas)), chunksize=8)
        _EIG = None
        queue = list(eig)

        def cached(K, M, k):
            lam, V = queue.pop(0)
            return lam[:k], V[:, :k]

        cs = O.heat_rot_coarse_space(op, mesh, part, prob.E, prob.heat_dirichlet_nodes, eig_solver=cached)
        self.coarse = O.CoarseSolver(op, cs.R0)
        t_coarse = time.perf_counter() - t0
        # level 1 + matvec workers, one strip of subdomains / row block each
        t0 = time.perf_counter()
        fidx = op.free_index()
        specs = []
        for rect in O.block_rects(mesh, spec.H, spec.delta):
            nodes = O.rect_nodes(mesh, *O.subdomain_node_rect(mesh, rect, True))
            idx = np.concatenate([fidx[nodes], fidx[nodes + mesh.n_nodes]])
            idx = idx[idx >= 0]
            if idx.size:
                specs.append(idx)
        self.n_subdomains = len(specs)
        self.specs = specs
        self.offs = np.concatenate([[0], np.cumsum([v.size for v in specs])]).astype(np.int64)
        self.p, self.q, self.r = _shared(n), _shared(n), _shared(n)
        self.ysh = _shared(int(self.offs[-1]))
        cut = [round(i * len(specs) / procs) for i in range(procs + 1)]
        rcut = [round(i * n / procs) for i in range(procs + 1)]
        ctx = mp.get_context("fork")
        self.conns, self.procs_ = [], []
        for w in range(procs):
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_worker, args=(b, op.matrix, (rcut[w], rcut[w + 1]), specs[cut[w]:cut[w + 1]],
                                                   self.offs[cut[w]:cut[w + 1]], self.p, self.q, self.r,
                                                   self.ysh), daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs_.append(pr)
        for c in self.conns:
            assert c.recv() == "ready"
        t_l1 = time.perf_counter() - t0
        self.n_free = n
        self.coarse_dim = cs.N_c
        self.info = {"t_assembly": t_asm, "t_coarse": t_coarse, "t_eig": cs.t_eig, "t_level1": t_l1,
                     "coarse_dim": cs.N_c, "mode_counts": cs.modes, "processes": procs}

    def _all(self, cmd):
        for c in self.conns:
            c.send(cmd)
        for c in self.conns:
            assert c.recv() == "done"

    def matvec(self, v):
        self.p[:] = v
        self._all("mv")
        return self.q.copy()

    def apply(self, r):
        """z = sum_i R_i^T K_i^-1 R_i r + R0^T K0^-1 R0 r (schwarz.py:76-84)."""
        self.r[:] = r
        self._all("l1")
        z = np.zeros(self.n_free)
        y, offs = self.ysh, self.offs
        for i, idx in enumerate(self.specs):  # the reference's summation order
            z[idx] += y[offs[i]:offs[i + 1]]
        z += self.coarse.apply(r)
        return z

    def close(self):
        for c in self.conns:
            try:
                c.send("quit")
                c.recv()
            except Exception:
                pass
        for pr in self.procs_:
            pr.join(timeout=10)
