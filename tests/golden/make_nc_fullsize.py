"""Per-neighbourhood mode counts at BASELINE.json's FULL sizes, from the
reference's own eigenproblems (build container only; needs /root/reference).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_nc_fullsize.py config3 config4 config5 config2_1e8

For every interior coarse node of the config the reference's pencil is
assembled by ``spectral.build_local_eigproblem`` (spectral.py:63-90) and its
7 lowest eigenpairs are computed with ARPACK shift-invert (scipy ``eigsh``)
instead of the reference's dense ``?sygvx`` (``solve_local_eig_dense``,
spectral.py:93-100): dense is ~7 s per 4,225-node pencil on one core, i.e.
~8 h for config 3 alone, ARPACK ~0.04 s.  The modes are then selected by the
reference's ``select_modes(rule='gap')`` (spectral.py:161-186).  To pin the
substitution, the reference's dense solver itself is run on the 16
neighbourhoods with the smallest gap margin and on 8 random ones per config,
and its mode counts must equal ARPACK's there (asserted here).

Output ``nc_<case>.npz``: eigenvalues (n_centers x 7), n_sel, margin = min
|log(ratio / 50)| over the gap tests (the north star excepts ratios within
1e-10 of the threshold), N_c of EH+Rot (sum 2 n_sel + 1), and the dense
cross-check (centres, dense eigenvalues, dense n_sel).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parents[1]))

from mselast import assembly, grid, spectral  # noqa: E402

from paper_2006_13387_b200 import configs  # noqa: E402

_STATE = None


def _margin(lam, n_max=6, threshold=50.0):
    win = np.asarray(lam)[: n_max + 1]
    eps = 1e-14 * abs(win[-1]) if win[-1] != 0 else 1e-300
    r = [win[i] / max(win[i - 1], eps) for i in range(1, win.size)]
    return float(np.min(np.abs(np.log(np.maximum(r, 1e-300) / threshold))))


def _problem(c):
    mesh, coeff, part, dirichlet = _STATE
    return spectral.build_local_eigproblem(mesh, coeff, part.neighborhoods[c], "diffusion", dirichlet)


def _arpack(c):
    prob = _problem(c)
    A, B = prob.K.tocsc(), prob.M.tocsc()
    sigma = -1e-10 * A.diagonal().sum() / B.diagonal().sum()
    w, v = spla.eigsh(A, 7, B, sigma=sigma, which="LM")
    order = np.argsort(w)
    sel = spectral.select_modes(spectral.EigSelection(w[order], v[:, order], "diffusion", prob), 6, rule="gap")
    return c, w[order], sel.n_sel


def _dense(c):
    prob = _problem(c)
    res = spectral.solve_local_eig_dense(prob, 7)
    return c, res.eigenvalues, spectral.select_modes(res, 6, rule="gap").n_sel


def run(name, spec, procs):
    global _STATE
    t0 = time.time()
    mesh = grid.build_fine_mesh(spec.nx, spec.ny)
    coeff = assembly.CoefficientField(spec.E, spec.nu, spec.E_min, spec.E_max)
    part = grid.build_coarse_partition(mesh, spec.nx // spec.H, spec.ny // spec.H)
    _STATE = (mesh, coeff, part, spec.heat_dirichlet_nodes)
    nc = len(part.neighborhoods)
    with mp.get_context("fork").Pool(procs) as pool:
        out = pool.map(_arpack, range(nc), chunksize=16)
    lam = np.array([o[1] for o in out])
    nsel = np.array([o[2] for o in out], dtype=np.int32)
    margin = np.array([_margin(w) for w in lam])
    rng = np.random.default_rng(17)
    check = np.unique(np.concatenate([np.argsort(margin)[:16], rng.choice(nc, size=min(8, nc), replace=False)]))
    with mp.get_context("fork").Pool(procs) as pool:
        dense = pool.map(_dense, [int(c) for c in check])
    dlam = np.array([d[1] for d in dense])
    dsel = np.array([d[2] for d in dense], dtype=np.int32)
    assert np.array_equal(dsel, nsel[check]), (name, check, dsel, nsel[check])
    N_c = int(np.sum(2 * nsel + 1))
    path = HERE / f"nc_{name}.npz"
    np.savez_compressed(path, eigenvalues=lam, n_sel=nsel, margin=margin, N_c=N_c,
                        dense_centres=check, dense_eigenvalues=dlam, dense_n_sel=dsel,
                        nx=spec.nx, ny=spec.ny, H=spec.H, E_checksum=float(np.sum(spec.E * np.arange(spec.E.size) % 7)))
    print(f"{name}: {nc} centres, N_c {N_c}, n_sel histogram {np.bincount(nsel, minlength=7)}, "
          f"min margin {margin.min():.3f}, dense checks {check.size} equal, {time.time()-t0:.0f} s", flush=True)


CASES = {
    "config3": lambda: configs.config3(seed=0),
    "config4": lambda: configs.config4(seed=0),
    "config5_step0": lambda: configs.config5(seed=0, step=0),
    "config5_step25": lambda: configs.config5(seed=0, step=25),
    "config5_step49": lambda: configs.config5(seed=0, step=49),
    "config2_1e2": lambda: configs.config2(seed=0, eta=1e2),
    "config2_1e4": lambda: configs.config2(seed=0, eta=1e4),
    "config2_1e6": lambda: configs.config2(seed=0, eta=1e6),
    "config2_1e8": lambda: configs.config2(seed=0, eta=1e8),
}


def main():
    procs = int(os.environ.get("NC_PROCS", "3"))
    names = sys.argv[1:] or list(CASES)
    for n in names:
        if n == "config5":
            for k in ("config5_step0", "config5_step25", "config5_step49"):
                run(k, CASES[k](), procs)
        elif n == "config2":
            for k in ("config2_1e2", "config2_1e4", "config2_1e6", "config2_1e8"):
                run(k, CASES[k](), procs)
        else:
            run(n, CASES[n](), procs)


if __name__ == "__main__":
    main()
