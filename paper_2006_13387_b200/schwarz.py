"""Two-level additive Schwarz preconditioner on the GPU (reference schwarz.py).

``build_preconditioner(tag, op, mesh, part, coeff, dirichlet_nodes, opts)``
keeps the reference signature (schwarz.py:176-211).  All seven Table-1
variants run on the GPU (``GPU_VARIANTS``): EH, EH+Rot, EH+Rot;Rand (heat
eigenproblems, gap rule), HH, HH+Rot (heat level 1) and EE, EE;Rand
(elasticity eigenproblems, rule 'fixed'); "None" is plain CG.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .assembly import ElasticityOperator


@dataclass(frozen=True)
class PreconditionerVariant:
    tag: str
    level1: str
    eig_kind: str | None
    randomized: bool
    enrich: bool


VARIANTS = {
    v.tag: v
    for v in [
        PreconditionerVariant("EE", "elasticity", "elasticity", False, False),
        PreconditionerVariant("EE;Rand", "elasticity", "elasticity", True, False),
        PreconditionerVariant("HH", "heat", "heat", False, False),
        PreconditionerVariant("HH+Rot", "heat", "heat", False, True),
        PreconditionerVariant("EH", "elasticity", "heat", False, False),
        PreconditionerVariant("EH+Rot", "elasticity", "heat", False, True),
        PreconditionerVariant("EH+Rot;Rand", "elasticity", "heat", True, True),
    ]
}
GPU_VARIANTS = ("EH", "EH+Rot", "EH+Rot;Rand", "HH", "HH+Rot", "EE", "EE;Rand")


def get_variant(tag):
    try:
        return VARIANTS[tag]
    except KeyError:
        raise ValueError(f"unknown preconditioner variant {tag!r}; choose from {sorted(VARIANTS)}") from None


@dataclass
class EigOptions:
    """schwarz.py:54-59"""

    n_max: int = 6
    rule: str | None = None  # None -> 'gap' for heat
    n_snapshots: int | None = None
    seed: int = 0


class IdentityPreconditioner:
    """The 'None' variant: plain CG."""

    coarse_dim = 0
    info = {}

    def apply(self, r):
        return r


class TwoLevelPreconditioner:
    """GPU-resident level-1 band factors + spectral coarse space + K0^-1."""

    def __init__(self, variant, op, handle, info):
        self.variant = variant
        self.op = op
        self.handle = handle
        self.n_free = op.n_free
        self.info = info

    @property
    def coarse_dim(self):
        return self.info["coarse_dim"]

    @property
    def mode_counts(self):
        return self.info["mode_counts"]

    def _call(self, fn, r):
        if r.shape[0] != self.n_free:
            raise ValueError("residual dimension mismatch")
        rp, keep, dev = _lib.vec_ptr(r)
        if dev:
            import torch

            z = torch.empty_like(keep)
            zp = C.c_void_p(z.data_ptr())
        else:
            z = np.empty(self.n_free)
            zp = C.c_void_p(z.ctypes.data)
        _lib.check(fn(self.handle, rp, zp), self.op._ctx.handle)
        return z

    def apply(self, r):
        """z = sum_i R_i^T K_i^-1 R_i r + R0^T K0^-1 R0 r (schwarz.py:76-84)."""
        return self._call(_lib.load().ms_precond_apply, r)

    def apply_coarse(self, r):
        """R0^T K0^-1 R0 r (CoarseOperator.apply_inverse, coarse.py:156-158)."""
        return self._call(_lib.load().ms_precond_apply_coarse, r)

    def bench_components(self, reps=20):
        """Each hot-path kernel timed alone (CUDA events), ms per launch."""
        out = np.zeros(8)
        _lib.check(_lib.load().ms_precond_bench(self.handle, int(reps), _lib.dptr(out)), self.op._ctx.handle)
        return {n: float(out[i]) for i, n in enumerate(_lib.BENCH_NAMES)}

    def coarse_matrix(self):
        N = self.coarse_dim
        K0 = np.empty((N, N))
        _lib.check(_lib.load().ms_precond_coarse_matrix(self.handle, _lib.dptr(K0)), self.op._ctx.handle)
        return K0

    def __del__(self):
        h = getattr(self, "handle", None)
        try:  # at interpreter exit the module globals may already be torn down
            if h is not None and h.value and _lib.alive():
                _lib.load().ms_precond_destroy(h)
        except Exception:
            pass
        self.handle = None


def randomized_forcings(mesh, part, dirichlet_nodes, n_snapshots, seed, kind="diffusion"):
    """Host forcings of solve_local_eig_randomized (spectral.py:119-121):
    centre k draws default_rng([seed, k]).uniform(-1, 1, (n_free_k, n_snap))
    over its free closed-neighbourhood dofs (schwarz.py:156-160); returned as
    [centre][snapshot][d * node] over all (2H+1)^2 nodes, zero at clamped
    nodes.  kind='elasticity' (d = 2): the free dofs are the x-dofs of the free
    nodes then their y-dofs (the reference's component-grouped order), stored
    as an x-plane followed by a y-plane."""
    NLx, NLy = 2 * part.mex + 1, 2 * part.mey + 1
    NL = NLx * NLy
    d = 2 if kind == "elasticity" else 1
    clamped = np.zeros(mesh.n_nodes, dtype=bool)
    clamped[np.asarray(dirichlet_nodes, dtype=np.int64)] = True
    F = np.zeros((part.n_neighborhoods, n_snapshots, d * NL))
    for k, (I, J) in enumerate(part.coarse_nodes):
        a0, b0 = (I - 1) * part.mex, (J - 1) * part.mey
        gids = ((b0 + np.arange(NLy))[:, None] * (mesh.nx + 1) + (a0 + np.arange(NLx))[None, :]).ravel()
        free = np.nonzero(~clamped[gids])[0]
        if d == 2:
            free = np.concatenate([free, NL + free])
        ns = min(n_snapshots, free.size)
        Fk = np.random.default_rng([seed, k]).uniform(-1.0, 1.0, size=(free.size, ns))
        F[k, :ns][:, free] = Fk.T
    return F


def build_preconditioner(tag, op, mesh, part, coeff, dirichlet_nodes, opts=None, *,
                         level1="neighborhoods", delta=None, use_coarse=True, local_solver="banded",
                         coarse_solve="inverse"):
    """Build a two-level preconditioner by variant name (schwarz.py:176-211).

    level1='neighborhoods' is the reference's layout (subdomains = omega_j);
    level1='blocks' uses delta-extended coarse blocks (the BASELINE configs).
    ``dirichlet_nodes`` are the whole nodes clamped in the heat eigenproblems.
    coarse_solve='inverse' applies an explicit packed K0^-1 (one SYMV per
    apply); 'cholesky' keeps the reference's arithmetic, the Cholesky factor
    and two triangular solves (cho_factor / cho_solve, coarse.py:143,154).
    """
    if tag == "None":
        return IdentityPreconditioner()
    variant = get_variant(tag)
    if tag not in GPU_VARIANTS:
        raise NotImplementedError(f"variant {tag!r} is not on the GPU path (supported: {GPU_VARIANTS})")
    if not isinstance(op, ElasticityOperator):
        raise TypeError("build_preconditioner needs the GPU ElasticityOperator from assemble_elasticity")
    opts = opts or EigOptions()
    elastic = variant.eig_kind == "elasticity"
    rule = opts.rule or ("fixed" if elastic else "gap")
    if rule not in ("gap", "fixed"):
        raise ValueError(f"unknown selection rule {rule!r}")
    if elastic and rule == "gap":  # spectral.py:176-177
        raise ValueError("gap rule is not reliable for elasticity eigenproblems")
    hd = np.ascontiguousarray(np.asarray(dirichlet_nodes, dtype=np.int64).ravel())
    o = _lib.PrecondOpts()
    o.Nx, o.Ny = part.Nx, part.Ny
    if level1 == "neighborhoods":
        o.level1_kind, o.delta = _lib.MS_LEVEL1_NEIGHBORHOODS, 0
    elif level1 == "blocks":
        if delta is None:
            raise ValueError("level1='blocks' needs the overlap delta")
        o.level1_kind, o.delta = _lib.MS_LEVEL1_BLOCKS, int(delta)
    else:
        raise ValueError(f"unknown level-1 layout {level1!r}")
    o.n_max = int(opts.n_max)
    o.gap_threshold = 50.0
    o.enrich = 1 if variant.enrich else 0
    o.fixed_rule = 1 if rule == "fixed" else 0
    if local_solver not in ("banded", "dense"):
        raise ValueError(f"unknown local solver {local_solver!r}")
    o.local_solver = _lib.MS_LOCAL_BANDED if local_solver == "banded" else _lib.MS_LOCAL_DENSE_INV
    o.use_coarse = 1 if use_coarse else 0
    if coarse_solve not in ("inverse", "cholesky"):
        raise ValueError(f"unknown coarse solve {coarse_solve!r}")
    o.coarse_solve = _lib.MS_COARSE_CHOLESKY if coarse_solve == "cholesky" else _lib.MS_COARSE_INVERSE
    o.level1_operator = _lib.MS_L1_HEAT if variant.level1 == "heat" else _lib.MS_L1_ELASTICITY
    o.eig_kind = _lib.MS_EIG_ELASTICITY if elastic else _lib.MS_EIG_HEAT
    o.heat_dirichlet_nodes = hd.ctypes.data_as(C.POINTER(C.c_int64)) if hd.size else None
    o.n_heat_dirichlet = hd.size
    F = None
    if variant.randomized:
        ns = opts.n_snapshots or (opts.n_max + 5)
        F = np.ascontiguousarray(randomized_forcings(mesh, part, hd, ns, opts.seed,
                                                     "elasticity" if elastic else "diffusion"))
        o.randomized, o.n_snapshots, o.snapshots = 1, ns, F.ctypes.data
    lib = _lib.load()
    h = C.c_void_p()
    _lib.check(lib.ms_precond_build(op.handle, C.byref(o), C.byref(h)), op._ctx.handle)
    inf = _lib.PrecondInfo()
    nc = (part.Nx - 1) * (part.Ny - 1) if use_coarse else 0
    counts = np.zeros(max(nc, 1), dtype=np.int32)
    evals = np.full((max(nc, 1), 7), np.nan)
    _lib.check(lib.ms_precond_info_get(h, C.byref(inf), _lib.iptr(counts), _lib.dptr(evals)))
    info = {
        "t_level1": inf.t_level1, "t_coarse": inf.t_coarse, "t_eig": inf.t_eig,
        "coarse_dim": inf.coarse_dim, "mode_counts": [int(c) for c in counts[:nc]],
        "basis_kind": "E" if elastic else ("H+Rot" if variant.enrich else "H"), "selection_rule": rule,
        "eig_solver": "randomized" if variant.randomized else "subspace",
        "eigenvalues": evals[:nc], "n_subdomains": inf.n_subdomains,
        "max_eig_passes": inf.max_eig_passes, "mean_eig_passes": inf.mean_eig_passes, "local_bytes": inf.local_bytes,
        "coarse_bytes": inf.coarse_bytes, "level1": level1, "level1_operator": variant.level1, "delta": delta, "local_solver": local_solver,
        "coarse_solve": coarse_solve, "level1_twisted": bool(inf.level1_twisted),
        "level1_copies": int(inf.level1_copies), "n_subdomains_local": int(inf.n_subdomains_local),
        "level1_unit": int(inf.level1_unit),
    }
    return TwoLevelPreconditioner(variant, op, h, info)
