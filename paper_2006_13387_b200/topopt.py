"""Minimum-compliance SIMP loop with preconditioner reuse, on the GPU.

Same names, defaults and semantics as the reference's ``topopt`` module
(topopt.py:1-216).  Every per-design-step array stays on
the device: the density filter and its adjoint, the SIMP map into the
operator's modulus, the compliance sensitivity and the optimality-criteria
multiplier bisection are sm_100a kernels behind the C ABI
(``ms_filter_*``, ``ms_problem_set_density``, ``ms_compliance_sensitivity``,
``ms_oc_update``).  Only the per-iteration log scalars come back to the host.

Functions accept numpy arrays or float64 CUDA tensors and return the same
kind (numpy in, numpy out); ``optimize`` keeps tensors internally and returns
numpy designs like the reference.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._context import default_context
from .assembly import CoefficientField, ElasticityOperator, LoadSpec, build_load_vector, vector_dirichlet_dofs
from .grid import build_coarse_partition, build_fine_mesh
from .krylov import pcg_solve
from .schwarz import EigOptions, build_preconditioner


@dataclass
class ReusePolicy:
    """Rebuild after ``period`` design steps or when the previous solve's PCG
    iteration count exceeds ``max_inner_iterations`` (topopt.py:20-32)."""

    period: int = 1
    max_inner_iterations: int | None = None

    def __post_init__(self):
        if self.period < 1:
            raise ValueError("reuse period must be >= 1")
        if self.max_inner_iterations is not None and self.max_inner_iterations < 1:
            raise ValueError("inner-iteration threshold must be >= 1")


@dataclass
class OptimizeConfig:
    """topopt.py:35-56 (same fields and defaults)."""

    nx: int = 60
    ny: int = 60
    Nx: int = 3
    Ny: int = 3
    volfrac: float = 0.3
    penal: float = 3.0
    filter_radius_factor: float = 2.5
    E_max: float = 1.0
    E_min: float | None = None
    nu: float = 0.3
    n_iterations: int = 100
    variant: str = "EH+Rot;Rand"
    eig_options: EigOptions = field(default_factory=EigOptions)
    reuse: ReusePolicy = field(default_factory=ReusePolicy)
    tol: float = 1e-6
    maxit: int = 2000
    move_limit: float = 0.2
    damping: float = 0.5
    load: LoadSpec | None = None
    solver: str = "pcg"


# ---------------------------------------------------------------------------
# host/device plumbing


def _is_tensor(x):
    return type(x).__module__.startswith("torch")


def _as_dev(x):
    """float64 CUDA tensor view/copy of x (numpy arrays are uploaded)."""
    import torch

    if _is_tensor(x):
        t = x.to(dtype=torch.float64)
        if not t.is_cuda:
            t = t.cuda()
        return t.contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64).ravel(), device="cuda")


def _out_like(x, t):
    return t if _is_tensor(x) else t.cpu().numpy()


def _ptr(t):
    import torch

    torch.cuda.synchronize(t.device)
    return C.c_void_p(t.data_ptr())


def dot(a, b, ctx=None):
    """Deterministic device dot product (volume / compliance logs)."""
    ctx = ctx or default_context()
    ta, tb = _as_dev(a), _as_dev(b)
    if ta.numel() != tb.numel():
        raise ValueError("dimension mismatch")
    out = C.c_double()
    _lib.check(_lib.load().ms_dot(ctx.handle, ta.numel(), _ptr(ta), _ptr(tb), C.byref(out)), ctx.handle)
    return float(out.value)


# ---------------------------------------------------------------------------
# density filter


class DensityFilter:
    """Linear cone filter with row-normalised weights (assembly.py:290-336).

    ``apply`` is W rho and ``adjoint`` W^T v, both bit-identical to the
    reference's CSR products (same weights, normalisation and summation order).
    """

    def __init__(self, mesh, radius, ctx=None):
        if radius < 0:
            raise ValueError("filter radius must be nonnegative")
        self.mesh = mesh
        self.radius = float(radius)
        self._ctx = ctx or default_context()
        h = C.c_void_p()
        _lib.check(_lib.load().ms_filter_create(self._ctx.handle, mesh.nx, mesh.ny, mesh.h, self.radius,
                                                C.byref(h)), self._ctx.handle)
        self.handle = h

    def _run(self, fn, x):
        t = _as_dev(x)
        if t.numel() != self.mesh.n_elements:
            raise ValueError("field does not match the mesh")
        import torch

        out = torch.empty_like(t)
        _lib.check(fn(self.handle, _ptr(t), C.c_void_p(out.data_ptr())), self._ctx.handle)
        return _out_like(x, out)

    def apply(self, rho):
        return self._run(_lib.load().ms_filter_apply, rho)

    def adjoint(self, v):
        return self._run(_lib.load().ms_filter_adjoint, v)

    def __del__(self):
        h = getattr(self, "handle", None)
        try:  # at interpreter exit the module globals may already be torn down
            if h is not None and h.value and _lib.alive():
                _lib.load().ms_filter_destroy(h)
        except Exception:
            pass
        self.handle = None


# ---------------------------------------------------------------------------
# sensitivity and OC update


def compliance_and_sensitivity(mesh, u_full, f_full, rho_f, penal, E_min, E_max, nu, ctx=None):
    """Compliance f^T u and its gradient wrt the filtered densities (topopt.py:59-70).

    Per element: -p rho^(p-1) (E_max - E_min) u_e^T k0 u_e, k0 the unit-modulus
    element stiffness; all entries are nonpositive.
    """
    ctx = ctx or default_context()
    tu, tf, tr = _as_dev(u_full), _as_dev(f_full), _as_dev(rho_f)
    if tu.numel() != mesh.n_dofs or tf.numel() != mesh.n_dofs or tr.numel() != mesh.n_elements:
        raise ValueError("field does not match the mesh")
    import torch

    sens = torch.empty_like(tr)
    g0 = C.c_double()
    _lib.check(_lib.load().ms_compliance_sensitivity(
        ctx.handle, mesh.nx, mesh.ny, float(nu), _ptr(tu), _ptr(tf), _ptr(tr), float(penal), float(E_min),
        float(E_max), C.byref(g0), C.c_void_p(sens.data_ptr())), ctx.handle)
    return float(g0.value), _out_like(rho_f, sens)


def oc_update(rho, dg, volumes, v_star, move=0.2, damping=0.5, filt=None, ctx=None):
    """Optimality-criteria step with Lagrange-multiplier bisection (topopt.py:73-107).

    ``dg`` is the compliance gradient wrt the design densities (<= 0).  The
    multiplier is bracketed, then bisected on the device until the (filtered)
    volume constraint is active: v^T rho_f(rho_new) = v_star.  Raises
    RuntimeError when no bracket is found, like the reference.
    """
    ctx = ctx or (filt._ctx if filt is not None else default_context())
    tr, td, tv = _as_dev(rho), _as_dev(dg), _as_dev(volumes)
    n = tr.numel()
    if td.numel() != n or tv.numel() != n:
        raise ValueError("dimension mismatch")
    import torch

    out = torch.empty_like(tr)
    evals = C.c_int()
    _lib.check(_lib.load().ms_oc_update(
        ctx.handle, n, filt.handle if filt is not None else None, _ptr(tr), _ptr(td), _ptr(tv), float(v_star),
        float(move), float(damping), C.c_void_p(out.data_ptr()), C.byref(evals)), ctx.handle)
    return _out_like(rho, out)


# ---------------------------------------------------------------------------
# the loop


@dataclass
class OptimizationResult:
    rho: np.ndarray
    rho_f: np.ndarray
    log: list
    coarse_build_time: float
    rebuilds: int

    @property
    def compliance_history(self):
        return [row["g0"] for row in self.log]


def optimize(config, callback=None):
    """Run the SIMP loop on the GPU; returns the final design and the
    per-iteration log (topopt.py:123-216)."""
    import torch

    if config.solver != "pcg":
        raise ValueError("the GPU loop solves the state with PCG; solver='direct' is the CPU oracle path")
    mesh = build_fine_mesh(config.nx, config.ny)
    part = build_coarse_partition(mesh, config.Nx, config.Ny)
    E_min = config.E_min if config.E_min is not None else 1e-6 * config.E_max
    filt = DensityFilter(mesh, config.filter_radius_factor * mesh.h)
    ctx = filt._ctx
    dirichlet = mesh.boundary_nodes()

    load = config.load or LoadSpec(body_force=(0.0, -1.0))
    f_host = build_load_vector(mesh, load)
    volumes_h = np.full(mesh.n_elements, mesh.h * mesh.h)
    v_star = config.volfrac * volumes_h.sum()

    free = np.setdiff1d(np.arange(mesh.n_dofs), vector_dirichlet_dofs(mesh, dirichlet))
    # the modulus is written on the device every step (ms_problem_set_density);
    # the coefficient record only carries nu and the bounds
    coeff = CoefficientField(np.full(mesh.n_elements, config.E_max), config.nu, E_min, config.E_max)
    op = ElasticityOperator(mesh, coeff, free, ctx=ctx)
    dev = torch.device("cuda", torch.cuda.current_device())
    f_full = torch.tensor(f_host, device=dev)
    free_t = torch.tensor(free, device=dev)
    b = f_full[free_t].contiguous()
    volumes = torch.tensor(volumes_h, device=dev)
    rho = torch.full((mesh.n_elements,), float(config.volfrac), dtype=torch.float64, device=dev)
    u_full = torch.zeros(mesh.n_dofs, dtype=torch.float64, device=dev)

    precond = None
    precond_age = 0
    last_inner = 0
    coarse_build_time = 0.0
    rebuilds = 0
    log = []

    def build():
        t0 = time.perf_counter()
        pc = build_preconditioner(config.variant, op, mesh, part, coeff, dirichlet, config.eig_options)
        return pc, time.perf_counter() - t0

    for it in range(config.n_iterations):
        rho_f = filt.apply(rho)
        op.set_density(rho_f, config.penal, E_min, config.E_max)

        due = (precond is None or precond_age >= config.reuse.period
               or (config.reuse.max_inner_iterations is not None
                   and last_inner > config.reuse.max_inner_iterations))
        if due:
            precond = None  # release the old factors before building the new ones
            precond, dt = build()
            coarse_build_time += dt
            precond_age = 0
            rebuilds += 1
        rebuilt = due
        u_free, report = pcg_solve(op, b, precond, tol=config.tol, maxit=config.maxit)
        if not report.converged:
            # stale preconditioner is the usual culprit: rebuild and retry once
            precond = None
            precond, dt = build()
            coarse_build_time += dt
            precond_age = 0
            rebuilds += 1
            rebuilt = True
            u_free, report = pcg_solve(op, b, precond, tol=config.tol, maxit=config.maxit)
            if not report.converged:
                raise RuntimeError(f"state solve failed at iteration {it}")
        precond_age += 1
        last_inner = report.iterations

        u_full.zero_()
        u_full[free_t] = u_free
        g0, sens_f = compliance_and_sensitivity(mesh, u_full, f_full, rho_f, config.penal, E_min,
                                                config.E_max, config.nu, ctx=ctx)
        dg = filt.adjoint(sens_f)
        rho = oc_update(rho, dg, volumes, v_star, config.move_limit, config.damping, filt)
        row = {
            "iteration": it,
            "g0": g0,
            "volume": dot(volumes, filt.apply(rho), ctx),
            "inner_iterations": report.iterations,
            "rebuilt": rebuilt,
            "cond_estimate": report.cond_estimate,
        }
        log.append(row)
        if callback is not None:
            callback(it, rho, row)

    rho_f = filt.apply(rho)
    return OptimizationResult(rho.cpu().numpy(), rho_f.cpu().numpy(), log, coarse_build_time, rebuilds)
