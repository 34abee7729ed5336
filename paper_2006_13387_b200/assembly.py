"""Elasticity operator on the GPU behind the reference's assembly API.

``assemble_elasticity`` (assembly.py:208-220 in the reference) returns an
operator object with the same duck type as ``SymmetricSparseOperator``
(``free_dofs``, ``n_free``, ``free_index()``, ``expand``, ``restrict``,
``matrix @ v``) whose matvec is the matrix-free sm_100a kernel.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._context import default_context


@dataclass
class CoefficientField:
    """Per-element modulus with bounds and Poisson ratio (assembly.py:21-52)."""

    values: np.ndarray
    nu: float
    E_min: float
    E_max: float

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=float).ravel()
        if self.E_min <= 0:
            raise ValueError("E_min must be positive")
        tol = 1e-12 * self.E_max
        if self.values.min() < self.E_min - tol or self.values.max() > self.E_max + tol:
            raise ValueError("element moduli out of [E_min, E_max]")

    @property
    def contrast(self):
        return self.E_max / self.E_min


@dataclass
class LoadSpec:
    """Point loads (node, component, magnitude) plus an optional uniform body force (assembly.py:55-60)."""

    point_loads: list = field(default_factory=list)
    body_force: tuple | None = None  # (fx, fy) per unit area


def build_load_vector(mesh, load):
    """Full-layout load vector (assembly.py:63-77): point loads, then the
    consistent body force (each element adds the row sums of its Q1 mass
    element to its corners, in element order)."""
    f = np.zeros(mesh.n_dofs)
    for node, comp, mag in load.point_loads:
        if not (0 <= node < mesh.n_nodes) or comp not in (0, 1):
            raise ValueError(f"invalid point load ({node}, {comp})")
        f[node + comp * mesh.n_nodes] += mag
    if load.body_force is not None:
        fx, fy = load.body_force
        h2 = mesh.h * mesh.h / 36.0
        corner = (h2 * np.array([[4.0, 2.0, 1.0, 2.0], [2.0, 4.0, 2.0, 1.0], [1.0, 2.0, 4.0, 2.0],
                                 [2.0, 1.0, 2.0, 4.0]])).sum(axis=1)
        nodal = np.zeros(mesh.n_nodes)
        np.add.at(nodal, mesh.element_nodes().ravel(), np.tile(corner, mesh.n_elements))
        f[: mesh.n_nodes] += fx * nodal
        f[mesh.n_nodes:] += fy * nodal
    return f


def simp_modulus(rho_f, p, E_min, E_max):
    """E = E_min + rho^p (E_max - E_min) (assembly.py:280-287)."""
    rho_f = np.asarray(rho_f, dtype=float)
    if rho_f.min() < -1e-12 or rho_f.max() > 1 + 1e-12:
        raise ValueError("density out of [0, 1]")
    if p < 1:
        raise ValueError("penalization exponent must be >= 1")
    return E_min + np.clip(rho_f, 0.0, 1.0) ** p * (E_max - E_min)


def vector_dirichlet_dofs(mesh, nodes):
    nodes = np.asarray(nodes, dtype=np.int64)
    return np.concatenate([nodes, nodes + mesh.n_nodes])


class ElasticityOperator:
    """Free-dof Q1 plane-stress operator held on the GPU."""

    def __init__(self, mesh, coeff, free_dofs, ctx=None):
        self.mesh = mesh
        self.coeff = coeff
        self.nu = float(coeff.nu)
        self.free_dofs = np.ascontiguousarray(free_dofs, dtype=np.int64)
        self.n_full = mesh.n_dofs
        if self.free_dofs.size == 0:
            raise ValueError("empty free-dof set")
        self._ctx = ctx or default_context()
        lib = _lib.load()
        h = C.c_void_p()
        E = np.ascontiguousarray(coeff.values, dtype=np.float64)
        _lib.check(lib.ms_problem_create(self._ctx.handle, mesh.nx, mesh.ny, mesh.h, self.nu,
                                         C.c_void_p(E.ctypes.data), C.c_void_p(self.free_dofs.ctypes.data),
                                         self.free_dofs.size, C.byref(h)), self._ctx.handle)
        self.handle = h

    # SymmetricSparseOperator duck type (assembly.py:150-182)
    @property
    def n_free(self):
        return int(self.free_dofs.size)

    @property
    def matrix(self):
        return self

    @property
    def shape(self):
        return (self.n_free, self.n_free)

    def free_index(self):
        idx = np.full(self.n_full, -1, dtype=np.int64)
        idx[self.free_dofs] = np.arange(self.n_free)
        return idx

    def expand(self, x_free):
        x = np.zeros(self.n_full)
        x[self.free_dofs] = x_free
        return x

    def restrict(self, x_full):
        return np.asarray(x_full)[self.free_dofs]

    def apply(self, p):
        """q = A p on the GPU (replaces ``op.matrix @ p``, krylov.py:90)."""
        if p.shape[0] != self.n_free:
            raise ValueError("vector dimension mismatch")
        pp, keep, dev = _lib.vec_ptr(p)
        if dev:
            import torch

            q = torch.empty_like(keep)
            qp = C.c_void_p(q.data_ptr())
        else:
            q = np.empty(self.n_free)
            qp = C.c_void_p(q.ctypes.data)
        _lib.check(_lib.load().ms_operator_apply(self.handle, pp, qp), self._ctx.handle)
        return q

    __matmul__ = apply

    # scipy views of the assembled matrix (the reference's ``op.matrix`` is a
    # CSR matrix, e.g. ``op.matrix.tocsc()`` for a direct solve): K is recovered
    # from 18 operator applies on the GPU -- the Q1 stencil couples a node only
    # to its 8 neighbours, so nodes of one colour (a mod 3, b mod 3) never share
    # a row, and one apply per (colour, component) yields all their columns.
    def tocsr(self):
        import scipy.sparse as sp

        if getattr(self, "_csr", None) is not None and self._csr_E is self.coeff:
            return self._csr.copy()
        mesh = self.mesh
        nnx, nny = mesh.nx + 1, mesh.ny + 1
        n_nodes = nnx * nny
        a = np.tile(np.arange(nnx), nny)
        b = np.repeat(np.arange(nny), nnx)
        fidx = self.free_index()
        rows, cols, vals = [], [], []
        for comp in range(2):
            for cb in range(3):
                for ca in range(3):
                    src_nodes = np.flatnonzero((a % 3 == ca) & (b % 3 == cb))
                    src = fidx[comp * n_nodes + src_nodes]
                    src_nodes, src = src_nodes[src >= 0], src[src >= 0]
                    if src.size == 0:
                        continue
                    v = np.zeros(self.n_free)
                    v[src] = 1.0
                    q = self.expand(self.apply(v))
                    # the source node of every row: the unique colour node within one step
                    sa = a - ((a - ca) % 3) + np.where((a - ca) % 3 == 2, 3, 0)
                    sb = b - ((b - cb) % 3) + np.where((b - cb) % 3 == 2, 3, 0)
                    ok = (sa >= 0) & (sa < nnx) & (sb >= 0) & (sb < nny)
                    snode = np.where(ok, sb * nnx + sa, 0)
                    scol = np.where(ok, fidx[comp * n_nodes + snode], -1)
                    for rc in range(2):
                        r_full = rc * n_nodes + np.arange(n_nodes)
                        r_free = fidx[r_full]
                        val = q[r_full]
                        keep = (r_free >= 0) & (scol >= 0) & (val != 0.0)
                        rows.append(r_free[keep])
                        cols.append(scol[keep])
                        vals.append(val[keep])
        K = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.n_free, self.n_free))
        K.sort_indices()
        self._csr, self._csr_E = K, self.coeff
        return K.copy()

    def tocsc(self):
        return self.tocsr().tocsc()

    def toarray(self):
        return self.tocsr().toarray()

    def diagonal(self):
        return self.tocsr().diagonal()

    def set_modulus(self, E):
        """Replace the per-element modulus in place (topopt.py:150-160); the
        same checks as CoefficientField (assembly.py:21-52) guard the copy."""
        E = np.ascontiguousarray(E, dtype=np.float64).ravel()
        if E.size != self.mesh.n_elements:
            raise ValueError("coefficient field does not match mesh")
        if not np.all(E > 0):
            raise ValueError("element moduli must be positive")
        _lib.check(_lib.load().ms_problem_set_modulus(self.handle, C.c_void_p(E.ctypes.data)),
                   self._ctx.handle)
        self._csr = None

    def set_density(self, rho_f, p, E_min, E_max):
        """E = simp_modulus(rho_f, p, E_min, E_max) computed on the device into the
        operator's modulus (assembly.py:280-287 + the re-assembly of topopt.py:161-164).
        rho_f: numpy array or float64 CUDA tensor of element densities."""
        pp, keep, _ = _lib.vec_ptr(rho_f)
        if keep.shape[0] != self.mesh.n_elements:
            raise ValueError("density field does not match mesh")
        _lib.check(_lib.load().ms_problem_set_density(self.handle, pp, float(p), float(E_min), float(E_max)),
                   self._ctx.handle)
        self._csr = None

    def __del__(self):
        h = getattr(self, "handle", None)
        try:  # at interpreter exit the module globals may already be torn down
            if h is not None and h.value and _lib.alive():
                _lib.load().ms_problem_destroy(h)
        except Exception:
            pass
        self.handle = None


def element_stiffness_elasticity(E, nu, h=1.0):
    """Plane-stress Q1 element stiffness (assembly.py:119-130): E times the
    unit matrix the kernels use, computed by the library with the reference's
    exact arithmetic (ms_unit_element; bitwise equal to
    ``_unit_elasticity_element``, assembly.py:100-116)."""
    if E <= 0:
        raise ValueError("modulus must be positive")
    if not (0 <= nu < 0.5):
        raise ValueError(f"Poisson ratio {nu} outside [0, 0.5)")
    K = np.empty(64)
    _lib.check(_lib.load().ms_unit_element(float(nu), _lib.dptr(K)))
    return E * K.reshape(8, 8)


def assemble_elasticity(mesh, coeff, dirichlet_nodes, constrained_dofs=None):
    """GPU operator over free dofs (assembly.py:208-220).

    ``dirichlet_nodes`` clamp whole nodes exactly as in the reference;
    ``constrained_dofs`` (full-dof ids) additionally allows component-wise
    constraints (MBB configs).
    """
    if coeff.values.size != mesh.n_elements:
        raise ValueError("coefficient field does not match mesh")
    cons = vector_dirichlet_dofs(mesh, dirichlet_nodes)
    if constrained_dofs is not None:
        cons = np.concatenate([cons, np.asarray(constrained_dofs, dtype=np.int64)])
    free = np.setdiff1d(np.arange(mesh.n_dofs), cons)
    return ElasticityOperator(mesh, coeff, free)
