"""CPU oracle for the two-level spectral Schwarz PCG path — TEST INFRASTRUCTURE.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The CUDA path (``paper_2006_13387_b200``)
never routes through it.

It is a numpy/scipy restatement of the reference package ``mselast``
(``/root/reference/pkg/src/mselast``), following the same third-party calls
(scipy CSR assembly, SuperLU ``splu``, LAPACK ``?sygvx`` via ``eigh``,
``cho_factor``/``cho_solve``) so that it reproduces the reference bit for bit
on the reference's own benchmark.  Each function cites the reference
file:line it restates.  Parity is PINNED: ``tests/test_oracle_pins.py``
checks it against ``tests/golden/*.npz``, which ``tests/golden/make_golden.py``
produced by running the unmodified reference in the build container.

Two extensions the BASELINE configs need are marked ADAPTER:
delta-extended level-1 blocks and component-wise constraints.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

# ---------------------------------------------------------------------------
# structured mesh (grid.py:14-65)


@dataclass(frozen=True)
class Mesh:
    nx: int
    ny: int
    h: float

    @property
    def n_nodes(self):
        return (self.nx + 1) * (self.ny + 1)

    @property
    def n_dofs(self):
        return 2 * self.n_nodes

    def xy(self):
        """Node coordinates, lexicographic (grid.py:37-42)."""
        X, Y = np.meshgrid(np.arange(self.nx + 1) * self.h, np.arange(self.ny + 1) * self.h)
        return np.column_stack([X.ravel(), Y.ravel()])

    def quad_nodes(self):
        """(n_el, 4) corners, counter-clockwise from lower-left (grid.py:44-49)."""
        jj, ii = np.divmod(np.arange(self.nx * self.ny), self.nx)
        n0 = jj * (self.nx + 1) + ii
        return np.stack([n0, n0 + 1, n0 + self.nx + 2, n0 + self.nx + 1], axis=1)

    def quad_dofs(self):
        """(n_el, 8) component-grouped dofs (grid.py:51-54)."""
        q = self.quad_nodes()
        return np.concatenate([q, q + self.n_nodes], axis=1)


def mesh_for(nx, ny, h=None):
    return Mesh(int(nx), int(ny), float(1.0 / nx if h is None else h))


def rect_nodes(mesh, a0, a1, b0, b1):
    """Global ids of nodes (a, b), a0<=a<=a1, b0<=b<=b1, lexicographic."""
    if a1 < a0 or b1 < b0:
        return np.zeros(0, dtype=np.int64)
    a = np.arange(a0, a1 + 1)
    b = np.arange(b0, b1 + 1)
    return (b[:, None] * (mesh.nx + 1) + a[None, :]).ravel().astype(np.int64)


# ---------------------------------------------------------------------------
# element matrices (assembly.py:83-147)

_G = (0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0))


def _grad_ref(xi, eta):
    """Rows d/dx, d/dy of the 4 bilinear shape functions (assembly.py:88-96)."""
    return np.array([[-(1 - eta), 1 - eta, eta, -eta], [-(1 - xi), -xi, xi, 1 - xi]])


def elasticity_element(nu):
    """Unit plane-stress Q1 stiffness, E=1 (assembly.py:100-116)."""
    D = np.array([[1.0, nu, 0.0], [nu, 1.0, 0.0], [0.0, 0.0, (1.0 - nu) / 2.0]]) / (1.0 - nu * nu)
    K = np.zeros((8, 8))
    for xi in _G:
        for eta in _G:
            g = _grad_ref(xi, eta)
            B = np.zeros((3, 8))
            B[0, :4], B[1, 4:], B[2, :4], B[2, 4:] = g[0], g[1], g[1], g[0]
            K += 0.25 * B.T @ D @ B
    return 0.5 * (K + K.T)


def laplace_element():
    """Unit-conductivity Q1 Laplacian (assembly.py:133-140)."""
    A = np.zeros((4, 4))
    for xi in _G:
        for eta in _G:
            g = _grad_ref(xi, eta)
            A += 0.25 * (np.outer(g[0], g[0]) + np.outer(g[1], g[1]))
    return A


def mass_element(h):
    """Exact Q1 scalar mass on a square of side h (assembly.py:143-147)."""
    pat = np.array([[4.0, 2.0, 1.0, 2.0], [2.0, 4.0, 2.0, 1.0], [1.0, 2.0, 4.0, 2.0], [2.0, 1.0, 2.0, 4.0]])
    return (h * h / 36.0) * pat


# ---------------------------------------------------------------------------
# assembly over free dofs (assembly.py:150-259)


@dataclass
class FreeOperator:
    """CSR over free dofs plus the free-dof map (assembly.py:150-182)."""

    matrix: sp.csr_matrix
    free_dofs: np.ndarray
    n_full: int

    @property
    def n_free(self):
        return self.free_dofs.size

    def free_index(self):
        m = np.full(self.n_full, -1, dtype=np.int64)
        m[self.free_dofs] = np.arange(self.free_dofs.size)
        return m


def _assemble_free(dofs, mats, n, free):
    """COO sum -> CSR -> 0.5(A+A^T) -> A[free][:, free] (assembly.py:185-196)."""
    w = dofs.shape[1]
    rows = np.repeat(dofs, w, axis=1).ravel()
    cols = np.tile(dofs, (1, w)).ravel()
    A = sp.coo_matrix((mats.ravel(), (rows, cols)), shape=(n, n)).tocsr()
    A = 0.5 * (A + A.T)
    if free.size == 0:
        raise ValueError("empty free-dof set")
    return FreeOperator(A[free][:, free].tocsr(), free, n)


def free_complement(n, constrained):
    """setdiff of constrained ids (assembly.py:203-205)."""
    return np.setdiff1d(np.arange(n), np.asarray(constrained, dtype=np.int64))


def elasticity_operator(mesh, E, nu, constrained_dofs):
    """K over free dofs; constraints are arbitrary full-dof ids (assembly.py:208-220).

    ADAPTER: the reference clamps whole nodes; passing component-wise ids here
    is the SURVEY.md §A.5 construction (``_assemble`` with a custom free set).
    """
    E = np.asarray(E, dtype=float).ravel()
    mats = E[:, None, None] * elasticity_element(float(nu))[None]
    return _assemble_free(mesh.quad_dofs(), mats, mesh.n_dofs, free_complement(mesh.n_dofs, constrained_dofs))


def whole_node_dofs(mesh, nodes):
    nodes = np.asarray(nodes, dtype=np.int64)
    return np.concatenate([nodes, nodes + mesh.n_nodes])


def heat_pencil(mesh, E, dirichlet_nodes):
    """Diffusion stiffness and E-weighted mass (assembly.py:223-259, diffusion kind)."""
    E = np.asarray(E, dtype=float).ravel()
    free = free_complement(mesh.n_nodes, dirichlet_nodes)
    K = _assemble_free(mesh.quad_nodes(), E[:, None, None] * laplace_element()[None], mesh.n_nodes, free)
    M = _assemble_free(mesh.quad_nodes(), E[:, None, None] * mass_element(mesh.h)[None], mesh.n_nodes, free)
    return K, M


# ---------------------------------------------------------------------------
# coarse partition, neighbourhoods and partition of unity (grid.py:107-219)


@dataclass
class Partition:
    """Coarse blocks and interior-coarse-node neighbourhoods (grid.py:117-141)."""

    mesh: Mesh
    Nx: int
    Ny: int

    def __post_init__(self):
        if self.mesh.nx % self.Nx or self.mesh.ny % self.Ny:
            raise ValueError("coarse mesh not nested in fine mesh")
        self.mex = self.mesh.nx // self.Nx
        self.mey = self.mesh.ny // self.Ny
        self.centers = [(I, J) for J in range(1, self.Ny) for I in range(1, self.Nx)]
        # element rectangles [ex0, ex1) x [ey0, ey1)
        self.omegas = [
            (max(0, (I - 1) * self.mex), min(self.mesh.nx, (I + 1) * self.mex),
             max(0, (J - 1) * self.mey), min(self.mesh.ny, (J + 1) * self.mey))
            for (I, J) in self.centers
        ]

    @property
    def n_centers(self):
        return len(self.centers)

    def center_xy(self, k):
        I, J = self.centers[k]
        return I * self.mex * self.mesh.h, J * self.mey * self.mesh.h


def pou_values(part):
    """chi_k on the closed omega_k nodes, renormalised by the hat sum (grid.py:172-207)."""
    mesh = part.mesh
    xy = mesh.xy()
    Hx, Hy = part.mex * mesh.h, part.mey * mesh.h
    ids, raw = [], []
    for k, (ex0, ex1, ey0, ey1) in enumerate(part.omegas):
        cx, cy = part.center_xy(k)
        nid = rect_nodes(mesh, ex0, ex1, ey0, ey1)
        p = xy[nid]
        raw.append(np.maximum(0.0, 1.0 - np.abs(p[:, 0] - cx) / Hx)
                   * np.maximum(0.0, 1.0 - np.abs(p[:, 1] - cy) / Hy))
        ids.append(nid)
    total = np.zeros(mesh.n_nodes)
    for nid, v in zip(ids, raw):
        np.add.at(total, nid, v)
    denom = np.where(total > 0.0, total, 1.0)
    return ids, [v / denom[nid] for nid, v in zip(ids, raw)]


# ---------------------------------------------------------------------------
# local heat eigenproblems and the gap rule (spectral.py:63-100, 161-186)


def local_heat_problem(mesh, E, rect, dirichlet_nodes):
    """Neumann heat pencil on omega (Dirichlet where globally clamped) (spectral.py:63-90)."""
    ex0, ex1, ey0, ey1 = rect
    pmesh = Mesh(ex1 - ex0, ey1 - ey0, mesh.h)
    Eloc = np.asarray(E).reshape(mesh.ny, mesh.nx)[ey0:ey1, ex0:ex1].ravel()
    gids = rect_nodes(mesh, ex0, ex1, ey0, ey1)
    local_dir = np.nonzero(np.isin(gids, np.asarray(dirichlet_nodes, dtype=np.int64)))[0]
    K, M = heat_pencil(pmesh, Eloc, local_dir)
    return K, M, pmesh


def lowest_eigenpairs(K, M, k, Z=None):
    """Dense generalized eigensolve, LAPACK ?sygvx (spectral.py:93-100)."""
    if k > K.matrix.shape[0]:
        raise ValueError("more modes requested than dofs")
    return sla.eigh(K.matrix.toarray(), M.matrix.toarray(), subset_by_index=[0, k - 1])


def lowest_eigenpairs_arpack(K, M, k):
    """Shift-invert ARPACK alternative to ?sygvx, same pencil and k.

    Used where the dense solve is too slow (the bench's bounded CPU sample and
    large parity cases); tests check it against ``lowest_eigenpairs`` on the
    golden neighbourhoods.  Vectors are M-orthonormal like eigh's.
    """
    A, B = K.matrix.tocsc(), M.matrix.tocsc()
    n = A.shape[0]
    if n <= 4 * k + 20:
        return lowest_eigenpairs(K, M, k)
    sigma = -1e-10 * A.diagonal().sum() / B.diagonal().sum()
    w, v = spla.eigsh(A, k, B, sigma=sigma, which="LM")
    order = np.argsort(w)
    w, v = w[order], v[:, order]
    v = v / np.sqrt(np.einsum("ij,ij->j", v, B @ v))
    return w, v


def randomized_eigenpairs(K, M, k, n_snapshots, seed, n_passes=4, Z=None):
    """Randomized snapshot eigen-approximation (spectral.py:103-158).

    Deflated shift-invert block iteration on uniform(-1,1) forcings drawn from
    ``default_rng(seed)``, enrichment with the near-null candidates Z (the
    constant for heat, the rigid-body modes for elasticity), SVD
    orthonormalisation with a 1e-10 rank cut, Rayleigh-Ritz.
    """
    if n_snapshots < k:
        raise ValueError("need at least k snapshots")
    A, B = K.matrix, M.matrix
    n = A.shape[0]
    rng = np.random.default_rng(seed)
    Z = np.ones((n, 1)) if Z is None else Z
    MZ = B @ Z
    G = Z.T @ MZ
    F = rng.uniform(-1.0, 1.0, size=(n, n_snapshots))
    F = F - MZ @ np.linalg.solve(G, Z.T @ F)

    def deflate(X):
        return X - Z @ np.linalg.solve(G, MZ.T @ X)

    sigma = 1e-8 * (A.diagonal().sum() / n)
    lu = spla.splu((A + sigma * B).tocsc())
    U = deflate(lu.solve(F))
    for _ in range(n_passes - 1):
        U, _ = np.linalg.qr(U)
        U = deflate(lu.solve(B @ U))
    W = np.hstack([U, Z])
    nrm = np.linalg.norm(W, axis=0)
    nrm[nrm == 0.0] = 1.0
    Q, s, _ = np.linalg.svd(W / nrm, full_matrices=False)
    Q = Q[:, s > 1e-10 * s[0]]
    Kr = Q.T @ (A @ Q)
    Mr = Q.T @ (B @ Q)
    w, v = sla.eigh(0.5 * (Kr + Kr.T), 0.5 * (Mr + Mr.T))
    m = min(k, w.size)
    return w[:m], Q @ v[:, :m]


def randomized_solver(n_max=6, n_snapshots=None, seed=0):
    """eig_solver hook for heat_rot_coarse_space: per-centre seed [seed, centre]
    (schwarz.py:156-160); n_snapshots defaults to n_max + 5."""
    counter = {"k": 0}

    def solve(K, M, kk, Z=None):
        centre = counter["k"]
        counter["k"] += 1
        ns = n_snapshots or (n_max + 5)
        return randomized_eigenpairs(K, M, kk, min(ns, K.n_free), [seed, centre], Z=Z)

    return solve


def gap_count(lam, n_max, threshold=50.0):
    """Gap rule (spectral.py:161-186): largest i<=n_max with l[i]/max(l[i-1],eps)>=thr."""
    if n_max < 1:
        raise ValueError("mode cap must be >= 1")
    win = np.asarray(lam)[: min(n_max + 1, len(lam))]
    eps = 1e-14 * abs(win[-1]) if win[-1] != 0 else 1e-300
    n = 1
    for i in range(1, win.size):
        if win[i] / max(win[i - 1], eps) >= threshold:
            n = i
    return min(n, n_max)


def gap_margin(lam, n_max, threshold=50.0):
    """min |log(ratio/threshold)| over the gap tests (parity-harness diagnostic)."""
    win = np.asarray(lam)[: min(n_max + 1, len(lam))]
    eps = 1e-14 * abs(win[-1]) if win[-1] != 0 else 1e-300
    r = [win[i] / max(win[i - 1], eps) for i in range(1, win.size)]
    return float(np.min(np.abs(np.log(np.maximum(r, 1e-300) / threshold)))) if r else np.inf


# ---------------------------------------------------------------------------
# coarse basis (coarse.py:33-133) and the coarse operator (coarse.py:136-168)


@dataclass
class CoarseSpace:
    R0: sp.csr_matrix
    modes: list  # selected heat modes per centre
    eigenvalues: list  # the k=min(n_max+1, dim) computed eigenvalues per centre
    eigvecs: list  # selected eigenvectors per centre (free local nodes x n_sel)
    t_eig: float = 0.0

    @property
    def N_c(self):
        return self.R0.shape[0]


class _Rows:
    """Sparse row accumulator dropping exact zeros (coarse.py:33-55)."""

    def __init__(self, ncols):
        self.ncols, self.r, self.c, self.v, self.n = ncols, [], [], [], 0

    def push(self, fx, fy, vx, vy):
        cols = np.concatenate([fx[fx >= 0], fy[fy >= 0]])
        vals = np.concatenate([vx[fx >= 0], vy[fy >= 0]])
        keep = vals != 0.0
        self.r.append(np.full(int(keep.sum()), self.n))
        self.c.append(cols[keep])
        self.v.append(vals[keep])
        self.n += 1

    def csr(self):
        if self.n == 0:
            return sp.csr_matrix((0, self.ncols))
        return sp.coo_matrix((np.concatenate(self.v), (np.concatenate(self.r), np.concatenate(self.c))),
                             shape=(self.n, self.ncols)).tocsr()


def heat_rot_coarse_space(op, mesh, part, E, dirichlet_nodes, n_max=6, threshold=50.0,
                          enrich=True, rule="gap", eig_solver=None):
    """EH(+Rot) coarse basis rows (schwarz.py:143-173, coarse.py:94-133).

    Rows: per centre, per selected mode, x-slot then y-slot; then (enrich) one
    localized rotation per centre, appended after all heat rows.
    """
    eig_solver = eig_solver or lowest_eigenpairs
    fidx = op.free_index()
    pou_ids, pou_vals = pou_values(part)
    chi_full = np.zeros(mesh.n_nodes)
    xy = mesh.xy()
    heat, rot = _Rows(op.n_free), _Rows(op.n_free)
    modes, lams, vecs = [], [], []
    t_eig = 0.0
    for k, rect in enumerate(part.omegas):
        t0 = time.perf_counter()
        K, M, pmesh = local_heat_problem(mesh, E, rect, dirichlet_nodes)
        kk = min(n_max + 1, K.n_free)
        lam, V = eig_solver(K, M, kk)
        n = gap_count(lam, n_max, threshold) if rule == "gap" else min(n_max, lam.size)
        t_eig += time.perf_counter() - t0
        modes.append(n)
        lams.append(lam)
        vecs.append(V[:, :n])
        gn = rect_nodes(mesh, *rect)
        chi_full[:] = 0.0
        chi_full[pou_ids[k]] = pou_vals[k]
        chi = chi_full[gn]
        fx, fy = fidx[gn], fidx[gn + mesh.n_nodes]
        zero = np.zeros_like(chi)
        for m in range(n):
            psi = np.zeros(pmesh.n_nodes)
            psi[K.free_dofs] = V[:, m]
            heat.push(fx, fy, chi * psi, zero)
            heat.push(fx, fy, zero, chi * psi)
        if enrich:
            cx, cy = part.center_xy(k)
            p = xy[gn]
            rot.push(fx, fy, chi * -(p[:, 1] - cy), chi * (p[:, 0] - cx))
    R0 = heat.csr()
    if enrich:
        R0 = sp.vstack([R0, rot.csr()]).tocsr()
    return CoarseSpace(R0, modes, lams, vecs, t_eig)


def local_elasticity_problem(mesh, E, nu, rect, dirichlet_nodes):
    """Neumann elasticity pencil on omega (spectral.py:63-90, kind 'elasticity'):
    K restricted to the patch elements with whole-node Dirichlet where the
    patch meets clamped nodes, M the E-weighted block-diagonal Q1 mass
    (assembly.py:236-259), both on the free patch dofs."""
    ex0, ex1, ey0, ey1 = rect
    pmesh = Mesh(ex1 - ex0, ey1 - ey0, mesh.h)
    Eloc = np.asarray(E).reshape(mesh.ny, mesh.nx)[ey0:ey1, ex0:ex1].ravel()
    gids = rect_nodes(mesh, ex0, ex1, ey0, ey1)
    local_dir = np.nonzero(np.isin(gids, np.asarray(dirichlet_nodes, dtype=np.int64)))[0]
    K = elasticity_operator(pmesh, Eloc, nu, whole_node_dofs(pmesh, local_dir))
    me = mass_element(mesh.h)
    blk = np.zeros((8, 8))
    blk[:4, :4] = me
    blk[4:, 4:] = me
    M = _assemble_free(pmesh.quad_dofs(), Eloc[:, None, None] * blk[None], pmesh.n_dofs, K.free_dofs)
    return K, M, pmesh


def rigid_body_modes(pmesh, free_dofs):
    """x/y translations and the rotation about the patch centroid
    (assembly.py:262-273 with LocalEigProblem.kernel_basis, spectral.py:37-44)."""
    xy = pmesh.xy()
    c = xy.mean(axis=0)
    n = pmesh.n_nodes
    Z = np.zeros((2 * n, 3))
    Z[:n, 0] = 1.0
    Z[n:, 1] = 1.0
    Z[:n, 2] = -(xy[:, 1] - c[1])
    Z[n:, 2] = xy[:, 0] - c[0]
    return Z[free_dofs]


def elasticity_coarse_space(op, mesh, part, E, nu, dirichlet_nodes, n_max=6, eig_solver=None):
    """EE / EE;Rand coarse space: per centre the min(n_max, k) lowest
    elasticity eigenvectors (rule 'fixed', schwarz.py:148-173), each giving one
    vector-valued basis row chi * psi (coarse.py:76-91)."""
    eig_solver = eig_solver or lowest_eigenpairs
    fidx = op.free_index()
    pou_ids, pou_vals = pou_values(part)
    chi_full = np.zeros(mesh.n_nodes)
    rows = _Rows(op.n_free)
    modes, lams, vecs = [], [], []
    t_eig = 0.0
    for k, rect in enumerate(part.omegas):
        t0 = time.perf_counter()
        K, M, pmesh = local_elasticity_problem(mesh, E, nu, rect, dirichlet_nodes)
        kk = min(n_max + 1, K.n_free)
        lam, V = eig_solver(K, M, kk, Z=rigid_body_modes(pmesh, K.free_dofs))
        n = min(n_max, lam.size)
        t_eig += time.perf_counter() - t0
        modes.append(n)
        lams.append(lam)
        vecs.append(V[:, :n])
        gn = rect_nodes(mesh, *rect)
        chi_full[:] = 0.0
        chi_full[pou_ids[k]] = pou_vals[k]
        chi = chi_full[gn]
        fx, fy = fidx[gn], fidx[gn + mesh.n_nodes]
        npn = pmesh.n_nodes
        for m in range(n):
            psi = np.zeros(2 * npn)
            psi[K.free_dofs] = V[:, m]
            rows.push(fx, fy, chi * psi[:npn], chi * psi[npn:])
    return CoarseSpace(rows.csr(), modes, lams, vecs, t_eig)


class CoarseSolver:
    """Dense K0 = R0 A R0^T, symmetrised, Cholesky (coarse.py:136-168)."""

    def __init__(self, op, R0):
        if R0.shape[1] != op.n_free:
            raise ValueError("basis and operator dimensions do not match")
        K0 = ((R0 @ op.matrix) @ R0.T).toarray()
        self.K0 = 0.5 * (K0 + K0.T)
        self.R0 = R0
        try:
            self.chol = sla.cho_factor(self.K0)
        except np.linalg.LinAlgError as exc:
            raise ValueError("coarse operator not positive definite: basis is rank deficient") from exc

    @property
    def dim(self):
        return self.K0.shape[0]

    def apply(self, r):
        return self.R0.T @ sla.cho_solve(self.chol, self.R0 @ r)


# ---------------------------------------------------------------------------
# level-1 subdomains (schwarz.py:97-109 and the ADAPTER of SURVEY.md §A.3)


def subdomain_node_rect(mesh, rect, keep_domain_boundary):
    """Kept node rectangle [a0,a1]x[b0,b1] of an element patch.

    keep_domain_boundary=False: nodes strictly inside the patch, exactly the
    reference's ``Patch.interior_node_ids`` (grid.py:100-104).
    keep_domain_boundary=True (ADAPTER): along each axis a node is kept when it
    is strictly inside the patch interval or lies on a patch side that is part
    of the domain boundary -- the local Dirichlet part is the closure of
    dD'_i inside the domain (tensor-product form).
    """
    ex0, ex1, ey0, ey1 = rect
    a0, a1, b0, b1 = ex0 + 1, ex1 - 1, ey0 + 1, ey1 - 1
    if keep_domain_boundary:
        if ex0 == 0:
            a0 = 0
        if ex1 == mesh.nx:
            a1 = mesh.nx
        if ey0 == 0:
            b0 = 0
        if ey1 == mesh.ny:
            b1 = mesh.ny
    return a0, a1, b0, b1


def block_rects(mesh, H, delta):
    """delta-extended non-overlapping HxH blocks, J-major (ADAPTER)."""
    out = []
    for J in range(mesh.ny // H):
        for I in range(mesh.nx // H):
            out.append((max(0, I * H - delta), min(mesh.nx, (I + 1) * H + delta),
                        max(0, J * H - delta), min(mesh.ny, (J + 1) * H + delta)))
    return out


def level1_solvers(op, mesh, rects, keep_domain_boundary):
    """(free idx, SuperLU solve) per subdomain (schwarz.py:97-109)."""
    fidx = op.free_index()
    out = []
    for rect in rects:
        nodes = rect_nodes(mesh, *subdomain_node_rect(mesh, rect, keep_domain_boundary))
        idx = np.concatenate([fidx[nodes], fidx[nodes + mesh.n_nodes]])
        idx = idx[idx >= 0]
        if idx.size == 0:
            continue
        out.append((idx, spla.splu(op.matrix[idx][:, idx].tocsc()).solve))
    return out


def heat_level1_solvers(op, mesh, E, rects, keep_domain_boundary):
    """HH / HH+Rot level 1 (schwarz.py:112-140): one scalar factor of the
    E-weighted diffusion matrix restricted to the subdomain's free nodes,
    applied to the x block and to the y block.  Needs whole-node constraints
    (the reference's layout assumption, schwarz.py:113-117)."""
    nn = mesh.n_nodes
    cons = np.setdiff1d(np.arange(mesh.n_dofs), op.free_dofs)
    cnodes = cons[cons < nn]
    if not np.array_equal(cnodes + nn, cons[cons >= nn]):
        raise ValueError("heat level-1 needs whole-node constraints")
    E = np.asarray(E, dtype=float).ravel()
    D = _assemble_free(mesh.quad_nodes(), E[:, None, None] * laplace_element()[None], nn,
                       free_complement(nn, cnodes))
    sindex = D.free_index()
    out = []
    for rect in rects:
        nodes = rect_nodes(mesh, *subdomain_node_rect(mesh, rect, keep_domain_boundary))
        sidx = sindex[nodes]
        sidx = sidx[sidx >= 0]
        if sidx.size == 0:
            continue
        lu = spla.splu(D.matrix[sidx][:, sidx].tocsc())
        m = sidx.size

        def solve(r, lu=lu, m=m):
            out_ = np.empty_like(r)
            out_[:m] = lu.solve(r[:m])
            out_[m:] = lu.solve(r[m:])
            return out_

        out.append((np.concatenate([sidx, sidx + D.n_free]), solve))
    return out


class TwoLevel:
    """Additive level-1 + coarse correction (schwarz.py:66-84)."""

    def __init__(self, level1, coarse, n_free, info=None):
        self.level1, self.coarse, self.n_free = level1, coarse, n_free
        self.info = info or {}

    @property
    def coarse_dim(self):
        return 0 if self.coarse is None else self.coarse.dim

    def apply(self, r, reverse=False):
        if r.shape[0] != self.n_free:
            raise ValueError("residual dimension mismatch")
        z = np.zeros_like(r)
        for idx, solve in (reversed(self.level1) if reverse else self.level1):
            z[idx] += solve(r[idx])
        if self.coarse is not None:
            z += self.coarse.apply(r)
        return z

    def level1_only(self, r):
        return self.level1_apply(r)

    def level1_apply(self, r):
        z = np.zeros_like(r)
        for idx, solve in self.level1:
            z[idx] += solve(r[idx])
        return z


# ---------------------------------------------------------------------------
# PCG with Lanczos extremes (krylov.py:17-134)


@dataclass
class Report:
    iterations: int = 0
    converged: bool = False
    residuals: list = field(default_factory=list)
    alphas: list = field(default_factory=list)
    betas: list = field(default_factory=list)
    cond_estimate: float | None = None
    ritz_min: float | None = None
    ritz_max: float | None = None
    timings: dict = field(default_factory=dict)


def lanczos_extremes(alphas, betas, upto=None):
    """Ritz extremes of the PCG tridiagonal (krylov.py:38-59)."""
    k = len(alphas) if upto is None else min(upto, len(alphas))
    if k == 0:
        return None, None
    d = np.array([1.0 / alphas[j] + (betas[j - 1] / alphas[j - 1] if j else 0.0) for j in range(k)])
    e = np.array([np.sqrt(betas[j]) / alphas[j] for j in range(k - 1)])
    if k == 1:
        return d[0], d[0]
    w = sla.eigh_tridiagonal(d, e, eigvals_only=True)
    return w[0], w[-1]


def pcg(A, b, M=None, tol=1e-6, maxit=2000):
    """PCG from x0=0, stop on ||r_k|| <= tol ||b|| of the recursive residual (krylov.py:81-134)."""
    if not (0.0 < tol < 1.0):
        raise ValueError("tolerance must be in (0, 1)")
    mv = (lambda v: A @ v) if (sp.issparse(A) or isinstance(A, np.ndarray)) else A
    prec = (lambda r: r) if M is None else (M if callable(M) else M.apply)
    t0 = time.perf_counter()
    rep = Report()
    x = np.zeros_like(b)
    r = b.copy()
    bn = np.linalg.norm(b)
    rep.residuals.append(1.0)
    if bn == 0.0:
        rep.converged = True
        return x, rep
    z = prec(r)
    p = z.copy()
    rz = r @ z
    for _ in range(maxit):
        q = mv(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        rep.iterations += 1
        rep.residuals.append(np.linalg.norm(r) / bn)
        rep.alphas.append(alpha)
        if rep.residuals[-1] <= tol:
            rep.converged = True
            break
        z = prec(r)
        rz_new = r @ z
        rep.betas.append(rz_new / rz)
        p = z + rep.betas[-1] * p
        rz = rz_new
    rep.ritz_min, rep.ritz_max = lanczos_extremes(rep.alphas, rep.betas)
    rep.cond_estimate = None if rep.ritz_min is None else rep.ritz_max / rep.ritz_min
    rep.timings["solve"] = time.perf_counter() - t0
    return x, rep


# ---------------------------------------------------------------------------
# drivers


@dataclass
class OracleProblem:
    mesh: Mesh
    op: FreeOperator
    E: np.ndarray
    nu: float
    b: np.ndarray
    heat_dirichlet_nodes: np.ndarray


def problem_from_spec(spec):
    mesh = mesh_for(spec.nx, spec.ny)
    op = elasticity_operator(mesh, spec.E, spec.nu, spec.constrained_dofs)
    return OracleProblem(mesh, op, np.asarray(spec.E, float), spec.nu,
                         spec.load_full[op.free_dofs], np.asarray(spec.heat_dirichlet_nodes, np.int64))


def build_two_level(prob, H, delta=None, n_max=6, threshold=50.0, enrich=True, rule="gap",
                    level1_mode="blocks", eig_solver=None, level1_op="elasticity", eig_kind="heat"):
    """EH(+Rot) preconditioner; level1_op='heat' gives HH(+Rot).

    level1_mode='neighborhoods': reference semantics (subdomains = omega_j,
    strictly interior nodes; schwarz.py:176-211).  'blocks': ADAPTER with
    delta-extended HxH blocks.
    """
    mesh = prob.mesh
    part = Partition(mesh, mesh.nx // H, mesh.ny // H)
    t0 = time.perf_counter()
    if level1_mode == "neighborhoods":
        rects, keep = part.omegas, False
    else:
        rects, keep = block_rects(mesh, H, delta), True
    if level1_op == "heat":
        l1 = heat_level1_solvers(prob.op, mesh, prob.E, rects, keep)
    else:
        l1 = level1_solvers(prob.op, mesh, rects, keep)
    t_l1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    if eig_kind == "elasticity":
        cs = elasticity_coarse_space(prob.op, mesh, part, prob.E, prob.nu, prob.heat_dirichlet_nodes, n_max,
                                     eig_solver)
    else:
        cs = heat_rot_coarse_space(prob.op, mesh, part, prob.E, prob.heat_dirichlet_nodes, n_max,
                                   threshold, enrich, rule, eig_solver)
    coarse = CoarseSolver(prob.op, cs.R0)
    t_c = time.perf_counter() - t0
    info = {"t_level1": t_l1, "t_coarse": t_c, "t_eig": cs.t_eig, "coarse_dim": cs.N_c,
            "mode_counts": cs.modes, "basis_kind": "E" if eig_kind == "elasticity" else ("H+Rot" if enrich else "H"),
            "selection_rule": "fixed" if eig_kind == "elasticity" else rule}
    P = TwoLevel(l1, coarse, prob.op.n_free, info)
    P.coarse_space = cs
    P.partition = part
    return P


# ---------------------------------------------------------------------------
# topology-optimisation caller: body-force load
# (assembly.py:63-77), SIMP + density filter (assembly.py:280-336),
# sensitivity, OC update and the reuse loop (topopt.py:20-216)


def body_force_load(mesh, fx, fy):
    """Consistent nodal load of a uniform body force (assembly.py:69-76):
    element mass-row sums scattered to the corners in element order."""
    corner = mass_element(mesh.h).sum(axis=1)
    nodal = np.zeros(mesh.n_nodes)
    np.add.at(nodal, mesh.quad_nodes().ravel(), np.tile(corner, mesh.nx * mesh.ny))
    f = np.zeros(mesh.n_dofs)
    f[: mesh.n_nodes] += fx * nodal
    f[mesh.n_nodes:] += fy * nodal
    return f


def simp(rho_f, p, E_min, E_max):
    """simp_modulus (assembly.py:280-287)."""
    rho_f = np.asarray(rho_f, dtype=float)
    if rho_f.min() < -1e-12 or rho_f.max() > 1 + 1e-12:
        raise ValueError("density out of [0, 1]")
    return E_min + np.clip(rho_f, 0.0, 1.0) ** p * (E_max - E_min)


class ConeFilter:
    """DensityFilter (assembly.py:290-336): W = diag(1/rowsum) C with
    C_ek = max(0, r - h |c_e - c_k|) over the offsets with positive weight.
    Built with the same scipy calls (COO -> CSR, row sums, diagonal scaling),
    which fixes the stored order (descending columns) and the rounding."""

    def __init__(self, mesh, radius):
        nx, ny, h = mesh.nx, mesh.ny, mesh.h
        reach = max(int(np.ceil(radius / h)) - 1, 0) if radius > 0 else 0
        stencil = []
        for di in range(-reach, reach + 1):
            for dj in range(-reach, reach + 1):
                d = h * np.hypot(di, dj)
                if radius - d > 0:
                    stencil.append((di, dj, max(radius - d, 0.0) if radius > 0 else 1.0))
        if not stencil:
            stencil = [(0, 0, max(radius, 0.0) if radius > 0 else 1.0)]
        e = np.arange(nx * ny)
        ii, jj = e % nx, e // nx
        r_, c_, v_ = [], [], []
        for di, dj, w in stencil:
            ik, jk = ii + di, jj + dj
            ok = (ik >= 0) & (ik < nx) & (jk >= 0) & (jk < ny)
            r_.append(e[ok])
            c_.append((jk * nx + ik)[ok])
            v_.append(np.full(int(ok.sum()), w))
        Cm = sp.coo_matrix((np.concatenate(v_), (np.concatenate(r_), np.concatenate(c_))),
                           shape=(nx * ny, nx * ny)).tocsr()
        self.W = (sp.diags(1.0 / np.asarray(Cm.sum(axis=1)).ravel()) @ Cm).tocsr()

    def apply(self, rho):
        return self.W @ np.asarray(rho, dtype=float).ravel()

    def adjoint(self, v):
        return self.W.T @ np.asarray(v, dtype=float).ravel()


def compliance_and_sensitivity(mesh, u_full, f_full, rho_f, p, E_min, E_max, nu):
    """topopt.py:59-70: g0 = f.u and -p rho^(p-1) (E_max-E_min) u_e^T k0 u_e."""
    g0 = float(f_full @ u_full)
    ue = u_full[mesh.quad_dofs()]
    energy = np.einsum("ni,ij,nj->n", ue, elasticity_element(nu), ue)
    return g0, -p * np.clip(rho_f, 0.0, 1.0) ** (p - 1) * (E_max - E_min) * energy


def oc_update(rho, dg, volumes, v_star, move=0.2, damping=0.5, filt=None):
    """topopt.py:73-107: bracket the multiplier (64 tries), then bisect
    (<= 200 steps) until the (filtered) volume is within 1e-8 of v_star."""
    rho = np.asarray(rho, dtype=float)
    gain = np.maximum(-np.asarray(dg, dtype=float), 0.0)

    def cand(lam):
        step = rho * (gain / (lam * volumes)) ** damping
        return np.clip(np.clip(step, rho - move, rho + move), 0.0, 1.0)

    def vol(lam):
        x = cand(lam)
        return volumes @ (filt.apply(x) if filt is not None else x)

    lo, hi = 1e-9, 1e9
    for _ in range(64):
        if vol(lo) >= v_star >= vol(hi):
            break
        lo, hi = 0.5 * lo, 2.0 * hi
    else:
        raise RuntimeError("OC bisection failed to bracket the volume constraint")
    for _ in range(200):
        mid = np.sqrt(lo * hi)
        v = vol(mid)
        if v > v_star:
            lo = mid
        else:
            hi = mid
        if abs(v - v_star) <= 1e-8 * v_star:
            break
    return cand(np.sqrt(lo * hi))


def optimize(nx=60, ny=60, Nx=3, Ny=3, volfrac=0.3, penal=3.0, radius_factor=2.5, E_max=1.0,
             E_min=None, nu=0.3, n_iterations=100, variant="EH+Rot;Rand", tol=1e-6, maxit=2000,
             move=0.2, damping=0.5, period=1, max_inner=None, seed=0):
    """The SIMP loop with preconditioner reuse (topopt.py:123-216), reference
    semantics: neighbourhood level-1, fully clamped boundary, body force
    (0, -1), rebuild when due or when the solve fails (once)."""
    mesh = mesh_for(nx, ny)
    E_min = 1e-6 * E_max if E_min is None else E_min
    filt = ConeFilter(mesh, radius_factor * mesh.h)
    bnodes = np.nonzero(_boundary_mask(mesh))[0]
    cons = whole_node_dofs(mesh, bnodes)
    f_full = body_force_load(mesh, 0.0, -1.0)
    volumes = np.full(nx * ny, mesh.h * mesh.h)
    v_star = volfrac * volumes.sum()
    rho = np.full(nx * ny, volfrac)
    enrich = "+Rot" in variant
    eig = randomized_solver(seed=seed) if variant.endswith(";Rand") else None
    P, age, last, rebuilds, log = None, 0, 0, 0, []
    for it in range(n_iterations):
        rho_f = filt.apply(rho)
        E = simp(rho_f, penal, E_min, E_max)
        op = elasticity_operator(mesh, E, nu, cons)
        prob = OracleProblem(mesh, op, E, nu, f_full[op.free_dofs], bnodes)

        def build():
            return build_two_level(prob, H=nx // Nx, level1_mode="neighborhoods", enrich=enrich,
                                   eig_solver=randomized_solver(seed=seed) if eig else None,
                                   level1_op="heat" if variant.startswith("HH") else "elasticity")

        due = P is None or age >= period or (max_inner is not None and last > max_inner)
        if due:
            P, age = build(), 0
            rebuilds += 1
        rebuilt = due
        u, rep = pcg(op.matrix, prob.b, P, tol=tol, maxit=maxit)
        if not rep.converged:
            P, age = build(), 0
            rebuilds += 1
            rebuilt = True
            u, rep = pcg(op.matrix, prob.b, P, tol=tol, maxit=maxit)
            if not rep.converged:
                raise RuntimeError(f"state solve failed at iteration {it}")
        age += 1
        last = rep.iterations
        u_full = np.zeros(mesh.n_dofs)
        u_full[op.free_dofs] = u
        g0, sens = compliance_and_sensitivity(mesh, u_full, f_full, rho_f, penal, E_min, E_max, nu)
        rho = oc_update(rho, filt.adjoint(sens), volumes, v_star, move, damping, filt)
        log.append({"iteration": it, "g0": g0, "volume": float(volumes @ filt.apply(rho)),
                    "inner_iterations": rep.iterations, "rebuilt": rebuilt})
    return rho, filt.apply(rho), log, rebuilds


def _boundary_mask(mesh):
    jj, ii = np.divmod(np.arange(mesh.n_nodes), mesh.nx + 1)
    return (ii == 0) | (ii == mesh.nx) | (jj == 0) | (jj == mesh.ny)
