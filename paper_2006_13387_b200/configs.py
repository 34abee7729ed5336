"""Seeded synthetic inputs for the five BASELINE.json configurations.

These are INPUT generators (host numpy), shared verbatim by the CUDA path and
by the CPU oracle so that both consume the identical fp64 modulus array E,
the identical constrained-dof list and the identical load.  No reference
dataset exists for this path: the reference's only
benchmark is its own frozen layout, which the golden fixtures carry as data.

Frozen choices (DESIGN.md §3 "Inputs"):

* mesh / dof conventions follow the reference (grid.py:1-6): nodes
  lexicographic ``j*(nx+1)+i``, elements ``j*nx+i``, dofs component-grouped
  (all x then all y).
* SIMP map E = E_min + clip(rho,0,1)**p (E_max-E_min), p=3, E_max=1
  (assembly.py:280-287).
* cone filter of radius r = 4h with row-normalised weights max(0, r-|d|)
  (the ``DensityFilter`` semantics, assembly.py:290-330), applied with array
  shifts instead of an explicit sparse matrix.
* "near-binary at ~V volume": standardise the filtered noise, then apply the
  tanh projection (beta=8, eta=0.5) to 0.5 + 0.5*(s - t) with the shift t
  chosen by bisection so that mean(rho) == V (to 1e-9).
* cantilever: whole nodes on the left edge clamped, unit downward point load
  at the right-edge midpoint node.  MBB (config 4): x-dofs of the left edge
  and the y-dof of the bottom-right node constrained; unit downward load at
  the top-left node; heat eigenproblems are pure Neumann.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NU = 0.3
SIMP_P = 3.0


@dataclass
class ProblemSpec:
    """Everything one solve needs, in the reference's conventions."""

    name: str
    nx: int
    ny: int
    E: np.ndarray  # (nx*ny,) fp64, row-major elements
    E_min: float
    E_max: float
    constrained_dofs: np.ndarray  # int64 full-dof ids (component-grouped)
    heat_dirichlet_nodes: np.ndarray  # whole nodes clamped in the heat eigenproblems
    load_full: np.ndarray  # (2*n_nodes,) fp64 load in the full dof layout
    H: int  # subdomain / coarse block size in elements
    delta: int  # overlap of the level-1 blocks, in elements
    nu: float = NU
    tol: float = 1e-8
    maxit: int = 5000
    meta: dict = field(default_factory=dict)

    @property
    def h(self) -> float:
        return 1.0 / self.nx

    @property
    def n_nodes(self) -> int:
        return (self.nx + 1) * (self.ny + 1)

    @property
    def n_dofs(self) -> int:
        return 2 * self.n_nodes

    @property
    def Nx(self) -> int:
        return self.nx // self.H

    @property
    def Ny(self) -> int:
        return self.ny // self.H

    def free_dofs(self) -> np.ndarray:
        mask = np.ones(self.n_dofs, dtype=bool)
        mask[self.constrained_dofs] = False
        return np.nonzero(mask)[0].astype(np.int64)

    def rhs(self) -> np.ndarray:
        return self.load_full[self.free_dofs()]


# ---------------------------------------------------------------------------
# building blocks


def simp(rho, p=SIMP_P, E_min=1e-6, E_max=1.0):
    rho = np.asarray(rho, dtype=np.float64)
    return E_min + np.clip(rho, 0.0, 1.0) ** p * (E_max - E_min)


def cone_filter(field2d: np.ndarray, radius_elems: float = 4.0) -> np.ndarray:
    """Row-normalised cone filter on an (ny, nx) element array."""
    ny, nx = field2d.shape
    reach = max(int(np.ceil(radius_elems)) - 1, 0)
    acc = np.zeros_like(field2d)
    wsum = np.zeros_like(field2d)
    ones = np.ones_like(field2d)
    for di in range(-reach, reach + 1):
        for dj in range(-reach, reach + 1):
            w = radius_elems - np.hypot(di, dj)
            if w <= 0.0:
                continue
            # target (j, i) receives source (j+dj, i+di) when inside the mesh
            ys = slice(max(0, -dj), min(ny, ny - dj))
            xs = slice(max(0, -di), min(nx, nx - di))
            ysrc = slice(ys.start + dj, ys.stop + dj)
            xsrc = slice(xs.start + di, xs.stop + di)
            acc[ys, xs] += w * field2d[ysrc, xsrc]
            wsum[ys, xs] += w * ones[ysrc, xsrc]
    return acc / wsum


def tanh_project(x, beta=8.0, eta=0.5):
    num = np.tanh(beta * eta) + np.tanh(beta * (x - eta))
    den = np.tanh(beta * eta) + np.tanh(beta * (1.0 - eta))
    return num / den


def filtered_noise_density(rng, nx, ny, volume, beta=8.0, radius=4.0):
    """Uniform noise -> cone filter -> standardise -> shifted tanh projection."""
    noise = rng.uniform(0.0, 1.0, size=(ny, nx))
    f = cone_filter(noise, radius)
    s = (f - f.mean()) / f.std()

    def rho_of(t):
        return tanh_project(np.clip(0.5 + 0.5 * (s - t), 0.0, 1.0), beta, 0.5)

    lo, hi = -10.0, 10.0  # mean(rho) decreases in t
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if rho_of(mid).mean() > volume:
            lo = mid
        else:
            hi = mid
        if hi - lo < 1e-13:
            break
    return np.clip(rho_of(0.5 * (lo + hi)), 0.0, 1.0).ravel()


def _node(nx, i, j):
    return j * (nx + 1) + i


def cantilever_bcs(nx, ny):
    n_nodes = (nx + 1) * (ny + 1)
    left = np.array([_node(nx, 0, j) for j in range(ny + 1)], dtype=np.int64)
    constrained = np.concatenate([left, left + n_nodes])
    load = np.zeros(2 * n_nodes)
    load[_node(nx, nx, ny // 2) + n_nodes] = -1.0
    return constrained, left, load


def mbb_bcs(nx, ny):
    n_nodes = (nx + 1) * (ny + 1)
    left = np.array([_node(nx, 0, j) for j in range(ny + 1)], dtype=np.int64)
    roller = _node(nx, nx, 0) + n_nodes
    constrained = np.sort(np.concatenate([left, [roller]])).astype(np.int64)
    load = np.zeros(2 * n_nodes)
    load[_node(nx, 0, ny) + n_nodes] = -1.0
    return constrained, np.zeros(0, dtype=np.int64), load


def random_squares(rng, nx, ny, count, side_lo, side_hi):
    rho = np.zeros((ny, nx))
    for _ in range(count):
        s = int(rng.integers(side_lo, side_hi + 1))
        i0 = int(rng.integers(0, nx - s + 1))
        j0 = int(rng.integers(0, ny - s + 1))
        rho[j0 : j0 + s, i0 : i0 + s] = 1.0
    return rho


def random_channels(rng, nx, ny, target, width_lo=1, width_hi=2):
    """Long thin straight channels at random orientation until `target` solid."""
    rho = np.zeros((ny, nx))
    ci = (np.arange(nx) + 0.5)[None, :]
    cj = (np.arange(ny) + 0.5)[:, None]
    while rho.mean() < target:
        x0, y0 = rng.uniform(0, nx), rng.uniform(0, ny)
        theta = rng.uniform(0.0, np.pi)
        length = rng.uniform(0.2, 0.8) * max(nx, ny)
        w = rng.uniform(width_lo, width_hi)
        dx, dy = np.cos(theta), np.sin(theta)
        # distance of centroids to the segment [(x0,y0), (x0,y0) + L (dx,dy)]
        t = np.clip((ci - x0) * dx + (cj - y0) * dy, 0.0, length)
        d2 = (ci - x0 - t * dx) ** 2 + (cj - y0 - t * dy) ** 2
        rho[d2 <= (0.5 * w) ** 2] = 1.0
    return rho


# ---------------------------------------------------------------------------
# the five configurations (BASELINE.json "configs", in order)


def _spec(name, nx, ny, rho, E_min, bcs, H, delta, **meta):
    constrained, heat_dir, load = bcs
    E = simp(rho.ravel(), E_min=E_min)
    return ProblemSpec(
        name=name, nx=nx, ny=ny, E=E, E_min=E_min, E_max=1.0,
        constrained_dofs=constrained, heat_dirichlet_nodes=heat_dir,
        load_full=load, H=H, delta=delta,
        meta=dict(meta, solid_fraction=float(np.mean(np.asarray(rho) > 0.5)),
                  volume=float(np.mean(rho))),
    )


def config1(seed=0, n=64, H=16, delta=1, solid=0.20):
    """64^2, 40 random squares (side 2-6) at ~20% solid, E_min 1e-6, cantilever, delta=1.

    40 independent squares of side U{2..6} cover ~15% on average (overlaps), so
    the layout is drawn by seeded rejection: successive draws of `count`
    squares from the same generator until the solid fraction is within 0.01
    of `solid` (BASELINE config 1's "40 inclusions at ~20% solid")."""
    rng = np.random.default_rng([1, seed])
    count = max(1, int(round(40 * (n / 64) ** 2)))
    for _ in range(100000):
        rho = random_squares(rng, n, n, count, 2, 6)
        if abs(rho.mean() - solid) <= 0.01:
            break
    else:  # pragma: no cover
        raise RuntimeError("config1: no layout near the target solid fraction")
    return _spec(f"config1[n={n},seed={seed}]", n, n, rho, 1e-6, cantilever_bcs(n, n), H, delta)


def config2(seed=0, eta=1e6, n=512, H=32, delta=2):
    """512^2 thin random channels (~15%) + sparse inclusions, contrast sweep."""
    rng = np.random.default_rng([2, seed])
    rho = random_channels(rng, n, n, 0.15)
    rho = np.maximum(rho, random_squares(rng, n, n, max(1, int(30 * (n / 512) ** 2)), 2, 5))
    return _spec(f"config2[n={n},eta={eta:g},seed={seed}]", n, n, rho, 1.0 / eta,
                 cantilever_bcs(n, n), H, delta, eta=eta)


def config3(seed=0, n=2048, H=32, delta=2, eta=1e6, volume=0.4, ny=None):
    """2048^2 filtered-noise tanh-projected density at 40% volume, eta 1e6.
    ny < n gives an n x ny strip of the same recipe (e.g. 2048 x 256: the
    512 subdomains one GPU owns when config 3 is split over 8)."""
    ny = ny or n
    rng = np.random.default_rng([3, seed])
    rho = filtered_noise_density(rng, n, ny, volume)
    name = f"config3[n={n},seed={seed}]" if ny == n else f"config3[{n}x{ny},seed={seed}]"
    return _spec(name, n, ny, rho.reshape(ny, n), 1.0 / eta, cantilever_bcs(n, ny), H, delta, eta=eta)


def config4(seed=0, nx=4096, ny=2048, H=32, delta=2, eta=1e9, volume=0.5):
    """4096x2048 MBB beam, filtered-noise density at 50%, eta 1e9."""
    rng = np.random.default_rng([4, seed])
    rho = filtered_noise_density(rng, nx, ny, volume)
    return _spec(f"config4[{nx}x{ny},seed={seed}]", nx, ny, rho.reshape(ny, nx), 1.0 / eta,
                 mbb_bcs(nx, ny), H, delta, eta=eta)


def config5_densities(seed=0, n=1024, steps=50, amplitude=0.05, volume=0.5):
    """Generator of the 50-step density sequence (rho_0 .. rho_{steps-1})."""
    rng = np.random.default_rng([5, seed])
    rho = filtered_noise_density(rng, n, n, volume)
    for _ in range(steps):
        yield rho
        f = cone_filter(rng.uniform(-1.0, 1.0, size=(n, n)))
        s = (f - f.mean()) / f.std()
        rho = np.clip(rho + amplitude * s.ravel(), 0.0, 1.0)


def config5(seed=0, step=0, n=1024, H=32, delta=2, eta=1e6):
    """Step `step` of the 1024^2 topology-optimisation-style sequence."""
    for k, rho in enumerate(config5_densities(seed, n, steps=step + 1)):
        if k == step:
            return _spec(f"config5[n={n},step={step},seed={seed}]", n, n, rho.reshape(n, n),
                         1.0 / eta, cantilever_bcs(n, n), H, delta, eta=eta, step=step)
    raise ValueError("step out of range")


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
