"""Structured mesh and coarse partition metadata (host side, no compute).

Same conventions and public names as the reference (grid.py:1-223): nodes
``j*(nx+1)+i``, elements ``j*nx+i``, component-grouped dofs, coarse
neighbourhoods around interior coarse nodes in J-major order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class FineMesh:
    nx: int
    ny: int
    h: float

    @property
    def n_nodes(self):
        return (self.nx + 1) * (self.ny + 1)

    @property
    def n_elements(self):
        return self.nx * self.ny

    @property
    def n_dofs(self):
        return 2 * self.n_nodes

    def node_id(self, i, j):
        return j * (self.nx + 1) + i

    def node_coords(self):
        X, Y = np.meshgrid(np.arange(self.nx + 1) * self.h, np.arange(self.ny + 1) * self.h)
        return np.column_stack([X.ravel(), Y.ravel()])

    def element_nodes(self):
        """(n_elements, 4) corner node ids, counter-clockwise from lower-left (grid.py:40-48)."""
        jj, ii = np.divmod(np.arange(self.n_elements), self.nx)
        n0 = jj * (self.nx + 1) + ii
        return np.stack([n0, n0 + 1, n0 + self.nx + 2, n0 + self.nx + 1], axis=1)

    def boundary_nodes(self):
        jj, ii = np.divmod(np.arange(self.n_nodes), self.nx + 1)
        on = (ii == 0) | (ii == self.nx) | (jj == 0) | (jj == self.ny)
        return np.nonzero(on)[0]


def build_fine_mesh(nx, ny, h=None):
    """grid.py:68-73"""
    if nx < 1 or ny < 1:
        raise ValueError(f"element counts must be positive, got ({nx}, {ny})")
    return FineMesh(int(nx), int(ny), float(1.0 / nx if h is None else h))


@dataclass(frozen=True)
class Patch:
    """Element rectangle [ex0, ex1) x [ey0, ey1) (grid.py:76-104)."""

    ex0: int
    ex1: int
    ey0: int
    ey1: int


class CoarsePartition:
    """Coarse blocks and interior-node neighbourhoods (grid.py:107-165)."""

    def __init__(self, mesh, Nx, Ny, include_boundary=False):
        if mesh.nx % Nx != 0 or mesh.ny % Ny != 0:
            raise ValueError(f"coarse mesh {Nx}x{Ny} not nested in fine mesh {mesh.nx}x{mesh.ny}")
        if include_boundary:
            raise NotImplementedError("include_boundary=True is not part of the EH+Rot GPU path")
        self.mesh = mesh
        self.Nx, self.Ny = int(Nx), int(Ny)
        self.mex, self.mey = mesh.nx // Nx, mesh.ny // Ny
        self.include_boundary = False
        self.coarse_nodes = [(I, J) for J in range(1, Ny) for I in range(1, Nx)]
        self.neighborhoods = [
            Patch(max(0, (I - 1) * self.mex), min(mesh.nx, (I + 1) * self.mex),
                  max(0, (J - 1) * self.mey), min(mesh.ny, (J + 1) * self.mey))
            for (I, J) in self.coarse_nodes
        ]

    @property
    def n_blocks(self):
        return self.Nx * self.Ny

    @property
    def n_neighborhoods(self):
        return len(self.coarse_nodes)

    def coarse_node_coords(self, k):
        I, J = self.coarse_nodes[k]
        return (I * self.mex * self.mesh.h, J * self.mey * self.mesh.h)


def build_coarse_partition(mesh, Nx, Ny, include_boundary=False):
    return CoarsePartition(mesh, Nx, Ny, include_boundary=include_boundary)
