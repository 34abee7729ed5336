"""Convenience driver: one BASELINE config (configs.ProblemSpec) end to end."""

from __future__ import annotations

import time

import numpy as np

from .assembly import CoefficientField, ElasticityOperator
from .grid import build_coarse_partition, build_fine_mesh
from .krylov import pcg_solve
from .schwarz import EigOptions, build_preconditioner


def setup_spec(spec, tag="EH+Rot", level1="blocks", local_solver="banded", coarse_solve="inverse"):
    mesh = build_fine_mesh(spec.nx, spec.ny)
    coeff = CoefficientField(spec.E, spec.nu, spec.E_min, spec.E_max)
    op = ElasticityOperator(mesh, coeff, spec.free_dofs())
    part = build_coarse_partition(mesh, spec.Nx, spec.Ny)
    t0 = time.perf_counter()
    pre = build_preconditioner(tag, op, mesh, part, coeff, spec.heat_dirichlet_nodes, EigOptions(),
                               level1=level1, delta=spec.delta if level1 == "blocks" else None,
                               local_solver=local_solver, coarse_solve=coarse_solve)
    pre.info["t_build_wall"] = time.perf_counter() - t0
    return mesh, op, pre


def solve_spec(spec, tag="EH+Rot", level1="blocks", tol=None, maxit=None):
    mesh, op, pre = setup_spec(spec, tag, level1)
    b = spec.rhs()
    x, rep = pcg_solve(op, b, pre, tol=tol or spec.tol, maxit=maxit or spec.maxit)
    return x, rep, pre, op
