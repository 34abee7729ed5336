"""CPU-only checks: the C-ABI library loads and exports what include/msgpu.h
declares (no CUDA calls), the host-side API logic, config generators, and the
oracle's ARPACK eigen path against the dense reference eigenvalues."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, load_golden
from oracle import mselast_oracle as O
from paper_2006_13387_b200 import _lib, configs
import paper_2006_13387_b200 as G

HEADER = ROOT / "include" / "msgpu.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ms_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    decl = declared_functions()
    assert decl, "no declarations parsed"
    assert set(decl) == set(_lib.EXPORTS), set(decl) ^ set(_lib.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name
    m = re.search(r"#define MSGPU_ABI_VERSION (\d+)", HEADER.read_text())
    assert lib.ms_abi_version() == int(m.group(1))


def test_status_codes_map_to_reference_exceptions():
    for code, exc in ((_lib.MS_E_INVALID, ValueError), (_lib.MS_E_NOT_SPD, ValueError),
                      (_lib.MS_E_NOMEM, MemoryError), (_lib.MS_E_CUDA, RuntimeError)):
        with pytest.raises(exc):
            _lib.check(code)
    _lib.check(_lib.MS_OK)


def _c_layout(struct, fields):
    """sizeof and offsetof of an ABI struct as gcc lays it out from the header."""
    import subprocess
    import tempfile

    body = "".join(f'printf("%zu ", offsetof({struct}, {f}));' for f in fields)
    src = (f'#include <stdio.h>\n#include <stddef.h>\n#include "msgpu.h"\n'
           f'int main(void){{ {body} printf("%zu\\n", sizeof({struct})); return 0; }}\n')
    with tempfile.TemporaryDirectory() as d:
        c, exe = Path(d) / "l.c", Path(d) / "l"
        c.write_text(src)
        subprocess.run(["gcc", "-I", str(HEADER.parent), str(c), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    return [int(v) for v in out]


@pytest.mark.parametrize("cls,struct", [(_lib.PrecondOpts, "ms_precond_opts"),
                                        (_lib.PrecondInfo, "ms_precond_info"),
                                        (_lib.Report, "ms_report"),
                                        (_lib.LinOp, "ms_linop")])
def test_struct_layouts_match_header(cls, struct):
    # every field offset and the size of the ctypes mirror equal the C layout
    import ctypes as C

    names = [f for f, _ in cls._fields_]
    got = [getattr(cls, f).offset for f in names] + [C.sizeof(cls)]
    assert got == _c_layout(struct, names)


def test_duck_typed_operands_map_to_linops():
    # the reference's pcg_solve operands (krylov.py:73-78, 90) classify without touching the GPU:
    # callables -> host-callback linops, wrong types -> TypeError, bad tolerance -> ValueError
    from paper_2006_13387_b200 import krylov

    cb = krylov._HostCallback(lambda v: 2.0 * v)
    lo = cb.linop()
    assert lo.kind == _lib.MS_LINOP_CALLBACK and lo.handle is None
    src = np.arange(4.0)
    dst = np.empty(4)
    assert cb.cb(None, _lib.dptr(src), _lib.dptr(dst), 4) == 0 and np.array_equal(dst, 2.0 * src)
    bad = krylov._HostCallback(lambda v: v[:2])  # wrong shape: carried as an error, status 1
    assert bad.cb(None, _lib.dptr(src), _lib.dptr(dst), 4) == 1 and isinstance(bad.error, ValueError)
    with pytest.raises(ValueError):
        G.pcg_solve(lambda v: v, np.ones(3), tol=2.0)
    with pytest.raises(TypeError):
        krylov._as_linops("not an operator", None)


def test_unit_element_bitwise_equals_reference():
    # assembly.py:100-116 evaluated by the library (host arithmetic, no GPU):
    # all 64 doubles identical to the reference's for both Poisson ratios
    g = load_golden("ref_elements.npz")
    for nu, key in ((0.3, "Ke0_nu03"), (0.25, "Ke0_nu025")):
        K = G.element_stiffness_elasticity(1.0, nu)
        assert np.array_equal(K, g[key]), (nu, np.argwhere(K != g[key]))
    assert np.array_equal(G.element_stiffness_elasticity(2.5, 0.3), 2.5 * g["Ke0_nu03"])
    with pytest.raises(ValueError):
        G.element_stiffness_elasticity(1.0, 0.5)


def test_variant_table_and_errors():
    assert set(G.VARIANTS) == {"EE", "EE;Rand", "HH", "HH+Rot", "EH", "EH+Rot", "EH+Rot;Rand"}
    assert G.get_variant("EH+Rot").enrich and not G.get_variant("EH").enrich
    with pytest.raises(ValueError):
        G.get_variant("XX")
    assert G.EigOptions().n_max == 6


def test_grid_and_coefficient_validation():
    with pytest.raises(ValueError):
        G.build_fine_mesh(0, 3)
    mesh = G.build_fine_mesh(8, 8)
    with pytest.raises(ValueError):
        G.build_coarse_partition(mesh, 3, 3)
    part = G.build_coarse_partition(mesh, 4, 4)
    assert part.n_neighborhoods == 9 and part.mex == 2
    with pytest.raises(ValueError):
        G.CoefficientField(np.full(64, 2.0), 0.3, 0.1, 1.0)
    assert np.allclose(G.simp_modulus([0.0, 1.0], 3, 1e-3, 1.0), [1e-3, 1.0])
    with pytest.raises(ValueError):
        G.simp_modulus([1.5], 3, 1e-3, 1.0)
    f = G.build_load_vector(mesh, G.LoadSpec([(3, 1, -1.0)]))
    assert f[3 + mesh.n_nodes] == -1.0 and f.sum() == -1.0


def test_config_boundary_conditions():
    c = configs.config1(seed=0)
    nn = c.n_nodes
    # cantilever: whole left-edge nodes clamped, unit downward load at right-edge midpoint
    left = np.arange(0, nn, c.nx + 1)
    assert np.array_equal(np.sort(c.constrained_dofs), np.sort(np.concatenate([left, left + nn])))
    assert c.load_full.sum() == -1.0 and c.load_full[(c.ny // 2) * (c.nx + 1) + c.nx + nn] == -1.0
    m = configs.config4(seed=0, nx=64, ny=32, H=16)
    nn = m.n_nodes
    assert m.heat_dirichlet_nodes.size == 0
    assert (64 + nn) in m.constrained_dofs and 0 in m.constrained_dofs and nn not in m.constrained_dofs
    assert m.load_full[32 * 65 + nn] == -1.0
    assert abs(configs.config3(seed=1, n=64, H=16).meta["volume"] - 0.4) < 1e-6


def test_config5_sequence_is_seeded_and_bounded():
    seq = list(configs.config5_densities(seed=0, n=32, steps=3))
    assert len(seq) == 3 and all(0.0 <= r.min() and r.max() <= 1.0 for r in seq)
    assert not np.array_equal(seq[0], seq[1])
    seq2 = list(configs.config5_densities(seed=0, n=32, steps=3))
    assert all(np.array_equal(a, b) for a, b in zip(seq, seq2))


def test_arpack_eigen_path_matches_dense_reference():
    g = load_golden("ref_bench100_eta1e+06.npz")
    mesh = O.mesh_for(100, 100)
    part = O.Partition(mesh, 10, 10)
    for k in (0, 40, 80):
        K, M, _ = O.local_heat_problem(mesh, g["E"], part.omegas[k], g["dirichlet_nodes"])
        w, v = O.lowest_eigenpairs_arpack(K, M, 7)
        assert np.allclose(w, g["eigenvalues"][k], rtol=1e-9, atol=1e-12 * abs(g["eigenvalues"][k]).max())
        assert O.gap_count(w, 6) == g["mode_counts"][k]


def test_bench_level1_dof_count_matches_oracle_blocks():
    import bench

    spec = configs.config1(seed=0)
    mesh = O.mesh_for(spec.nx, spec.ny)
    total = 0
    for rect in O.block_rects(mesh, spec.H, spec.delta):
        a0, a1, b0, b1 = O.subdomain_node_rect(mesh, rect, True)
        total += 2 * (a1 - a0 + 1) * (b1 - b0 + 1)
    assert bench.level1_dofs(spec) == total


def test_product_path_has_no_cpu_fallback(tmp_path):
    with pytest.raises(ImportError):
        _lib.load(tmp_path / "missing.so")
    mesh = G.build_fine_mesh(4, 4)
    part = G.build_coarse_partition(mesh, 2, 2)
    coeff = G.CoefficientField(np.ones(16), 0.3, 1.0, 1.0)
    with pytest.raises(TypeError):
        G.build_preconditioner("EH+Rot", object(), mesh, part, coeff, [])
    with pytest.raises(TypeError):
        G.build_preconditioner("EE", object(), mesh, part, coeff, [])
    with pytest.raises(ValueError):
        G.build_preconditioner("XX", object(), mesh, part, coeff, [])
    assert set(G.GPU_VARIANTS) == set(G.VARIANTS)
    with pytest.raises(TypeError):
        G.pcg_solve("not an operator", np.ones(3))
    # a foreign matrix is a valid operand (krylov.py:90) and runs on the GPU: without one the
    # solve fails loudly instead of falling back to a host loop
    import torch

    if not torch.cuda.is_available():
        with pytest.raises(_lib.MsError):
            G.pcg_solve(np.eye(3), np.ones(3))


def test_topopt_host_pieces():
    """ReusePolicy validation and config defaults (topopt.py:20-56); the
    body-force load vector is bit-identical to the reference's."""
    from paper_2006_13387_b200 import topopt as T

    with pytest.raises(ValueError):
        T.ReusePolicy(period=0)
    with pytest.raises(ValueError):
        T.ReusePolicy(period=1, max_inner_iterations=0)
    c = T.OptimizeConfig()
    assert (c.nx, c.ny, c.Nx, c.Ny, c.volfrac, c.penal, c.filter_radius_factor, c.variant, c.tol, c.maxit,
            c.move_limit, c.damping, c.solver) == (60, 60, 3, 3, 0.3, 3.0, 2.5, "EH+Rot;Rand", 1e-6, 2000,
                                                   0.2, 0.5, "pcg")
    g = load_golden("ref_topopt_units.npz")
    mesh = G.build_fine_mesh(16, 16)
    assert np.array_equal(G.build_load_vector(mesh, G.LoadSpec(body_force=(0.0, -1.0))), g["sens_f"])
    with pytest.raises(ValueError):
        T.optimize(T.OptimizeConfig(solver="direct"))


@pytest.mark.parametrize("kind", ["diffusion", "elasticity"])
def test_randomized_forcings_follow_reference_dof_order(kind):
    """Forcing k is default_rng([seed, k]).uniform over the local problem's
    free dofs in the reference's order (spectral.py:119-121): nodes ascending,
    x-dofs then y-dofs for elasticity."""
    from paper_2006_13387_b200.schwarz import randomized_forcings

    mesh_o = O.mesh_for(20, 20)
    part_o = O.Partition(mesh_o, 4, 4)
    mesh = G.build_fine_mesh(20, 20)
    part = G.build_coarse_partition(mesh, 4, 4)
    clamped = np.nonzero((np.arange(mesh.n_nodes) % 21 == 0))[0]  # left edge
    F = randomized_forcings(mesh, part, clamped, 11, 5, kind)
    E = np.ones(400)
    for k in (0, 3, 8):
        if kind == "elasticity":
            K, M, pm = O.local_elasticity_problem(mesh_o, E, 0.3, part_o.omegas[k], clamped)
        else:
            K, M, pm = O.local_heat_problem(mesh_o, E, part_o.omegas[k], clamped)
        ref = np.random.default_rng([5, k]).uniform(-1.0, 1.0, size=(K.n_free, 11))
        full = np.zeros((F.shape[2], 11))
        full[K.free_dofs] = ref
        assert np.array_equal(F[k].T, full)


def test_condition_estimate_helpers_follow_reference():
    """krylov.py:38-70: the Lanczos tridiagonal is bitwise the reference's loop;
    long solves take the two extreme Ritz values by bisection, which agree with
    the full spectrum to round-off."""
    import scipy.linalg as sla

    from paper_2006_13387_b200 import krylov as K

    rng = np.random.default_rng(7)
    for k in (1, 2, 3, 40, 600, 3000):
        a = list(rng.uniform(0.05, 1.0, k))
        b = list(rng.uniform(0.0, 0.95, max(k - 1, 0)))
        d, e = K._lanczos_tridiagonal(a, b)
        dr, er = np.empty(k), np.empty(max(k - 1, 0))
        for j in range(k):  # the reference's loop
            dr[j] = 1.0 / a[j]
            if j > 0:
                dr[j] += b[j - 1] / a[j - 1]
            if j < k - 1:
                er[j] = np.sqrt(b[j]) / a[j]
        assert np.array_equal(d, dr) and np.array_equal(e, er)
        lo, hi = K._ritz_extremes(a, b)
        w = sla.eigh_tridiagonal(dr, er, eigvals_only=True) if k > 1 else dr
        assert lo == pytest.approx(w[0], rel=1e-10) and hi == pytest.approx(w[-1], rel=1e-12)
    assert K._ritz_extremes([], []) == (None, None)
    assert K._ritz_extremes([1.0, float("nan")], [0.5]) == (None, None)


def test_parallel_reference_arm_reproduces_sequential_oracle():
    """bench.py --impl reference runs the oracle on all host cores
    (oracle/parallel_ref.py): the worker-split operator and the level-1 sum
    are bit-identical to the sequential oracle (CSR rows unchanged; local
    solutions added in the reference's subdomain order)."""
    from oracle.parallel_ref import ParallelReference

    spec = configs.config3(seed=0, n=128)
    R = ParallelReference(spec, procs=3)
    try:
        prob = R.prob
        rng = np.random.default_rng(4)
        p = rng.standard_normal(R.n_free)
        assert np.array_equal(R.matvec(p), prob.op.matrix @ p)
        l1 = O.level1_solvers(prob.op, prob.mesh, O.block_rects(prob.mesh, spec.H, spec.delta), True)
        z_seq = np.zeros(R.n_free)
        for idx, solve in l1:
            z_seq[idx] += solve(p[idx])
        z_seq_full = z_seq + R.coarse.apply(p)  # coarse added last, as in schwarz.py:83
        assert np.array_equal(R.apply(p), z_seq_full)
        assert R.coarse_dim == sum(2 * m + 1 for m in R.info["mode_counts"])
    finally:
        R.close()
