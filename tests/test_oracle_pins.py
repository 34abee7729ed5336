"""Pin the CPU oracle against outputs of the unmodified reference.

The fixtures in tests/golden/ were produced by tests/golden/make_golden.py,
which runs the reference package itself.  These tests need no GPU.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import mselast_oracle as O
from paper_2006_13387_b200 import configs


def test_element_matrices_bitwise():
    g = load_golden("ref_elements.npz")
    assert np.array_equal(O.elasticity_element(0.3), g["Ke0_nu03"])
    assert np.array_equal(O.elasticity_element(0.25), g["Ke0_nu025"])
    assert np.array_equal(O.laplace_element(), g["lap"])
    assert np.array_equal(O.mass_element(0.01), g["mass_h001"])


def _bench_problem(g):
    mesh = O.mesh_for(100, 100)
    op = O.elasticity_operator(mesh, g["E"], 0.3, O.whole_node_dofs(mesh, g["dirichlet_nodes"]))
    assert np.array_equal(op.free_dofs, g["free_dofs"])
    return O.OracleProblem(mesh, op, g["E"], 0.3, g["b"], g["dirichlet_nodes"])


@pytest.mark.parametrize("eta", ["1", "1e+06"])
def test_reference_benchmark_cell(eta):
    """Reference semantics (subdomains = omega_j), 100^2/10^2, EH+Rot."""
    g = load_golden(f"ref_bench100_eta{eta}.npz")
    prob = _bench_problem(g)
    P = O.build_two_level(prob, H=10, level1_mode="neighborhoods")
    assert P.coarse_dim == int(g["coarse_dim"])
    assert np.array_equal(np.array(P.info["mode_counts"]), g["mode_counts"])
    lam = np.array(P.coarse_space.eigenvalues)
    assert np.allclose(lam, g["eigenvalues"], rtol=1e-12, atol=1e-12 * np.abs(g["eigenvalues"]).max())
    z = P.apply(g["apply_r"])
    assert np.linalg.norm(z - g["apply_z"]) <= 1e-13 * np.linalg.norm(g["apply_z"])
    for tol in ("1e-06", "1e-08"):
        x, rep = O.pcg(prob.op.matrix, prob.b, P, tol=float(tol), maxit=2000)
        assert rep.iterations == int(g[f"iters_{tol}"])
        xr = g[f"x_{tol}"]
        assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)
        assert rep.cond_estimate == pytest.approx(float(g[f"cond_{tol}"]), rel=1e-8)


def _adapter_check(name, apply_only=False, level1_op="elasticity"):
    g = load_golden(name)
    spec = configs.ProblemSpec(
        name=name, nx=int(g["nx"]), ny=int(g["ny"]), E=g["E"], E_min=float(g["E"].min()),
        E_max=1.0, constrained_dofs=g["constrained_dofs"],
        heat_dirichlet_nodes=g["heat_dirichlet_nodes"], load_full=g["load_full"],
        H=int(g["H"]), delta=int(g["delta"]), nu=float(g["nu"]))
    prob = O.problem_from_spec(spec)
    P = O.build_two_level(prob, H=spec.H, delta=spec.delta, level1_mode="blocks", level1_op=level1_op)
    assert P.coarse_dim == int(g["coarse_dim"])
    assert np.array_equal(np.array(P.info["mode_counts"]), g["mode_counts"])
    assert np.allclose(P.coarse.K0, g["K0"], rtol=0, atol=1e-13 * np.abs(g["K0"]).max())
    z = P.apply(g["apply_r"])
    assert np.linalg.norm(z - g["apply_z"]) <= 1e-12 * np.linalg.norm(g["apply_z"])
    if apply_only:
        return
    x, rep = O.pcg(prob.op.matrix, prob.b, P, tol=float(g["tol"]), maxit=5000)
    assert rep.iterations == int(g["iters"])
    assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])


def test_config1_adapter_matches_reference_composition():
    _adapter_check("ref_config1.npz")


def test_mbb_componentwise_adapter_matches_reference_composition():
    _adapter_check("ref_mbb_64x32.npz")


def test_gap_rule_examples():
    # spectral.py:161-186 semantics
    assert O.gap_count([0.0, 1.0, 1.1, 2.0, 3.0, 4.0, 5.0], 6) == 1
    assert O.gap_count([1e-6, 2e-6, 1.0, 2.0, 3.0, 4.0, 5.0], 6) == 2
    assert O.gap_count([1e-8, 1e-6, 1e-4, 1e-2, 1.0, 1e2, 1e4], 6) == 6
    assert O.gap_count([1.0, 2.0], 6) == 1


def test_configs_are_deterministic():
    a = configs.config1(seed=3)
    b = configs.config1(seed=3)
    assert np.array_equal(a.E, b.E)
    c = configs.config3(seed=0, n=64, H=16)
    assert abs(c.meta["volume"] - 0.4) < 1e-6
    assert c.E.min() >= 1e-6 - 1e-18 and c.E.max() <= 1.0


@pytest.mark.parametrize("eta", ["1", "1e+06"])
def test_randomized_variant_matches_reference(eta):
    """EH+Rot;Rand: the oracle's restatement of solve_local_eig_randomized
    (spectral.py:103-158, seeds [0, centre]) reproduces the reference."""
    g = load_golden(f"ref_bench100_rand_eta{eta}.npz")
    mesh = O.mesh_for(100, 100)
    op = O.elasticity_operator(mesh, g["E"], 0.3, O.whole_node_dofs(mesh, g["dirichlet_nodes"]))
    prob = O.OracleProblem(mesh, op, g["E"], 0.3, g["b"], g["dirichlet_nodes"])
    P = O.build_two_level(prob, H=10, level1_mode="neighborhoods", eig_solver=O.randomized_solver())
    lam = np.array(P.coarse_space.eigenvalues)
    assert np.allclose(lam, g["eigenvalues"], rtol=1e-10, atol=1e-12 * np.abs(g["eigenvalues"]).max())
    assert P.coarse_dim == int(g["coarse_dim"])
    assert np.array_equal(np.array(P.info["mode_counts"]), g["mode_counts"])
    z = P.apply(g["apply_r"])
    assert np.linalg.norm(z - g["apply_z"]) <= 1e-12 * np.linalg.norm(g["apply_z"])
    x, rep = O.pcg(prob.op.matrix, prob.b, P, tol=1e-8, maxit=2000)
    assert rep.iterations == int(g["iters"])
    assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])


@pytest.mark.parametrize("name,enrich", [("ref_bench100_hhrot_eta1.npz", True),
                                         ("ref_bench100_hhrot_eta1e+06.npz", True),
                                         ("ref_bench100_hh_eta1e+06.npz", False)])
def test_heat_level1_variants_match_reference(name, enrich):
    """HH / HH+Rot (schwarz.py:112-140): scalar level-1 factor on both blocks."""
    g = load_golden(name)
    mesh = O.mesh_for(100, 100)
    op = O.elasticity_operator(mesh, g["E"], 0.3, O.whole_node_dofs(mesh, g["dirichlet_nodes"]))
    prob = O.OracleProblem(mesh, op, g["E"], 0.3, g["b"], g["dirichlet_nodes"])
    P = O.build_two_level(prob, H=10, level1_mode="neighborhoods", enrich=enrich, level1_op="heat")
    assert P.coarse_dim == int(g["coarse_dim"])
    assert np.array_equal(np.array(P.info["mode_counts"]), g["mode_counts"])
    r = g["apply_r"]
    assert np.linalg.norm(P.level1_apply(r) - g["level1_z"]) <= 1e-13 * np.linalg.norm(g["level1_z"])
    assert np.linalg.norm(P.apply(r) - g["apply_z"]) <= 1e-12 * np.linalg.norm(g["apply_z"])
    x, rep = O.pcg(prob.op.matrix, prob.b, P, tol=1e-8, maxit=2000)
    assert rep.iterations == int(g["iters"])
    assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])


def test_config1_heat_level1_adapter_matches_reference_composition():
    _adapter_check("ref_config1_hhrot.npz", level1_op="heat")


# ---------------------------------------------------------------------------
# SIMP caller (row f2)


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_cone_filter_bitwise(tag):
    g = load_golden("ref_topopt_units.npz")
    nx, ny = g[f"filt_{tag}_shape"]
    filt = O.ConeFilter(O.mesh_for(int(nx), int(ny)), float(g[f"filt_{tag}_radius"]))
    assert np.array_equal(filt.apply(g[f"filt_{tag}_x"]), g[f"filt_{tag}_Wx"])
    assert np.array_equal(filt.adjoint(g[f"filt_{tag}_v"]), g[f"filt_{tag}_WTv"])


def test_sensitivity_and_oc_units():
    g = load_golden("ref_topopt_units.npz")
    mesh = O.mesh_for(16, 16)
    assert np.array_equal(O.body_force_load(mesh, 0.0, -1.0), g["sens_f"])
    assert np.array_equal(O.simp(g["sens_rho"], 3.0, 1e-6, 1.0), g["sens_E"])
    g0, sens = O.compliance_and_sensitivity(mesh, g["sens_u"], g["sens_f"], g["sens_rho"], 3.0, 1e-6, 1.0, 0.3)
    assert g0 == pytest.approx(float(g["sens_g0"]), rel=1e-14)
    assert np.allclose(sens, g["sens_sens"], rtol=1e-13, atol=0)
    new = O.oc_update(g["oc_rho"], g["oc_dg"], g["oc_vol"], float(g["oc_vstar"]), move=0.15)
    assert np.array_equal(new, g["oc_new"])
    filt = O.ConeFilter(O.mesh_for(30, 20), 2.5 / 30)
    new = O.oc_update(g["ocf_rho"], g["ocf_dg"], g["ocf_vol"], float(g["ocf_vstar"]), filt=filt)
    assert np.array_equal(new, g["ocf_new"])
    with pytest.raises(RuntimeError):
        O.oc_update(np.full(20, 0.9), np.full(20, -1.0), np.ones(20), 2.0, move=0.01)


@pytest.mark.parametrize("name,variant", [("ehrot", "EH+Rot"), ("rand_reuse3", "EH+Rot;Rand"),
                                          ("hhrot_thresh", "HH+Rot")])
def test_optimize_loop_matches_reference(name, variant):
    g = load_golden(f"ref_topopt_{name}.npz")
    mi = int(g["max_inner"])
    rho, rho_f, log, rebuilds = O.optimize(nx=40, ny=40, Nx=4, Ny=4, n_iterations=6, volfrac=0.3,
                                           variant=variant, tol=1e-8, period=int(g["period"]),
                                           max_inner=mi or None)
    assert [r["rebuilt"] for r in log] == list(g["rebuilt"]) and rebuilds == int(g["rebuilds"])
    assert [r["inner_iterations"] for r in log] == list(g["inner"])
    assert np.allclose([r["g0"] for r in log], g["g0"], rtol=1e-10, atol=0)
    assert np.allclose(rho, g["rho"], rtol=0, atol=1e-9)


@pytest.mark.parametrize("name", ["ee_eta1", "ee_eta1e+06", "ee_rand_eta1", "ee_rand_eta1e+06"])
def test_elasticity_eigen_variants_match_reference(name):
    """EE / EE;Rand (row f4): elasticity eigenproblems, rule 'fixed'."""
    g = load_golden(f"ref_bench100_{name}.npz")
    mesh = O.mesh_for(100, 100)
    op = O.elasticity_operator(mesh, g["E"], 0.3, O.whole_node_dofs(mesh, g["dirichlet_nodes"]))
    prob = O.OracleProblem(mesh, op, g["E"], 0.3, g["b"], g["dirichlet_nodes"])
    eig = O.randomized_solver() if "rand" in name else None
    P = O.build_two_level(prob, H=10, level1_mode="neighborhoods", eig_kind="elasticity", eig_solver=eig)
    assert P.coarse_dim == int(g["coarse_dim"])
    assert np.array_equal(np.array(P.info["mode_counts"]), g["mode_counts"])
    lam = np.array(P.coarse_space.eigenvalues)
    scale = np.abs(g["eigenvalues"]).max()
    assert np.allclose(lam, g["eigenvalues"], rtol=1e-9, atol=1e-12 * scale)
    z = P.apply(g["apply_r"])
    assert np.linalg.norm(z - g["apply_z"]) <= 1e-11 * np.linalg.norm(g["apply_z"])
    x, rep = O.pcg(prob.op.matrix, prob.b, P, tol=1e-8, maxit=2000)
    assert rep.iterations == int(g["iters"])
    assert np.linalg.norm(x - g["x"]) <= 1e-9 * np.linalg.norm(g["x"])

