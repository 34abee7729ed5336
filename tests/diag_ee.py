"""Diagnostic (not collected): EE eigenvalue/apply agreement on the bench cell."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np

import paper_2006_13387_b200 as G
from conftest import load_golden

for name, tag in [("ee_rand_eta1e+06", "EE;Rand")]:
    g = load_golden(f"ref_bench100_{name}.npz")
    mesh = G.build_fine_mesh(100, 100)
    coeff = G.CoefficientField(g["E"], 0.3, float(g["E"].min()), 1.0)
    op = G.ElasticityOperator(mesh, coeff, g["free_dofs"])
    part = G.build_coarse_partition(mesh, 10, 10)
    try:
        pre = G.build_preconditioner(tag, op, mesh, part, coeff, g["dirichlet_nodes"])
    except Exception as e:
        print(name, "build failed", e)
        continue
    lam, ref = pre.info["eigenvalues"], g["eigenvalues"]
    scale = np.abs(ref).max(axis=1, keepdims=True)
    ratio = np.abs(lam - ref) / (1e-4 * np.abs(ref) + 1e-9 * scale)
    k, j = np.unravel_index(np.argmax(ratio), ratio.shape)
    print(name, "N_c", pre.coarse_dim, int(g["coarse_dim"]), "worst", ratio.max(), "at", k, j)
    print("  gpu", lam[k]); print("  ref", ref[k])
    z = pre.apply(g["apply_r"])
    print("  apply rel", np.linalg.norm(z - g["apply_z"]) / np.linalg.norm(g["apply_z"]))
    x, rep = G.pcg_solve(op, g["b"], pre, tol=1e-8, maxit=2000)
    print("  iters", rep.iterations, int(g["iters"]), "x rel", np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]),
          "passes", pre.info["max_eig_passes"], pre.info["mean_eig_passes"])
