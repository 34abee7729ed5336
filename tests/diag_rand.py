import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import load_golden
import paper_2006_13387_b200 as G
g = load_golden("ref_bench100_rand_eta1e+06.npz")
mesh = G.build_fine_mesh(100, 100)
coeff = G.CoefficientField(g["E"], 0.3, float(g["E"].min()), 1.0)
op = G.ElasticityOperator(mesh, coeff, g["free_dofs"])
part = G.build_coarse_partition(mesh, 10, 10)
pre = G.build_preconditioner("EH+Rot;Rand", op, mesh, part, coeff, g["dirichlet_nodes"])
lam, ref = pre.info["eigenvalues"], g["eigenvalues"]
rel = np.abs(lam - ref) / np.abs(ref)
print("coarse", pre.coarse_dim, g["coarse_dim"], "modes equal", np.array_equal(np.array(pre.mode_counts), g["mode_counts"]))
bad = np.argsort(-rel.max(axis=1))[:6]
np.set_printoptions(precision=10, linewidth=200)
for k in bad:
    print(k, rel[k].max(), "\n gpu", lam[k], "\n ref", ref[k])
print("nan rows", np.nonzero(np.isnan(lam).any(axis=1))[0])
scale = np.abs(ref).max(axis=1, keepdims=True)
badm = ~(np.abs(lam - ref) <= 1e-7 * np.abs(ref) + 1e-10 * scale)
for k in np.nonzero(badm.any(axis=1))[0][:5]:
    print("fail", k, "\n gpu", lam[k], "\n ref", ref[k])
