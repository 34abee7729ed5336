"""GPU diagnostic: iteration counts of the golden adapter cases under the GPU
path's own arithmetic variants (level-1 plain / twisted sweeps, coarse solve
by explicit inverse / Cholesky), next to the reference's measured band."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import load_golden  # noqa: E402
from paper_2006_13387_b200 import configs, pcg_solve  # noqa: E402
from paper_2006_13387_b200.solve import setup_spec  # noqa: E402

names = sys.argv[1:] or ["ref_config1.npz", "ref_config2_n128.npz", "ref_config2_n128_eta1e8.npz",
                         "ref_config5_n128_step3.npz", "ref_config5_n64_step0.npz", "ref_config3_n128.npz",
                         "ref_mbb_64x32.npz"]
for name in names:
    g = load_golden(name)
    spec = configs.ProblemSpec(name="golden", nx=int(g["nx"]), ny=int(g["ny"]), E=g["E"], E_min=float(g["E"].min()),
                               E_max=1.0, constrained_dofs=g["constrained_dofs"],
                               heat_dirichlet_nodes=g["heat_dirichlet_nodes"], load_full=g["load_full"],
                               H=int(g["H"]), delta=int(g["delta"]), nu=float(g["nu"]))
    band = np.concatenate([[int(g["iters"])], g["jitter_iters"]])
    rows = []
    for tw in ("0", "1"):
        os.environ["MS_L1_TWIST"] = tw
        for mode in ("inverse", "cholesky"):
            mesh, op, pre = setup_spec(spec, "EH+Rot", coarse_solve=mode)
            z = pre.apply(g["apply_r"])
            x, rep = pcg_solve(op, spec.rhs(), pre, tol=float(g["tol"]), maxit=20000)
            rows.append(f"tw{tw}/{mode}: {rep.iterations} x {np.linalg.norm(x - g['x']) / np.linalg.norm(g['x']):.1e} "
                        f"z {np.linalg.norm(z - g['apply_z']) / np.linalg.norm(g['apply_z']):.1e}")
    print(f"{name}: ref {int(g['iters'])} band [{band.min()}, {band.max()}] spread {g['jitter_x'].max():.1e} | "
          + " | ".join(rows), flush=True)
