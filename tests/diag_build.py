"""Diagnostic (not collected): build-time split (level-1 factors, eigensolves,
K0 + inverse) for config 5 (1024^2) and config 3 (2048^2)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_13387_b200 import configs
from paper_2006_13387_b200.solve import setup_spec

for name, spec in (("config5", configs.config5(seed=0, n=1024)), ("config3", configs.config3(seed=0, n=2048))):
    for rep in range(2):
        t0 = time.perf_counter()
        mesh, op, pre = setup_spec(spec)
        t = time.perf_counter() - t0
        i = pre.info
        print(name, rep, f"wall {t:.3f} s  t_level1 {i['t_level1']:.3f}  t_eig {i['t_eig']:.3f}  "
              f"t_coarse(incl eig) {i['t_coarse']:.3f}  max_passes {i.get('max_eig_passes')}  N_c {pre.coarse_dim}", flush=True)
        del pre, op
