"""Diagnostic (not collected): level-1 kernel time per launch for a variant
on config 3 (bench_components), for alternative library builds given as
arguments (MSGPU_LIB is set per subprocess)."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2006_13387_b200 import configs
    from paper_2006_13387_b200.solve import setup_spec

    tag, n = sys.argv[2], int(sys.argv[3])
    spec = configs.config3(seed=0, n=n)
    mesh, op, pre = setup_spec(spec, tag)
    c = pre.bench_components(reps=20)
    gb = (pre.info["local_bytes"]) / 1e9
    print(json.dumps({"lib": os.environ.get("MSGPU_LIB"), "tag": tag, "level1_ms": c["level1"],
                      "factor_GB": gb, "GBs": gb / (c["level1"] * 1e-3), "all": c}), flush=True)
    sys.exit(0)

tag = os.environ.get("TAG", "HH+Rot")
n = os.environ.get("N", "2048")
for lib in sys.argv[1:]:
    env = dict(os.environ, MSGPU_LIB=os.path.abspath(lib))
    subprocess.run([sys.executable, __file__, "--one", tag, n], env=env, check=False)
