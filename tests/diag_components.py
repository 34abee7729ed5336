"""Per-kernel microbenchmark of the hot path on config 3 (GPU)."""
import json, sys
sys.path.insert(0, ".")
from paper_2006_13387_b200 import configs
from paper_2006_13387_b200.solve import setup_spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
spec = configs.config3(seed=0, n=n)
mesh, op, pre = setup_spec(spec)
print(json.dumps({"n": n, "ms": pre.bench_components(20)}))
