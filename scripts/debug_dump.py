import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SKY_DEBUG_DUMP"] = "gpurun_out/dump_u.bin"
from paper_2411_14968_b200 import Engine, generate
from paper_2411_14968_b200.configs import make_config
os.makedirs("gpurun_out", exist_ok=True)
eng = Engine(0)
w = make_config(2, 100_000)
x = generate(w.kind, w.n, w.d, 42)
r = eng.run(x, w.config, w.normalized)
print(r.metrics.union_size, r.metrics.dom_exact_checks, r.metrics.tests_merge)
