"""Per-launch timeline of one run (engine option `timeline`): host issue time vs
device completion time of every counted launch, for the last of 4 runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_14968_b200 import Engine, generate
from paper_2411_14968_b200.configs import make_config
import torch
eng = Engine(0)
eng.set_option("timeline", 1)
w = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
x = generate(w.kind, w.n, w.d, 42)
xd = torch.from_numpy(x).cuda()
for i in range(4):
    if i == 3:
        print("=== last run", file=sys.stderr, flush=True)
    r = eng.run(None, w.config, w.normalized, device_ptr=xd.data_ptr(), n=w.n, d=w.d)
    print(f"run {i}: gpu_total {r.metrics.total_ms:.3f}", file=sys.stderr, flush=True)
