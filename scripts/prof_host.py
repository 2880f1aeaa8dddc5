import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_14968_b200 import Engine, generate
from paper_2411_14968_b200.configs import make_config
import torch
eng = Engine(0)
eng.set_option("profile_host", 1)
eng.set_option("kernel_events", 1)
w = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
x = generate(w.kind, w.n, w.d, 42)
xd = torch.from_numpy(x).cuda()
for i in range(3):
    t0 = time.perf_counter()
    r = eng.run(None, w.config, w.normalized, device_ptr=xd.data_ptr(), n=w.n, d=w.d)
    print(f"run {i}: wall {1e3*(time.perf_counter()-t0):.3f} ms gpu_total {r.metrics.total_ms:.3f} phases "
          f"{r.metrics.partition_ms:.3f} {r.metrics.local_ms:.3f} {r.metrics.merge_ms:.3f} dom {r.metrics.dom_kernel_ms:.3f}",
          file=sys.stderr, flush=True)
