"""Where the host time after the last device sync goes: the C call vs the
Python result marshalling, per run (config from argv)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_2411_14968_b200 import Engine, generate, abi
from paper_2411_14968_b200.configs import make_config
import torch
eng = Engine(0)
w = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
x = generate(w.kind, w.n, w.d, 42)
xd = torch.from_numpy(x).cuda()
cfg = w.config.to_c()
for i in range(5):
    res = abi.SkyResult()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = eng._lib.sky_run(eng._h, C.c_void_p(xd.data_ptr()), w.n, w.d, int(w.normalized), 1, C.byref(cfg), C.byref(res))
    t1 = time.perf_counter()
    r = eng._result(res, w.config)
    t2 = time.perf_counter()
    print(f"run {i}: sky_run {1e3*(t1-t0):.3f} ms (gpu_total {r.metrics.total_ms:.3f}) _result {1e3*(t2-t1):.3f} ms ids {r.skyline.size}",
          flush=True)
