import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
from paper_2411_14968_b200 import Engine, generate, LocalAlgo
from paper_2411_14968_b200.configs import make_config
from paper_2411_14968_b200 import abi
eng = Engine(0)
for idx, n in ((4, 400_000), (2, 1_000_000)):
    w = make_config(idx, n)
    x = generate(w.kind, w.n, w.d, 42)
    for algo in (LocalAlgo.SFS, LocalAlgo.BNL):
        w.config.local_algo = algo
        cfg = w.config.to_c(); res = abi.SkyResult()
        rc = eng._lib.sky_run(eng._h, x.ctypes.data_as(C.c_void_p), w.n, w.d, int(w.normalized), 0, C.byref(cfg), C.byref(res))
        print(idx, algo.name, 'rc', rc, 'ms', round(res.total_ms, 2), 'local', round(res.local_ms, 2), 'merge', round(res.merge_ms, 2),
              'tests l/m', res.tests_local, res.tests_merge, 'exact all', res.dom_exact_checks, 'exact merge', res.exact_checks_merge, flush=True)
        eng._lib.sky_result_free(C.byref(res))
