import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_14968_b200 import Engine, generate
from paper_2411_14968_b200.configs import make_config
eng = Engine(0)
w = make_config(int(sys.argv[1]))
x = generate(w.kind, w.n, w.d, 42)
r = eng.run(x, w.config, w.normalized)
ls = np.array(r.metrics.local_skyline_sizes)
print("P", len(ls), "U", ls.sum(), "min", ls.min(), "mean", round(ls.mean(), 1), "max", ls.max(), "top5", np.sort(ls)[-5:], "argmax", ls.argmax())
print("sizes head", ls[:8], "tail", ls[-8:])
