import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SKY_DEBUG_HITS"] = "1"
import numpy as np
from paper_2411_14968_b200 import Engine, generate
eng = Engine(0)
rng = np.random.default_rng(0)
for name, x in (("uniform6", rng.random((20000, 6), dtype=np.float32)), ("anti6", generate(2, 20000, 6, 1)), ("anti10", generate(4, 20000, 10, 1))):
    r = x[:5000]; c = x[5000:]
    keep = eng.relative_skyline(r, c)
    print(name, "kept", int(keep.sum()), flush=True)
