"""GPU generation of the BASELINE inputs (sky_generate_device) against the
host generator (sky_generate, include/skyline_baseline_gen.h): identical
float32 rows, compared by SHA-256 at every BASELINE config's full size and
elementwise on small odd shapes (partial chunks, d from 1 to 16)."""
import hashlib

import numpy as np
import pytest

from paper_2411_14968_b200 import Engine, generate
from paper_2411_14968_b200.configs import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    e = Engine(0)
    yield e
    e.close()


def device_rows(eng, kind, n, d, seed):
    import torch
    t = torch.empty((n, d), dtype=torch.float32, device="cuda:0")
    torch.cuda.synchronize()
    eng.generate_device(kind, n, d, seed, t.data_ptr())
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("i", [1, 2, 3, 4, 5])
def test_full_size_matches_host(eng, i):
    w = make_config(i)
    host = generate(w.kind, w.n, w.d, 42)
    dev = device_rows(eng, w.kind, w.n, w.d, 42)
    if not np.array_equal(host, dev):
        bad = np.argwhere(host != dev)
        pytest.fail(f"config {i}: {len(bad)} values differ, first at {bad[:3].tolist()}")
    assert hashlib.sha256(dev.tobytes()).hexdigest() == hashlib.sha256(host.tobytes()).hexdigest()


@pytest.mark.parametrize("kind", [1, 2, 3, 4, 5])
def test_small_shapes(eng, kind):
    for n, d, seed in ((1, 1, 0), (65537, 3, 7), (100, 16, 9), (200000, 6, 11), (70000, 10, 5)):
        host = generate(kind, n, d, seed)
        dev = device_rows(eng, kind, n, d, seed)
        assert np.array_equal(host, dev), (kind, n, d, seed, int((host != dev).sum()))
