"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only entry points behave (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np

from paper_2411_14968_b200 import abi, generate, plan_lpt, plan_split, snap_slices

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = abi.load()
    with open(os.path.join(ROOT, "include", "skyline_b200.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"SKY_API\s+[\w\s\*]+?\b(sky_\w+)\s*\(", hdr))
    assert declared == set(abi.EXPORTED), declared ^ set(abi.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.sky_abi_version() == 3


def test_config_struct_layout_matches_header():
    # offsets of the C struct as compiled by gcc, via a tiny C probe
    import subprocess
    import tempfile
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "skyline_b200.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(sky_config), offsetof(sky_config, rep_q),
        offsetof(sky_config, count_tests), sizeof(sky_result), offsetof(sky_result, kernel_launches),
        offsetof(sky_result, stream_kernel_ms), offsetof(sky_result, stream_bytes));
 return 0;}
'''
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "probe.c")
        open(p, "w").write(src)
        exe = os.path.join(td, "probe")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), p, "-o", exe], check=True)
        vals = list(map(int, subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()))
    assert vals == [C.sizeof(abi.SkyConfig), abi.SkyConfig.rep_q.offset, abi.SkyConfig.count_tests.offset,
                    C.sizeof(abi.SkyResult), abi.SkyResult.kernel_launches.offset,
                    abi.SkyResult.stream_kernel_ms.offset, abi.SkyResult.stream_bytes.offset]


def test_snap_slices_known_answers():
    # test_partition.cpp:228-234
    assert snap_slices(16, 4) == 2
    assert snap_slices(120, 4) == 3
    assert snap_slices(120, 3) == 5
    assert snap_slices(120, 2) == 11
    assert snap_slices(120, 1) == 120
    assert snap_slices(1, 3) == 1
    assert snap_slices(64, 5) == 2  # config 2: 64 angular partitions at d=6 -> m=2 (32 cells)


def test_generators_deterministic_and_in_spec():
    for kind, d in ((1, 4), (2, 6), (3, 8), (4, 10), (5, 5)):
        a = generate(kind, 70_000, d, 42)
        b = generate(kind, 70_000, d, 42)
        assert np.array_equal(a, b)
        assert not np.array_equal(a, generate(kind, 70_000, d, 43))
        assert a.dtype == np.float32 and a.shape == (70_000, d)
        assert np.isfinite(a).all() and (a >= 0).all()
        if kind == 5:
            assert set(np.unique(a).tolist()) <= set(float(v) for v in range(16))
        else:
            assert (a <= 1).all()
        if kind == 1:
            assert (a < 1).all()
        if kind in (2, 4):
            # |sum(x) - d s| <= 0.01 d with s ~ N(0.5, 0.0625): sums concentrate near d/2
            s = a.astype(np.float64).sum(1)
            assert abs(s.mean() - d / 2) < 0.05 * d
            assert np.corrcoef(a[:, 0], a[:, 1])[0, 1] < 0


def test_plan_helpers():
    w = np.array([10, 1, 7, 3, 3, 9], np.uint64)
    owner = plan_lpt(w, 3)
    loads = [int(w[owner == r].sum()) for r in range(3)]
    assert sorted(loads) == [10, 11, 12] or max(loads) - min(loads) <= 3
    b = plan_split(np.ones(100, np.uint64), 4)
    assert b.tolist() == [0, 25, 50, 75, 100]
    b = plan_split(np.arange(10, dtype=np.uint64), 2)
    assert b[0] == 0 and b[-1] == 10 and 0 < b[1] < 10
