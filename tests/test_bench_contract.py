"""bench.py contract checks that run without a GPU.

* `--impl reference` runs the reference's own CPU engine (oracle/_ref) and
  must not load the product library (its input comes from the generator
  compiled into oracle/_ref).
* Both arms emit the same `config` object.
"""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_loads_only_the_reference():
    code = r'''
import json, sys
sys.argv = ["bench.py", "--impl", "reference", "--config", "1", "--n", "20000", "--steps", "1", "--warmup", "0"]
import bench
bench.run_reference_arm(bench.parse())
maps = open("/proc/self/maps").read()
print("MAPS", json.dumps(sorted({l.split()[-1] for l in maps.splitlines() if l.endswith(".so")})))
'''
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    libs = json.loads(lines[-1][len("MAPS "):])
    assert not any("libskyline_b200" in p for p in libs), libs
    assert any(p.endswith("oracle/_ref/libskyref.so") for p in libs), libs


def test_config_object_identical_in_both_arms():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2411_14968_b200.configs import make_config
    for i in range(1, 6):
        w = make_config(i)
        c = bench.bench_config(w)
        assert set(c) == {"workload", "n", "d", "description", "l2"}
        assert c == bench.bench_config(make_config(i))
