"""The steps either side of the hot path, host side of
libskyline_b200.so: the reference's dataset generators (datagen.cpp:16-57,
127-151), CSV ingest with min-max normalisation (datagen.cpp:60-218) and CSV
output (datagen.cpp:220-238), pinned to fixtures produced by the reference
itself (tests/golden/make_golden.py) and, where oracle/_ref is built, live."""
import hashlib
import os

import numpy as np
import pytest

import oracle as O
from paper_2411_14968_b200 import ConfigError, DataError, IoError, generate_family, ingest_csv, normalize, write_csv
from paper_2411_14968_b200 import abi


def test_generators_match_reference_fixtures(golden):
    for g in golden["dataio"]["generate"]:
        x = generate_family(g["dist"], g["n"], g["d"], g["seed"])
        assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == g["sha256"], g
        assert x[:3].tolist() == g["head"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_generators_match_reference_live():
    for dist in (0, 1, 2):
        for d in (1, 2, 6, 11):
            assert np.array_equal(generate_family(dist, 2500, d, 1000 + d), O.ref_generate(dist, 2500, d, 1000 + d))


def test_ingest_matches_reference_fixtures(golden, tmp_path):
    err = {1: ConfigError, 3: Exception, 4: DataError, 5: IoError}
    for case in golden["dataio"]["ingest"]:
        path = tmp_path / (case["name"] + ".csv")
        path.write_bytes(case["text"].encode())
        if "error" in case:
            with pytest.raises(err[case["error"]]):
                ingest_csv(str(path), case["columns"], case["maximize"])
            continue
        got = ingest_csv(str(path), case["columns"], case["maximize"])
        assert list(got.shape) == case["shape"], case["name"]
        assert [[v.hex() for v in r] for r in got.tolist()] == case["rows_hex"], case["name"]


def test_ingest_errors(tmp_path):
    with pytest.raises(IoError):
        ingest_csv(str(tmp_path / "missing.csv"))
    p = tmp_path / "a.csv"
    p.write_text("a,b\n1,2\n")
    lib = abi.load()
    import ctypes as C
    cols = (C.c_char_p * 2)(b"a", b"b")
    flags = (C.c_uint8 * 3)(1, 0, 1)
    rows = C.POINTER(C.c_double)()
    n, d = C.c_uint64(), C.c_uint32()
    # three directions for two columns (datagen.cpp:173-175, 195-197)
    rc = lib.sky_ingest_csv(str(p).encode(), cols, 2, flags, 3, C.byref(rows), C.byref(n), C.byref(d))
    assert rc == abi.SKY_E_CONFIG and b"directions" in lib.sky_host_error()


def test_write_csv_matches_reference_bytes(golden, tmp_path):
    w = golden["dataio"]["write_csv"]
    rows = np.array([[float.fromhex(v) for v in r] for r in w["rows_hex"]])
    path = tmp_path / "w.csv"
    write_csv(str(path), rows)
    assert path.read_text() == w["text"]
    # and the round trip through ingest is exact up to the min-max rescale
    back = ingest_csv(str(path))
    assert np.array_equal(back, normalize(rows))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_ingest_live_vs_reference(tmp_path):
    rng = np.random.default_rng(8)
    x = rng.normal(size=(400, 5)) * 1e3
    x[rng.random(x.shape) < 0.01] = np.nan  # dropped rows ("nan" does not parse as finite)
    path = str(tmp_path / "r.csv")
    with open(path, "w") as f:
        f.write("c0, c1 ,c2,c3,c4\n")
        for r in x:
            f.write(",".join("" if np.isnan(v) and rng.random() < 0.5 else repr(float(v)) for v in r) + "\n")
    for cols, mx in ((None, None), (["c4", "c1"], ["c1"]), (["c2"], None)):
        assert np.array_equal(ingest_csv(path, cols, mx), O.ref_ingest_csv(path, cols, mx))
