"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU checkers.

* ``liboracle.so``      — oracle/sky_oracle.c, a plain-C restatement of the
  reference engine (each function cites the reference file:line it follows).
* ``_ref/libskyref.so`` — the reference engine itself, compiled in place from
  /root/reference by ``make -C oracle ref`` (git-ignored, travels to the GPU
  box with the snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2411_14968_b200.abi import SkyConfig

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libskyref.so")


class _OracleResult(C.Structure):
    _fields_ = [
        ("ids", C.POINTER(C.c_int64)),
        ("n_ids", C.c_uint64),
        ("effective_p", C.c_uint64),
        ("union_size", C.c_uint64),
        ("filtered_count", C.c_uint64),
        ("final_size", C.c_uint64),
        ("n_reps", C.c_uint64),
        ("local_skyline_sizes", C.POINTER(C.c_uint64)),
        ("tests_reps", C.c_uint64),
        ("tests_local", C.c_uint64),
        ("tests_merge", C.c_uint64),
    ]


class _RefResult(C.Structure):
    _fields_ = [
        ("ids", C.POINTER(C.c_int64)),
        ("n_ids", C.c_uint64),
        ("effective_p", C.c_uint64),
        ("union_size", C.c_uint64),
        ("filtered_count", C.c_uint64),
        ("final_size", C.c_uint64),
        ("n_reps", C.c_uint64),
        ("local_skyline_sizes", C.POINTER(C.c_uint64)),
        ("partition_ms", C.c_double),
        ("local_ms", C.c_double),
        ("merge_ms", C.c_double),
        ("run_ms", C.c_double),
    ]


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle [ref]). The reference build needs
    /root/reference, which exists only in the build container."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


_oracle = None
_ref = None
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(_f32p)


def _rows(a):
    """(array, pointer, is_f64): float64 arrays stay FP64 (the reference's
    own coordinate type), anything else becomes float32."""
    if np.asarray(a).dtype == np.float64:
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.ndim == 1:
            a = a.reshape(-1, 1) if a.size else a.reshape(0, 0)
        return a, a.ctypes.data_as(_f64p), True
    a, p = _f32(a)
    return a, p, False


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_run.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(SkyConfig), C.POINTER(_OracleResult)]
        lib.oracle_run_f64.argtypes = [_f64p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(SkyConfig),
                                       C.POINTER(_OracleResult)]
        lib.oracle_result_free.argtypes = [C.POINTER(_OracleResult)]
        lib.oracle_assign.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(SkyConfig), _u64p, _u64p]
        lib.oracle_bruteforce.argtypes = [_f32p, C.c_uint64, C.c_uint32, _i64p]
        lib.oracle_bruteforce.restype = C.c_uint64
        lib.oracle_relative_skyline.argtypes = [_f32p, C.c_uint64, _f32p, C.c_uint64, C.c_uint32, _u8p]
        lib.oracle_snap_slices.argtypes = [C.c_uint64, C.c_uint64]
        lib.oracle_snap_slices.restype = C.c_uint64
        lib.oracle_angular_index.argtypes = [_f32p, C.c_uint32, C.c_uint64]
        lib.oracle_angular_index.restype = C.c_uint64
        lib.oracle_grid_index.argtypes = [_f32p, C.c_uint32, C.c_uint64]
        lib.oracle_grid_index.restype = C.c_uint64
        lib.oracle_random_permutation.argtypes = [C.c_uint64, C.c_uint64, _u64p]
        lib.oracle_representatives.argtypes = [_f32p, C.c_uint64, C.c_uint32, _u64p, C.c_uint64, C.c_uint64, _i64p]
        lib.oracle_representatives.restype = C.c_uint64
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(REF_SO)
        lib.skyref_run.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(SkyConfig), C.POINTER(_RefResult)]
        lib.skyref_run_f64.argtypes = [_f64p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(SkyConfig),
                                       C.POINTER(_RefResult)]
        lib.skyref_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _f64p]
        lib.skyref_ingest_csv.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_uint32, _u8p, C.c_uint32,
                                          C.POINTER(_f64p), _u64p, C.POINTER(C.c_uint32)]
        lib.skyref_write_csv.argtypes = [C.c_char_p, _f64p, C.c_uint64, C.c_uint32]
        lib.skyref_free.argtypes = [C.c_void_p]
        lib.skyref_result_free.argtypes = [C.POINTER(_RefResult)]
        lib.skyref_assign.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(SkyConfig), _u64p, _u64p]
        lib.skyref_bruteforce.argtypes = [_f32p, C.c_uint64, C.c_uint32, _i64p]
        lib.skyref_bruteforce.restype = C.c_uint64
        lib.skyref_sfs.argtypes = [_f32p, C.c_uint64, C.c_uint32, _i64p]
        lib.skyref_sfs.restype = C.c_uint64
        lib.skyref_relative_skyline.argtypes = [_f32p, C.c_uint64, _f32p, C.c_uint64, C.c_uint32, _u8p]
        lib.skyref_snap_slices.argtypes = [C.c_uint64, C.c_uint64]
        lib.skyref_snap_slices.restype = C.c_uint64
        lib.skyref_angular_index.argtypes = [_f32p, C.c_uint32, C.c_uint64]
        lib.skyref_angular_index.restype = C.c_uint64
        lib.skyref_grid_index.argtypes = [_f32p, C.c_uint32, C.c_uint64]
        lib.skyref_grid_index.restype = C.c_uint64
        lib.skyref_representatives.argtypes = [_f32p, C.c_uint64, C.c_uint32, _u64p, C.c_uint64, C.c_uint64, _i64p]
        lib.skyref_representatives.restype = C.c_uint64
        lib.skyref_hardware_concurrency.restype = C.c_int
        lib.skyref_generate_baseline.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, _f32p]
        _ref = lib
    return _ref


class CpuRun(dict):
    """Result of a CPU run: ids (np.int64), metrics, optional timings."""


def _to_run(res, p_count, extra):
    out = CpuRun()
    out["ids"] = np.ctypeslib.as_array(res.ids, shape=(res.n_ids,)).copy() if res.n_ids else np.zeros(0, np.int64)
    out["effective_p"] = int(res.effective_p)
    out["union_size"] = int(res.union_size)
    out["filtered_count"] = int(res.filtered_count)
    out["final_size"] = int(res.final_size)
    out["local_skyline_sizes"] = (
        np.ctypeslib.as_array(res.local_skyline_sizes, shape=(p_count,)).copy() if p_count else np.zeros(0, np.uint64)
    )
    out.update(extra)
    return out


class CpuError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"status {code}")
        self.code = code


def oracle_run(points, cfg: SkyConfig, normalized: bool = True) -> CpuRun:
    lib = oracle_lib()
    a, p, f64 = _rows(points)
    n, d = a.shape
    res = _OracleResult()
    rc = (lib.oracle_run_f64 if f64 else lib.oracle_run)(p, n, d, int(normalized), C.byref(cfg), C.byref(res))
    if rc:
        raise CpuError(rc)
    try:
        return _to_run(res, res.effective_p, {
            "n_reps": int(res.n_reps), "tests_reps": int(res.tests_reps),
            "tests_local": int(res.tests_local), "tests_merge": int(res.tests_merge)})
    finally:
        lib.oracle_result_free(C.byref(res))


def ref_run(points, cfg: SkyConfig, normalized: bool = True) -> CpuRun:
    lib = ref_lib()
    a, p, f64 = _rows(points)
    n, d = a.shape
    res = _RefResult()
    rc = (lib.skyref_run_f64 if f64 else lib.skyref_run)(p, n, d, int(normalized), C.byref(cfg), C.byref(res))
    if rc:
        raise CpuError(rc)
    try:
        return _to_run(res, res.effective_p, {
            "partition_ms": res.partition_ms, "local_ms": res.local_ms,
            "merge_ms": res.merge_ms, "run_ms": res.run_ms})
    finally:
        lib.skyref_result_free(C.byref(res))


def oracle_assign(points, cfg: SkyConfig, normalized=True, ref=False):
    lib = ref_lib() if ref else oracle_lib()
    fn = lib.skyref_assign if ref else lib.oracle_assign
    a, p = _f32(points)
    n, d = a.shape
    out = np.zeros(max(n, 1), np.uint64)
    cnt = C.c_uint64(0)
    rc = fn(p, n, d, int(normalized), C.byref(cfg), out.ctypes.data_as(_u64p), C.byref(cnt))
    if rc:
        raise CpuError(rc)
    return out[:n], int(cnt.value)


def bruteforce(points, ref=False):
    lib = ref_lib() if ref else oracle_lib()
    fn = lib.skyref_bruteforce if ref else lib.oracle_bruteforce
    a, p = _f32(points)
    n, d = a.shape
    out = np.zeros(max(n, 1), np.int64)
    k = fn(p, n, d, out.ctypes.data_as(_i64p))
    return out[:k]


def relative_skyline(r, c, ref=False):
    lib = ref_lib() if ref else oracle_lib()
    fn = lib.skyref_relative_skyline if ref else lib.oracle_relative_skyline
    ra, rp = _f32(r)
    ca, cp = _f32(c)
    keep = np.zeros(max(len(ra), 1), np.uint8)
    fn(rp, len(ra), cp, len(ca), ra.shape[1], keep.ctypes.data_as(_u8p))
    return keep[: len(ra)].astype(bool)


def representatives(points, partition_of, p, q, ref=False):
    lib = ref_lib() if ref else oracle_lib()
    fn = lib.skyref_representatives if ref else lib.oracle_representatives
    a, ap = _f32(points)
    n, d = a.shape
    po = np.ascontiguousarray(partition_of, dtype=np.uint64)
    out = np.zeros(max(n, 1), np.int64)
    k = fn(ap, n, d, po.ctypes.data_as(_u64p), p, q, out.ctypes.data_as(_i64p))
    return out[:k]


def random_permutation(n, seed):
    out = np.zeros(max(n, 1), np.uint64)
    oracle_lib().oracle_random_permutation(n, seed, out.ctypes.data_as(_u64p))
    return out[:n]


def ref_generate_baseline(kind: int, n: int, d: int, seed: int = 42) -> np.ndarray:
    """BASELINE.json input `kind` (1..5) as float32 n x d, built inside
    oracle/_ref/libskyref.so from include/skyline_baseline_gen.h — the same
    bytes as the product's sky_generate, without loading the product."""
    out = np.empty((n, d), np.float32)
    rc = ref_lib().skyref_generate_baseline(kind, n, d, seed, out.ctypes.data_as(_f32p))
    if rc:
        raise CpuError(rc)
    return out


def ref_generate(dist: int, n: int, d: int, seed: int) -> np.ndarray:
    """skyline::generate (datagen.cpp:127-151) of the reference itself:
    dist 0 uniform, 1 correlated, 2 anticorrelated; FP64 rows."""
    out = np.zeros((n, d), np.float64)
    rc = ref_lib().skyref_generate(dist, n, d, seed, out.ctypes.data_as(_f64p))
    if rc:
        raise CpuError(rc)
    return out


def ref_ingest_csv(path: str, columns=None, maximize=None) -> np.ndarray:
    """skyline::ingest_csv of the reference itself (raises CpuError)."""
    lib = ref_lib()
    cols = list(columns or [])
    arr = (C.c_char_p * max(1, len(cols)))(*[c.encode() for c in cols])
    mx = list(maximize or [])
    flags = np.array([1 if c in mx else 0 for c in cols], np.uint8) if mx else np.zeros(1, np.uint8)
    rows = _f64p()
    n = C.c_uint64(0)
    d = C.c_uint32(0)
    rc = lib.skyref_ingest_csv(path.encode(), arr, len(cols), flags.ctypes.data_as(_u8p), len(cols) if mx else 0,
                               C.byref(rows), C.byref(n), C.byref(d))
    if rc:
        raise CpuError(rc)
    try:
        return np.ctypeslib.as_array(rows, shape=(n.value, d.value)).copy()
    finally:
        lib.skyref_free(rows)


def ref_write_csv(path: str, rows) -> None:
    a = np.ascontiguousarray(rows, dtype=np.float64)
    rc = ref_lib().skyref_write_csv(path.encode(), a.ctypes.data_as(_f64p), a.shape[0], a.shape[1])
    if rc:
        raise CpuError(rc)
