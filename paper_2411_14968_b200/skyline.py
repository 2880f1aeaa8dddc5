"""Host-side mirror of the reference engine API (reference
proj/include/skyline/{engine,partition,filter,core}.hpp) over the C ABI.

Names, argument meanings and error behaviour follow the reference:

    reference (C++)                          here
    ---------------------------------------  ----------------------------------
    skyline::Strategy        partition.hpp:14  Strategy
    skyline::PartitionConfig partition.hpp:21  PartitionConfig
    skyline::FilterKind      engine.hpp:19     FilterKind
    skyline::RepSelection    filter.hpp:21     RepSelection
    skyline::MergeKind       engine.hpp:25     MergeKind
    skyline::EngineConfig    engine.hpp:30     EngineConfig (+ local_algo, bnl_window_cap)
    skyline::PhaseMetrics    engine.hpp:40     PhaseMetrics
    skyline::RunResult       engine.hpp:50     RunResult
    skyline::run             engine.hpp:88     Engine.run / run
    skyline::make_assignment partition.hpp:102 Engine.make_assignment
    skyline::snap_slices     partition.hpp:99  snap_slices
    skyline::relative_skyline core.hpp:79      Engine.relative_skyline
    skyline::sfs             sequential.hpp:29 Engine.sfs
    select_representatives_sorted filter.hpp:46 Engine.select_representatives_sorted
    SkylineError hierarchy   core.hpp:13-34    SkylineError, ConfigError, ...

Every call runs on the GPU through libskyline_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi


# ----------------------------------------------------------------- errors
class SkylineError(RuntimeError):
    code = 12


class ConfigError(SkylineError):
    code = 1


class DimensionError(SkylineError):
    code = 2


class NormalizationError(SkylineError):
    code = 3


class DataError(SkylineError):
    code = 4


class IoError(SkylineError):
    code = 5


class CudaError(SkylineError):
    code = 10


class NcclError(SkylineError):
    code = 11


_ERRORS = {1: ConfigError, 2: DimensionError, 3: NormalizationError, 4: DataError, 5: IoError,
           10: CudaError, 11: NcclError, 12: SkylineError}


def _raise(rc: int, msg: str = ""):
    if rc != abi.SKY_OK:
        raise _ERRORS.get(rc, SkylineError)(msg or abi.STATUS_NAMES.get(rc, str(rc)))


# ------------------------------------------------------------------ enums
class Strategy(enum.IntEnum):
    Random = 0
    Grid = 1
    Angular = 2
    Sliced = 3


class FilterKind(enum.IntEnum):
    None_ = 0
    GridFilter = 1
    Representative = 2


class RepSelection(enum.IntEnum):
    Sorted = 0
    Region = 1
    Random = 2


class MergeKind(enum.IntEnum):
    Sequential = 0
    NoSeq = 1


class LocalAlgo(enum.IntEnum):
    SFS = 0
    BNL = 1


@dataclass
class PartitionConfig:
    strategy: Strategy = Strategy.Random
    p: int = 1
    m: int = 0
    seed: int = 0
    slice_dim: int = 0


_RF = abi.SKY_RESULT_FIELDS
_ZERO_COPY_IDS = 1 << 16  # ids from which RunResult.skyline is a view of the library's buffer


class _ResultOwner:
    """Keeps a sky_result alive for the arrays that view its buffers."""

    def __init__(self, lib, res):
        self._lib = lib
        self._res = res

    def __del__(self):
        try:
            self._lib.sky_result_free(C.byref(self._res))
        except Exception:
            pass


@dataclass
class EngineConfig:
    partition: PartitionConfig = field(default_factory=PartitionConfig)
    filter: FilterKind = FilterKind.None_
    rep_selection: RepSelection = RepSelection.Sorted
    rep_q: int = 5
    merge: MergeKind = MergeKind.Sequential
    workers: int = 1
    seed: int = 0
    local_algo: LocalAlgo = LocalAlgo.SFS
    bnl_window_cap: int = 4096
    count_tests: bool = True

    def to_c(self) -> abi.SkyConfig:
        p = self.partition
        return abi.SkyConfig.make(
            strategy=int(p.strategy), p=int(p.p), m=int(p.m), seed=int(p.seed), slice_dim=int(p.slice_dim),
            filter=int(self.filter), rep_selection=int(self.rep_selection), rep_q=int(self.rep_q),
            merge=int(self.merge), workers=int(self.workers), local_algo=int(self.local_algo),
            bnl_window_cap=int(self.bnl_window_cap), count_tests=int(bool(self.count_tests)),
            rep_seed=int(self.seed))


@dataclass
class PhaseMetrics:
    partition_ms: float = 0.0
    local_ms: float = 0.0
    merge_ms: float = 0.0
    local_skyline_sizes: List[int] = field(default_factory=list)
    union_size: int = 0
    filtered_count: int = 0
    final_size: int = 0
    # B200 extensions
    total_ms: float = 0.0
    tests_reps: int = 0
    tests_local: int = 0
    tests_merge: int = 0
    n_reps: int = 0
    angular_host_fixups: int = 0
    kernel_launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    dom_launches: int = 0
    dom_kernel_ms: float = 0.0
    dom_tests: int = 0
    stream_launches: int = 0
    stream_kernel_ms: float = 0.0
    stream_bytes: int = 0
    dom_exact_checks: int = 0
    # multi-GPU
    world: int = 1
    sharded: bool = False
    exchange_bytes: int = 0
    local_rows: int = 0

    @property
    def tests_total(self) -> int:
        return self.tests_reps + self.tests_local + self.tests_merge


@dataclass
class RunResult:
    skyline: np.ndarray  # int64 ids, ascending
    metrics: PhaseMetrics
    config: EngineConfig
    effective_p: int
    input_size: int
    input_dim: int


def snap_slices(target_p: int, k: int) -> int:
    out = C.c_uint64(0)
    _raise(abi.load().sky_snap_slices(target_p, k, C.byref(out)))
    return int(out.value)


def _as_rows(points) -> np.ndarray:
    """float32 rows, or float64 rows when some value is not a float32."""
    a = np.asarray(points)
    if a.dtype == np.float64:
        a64 = np.ascontiguousarray(a)
        if a64.ndim == 2 and not np.array_equal(a64.astype(np.float32).astype(np.float64), a64, equal_nan=True):
            return a64
    return _as_points(a)


def _as_points(points) -> np.ndarray:
    a = np.ascontiguousarray(points, dtype=np.float32)
    if a.ndim == 1:
        a = a.reshape(-1, 1) if a.size else a.reshape(0, 0)
    if a.ndim != 2:
        raise DimensionError("points must be a 2-D array (n x d)")
    return a


class Engine:
    """One GPU context (device, stream, device arena). Not thread-safe: one
    call in flight per Engine, as in the C ABI."""

    def __init__(self, device: int = 0):
        self._lib = abi.load()
        h = C.c_void_p()
        rc = self._lib.sky_ctx_create(device, C.byref(h))
        _raise(rc, "sky_ctx_create failed (is a CUDA device visible?)")
        self._h = h
        self.device = device

    @classmethod
    def group(cls, devices, loopback: bool = False) -> "Engine":
        """One process driving several GPUs (rank r on devices[r]): run()
        shards the rows over the ranks and returns the whole result. NCCL
        between distinct devices; `loopback` (implied when a device repeats)
        exchanges by event-ordered device copies, so every rank may share
        one GPU."""
        self = cls.__new__(cls)
        self._lib = abi.load()
        devs = [int(x) for x in devices]
        arr = (C.c_int * len(devs))(*devs)
        h = C.c_void_p()
        rc = self._lib.sky_ctx_create_group(arr, len(devs), abi.SKY_GROUP_LOOPBACK if loopback else 0, C.byref(h))
        _raise(rc, "sky_ctx_create_group failed")
        self._h = h
        self.device = devs[0]
        return self

    @classmethod
    def peers(cls, devices) -> list:
        """Rank engines of one process that exchange through device copies;
        each is used like Engine.distributed from its own thread (run /
        run_shard called concurrently). Devices may repeat."""
        lib = abi.load()
        devs = [int(x) for x in devices]
        arr = (C.c_int * len(devs))(*devs)
        hs = (C.c_void_p * len(devs))()
        _raise(lib.sky_ctx_create_peers(arr, len(devs), hs), "sky_ctx_create_peers failed")
        out = []
        for r, dev in enumerate(devs):
            e = cls.__new__(cls)
            e._lib = lib
            e._h = C.c_void_p(hs[r])
            e.device = dev
            out.append(e)
        return out

    @property
    def world(self) -> int:
        r, w = C.c_int(0), C.c_int(0)
        self._lib.sky_ctx_world(self._h, C.byref(r), C.byref(w))
        return int(w.value)

    @property
    def rank(self) -> int:
        r, w = C.c_int(0), C.c_int(0)
        self._lib.sky_ctx_world(self._h, C.byref(r), C.byref(w))
        return int(r.value)

    def set_option(self, name: str, value: int):
        """Engine option (sky_ctx_set_option): stream, host_merge, cap_sync,
        sfs_tile, sfs_chunk, sfs_head, merge_tile, merge_head, grain_items,
        profile_host, timeline."""
        self._err(self._lib.sky_ctx_set_option(self._h, name.encode(), int(value)))

    DEFAULT_OPTIONS = {"stream": -1, "host_merge": 0, "cap_sync": -1, "sfs_tile": 0, "sfs_chunk": 2048,
                       "sfs_head": 2048, "merge_tile": 0, "merge_head": 4096, "grain_items": 4, "bnl_block": 1024, "merge_index": 1, "merge_cell_rows": 1024, "range_par": 4, "sfs_auto_chunk": 1, "wave_growth": 4, "wave_split_mpairs": 8192, "profile_host": 0,
                       "timeline": 0, "small_tail": 1, "kernel_events": 0}

    def reset_options(self):
        for k, v in self.DEFAULT_OPTIONS.items():
            self.set_option(k, v)

    def issue_peak(self, d: int, k: int = 0, ctas_per_sm: int = 2, iters: int = 20000) -> float:
        """Measured pair tests/s of the dominance core's packed-code loop on
        every SM (sky_issue_peak): the dominance roofline denominator (k = 0:
        the best over the kernel's shapes)."""
        v = C.c_double(0.0)
        self._err(self._lib.sky_issue_peak(self._h, int(d), int(k), int(ctas_per_sm), int(iters), C.byref(v)))
        return float(v.value)

    def generate_device(self, kind: int, n: int, d: int, seed: int, device_ptr: int):
        """The BASELINE synthetic rows (as `generate`) written by the GPU into
        n*d float32 of device memory at device_ptr (sky_generate_device)."""
        self._err(self._lib.sky_generate_device(self._h, int(kind), int(n), int(d), int(seed),
                                                C.c_void_p(device_ptr)))

    def set_sharded(self, on: bool = True):
        """Take the sharded multi-rank path even on one rank (tests)."""
        self._err(self._lib.sky_ctx_set_sharded(self._h, int(bool(on))))

    @classmethod
    def distributed(cls, device: int, rank: int, world: int, unique_id: bytes) -> "Engine":
        """A rank of a multi-GPU engine (one process per GPU): every rank
        calls run() on the same input; the local and merge phases are
        sharded over the ranks with NCCL and every rank gets the result."""
        self = cls.__new__(cls)
        self._lib = abi.load()
        h = C.c_void_p()
        buf = (C.c_uint8 * len(unique_id)).from_buffer_copy(unique_id)
        rc = self._lib.sky_ctx_create_dist(device, rank, world, buf, C.byref(h))
        _raise(rc, "sky_ctx_create_dist failed")
        self._h = h
        self.device = device
        return self

    def close(self):
        if getattr(self, "_h", None):
            self._lib.sky_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _err(self, rc):
        if rc != abi.SKY_OK:
            msg = self._lib.sky_last_error(self._h)
            _raise(rc, msg.decode() if msg else "")

    def set_stream(self, stream_ptr: Optional[int]):
        self._lib.sky_ctx_set_stream(self._h, C.c_void_p(stream_ptr or 0))

    # skyline::run (engine.hpp:88)
    def run(self, points, config: EngineConfig, normalized: bool = True, *, device_ptr: Optional[int] = None,
            n: Optional[int] = None, d: Optional[int] = None, dtype=np.float32) -> RunResult:
        """Run the engine (skyline::run). `points` is an (n, d) host array, or
        pass device_ptr/n/d (and dtype) for rows already resident on the GPU.
        float64 rows take the exact FP64 path (sky_run_f64) unless every value
        is a float32, in which case both paths give the same result and the
        float32 one is used."""
        cfg = config.to_c()
        res = abi.SkyResult()
        if device_ptr is not None:
            fn = self._lib.sky_run_f64 if np.dtype(dtype) == np.float64 else self._lib.sky_run
            rc = fn(self._h, C.c_void_p(device_ptr), n, d, int(normalized), 1, C.byref(cfg), C.byref(res))
        else:
            a = _as_rows(points)
            n, d = a.shape
            fn = self._lib.sky_run_f64 if a.dtype == np.float64 else self._lib.sky_run
            rc = fn(self._h, a.ctypes.data_as(C.c_void_p), n, d, int(normalized), 0, C.byref(cfg), C.byref(res))
        self._err(rc)
        return self._result(res, config)

    def run_shard(self, points, config: EngineConfig, normalized: bool = True, *, device_ptr: Optional[int] = None,
                  n: Optional[int] = None, d: Optional[int] = None) -> RunResult:
        """skyline::run over rows sharded across the ranks of a distributed
        engine (sky_run_shard): `points` are this rank's consecutive rows
        (rank 0's first); every rank gets the whole result."""
        cfg = config.to_c()
        res = abi.SkyResult()
        if device_ptr is not None:
            rc = self._lib.sky_run_shard(self._h, C.c_void_p(device_ptr), n, d, int(normalized), 1, C.byref(cfg),
                                         C.byref(res))
        else:
            a = _as_points(points)
            n, d = a.shape
            rc = self._lib.sky_run_shard(self._h, a.ctypes.data_as(C.c_void_p), n, d, int(normalized), 0,
                                         C.byref(cfg), C.byref(res))
        self._err(rc)
        return self._result(res, config)

    def _result(self, res, config) -> RunResult:
        owned = False
        try:
            # every scalar of the result in one unpack (no per-field ctypes
            # fetch); ids by memmove instead of np.ctypeslib.as_array (~10 us
            # of array-interface setup per call, inside the caller's timed
            # region)
            v = abi.SKY_RESULT_STRUCT.unpack_from(res)
            f = _RF
            nid = v[f["n_ids"]]
            if nid >= _ZERO_COPY_IDS:
                # megabytes of ids: a view of the library's buffer instead of
                # a fresh array (its page faults and the copy cost ~2 ms on
                # 700k ids); the buffer goes back to the library when the
                # last view of it is collected
                buf = (C.c_int64 * nid).from_address(v[f["ids"]])
                buf._owner = _ResultOwner(self._lib, res)
                owned = True
                ids = np.frombuffer(buf, dtype=np.int64)
            else:
                ids = np.empty(nid, np.int64)
                if nid:
                    C.memmove(ids.ctypes.data, v[f["ids"]], nid * 8)
            P = v[f["effective_p"]]
            sizes_a = np.empty(P, np.uint64)
            if P:
                C.memmove(sizes_a.ctypes.data, v[f["local_skyline_sizes"]], P * 8)
            m = PhaseMetrics(
                v[f["partition_ms"]], v[f["local_ms"]], v[f["merge_ms"]], sizes_a.tolist(), v[f["union_size"]],
                v[f["filtered_count"]], v[f["final_size"]], v[f["total_ms"]], v[f["tests_reps"]],
                v[f["tests_local"]], v[f["tests_merge"]], v[f["n_reps"]], v[f["angular_host_fixups"]],
                v[f["kernel_launches"]], v[f["h2d_bytes"]], v[f["d2h_bytes"]], v[f["dom_launches"]],
                v[f["dom_kernel_ms"]], v[f["dom_tests"]], v[f["stream_launches"]], v[f["stream_kernel_ms"]],
                v[f["stream_bytes"]], v[f["dom_exact_checks"]], v[f["world"]] or 1, bool(v[f["sharded"]]),
                v[f["exchange_bytes"]], v[f["local_rows"]])
            return RunResult(ids, m, config, P, v[f["input_size"]], v[f["input_dim"]])
        finally:
            if not owned:
                self._lib.sky_result_free(C.byref(res))

    # skyline::make_assignment (partition.hpp:102)
    def make_assignment(self, points, partition: PartitionConfig, normalized: bool = True):
        a = _as_points(points)
        n, d = a.shape
        cfg = EngineConfig(partition=partition).to_c()
        out = np.zeros(max(n, 1), np.uint64)
        P = C.c_uint64(0)
        rc = self._lib.sky_assign(self._h, a.ctypes.data_as(C.POINTER(C.c_float)), n, d, int(normalized),
                                  C.byref(cfg), out.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(P))
        self._err(rc)
        return out[:n], int(P.value)

    # skyline::relative_skyline (core.hpp:79): boolean keep mask over r
    def relative_skyline(self, r, c):
        ra = _as_points(r)
        ca = _as_points(c)
        d = ra.shape[1] if ra.size else (ca.shape[1] if ca.size else 0)
        if ra.size and ca.size and ra.shape[1] != ca.shape[1]:
            raise DimensionError("relative skyline over relations of unequal dimensionality")
        keep = np.ones(max(len(ra), 1), np.uint8)
        tests = C.c_uint64(0)
        rc = self._lib.sky_relative_skyline(self._h, ra.ctypes.data_as(C.POINTER(C.c_float)), len(ra),
                                            ca.ctypes.data_as(C.POINTER(C.c_float)), len(ca), d,
                                            keep.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(tests))
        self._err(rc)
        return keep[: len(ra)].astype(bool)

    # skyline::sfs / skyline_bruteforce: skyline ids ascending
    def sfs(self, points) -> np.ndarray:
        a = _as_points(points)
        n, d = a.shape
        ptr = C.POINTER(C.c_int64)()
        k = C.c_uint64(0)
        t = C.c_uint64(0)
        rc = self._lib.sky_skyline(self._h, a.ctypes.data_as(C.POINTER(C.c_float)), n, d, C.byref(ptr),
                                   C.byref(k), C.byref(t))
        self._err(rc)
        try:
            return np.ctypeslib.as_array(ptr, shape=(k.value,)).copy() if k.value else np.zeros(0, np.int64)
        finally:
            self._lib.sky_free(ptr)

    skyline = sfs

    # select_representatives_sorted + prune_dominated_reps (filter.hpp:46,67)
    def select_representatives_sorted(self, points, partition_of, p: int, q: int) -> np.ndarray:
        a = _as_points(points)
        n, d = a.shape
        po = np.ascontiguousarray(partition_of, dtype=np.uint64)
        ptr = C.POINTER(C.c_int64)()
        k = C.c_uint64(0)
        rc = self._lib.sky_representatives(self._h, a.ctypes.data_as(C.POINTER(C.c_float)), n, d,
                                           po.ctypes.data_as(C.POINTER(C.c_uint64)), p, q, C.byref(ptr),
                                           C.byref(k))
        self._err(rc)
        try:
            return np.ctypeslib.as_array(ptr, shape=(k.value,)).copy() if k.value else np.zeros(0, np.int64)
        finally:
            self._lib.sky_free(ptr)


_default: Optional[Engine] = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(0)
    return _default


def run(points, config: EngineConfig, normalized: bool = True) -> RunResult:
    """skyline::run on the default GPU context."""
    return default_engine().run(points, config, normalized)


def generate(kind: int, n: int, d: int, seed: int) -> np.ndarray:
    """Synthetic BASELINE inputs (host, deterministic): kind 1 uniform,
    2/4 anti-correlated, 3 correlated, 5 integers in [0,16)."""
    out = np.empty((n, d), np.float32)
    rc = abi.load().sky_generate(kind, n, d, seed, out.ctypes.data_as(C.POINTER(C.c_float)))
    _raise(rc)
    return out


class Distribution(enum.IntEnum):
    """datagen.hpp:12-16"""
    Uniform = 0
    Correlated = 1
    Anticorrelated = 2


def _host_raise(rc: int):
    if rc != abi.SKY_OK:
        _raise(rc, abi.load().sky_host_error().decode(errors="replace"))


def generate_family(distribution, n: int, d: int, seed: int) -> np.ndarray:
    """skyline::generate (datagen.cpp:127-151): FP64 rows identical to the
    reference's for (distribution, n, d, seed)."""
    out = np.empty((n, d), np.float64)
    _host_raise(abi.load().sky_generate_family(int(distribution), n, d, seed,
                                               out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def normalize(rows) -> np.ndarray:
    """skyline::normalize (datagen.cpp:153-168): column min-max to [0,1]."""
    a = np.array(rows, dtype=np.float64, order="C", copy=True)
    n, d = a.shape
    _host_raise(abi.load().sky_normalize(a.ctypes.data_as(C.POINTER(C.c_double)), n, d))
    return a


def ingest_csv(path: str, columns=None, maximize=None) -> np.ndarray:
    """skyline::ingest_csv (datagen.cpp:170-218): selected columns (all when
    None), `maximize` = column names where larger raw values are better."""
    lib = abi.load()
    cols = list(columns or [])
    arr = (C.c_char_p * max(1, len(cols)))(*[c.encode() for c in cols])
    mx = list(maximize or [])
    if mx and not cols:
        raise ConfigError("maximize needs explicit columns")
    flags = np.array([1 if c in mx else 0 for c in cols], np.uint8) if mx else np.zeros(1, np.uint8)
    rows = C.POINTER(C.c_double)()
    n = C.c_uint64(0)
    d = C.c_uint32(0)
    _host_raise(lib.sky_ingest_csv(path.encode(), arr, len(cols), flags.ctypes.data_as(C.POINTER(C.c_uint8)),
                                   len(cols) if mx else 0, C.byref(rows), C.byref(n), C.byref(d)))
    try:
        return np.ctypeslib.as_array(rows, shape=(n.value, d.value)).copy()
    finally:
        lib.sky_free(rows)


def write_csv(path: str, rows) -> None:
    """skyline::write_csv (datagen.cpp:220-238)."""
    a = np.ascontiguousarray(rows, dtype=np.float64)
    n, d = a.shape
    _host_raise(abi.load().sky_write_csv(path.encode(), a.ctypes.data_as(C.POINTER(C.c_double)), n, d))


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _raise(abi.load().sky_nccl_unique_id(buf, 128))
    return bytes(buf)


def plan_local_shards(off, ranks: int) -> np.ndarray:
    """Partition ranges per rank for the local phase (what sky_run uses)."""
    o = np.ascontiguousarray(off, dtype=np.uint32)
    b = np.zeros(ranks + 1, np.uint32)
    _raise(abi.load().sky_plan_local_shards(o.ctypes.data_as(C.POINTER(C.c_uint32)), len(o) - 1, ranks,
                                            b.ctypes.data_as(C.POINTER(C.c_uint32))))
    return b


def plan_merge_shards(offu, ranks: int, config: EngineConfig, d: int, m: int = 0) -> np.ndarray:
    """Candidate-partition ranges per rank for the merge phase."""
    o = np.ascontiguousarray(offu, dtype=np.uint32)
    b = np.zeros(ranks + 1, np.uint32)
    cfg = config.to_c()
    _raise(abi.load().sky_plan_merge_shards(o.ctypes.data_as(C.POINTER(C.c_uint32)), len(o) - 1, ranks,
                                            C.byref(cfg), d, m, b.ctypes.data_as(C.POINTER(C.c_uint32))))
    return b


def plan_lpt(weights, ranks: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, dtype=np.uint64)
    owner = np.zeros(max(len(w), 1), np.int32)
    _raise(abi.load().sky_plan_lpt(w.ctypes.data_as(C.POINTER(C.c_uint64)), len(w), ranks,
                                   owner.ctypes.data_as(C.POINTER(C.c_int32))))
    return owner[: len(w)]


def plan_split(cost, ranks: int) -> np.ndarray:
    c = np.ascontiguousarray(cost, dtype=np.uint64)
    prefix = np.zeros(len(c) + 1, np.uint64)
    np.cumsum(c, out=prefix[1:])
    bounds = np.zeros(ranks + 1, np.uint64)
    _raise(abi.load().sky_plan_split(prefix.ctypes.data_as(C.POINTER(C.c_uint64)), len(c), ranks,
                                     bounds.ctypes.data_as(C.POINTER(C.c_uint64))))
    return bounds
