"""ctypes view of include/skyline_b200.h (the C ABI) and the library loader.

The shared library ``libskyline_b200.so`` is built in-tree by
``paper_2411_14968_b200/build.py`` (nvcc, sm_100a). Loading fails loudly when
it is missing: there is no CPU or Python fallback for the engine.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libskyline_b200.so")

SKY_OK = 0
SKY_E_CONFIG, SKY_E_DIMENSION, SKY_E_NORMALIZATION, SKY_E_DATA, SKY_E_IO = 1, 2, 3, 4, 5
STATUS_NAMES = {
    0: "OK", 1: "ConfigError", 2: "DimensionError", 3: "NormalizationError",
    4: "DataError", 5: "IoError", 10: "CudaError", 11: "NcclError", 12: "InternalError",
}


class SkyConfig(C.Structure):
    """sky_config — EngineConfig (engine.hpp:30-38) + PartitionConfig
    (partition.hpp:21-27) + B200 extensions."""

    _fields_ = [
        ("strategy", C.c_int32),
        ("p", C.c_uint64),
        ("m", C.c_uint64),
        ("seed", C.c_uint64),
        ("slice_dim", C.c_uint64),
        ("filter", C.c_int32),
        ("rep_selection", C.c_int32),
        ("rep_q", C.c_uint64),
        ("merge", C.c_int32),
        ("workers", C.c_uint64),
        ("local_algo", C.c_int32),
        ("bnl_window_cap", C.c_uint32),
        ("count_tests", C.c_int32),
        ("rep_seed", C.c_uint64),
    ]

    @classmethod
    def make(cls, strategy=0, p=1, m=0, seed=0, slice_dim=0, filter=0, rep_selection=0,
             rep_q=5, merge=0, workers=1, local_algo=0, bnl_window_cap=4096, count_tests=1, rep_seed=None):
        # rep_seed defaults to the partition seed, as the reference CLI sets both
        return cls(strategy, p, m, seed, slice_dim, filter, rep_selection, rep_q, merge,
                   workers, local_algo, bnl_window_cap, count_tests, seed if rep_seed is None else rep_seed)

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class SkyResult(C.Structure):
    _fields_ = [
        ("ids", C.POINTER(C.c_int64)),
        ("n_ids", C.c_uint64),
        ("effective_p", C.c_uint64),
        ("input_size", C.c_uint64),
        ("input_dim", C.c_uint64),
        ("union_size", C.c_uint64),
        ("filtered_count", C.c_uint64),
        ("final_size", C.c_uint64),
        ("local_skyline_sizes", C.POINTER(C.c_uint64)),
        ("partition_ms", C.c_double),
        ("local_ms", C.c_double),
        ("merge_ms", C.c_double),
        ("total_ms", C.c_double),
        ("tests_reps", C.c_uint64),
        ("tests_local", C.c_uint64),
        ("tests_merge", C.c_uint64),
        ("n_reps", C.c_uint64),
        ("angular_host_fixups", C.c_uint64),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("kernel_launches", C.c_uint32),
        ("dom_launches", C.c_uint32),
        ("dom_kernel_ms", C.c_double),
        ("dom_tests", C.c_uint64),
        ("dom_exact_checks", C.c_uint64),
        ("exact_checks_merge", C.c_uint64),
        ("stream_launches", C.c_uint32),
        ("stream_kernel_ms", C.c_double),
        ("stream_bytes", C.c_uint64),
        ("world", C.c_uint32),
        ("sharded", C.c_uint32),
        ("exchange_bytes", C.c_uint64),
        ("local_rows", C.c_uint64),
    ]


def _struct_of(cstruct):
    """struct.Struct with the C layout of a ctypes.Structure of scalars and
    pointers: one unpack reads every field (a ctypes attribute fetch per field
    costs ~20 us per result, inside a caller's timed region)."""
    import struct
    codes = {C.c_double: "d", C.c_float: "f", C.c_uint64: "Q", C.c_int64: "q", C.c_uint32: "I", C.c_int32: "i"}
    fmt = "@" + "".join(codes.get(t, "P") for _, t in cstruct._fields_)
    st = struct.Struct(fmt)
    assert st.size == C.sizeof(cstruct), (st.size, C.sizeof(cstruct))
    return st


SKY_RESULT_STRUCT = _struct_of(SkyResult)
SKY_RESULT_FIELDS = {name: k for k, (name, _) in enumerate(SkyResult._fields_)}


# Every symbol include/skyline_b200.h declares; tests check the library
# exports all of them.
EXPORTED = [
    "sky_ctx_create", "sky_ctx_destroy", "sky_nccl_unique_id", "sky_ctx_create_dist",
    "sky_last_error", "sky_ctx_set_stream",
    "sky_config_default", "sky_run", "sky_run_f64", "sky_result_free", "sky_assign",
    "sky_snap_slices", "sky_relative_skyline", "sky_skyline",
    "sky_representatives", "sky_free", "sky_generate", "sky_plan_lpt",
    "sky_plan_split", "sky_plan_local_shards", "sky_plan_merge_shards", "sky_abi_version",
    "sky_generate_family", "sky_normalize", "sky_ingest_csv", "sky_write_csv", "sky_host_error",
    "sky_ctx_create_group", "sky_ctx_world", "sky_ctx_set_sharded", "sky_run_shard", "sky_ctx_set_option",
    "sky_ctx_create_peers", "sky_issue_peak", "sky_device_count", "sky_generate_device",
]

SKY_GROUP_LOOPBACK = 1

_lib = None
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_f32p = C.POINTER(C.c_float)


def load():
    """Load libskyline_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2411_14968_b200.build` "
            "(nvcc -gencode arch=compute_100a,code=sm_100a). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    lib.sky_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    lib.sky_ctx_destroy.argtypes = [vp]
    lib.sky_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8), C.c_uint64]
    lib.sky_ctx_create_dist.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(vp)]
    lib.sky_ctx_create_group.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int, C.POINTER(vp)]
    lib.sky_ctx_create_peers.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
    lib.sky_ctx_world.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.sky_ctx_set_sharded.argtypes = [vp, C.c_int]
    lib.sky_ctx_set_option.argtypes = [vp, C.c_char_p, C.c_int64]
    lib.sky_run_shard.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_int, C.c_int,
                                  C.POINTER(SkyConfig), C.POINTER(SkyResult)]
    lib.sky_last_error.argtypes = [vp]
    lib.sky_last_error.restype = C.c_char_p
    lib.sky_ctx_set_stream.argtypes = [vp, vp]
    lib.sky_config_default.argtypes = [C.POINTER(SkyConfig)]
    lib.sky_run.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_int, C.c_int,
                            C.POINTER(SkyConfig), C.POINTER(SkyResult)]
    lib.sky_run_f64.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_int, C.c_int,
                            C.POINTER(SkyConfig), C.POINTER(SkyResult)]
    lib.sky_generate_family.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(C.c_double)]
    lib.sky_normalize.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_uint32]
    lib.sky_ingest_csv.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_uint32, _u8p, C.c_uint32,
                                   C.POINTER(C.POINTER(C.c_double)), _u64p, C.POINTER(C.c_uint32)]
    lib.sky_write_csv.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_uint64, C.c_uint32]
    lib.sky_host_error.restype = C.c_char_p
    lib.sky_result_free.argtypes = [C.POINTER(SkyResult)]
    lib.sky_assign.argtypes = [vp, _f32p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(SkyConfig), _u64p, _u64p]
    lib.sky_snap_slices.argtypes = [C.c_uint64, C.c_uint64, _u64p]
    lib.sky_relative_skyline.argtypes = [vp, _f32p, C.c_uint64, _f32p, C.c_uint64, C.c_uint32, _u8p, _u64p]
    lib.sky_skyline.argtypes = [vp, _f32p, C.c_uint64, C.c_uint32, C.POINTER(_i64p), _u64p, _u64p]
    lib.sky_representatives.argtypes = [vp, _f32p, C.c_uint64, C.c_uint32, _u64p, C.c_uint64, C.c_uint64,
                                        C.POINTER(_i64p), _u64p]
    lib.sky_free.argtypes = [vp]
    lib.sky_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, _f32p]
    lib.sky_plan_lpt.argtypes = [_u64p, C.c_uint64, C.c_int, C.POINTER(C.c_int32)]
    lib.sky_plan_split.argtypes = [_u64p, C.c_uint64, C.c_int, _u64p]
    _u32p = C.POINTER(C.c_uint32)
    lib.sky_plan_local_shards.argtypes = [_u32p, C.c_uint64, C.c_int, _u32p]
    lib.sky_plan_merge_shards.argtypes = [_u32p, C.c_uint64, C.c_int, C.POINTER(SkyConfig), C.c_uint32, C.c_uint64,
                                          _u32p]
    lib.sky_issue_peak.argtypes = [vp, C.c_uint32, C.c_int, C.c_int, C.c_uint32, C.POINTER(C.c_double)]
    lib.sky_device_count.restype = C.c_int
    lib.sky_generate_device.argtypes = [vp, C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, vp]
    lib.sky_abi_version.restype = C.c_int
    _lib = lib
    return lib
