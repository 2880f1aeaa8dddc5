"""B200-native two-phase parallel skyline engine (arXiv 2411.14968 hot path).

The engine lives in libskyline_b200.so (hand-written sm_100a CUDA kernels +
C++ host orchestration behind the C ABI in include/skyline_b200.h); this
package is the host-side mirror of the reference's engine API.
"""
from .skyline import (  # noqa: F401
    ConfigError, CudaError, DataError, DimensionError, Distribution, Engine, EngineConfig, FilterKind, IoError, LocalAlgo,
    MergeKind, NcclError, NormalizationError, PartitionConfig, PhaseMetrics, RepSelection, RunResult,
    SkylineError, Strategy, default_engine, generate, generate_family, ingest_csv, nccl_unique_id, normalize, plan_local_shards, plan_lpt, plan_merge_shards,
    plan_split, run, snap_slices, write_csv,
)
from .configs import BASELINE_CONFIGS, make_config  # noqa: F401
