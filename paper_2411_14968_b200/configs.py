"""The five BASELINE.json configurations as engine configs + input recipes.

Synthetic inputs stand in for the paper's UNI/ANT/CORR families; they are
generated on the host by sky_generate (deterministic for (kind, n, d, seed)).
q for configs 3-5 is the reference default rep_q = 5 (engine.hpp:34;
SURVEY.md 0.4). Config 2's 64 angular partitions snap to m = 2, i.e. 32
effective partitions (partition.cpp:220-245).
"""
from __future__ import annotations

from dataclasses import dataclass

from .skyline import EngineConfig, FilterKind, LocalAlgo, MergeKind, PartitionConfig, Strategy

DATA_SEED = 42


@dataclass(frozen=True)
class Workload:
    name: str
    kind: int          # sky_generate kind
    n: int
    d: int
    normalized: bool
    config: EngineConfig
    description: str


def make_config(idx: int, n: int | None = None) -> Workload:
    if idx == 1:
        cfg = EngineConfig(partition=PartitionConfig(Strategy.Random, p=8, seed=DATA_SEED),
                           filter=FilterKind.None_, merge=MergeKind.Sequential, local_algo=LocalAlgo.SFS)
        return Workload("c1_uniform_d4_random8_sfs_seq", 1, n or 100_000, 4, True, cfg,
                        "uniform N=100k d=4, random 8, SFS, sequential merge, no filter")
    if idx == 2:
        cfg = EngineConfig(partition=PartitionConfig(Strategy.Angular, p=64),
                           filter=FilterKind.Representative, rep_q=8, merge=MergeKind.NoSeq,
                           local_algo=LocalAlgo.SFS)
        return Workload("c2_anticorr_d6_angular64_q8_noseq", 2, n or 1_000_000, 6, True, cfg,
                        "anti-correlated N=1M d=6, angular 64 (->32), reps q=8, NoSeq")
    if idx == 3:
        cfg = EngineConfig(partition=PartitionConfig(Strategy.Grid, p=256, m=2),
                           filter=FilterKind.Representative, rep_q=5, merge=MergeKind.NoSeq,
                           local_algo=LocalAlgo.SFS)
        return Workload("c3_corr_d8_grid2_q5_noseq", 3, n or 10_000_000, 8, True, cfg,
                        "correlated N=10M d=8, grid m=2 (256 cells), reps q=5, NoSeq")
    if idx == 4:
        cfg = EngineConfig(partition=PartitionConfig(Strategy.Sliced, p=128, slice_dim=0),
                           filter=FilterKind.Representative, rep_q=5, merge=MergeKind.NoSeq,
                           local_algo=LocalAlgo.BNL, bnl_window_cap=4096)
        return Workload("c4_anticorr_d10_sliced128_bnl4096_q5_noseq", 4, n or 4_000_000, 10, True, cfg,
                        "anti-correlated N=4M d=10, sliced 128 on x0, BNL window 4096, reps q=5, NoSeq")
    if idx == 5:
        cfg = EngineConfig(partition=PartitionConfig(Strategy.Random, p=32, seed=DATA_SEED),
                           filter=FilterKind.Representative, rep_q=5, merge=MergeKind.NoSeq,
                           local_algo=LocalAlgo.SFS)
        return Workload("c5_ints16_d5_random32_q5_noseq", 5, n or 2_000_000, 5, False, cfg,
                        "integers [0,16) N=2M d=5, random 32, reps q=5, NoSeq")
    raise ValueError(idx)


BASELINE_CONFIGS = {i: make_config(i) for i in range(1, 6)}
