"""Multi-rank engine on one B200: the sharded phase 1 (shard.cu), the
replicated phase 1 (run_impl's world > 1 branch), the exchanges (comm.cpp)
and the group / peer / distributed contexts, against the reference goldens
and the oracle. Bit-exact: ids, effective_p, union_size, filtered_count,
final_size, local_skyline_sizes.

The ranks run as host threads of this process. Loopback ranks exchange by
event-ordered device copies (no kernel waits on another rank), so several
ranks may share the one GPU of the box; the NCCL backend is exercised with a
real one-rank communicator (ncclCommInitAll / ncclCommInitRank).
"""
import threading

import numpy as np
import pytest

import oracle as O
from paper_2411_14968_b200 import (DataError, Engine, EngineConfig, FilterKind, LocalAlgo, MergeKind,
                                   PartitionConfig, RepSelection, Strategy, generate, nccl_unique_id)
from paper_2411_14968_b200.abi import SkyConfig
from paper_2411_14968_b200.configs import make_config

pytestmark = pytest.mark.gpu


def to_engine_config(d):
    return EngineConfig(partition=PartitionConfig(Strategy(d["strategy"]), d["p"], d["m"], d["seed"], d["slice_dim"]),
                        filter=FilterKind(d["filter"]), rep_q=d["rep_q"], merge=MergeKind(d["merge"]),
                        rep_selection=RepSelection(d.get("rep_selection", 0)), seed=d.get("rep_seed", d["seed"]),
                        workers=max(1, d["workers"]), local_algo=LocalAlgo(d.get("local_algo", 0)),
                        bnl_window_cap=d.get("bnl_window_cap", 4096) or 4096)


def same(r, exp, tag):
    assert np.array_equal(r.skyline, np.asarray(exp["ids"], np.int64)), tag
    m = r.metrics
    assert r.effective_p == exp["effective_p"], tag
    assert m.union_size == exp["union_size"], (tag, m.union_size, exp["union_size"])
    assert m.filtered_count == exp["filtered_count"], (tag, m.filtered_count, exp["filtered_count"])
    assert m.final_size == exp["final_size"], tag
    assert list(m.local_skyline_sizes) == [int(v) for v in exp["local_skyline_sizes"]], tag


@pytest.fixture(scope="module", params=[2, 3])
def group(request):
    e = Engine.group([0] * request.param, loopback=True)
    assert e.world == request.param
    yield e
    e.close()


def sharded_cases():
    rng = np.random.default_rng(11)
    out = []
    for strat, p in ((Strategy.Random, 7), (Strategy.Grid, 16), (Strategy.Angular, 9), (Strategy.Sliced, 11)):
        for filt in (FilterKind.None_, FilterKind.Representative):
            for merge in (MergeKind.Sequential, MergeKind.NoSeq):
                for algo in (LocalAlgo.SFS, LocalAlgo.BNL):
                    d = int(rng.integers(2, 7))
                    n = int(rng.integers(500, 6000))
                    kind = int(rng.integers(0, 3))
                    if kind == 0:
                        x = rng.random((n, d), dtype=np.float32)
                    elif kind == 1:
                        x = generate(2, n, d, int(rng.integers(1 << 30)))
                    else:  # ties: lattice values (sliced tie runs straddle boundaries)
                        x = (rng.integers(0, 5, (n, d)) / 4).astype(np.float32)
                    cfg = EngineConfig(partition=PartitionConfig(strat, p=p, seed=int(rng.integers(100))),
                                       filter=filt, rep_q=int(rng.integers(1, 9)), merge=merge, local_algo=algo,
                                       bnl_window_cap=64)
                    out.append((x, cfg))
    return out


def test_group_sharded_vs_oracle(group):
    """Every strategy x filter x merge x local algorithm on the sharded path
    (and the replicated one where the input needs it) equals the oracle."""
    for k, (x, cfg) in enumerate(sharded_cases()):
        exp = O.oracle_run(x, cfg.to_c(), True)
        r = group.run(x, cfg, True)
        assert r.metrics.world == group.world
        same(r, exp, (group.world, k, cfg.partition.strategy.name, cfg.filter.name, cfg.merge.name))


def test_group_plane_matches_reference(group, golden):
    """The reference-generated configuration plane (grid filtering, Region /
    Random representatives: the replicated phase 1; the rest sharded)."""
    arr = golden["plane_arrays"]
    for case in golden["plane"][:: 3 if group.world == 3 else 1]:
        key = case["key"]
        cfg = to_engine_config(case["cfg"])
        r = group.run(arr[key + "_x"], cfg, case["normalized"])
        assert np.array_equal(r.skyline, arr[key + "_ids"]), key
        assert r.metrics.local_skyline_sizes == arr[key + "_lss"].tolist(), key
        assert r.metrics.union_size == case["union_size"] and r.metrics.filtered_count == case["filtered_count"], key


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_group_baseline_configs_reduced(group, golden, idx):
    c = [c for c in golden["configs"] if c["config"] == idx][0]
    arr = golden["config_arrays"]
    x = generate(c["kind"], c["n"], c["d"], c["seed"])
    w = make_config(idx)
    r = group.run(x, w.config, c["normalized"])
    assert r.metrics.sharded, idx
    assert np.array_equal(r.skyline, arr[f"c{idx}_ids"]), idx
    assert r.metrics.local_skyline_sizes == arr[f"c{idx}_lss"].tolist(), idx
    assert r.metrics.union_size == c["union_size"] and r.metrics.filtered_count == c["filtered_count"], idx


def test_group_edge_cases(group):
    """Fewer rows than ranks (ranks without rows), ranks without partitions,
    empty input, duplicates, and errors raised identically by every rank."""
    W = group.world
    cfgs = [EngineConfig(partition=PartitionConfig(Strategy.Random, p=5, seed=1), filter=FilterKind.Representative,
                         rep_q=2, merge=MergeKind.NoSeq),
            EngineConfig(partition=PartitionConfig(Strategy.Sliced, p=1), merge=MergeKind.NoSeq),
            EngineConfig(partition=PartitionConfig(Strategy.Grid, p=4), filter=FilterKind.Representative, rep_q=3,
                         merge=MergeKind.NoSeq, local_algo=LocalAlgo.BNL)]
    rng = np.random.default_rng(5)
    for n in (0, 1, W - 1, W, 7):
        x = rng.random((n, 3), dtype=np.float32)
        for cfg in cfgs:
            exp = O.oracle_run(x, cfg.to_c(), True)
            same(group.run(x, cfg, True), exp, (W, n, cfg.partition.strategy.name))
    x = np.repeat(rng.random((4, 3), dtype=np.float32), 500, axis=0)
    for cfg in cfgs:
        same(group.run(x, cfg, True), O.oracle_run(x, cfg.to_c(), True), ("dups", cfg.partition.strategy.name))
    # a NaN in the last rank's rows: every rank reports the DataError
    x = rng.random((3000, 4), dtype=np.float32)
    x[-1, 2] = np.nan
    with pytest.raises(DataError):
        group.run(x, cfgs[0], True)
    # the group is usable after the error
    x = rng.random((3000, 4), dtype=np.float32)
    same(group.run(x, cfgs[0], True), O.oracle_run(x, cfgs[0].to_c(), True), "after error")


def test_group_f64_rows(group):
    """FP64 rows (replicated phase 1 on every rank) equal the oracle."""
    rng = np.random.default_rng(9)
    base = rng.random((1500, 4))
    x = np.concatenate([base, base + 1e-12])  # differences below float32 resolution
    x = np.minimum(x, 1.0)
    cfg = EngineConfig(partition=PartitionConfig(Strategy.Sliced, p=6), filter=FilterKind.Representative, rep_q=3,
                       merge=MergeKind.NoSeq)
    exp = O.oracle_run(x, cfg.to_c(), True)
    same(group.run(x, cfg, True), exp, "f64")


def _run_peers(engines, fn):
    """fn(rank, engine) on every rank concurrently (one thread per rank)."""
    out = [None] * len(engines)
    err = [None] * len(engines)

    def body(r):
        try:
            out[r] = fn(r, engines[r])
        except Exception as e:  # noqa: BLE001
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(len(engines))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("W", [2, 3])
def test_peers_run_shard(W):
    """sky_run_shard: each rank passes only its own rows (unequal shards,
    one empty), as torchrun ranks do; every rank returns the reference
    result. Also device-resident shards."""
    import torch
    peers = Engine.peers([0] * W)
    try:
        for idx, n in ((2, 40_000), (4, 12_000), (5, 60_000), (1, 30_000), (3, 150_000)):
            w = make_config(idx, n)
            x = generate(w.kind, w.n, w.d, 42)
            exp = O.oracle_run(x, w.config.to_c(), w.normalized)
            cuts = [0] + sorted(int(v) for v in np.random.default_rng(idx).integers(0, n, W - 1)) + [n]
            cuts[1] = cuts[0]  # rank 0 holds no rows
            res = _run_peers(peers, lambda r, e: e.run_shard(x[cuts[r]:cuts[r + 1]], w.config, w.normalized))
            for r in range(W):
                same(res[r], exp, (idx, W, r))
            dev = [torch.from_numpy(x[cuts[r]:cuts[r + 1]].copy()).cuda() for r in range(W)]
            torch.cuda.synchronize()
            res = _run_peers(peers, lambda r, e: e.run_shard(None, w.config, w.normalized,
                                                              device_ptr=dev[r].data_ptr(), n=cuts[r + 1] - cuts[r],
                                                              d=w.d))
            same(res[0], exp, (idx, W, "device"))
    finally:
        for e in peers:
            e.close()


def test_nccl_one_rank_sharded():
    """The sharded path through real NCCL communicators (one rank: the
    all-reduces and copies run as NCCL launches), both constructors."""
    dist = Engine.distributed(0, 0, 1, nccl_unique_id())
    grp = Engine.group([0])
    try:
        dist.set_sharded(True)
        grp.set_sharded(True)
        for idx, n in ((2, 30_000), (4, 8_000), (3, 200_000), (5, 50_000), (1, 20_000)):
            w = make_config(idx, n)
            x = generate(w.kind, w.n, w.d, 42)
            exp = O.oracle_run(x, w.config.to_c(), w.normalized)
            for e in (dist, grp):
                r = e.run(x, w.config, w.normalized)
                assert r.metrics.sharded
                same(r, exp, (idx, e.world))
            same(dist.run_shard(x, w.config, w.normalized), exp, (idx, "shard"))
    finally:
        dist.close()
        grp.close()


def test_single_rank_forced_sharded(engine):
    """The sharded path on a plain one-GPU context (loopback of one)."""
    e = Engine(0)
    try:
        e.set_sharded(True)
        for x, cfg in sharded_cases()[::2]:
            same(e.run(x, cfg, True), O.oracle_run(x, cfg.to_c(), True), cfg.partition.strategy.name)
    finally:
        e.close()


@pytest.mark.parametrize("i", [1, 2, 3, 4, 5])
def test_full_size_group_matches_reference(i):
    """Full BASELINE sizes through two sharded loopback ranks on the one GPU:
    the reference's own result (tests/golden/full, from oracle/_ref)."""
    import hashlib

    from test_full_size import _check, load
    g, ids = load(i)
    w = make_config(i)
    x = generate(w.kind, w.n, w.d, 42)
    assert hashlib.sha256(x.tobytes()).hexdigest() == g["input_sha256"]
    e = Engine.group([0, 0], loopback=True)
    try:
        r = e.run(x, w.config, w.normalized)
        assert r.metrics.sharded and r.metrics.world == 2
        _check(r, g, ids, f"c{i} W=2")
    finally:
        e.close()


def test_group_sliced_many_tie_runs(group):
    """Sliced partitions whose boundaries fall inside many tie runs of the
    slice attribute (the run table is laid out identically on every rank,
    whatever order the device lists the runs in)."""
    rng = np.random.default_rng(21)
    for it in range(3):
        x = rng.random((20000, 4), dtype=np.float32)
        x[:, 0] = (rng.integers(0, 40, 20000) / 39).astype(np.float32)
        for p, filt in ((64, FilterKind.Representative), (127, FilterKind.None_)):
            cfg = EngineConfig(partition=PartitionConfig(Strategy.Sliced, p=p), filter=filt, rep_q=3,
                               merge=MergeKind.NoSeq)
            same(group.run(x, cfg, True), O.oracle_run(x, cfg.to_c(), True), (it, p))
