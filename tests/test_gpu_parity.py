"""GPU parity: the sm_100a engine (through the C ABI) against the reference
goldens and the oracle. Integer/index work, so every check is bit-exact:
skyline id sets, effective_p, union_size, filtered_count, final_size and
local_skyline_sizes."""
import hashlib

import numpy as np
import pytest

import oracle as O
from paper_2411_14968_b200 import (ConfigError, DataError, DimensionError, EngineConfig, FilterKind, LocalAlgo,
                                   MergeKind, NormalizationError, PartitionConfig, RepSelection, Strategy, generate)
from paper_2411_14968_b200.abi import SkyConfig
from paper_2411_14968_b200.configs import make_config

pytestmark = pytest.mark.gpu


def to_engine_config(d):
    return EngineConfig(partition=PartitionConfig(Strategy(d["strategy"]), d["p"], d["m"], d["seed"], d["slice_dim"]),
                        filter=FilterKind(d["filter"]), rep_q=d["rep_q"], merge=MergeKind(d["merge"]),
                        rep_selection=RepSelection(d.get("rep_selection", 0)), seed=d.get("rep_seed", d["seed"]),
                        workers=max(1, d["workers"]), local_algo=LocalAlgo(d.get("local_algo", 0)),
                        bnl_window_cap=d.get("bnl_window_cap", 4096) or 4096)


def check_metrics(res, exp, tag):
    m = res.metrics
    assert res.effective_p == exp["effective_p"], tag
    assert m.union_size == exp["union_size"], (tag, m.union_size, exp["union_size"])
    assert m.filtered_count == exp["filtered_count"], (tag, m.filtered_count, exp["filtered_count"])
    assert m.final_size == exp["final_size"], tag


def test_known_answers(engine, golden):
    for ka in golden["known_answers"]:
        k = ka["kind"]
        if k == "skyline":
            got = engine.sfs(np.array(ka["points"], np.float32)).tolist()
        elif k == "relative":
            got = engine.relative_skyline(np.array(ka["r"], np.float32), np.array(ka["c"], np.float32)).astype(int).tolist()
        elif k in ("grid_index", "angular_index"):
            x = np.array([ka["x"]], np.float32)
            strat = Strategy.Grid if k == "grid_index" else Strategy.Angular
            po, _ = engine.make_assignment(x, PartitionConfig(strat, p=1, m=ka["m"]))
            got = int(po[0])
        elif k == "snap":
            from paper_2411_14968_b200 import snap_slices
            got = snap_slices(ka["p"], ka["k"])
        elif k == "assign":
            c = ka["cfg"]
            po, cnt = engine.make_assignment(np.array(ka["points"], np.float32),
                                             PartitionConfig(Strategy(c["strategy"]), p=c["p"]), ka["normalized"])
            got = po.astype(int).tolist()
            assert cnt == ka["count"]
        elif k == "run":
            r = engine.run(np.array(ka["points"], np.float32), to_engine_config(ka["cfg"]), ka["normalized"])
            got = r.skyline.tolist()
            assert r.metrics.local_skyline_sizes == ka["local_skyline_sizes"], ka["src"]
        elif k == "reps":
            got = engine.select_representatives_sorted(np.array(ka["points"], np.float32), ka["partition_of"],
                                                       ka["p"], ka["q"]).tolist()
        else:
            raise AssertionError(k)
        assert got == ka["expect"], (ka["src"], got, ka["expect"])


@pytest.mark.parametrize("local_algo", [LocalAlgo.SFS, LocalAlgo.BNL])
def test_plane_matches_reference(engine, golden, local_algo):
    arr = golden["plane_arrays"]
    for case in golden["plane"]:
        key = case["key"]
        cfg = to_engine_config(case["cfg"])
        cfg.local_algo = local_algo
        cfg.bnl_window_cap = 64  # small window: forces overflow passes
        r = engine.run(arr[key + "_x"], cfg, case["normalized"])
        assert np.array_equal(r.skyline, arr[key + "_ids"]), key
        assert r.metrics.local_skyline_sizes == arr[key + "_lss"].tolist(), key
        check_metrics(r, case, key)


@pytest.mark.parametrize("local_algo", [LocalAlgo.SFS, LocalAlgo.BNL])
def test_plane64_matches_reference(engine, golden, local_algo):
    """FP64 rows through sky_run_f64: the reference's generators and a k/7
    lattice whose values are not float32 (rounding creates ties the doubles
    do not have)."""
    arr = golden["plane64_arrays"]
    for case in golden["plane64"]:
        key = case["key"]
        x = arr[case["x"]]
        cfg = to_engine_config(case["cfg"])
        cfg.local_algo = local_algo
        cfg.bnl_window_cap = 64
        r = engine.run(x, cfg, case["normalized"])
        assert np.array_equal(r.skyline, arr[key + "_ids"]), key
        assert r.metrics.local_skyline_sizes == arr[key + "_lss"].tolist(), key
        check_metrics(r, case, key)


def test_f64_large_vs_oracle(engine):
    """FP64 rows at BASELINE-like sizes: near-ties below float32 resolution."""
    rng = np.random.default_rng(3)
    for it, (strat, filt, sel) in enumerate([(2, 2, 0), (3, 2, 0), (0, 0, 0), (1, 2, 1), (3, 2, 2), (1, 1, 0)]):
        n, d = 30000, 4 + it % 3
        base = (rng.integers(0, 1 << 20, (n, d)) / float(1 << 20))
        x = np.clip(base + rng.integers(-2, 3, (n, d)) * 2.0 ** -40, 0.0, 1.0)  # differences below float32 ulp
        cfg = SkyConfig.make(strategy=strat, p=16, seed=it, slice_dim=0, filter=filt, rep_q=4, merge=1,
                             rep_selection=sel)
        exp = O.oracle_run(x, cfg, True)
        for algo in (LocalAlgo.SFS, LocalAlgo.BNL):
            ecfg = to_engine_config(cfg.as_dict())
            ecfg.local_algo = algo
            r = engine.run(x, ecfg, True)
            assert np.array_equal(r.skyline, exp["ids"]), (it, algo)
            assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), (it, algo)
            check_metrics(r, exp, (it, algo))


@pytest.mark.parametrize("cfg_idx", [1, 2, 3, 4, 5])
def test_baseline_configs_reduced(engine, golden, cfg_idx):
    c = [c for c in golden["configs"] if c["config"] == cfg_idx][0]
    arr = golden["config_arrays"]
    x = generate(c["kind"], c["n"], c["d"], c["seed"])
    assert hashlib.sha256(x.tobytes()).hexdigest() == c["sha256"]
    w = make_config(cfg_idx)
    for algo in (w.config.local_algo, LocalAlgo.SFS if w.config.local_algo == LocalAlgo.BNL else LocalAlgo.BNL):
        w.config.local_algo = algo
        r = engine.run(x, w.config, c["normalized"])
        assert np.array_equal(r.skyline, arr[f"c{cfg_idx}_ids"]), (cfg_idx, algo)
        assert r.metrics.local_skyline_sizes == arr[f"c{cfg_idx}_lss"].tolist(), (cfg_idx, algo)
        check_metrics(r, c, cfg_idx)


def test_random_configs_vs_oracle(engine):
    rng = np.random.default_rng(11)
    for it in range(120):
        d = int(rng.integers(1, 13))
        n = int(rng.integers(0, 3000))
        kind = it % 4
        if kind == 0:
            x = rng.random((n, d), dtype=np.float32)
        elif kind == 1:
            x = (rng.integers(0, 5, (n, d)) / 4).astype(np.float32)
        elif kind == 2:
            x = rng.integers(0, 7, (n, d)).astype(np.float32)
        else:
            x = generate(2, max(n, 1), d, it)[:n] if d > 1 else rng.random((n, d), dtype=np.float32)
        norm = kind != 2
        strat = int(rng.integers(0, 4))
        filt = int(rng.choice([0, 2] + ([1] if strat == 1 else [])))
        cfg = SkyConfig.make(strategy=strat, p=int(rng.integers(1, 40)), seed=int(rng.integers(0, 1000)),
                             slice_dim=int(rng.integers(0, d)), filter=filt, rep_q=int(rng.integers(1, 9)),
                             merge=int(rng.integers(0, 2)), workers=1, rep_selection=int(rng.integers(0, 3)))
        ecfg = to_engine_config(cfg.as_dict())
        ecfg.local_algo = LocalAlgo(it % 2)
        ecfg.bnl_window_cap = int(rng.choice([32, 256, 4096]))
        try:
            exp = O.oracle_run(x, cfg, norm)
        except O.CpuError as e:
            with pytest.raises(Exception) as ei:
                engine.run(x, ecfg, norm)
            assert getattr(ei.value, "code", None) == e.code, (it, e.code, ei.value)
            continue
        r = engine.run(x, ecfg, norm)
        tag = (it, n, d, strat, filt, cfg.merge, ecfg.local_algo)
        assert np.array_equal(r.skyline, exp["ids"]), tag
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), tag
        check_metrics(r, exp, tag)


@pytest.mark.parametrize("cfg_idx", [2, 3, 4, 5])
@pytest.mark.parametrize("sel", [RepSelection.Region, RepSelection.Random])
def test_rep_selection_configs_vs_oracle(engine, cfg_idx, sel):
    """Region / Random representatives (filter.cpp:88-137) on BASELINE-shaped
    inputs; C4 (sliced) exercises the exact scan order of Random picks."""
    w = make_config(cfg_idx, {2: 40000, 3: 60000, 4: 20000, 5: 40000}[cfg_idx])
    x = generate(w.kind, w.n, w.d, 7)
    w.config.rep_selection = sel
    cfg = w.config.to_c()
    try:
        exp = O.oracle_run(x, cfg, w.normalized)
    except O.CpuError as e:
        with pytest.raises(Exception) as ei:
            engine.run(x, w.config, w.normalized)
        assert getattr(ei.value, "code", None) == e.code
        return
    r = engine.run(x, w.config, w.normalized)
    assert np.array_equal(r.skyline, exp["ids"]), (cfg_idx, sel)
    assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist()
    check_metrics(r, exp, (cfg_idx, sel))


def test_skyline_and_relative_vs_oracle(engine):
    rng = np.random.default_rng(5)
    for it in range(30):
        d = int(rng.integers(1, 11))
        x = (rng.integers(0, 6, (int(rng.integers(1, 5000)), d)) / 5).astype(np.float32) if it % 2 else \
            rng.random((int(rng.integers(1, 5000)), d), dtype=np.float32)
        assert np.array_equal(engine.sfs(x), O.bruteforce(x) if len(x) < 1500 else O.oracle_run(
            x, SkyConfig.make(strategy=3, p=1), True)["ids"])
        c = x[rng.integers(0, len(x), int(rng.integers(1, 300)))] * np.float32(0.9)
        assert np.array_equal(engine.relative_skyline(x, c), O.relative_skyline(x, c))


def test_edge_cases(engine):
    cfg = EngineConfig(partition=PartitionConfig(Strategy.Sliced, p=4))
    r = engine.run(np.zeros((0, 3), np.float32), cfg)
    assert r.skyline.size == 0 and r.effective_p == 4
    one = np.array([[0.5, 0.5]], np.float32)
    for s in (Strategy.Random, Strategy.Grid, Strategy.Sliced, Strategy.Angular):
        assert engine.run(one, EngineConfig(partition=PartitionConfig(s, p=3))).skyline.tolist() == [0]
    dup = np.ones((1000, 4), np.float32) * 0.25
    assert engine.run(dup, EngineConfig(partition=PartitionConfig(Strategy.Random, p=7),
                                        filter=FilterKind.Representative, merge=MergeKind.NoSeq)).skyline.size == 1000
    # errors (engine.cpp:19-32, core.cpp:21-46, partition.cpp:26-29)
    x = np.random.default_rng(0).random((10, 2), dtype=np.float32)
    with pytest.raises(ConfigError):
        engine.run(x, EngineConfig(workers=0))
    with pytest.raises(ConfigError):
        engine.run(x, EngineConfig(partition=PartitionConfig(p=0)))
    with pytest.raises(ConfigError):
        engine.run(x, EngineConfig(partition=PartitionConfig(Strategy.Sliced), filter=FilterKind.GridFilter))
    with pytest.raises(ConfigError):
        engine.run(x, EngineConfig(filter=FilterKind.Representative, rep_q=0))
    with pytest.raises(DimensionError):
        engine.run(x[:, :1], EngineConfig(partition=PartitionConfig(Strategy.Angular)))
    with pytest.raises(NormalizationError):
        engine.run(np.array([[3.0, 1.0], [0.5, 2.0]], np.float32), EngineConfig(partition=PartitionConfig(Strategy.Grid)),
                   normalized=False)
    with pytest.raises(DataError):
        engine.run(np.array([[-1.0, 1.0]], np.float32), EngineConfig())
    with pytest.raises(DataError):
        engine.run(np.array([[np.nan, 1.0]], np.float32), EngineConfig())
    with pytest.raises(DataError):
        engine.run(np.array([[0.5, 1.5]], np.float32), EngineConfig(), normalized=True)


def _dominated_by_any(x, t):
    return bool(np.any(np.all(x <= t, axis=1) & np.any(x < t, axis=1)))


@pytest.mark.parametrize("cfg_idx", [1, 2, 3, 4, 5])
def test_full_size_properties(engine, cfg_idx):
    """BASELINE sizes: output is sorted, unique, an antichain on a sample, no
    sampled output row is dominated by any input row, and sampled
    non-output rows are dominated by some output row."""
    w = make_config(cfg_idx)
    x = generate(w.kind, w.n, w.d, 42)
    r = engine.run(x, w.config, w.normalized)
    ids = r.skyline
    assert ids.size > 0 and np.all(np.diff(ids) > 0)
    assert r.metrics.final_size == ids.size <= r.metrics.union_size
    assert r.metrics.union_size == sum(r.metrics.local_skyline_sizes)
    assert r.metrics.union_size <= w.n - r.metrics.filtered_count
    rng = np.random.default_rng(cfg_idx)
    sky = x[ids]
    for t in rng.choice(ids, min(25, ids.size), replace=False):
        assert not _dominated_by_any(x, x[t]), t
    mask = np.ones(w.n, bool)
    mask[ids] = False
    others = np.flatnonzero(mask)
    for t in rng.choice(others, min(200, others.size), replace=False):
        assert _dominated_by_any(sky, x[t]), t
    # determinism (workers-invariance analogue, test_engine.cpp:246-258)
    r2 = engine.run(x, w.config, w.normalized)
    assert np.array_equal(r2.skyline, ids)
    assert r2.metrics.local_skyline_sizes == r.metrics.local_skyline_sizes


def test_full_c1_vs_oracle(engine):
    w = make_config(1)
    x = generate(w.kind, w.n, w.d, 42)
    exp = O.oracle_run(x, w.config.to_c(), w.normalized)
    r = engine.run(x, w.config, w.normalized)
    assert np.array_equal(r.skyline, exp["ids"])
    assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist()
    check_metrics(r, exp, "c1")


@pytest.mark.parametrize("n,p,seed", [(2, 1, 0), (3, 2, 5), (1000, 7, 42), (65_537, 32, 42), (2_000_000, 32, 42),
                                      (100_000, 8, 42), (300_001, 5, 123456789)])
def test_random_assignment_matches_reference_shuffle(engine, n, p, seed):
    """assign_random (partition.cpp:36-54) resolved on the GPU must equal the
    sequential Fisher-Yates with mt19937_64 (rng.hpp:40-60)."""
    x = np.zeros((n, 2), np.float32)
    po, cnt = engine.make_assignment(x, PartitionConfig(Strategy.Random, p=p, seed=seed))
    perm = O.random_permutation(n, seed)
    exp = np.empty(n, np.uint64)
    exp[perm] = np.arange(n, dtype=np.uint64) % p
    assert cnt == p
    assert np.array_equal(po, exp)


def test_distributed_context_single_rank():
    """The NCCL-backed context (world = 1 on this box) runs the same path and
    returns the reference result."""
    from paper_2411_14968_b200 import Engine, nccl_unique_id
    eng = Engine.distributed(0, 0, 1, nccl_unique_id())
    try:
        for idx, n in ((2, 30_000), (4, 8_000), (3, 200_000)):
            w = make_config(idx, n)
            x = generate(w.kind, w.n, w.d, 42)
            exp = O.oracle_run(x, w.config.to_c(), w.normalized)
            r = eng.run(x, w.config, w.normalized)
            assert np.array_equal(r.skyline, exp["ids"])
            assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist()
    finally:
        eng.close()


@pytest.mark.parametrize("stream", ["1", "0"])
def test_stream_path_forced(engine, golden, options, stream):
    """The stream path (sorted representatives from per-partition candidate
    buckets, row-order prefilter that appends survivor keys, survivors-only
    sort; engine.cu `stream`) and the sorted path, each forced at sizes the
    oracle finishes quickly: the golden plane, the reduced BASELINE configs
    and random configurations."""
    options(stream=int(stream))
    test_plane_matches_reference(engine, golden, LocalAlgo.SFS)
    for idx in (2, 3, 5):
        test_baseline_configs_reduced(engine, golden, idx)
    test_random_configs_vs_oracle(engine)


@pytest.mark.parametrize("cap_sync", [1, 0])
def test_filtered_capacity_modes(engine, golden, options, cap_sync):
    """Both sizings of the filtered set (engine.cu kExactCapRows): the exact
    count read back before the local phase, and the input's size as capacity
    with every later pass bounded by the device count; SFS and BNL (small
    window: overflow passes) local phases."""
    options(cap_sync=cap_sync)
    test_plane_matches_reference(engine, golden, LocalAlgo.SFS)
    test_plane_matches_reference(engine, golden, LocalAlgo.BNL)
    for idx in (1, 2, 3, 4, 5):
        test_baseline_configs_reduced(engine, golden, idx)
    test_random_configs_vs_oracle(engine)


def test_stream_path_bucket_overflow(engine, options):
    """Candidate buckets that fill up (duplicate-heavy rows, rows sorted by
    partition): the run is redone with 8,192-slot buckets, and on the sorted
    path when those overflow too (20,000 identical rows), with identical
    results."""
    options(stream=1)
    rng = np.random.default_rng(3)
    cases = [
        np.zeros((6000, 3), np.float32),                                   # every row identical
        np.zeros((20000, 3), np.float32),                                  # more duplicates than the large buckets hold
        np.repeat(rng.random((3, 4), dtype=np.float32), 3000, axis=0),     # three values, 3000 copies
        np.sort(rng.random((20000, 4), dtype=np.float32), axis=0),         # partitions concentrated by row
        rng.integers(0, 3, (20000, 5)).astype(np.float32) / 2,             # lattice ties
    ]
    for k, x in enumerate(cases):
        for strat, p in ((1, 2), (0, 16), (2, 16)):
            cfg = SkyConfig.make(strategy=strat, p=p, m=p if strat == 1 else 0, seed=k, filter=2, rep_q=5, merge=1,
                                 workers=1)
            exp = O.oracle_run(x, cfg, True)
            r = engine.run(x, to_engine_config(cfg.as_dict()), True)
            assert np.array_equal(r.skyline, exp["ids"]), (k, strat)
            check_metrics(r, exp, (k, strat))
            assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), (k, strat)


@pytest.mark.parametrize("m", [2, 3, 4, 8])
def test_angular_boundaries_vs_oracle(engine, m):
    """Angular partition ids on lattice rows that sit exactly on slice
    boundaries (x_i^2 == tail sums, zeros, -0.0): the tangent-ratio filter
    (k_prep_stream) must defer every such row to the exact FP64 path."""
    rng = np.random.default_rng(100 + m)
    for d in (2, 3, 4, 6):
        x = (rng.integers(0, 5, (3000, d)) / 4).astype(np.float32)
        x[:50] = 0.0
        x[50:100, 0] = -0.0
        x[100:110] = 0.5
        cfg = SkyConfig.make(strategy=2, p=m ** (d - 1), m=m, seed=1, filter=0, merge=1, workers=1)
        exp = O.oracle_run(x, cfg, True)
        r = engine.run(x, to_engine_config(cfg.as_dict()), True)
        assert np.array_equal(r.skyline, exp["ids"]), (m, d)
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), (m, d)
        po, _ = engine.make_assignment(x, PartitionConfig(Strategy.Angular, p=m ** (d - 1), m=m))
        epo, _ = O.oracle_assign(x, cfg, True)
        assert np.array_equal(np.asarray(po), np.asarray(epo)), (m, d)


@pytest.mark.parametrize("m", [2, 4])
def test_angular_many_boundary_rows(engine, m):
    """Integer rows put hundreds of thousands of angles exactly on a slice
    boundary (x_i == x_j gives atan2 = pi/4): all of them are decided on the
    device (no host fix-up, no cap). Partition ids vs the
    reference itself, and a full run vs the reference."""
    x = generate(5, 2_000_000, 5, 42)
    cfg = SkyConfig.make(strategy=2, p=m ** 4, m=m, seed=1, filter=2, rep_q=5, merge=1, workers=8)
    po, _ = engine.make_assignment(x, PartitionConfig(Strategy.Angular, p=m ** 4, m=m), False)
    if O.ref_available():
        epo, _ = O.oracle_assign(x, cfg, False, ref=True)
        assert np.array_equal(np.asarray(po), np.asarray(epo))
        exp = O.ref_run(x, cfg, False)
    else:
        exp = O.oracle_run(x, cfg, False)
    r = engine.run(x, to_engine_config(cfg.as_dict()), False)
    assert r.metrics.angular_host_fixups == 0
    assert np.array_equal(r.skyline, exp["ids"])
    check_metrics(r, exp, m)
    assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist()


def test_angular_libm_latitude_rows_vs_oracle(engine):
    """k/7 lattice rows whose angle sits within one ulp of pi/4 (y = sqrt(x^2)
    rounded, not equal to x): the reference's slice depends on the host
    libm's rounding there, so those rows take the batched host fix-up."""
    rng = np.random.default_rng(7)
    x = (rng.integers(0, 8, (200_000, 3)) / 7).astype(np.float64)
    for m in (2, 4):
        cfg = SkyConfig.make(strategy=2, p=m ** 2, m=m, seed=1, filter=0, merge=1, workers=1)
        epo, _ = O.oracle_assign(x.astype(np.float32), cfg, True)
        po, _ = engine.make_assignment(x.astype(np.float32), PartitionConfig(Strategy.Angular, p=m ** 2, m=m))
        assert np.array_equal(np.asarray(po), np.asarray(epo)), m
        exp = O.oracle_run(x, cfg, True)
        r = engine.run(x, to_engine_config(cfg.as_dict()), True)
        assert np.array_equal(r.skyline, exp["ids"]), m
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), m


def test_stream_path_many_representatives(engine, options):
    """Stream path with more representatives than its shared-memory
    reservation (256): the prefilter reads the rest from global memory."""
    options(stream=1)
    for d, m, q in ((7, 2, 8), (5, 3, 6)):
        x = generate(2, 60000, d, 5)
        cfg = SkyConfig.make(strategy=2, p=m ** (d - 1), m=m, seed=3, filter=2, rep_q=q, merge=1, workers=1)
        exp = O.oracle_run(x, cfg, True)
        r = engine.run(x, to_engine_config(cfg.as_dict()), True)
        assert r.metrics.n_reps > 256, r.metrics.n_reps
        assert np.array_equal(r.skyline, exp["ids"]), (d, m)
        check_metrics(r, exp, (d, m))
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), (d, m)


@pytest.mark.parametrize("host_merge", ["0", "1"])
def test_device_merge_vs_oracle(engine, options, host_merge):
    """The all-pairs merge planned on the device with the ids written to
    mapped host memory (one round trip per step) and the host-planned merge,
    on inputs whose filtered set is large enough to take the device path."""
    options(host_merge=int(host_merge))
    for strat, p, merge, seed in ((2, 64, 1, 1), (0, 16, 1, 2), (0, 8, 0, 3)):
        x = generate(2, 150000, 6, seed)
        cfg = SkyConfig.make(strategy=strat, p=p, seed=seed, filter=2, rep_q=8, merge=merge, workers=1)
        exp = O.oracle_run(x, cfg, True)
        r = engine.run(x, to_engine_config(cfg.as_dict()), True)
        tag = (strat, p, merge, host_merge)
        assert np.array_equal(r.skyline, exp["ids"]), tag
        check_metrics(r, exp, tag)
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), tag


def test_chunked_input_copy_vs_oracle(engine):
    """Host inputs of 4 MB and more are copied in four chunks whose prep
    starts as each lands: the same result as the oracle (angular, sliced)."""
    x = generate(2, 200000, 6, 9)
    assert x.nbytes >= 4 << 20
    for strat, p in ((2, 64), (3, 16)):
        cfg = SkyConfig.make(strategy=strat, p=p, seed=4, filter=2, rep_q=8, merge=1, workers=1)
        exp = O.oracle_run(x, cfg, True)
        r = engine.run(x, to_engine_config(cfg.as_dict()), True)
        assert np.array_equal(r.skyline, exp["ids"]), strat
        check_metrics(r, exp, strat)
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), strat


def test_repeated_runs_reuse_buffers(engine):
    """Repeated runs of one shape (arena buffers, pinned result memory and
    launch-shape caches reused), then another input: every run exact."""
    x = generate(2, 150000, 6, 21)
    cfg = SkyConfig.make(strategy=2, p=64, seed=2, filter=2, rep_q=8, merge=1, workers=1)
    exp = O.oracle_run(x, cfg, True)
    ecfg = to_engine_config(cfg.as_dict())
    for it in range(5):
        r = engine.run(x, ecfg, True)
        assert np.array_equal(r.skyline, exp["ids"]), it
        check_metrics(r, exp, it)
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), it
    # a different input afterwards (other key or the same one): still exact
    y = generate(2, 150000, 6, 22)
    exp2 = O.oracle_run(y, cfg, True)
    for it in range(3):
        r = engine.run(y, ecfg, True)
        assert np.array_equal(r.skyline, exp2["ids"]), ("y", it)
        check_metrics(r, exp2, ("y", it))


@pytest.mark.parametrize("small_tail", ["1", "0"])
def test_stream_small_tail_vs_oracle(engine, options, small_tail):
    """Stream path whose prefilter leaves at most kSmallCap (4096) rows: the
    fused tail (small.cu: sort, local skylines, union, merge, ids in five
    launches and one round trip) against the oracle, and the general tail
    (small_tail=0) on the same inputs; inputs with more survivors make the
    fused tail decline and hand over to the general one."""
    options(stream=1, small_tail=int(small_tail))
    rng = np.random.default_rng(11)
    cases = [
        (generate(3, 200_000, 8, 3), 1, 2, 256),                           # C3-like: correlated, grid 2^8
        (np.zeros((3000, 3), np.float32), 1, 2, 8),                         # identical rows: all survive, no dominance
        ((rng.integers(0, 3, (20000, 5)) / 2).astype(np.float32), 1, 3, 243),  # lattice ties
        (generate(2, 50_000, 4, 4), 1, 4, 256),                             # anticorrelated: > 4096 survivors
        (generate(1, 100_000, 5, 5), 0, 0, 32),                             # random partitions
        (generate(1, 100_000, 6, 6), 2, 2, 32),                             # angular
        (generate(5, 100_000, 5, 7), 0, 0, 16),                             # integer rows, one dominator
    ]
    for k, (x, strat, m, p) in enumerate(cases):
        cfg = SkyConfig.make(strategy=strat, p=p, m=m, seed=k, filter=2, rep_q=5, merge=1, workers=1)
        normalized = bool(x.max() <= 1.0)
        exp = O.oracle_run(x, cfg, normalized)
        r = engine.run(x, to_engine_config(cfg.as_dict()), normalized)
        tag = (k, small_tail)
        assert np.array_equal(r.skyline, exp["ids"]), tag
        check_metrics(r, exp, tag)
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), tag


@pytest.mark.parametrize("m,d", [(2, 3), (3, 4), (5, 3), (1, 4), (2, 10), (4, 9), (2, 17)])
def test_grid_filter_cell_antichain_vs_oracle(engine, m, d):
    """grid_filter (filter.cpp:37-50) on the device: the per-axis prefix OR of
    the cell occupancy against the reference's pair loop, from a handful of
    cells up to m^d = 262,144 (the multi-launch path, above 32,768 cells)."""
    rng = np.random.default_rng(m * 100 + d)
    for n, spread in ((400, 1.0), (3000, 1.0), (3000, 0.45)):
        x = rng.random((n, d), dtype=np.float32)
        # rows pushed towards the far corner leave the near cells empty, so
        # few cells are filtered; the full spread filters most of them
        x = (1.0 - spread + spread * x).astype(np.float32)
        for merge in (0, 1):
            cfg = SkyConfig.make(strategy=1, p=m ** d, filter=1, merge=merge, workers=1)
            exp = O.oracle_run(x, cfg, True)
            r = engine.run(x, to_engine_config(cfg.as_dict()), True)
            tag = (m, d, n, spread, merge)
            assert np.array_equal(r.skyline, exp["ids"]), tag
            assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), tag
            check_metrics(r, exp, tag)


@pytest.mark.parametrize("d", [17, 24, 32])
def test_wide_rows_vs_oracle(engine, d):
    """16 < d <= 32 runs on the exact-compare core (no packed codes): every
    strategy x filter x merge x local algorithm against the oracle."""
    rng = np.random.default_rng(d)
    for n in (1, 1500):
        x = rng.random((n, d), dtype=np.float32)
        x[:, : d - 3] = np.round(x[:, : d - 3] * 2) / 2  # few distinct values: the skyline is a fraction of the rows
        for strat in range(4):
            for filt in ((0, 1, 2) if strat == 1 else (0, 2)):
                for merge in (0, 1):
                    for algo in (0, 1):
                        sel = (strat + merge + algo) % 3 if filt == 2 else 0
                        p = 2 ** 17 if strat == 1 and d == 17 else 9
                        cfg = SkyConfig.make(strategy=strat, p=p, seed=3, slice_dim=d - 1, filter=filt, rep_q=4,
                                             merge=merge, workers=1, rep_selection=sel)
                        try:
                            exp = O.oracle_run(x, cfg, True)
                        except O.CpuError:
                            continue  # e.g. a grid whose m^d overflows: covered by test_edge_cases
                        ecfg = to_engine_config(cfg.as_dict())
                        ecfg.local_algo = LocalAlgo(algo)
                        ecfg.bnl_window_cap = 64
                        r = engine.run(x, ecfg, True)
                        tag = (d, n, strat, filt, merge, algo, sel)
                        assert np.array_equal(r.skyline, exp["ids"]), tag
                        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), tag
                        check_metrics(r, exp, tag)


@pytest.mark.parametrize("d", [16, 20])
def test_bnl_many_passes(engine, d):
    """BNL with a 16-tuple window over one partition of mostly incomparable
    rows: more than 256 overflow passes (the window records its tuples' pass
    modulo 256; the d > 16 kernel used to spin forever past pass 255)."""
    rng = np.random.default_rng(7)
    x = (rng.integers(0, 4, (12000 if d == 16 else 6000, d)) / 3).astype(np.float32)
    cfg = SkyConfig.make(strategy=3, p=1, slice_dim=0, merge=1, workers=1)
    exp = O.oracle_run(x, cfg, True)
    assert len(exp["ids"]) > 256 * 16
    ecfg = to_engine_config(cfg.as_dict())
    ecfg.local_algo = LocalAlgo.BNL
    ecfg.bnl_window_cap = 16
    r = engine.run(x, ecfg, True)
    assert np.array_equal(r.skyline, exp["ids"])
    check_metrics(r, exp, d)


@pytest.mark.parametrize("case", [
    # (d, data, strategy, p, q, rep_selection): thousands of representatives (past the prefilter's shared
    # memory) and partition counts past the streamed prep pass's per-partition tables
    (11, "uniform", 1, 3 ** 11, 1, 0),
    (16, "lattice", 1, 2 ** 16, 30, 1),
    (16, "lattice", 1, 2 ** 16, 8, 2),
    (11, "f64", 3, 1000, 30, 2),
    (8, "uniform", 0, 5000, 100, 0),
])
def test_many_representatives_and_partitions(engine, case):
    d, data, strat, p, q, sel = case
    rng = np.random.default_rng(d * 1000 + q)
    n = 5000
    if data == "uniform":
        x = rng.random((n, d), dtype=np.float32)
    elif data == "lattice":
        x = (rng.integers(0, 4, (n, d)) / 3).astype(np.float32)
    else:
        x = np.clip(rng.integers(0, 1 << 12, (n, d)) / float(1 << 12) + rng.integers(-2, 3, (n, d)) * 2.0 ** -40, 0, 1)
    for merge in (0, 1):
        cfg = SkyConfig.make(strategy=strat, p=p, seed=9, slice_dim=d - 1, filter=2, rep_q=q, merge=merge, workers=1,
                             rep_selection=sel)
        exp = O.oracle_run(x, cfg, True)
        for algo in (LocalAlgo.SFS, LocalAlgo.BNL):
            ecfg = to_engine_config(cfg.as_dict())
            ecfg.local_algo = algo
            r = engine.run(x, ecfg, True)
            tag = (case, merge, algo)
            assert np.array_equal(r.skyline, exp["ids"]), tag
            assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), tag
            check_metrics(r, exp, tag)


def test_baseline_sized_random_configs_vs_reference(engine):
    """Random configurations at BASELINE-like sizes (100k-1.5M rows of the
    BASELINE generators) with the engine's default options, so the stream
    path (inputs over 32 MB), the device-planned merges and the indexed merge
    take their production branches, against the reference itself
    (oracle/_ref, all host threads). scripts/fuzz_gpu_big.py runs the long
    version of this sweep."""
    if not O.ref_available():
        pytest.skip("oracle/_ref/libskyref.so was not built")
    import os
    rng = np.random.default_rng(2411)
    for it in range(16):
        d = int(rng.choice([3, 4, 5, 6, 8]))
        n = int(rng.choice([100_000, 300_000, 1_000_000, 1_500_000]))
        kind = int(rng.choice([1, 3, 3, 5, 2]))
        if kind == 2 and n > 300_000:
            kind = 3
        x = generate(kind, n, d, int(rng.integers(1 << 30)))
        norm = kind != 5
        strat = int(rng.integers(0, 4))
        filt = int(rng.choice([0, 2, 2] + ([1] if strat == 1 else [])))
        p = int(rng.choice([2, 3])) ** d if strat == 1 else int(rng.choice([8, 32, 128, 500]))
        if kind == 5 and strat == 1:  # integers are outside [0, 1]: the grid raises (test_edge_cases)
            strat, p, filt = 0, 32, 2 if filt == 1 else filt
        sel = int(rng.choice([0, 0, 1, 2])) if filt == 2 and norm else 0
        cfg = SkyConfig.make(strategy=strat, p=p, seed=int(rng.integers(0, 1000)), slice_dim=int(rng.integers(0, d)),
                             filter=filt, rep_q=int(rng.choice([1, 5, 8, 20])), merge=int(rng.integers(0, 2)),
                             workers=os.cpu_count() or 8, rep_selection=sel)
        exp = O.ref_run(x, cfg, norm)
        ecfg = to_engine_config(cfg.as_dict())
        ecfg.local_algo = LocalAlgo(it % 2)
        r = engine.run(x, ecfg, norm)
        tag = (it, n, d, kind, strat, p, filt, sel, cfg.merge, it % 2)
        assert np.array_equal(r.skyline, exp["ids"]), tag
        assert r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist(), tag
        check_metrics(r, exp, tag)
