"""Multi-rank decomposition of sky_run, on CPU with gloo (world_size 2).

The NCCL path of libskyline_b200 shards the local phase by the partition
ranges of sky_plan_local_shards and the merge by the candidate-partition
ranges of sky_plan_merge_shards, all-gathering local skylines and survivor
ids. Here two gloo processes execute that exact decomposition, with the CPU
oracle standing in for the GPU kernels, and must reproduce the
single-process reference result (ids and local_skyline_sizes)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2411_14968_b200 import (EngineConfig, FilterKind, MergeKind, PartitionConfig, Strategy,
                                   plan_local_shards, plan_merge_shards, snap_slices)


def _cases():
    rng = np.random.default_rng(3)
    out = []
    for strat in (Strategy.Random, Strategy.Grid, Strategy.Angular, Strategy.Sliced):
        for filt in (FilterKind.None_, FilterKind.Representative):
            for merge in (MergeKind.Sequential, MergeKind.NoSeq):
                d = 3
                x = rng.random((700, d), dtype=np.float32) if strat != Strategy.Grid or True else None
                if strat == Strategy.Sliced:
                    x[:200] = (rng.integers(0, 4, (200, d)) / 3).astype(np.float32)  # ties on the slice dim
                cfg = EngineConfig(partition=PartitionConfig(strat, p=7, seed=5, slice_dim=0), filter=filt, rep_q=3,
                                   merge=merge)
                out.append((x, cfg))
    return out


def _pd(strategy, i, P, m, d, sizes):
    """potential_dominators (engine.cpp:74-114) as partition indices."""
    if strategy in (Strategy.Random, Strategy.Angular):
        return [j for j in range(P) if j != i]
    if strategy == Strategy.Sliced:
        return list(range(i))
    ci = [(i // m ** k) % m for k in range(d)]
    res = []
    for j in range(P):
        if j == i or sizes[j] == 0:
            continue
        cj = [(j // m ** k) % m for k in range(d)]
        if cj != ci and all(a <= b for a, b in zip(cj, ci)):
            res.append(j)
    return res


def _rank_run(rank, world, x, cfg):
    c = cfg.to_c()
    po, P = O.oracle_assign(x, c, True)
    d = x.shape[1]
    m = cfg.partition.m or (snap_slices(cfg.partition.p, d) if cfg.partition.strategy == Strategy.Grid else
                            snap_slices(cfg.partition.p, d - 1) if cfg.partition.strategy == Strategy.Angular else 0)
    parts = [np.flatnonzero(po == p) for p in range(P)]
    # phase 1a (replicated): representatives + prefilter
    if cfg.filter == FilterKind.Representative:
        reps = O.representatives(x, po, P, cfg.rep_q)
        parts = [ix[O.relative_skyline(x[ix], x[reps])] if len(ix) and len(reps) else ix for ix in parts]
    off = np.zeros(P + 1, np.uint32)
    off[1:] = np.cumsum([len(ix) for ix in parts])
    # local phase: this rank's partition range
    b = plan_local_shards(off, world)
    mine = {p: parts[p][np.asarray(O.bruteforce(x[parts[p]]), dtype=np.int64)] if len(parts[p]) else parts[p]
            for p in range(int(b[rank]), int(b[rank + 1]))}
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    locals_ = {}
    for g in gathered:
        assert not (set(g) & set(locals_)), "partition computed by two ranks"
        locals_.update(g)
    assert sorted(locals_) == list(range(P)), "partition not covered"
    sizes = [len(locals_[p]) for p in range(P)]
    offu = np.zeros(P + 1, np.uint32)
    offu[1:] = np.cumsum(sizes)
    # merge phase: this rank's candidate partitions
    mb = plan_merge_shards(offu, world, cfg, d, m)
    surv = []
    for i in range(int(mb[rank]), int(mb[rank + 1])):
        u = locals_[i]
        if not len(u):
            continue
        if cfg.merge == MergeKind.Sequential:
            comp = np.concatenate([locals_[j] for j in range(P)])
        else:
            pdl = _pd(cfg.partition.strategy, i, P, m, d, sizes)
            comp = np.concatenate([locals_[j] for j in pdl]) if pdl else np.zeros(0, np.int64)
        keep = O.relative_skyline(x[u], x[comp]) if len(comp) else np.ones(len(u), bool)
        surv.extend(u[keep].tolist())
    allsurv = [None] * world
    dist.all_gather_object(allsurv, surv)
    ids = np.sort(np.array([v for s in allsurv for v in s], np.int64))
    return ids, sizes


def _first_q(x, rows, q):
    """The first q rows by (FP64 coordinate sum, lex coords, id)
    (filter.cpp:74-79), rows ascending ids."""
    if not len(rows):
        return rows
    xr = x[rows].astype(np.float64)
    s = np.zeros(len(rows))
    for j in range(x.shape[1]):
        s = s + xr[:, j]  # left to right, as coord_sum
    keys = [rows] + [xr[:, j] for j in range(x.shape[1] - 1, -1, -1)] + [s]
    return rows[np.lexsort(keys)][:q]


def _rank_run_sharded(rank, world, x, cfg):
    """shard.cu's phase 1 restated: this rank's rows only, shard-local first q
    per partition, all-gathered, global first q of the W*q candidates,
    pruned; prefilter of the own rows; survivors routed to partition owners;
    local skylines by the owners; then the merge of _rank_run."""
    c = cfg.to_c()
    po, P = O.oracle_assign(x, c, True)
    N, d = x.shape
    r0, r1 = N * rank // world, N * (rank + 1) // world
    own = np.arange(r0, r1)
    q = min(cfg.rep_q, N)
    survivors = own
    if cfg.filter == FilterKind.Representative:
        picks = {p: _first_q(x, own[po[own] == p], q).tolist() for p in range(P)}
        gathered = [None] * world
        dist.all_gather_object(gathered, picks)
        cand = []
        for p in range(P):
            allp = np.array(sorted(v for g in gathered for v in g[p]), np.int64)
            cand.extend(_first_q(x, allp, q).tolist())
        cand = np.array(cand, np.int64)
        reps = cand[O.bruteforce(x[cand])] if len(cand) else cand  # prune_dominated_reps
        assert np.array_equal(np.sort(reps), O.representatives(x, po, P, cfg.rep_q)), "global reps differ"
        if len(reps) and len(own):
            survivors = own[O.relative_skyline(x[own], x[reps])]
    # routing: owners of contiguous partition ranges balanced by |r_i|^2
    counts = np.bincount(po[survivors].astype(np.int64), minlength=P)
    allc = [None] * world
    dist.all_gather_object(allc, counts.tolist())
    tot = np.sum(np.array(allc, np.int64), axis=0)
    offs = np.zeros(P + 1, np.uint32)
    offs[1:] = np.cumsum(tot)
    pr = plan_local_shards(offs, world)
    outbox = [[int(v) for v in survivors if pr[k] <= po[v] < pr[k + 1]] for k in range(world)]
    inbox = [None] * world
    dist.all_gather_object(inbox, outbox)
    mine = np.array(sorted(v for box in inbox for v in box[rank]), np.int64)
    local = {}
    for p in range(int(pr[rank]), int(pr[rank + 1])):
        rows = mine[po[mine] == p]
        local[p] = rows[np.asarray(O.bruteforce(x[rows]), dtype=np.int64)] if len(rows) else rows
    return local, int(N - offs[P])


def _worker_sharded(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for k, (x, cfg) in enumerate(_cases()):
            local, filtered = _rank_run_sharded(rank, world, x, cfg)
            gathered = [None] * world
            dist.all_gather_object(gathered, local)
            if rank == 0:
                ref = O.oracle_run(x, cfg.to_c(), True)
                merged = {}
                for g in gathered:
                    merged.update(g)
                sizes = [len(merged.get(p, [])) for p in range(len(ref["local_skyline_sizes"]))]
                results[k] = (sizes == ref["local_skyline_sizes"].astype(int).tolist(),
                              filtered == int(ref["filtered_count"]))
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for k, (x, cfg) in enumerate(_cases()):
            ids, sizes = _rank_run(rank, world, x, cfg)
            if rank == 0:
                ref = O.oracle_run(x, cfg.to_c(), True)
                results[k] = (np.array_equal(ids, ref["ids"]),
                              sizes == ref["local_skyline_sizes"].astype(int).tolist())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_decomposition_matches_single_process(world):
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        results = mgr.dict()
        mp.start_processes(_worker, args=(world, _free_port(), results), nprocs=world, join=True,
                           start_method="spawn")
        res = dict(results)
    assert len(res) == len(_cases())
    for k, (ok_ids, ok_sizes) in res.items():
        assert ok_ids and ok_sizes, k


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_phase1_matches_single_process(world):
    """Row-sharded phase 1 (shard.cu): shard-local representative picks merged
    into the global first q reproduce the reference's representatives, and
    the routed, owner-computed local skylines and the filtered count equal
    the single-process result."""
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        results = mgr.dict()
        mp.start_processes(_worker_sharded, args=(world, _free_port(), results), nprocs=world, join=True,
                           start_method="spawn")
        res = dict(results)
    assert len(res) == len(_cases())
    for k, (ok_sizes, ok_filtered) in res.items():
        assert ok_sizes and ok_filtered, k


def test_shard_plans_cover_and_balance():
    off = np.array([0, 10, 10, 500, 520, 530, 2000], np.uint32)
    for w in (1, 2, 3, 4, 8):
        b = plan_local_shards(off, w)
        assert b[0] == 0 and b[-1] == len(off) - 1 and np.all(np.diff(b.astype(int)) >= 0)
    cfg = EngineConfig(partition=PartitionConfig(Strategy.Sliced, p=6), merge=MergeKind.NoSeq)
    b = plan_merge_shards(off, 2, cfg, 4)
    # sliced: later slices carry more potential dominators -> the split leans late
    assert 0 < b[1] <= 6 and b[-1] == 6
