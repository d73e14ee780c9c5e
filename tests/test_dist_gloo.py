"""World-size-2 gloo tests (CPU) of the point-sharded path's host logic: shard
ranges, the ncclUniqueId broadcast, max-over-ranks timing, and the algebra of the per-iteration
packed allreduce — per-rank partial [sums | counts | SSE | changed] from each shard, summed
across ranks and finalised, equal the single-process Lloyd step (oracle on the full data)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_12208_b200 import dist as pd
        out = {}
        # 1. shard ranges
        n = 100_003
        out["shard"] = pd.shard_range(n, world, rank)
        # 2. unique-id broadcast (rank 0's bytes reach every rank)
        nid = bytes(range(128)) if rank == 0 else None
        out["nid"] = pd.broadcast_nccl_id(nid)
        # 3. max over ranks
        out["max"] = pd.max_over_ranks(float(rank) * 2.5 + 1.0)
        # 4. packed allreduce algebra on a C5-shaped (reduced) problem
        N, k = 6_000, 24
        X, _, _ = synth.make("c3_blobs_1m_d64", n=N, seed=7)
        Xn, _, _ = oracle.normalize(X, "zscore", work="fp32")
        Xn = Xn.astype(np.float32).astype(np.float64)
        C = Xn[:k].copy()
        r0, r1 = pd.shard_range(N, world, rank)
        st = oracle.step(Xn[r0:r1], C, work="fp32", dist="fp16")
        L = pd.packed_layout(k, 64)
        buf = np.zeros(L["total"])
        buf[L["sums"]:L["counts"]] = st["sums"].ravel()
        buf[L["counts"]:L["sse"]] = st["counts"]
        buf[L["sse"]] = np.maximum(st["dmin"], 0).sum()
        buf[L["changed"]] = (r1 - r0)
        t = torch.from_numpy(buf)
        tdist.all_reduce(t)
        g = t.numpy()
        cnt = g[L["counts"]:L["sse"]]
        sums = g[L["sums"]:L["counts"]].reshape(k, 64)
        newc = np.where(cnt[:, None] > 0,
                        (sums / np.maximum(cnt, 1)[:, None]).astype(np.float32).astype(np.float64),
                        C)
        out["cnt"], out["newc"], out["sse"], out["changed"] = cnt, newc, g[L["sse"]], g[L["changed"]]
        q.put((rank, out))
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shard ranges: disjoint, ordered, covering [0, n)
    assert res[0]["shard"] == (0, 50_002) and res[1]["shard"] == (50_002, 100_003)
    assert res[0]["nid"] == res[1]["nid"] == bytes(range(128))
    assert res[0]["max"] == res[1]["max"] == 3.5
    # allreduced partials == full-data Lloyd step, identical on both ranks
    N, k = 6_000, 24
    X, _, _ = synth.make("c3_blobs_1m_d64", n=N, seed=7)
    Xn, _, _ = oracle.normalize(X, "zscore", work="fp32")
    Xn = Xn.astype(np.float32).astype(np.float64)
    full = oracle.step(Xn, Xn[:k].copy(), work="fp32", dist="fp16")
    for r in (0, 1):
        assert np.array_equal(res[r]["cnt"], full["counts"])
        assert np.array_equal(res[r]["newc"], res[0]["newc"])
        assert np.allclose(res[r]["newc"], full["centroids"], rtol=2e-7, atol=1e-7)
        assert res[r]["changed"] == N
        assert abs(res[r]["sse"] - np.maximum(full["dmin"], 0).sum()) <= 1e-9 * res[r]["sse"]


def _fx_q_vec(x, e):
    """Vectorised host model of k_update.cu fx_q (see tests/test_fx_grid.py): per-feature
    exponents e (2^e > max |x|), float32 IEEE round-to-nearest operations."""
    x = x.astype(np.float32)
    c1 = (1.5 * np.exp2(e + 1.0)).astype(np.float32)
    c2 = (1.5 * np.exp2(e - 22.0)).astype(np.float32)
    t1 = (x + c1).astype(np.float32)
    r = (x - (t1 - c1).astype(np.float32)).astype(np.float32)
    t2 = (r + c2).astype(np.float32)
    i1 = t1.view(np.int32).astype(np.int64) - c1.view(np.int32).astype(np.int64)
    i2 = t2.view(np.int32).astype(np.int64) - c2.view(np.int32).astype(np.int64)
    return i1, i2


def _fx_worker(rank, world, port, q):
    """One rank of the fixed-point exchange (R9): per-feature grid from
    the max-allreduced column maxima, this shard's int64 totals (sum of i1, sum of i2) and int32
    counts per cluster, int64 / int32 sum allreduces."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_12208_b200 import dist as pd
        N, k, d = 7_001, 17, 24
        X, _, _ = synth.make("c3_blobs_1m_d64", n=N, seed=11)
        X = X[:, :d].astype(np.float32)
        lab = oracle.assign(X, X[:k], work="fp32", dist="fp32")[0]
        r0, r1 = pd.shard_range(N, world, rank)
        amax = torch.from_numpy(np.abs(X[r0:r1]).max(0).astype(np.float32))
        tdist.all_reduce(amax, op=tdist.ReduceOp.MAX)
        e = np.frexp(amax.numpy().astype(np.float64))[1].astype(np.float64)
        i1, i2 = _fx_q_vec(X[r0:r1], e[None, :])
        Shi = np.zeros((k, d), np.int64)
        Slo = np.zeros((k, d), np.int64)
        np.add.at(Shi, lab[r0:r1], i1)
        np.add.at(Slo, lab[r0:r1], i2)
        cnt = np.bincount(lab[r0:r1], minlength=k).astype(np.int32)
        ts = [torch.from_numpy(Shi), torch.from_numpy(Slo), torch.from_numpy(cnt)]
        for t in ts:
            tdist.all_reduce(t)
        q.put((rank, {"Shi": ts[0].numpy(), "Slo": ts[1].numpy(), "cnt": ts[2].numpy(),
                      "e": e}))
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_fixed_point_totals():
    """The fp32-work exchange of the library (int64 totals of the grid integers, int32 counts):
    the allreduced totals equal the single-process totals EXACTLY (integer sums are order-free),
    and the finalised centres round_fp32((Shi 2^23 + Slo) g / count) are the rounded exact means
    of eq:center to one ulp — identical on every rank."""
    from fractions import Fraction
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fx_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, k, d = 7_001, 17, 24
    X, _, _ = synth.make("c3_blobs_1m_d64", n=N, seed=11)
    X = X[:, :d].astype(np.float32)
    lab = oracle.assign(X, X[:k], work="fp32", dist="fp32")[0]
    e = np.frexp(np.abs(X).max(0).astype(np.float64))[1].astype(np.float64)
    assert np.array_equal(res[0]["e"], e) and np.array_equal(res[1]["e"], e)
    i1, i2 = _fx_q_vec(X, e[None, :])
    Shi = np.zeros((k, d), np.int64)
    Slo = np.zeros((k, d), np.int64)
    np.add.at(Shi, lab, i1)
    np.add.at(Slo, lab, i2)
    for r in (0, 1):
        assert np.array_equal(res[r]["Shi"], Shi) and np.array_equal(res[r]["Slo"], Slo)
        assert np.array_equal(res[r]["cnt"], np.bincount(lab, minlength=k))
    st = oracle.step(X.astype(np.float64), X[:k].astype(np.float64), work="fp32", dist="fp32")
    assert np.array_equal(st["labels"], lab)
    for j in range(k):
        m = int(res[0]["cnt"][j])
        for t in range(d):
            g = Fraction(2) ** int(e[t] - 45)
            tot = Fraction(int(Shi[j, t]) * 2 ** 23 + int(Slo[j, t])) * g
            c = np.float32(float(tot / m))
            exact = sum(Fraction(float(v)) for v in X[lab == j, t]) / m
            ulp = abs(float(np.spacing(np.float32(float(exact)))))
            assert abs(Fraction(float(c)) - exact) <= Fraction(ulp), (j, t)
            assert abs(float(c) - st["centroids"][j, t]) <= ulp


def test_shard_range_properties():
    from paper_2407_12208_b200.dist import shard_range
    for n in (1, 7, 1000, 10_000_000):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
