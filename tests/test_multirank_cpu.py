"""Multi-rank host logic on CPU (gloo, world size 2): the row-sharded exchange protocol of
SURVEY.md §8(e) reproduced with the oracle — no GPU needed.

* per-rank int64 node histograms all-reduced (SUM) equal the unsharded histogram (C1 in §5);
* the global strided cut sample assembled from per-rank samples (all-gather of fixed-size padded
  samples, re-packed by rank prefix — what binning.cu does) equals the single-process sample;
* shards of the C3/C4 generator tile the global row range and never split an Eq. (4) group.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sample_rows(n_global, row_offset, n):
    cap = 1 << 20
    s = max(1, -(-n_global // cap))
    i0 = (s - row_offset % s) % s
    return np.arange(i0, n, s)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # ---- histogram all-reduce
        rng = np.random.default_rng(0)
        n, F = 5000, 8
        codes = rng.integers(0, 40, (n, F)).astype(np.uint8)
        qg = rng.integers(-(1 << 14), (1 << 14) + 1, n).astype(np.int32)
        qh = rng.integers(0, (1 << 14) + 1, n).astype(np.int32)
        lo, hi = rank * n // world, (rank + 1) * n // world
        Hg, Hh = oracle.node_hist(codes[lo:hi], np.arange(hi - lo), qg[lo:hi], qh[lo:hi])
        tg, th = torch.from_numpy(Hg), torch.from_numpy(Hh)
        dist.all_reduce(tg, op=dist.ReduceOp.SUM)
        dist.all_reduce(th, op=dist.ReduceOp.SUM)
        Fg, Fh = oracle.node_hist(codes, np.arange(n), qg, qh)
        ok_hist = bool(np.array_equal(tg.numpy(), Fg) and np.array_equal(th.numpy(), Fh))
        # ---- global cut sample from per-rank samples
        n_global = (1 << 21) + 12345
        X = (np.arange(n_global) % 977).astype(np.float32)[:, None]
        lo, hi = rank * n_global // world, (rank + 1) * n_global // world
        mine = X[lo:hi][_sample_rows(n_global, lo, hi - lo), 0]
        meta = torch.tensor([lo, hi - lo], dtype=torch.int64)
        metas = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(metas, meta)
        m_r = [len(_sample_rows(n_global, int(m[0]), int(m[1]))) for m in metas]
        m_pad = max(m_r)
        buf = torch.zeros(m_pad, dtype=torch.float32)
        buf[:len(mine)] = torch.from_numpy(mine)
        bufs = [torch.zeros(m_pad, dtype=torch.float32) for _ in range(world)]
        dist.all_gather(bufs, buf)
        glob = np.concatenate([bufs[r][:m_r[r]].numpy() for r in range(world)])
        ref = X[_sample_rows(n_global, 0, n_global), 0]
        ok_sample = bool(np.array_equal(glob, ref))
        # cuts from the assembled sample == cuts of the whole column
        ct, nc = oracle.cuts(glob[:, None])
        ct2, nc2 = oracle.cuts(X, n_global=n_global)
        ok_cuts = bool(nc[0] == nc2[0] and np.array_equal(ct[0, :nc[0]], ct2[0, :nc2[0]]))
        q.put((rank, ok_hist, ok_sample, ok_cuts))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_histogram_allreduce_and_cut_sample():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_hist, ok_sample, ok_cuts in res:
        assert ok_hist and ok_sample and ok_cuts, (rank, ok_hist, ok_sample, ok_cuts)


def test_scaled_shards_tile_rows_and_keep_groups():
    n_llm, world = 1000, 4
    shards = [synth.make_scaled(n_llm, r, world) for r in range(world)]
    offs = [s.row_offset for s in shards]
    assert offs[0] == 0
    for a, b in zip(shards, shards[1:]):
        assert a.row_offset + a.n == b.row_offset
    assert shards[-1].row_offset + shards[-1].n == shards[0].n_global == n_llm * 8 * 16
    groups = [set(zip(s.llm_id.tolist(), s.prof_id.tolist())) for s in shards]
    for i in range(world):
        for j in range(i + 1, world):
            assert not (groups[i] & groups[j])
    full = synth.make_scaled(n_llm)
    assert np.array_equal(np.concatenate([s.X for s in shards]), full.X)
    assert np.array_equal(np.concatenate([s.y for s in shards]), full.y)
