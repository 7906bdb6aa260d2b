"""Data-parallel path on CPU (gloo, world size 2): the DataParallel driver of
paper_2504_04315_b200/dp.py with an oracle-backed trainer plugged in.

Checks the one exchange step of the method (C-A13): with every
rank scaling by 1/N_global, the allreduced gradient equals the union-batch
gradient, the replicas stay bitwise identical after several optimiser steps,
and the reduced statistics equal the union batch's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_04315_b200.dp import DataParallel, shard_range
from tests.test_oracle_npm import tiny_cfg, random_params, random_batch


PAD = 264   # the library's buffer padding past n_params (npm.h npm_shard_range)


class OracleTrainer:
    """DataParallel protocol backed by the float64 oracle (test double),
    including the ZeRO-1 building blocks with the library's shard layout."""

    def __init__(self, cfg, params):
        from oracle import npm as onpm
        self.onpm = onpm
        self.state = onpm.State(cfg, params.copy())
        self.n = params.size
        self.gbuf = torch.zeros(self.n + PAD, dtype=torch.float64)
        self.grads = self.gbuf[:self.n]
        self.pbuf = torch.zeros(self.n + PAD, dtype=torch.float64)

    def shard_range(self, rank, world):
        chunk = ((self.n + world - 1) // world + 3) // 4 * 4
        b = rank * chunk
        return b, max(0, min(chunk, self.n - b)), chunk

    def optimizer_step_shard(self, rank, world, want_stats):
        from oracle import adam as oadam
        st, c = self.state, self.state.cfg
        b, cnt, _ = self.shard_range(rank, world)
        g = self.gbuf[:self.n].numpy()[b:b + cnt].copy()
        st.t += 1
        sl = slice(b, b + cnt)
        p, m, v, _, nnf = oadam.adam_ema_step(st.params[sl], g, st.m[sl], st.v[sl], st.ema[sl], st.t,
                                              self.onpm.grid_mask(c)[sl], c.lr, c.beta1, c.beta2, c.adam_eps,
                                              c.ema_decay)
        st.params[sl], st.m[sl], st.v[sl] = p, m, v
        self.gbuf.zero_()
        return dict(grad_norm_sq=float(np.sum(np.where(np.isfinite(g), g, 0.0) ** 2)), n_nonfinite_grad=nnf)

    def param_tensor(self, count):
        self.pbuf[:self.n] = torch.from_numpy(self.state.params)
        return self.pbuf[:count]

    def ema_update(self):
        st, d = self.state, self.state.cfg.ema_decay
        st.params = self.pbuf[:self.n].numpy().copy()
        st.ema = d * st.ema + (1 - d) * st.params

    def accumulate(self, q, wi, target, spdf, n_global, want_stats):
        g, st = self.onpm.gradient(self.state.cfg, self.state.params, q, wi, target, spdf, n_global)
        self.grads += torch.from_numpy(g)
        return st

    def optimizer_step(self, want_stats):
        g = self.grads.numpy().copy()
        nnf = self.onpm.optimizer_step(self.state, g)
        self.grads.zero_()
        return dict(grad_norm_sq=float((g ** 2).sum()), n_nonfinite_grad=nnf)

    def grad_tensor(self, count=None):
        return self.grads if count is None else self.gbuf[:count]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(n, seed):
    cfg = tiny_cfg()
    rng = np.random.default_rng(seed)
    q, wi, tgt, pdf = random_batch(cfg, rng, n)
    return cfg, dict(x=q["x"]), wi, tgt, pdf


def _worker(rank, world, port, n, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, q, wi, tgt, pdf = _batch(n, 5)
    params = random_params(cfg, np.random.default_rng(6))
    tr = OracleTrainer(cfg, params)
    dp = DataParallel(tr, world)
    a, b = shard_range(n, rank, world)
    sl = lambda x: np.ascontiguousarray(x[..., a:b])
    stats = []
    for _ in range(steps):
        stats.append(dp.train_step(dict(x=sl(q["x"])), sl(wi), sl(tgt), sl(pdf), n_global=n, want_stats=True))
    out[rank] = (tr.state.params.copy(), tr.state.ema.copy(), stats)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [e - s for s, e in parts]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_step_equals_union_batch():
    n, steps, world = 61, 3, 2   # ragged: shards of 31 and 30 records
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, n, steps, out), nprocs=world, join=True)
    p0, e0, s0 = out[0]
    p1, e1, s1 = out[1]
    # replicas bitwise identical (same reduced bytes, same deterministic optimiser)
    assert np.array_equal(p0, p1) and np.array_equal(e0, e1)
    # single-process union batch
    cfg, q, wi, tgt, pdf = _batch(n, 5)
    tr = OracleTrainer(cfg, random_params(cfg, np.random.default_rng(6)))
    ref_stats = [DataParallel(tr, 1).train_step(q, wi, tgt, pdf, n_global=n, want_stats=True) for _ in range(steps)]
    assert np.allclose(p0, tr.state.params, rtol=1e-12, atol=1e-14)
    assert np.allclose(e0, tr.state.ema, rtol=1e-12, atol=1e-14)
    for a, b in zip(s0, ref_stats):
        assert a["n_used"] == b["n_used"] and a["n_dropped"] == b["n_dropped"]
        assert np.isclose(a["loss_proxy"], b["loss_proxy"], rtol=1e-12)
        assert np.isclose(a["grad_norm_sq"], b["grad_norm_sq"], rtol=1e-10)


def _stream_worker(rank, world, port, n, micro_local, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, q, wi, tgt, pdf = _batch(n, 8)
    tr = OracleTrainer(cfg, random_params(cfg, np.random.default_rng(9)))
    dp = DataParallel(tr, world)
    a, b = shard_range(n, rank, world)

    def make_slice(s0, s1):
        sl = lambda x: np.ascontiguousarray(x[..., a + s0:a + s1])
        return dict(x=sl(q["x"])), sl(wi), sl(tgt), sl(pdf)

    stats = dp.train_stream(make_slice, b - a, micro_local, want_stats=True)
    out[rank] = (tr.state.params.copy(), tr.state.t, stats)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_micro_step_stream_equals_union_micro_batches():
    # f-3 with one exchange per micro-step: micro-step j is one optimisation
    # step over the union of both ranks' slice j
    n, micro_local, world = 60, 12, 2      # shards of 30 -> slices 12, 12, 6
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_stream_worker, args=(world, port, n, micro_local, out), nprocs=world, join=True)
    p0, t0, s0 = out[0]
    p1, t1, s1 = out[1]
    assert np.array_equal(p0, p1) and t0 == t1 == 3
    from oracle import npm as onpm
    cfg, q, wi, tgt, pdf = _batch(n, 8)
    st = onpm.State(cfg, random_params(cfg, np.random.default_rng(9)))
    shards = [shard_range(n, r, world) for r in range(world)]
    for j in range(3):
        idx = np.concatenate([np.arange(a + j * micro_local, min(a + (j + 1) * micro_local, b)) for a, b in shards])
        _, ref = onpm.train_step(st, dict(x=q["x"][:, idx]), wi[:, idx], tgt[..., idx], pdf[idx], idx.size)
        assert s0[j]["n_used"] == ref["n_used"] and np.isclose(s0[j]["loss_proxy"], ref["loss_proxy"], rtol=1e-12)
    assert np.allclose(p0, st.params, rtol=1e-12, atol=1e-14)


def _ragged_worker(rank, world, port, n, micro_local, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, q, wi, tgt, pdf = _batch(n, 10)
    tr = OracleTrainer(cfg, random_params(cfg, np.random.default_rng(11)))
    dp = DataParallel(tr)            # world and N_global from the process group
    a, b = shard_range(n, rank, world)
    sl = lambda x, s0, s1: np.ascontiguousarray(x[..., a + s0:a + s1])
    # one full-shard step with N_global inferred (31 + 30 records)
    st1 = dp.train_step(dict(x=sl(q["x"], 0, b - a)), sl(wi, 0, b - a), sl(tgt, 0, b - a), sl(pdf, 0, b - a),
                        n_local=b - a, want_stats=True)
    # then a micro-step stream whose last step is empty on rank 1
    stats = dp.train_stream(lambda s0, s1: (dict(x=sl(q["x"], s0, s1)), sl(wi, s0, s1), sl(tgt, s0, s1),
                                            sl(pdf, s0, s1)), b - a, micro_local, want_stats=True)
    out[rank] = (tr.state.params.copy(), tr.state.t, st1, stats)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_unequal_shards_infer_n_global_and_stream_stays_in_step():
    # N_global is the sum of the (unequal) shard sizes, and both
    # ranks run the same number of micro-steps (rank 1's last slice is empty)
    n, micro_local, world = 61, 15, 2      # shards 31 (15, 15, 1) and 30 (15, 15, 0)
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ragged_worker, args=(world, port, n, micro_local, out), nprocs=world, join=True)
    p0, t0, a0, s0 = out[0]
    p1, t1, a1, s1 = out[1]
    assert np.array_equal(p0, p1) and t0 == t1 == 4
    from oracle import npm as onpm
    cfg, q, wi, tgt, pdf = _batch(n, 10)
    st = onpm.State(cfg, random_params(cfg, np.random.default_rng(11)))
    _, ref = onpm.train_step(st, q, wi, tgt, pdf, n)
    assert a0["n_used"] == ref["n_used"] and np.isclose(a0["loss_proxy"], ref["loss_proxy"], rtol=1e-12)
    shards = [shard_range(n, r, world) for r in range(world)]
    for j in range(3):
        idx = np.concatenate([np.arange(a + j * micro_local, min(a + (j + 1) * micro_local, b)) for a, b in shards])
        _, ref = onpm.train_step(st, dict(x=q["x"][:, idx]), wi[:, idx], tgt[..., idx], pdf[idx], idx.size)
        assert s0[j]["n_used"] == ref["n_used"] and np.isclose(s0[j]["loss_proxy"], ref["loss_proxy"], rtol=1e-12)
    assert np.allclose(p0, st.params, rtol=1e-12, atol=1e-14)


def _zero1_worker(rank, world, port, n, steps, zero1, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, q, wi, tgt, pdf = _batch(n, 12)
    tr = OracleTrainer(cfg, random_params(cfg, np.random.default_rng(13)))
    dp = DataParallel(tr, world, zero1=zero1)
    a, b = shard_range(n, rank, world)
    sl = lambda x: np.ascontiguousarray(x[..., a:b])
    stats = [dp.train_step(dict(x=sl(q["x"])), sl(wi), sl(tgt), sl(pdf), n_global=n, want_stats=True)
             for _ in range(steps)]
    out[(zero1, rank)] = (tr.state.params.copy(), tr.state.m.copy(), tr.state.v.copy(), tr.state.ema.copy(), stats)
    dist.barrier()
    dist.destroy_process_group()


def test_zero1_sharded_optimiser_equals_replicated_bit_for_bit():
    """SURVEY 8(e) c5 schedule: reduce-scatter -> Adam on 1/P -> all-gather ->
    local EMA gives bit for bit the replicated allreduce + Adam + EMA update
    (2 ranks: the two-term sums are order-free), on every rank, over several
    steps, with ragged shards (n_params not a multiple of 4 P) and the grid-skip
    rule crossing a shard boundary."""
    n, steps, world = 41, 3, 2
    mgr = mp.Manager()
    out = mgr.dict()
    for zero1 in (False, True):
        mp.spawn(_zero1_worker, args=(world, _free_port(), n, steps, zero1, out), nprocs=world, join=True)
    ref = out[(False, 0)]
    tr = OracleTrainer(tiny_cfg(), random_params(tiny_cfg(), np.random.default_rng(13)))
    for rank in range(world):
        got = out[(True, rank)]
        # parameters and EMA: replicated, identical everywhere
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[3], ref[3])
        # Adam moments: each rank keeps only its own shard's (ZeRO-1)
        b, c, _ = tr.shard_range(rank, world)
        assert np.array_equal(got[1][b:b + c], ref[1][b:b + c]) and np.array_equal(got[2][b:b + c], ref[2][b:b + c])
        for sa, sb in zip(got[4], ref[4]):
            assert sa["n_nonfinite_grad"] == sb["n_nonfinite_grad"]
            assert np.isclose(sa["grad_norm_sq"], sb["grad_norm_sq"], rtol=1e-12)
    assert not np.array_equal(ref[0], tr.state.params)
    # the shards of this tiny model are ragged and the grid-skip boundary
    # (n_mlp) falls inside rank 0's shard
    assert tr.n % (4 * world) != 0
    b1, _, _ = tr.shard_range(1, world)
    assert 0 < tiny_cfg().n_mlp < b1
