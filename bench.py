#!/usr/bin/env python
"""Benchmark of the NPM hot path (arXiv 2504.04315) on B200.

One STEP = one pass of the whole hot path over one batch of synthetic input
(DESIGN.md "Measurement"): a guided query wave -- npm_sample with the fused pdf
at caller directions (encode -> decode -> Table 1 -> sample + pdf) over n
queries -- followed by one optimisation step -- npm_accumulate_grads (Eq. 9
head -> backprop -> grid scatter-add) over n records, [gradient allreduce over
NCCL when N > 1], npm_optimizer_step (Adam + EMA).  n = BASELINE configs[1]
(c2: 1280 x 720 = 921,600) per GPU; N > 1 is weak scaling with the gradient
allreduced every step.

value   = (queries + training records) processed by all ranks / device time,
          i.e. 2 n N / t_step ("samples/s": one query and one record per
          pixel-sample); train_samples_per_s and queries_per_s are the two
          phases timed separately inside the same steps.
e2e     = the same metric through the C ABI with HOST (pinned) buffers, the
          host<->device copies inside the timed region.
Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import synth  # noqa: E402
from workloads.configs import CONFIGS  # noqa: E402

METRIC = "NPM training samples/sec and guided pdf+sample queries/sec at 1/2/4/8 B200"
UNIT = "samples/s"
WORKLOAD = "c2"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()

    def summary(self):
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
_W = {}


def _oracle_worker_init(name, seed):
    """Pool initializer: the worker's copy of the model state (float64 oracle,
    1 BLAS thread per process so the pool uses exactly its cores)."""
    from threadpoolctl import threadpool_limits
    from oracle import npm as onpm
    _W["limits"] = threadpool_limits(limits=1)
    cfg = onpm.Config(**CONFIGS[name]["model"])
    _W["cfg"] = cfg
    _W["p"] = synth.random_params(cfg.layer_dims, cfg.n_grid, cfg.n_lobes, seed=seed).astype(np.float64)
    _W["ema"] = _W["p"].copy()


def _oracle_shard(task):
    """One shard of the hot path in the oracle: decode + sample + pdf at the
    caller directions for the shard's queries, Eq. 9 gradient over its records
    (scaled by 1/N_global).  Returns the shard's gradient vector."""
    from oracle import npm as onpm, vmf as ovmf
    cfg = _W["cfg"]
    q, t, u, n_global = task
    _, act = onpm.decode(cfg, _W["ema"], q["cond"])
    ovmf.sample(act, u, cfg.n_lobes)
    ovmf.mixture_pdf(q["wq"], act)
    g, _ = onpm.gradient(cfg, _W["p"], t["cond"], t["wi"], t["target"], t["pdf"], n_global)
    return g


class OracleRunner:
    """The float64 oracle as it stands, run on all host cores: queries and
    records are cut into contiguous shards, one per process (forward and the
    per-record gradient are independent per sample); the parent sums the
    shards' gradients in a fixed order and runs Adam + EMA once (SURVEY 8(d)
    "multiprocessing over contiguous sample shards on all host cores")."""

    def __init__(self, name, seed=0, cores=None):
        import multiprocessing as mp
        from oracle import npm as onpm
        self.name, self.seed = name, seed
        self.cores = cores or os.cpu_count() or 1
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_oracle_worker_init, initargs=(name, seed))
        cfg = onpm.Config(**CONFIGS[name]["model"])
        self.state = onpm.State(cfg, synth.random_params(cfg.layer_dims, cfg.n_grid, cfg.n_lobes,
                                                         seed=seed).astype(np.float64))
        self.prod = cfg.mode == onpm.PRODUCT
        self.batches = {}

    def _batch(self, n, seed):
        from oracle import philox as ophilox
        if (n, seed) not in self.batches:
            qb = synth.query_batch(n, seed=seed + 1, product=self.prod)
            tb = synth.training_batch(n, seed=seed + 2, product=self.prod)
            cond = lambda b, a, e: dict(x=b["x"][:, a:e], **(dict(
                wo=b["wo"][:, a:e].astype(np.float64), n=b["nrm"][:, a:e].astype(np.float64),
                rough=b["rough"][a:e].astype(np.float64)) if self.prod else {}))
            u = ophilox.sample_uniforms(n, 1234, 0)
            tasks = []
            for k in range(self.cores):
                a, e = n * k // self.cores, n * (k + 1) // self.cores
                tasks.append((dict(cond=cond(qb, a, e), wq=qb["wq"][:, a:e].astype(np.float64)),
                              dict(cond=cond(tb, a, e), wi=tb["wi"][:, a:e].astype(np.float64),
                                   target=tb["target"][..., a:e].astype(np.float64),
                                   pdf=tb["pdf"][a:e].astype(np.float64)), u[:, a:e], n))
            self.batches = {(n, seed): tasks}
        return self.batches[(n, seed)]

    def step(self, n, seed=0):
        """One step on n queries + n records; returns its wall time (s)."""
        from oracle import npm as onpm
        tasks = self._batch(n, seed)
        t0 = time.perf_counter()
        g = None
        for gk in self.pool.map(_oracle_shard, tasks, chunksize=1):   # fixed (shard) order
            g = gk if g is None else g + gk
        onpm.optimizer_step(self.state, g)
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def host_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"os_cpu_count": os.cpu_count(), "lscpu_model": model, "threads_per_process": 1}


def cpu_baseline(name, budget_s=20.0):
    """The oracle on all host cores: the full per-step workload when it fits
    the time budget (c1, c2 on a many-core host), else a bounded sample
    (n scaled down to ~budget_s)."""
    n_full = CONFIGS[name]["n"]
    r = OracleRunner(name)
    try:
        n0 = min(n_full, 1 << 13) * r.cores
        n0 = min(n0, n_full)
        dt0 = r.step(n0, seed=1)
        n = n_full if dt0 * n_full / n0 <= budget_s else int(max(n0, n0 * budget_s / max(dt0, 1e-3)))
        dt = r.step(n)
    finally:
        r.close()
    return {"value": 2 * n / dt, "unit": UNIT, "cores": r.cores, "kind": "oracle",
            "sample": "%s workload, %d queries + %d records, one step%s (float64 numpy oracle, %d processes x 1 "
                      "thread, contiguous shards; gradient summed in shard order, Adam + EMA over all %s params "
                      "in the parent)" % (name, n, n, " (the full step)" if n == n_full else " (bounded sample)",
                                          r.cores, name),
            "host": host_info(), "seconds": dt}


def run_reference(args, rank):
    """--impl reference: the oracle on all host cores, same metric/config."""
    if rank != 0:
        return
    name = args.workload
    n_full = CONFIGS[name]["n"]
    r = OracleRunner(name)
    try:
        n0 = min(n_full, (1 << 13) * r.cores)
        dt0 = r.step(n0, seed=1)
        # the whole --steps/--warmup run within ~3 minutes
        per_step = 150.0 / max(1, args.steps + args.warmup)
        n = n_full if dt0 * n_full / n0 <= per_step else int(max(n0, n0 * per_step / max(dt0, 1e-3)))
        for _ in range(args.warmup):
            r.step(n)
        ts = [r.step(n) for _ in range(args.steps)]
    finally:
        r.close()
    t = float(np.sum(ts))
    v = 2 * n * args.steps / t
    sample = ("%d queries + %d records per step of the %s workload%s; float64 oracle on %d processes x 1 thread"
              % (n, n, name, " (the full step)" if n == n_full else " (bounded sample)", r.cores))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": name + (" (full step)" if n == n_full else
                                                               " (bounded sample: %d queries + %d records per step)"
                                                               % (n, n)), "n_per_gpu": n},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": r.cores, "kind": "oracle", "sample": sample,
                             "host": host_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=WORKLOAD, choices=list(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-strong", action="store_true", help="skip the c3 strong-scaling block")
    ap.add_argument("--native-comm", action="store_true",
                    help="GRADS allreduce through the library's own NCCL communicator (npm_comm_init)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import torch.distributed as dist
    from paper_2504_04315_b200 import npm
    from paper_2504_04315_b200.dp import DataParallel

    torch.cuda.set_device(local)
    distributed = "WORLD_SIZE" in os.environ   # launched by torchrun (also world size 1)
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    name = args.workload
    cfg = CONFIGS[name]
    n = cfg["n"] if name != "c3" else cfg["n_global"] // world
    m = npm.Model(local, **cfg["model"])
    dp = DataParallel(m, world, force_allreduce=distributed, native=args.native_comm and distributed)
    # inputs resident in HBM (device-timed value)
    qb = synth.query_batch(n, seed=100 + rank, product=m.product)
    tb = synth.training_batch(n, seed=200 + rank, product=m.product)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    qx, wq = T(qb["x"]), T(qb["wq"])
    tx, twi, ttg, tpd = T(tb["x"]), T(tb["wi"]), T(tb["target"]), T(tb["pdf"])
    extra_q = [T(qb["wo"]), T(qb["nrm"]), T(qb["rough"])] if m.product else [None, None, None]
    extra_t = [T(tb["wo"]), T(tb["nrm"]), T(tb["rough"])] if m.product else [None, None, None]
    qq = m.query(qx, *extra_q)
    qt = m.query(tx, *extra_t)
    wi_o, pdf_o, pdfq_o = (torch.empty(3, n, device=dev), torch.empty(n, device=dev),
                           torch.empty(n, device=dev))
    stream = torch.cuda.current_stream(dev).cuda_stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def step(i, ev=None):
        npm.npm_sample(m.h, qq, None, 0xC0FFEE, i * n, True, wi_o[0], wi_o[1], wi_o[2], pdf_o, wq[0], wq[1],
                       wq[2], pdfq_o, stream=stream)
        if ev is not None:
            ev.record()
        dp.train_step(qt, twi, ttg, tpd, n_local=n, n_global=n * world)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    launches0 = m.launches
    npm.npm_profile_reset(m.h)
    npm.npm_profile_enable(m.h, True)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e2 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()                     # L2 flush between timed steps (not timed)
            e0[i].record()
            step(args.warmup + i, e1[i])
            e2[i].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = m.launches - launches0
    npm.npm_profile_enable(m.h, False)
    prof = npm.npm_profile_read(m.h)
    t_q = sum(a.elapsed_time(b) for a, b in zip(e0, e1)) / 1e3
    t_t = sum(a.elapsed_time(b) for a, b in zip(e1, e2)) / 1e3
    tt = torch.tensor([t_q + t_t, t_q, t_t], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_tot, t_q, t_t = tt.tolist()
    K = args.steps
    value = 2 * n * world * K / t_tot

    # ---- f-1 context: combined BSDF/guide sampling (alpha = 0.5) over the same n
    # queries and the record unwind of n records (8-vertex paths), device-timed
    def timed_ms(fn, reps=5):
        fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            fn()
            a1.record()
            torch.cuda.synchronize()
            ts.append(a0.elapsed_time(a1))
        return float(np.median(ts))

    nv = np.random.default_rng(300 + rank).normal(size=(3, n))
    nrm = T((nv / np.linalg.norm(nv, axis=0)).astype(np.float32))
    cw, cp, cg = torch.empty(3, n, device=dev), torch.empty(n, device=dev), torch.empty(n, device=dev)
    ct = torch.empty(n, dtype=torch.int32, device=dev)
    t_comb = timed_ms(lambda: npm.npm_combined_sample(m.h, qq, nrm[0], nrm[1], nrm[2], 0.5, None, 0xC0FFEE, 0, True,
                                                      cw[0], cw[1], cw[2], cp, cg, ct, stream=stream))
    Dp, npaths = 8, n // 8
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    le_ = torch.rand(3, Dp, npaths, device=dev, generator=g)
    fs_ = torch.rand(3, Dp, npaths, device=dev, generator=g)
    cs_ = torch.rand(Dp, npaths, device=dev, generator=g)
    pd_ = torch.rand(Dp, npaths, device=dev, generator=g) + 0.05
    dp_ = torch.randint(0, Dp + 1, (npaths,), device=dev, dtype=torch.int32, generator=g)
    tg_ = torch.empty(3, Dp, npaths, device=dev)
    t_unw = timed_ms(lambda: npm.npm_unwind_records(m.h, le_, fs_, cs_, pd_, dp_, 3, Dp, npaths, 0, tg_, stream=stream))
    pq_ = torch.empty(n, device=dev)
    t_cos = timed_ms(lambda: npm.npm_sample_cosine_product(m.h, qq, nrm[0], nrm[1], nrm[2], 2.1438, None, 0xC0FFEE, 0,
                                                           True, cw[0], cw[1], cw[2], cp, wq[0], wq[1], wq[2], pq_,
                                                           stream=stream))
    f2 = {"cosine_product_sample_plus_pdf_ms": t_cos, "queries_per_s": n / (t_cos / 1e3), "kappa_c": 2.1438}
    # ---- f-4 context (c2 shape): one training step (Eq. 9 kernel + Adam) per objective on
    # the same records and parameters: KL (the bench's), Pearson chi^2 (C-A31), the
    # variance-aware target (C-A35) and KL + the learned selection probability (C-A34)
    f4 = None
    if name in ("c2", "c1") and world == 1:
        try:
            wsq = (twi * T(tb["nrm"])).sum(0).clamp_min(0) / np.pi   # the records' stand-in BSDF pdf (C-A24)
            p0 = m.get(npm.BUF_PARAMS)
            f4 = {}
            for key, kw in (("kl", {}), ("chi2", {"divergence": 1}), ("variance_aware", {"divergence": 2}),
                            ("learned_alpha", {"learn_alpha": 1})):
                m4 = npm.Model(local, **dict(cfg["model"], **kw))
                if "learn_alpha" in kw:
                    pf = torch.zeros(m4.n_params, device=dev)
                    pf[:p0.numel()] = p0
                    m4.set(npm.BUF_PARAMS, pf)
                    q4 = m4.query(tx, bsdf_pdf=wsq)
                else:
                    m4.set(npm.BUF_PARAMS, p0)
                    q4 = m4.query(tx)
                t4 = timed_ms(lambda: (m4.accumulate_grads(q4, twi, ttg, tpd, want_stats=False),
                                       m4.optimizer_step(False)))
                f4[key] = {"train_step_ms": t4, "records_per_s": n / (t4 / 1e3)}
                m4.close()
        except Exception as exc:   # context only; never fail the bench line on it
            f4 = {"error": str(exc)}
    f1 = {"combined_sample_ms": t_comb, "combined_sample_queries_per_s": n / (t_comb / 1e3), "alpha": 0.5,
          "unwind_ms": t_unw, "unwind_records_per_s": Dp * npaths / (t_unw / 1e3),
          "unwind_bytes_per_record": 4 * (3 + 3 + 1 + 1 + 3) + 4 / Dp,
          "unwind_gb_s": (4 * 11 * Dp * npaths + 4 * npaths) / (t_unw / 1e3) / 1e9}

    # ---- e2e: same step through the C ABI with pinned HOST buffers ------------------------
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hqx, hwq = pin(qb["x"]), pin(qb["wq"])
    htx, htwi, httg, htpd = pin(tb["x"]), pin(tb["wi"]), pin(tb["target"]), pin(tb["pdf"])
    hex_q = [pin(qb["wo"]), pin(qb["nrm"]), pin(qb["rough"])] if m.product else [None, None, None]
    hex_t = [pin(tb["wo"]), pin(tb["nrm"]), pin(tb["rough"])] if m.product else [None, None, None]
    hq = npm.make_query(n, hqx[0], hqx[1], hqx[2], *(
        [hex_q[0][0], hex_q[0][1], hex_q[0][2], hex_q[1][0], hex_q[1][1], hex_q[1][2], hex_q[2]] if m.product else []))
    ht = npm.make_query(n, htx[0], htx[1], htx[2], *(
        [hex_t[0][0], hex_t[0][1], hex_t[0][2], hex_t[1][0], hex_t[1][1], hex_t[1][2], hex_t[2]] if m.product else []))
    hwi, hpdf, hpdfq = pin(np.zeros((3, n), np.float32)), pin(np.zeros(n, np.float32)), pin(np.zeros(n, np.float32))
    n_in_f = 3 + (7 if m.product else 0)
    h2d = n * 4 * (n_in_f + 3) + n * 4 * (n_in_f + 3 + ttg.shape[0] + 1)
    d2h = n * 4 * 5 + 8 * 6

    import ctypes
    hstats = torch.zeros(ctypes.sizeof(npm.npm_step_stats), dtype=torch.uint8).pin_memory()

    frame_call = world == 1 or args.native_comm   # the exchange then runs inside the library

    def e2e_step(i):
        if frame_call:
            # one host call per frame: queries + records through ONE chunked
            # host<->device pipeline, then the optimiser (npm_frame_step)
            npm.npm_frame_step(m.h, hq, None, 0xC0FFEE, i * n, True, hwi[0], hwi[1], hwi[2], hpdf, hwq[0], hwq[1],
                               hwq[2], hpdfq, ht, htwi[0], htwi[1], htwi[2], httg, httg.shape[0], htpd, n * world,
                               want_stats=False, stream=stream)
        else:
            npm.npm_sample(m.h, hq, None, 0xC0FFEE, i * n, True, hwi[0], hwi[1], hwi[2], hpdf, hwq[0], hwq[1],
                           hwq[2], hpdfq, stream=stream)
            dp.train_step(ht, htwi, httg, htpd, n_local=n, n_global=n * world, want_stats=False)
        # the step's loss read back to pinned host memory every step, without a
        # host synchronisation per step (the timed region ends with one)
        npm.npm_step_stats_async(m.h, hstats.data_ptr(), stream=stream)

    for i in range(2):
        e2e_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record()
    th0 = time.perf_counter()
    for i in range(K):
        e2e_step(i)
    host_enqueue_ms = (time.perf_counter() - th0) * 1e3 / K   # host time to enqueue one step (diagnostic)
    ee1.record()
    torch.cuda.synchronize()
    te = torch.tensor([ee0.elapsed_time(ee1) / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = 2 * n * world * K / te.item()

    # ---- c3 strong scaling: N_global = 2^23 training records per
    # optimisation step, sharded contiguously over the ranks (n_global / N each),
    # one allreduce of GRADS + Adam per step; the same model shape as c2
    strong = None
    if name == "c2" and not args.no_strong:
        from paper_2504_04315_b200.dp import shard_range
        ng = CONFIGS["c3"]["n_global"]
        a3, e3 = shard_range(ng, rank, world)
        n3 = e3 - a3
        sb3 = synth.training_batch(n3, seed=400 + rank, product=m.product)
        sx3, sw3, st3, sp3 = T(sb3["x"]), T(sb3["wi"]), T(sb3["target"]), T(sb3["pdf"])
        q3 = m.query(sx3, *([T(sb3["wo"]), T(sb3["nrm"]), T(sb3["rough"])] if m.product else []))
        for _ in range(2):
            dp.train_step(q3, sw3, st3, sp3, n_local=n3, n_global=ng)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        k3 = 5
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(k3):
            dp.train_step(q3, sw3, st3, sp3, n_local=n3, n_global=ng)
        a1.record()
        torch.cuda.synchronize()
        t3 = torch.tensor([a0.elapsed_time(a1) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t3, op=dist.ReduceOp.MAX)
        t3v = t3.item() / k3
        strong = {"workload": "c3: 2^23 training records per optimisation step over all ranks (strong scaling)",
                  "n_global": ng, "n_per_gpu": n3, "steps": k3, "ms_per_step": 1e3 * t3v,
                  "train_samples_per_s": ng / t3v, "scaling": "strong",
                  "note": "device time, max over ranks; inputs resident; includes the GRADS allreduce and Adam"}
        del sx3, sw3, st3, sp3, q3

    # ---- the paper's own workloads, as context (RTX 3070): a training step on a
    # 2^18-record batch (~10 ms) and one guided evaluation of a 1280x720 frame (~3 ms)
    paper_ctx = None
    if name == "c2" and n >= (1 << 18):
        k18 = 1 << 18
        C = lambda t2: t2[..., :k18].contiguous()
        q18 = m.query(C(tx), *[C(e) if e is not None else None for e in extra_t])
        w18, t18, p18 = C(twi), C(ttg), C(tpd)
        for _ in range(3):
            dp.train_step(q18, w18, t18, p18, n_local=k18, n_global=k18 * world)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            flush.zero_()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            dp.train_step(q18, w18, t18, p18, n_local=k18, n_global=k18 * world)
            a1.record()
            torch.cuda.synchronize()
            ts.append(a0.elapsed_time(a1))
        # f-3: the whole frame batch as 2^18-record micro-steps, one call
        tsm = []
        for _ in range(5):
            flush.zero_()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            m.train_stream(qt, twi, ttg, tpd, micro_batch=k18, want_stats=False)
            a1.record()
            torch.cuda.synchronize()
            tsm.append(a0.elapsed_time(a1))
        f3 = {"frame_records": n, "micro_batch": k18, "micro_steps": (n + k18 - 1) // k18,
              "ms": float(np.median(tsm)), "records_per_s": n / (float(np.median(tsm)) / 1e3)}
        paper_ctx = {"train_step_2e18_records_ms": float(np.median(ts)), "paper_rtx3070_ms": 10.0,
                     "f3_micro_step_stream": f3,
                     "eval_1280x720_sample_plus_pdf_ms": 1e3 * t_q / K, "paper_eval_rtx3070_ms": 3.0,
                     "note": "paper numbers are another machine's (RTX 3070, P:309, P:482): context only"}
    # ---- roofline of the dominant kernel -----------------------------------------------------
    hbm, bf16, bf16s, src = peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][1])
    kname, (kl, kms) = dom
    L, F = m.L, m.F
    gather = 8 * L * F * 4
    per_unit = {  # algorithmic bytes per sample
        "query": 12 + 12 + gather + 12 + 4 + 4,          # x, caller dir, gathers, sample w + pdf, pdf_q
        "train_fused": 12 + 12 + 4 * ttg.shape[0] + 4 + 2 * gather,   # records + gathers + scatter-add
        "train_forward": 12 + 12 + 4 * ttg.shape[0] + 4 + gather,
        "train_backward": 12 + gather,                   # x (re-derive corners) + scatter-add
        "weight_grad": 0, "adam": 0, "encode": 12 + gather + 4 * L * F,
    }
    units = n * K
    if kname == "adam":
        algo = 40 * m.n_params * kl
    else:
        algo = per_unit.get(kname, 0) * units
    achieved = algo / (kms / 1e3) / 1e9 if kms > 0 else 0.0
    traffic = None   # dram bytes per launch from the committed ncu --set full capture (profiles/traffic.json)
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if tj.get("workload") == name:
            traffic = tj["dram_bytes_per_launch"].get(kname)
    except Exception:
        pass
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": traffic, "traffic_source": "profiles/traffic.json (ncu --set full)" if traffic else None,
            "algorithmic_bytes_per_launch": per_unit.get(kname, 0) * n,
            "kernel": kname, "kernel_ms_per_launch": kms / max(kl, 1),
            "kernel_share_of_step": (kms / 1e3) / t_tot if t_tot > 0 else None, "peak_source": src,
            "per_unit_bytes": per_unit.get(kname), "units_per_launch": n}

    # grid-access ceiling: the same number of uniformly random 16-B
    # gathers / v4 scatter-adds into a table of this model's size, timed by the
    # library's probe kernels (include/npm.h npm_probe_grid_access).  For
    # L2-resident tables this, not HBM, bounds the fused kernels' grid stage.
    try:
        ents = m.n_grid // F
        tg = npm.npm_probe_grid_access(local, ents, n, L, 0)
        ts_ = npm.npm_probe_grid_access(local, ents, n, L, 1)
        acc = 8 * L * n
        probe = {"table_entries": ents, "table_mb": 16 * ents / 1e6, "accesses_per_launch": acc,
                 "gather_ms": tg, "scatter_ms": ts_,
                 "gathers_per_s": acc / (tg / 1e3), "scatter_adds_per_s": acc / (ts_ / 1e3)}
        for k, need in (("query", tg), ("train_fused", tg + ts_)):
            if k in prof and prof[k][0]:
                probe["%s_frac_of_probe" % k] = need / (prof[k][1] / prof[k][0])
        roof["grid_access_probe"] = probe
    except Exception as exc:   # the probe is context; never fail the bench line on it
        roof["grid_access_probe"] = {"error": str(exc)}

    # decoder tensor-core work (algorithmic MACs of the 64-wide MLP; split-bf16 issues 3x)
    dims = [(m.cfg.n_levels * m.F + (33 if m.product else 0), m.cfg.mlp_width)]
    dims += [(m.cfg.mlp_width, m.cfg.mlp_width)] * (m.cfg.mlp_linear_layers - 2)
    dims += [(m.cfg.mlp_width, 4 * m.K)]
    fwd_flop = 2 * sum(i * o for i, o in dims)
    t_dec = {k: v for k, v in prof.items() if k in ("query", "train_fused")}
    tens = {}
    for k, (kl2, kms2) in t_dec.items():
        fl = (fwd_flop if k == "query" else 3 * fwd_flop) * n * kl2
        tens[k] = {"algorithmic_tflops": fl / (kms2 / 1e3) / 1e12 if kms2 else None,
                   "issued_tflops_split_bf16x3": 3 * fl / (kms2 / 1e3) / 1e12 if kms2 else None,
                   "peak_bf16_tflops": bf16, "flop_per_sample": fl / (n * kl2)}
    roof["decoder_tensor"] = tens
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(name)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
                "ms_per_step": 1e3 * t_tot / K, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32 (decoder MMAs split-bf16x3, f32 accumulate)", "data": "synthetic",
                "config": {"workload": "%s: %s" % (name, "per-frame batch 1280x720 queries + records per GPU, "
                                                   "K=8, L=8 (D 8..86, T=2^18), 3x64 MLP" if name == "c2" else name),
                           "n_per_gpu": n, "l2": "flushed between timed steps (512 MB write)",
                           "parallelism": "dp%d" % world},
                "train_samples_per_s": n * world * K / t_t, "queries_per_s": n * world * K / t_q,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "host_enqueue_ms_per_step": host_enqueue_ms,
                        "call": "npm_frame_step (one pipeline per frame)" if frame_call else
                                "npm_sample + DataParallel.train_step (torch.distributed exchange)"},
                "gpu_launches": launches, "gpu_launches_per_step": launches / K,
                "roofline": roof, "kernels": {k: {"launches": v[0], "ms": v[1]} for k, v in prof.items() if v[0]},
                "clocks": clk.summary(), "cpu_baseline": cpu, "strong_c3": strong, "paper_context": paper_ctx,
                "f1_guided_mis": f1,
                "f2_cosine_product": f2,
                "f4_objectives": f4}
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
