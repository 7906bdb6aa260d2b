"""Small workloads for compute-sanitizer (memcheck / synccheck / racecheck):
every library entry point on c1 and on a small c2 / c4 batch, including the
binned query path (n >= 65,536), both training kernels (warp-specialised and
the r01 two-group one), the host-pointer pipeline (npm_frame_step, n >=
131,072), the ZeRO-1 building blocks and the f-1 / f-2 calls.
usage: compute-sanitizer --tool memcheck python tools/san_small.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_04315_b200 import npm  # noqa: E402
from workloads import synth  # noqa: E402
from workloads.configs import CONFIGS  # noqa: E402


def run(name, n, ws):
    os.environ["NPM_TRAIN_WS"] = str(ws)
    m = npm.Model(0, **CONFIGS[name]["model"])
    prod = m.product
    b = synth.training_batch(n, seed=1, product=prod, rgb=True, nan_rate=1e-3)
    q = m.query(b["x"], b["wo"], b["nrm"], b["rough"])
    m.train_step(q, b["wi"], b["target"], b["pdf"])
    qb = synth.query_batch(n, seed=2, product=prod)
    qq = m.query(qb["x"], qb["wo"], qb["nrm"], qb["rough"])
    m.sample(qq, seed=1, wq=qb["wq"])
    m.decode(qq)
    m.pdf(qq, qb["wq"])
    m.encode(qq)
    m.encode_debug(qq)
    if not prod:
        m.combined_sample(qq, qb["nrm"], alpha=0.5, seed=3)
        m.sample_cosine_product(qq, qb["nrm"], seed=4, wq=qb["wq"])
    # ZeRO-1 building blocks on a one-rank "world" of 2 (shard 0 and 1 in turn)
    m.accumulate_grads(q, b["wi"], b["target"], b["pdf"])
    npm.npm_optimizer_step_shard(m.h, 0, 2, True, m._stream())
    npm.npm_optimizer_step_shard(m.h, 1, 2, True, m._stream())
    npm.npm_ema_update(m.h, m._stream())
    m.train_stream(q, b["wi"], b["target"], b["pdf"], micro_batch=max(1, n // 3))
    print(name, n, "ws=%d" % ws, "ok", flush=True)
    m.close()


def objectives(n):
    """f-4' learned selection probability (C-A34) and f-4 variance-aware target (C-A35)."""
    from oracle import guide   # stand-in BSDF pdf of the records' directions (input data only)
    os.environ["NPM_TRAIN_WS"] = "1"
    b = synth.training_batch(n, seed=8, rgb=True, nan_rate=1e-3)
    pb = guide.bsdf_pdf(b["nrm"].astype(np.float64), b["wi"].astype(np.float64)).astype(np.float32)
    m = npm.Model(0, learn_alpha=1, **CONFIGS["c2"]["model"])
    m.train_step(m.query(b["x"], bsdf_pdf=pb), b["wi"], b["target"], b["pdf"])
    m.combined_sample(m.query(b["x"]), b["nrm"], alpha=0.5, seed=3)
    m.close()
    m = npm.Model(0, **dict(CONFIGS["c2"]["model"], divergence=2))
    m.train_step(m.query(b["x"]), b["wi"], b["target"], b["pdf"])
    print("objectives", n, "ok", flush=True)
    m.close()


def frame(n):
    import torch
    os.environ["NPM_TRAIN_WS"] = "1"
    m = npm.Model(0, **CONFIGS["c2"]["model"])
    b, tb = synth.query_batch(n, seed=5), synth.training_batch(n, seed=6)
    H = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hx, hw, tx, twi, ttg, tpd = H(b["x"]), H(b["wq"]), H(tb["x"]), H(tb["wi"]), H(tb["target"]), H(tb["pdf"])
    hq, ht = npm.make_query(n, hx[0], hx[1], hx[2]), npm.make_query(n, tx[0], tx[1], tx[2])
    wi, pdf, pdfq = H(np.zeros((3, n), np.float32)), H(np.zeros(n, np.float32)), H(np.zeros(n, np.float32))
    npm.npm_frame_step(m.h, hq, None, 7, 0, 1, wi[0], wi[1], wi[2], pdf, hw[0], hw[1], hw[2], pdfq, ht, twi[0], twi[1],
                       twi[2], ttg, 1, tpd, n)
    print("frame_step", n, "ok", flush=True)
    m.close()


if __name__ == "__main__":
    run("c1", 4096, 1)
    run("c2", 70000, 1)
    run("c2", 70000, 0)
    run("c4", 20000, 0)
    run("c4", 20000, 1)
    objectives(20000)
    frame(140000)
