"""Measurement experiment (not part of the product): time the fused training
kernel at c2 under different record orders / knobs, to see what the grid
stage costs.  Usage: python tools/train_exp.py <variant>  (prints one line).
Variants: shuffled, alpha (a learn_alpha model), va (the variance-aware target), sorted (records Morton-sorted on the host by their
finest-level cell), and the env knobs NPM_DEBUG (bit 0: skip the scatter),
NPM_BIN_TRAIN, NPM_PRIV set by the caller."""
import os
import sys
import json

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def morton_order(x, bits=7):
    u = np.clip((x + 1.0) / 2.0, 0, 1 - 1e-7)
    c = (u * (1 << bits)).astype(np.uint64)
    key = np.zeros(x.shape[1], np.uint64)
    for b in range(bits):
        for a in range(3):
            key |= ((c[a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return np.argsort(key, kind="stable")


def main():
    import torch
    from paper_2504_04315_b200 import npm
    from workloads import synth
    from workloads.configs import CONFIGS
    variant = sys.argv[1] if len(sys.argv) > 1 else "shuffled"
    name = os.environ.get("EXP_WORKLOAD", "c2")
    cfg = CONFIGS[name]
    n = cfg["n"]
    alpha = variant == "alpha"     # learn_alpha model (f-4', C-A34): the selection head's cost
    model = dict(cfg["model"], divergence=2) if variant == "va" else cfg["model"]   # C-A35
    m = npm.Model(0, learn_alpha=int(alpha), **model)
    tb = synth.training_batch(n, seed=200)
    if variant == "sorted":
        o = morton_order(tb["x"])
        tb = {k: (v[..., o] if isinstance(v, np.ndarray) and v.shape[-1] == n else v) for k, v in tb.items()}
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    pb = None
    if alpha:
        from oracle import guide   # measurement tool: the stand-in BSDF pdf of the records' directions
        pb = T(guide.bsdf_pdf(tb["nrm"].astype(np.float64), tb["wi"].astype(np.float64)).astype(np.float32))
    q = m.query(T(tb["x"]), bsdf_pdf=pb)
    wi, tg, pd = T(tb["wi"]), T(tb["target"]), T(tb["pdf"])
    for _ in range(3):
        m.accumulate_grads(q, wi, tg, pd, want_stats=False)
        m.optimizer_step(False)
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    npm.npm_profile_reset(m.h)
    npm.npm_profile_enable(m.h, True)
    for _ in range(10):
        flush.zero_()
        m.accumulate_grads(q, wi, tg, pd, want_stats=False)
        m.optimizer_step(False)
    torch.cuda.synchronize()
    prof = npm.npm_profile_read(m.h)
    out = {k: round(v[1] / v[0] * 1e3, 1) for k, v in prof.items() if v[0]}
    print(json.dumps({"variant": variant, "env": {k: v for k, v in os.environ.items() if k.startswith("NPM_")},
                      "us_per_launch": out}), flush=True)


if __name__ == "__main__":
    main()
