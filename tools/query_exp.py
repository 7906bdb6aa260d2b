"""Measurement experiment (not part of the product): time the fused query
kernel (npm_sample with the fused pdf at caller directions) at c2.
usage: python tools/query_exp.py  (prints one JSON line; NPM_* env knobs apply)"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2504_04315_b200 import npm
    from workloads import synth
    from workloads.configs import CONFIGS
    name = os.environ.get("EXP_WORKLOAD", "c2")
    cfg = CONFIGS[name]
    n = cfg["n"]
    m = npm.Model(0, **cfg["model"])
    prod = cfg["model"].get("mode", 0) == 1
    qb = synth.query_batch(n, seed=100, product=prod)
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    q = m.query(T(qb["x"]), *([T(qb["wo"]), T(qb["nrm"]), T(qb["rough"])] if prod else []))
    wq = T(qb["wq"])
    for i in range(3):
        m.sample(q, seed=1, offset=i * n, use_ema=True, wq=wq)
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    npm.npm_profile_reset(m.h)
    npm.npm_profile_enable(m.h, True)
    for i in range(10):
        flush.zero_()
        m.sample(q, seed=1, offset=i * n, use_ema=True, wq=wq)
    torch.cuda.synchronize()
    prof = npm.npm_profile_read(m.h)
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("NPM_")},
                      "us_per_launch": {k: round(v[1] / v[0] * 1e3, 1) for k, v in prof.items() if v[0]}}), flush=True)


if __name__ == "__main__":
    main()
