"""Measurement experiment (not part of the product): the training gradient's
rel-L2 error against the float64 oracle, whole vector and worst block, for the
library NPM_LIB points at (precision variants of the backward MMAs).
Usage: python tools/grad_err.py  (prints one line)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from workloads import synth
    from tests.helpers import rel_l2
    from tests.test_gpu_parity import make_pair, gq, grad_blocks
    from paper_2504_04315_b200 import npm
    from oracle import npm as onpm
    out = []
    for name, n, rgb, seed in (("c1", 4096, False, 17), ("c2", 20000, True, 17), ("c2", 20000, False, 5)):
        m, ocfg, p = make_pair(name)
        b = synth.training_batch(n, seed=seed, rgb=rgb, nan_rate=1e-3)
        m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))
        m.accumulate_grads(gq(m, b), b["wi"], b["target"], b["pdf"], n_global=2 * n)
        g = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
        og, _ = onpm.gradient(ocfg, p, dict(x=b["x"]), b["wi"].astype(np.float64), b["target"].astype(np.float64),
                              b["pdf"].astype(np.float64), 2 * n)
        worst = {}
        for kind, a, e in grad_blocks(ocfg):
            if np.linalg.norm(og[a:e]) > 0:
                worst[kind] = max(worst.get(kind, 0.0), rel_l2(g[a:e], og[a:e]))
        out.append(f"{name}{'rgb' if rgb else ''} all {rel_l2(g, og):.2e} " +
                   " ".join(f"{k} {v:.2e}" for k, v in worst.items()))
    print(" | ".join(out))


if __name__ == "__main__":
    main()
