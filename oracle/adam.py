"""Adam + EMA ("fixed learning rate of 0.005 ... Adam ... we also apply
exponential moving average (EMA) to the weights").

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

Readings C-A14 / C-O17: beta1 0.9, beta2 0.999, eps 1e-8, bias
correction with the global step t; MLP parameters always updated (a
non-finite gradient is zeroed and counted); grid parameters are skipped
(p, m, v unchanged) iff their gradient is exactly 0 ("touched Phi_E entries",
S:360; a non-finite grid gradient is zeroed, counted, and therefore skipped).
C-A15 / C-O18: EMA over all parameters after Adam, e = d e + (1 - d) p,
d = 0.99, e_0 = p_0.
"""
import numpy as np


def adam_ema_step(p, g, m, v, e, t, is_grid, lr=5e-3, beta1=0.9, beta2=0.999,
                  eps=1e-8, ema_decay=0.99):
    """One optimiser step at global step t (already incremented, t >= 1).
    All arrays float64 1-D of equal length; is_grid bool mask.
    Returns (p, m, v, e, n_nonfinite)."""
    p, m, v, e = p.copy(), m.copy(), v.copy(), e.copy()
    nonfinite = ~np.isfinite(g)
    g = np.where(nonfinite, 0.0, g)
    upd = ~(is_grid & (g == 0.0))
    m_new = beta1 * m + (1 - beta1) * g
    v_new = beta2 * v + (1 - beta2) * g * g
    mhat = m_new / (1 - beta1 ** t)
    vhat = v_new / (1 - beta2 ** t)
    p_new = p - lr * mhat / (np.sqrt(vhat) + eps)
    p = np.where(upd, p_new, p)
    m = np.where(upd, m_new, m)
    v = np.where(upd, v_new, v)
    e = ema_decay * e + (1 - ema_decay) * p
    return p, m, v, e, int(nonfinite.sum())
