"""Shared test helpers: oracle <-> library configuration mapping, tolerance
checks (SURVEY §8(c) parity table)."""
import numpy as np

from workloads.configs import CONFIGS


def oracle_config(name_or_model):
    from oracle import npm as onpm
    m = CONFIGS[name_or_model]["model"] if isinstance(name_or_model, str) else name_or_model
    return onpm.Config(**m)


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
