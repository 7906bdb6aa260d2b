"""Spherical-harmonics input encoding for omega_o and the surface normal
("encode them using the spherical harmonics basis", citing
Ref-NeRF).  TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

Reading C-A20 / C-O6: 4 bands (l = 0..3, 16 coefficients), real orthonormal
basis, l-major with m ascending (index l^2 + l + m), no Condon-Shortley phase
(S:187-195).  Written from the textbook definition

  Y_l^m = sqrt(2) K_l^m cos(m phi) P_l^m(cos theta)        m > 0
  Y_l^0 = K_l^0 P_l^0(cos theta)
  Y_l^m = sqrt(2) K_l^|m| sin(|m| phi) P_l^|m|(cos theta)  m < 0
  K_l^m = sqrt((2l+1)/(4 pi) (l-m)!/(l+m)!)

with the associated Legendre functions by the standard recurrence.
"""
import math
import numpy as np


def assoc_legendre(l, m, x):
    """P_l^m(x), m >= 0, without the (-1)^m Condon-Shortley phase."""
    pmm = np.ones_like(x)
    if m > 0:
        somx2 = np.sqrt(np.maximum(1.0 - x * x, 0.0))
        fact = 1.0
        for _ in range(m):
            pmm = pmm * fact * somx2
            fact += 2.0
    if l == m:
        return pmm
    pmmp1 = x * (2 * m + 1) * pmm
    if l == m + 1:
        return pmmp1
    pll = None
    for ll in range(m + 2, l + 1):
        pll = ((2 * ll - 1) * x * pmmp1 - (ll + m - 1) * pmm) / (ll - m)
        pmm, pmmp1 = pmmp1, pll
    return pll


def sh_encode(w, bands=4):
    """w: [3, n] unit vectors.  Returns [bands^2, n] float64."""
    w = np.asarray(w, np.float64)
    z = np.clip(w[2], -1.0, 1.0)
    phi = np.arctan2(w[1], w[0])
    out = np.zeros((bands * bands, w.shape[1]))
    for l in range(bands):
        for m in range(-l, l + 1):
            am = abs(m)
            k = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - am) / math.factorial(l + am))
            p = assoc_legendre(l, am, z)
            if m > 0:
                y = math.sqrt(2.0) * k * np.cos(am * phi) * p
            elif m < 0:
                y = math.sqrt(2.0) * k * np.sin(am * phi) * p
            else:
                y = k * p
            out[l * l + l + m] = y
    return out
