"""Least-squares fit of e^r on |r| <= ln2/2 (a0 = a1 = 1 fixed) for the LavaMD
exp (csrc/apps.cuh lava_exp, oracle/hpac_oracle.c)."""
import numpy as np

L = np.log(2) / 2 * 1.001
deg, n = 11, 2000
t = np.cos(np.pi * (np.arange(n) + 0.5) / n) * L
f = (np.expm1(t) - t) / t ** 2
c, *_ = np.linalg.lstsq(np.vander(t, deg - 1, increasing=True), f, rcond=None)
coeffs = np.concatenate([[1.0, 1.0], c])
print([float(v).hex() for v in coeffs[::-1]])
