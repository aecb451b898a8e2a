"""Shared helpers for the fastmath accuracy tests: sample points and ulp
errors against mpmath (40 digits)."""
from __future__ import annotations

import mpmath as mp
import numpy as np

mp.mp.dps = 40
BOUNDS = {"exp": 1.0, "log": 1.0, "erfc": 4.0, "rcp": 1.0}


def samples(kind, seed=7, m=600):
    rng = np.random.default_rng(seed)
    if kind == "exp":
        return np.concatenate([rng.uniform(-745, 709, m), rng.uniform(-1, 1, m), rng.uniform(-0.2, 0, m)])
    if kind == "log":
        return np.concatenate([np.exp(rng.uniform(-700, 700, m)), rng.uniform(0.5, 2, m),
                               1 + rng.uniform(-1e-6, 1e-6, m), [5e-320, 1e-310, 1.0]])
    if kind == "erfc":
        return np.concatenate([rng.uniform(-6, 26, m), rng.uniform(-2, 2, m), rng.uniform(0, 8, m)])
    return np.concatenate([rng.uniform(0.1, 10, m), np.exp(rng.uniform(-690, 690, m))])


def reference(kind, x):
    f = {"exp": mp.exp, "log": mp.log, "erfc": mp.erfc, "rcp": lambda v: 1 / v}[kind]
    return [f(mp.mpf(float(v))) for v in x]


def ulp_errors(y, ref):
    out = np.empty(len(y))
    for i, (a, r) in enumerate(zip(y, ref)):
        rf = abs(float(r))
        ulp = np.spacing(rf) if rf >= 2.2250738585072014e-308 else 5e-324
        out[i] = float(abs(mp.mpf(float(a)) - r) / ulp)
    return out
