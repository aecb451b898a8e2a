"""Randomised region configurations shared by the parity suites.

A case is a pure TABLE region (any reference Region whose evaluate is a
function of the work index, engine.hpp:19-25) plus grid, mapping and spec.
The same case runs through the CUDA engine (GPU tests), the C restatement
(oracle/liboracle.so) and the reference itself (oracle/_ref).
"""
from __future__ import annotations

import copy
from dataclasses import dataclass

import numpy as np

from paper_2308_16877_b200 import abi
from paper_2308_16877_b200 import engine as E

INF = float("inf")


@dataclass
class Case:
    grid: E.GridConfig
    n: int
    mapping: int
    in_dims: int
    out_dims: int
    inputs: np.ndarray | None
    table: np.ndarray
    encounters: np.ndarray | None
    accumulate: bool
    barrier: bool
    spec: object
    init: np.ndarray

    def region(self, out, xp=np):
        """Region over buffers `out` (numpy for oracle/ref, torch for CUDA)."""
        return E.table_region(self.inputs if xp is np else xp(self.inputs),
                              self.table if xp is np else xp(self.table), out,
                              input_dims=self.in_dims, output_dims=self.out_dims,
                              encounters=self.encounters if xp is np else (None if self.encounters is None else xp(self.encounters)),
                              accumulate=self.accumulate, barrier=self.barrier)

    def describe(self):
        s = self.spec
        sd = None if s is None else {f: getattr(s, f) for f, _ in s._fields_}
        return dict(grid=self.grid, n=self.n, mapping=self.mapping, in_dims=self.in_dims,
                    out_dims=self.out_dims, enc=self.encounters is not None,
                    acc=self.accumulate, barrier=self.barrier, spec=sd)


def _values(rng, kind, n, tid, step, lane, dims):
    """Output/input streams with temporal structure (constant, drift, noise,
    lane-split, small discrete set for iACT hits)."""
    out = np.empty((n, dims))
    for d in range(dims):
        if kind == "const":
            out[:, d] = 7.5 + d
        elif kind == "drift":
            out[:, d] = 50.0 * (1.0 + 1e-3 * step) + d
        elif kind == "noise":
            out[:, d] = rng.uniform(1.0, 2.0, n)
        elif kind == "lanesplit":
            out[:, d] = np.where(lane % 3 == 0, 1.0 + 0.37 * np.arange(n), 42.0 + d)
        elif kind == "discrete":
            out[:, d] = rng.integers(0, 3, n).astype(np.float64)
        elif kind == "tidconst":
            out[:, d] = 1.0 + (tid % 5) + 0.001 * rng.integers(0, 2, n)
        elif kind == "zero_mean":
            out[:, d] = np.where(rng.random(n) < 0.5, -1.0, 1.0) * (lane % 2)
        else:
            raise ValueError(kind)
    return out


def random_case(rng, allow_random_perfo=False, allow_per_team=True, max_threads=96,
                allow_generic_ws=True):
    ws_choices = [1, 2, 4, 8, 16, 32] + ([3, 6, 12, 64] if allow_generic_ws else [])
    ws = int(rng.choice(ws_choices))
    mult = int(rng.integers(1, 4))
    tpt = ws * mult
    while tpt > max_threads and mult > 1:
        mult -= 1
        tpt = ws * mult
    teams = int(rng.integers(1, 4))
    ipt = int(rng.integers(1, 9))
    mapping = abi.MAP_PER_TEAM if (allow_per_team and rng.random() < 0.2) else abi.MAP_PER_THREAD
    cap = teams * ipt * (1 if mapping == abi.MAP_PER_TEAM else tpt)
    n = int(rng.integers(0, cap + 1)) if rng.random() < 0.3 else cap
    budget = 48 * 1024 if rng.random() < 0.85 else int(rng.choice([16, 64, 256, 1024, 4096]))
    grid = E.GridConfig(teams, tpt, ws, ipt, budget)

    G = teams * tpt
    idx = np.arange(n)
    if mapping == abi.MAP_PER_THREAD:
        step = idx // G
        tid = idx % G
        lane = (tid % tpt) % ws
    else:
        step = idx // teams
        tid = idx % teams
        lane = np.zeros(n, dtype=np.int64)

    tech = rng.choice(["none", "taf", "iact", "perfo"], p=[0.1, 0.35, 0.3, 0.25])
    in_dims = int(rng.integers(1, 4)) if tech == "iact" else int(rng.integers(0, 3))
    out_dims = int(rng.integers(1, 3))
    kind_out = rng.choice(["const", "drift", "noise", "lanesplit", "discrete", "tidconst", "zero_mean"])
    table = _values(rng, kind_out, n, tid, step, lane, out_dims)
    inputs = None
    if in_dims > 0:
        kind_in = rng.choice(["discrete", "noise", "const", "tidconst"])
        inputs = _values(rng, kind_in, n, tid, step, lane, in_dims)
    encounters = None
    if mapping == abi.MAP_PER_THREAD and rng.random() < 0.2:
        encounters = rng.integers(1, 4, n).astype(np.int32)
    level = int(rng.choice([0, 1, 2]))
    spec = None
    if tech == "taf":
        spec = E.taf(int(rng.integers(1, 6)), int(rng.integers(1, 9)),
                     float(rng.choice([0.0, 0.01, 0.1, 0.5, 1.5, INF])), level)
    elif tech == "iact":
        tpw = None
        if rng.random() < 0.6:
            divs = [d for d in range(1, ws + 1) if ws % d == 0]
            tpw = int(rng.choice(divs))
        spec = E.iact(int(rng.integers(1, 5)), float(rng.choice([0.0, 0.3, 0.5, 1.5, INF])), tpw, level)
    elif tech == "perfo":
        kinds = ["small", "large", "ini", "fini", "herded_small", "herded_large"]
        if allow_random_perfo:
            kinds.append("random")
        k = str(rng.choice(kinds))
        if k in ("ini", "fini", "random"):
            arg = int(rng.integers(1, 100))
        else:
            arg = int(rng.integers(2, 7))
        spec = E.perfo(k, arg, level, seed=int(rng.integers(0, 2**31)))
        if k in ("ini", "fini"):
            encounters = None
    accumulate = encounters is not None and rng.random() < 0.5
    barrier = rng.random() < 0.1
    init = np.full((n, out_dims), -1.0)
    return Case(grid, n, mapping, in_dims, out_dims, inputs, table, encounters, accumulate,
                barrier, spec, init)


def clone_spec(spec):
    return None if spec is None else copy.copy(spec)
