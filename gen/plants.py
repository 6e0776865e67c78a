"""Constructed (planted) inputs for the oracle pins and the GPU edge-case tests.

Like the rest of `gen`, this module holds no arithmetic of the method: it
only writes Tier-1 inputs (integer counters, cycles, runtimes, optimization
bits) whose labels rt(before) / rt(after) follow a chosen rule, so that the
method's result is known in closed form.  Each builder names the passage
whose rule it exercises.
"""
from __future__ import annotations

import numpy as np

from .configs import Config, Scenarios, _bits, make_config
from .synth import Dataset

GENERIC = [f"O{j}" for j in range(6)]
POW2_FACTORS = (2.0, 0.5, 4.0, 0.25)   # label of every pair of optimization id o: POW2_FACTORS[o % 4]


def clamp_plant(x_held: float = 3.0, ac_held: float = 1.5, seed: int = 327) -> Config:
    """S:327 ("clamp predictions <= 0 to 0.01 before ranking"): one program,
    two counters (counter 1 constant, hence inactive, D3), LOO over the 64
    versions, only optimization 0 (bit 0) scored.  For every before version
    v != 0 the rate of counter 0 lies in [1, 2] and the label is planted on
    the line AC = 2.1 - x; version 0 has x = x_held and AC = ac_held.  Split 0
    holds out version 0: its 31 training pairs lie exactly on the line, so
    the ridge prediction is 2.1 - x_held up to the ridge bias (x_held = 3 ->
    EX ~ -0.9, clamped; x_held = 2.05 -> EX ~ 0.05, kept)."""
    rng = np.random.default_rng(seed)
    V, C = 64, 2
    cycles = np.full(V, 1_000_000.0)
    x = rng.uniform(1.0, 2.0, size=V)
    x[0] = x_held
    counters = np.zeros((V, C))
    counters[:, 0] = np.rint(x * 1e6)
    counters[:, 1] = 500_000.0
    xr = counters[:, 0] / 1e6            # the integer counters' exact rates
    rt = np.zeros(V)
    for v in range(0, V, 2):
        rt[v] = 10.0
        f = ac_held if v == 0 else 2.1 - xr[v]
        rt[v | 1] = rt[v] / f
    ob = np.array([[0, 1, 2, 3, 4, 5]], dtype=np.int8)
    ds = Dataset(1, 1, 1, 6, C, 6, counters, cycles, rt, ob, list(GENERIC), ["P0"])
    sc = Scenarios(kind="loo", n_splits=64, group_words=1, pool_groups=_bits([0], 1), opt_mask=1)
    return Config("clamp", ds, sc, f"S:327 clamp plant, held-out x = {x_held}")


def pow2_lattice(name: str = "C1", **kw) -> Config:
    """Perfect-predictor identity: config `name` with its
    runtimes replaced by rt(p, v) = 64 * prod 1 / POW2_FACTORS[o % 4] over the
    optimizations o of program p whose bit opt_bit[p][o] is set in v.  Every
    pair of optimization id o then has the label POW2_FACTORS[o % 4] exactly,
    in every program (powers of two: every runtime and every ratio is exact),
    and a fit on constant labels predicts that label exactly, so EX = AC."""
    cfg = make_config(name, **kw)
    ds = cfg.dataset
    V = 1 << ds.n_opt_bits
    rt = np.empty(ds.n_slots)
    for g in range(ds.n_groups):
        p = g // (ds.n_inputs * ds.n_runs)
        for v in range(V):
            r = 64.0
            for o in range(ds.n_opt_ids):
                b = int(ds.opt_bit[p, o])
                if b >= 0 and (v >> b) & 1:
                    r /= POW2_FACTORS[o % 4]
            rt[g * V + v] = r
    ds.runtime_ms = rt
    cfg.name = f"{name}-pow2"
    return cfg


def untrained_groups_split(cfg: Config | None = None) -> Config:
    """R18 (n = 0 -> untrained): on config C2's BH+NB lattice, splits that
    train on BH groups only and test on NB groups while scoring all ten
    optimization ids -- the NB-only ones (absent from BH, opt_bit = -1) have
    no training pair but NB test cases.  Plus the mirror split and one that
    trains on a single run."""
    cfg = cfg or make_config("C2")
    ds = cfg.dataset
    I, R = ds.n_inputs, ds.n_runs
    G = ds.n_groups
    gid = lambda p, i, r: (p * I + i) * R + r
    bh = [gid(0, i, r) for i in range(I) for r in range(R)]
    nb = [gid(1, i, r) for i in range(I) for r in range(R)]
    rows = [(bh, nb), (nb, bh), ([gid(0, 0, 0)], nb[:3] + bh[3:6])]
    W = (G + 63) // 64
    tr = np.stack([_bits(a, W) for a, _ in rows])
    te = np.stack([_bits(b, W) for _, b in rows])
    om = np.full(len(rows), (1 << ds.n_opt_ids) - 1, dtype=np.uint32)
    sc = Scenarios(kind="groups", n_splits=len(rows), group_words=W, train_groups=tr, test_groups=te,
                   split_opt_masks=om)
    return Config("C2-untrained", ds, sc, "R18: optimizations with test cases and no training pair")
