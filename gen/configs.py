"""The five workload configs of BASELINE.json as concrete synthetic inputs.

SURVEY §8(d) "The five configs".  A config = a dataset (gen.synth) + a
scenario batch description.  The description only *names* the scenarios
(which groups are train/test, which feature subsets, which seed); turning it
into slot membership is the method's job and happens independently in the
oracle and in the CUDA path.

Scenario s of a batch is (feature-mask index f, split index k) with
s = f * n_splits + k.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .synth import BH_OPTS, NB_OPTS, OPT_NAMES_C2, TABLE1, Dataset, generate

GENERIC_OPTS = [f"O{j}" for j in range(6)]


@dataclass
class Scenarios:
    """Mirror of `sr_scenarios` in include/speedrec.h (plain data)."""
    kind: str                                   # "groups" | "loo" | "random"
    n_splits: int
    group_words: int
    train_groups: Optional[np.ndarray] = None   # uint64 [n_splits][group_words]  (groups)
    test_groups: Optional[np.ndarray] = None    # uint64 [n_splits][group_words]  (groups)
    split_opt_masks: Optional[np.ndarray] = None  # uint32 [n_splits] scored optimization ids (groups)
    pool_groups: Optional[np.ndarray] = None    # uint64 [group_words]            (loo)
    seed: int = 0                               # (random)
    opt_mask: int = 0xFFFFFFFF                  # scored optimization ids when split_opt_masks is None
    n_masks: int = 1
    feature_masks: Optional[np.ndarray] = None  # uint64 [n_masks][2]; None = all counters
    all_subsets_k: int = 0                      # >0: feature mask f = all subsets of counters [0,k)
    aggregate_folds: bool = False               # C5: reduce rows over splits per mask

    @property
    def n_scenarios(self) -> int:
        return self.n_splits * self.n_masks


@dataclass
class Config:
    name: str
    dataset: Dataset
    scenarios: Scenarios
    description: str


def _bits(groups, words):
    out = np.zeros(words, dtype=np.uint64)
    for g in groups:
        out[g // 64] |= np.uint64(1) << np.uint64(g % 64)
    return out


def table2_scenarios(ds: Dataset, opt_names) -> Scenarios:
    """All 240 instantiations of the paper's Table 2 experiments.

    Programs: p=0 BH, p=1 NB; group g = (p*I + i)*R + r.
      Exp 1 (p,i,r):      train {(p,i,r)}, test {(p,i,*)}   -- test includes train
      Exp 2 (p,i,r):      train {(p,i,r)}, test {(p,i,r'!=r)}
      Exp 3 (p,i,r):      train {(p,i,r'!=r)}, test {(p,i,r)}
      Exp 4 (p,i,i',r'):  train {(p,i,*)}, test {(p,i',r')}, i'!=i
      Exp 5 (i,i',r'):    train {(BH,i,*)}, test {(NB,i',r')}; FTZ, RSQRT only
      Exp 6 (i,i',r'):    train {(NB,i,*)}, test {(BH,i',r')}; FTZ, RSQRT only
    Scored optimizations: the program's six for Exp 1-4; {FTZ, RSQRT} for Exp 5/6.
    Order: Exp 1..6, then loops in the order written above (reading R15).
    """
    P, I, R = ds.n_programs, ds.n_inputs, ds.n_runs
    assert P in (1, 2)          # 1: BH alone (config BH6, Exp 1-4)
    G = P * I * R
    W = (G + 63) // 64
    gid = lambda p, i, r: (p * I + i) * R + r
    prog_mask = []
    for p in range(P):
        mk = 0
        for o in range(ds.n_opt_ids):
            if ds.opt_bit[p, o] >= 0:
                mk |= 1 << o
        prog_mask.append(mk)
    shared = (1 << opt_names.index("FTZ")) | (1 << opt_names.index("RSQRT"))
    rows = []  # (train groups, test groups, opt mask, exp id)
    for p in range(P):
        for i in range(I):
            for r in range(R):
                rows.append(([gid(p, i, r)], [gid(p, i, rr) for rr in range(R)], prog_mask[p], 1))
    for p in range(P):
        for i in range(I):
            for r in range(R):
                rows.append(([gid(p, i, r)], [gid(p, i, rr) for rr in range(R) if rr != r], prog_mask[p], 2))
    for p in range(P):
        for i in range(I):
            for r in range(R):
                rows.append(([gid(p, i, rr) for rr in range(R) if rr != r], [gid(p, i, r)], prog_mask[p], 3))
    for p in range(P):
        for i in range(I):
            for i2 in range(I):
                if i2 == i:
                    continue
                for r2 in range(R):
                    rows.append(([gid(p, i, rr) for rr in range(R)], [gid(p, i2, r2)], prog_mask[p], 4))
    for ptrain, ptest, e in (((0, 1, 5), (1, 0, 6)) if P == 2 else ()):
        for i in range(I):
            for i2 in range(I):
                for r2 in range(R):
                    rows.append(([gid(ptrain, i, rr) for rr in range(R)], [gid(ptest, i2, r2)], shared, e))
    n = len(rows)
    tr = np.zeros((n, W), dtype=np.uint64)
    te = np.zeros((n, W), dtype=np.uint64)
    om = np.zeros(n, dtype=np.uint32)
    for k, (a, b, mk, _) in enumerate(rows):
        tr[k] = _bits(a, W)
        te[k] = _bits(b, W)
        om[k] = mk
    sc = Scenarios(kind="groups", n_splits=n, group_words=W, train_groups=tr, test_groups=te,
                   split_opt_masks=om)
    sc.experiment = np.array([e for *_, e in rows], dtype=np.int32)
    return sc


def make_config(name: str, n_splits: Optional[int] = None, n_masks_k: Optional[int] = None,
                n_programs: Optional[int] = None) -> Config:
    """Build config C1..C5; optional overrides shrink it for tests."""
    c = int(name[1]) if name[1].isdigit() else 6
    dseed, sseed = 1910 + c, 7776 + c
    if name == "C1":
        ds = generate(n_programs=1, n_inputs=1, n_runs=1, n_counters=32, seed=dseed,
                      opt_names=BH_OPTS, program_opts=[BH_OPTS], program_names=["BH"],
                      small_opt="FTZ")
        sc = Scenarios(kind="loo", n_splits=64, group_words=1, pool_groups=_bits([0], 1))
        desc = "1 program x 64 variants, 32 counters, leave-one-variant-out, 6 opts"
    elif name == "C2":
        ds = generate(n_programs=2, n_inputs=4, n_runs=3, n_counters=32, seed=dseed,
                      opt_names=OPT_NAMES_C2, program_opts=[BH_OPTS, NB_OPTS],
                      program_names=["BH", "NB"],
                      input_sizes=[TABLE1["BH"][:4], TABLE1["NB"]], small_opt="FTZ")
        sc = table2_scenarios(ds, OPT_NAMES_C2)
        desc = "BH+NB x 4 inputs x 3 runs x 64 variants, 32 counters, all 240 Table-2 instantiations"
    elif name == "BH6":
        # NEXT-3: Barnes-Hut with all six Table-1 inputs, Table-2 Exp 1-4
        ds = generate(n_programs=1, n_inputs=6, n_runs=3, n_counters=32, seed=1910 + 6,
                      opt_names=OPT_NAMES_C2, program_opts=[BH_OPTS], program_names=["BH"],
                      input_sizes=[TABLE1["BH"]], small_opt="FTZ")
        sc = table2_scenarios(ds, OPT_NAMES_C2)
        desc = "BH x 6 inputs (Table 1) x 3 runs x 64 variants, 32 counters, Table-2 Exp 1-4 (144)"
    elif name == "C3":
        # n_programs=1: one group, so a fit's n ~ Bin(32, 1/4) reaches the
        # degenerate fits n = 0 (R18 untrained), 1, 2, 3 (parity edge cases)
        P = n_programs or 2
        ds = generate(n_programs=P, n_inputs=1, n_runs=1, n_counters=64, seed=dseed,
                      opt_names=GENERIC_OPTS, program_opts=[GENERIC_OPTS] * P,
                      small_opt="O0")
        sc = Scenarios(kind="random", n_splits=n_splits or 1_000_000, group_words=1, seed=sseed)
        desc = f"{P} programs x 64 variants, 64 counters, random slot splits"
    elif name == "C4":
        P = n_programs or 1024
        ds = generate(n_programs=P, n_inputs=1, n_runs=1, n_counters=128, seed=dseed,
                      opt_names=GENERIC_OPTS, program_opts=[GENERIC_OPTS] * P, small_opt="O0")
        sc = Scenarios(kind="random", n_splits=n_splits or 10_000_000,
                       group_words=(P + 63) // 64, seed=sseed)
        desc = f"{P} programs x 64 variants, 128 counters, random slot splits"
    elif name == "C5":
        k = n_masks_k if n_masks_k is not None else 20
        ds = generate(n_programs=2, n_inputs=1, n_runs=1, n_counters=20, seed=dseed,
                      opt_names=GENERIC_OPTS, program_opts=[GENERIC_OPTS, GENERIC_OPTS],
                      small_opt="O0")
        sc = Scenarios(kind="loo", n_splits=128, group_words=1, pool_groups=_bits([0, 1], 1),
                       n_masks=1 << k, all_subsets_k=k, aggregate_folds=True)
        desc = f"2 programs x 64 variants, 20 counters, all 2^{k} feature subsets x 128 LOO folds"
    else:
        raise ValueError(name)
    if n_splits is not None and sc.kind != "random":
        sc.n_splits = min(sc.n_splits, n_splits)
        if sc.kind == "groups":
            sc.train_groups = sc.train_groups[:sc.n_splits]
            sc.test_groups = sc.test_groups[:sc.n_splits]
            sc.split_opt_masks = sc.split_opt_masks[:sc.n_splits]
    return Config(name, ds, sc, desc)


CONFIGS = ["C1", "C2", "C3", "C4", "C5"]
