"""GPU parity of the Tier-3 rule sweep (sr_sweep) vs the
oracle: the paper's rule (readings R8-R10, R13) applied by the oracle's
own rank-and-filter (or_rank) once per (threshold, list length) to the
oracle's own EX of every test version, counts of recommendations and of
recommendations with AC > 1 (R11) pooled over the scenarios.  Integer
results: exact equality (scenarios with guard cases, reading R21, excluded
from the comparison batch by construction of the check)."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


def _oracle_sweep(cfg, first, count, thr, cnt, learner=0, k=10):
    ds, sc = cfg.dataset, cfg.scenarios
    if learner == 2:      # M5P (NEXT-2): the model-tree oracle
        from oracle import m5
        ref = m5.evaluate(ds, sc, first, count)
    else:
        ref = oracle.evaluate(ds, sc, first, count, want_ex=True, learner=learner, k_nn=k)
    assert ref["scn"]["n_guard"].sum() == 0
    G, O = ds.n_groups, ds.n_opt_ids
    rt = ds.runtime_ms
    rec = np.zeros((len(thr), len(cnt)), np.int64)
    hit = np.zeros_like(rec)
    for s in range(count):
        trained = ref["opt"]["n_train"][s] > 0
        for g in range(G):
            p = g // (ds.n_inputs * ds.n_runs)
            for v in range(64):
                ids, exs, acs = [], [], []
                for o in range(O):
                    b = int(ds.opt_bit[p, o])
                    if b < 0 or (v >> b) & 1 or not trained[o]:
                        continue
                    kk = (v & ((1 << b) - 1)) | ((v >> (b + 1)) << b)
                    e = ref["ex"][s, o, g * 32 + kk]
                    if e == 0.0:          # not a test case of this scenario
                        continue
                    ids.append(o)
                    exs.append(e)
                    acs.append(rt[g * 64 + v] / rt[g * 64 + (v | (1 << b))])
                if not ids:
                    continue
                for i, th in enumerate(thr):
                    for j, K in enumerate(cnt):
                        _, r = oracle.rank(np.array(exs), np.array(ids), th, int(K))
                        rec[i, j] += len(r)
                        hit[i, j] += sum(acs[ids.index(o)] > 1.0 for o in r)
    return rec, hit


@pytest.mark.parametrize("name, kw, count, learner", [
    ("C2", {}, 240, 0),
    ("C3", dict(n_splits=300), 300, 0),
    ("C1", {}, 64, 1),
    ("C1", {}, 64, 2),
])
def test_sweep_matches_the_rule_applied_per_setting(name, kw, count, learner):
    from paper_1910_07776_b200 import Context, default_params
    cfg = gen.make_config(name, **kw)
    thr = np.array([0.5, 0.9, 1.0, 1.02, 1.05, 1.1, 1.2, 1.5])
    cnt = np.array([1, 3, 6])
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    rec, hit = ctx.sweep(thr, cnt, 0, count, params=default_params(learner=learner))
    # the default rule (theta 1.05, K 3) is the same count sr_evaluate reports
    got = ctx.evaluate(0, count, params=default_params(learner=learner))
    ctx.close()
    i, j = list(thr).index(1.05), list(cnt).index(3)
    assert rec[i, j] == got["scn"]["n_rec"].sum() and hit[i, j] == got["scn"]["n_rec_hit"].sum()
    r_ref, h_ref = _oracle_sweep(cfg, 0, count, thr, cnt, learner=learner)
    assert np.array_equal(rec, r_ref), (rec, r_ref)
    assert np.array_equal(hit, h_ref), (hit, h_ref)
    # monotone in both knobs
    assert np.all(np.diff(rec, axis=0) <= 0) and np.all(np.diff(rec, axis=1) >= 0)


def test_sweep_argument_errors():
    from paper_1910_07776_b200 import Context, SpeedrecError
    cfg = gen.make_config("C1")
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    with pytest.raises(SpeedrecError, match="ascending"):
        ctx.sweep([1.1, 1.0], [3])
    with pytest.raises(SpeedrecError, match="max_counts"):
        ctx.sweep([1.0], [0])
    ctx.close()
