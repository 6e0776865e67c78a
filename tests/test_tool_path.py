"""Tool path of the boundary (include/speedrec.h): sr_fit (GPU), sr_predict and
sr_recommend (host functions of the library; SPEC train_all S:282,
predict_all S:291, rank_and_filter S:300).

sr_predict / sr_recommend are pinned on CPU against exact arithmetic, the
SPEC's worked examples and the oracle's rank; sr_fit (GPU) is checked by
predicting every test case of a scenario from the fitted models and comparing
with the oracle's EX (1e-9 relative).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


@pytest.fixture(scope="module")
def S():
    from paper_1910_07776_b200 import build, speedrec
    build.build_library()
    return speedrec


def test_predict_exact_dot_product(S):
    rng = np.random.default_rng(5)
    O, C = 6, 37
    coef = rng.normal(size=(O, C + 1))
    coef[2, 0] = np.nan                       # no model for id 2
    coef[4, 0] = -1e3                         # forces a clamp
    counters = np.round(rng.uniform(0, 1e6, size=C))
    cycles = 7.06e5 * 3.0
    ex = S.predict(coef, counters, cycles)
    for o in range(O):
        if o == 2:
            assert np.isnan(ex[o])
            continue
        x = [Fraction(float(c) / cycles) for c in counters]      # IEEE rates
        exact = Fraction(float(coef[o, 0])) + sum(Fraction(float(u)) * xc for u, xc in zip(coef[o, 1:], x))
        if exact <= 0:
            assert ex[o] == 0.01                 # S:327 clamp
        else:
            assert abs(Fraction(float(ex[o])) - exact) <= Fraction(1, 10 ** 12) * max(1, abs(exact))


def test_predict_rejects_bad_profiles(S):
    coef = np.zeros((2, 4))
    with pytest.raises(S.SpeedrecError):
        S.predict(coef, np.array([1.0, -1.0, 0.0]), 10.0)          # negative counter
    with pytest.raises(S.SpeedrecError):
        S.predict(coef, np.array([1.0, 1.0, 0.0]), 0.0)            # cycles <= 0
    with pytest.raises(S.SpeedrecError):
        S.predict(coef, np.array([1.0, np.inf, 0.0]), 5.0)


def test_recommend_spec_examples(S):
    g = json.load(open(GOLDEN))["rank_and_filter"]
    for case in g["cases"]:
        names = sorted(case["ids"], key=lambda k: case["ids"][k])
        ex = np.array([case["pred"][k] for k in names])
        p = S.default_params(threshold=case["threshold"], max_count=case["max_count"])
        got = S.recommend(ex, params=p)
        assert [names[i] for i in got] == case["expect"], case


def test_recommend_matches_oracle_rank(S):
    rng = np.random.default_rng(9)
    for trial in range(2000):
        n = int(rng.integers(0, 11))
        ex = np.round(rng.uniform(0.8, 1.4, size=n), 2)        # many exact ties
        cand = rng.random(n) < 0.8
        ex[rng.random(n) < 0.1] = np.nan                        # untrained ids
        thr = float(rng.choice([1.0, 1.05, 1.2]))
        k = int(rng.integers(1, 9))
        got = S.recommend(ex, cand, params=S.default_params(threshold=thr, max_count=k))
        ids = np.flatnonzero(cand & ~np.isnan(ex)).astype(np.int32)
        _, want = oracle.rank(ex[ids], ids, threshold=thr, max_count=k)
        assert got == want, (ex, cand, thr, k)


def _slot_of(g, b, k):
    """before slot of pair k of group g for bit b (P:118 pair rank)."""
    v = (k & ((1 << b) - 1)) | ((k >> b) << (b + 1))
    return g * 64 + v


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw,scen", [("C1", {}, [0, 17, 63]), ("C2", {}, [0, 30, 100, 239]),
                                          ("C3", dict(n_splits=500), [0, 499]),
                                          ("C5", dict(n_masks_k=4), [0, 1000, 2047]),
                                          ("C4", dict(n_splits=4, n_programs=96), [1])])
def test_fit_predicts_the_oracle_ex(S, name, kw, scen):
    cfg = gen.make_config(name, **kw)
    ds, sc = cfg.dataset, cfg.scenarios
    ctx = S.Context(0)
    ctx.load(ds)
    ctx.define_scenarios(sc)
    worst = 0.0
    for s in scen:
        coef = ctx.fit(s)
        ref = oracle.evaluate(ds, sc, s, 1, want_ex=True)
        I_R = ds.n_inputs * ds.n_runs
        for o in range(ds.n_opt_ids):
            trained = ref["opt"]["n_train"][0, o] > 0
            assert np.isnan(coef[o, 0]) == (not trained)
            if not trained:
                continue
            for j in np.flatnonzero(ref["ex"][0, o]):
                g, k = divmod(int(j), 32)
                b = int(ds.opt_bit[g // I_R, o])
                t = _slot_of(g, b, k)
                e = S.predict(coef[o:o + 1], ds.counters[t], ds.cycles[t])[0]
                r = ref["ex"][0, o, j]
                err = abs(e - r) / max(1.0, abs(r))
                worst = max(worst, err)
                assert err <= 1e-9, (s, o, j, e, r)
    ctx.close()
    print(name, "sr_fit -> sr_predict worst rel err", worst)


@pytest.mark.gpu
def test_fit_rejects_ibk_and_bad_state(S):
    cfg = gen.make_config("C1")
    ctx = S.Context(0)
    with pytest.raises(S.SpeedrecError):
        ctx.fit(0)                                              # no dataset
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    with pytest.raises(S.SpeedrecError, match="IBK"):
        ctx.fit(0, S.default_params(learner=1))
    with pytest.raises(S.SpeedrecError):
        ctx.fit(64)                                             # out of range
    ctx.close()


@pytest.mark.gpu
def test_tier1_ingested_dataset_end_to_end(S):
    """NEXT-4: the C2 lattice exported to canonical CSV and ingested again
    (paper_1910_07776_b200.tier1) gives the same batched results as the
    generated arrays (all 240 Table-2 scenarios, bit-identical), and the
    single-profile tool path (sr_fit -> sr_predict -> sr_recommend) runs on it."""
    from paper_1910_07776_b200 import Context, predict, recommend
    from paper_1910_07776_b200 import tier1 as T
    cfg = gen.make_config("C2")
    ds2, info = T.to_dataset(T.parse_canonical_csv(T.serialize_canonical_csv(T.dataset_to_records(cfg.dataset))))
    outs = []
    for ds in (cfg.dataset, ds2):
        ctx = Context(0)
        ctx.load(ds)
        n = ctx.define_scenarios(cfg.scenarios)
        outs.append(ctx.evaluate(0, n, want_ex=True, want_recs=True))
        if ds is ds2:
            coef = ctx.fit(0)
            prof = ds2.counters[5]
            ex = predict(coef, prof, float(ds2.cycles[5]))
            rec = recommend(ex)
            assert np.all(np.isfinite(ex[coef[:, 0] == coef[:, 0]]))
            assert len(rec) <= 3
        ctx.close()
    a, b = outs
    for k in ("ex", "recs"):
        assert np.array_equal(a[k], b[k]), k
    for part in ("opt", "scn"):
        for f in a[part].dtype.names:
            assert np.array_equal(a[part][f], b[part][f]), (part, f)
