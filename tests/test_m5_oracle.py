"""Pins of the M5P oracle (oracle/m5.py, NEXT-2) -- CPU only.

Against what the paper and SPEC fix: SPEC's worked examples (S:219-221,
S:226-228), closed forms (SDR of {1,1,5,5}; the smoothing recurrence), the
invariants S:241-245 (SDR >= 0, coefficient confinement, constant-label
collapse, label shift), brute force (the chosen split maximises SDR over an
independent enumeration), and recovery of a noiseless linear label."""
import math
import random

import numpy as np
import pytest

from oracle import m5


def test_constant_labels_single_leaf():
    X = [[float(i), float(i % 3)] for i in range(12)]
    y = [1.25] * 12
    root = m5.m5_build(X, y)
    assert root.leaf
    for x in ([0.0, 0.0], [100.0, -5.0]):
        assert m5.m5_predict(root, x) == 1.25


def test_sdr_worked_example():
    # labels {1,1,5,5} split perfectly -> SDR = 2.0 - 0.5*0 - 0.5*0 = 2.0 (population sd)
    assert m5.sd_pop([1, 1, 5, 5]) == 2.0
    assert m5.sdr([1, 1, 5, 5], [True, True, False, False]) == 2.0
    X = [[0.0], [0.1], [0.9], [1.0]]
    a, thr, s = m5.best_split(X, [1.0, 1.0, 5.0, 5.0], [0, 1, 2, 3])
    assert (a, thr, s) == (0, 0.5, 2.0)


def test_best_split_is_the_brute_force_maximum():
    rng = random.Random(7)
    for _ in range(30):
        n, d = rng.randint(4, 14), rng.randint(1, 4)
        X = [[rng.choice([0.0, 0.25, 0.5, 0.75, 1.0]) for _ in range(d)] for _ in range(n)]
        y = [rng.uniform(0.5, 1.5) for _ in range(n)]
        got = m5.best_split(X, y, list(range(n)))
        # independent enumeration with numpy variances
        cands = []
        for a in range(d):
            col = np.array([r[a] for r in X])
            vals = np.unique(col)
            for lo, hi in zip(vals[:-1], vals[1:]):
                thr = (lo + hi) / 2
                L, R = np.array(y)[col <= thr], np.array(y)[col > thr]
                s = np.std(y) - len(L) / n * np.std(L) - len(R) / n * np.std(R)
                cands.append((s, -a, -thr))
        if not cands:
            assert got is None
            continue
        smax = max(c[0] for c in cands)
        assert got[2] >= smax - 1e-12
        assert got[2] >= -1e-15                      # S:241 SDR non-negativity


def test_noiseless_linear_label_recovered():
    # label = 1 + 0.5 f1 - 0.3 f2 over 200 instances -> held-out RMSE < 0.01
    rng = np.random.default_rng(3)
    Xtr = rng.uniform(0, 1, size=(200, 2))
    ytr = 1 + 0.5 * Xtr[:, 0] - 0.3 * Xtr[:, 1]
    root = m5.m5_build(Xtr.tolist(), ytr.tolist())
    Xte = rng.uniform(0, 1, size=(100, 2))
    pred = np.array([m5.m5_predict(root, x) for x in Xte.tolist()])
    rmse = math.sqrt(float(np.mean((pred - (1 + 0.5 * Xte[:, 0] - 0.3 * Xte[:, 1])) ** 2)))
    assert rmse < 0.01


def _random_tree(seed, n=40, d=3):
    rng = np.random.default_rng(seed)
    X = rng.uniform(0, 1, size=(n, d))
    y = np.where(X[:, 0] > 0.5, 1.3, 0.8) + 0.2 * X[:, 1] + 0.01 * rng.standard_normal(n)
    return X.tolist(), y.tolist()


@pytest.mark.parametrize("seed", range(6))
def test_coefficient_confinement_and_leaf_models(seed):
    """a node's model uses only features split on in its
    subtree; original leaves are intercept-only."""
    X, y = _random_tree(seed)
    root = m5.m5_build(X, y)

    def splits_below(nd):
        if nd.leaf:
            return set()
        return {nd.feature} | splits_below(nd.left) | splits_below(nd.right)

    for nd in m5.walk(root):
        used = {a for a, w in nd.model[1].items() if w != 0.0}
        assert used <= set(nd.allowed)
        if not nd.leaf:
            assert set(nd.allowed) >= splits_below(nd)


@pytest.mark.parametrize("seed", range(4))
def test_label_shift_shifts_predictions(seed):
    """adding c to every label shifts every prediction by c (splits and
    SDR are shift-invariant; intercepts absorb the shift)."""
    X, y = _random_tree(seed)
    c = 0.375
    r0, r1 = m5.m5_build(X, y), m5.m5_build(X, [v + c for v in y])
    rng = np.random.default_rng(seed + 100)
    for x in rng.uniform(0, 1, size=(20, 3)).tolist():
        assert abs(m5.m5_predict(r1, x) - (m5.m5_predict(r0, x) + c)) <= 1e-9


def test_smoothing_recurrence_by_hand():
    """a two-leaf model with hand-set models and counts; the smoothed
    value follows p' = (n p + k q)/(n + k) with n the count of the node below."""
    root = m5.Node(list(range(30)))
    left, right = m5.Node(list(range(12))), m5.Node(list(range(12, 30)))
    root.feature, root.thr, root.left, root.right = 0, 0.5, left, right
    root.model = (1.0, {0: 2.0})
    left.model, right.model = (3.0, {}), (-1.0, {})
    x = [0.25]
    q = 1.0 + 2.0 * 0.25
    assert m5.m5_predict(root, x) == (12 * 3.0 + 15 * q) / (12 + 15)
    x = [0.5]                                         # boundary -> left
    assert m5.m5_predict(root, x) == (12 * 3.0 + 15 * (1.0 + 2.0 * 0.5)) / 27


def test_stop_rules():
    # |T| < 4 -> leaf; sd below 5 % of the root's -> leaf
    X = [[0.0], [1.0], [2.0]]
    assert m5.m5_build(X, [1.0, 2.0, 3.0]).leaf
    X = [[float(i)] for i in range(8)]
    y = [1.0, 1.0, 1.0, 1.0, 9.0, 9.0, 9.0, 9.0 + 1e-9]
    root = m5.m5_build(X, y)
    assert not root.leaf or root.model is not None
    with pytest.raises(ValueError):
        m5.m5_build([], [])


def test_ridge_fit_exact_on_planted_line():
    X = [[0.0], [0.25], [0.5], [1.0]]
    y = [2.0, 2.5, 3.0, 4.0]                         # y = 2 + 2x exactly
    b, w = m5.ridge_fit(X, y, [0, 1, 2, 3], [0], lam=0.0)
    assert b == 2.0 and w[0] == 2.0


def test_scenario_plumbing_matches_the_c_oracle():
    """oracle/m5.evaluate with learner="ridge" runs the same path as the C
    oracle's ridge learner (pairs, membership, scaling, clamp, scores,
    ranking), so counts, fingerprints and recommendations agree exactly and
    EX within 1e-9 on C1 (LOO) and C2 (GROUPS, Table-2 Exp 1/4/5)."""
    import gen
    import oracle
    for name, scen in (("C1", [0, 17, 40]), ("C2", [0, 100, 190])):
        cfg = gen.make_config(name)
        for s in scen:
            got = m5.evaluate(cfg.dataset, cfg.scenarios, s, 1, learner="ridge")
            ref = oracle.evaluate(cfg.dataset, cfg.scenarios, s, 1, want_ex=True)
            for f in ("n_train", "n_test", "n_correct", "n_clamped", "fp_train", "fp_test"):
                assert np.array_equal(got["opt"][f], ref["opt"][f]), (name, s, f)
            for f in ("n_rec", "n_rec_hit", "n_untrained"):
                assert np.array_equal(got["scn"][f], ref["scn"][f]), (name, s, f)
            err = np.abs(got["ex"] - ref["ex"]) / np.maximum(1.0, np.abs(ref["ex"]))
            assert err.max() <= 1e-9, (name, s, err.max())


def test_m5_scenarios_run_and_score():
    """M5P on C1 scenarios: every test case predicted, finite, scored."""
    import gen
    cfg = gen.make_config("C1")
    r = m5.evaluate(cfg.dataset, cfg.scenarios, 0, 4)
    opt = r["opt"]
    assert (opt["n_test"].sum() > 0) and np.isfinite(r["ex"]).all()
    assert (opt["n_correct"] <= opt["n_test"]).all()
