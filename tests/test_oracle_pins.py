"""Pins of the oracle against what the paper, SPEC and mathematics fix.

None of these tests retypes the oracle's own formula: each compares it with
a worked example (tests/golden/spec_examples.json, cited), exact rational
arithmetic (fractions.Fraction), a closed form, an invariant, an independent
brute-force enumeration, or a library routine on a special case.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle
from gen.synth import Dataset

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
M64 = 2**64 - 1


# --------------------------------------------------------------------- Tier 1
def test_rates_worked_examples():
    for case in GOLD["normalize"]["cases"]:
        c = np.array([case["counters"]], dtype=np.float64)
        cyc = np.array([case["cycles"]], dtype=np.float64)
        if "scaled_by" in case:
            k = case["scaled_by"]
            np.testing.assert_array_equal(oracle.rates(c * k, cyc * k)[0], case["expect"])
        np.testing.assert_array_equal(oracle.rates(c, cyc)[0], case["expect"])


def test_rates_scale_invariance():
    # multiplying cycles and all counters by the same constant leaves
    # the vector unchanged within 1e-12 relative.
    rng = np.random.default_rng(0)
    c = np.rint(rng.uniform(0, 1e7, size=(50, 16)))
    cyc = np.rint(rng.uniform(1e5, 1e8, size=50))
    base = oracle.rates(c, cyc)
    for k in (3.0, 7.5, 1e3):
        np.testing.assert_allclose(oracle.rates(c * k, cyc * k), base, rtol=1e-12, atol=0)


# ----------------------------------------------------------- split hashing
def _py_mix(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def test_mix64_public_test_vector():
    g = int(GOLD["splitmix64"]["gamma"], 16)
    for k, out in enumerate(GOLD["splitmix64"]["outputs"]):
        assert oracle.mix64((k * g) & M64) == int(out, 16)


def test_split_word_independent_python():
    rng = np.random.default_rng(1)
    for _ in range(200):
        seed, split, word = (int(v) for v in rng.integers(0, 2**62, size=3))
        expect = _py_mix((_py_mix(seed ^ _py_mix(split)) + word) & M64)
        assert oracle.split_word(seed, split, word) == expect


# ----------------------------------------------------------- lattice / pairs
def _brute_pairs(ds, tr, te, o):
    """Independent enumeration of (training pairs, test cases) by brute force
    over all slot pairs that differ in exactly optimization o's bit."""
    V = 1 << ds.n_opt_bits
    G = ds.n_groups
    ntr = nte = 0
    fptr = fpte = 0
    for g in range(G):
        p = g // (ds.n_inputs * ds.n_runs)
        b = int(ds.opt_bit[p, o])
        if b < 0:
            continue
        befores = sorted(v for v in range(V) if not (v >> b) & 1)
        assert len(befores) == V // 2       # P:118 "32 versions ... do not ... include"
        for k, v in enumerate(befores):
            t, a = g * V + v, g * V + (v | (1 << b))
            assert bin((t ^ a)).count("1") == 1
            pid = (g * ds.n_opt_ids + o) * (V // 2) + k
            if tr[t] and tr[a]:
                ntr += 1
                fptr ^= _py_mix(pid)
            if te[t]:
                nte += 1
                fpte ^= _py_mix(pid)
    return ntr, nte, fptr, fpte


def test_random_split_counts_and_fingerprints_brute_force():
    cfg = gen.make_config("C3", n_splits=12)
    ds, sc = cfg.dataset, cfg.scenarios
    r = oracle.evaluate(ds, sc, 0, 12)
    N = ds.n_slots
    for s in range(12):
        tr = [(_py_mix((_py_mix(sc.seed ^ _py_mix(s)) + t // 64) & M64) >> (t % 64)) & 1 for t in range(N)]
        te = [1 - v for v in tr]
        for o in range(ds.n_opt_ids):
            row = r["opt"][s, o]
            ntr, nte, fptr, fpte = _brute_pairs(ds, tr, te, o)
            assert (row["n_train"], row["n_test"]) == (ntr, nte)
            assert (int(row["fp_train"]), int(row["fp_test"])) == (fptr, fpte)


def test_loo_removes_exactly_one_pair():
    # "always leaves 32 feature vectors"; LOO over one 64-version group:
    # every optimization keeps 31 training pairs; the held-out version is a
    # test case exactly for the optimizations it lacks (6 - popcount).
    cfg = gen.make_config("C1")
    r = oracle.evaluate(cfg.dataset, cfg.scenarios, 0, 64)
    for v in range(64):
        row = r["opt"][v]
        assert (row["n_train"] == 31).all()
        assert list(row["n_test"]) == [1 - ((v >> b) & 1) for b in range(6)]


def test_table2_counts():
    cfg = gen.make_config("C2")
    ds, sc = cfg.dataset, cfg.scenarios
    assert sc.n_splits == 240
    r = oracle.evaluate(ds, sc, 0, 240)
    ftz, rsq = ds.opt_names.index("FTZ"), ds.opt_names.index("RSQRT")
    for s in range(240):
        e = str(int(sc.experiment[s]))
        n, t = GOLD["table2_counts"]["per_experiment"][e]
        om = int(sc.split_opt_masks[s])
        for o in range(ds.n_opt_ids):
            row = r["opt"][s, o]
            if (om >> o) & 1:
                assert (row["n_train"], row["n_test"]) == (n, t), (s, e, o)
            else:
                assert row["n_train"] == 0 and row["n_test"] == 0
        if e in ("5", "6"):
            assert om == (1 << ftz) | (1 << rsq)


# ------------------------------------------------------------------ scaling
def test_scale_invariants():
    rng = np.random.default_rng(2)
    X = rng.uniform(0, 1, size=(20, 6))
    X[:, 3] = 0.25                                       # constant feature -> dropped
    Xt = rng.uniform(-0.5, 1.5, size=(7, 6))
    Xs, Xts, act = oracle.scale(X, Xt)
    assert list(act) == [0, 1, 2, 4, 5]
    assert (Xs.min(0) == 0).all() and (Xs.max(0) == 1).all()   # exact in IEEE
    # power-of-two rescaling of a raw feature is exact -> identical scaled values
    X2, Xt2 = X.copy(), Xt.copy()
    X2[:, 1] *= 8.0
    Xt2[:, 1] *= 8.0
    Xs2, Xts2, _ = oracle.scale(X2, Xt2)
    np.testing.assert_array_equal(Xs2, Xs)
    np.testing.assert_array_equal(Xts2, Xts)
    # permuting features permutes the scaled columns
    perm = [5, 2, 0, 4, 1, 3]
    Xs3, Xts3, act3 = oracle.scale(X[:, perm], Xt[:, perm])
    for j, a in enumerate(act3):
        k = list(act).index(perm[a])
        np.testing.assert_array_equal(Xs3[:, j], Xs[:, k])


# --------------------------------------------------------------- ridge fit
def _exact_ridge(Xs, y, Xts, lam):
    """Exact rational ridge with unpenalized intercept, UNcentred augmented
    normal equations (a different route than the oracle's centred one):
    ([1 X]^T [1 X] + diag(0, lam..lam)) beta = [1 X]^T y."""
    n, d = Xs.shape
    A = [[Fraction(1)] + [Fraction(float(v)) for v in row] for row in Xs]
    Y = [Fraction(float(v)) for v in y]
    L = Fraction(lam)
    p = d + 1
    M = [[sum(A[i][a] * A[i][b] for i in range(n)) + (L if (a == b and a > 0) else 0)
          for b in range(p)] + [sum(A[i][a] * Y[i] for i in range(n))] for a in range(p)]
    for c in range(p):                                   # Gauss-Jordan, exact
        piv = next(r for r in range(c, p) if M[r][c] != 0)
        M[c], M[piv] = M[piv], M[c]
        for r in range(p):
            if r != c and M[r][c] != 0:
                f = M[r][c] / M[c][c]
                M[r] = [M[r][k] - f * M[c][k] for k in range(p + 1)]
    beta = [M[a][p] / M[a][a] for a in range(p)]
    return [beta[0] + sum(beta[1 + a] * Fraction(float(v)) for a, v in enumerate(row)) for row in Xts]


@pytest.mark.parametrize("n,d", [(8, 3), (5, 3), (3, 3), (2, 2), (6, 1), (4, 3)])
def test_fit_exact_rational_bruteforce(n, d):
    rng = np.random.default_rng(100 + 10 * n + d)
    for lam in (1e-8, 0.5):
        X = rng.uniform(0, 1, size=(n, d))
        Xs, Xts, _ = oracle.scale(X, rng.uniform(-0.2, 1.2, size=(4, d)))
        y = rng.uniform(0.6, 1.4, size=n)
        ex, _ = oracle.fit_predict(Xs, y, Xts, ridge=lam)
        exact = _exact_ridge(Xs, y, Xts, lam)
        for e, q in zip(ex, exact):
            assert abs(Fraction(float(e)) - q) <= abs(q) * Fraction(1, 2**52) + Fraction(1, 10**30)


def test_fit_planted_linear_model_recovered():
    # Overdetermined, lambda = 0: coefficients of y = c0 + c.x' recovered.
    rng = np.random.default_rng(3)
    Xs = rng.uniform(0, 1, size=(40, 5))
    c0, c = 1.1, np.array([0.3, -0.2, 0.05, 0.0, 0.4])
    y = c0 + Xs @ c
    Xts = rng.uniform(0, 1, size=(10, 5))
    ex, coef = oracle.fit_predict(Xs, y, Xts, ridge=0.0)
    np.testing.assert_allclose(coef, np.r_[c0, c], rtol=0, atol=1e-13)
    np.testing.assert_allclose(ex, c0 + Xts @ c, rtol=0, atol=1e-13)
    # lambda = 1e-8: within the ridge-bias bound lambda*|w|/sigma_min^2
    ex2, _ = oracle.fit_predict(Xs, y, Xts, ridge=1e-8)
    Xc = Xs - Xs.mean(0)
    smin2 = np.linalg.svd(Xc, compute_uv=False)[-1] ** 2
    bound = 1e-8 * np.linalg.norm(c) / smin2 * np.abs(Xts - Xs.mean(0)).sum(1).max() * 2
    assert np.max(np.abs(ex2 - (c0 + Xts @ c))) <= bound


def test_fit_lstsq_special_case():
    # lambda -> 0 on a well-conditioned overdetermined fit = ordinary least squares.
    rng = np.random.default_rng(4)
    Xs = rng.uniform(0, 1, size=(60, 8))
    y = rng.uniform(0.5, 1.5, size=60)
    Xts = rng.uniform(0, 1, size=(9, 8))
    ex, _ = oracle.fit_predict(Xs, y, Xts, ridge=0.0)
    A = np.c_[np.ones(60), Xs]
    beta = np.linalg.lstsq(A, y, rcond=None)[0]
    np.testing.assert_allclose(ex, np.c_[np.ones(9), Xts] @ beta, rtol=1e-12, atol=1e-12)


def test_fit_label_shift_and_constant_labels():
    rng = np.random.default_rng(5)
    for n, d in ((31, 32), (16, 64), (63, 20)):          # under- and overdetermined
        Xs, Xts, _ = oracle.scale(rng.uniform(0, 1, (n, d)), rng.uniform(0, 1, (7, d)))
        y = rng.uniform(0.6, 1.4, n)
        ex, _ = oracle.fit_predict(Xs, y, Xts)
        ex2, _ = oracle.fit_predict(Xs, y + 0.5, Xts)     # S:246 label shift
        np.testing.assert_allclose(ex2, ex + 0.5, rtol=0, atol=1e-12)
        exc, _ = oracle.fit_predict(Xs, np.full(n, 1.23), Xts)
        np.testing.assert_array_equal(exc, 1.23)


def test_fit_degenerate_cases():
    y1 = np.array([1.37])
    ex, _ = oracle.fit_predict(np.zeros((1, 0)), y1, np.zeros((3, 0)))
    np.testing.assert_array_equal(ex, 1.37)             # n = 1 -> EX = y_1
    y = np.array([0.9, 1.2, 1.5])
    ex, _ = oracle.fit_predict(np.zeros((3, 0)), y, np.zeros((2, 0)))
    assert np.all(np.abs(ex - 1.2) <= 2.3e-16)           # d_eff = 0 -> EX = ybar


def test_fit_feature_permutation_invariance():
    rng = np.random.default_rng(6)
    for n, d in ((16, 64), (40, 8)):
        Xs, Xts, _ = oracle.scale(rng.uniform(0, 1, (n, d)), rng.uniform(0, 1, (9, d)))
        y = rng.uniform(0.6, 1.4, n)
        perm = rng.permutation(d)
        ex, _ = oracle.fit_predict(Xs, y, Xts)
        exp_, _ = oracle.fit_predict(Xs[:, perm], y, Xts[:, perm])
        np.testing.assert_allclose(exp_, ex, rtol=1e-15, atol=1e-15)


def test_fit_dual_identity_training_residual():
    # Underdetermined ridge: training residual y_c - Xc w = lambda * alpha with
    # alpha = (Xc Xc^T + lambda I)^-1 y_c (exact algebra).  Predicting the
    # training rows themselves gives EX_i = y_i - lambda*alpha_i.
    rng = np.random.default_rng(7)
    n, d = 6, 12
    Xs, _, _ = oracle.scale(rng.uniform(0, 1, (n, d)), np.zeros((0, d)))
    y = rng.uniform(0.6, 1.4, n)
    lam = 1e-3
    ex, _ = oracle.fit_predict(Xs, y, Xs, ridge=lam)
    F = lambda v: Fraction(float(v))
    Xc = [[F(Xs[i, a]) - sum(F(Xs[k, a]) for k in range(n)) / n for a in range(d)] for i in range(n)]
    yc = [F(y[i]) - sum(F(v) for v in y) / n for i in range(n)]
    K = [[sum(Xc[i][a] * Xc[j][a] for a in range(d)) + (Fraction(lam) if i == j else 0) for j in range(n)]
         for i in range(n)]
    M = [K[i] + [yc[i]] for i in range(n)]
    for c in range(n):
        for r in range(n):
            if r != c:
                f = M[r][c] / M[c][c]
                M[r] = [M[r][k] - f * M[c][k] for k in range(n + 1)]
    alpha = [M[i][n] / M[i][i] for i in range(n)]
    for i in range(n):
        q = F(y[i]) - Fraction(lam) * alpha[i]
        assert abs(Fraction(float(ex[i])) - q) <= abs(q) * Fraction(1, 2**52)


# ------------------------------------------------------------------- Tier 3
def test_rank_worked_examples():
    for case in GOLD["rank_and_filter"]["cases"]:
        names = list(case["pred"])
        ex = [case["pred"][k] for k in names]
        ids = [case["ids"][k] for k in names]
        _, rec = oracle.rank(ex, ids, case["threshold"], case["max_count"])
        inv = {v: k for k, v in case["ids"].items()}
        assert [inv[i] for i in rec] == case["expect"]


def test_rank_properties():
    rng = np.random.default_rng(8)
    for _ in range(2000):
        k = int(rng.integers(1, 10))
        ex = rng.choice([0.8, 1.0, 1.05, 1.2, 2.0], size=k) if rng.random() < 0.3 else rng.uniform(0.5, 1.6, k)
        ids = rng.permutation(16)[:k]
        th = float(rng.uniform(0.9, 1.3))
        mc = int(rng.integers(1, 6))
        order, rec = oracle.rank(ex, ids, th, mc)
        pos = {i: j for j, i in enumerate(ids)}
        vals = [ex[pos[i]] for i in order]
        assert all(vals[j] > vals[j + 1] or (vals[j] == vals[j + 1] and order[j] < order[j + 1])
                   for j in range(k - 1))                                       # ordering soundness
        assert len(rec) <= mc and all(ex[pos[i]] >= th for i in rec)
        _, rec_hi = oracle.rank(ex, ids, th + 0.1, mc)                          # threshold monotonicity
        assert rec_hi == rec[:len(rec_hi)]
        order2, _ = oracle.rank(np.exp(3 * ex) - 7, ids, -1e300, 100)           # monotone invariance
        assert order2 == order


def test_sign_accuracy_worked_example():
    g = GOLD["sign_accuracy"]
    correct = sum(oracle.sign_correct(e, a) for e, a in zip(g["ex"], g["ac"]))
    assert correct == g["expect_correct"]
    assert oracle.sign_correct(1.0, 1.0) and oracle.sign_correct(1.0, 0.5) and not oracle.sign_correct(1.0, 1.1)


# -------------------------------------------------------- end-to-end plants
def _plant_dataset(seed, C=4, y_of=None):
    """One program, one input, one run; labels planted per optimization."""
    rng = np.random.default_rng(seed)
    V = 64
    counters = np.rint(rng.uniform(1e3, 1e6, size=(V, C)))
    cycles = np.rint(rng.uniform(1e6, 2e6, size=V))
    x = counters / cycles[:, None]
    return counters, cycles, x


def test_pipeline_planted_linear_speedup():
    # rt(v | 2^b) = rt(v) / f(x(v)) for bit-clear v, f linear in raw rates
    # (hence in min-max scaled ones): with LOO (n = 31 > d_eff + 1 = 5) the
    # prediction of the held-out case recovers f within the ridge bias, so
    # every sign is right and every AC/EX ratio is 1 within 1e-6.
    counters, cycles, x = _plant_dataset(9)
    b = 2
    rng = np.random.default_rng(10)
    rt = rng.uniform(5, 10, size=64)
    coef = np.array([0.4, -0.3, 0.2, 0.1])
    for v in range(64):
        if not (v >> b) & 1:
            f = 0.7 + x[v] @ coef * 3.0
            rt[v | (1 << b)] = rt[v] / f
    ob = np.array([[0, 1, 2, 3, 4, 5]], dtype=np.int8)
    ds = Dataset(1, 1, 1, 6, 4, 6, counters, cycles, rt, ob, [f"O{j}" for j in range(6)], ["P0"])
    sc = gen.configs.Scenarios(kind="loo", n_splits=64, group_words=1,
                               pool_groups=np.array([1], dtype=np.uint64), opt_mask=1 << b)
    r = oracle.evaluate(ds, sc, 0, 64, want_ex=True)
    rows = r["opt"][:, b]
    sel = rows["n_test"] > 0
    assert sel.sum() == 32
    assert (rows["n_correct"][sel] == 1).all()
    np.testing.assert_allclose(rows["sum_ratio"][sel], 1.0, rtol=0, atol=1e-6)


def test_pipeline_recommendation_rule():
    # SPEC acceptance #7 analogue: optimization 0 halves the runtime (AC = 2
    # exactly), optimization 1 slows it (AC = 0.8).  Constant labels give
    # EX = AC exactly, so every test version lacking bit 0 gets exactly one
    # recommendation, [0], and it is a hit; versions with bit 0 get none.
    counters, cycles, _ = _plant_dataset(11)
    v = np.arange(64)
    rt = 8.0 * np.where(v & 1, 0.5, 1.0) * np.where(v & 2, 1.25, 1.0)
    ob = np.array([[0, 1, 2, 3, 4, 5]], dtype=np.int8)
    ds = Dataset(1, 1, 1, 6, 4, 6, counters, cycles, rt, ob, [f"O{j}" for j in range(6)], ["P0"])
    sc = gen.configs.Scenarios(kind="loo", n_splits=64, group_words=1,
                               pool_groups=np.array([1], dtype=np.uint64), opt_mask=0b11)
    r = oracle.evaluate(ds, sc, 0, 64, want_recs=True)
    for s in range(64):
        recs = r["recs"][s, s]
        if s & 1:
            assert list(recs) == [-1, -1, -1]
        else:
            assert list(recs) == [0, -1, -1]
    assert r["scn"]["n_rec"].sum() == 32 and r["scn"]["n_rec_hit"].sum() == 32
    assert (r["opt"][:, 0]["n_correct"] == r["opt"][:, 0]["n_test"]).all()


def test_mask_aggregation_ranking_rule():
    # O8: per-mask sums over folds; rank by (sum correct desc, mask id asc).
    n_masks, folds, O = 5, 3, 2
    opt = np.zeros((n_masks * folds, O), dtype=oracle.OPT_SCORE_DTYPE)
    scn = np.zeros(n_masks * folds, dtype=oracle.SCN_SCORE_DTYPE)
    correct = {0: 4, 1: 7, 2: 7, 3: 1, 4: 9}
    for m, c in correct.items():
        for f in range(folds):
            opt[m * folds + f, 0]["n_correct"] = c if f == 0 else 0
            opt[m * folds + f, :]["n_test"] = 2
            scn[m * folds + f]["n_rec"] = 1
    rows, top = oracle.aggregate_masks(opt, scn, folds, first_mask=10, top_k=3)
    assert list(rows["n_correct"]) == [4, 7, 7, 1, 9]
    assert (rows["n_test"] == 12).all() and (rows["n_rec"] == 3).all()
    assert list(top) == [14, 11, 12]


# ------------------------------------------------------------ IBK (NEXT-1)
def _knn_brute(Xs, y, Xts, k):
    """Independent brute force: exact rational distances, stable
    sort by (distance, stored index), arithmetic mean of the k labels."""
    out = []
    for q in Xts:
        D = [sum((Fraction(float(a)) - Fraction(float(b))) ** 2 for a, b in zip(q, row)) for row in Xs]
        order = sorted(range(len(Xs)), key=lambda i: (D[i], i))[:min(k, len(Xs))]
        out.append(float(sum(Fraction(float(y[i])) for i in order) / len(order)))
    return np.array(out)


def test_knn_spec_examples():
    rng = np.random.default_rng(20)
    X = rng.uniform(0, 1, (12, 5))
    y = rng.uniform(0.5, 1.5, 12)
    np.testing.assert_array_equal(oracle.knn_predict(X, y, X, k=1), y)           # S:210 identity, k=1
    ex = oracle.knn_predict(X, y, rng.uniform(0, 1, (4, 5)), k=50)                # S:211 k >= n
    np.testing.assert_allclose(ex, y.mean(), rtol=0, atol=1e-15)


def test_knn_matches_bruteforce():
    rng = np.random.default_rng(21)
    for trial in range(120):
        n, d = int(rng.integers(1, 51)), int(rng.integers(1, 9))
        X = rng.uniform(0, 1, (n, d))
        if trial % 4 == 0:
            X[rng.integers(0, n, n // 2)] = X[0]                                   # duplicates -> ties
        y = rng.uniform(0.5, 1.5, n)
        Xt = rng.uniform(-0.2, 1.2, (3, d))
        for k in (1, 3, 10):
            np.testing.assert_allclose(oracle.knn_predict(X, y, Xt, k=k), _knn_brute(X, y, Xt, k),
                                       rtol=0, atol=1e-9)


def test_knn_permutation_and_shift_invariance():
    rng = np.random.default_rng(22)
    X = rng.uniform(0, 1, (30, 6))
    y = rng.uniform(0.5, 1.5, 30)
    Xt = rng.uniform(0, 1, (10, 6))
    ex = oracle.knn_predict(X, y, Xt, k=10)
    perm = rng.permutation(30)
    np.testing.assert_allclose(oracle.knn_predict(X[perm], y[perm], Xt, k=10), ex, rtol=0, atol=1e-15)
    np.testing.assert_allclose(oracle.knn_predict(X, y + 0.25, Xt, k=10), ex + 0.25, rtol=0, atol=1e-14)


def test_knn_pipeline_exact_recall_exp1():
    # SPEC acceptance #5 analogue ("IBK ... is therefore able to predict
    # the speedup of the training data exactly"): Exp 1 tests the training run
    # itself; with k = 1 every test case of the training group is its own
    # nearest neighbour (distance 0), so EX == AC exactly there.
    cfg = gen.make_config("C2")
    sc = cfg.scenarios
    r = oracle.evaluate(cfg.dataset, sc, 0, 24, want_ex=True, learner=1, k_nn=1)
    ds = cfg.dataset
    O, G = ds.n_opt_ids, ds.n_groups
    V = 64
    for s in range(24):                                   # Exp 1 instantiations
        g_train = int(np.log2(int(sc.train_groups[s][0])))
        p = g_train // (ds.n_inputs * ds.n_runs)
        for o in range(O):
            b = int(ds.opt_bit[p, o])
            if b < 0:
                continue
            for k in range(32):
                v = ((k >> b) << (b + 1)) | (k & ((1 << b) - 1))
                ac = ds.runtime_ms[g_train * V + v] / ds.runtime_ms[g_train * V + (v | (1 << b))]
                assert r["ex"][s, o, g_train * 32 + k] == ac


# ---------------------------------------------- clamp rule (reading R7)
def test_pipeline_clamp_rule():
    # gen.plants.clamp_plant: split 0 holds out version 0, whose feature lies
    # outside the training range of a planted line AC = 2.1 - x; the ridge
    # extrapolates to 2.1 - 3 = -0.9 (ridge bias ~1e-8), so S:327 applies:
    # EX := 0.01, the case is flagged, and the ratio and the sign decision use
    # the clamped value (AC / 0.01; 0.01 <= 1 while AC = 1.5 > 1: incorrect).
    from gen.plants import clamp_plant
    cfg = clamp_plant(x_held=3.0, ac_held=1.5)
    r = oracle.evaluate(cfg.dataset, cfg.scenarios, 0, 1, want_ex=True, want_recs=True)
    row = r["opt"][0, 0]
    assert (row["n_train"], row["n_test"]) == (31, 1)
    assert row["n_clamped"] == 1 and row["n_correct"] == 0
    assert r["ex"][0, 0, 0] == 0.01                        # the stored EX is the floor itself
    assert row["sum_ratio"] == row["min_ratio"] == row["max_ratio"] == 1.5 / 0.01
    assert r["scn"][0]["n_rec"] == 0                        # 0.01 < 1.05: not recommended
    # the same fit without the clamp rule: the unclamped prediction is the line
    Xs, Xts, _ = oracle.scale(oracle.rates(cfg.dataset.counters, cfg.dataset.cycles)[2::2],
                              oracle.rates(cfg.dataset.counters, cfg.dataset.cycles)[0:1])
    y = cfg.dataset.runtime_ms[2::2] / cfg.dataset.runtime_ms[3::2]
    ex, _ = oracle.fit_predict(Xs, y, Xts)
    assert abs(ex[0] - (2.1 - 3.0)) < 1e-6


def test_pipeline_clamp_keeps_positive_predictions():
    # the other side of the rule: EX ~ 2.1 - 2.05 = 0.05 > 0 is kept as is
    from gen.plants import clamp_plant
    cfg = clamp_plant(x_held=2.05, ac_held=0.7)
    r = oracle.evaluate(cfg.dataset, cfg.scenarios, 0, 1, want_ex=True)
    row = r["opt"][0, 0]
    assert row["n_clamped"] == 0
    assert abs(r["ex"][0, 0, 0] - 0.05) < 1e-6
    assert abs(row["sum_ratio"] - 0.7 / 0.05) < 1e-3
    assert row["n_correct"] == 1                            # 0.05 <= 1 and 0.7 <= 1


# --------------------------- perfect / constant predictor
def _brute_test_ac(ds, sc, s, o):
    """Independent brute force: the AC of every test case of (scenario s, o),
    for LOO / GROUPS splits (membership written out from the definitions)."""
    V = 1 << ds.n_opt_bits
    out = []
    for g in range(ds.n_groups):
        p = g // (ds.n_inputs * ds.n_runs)
        b = int(ds.opt_bit[p, o])
        if b < 0:
            continue
        for v in range(V):
            if (v >> b) & 1:
                continue
            t = g * V + v
            if sc.kind == "loo":
                test = t == s
            else:
                test = (int(sc.test_groups[s][g // 64]) >> (g % 64)) & 1
            if test:
                out.append(ds.runtime_ms[t] / ds.runtime_ms[t | (1 << b)])
    return out


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_pipeline_perfect_predictor_identity(name):
    # S:383 / S:407: a predictor with EX = AC scores 100 % and every AC/EX is 1.
    # (a) the ridge learner itself on gen.plants.pow2_lattice: every pair of an
    #     optimization has the same (power-of-two) label, a fit on constant
    #     labels predicts that label exactly (O4(4)), so EX = AC exactly;
    # (b) the test-only stub learner EX := AC on the unmodified config.
    from gen.plants import pow2_lattice
    for cfg, learner in ((pow2_lattice(name), 0), (gen.make_config(name), oracle.LEARNER_PERFECT_STUB)):
        n = cfg.scenarios.n_scenarios
        r = oracle.evaluate(cfg.dataset, cfg.scenarios, 0, n, want_ex=True, learner=learner)
        o, sc = r["opt"], r["scn"]
        live = o["n_test"] > 0
        assert live.sum() > 0
        assert (o["n_correct"] == o["n_test"]).all()
        assert (o["n_clamped"] == 0).all()
        assert (o["sum_ratio"][live] == o["n_test"][live]).all()
        assert (o["min_ratio"][live] == 1.0).all() and (o["max_ratio"][live] == 1.0).all()
        assert (sc["n_rec_hit"] == sc["n_rec"]).all() and sc["n_rec"].sum() > 0


def test_pipeline_constant_predictor_stub():
    # with EX := 1 every ratio AC/EX equals AC; EX = 1 is "no gain"
    # (R11), so exactly the cases with AC <= 1 are correct; 1 < 1.05:
    # no recommendation; EX = 1 lies on the sign boundary, so every test case
    # is a guard case (R21).
    from fractions import Fraction
    for name in ("C1", "C2"):
        cfg = gen.make_config(name)
        ds, scd = cfg.dataset, cfg.scenarios
        n = min(scd.n_scenarios, 60)
        r = oracle.evaluate(ds, scd, 0, n, learner=oracle.LEARNER_CONSTANT_STUB)
        for s in range(n):
            om = int(scd.split_opt_masks[s]) if scd.split_opt_masks is not None else 0xFFFFFFFF
            for o in range(ds.n_opt_ids):
                row = r["opt"][s, o]
                if not (om >> o) & 1 or row["n_test"] == 0:
                    continue
                ac = _brute_test_ac(ds, scd, s, o)
                assert len(ac) == row["n_test"]
                assert row["n_correct"] == sum(a <= 1.0 for a in ac)
                assert row["min_ratio"] == min(ac) and row["max_ratio"] == max(ac)
                exact = sum(Fraction(a) for a in ac)
                assert abs(Fraction(float(row["sum_ratio"])) - exact) <= exact * Fraction(1, 2**52)
        assert (r["scn"]["n_rec"][:n] == 0).all()
        assert (r["scn"]["n_guard"][:n] >= r["opt"]["n_test"][:n].sum(1)).all()


# ------------------------------------------------------------- kappa^ (O4)
def test_kappa_closed_form_and_bound():
    # Orthogonal centred columns: G = diag(|x_a - xbar_a|^2) + lambda I, so the
    # Cholesky pivots are the diagonal and kappa^ = max/min of it exactly.
    Xs = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 3.0], [1.0, 3.0]])
    y = np.array([1.0, 1.2, 0.9, 1.4])
    lam = 1e-8
    for prec in ("quad", "ld"):
        _, _, kap = oracle.fit_predict(Xs, y, Xs, ridge=lam, precision=prec, want_kappa=True)
        assert abs(kap - (9.0 + lam) / (1.0 + lam)) <= 1e-14 * kap
    # general case: 1 <= kappa^ <= cond_2(G) (pivots lie inside the spectrum)
    rng = np.random.default_rng(30)
    for n, d in ((40, 6), (10, 20), (200, 70)):
        Xs = rng.uniform(0, 1, (n, d))
        _, _, kap = oracle.fit_predict(Xs, rng.uniform(0.6, 1.4, n), Xs[:2], want_kappa=True)
        Xc = Xs - Xs.mean(0)
        ev = np.linalg.eigvalsh(Xc.T @ Xc + 1e-8 * np.eye(d))
        assert 1.0 <= kap <= ev[-1] / ev[0] * (1 + 1e-6)


# ---------------------------- long-double fits (SURVEY 8(c) precision policy)
@pytest.mark.parametrize("n,d", [(8, 3), (5, 3), (6, 1)])
def test_fit_ld_exact_rational_bruteforce(n, d):
    rng = np.random.default_rng(200 + 10 * n + d)
    X = rng.uniform(0, 1, size=(n, d))
    Xs, Xts, _ = oracle.scale(X, rng.uniform(-0.2, 1.2, size=(4, d)))
    y = rng.uniform(0.6, 1.4, size=n)
    ex, _ = oracle.fit_predict(Xs, y, Xts, ridge=1e-8, precision="ld")
    exact = _exact_ridge(Xs, y, Xts, 1e-8)
    for e, q in zip(ex, exact):
        assert abs(Fraction(float(e)) - q) <= abs(q) * Fraction(1, 2**50)


def test_fit_ld_planted_model_at_c4_width():
    # p > 65 overdetermined (the only regime the policy sends to long double):
    # a planted y = c0 + Xs c with lambda = 0 is recovered, and with lambda =
    # 1e-8 the long-double and quad predictions agree far inside the 1e-9 bar.
    rng = np.random.default_rng(31)
    n, d = 1024, 128
    Xs = rng.uniform(0, 1, size=(n, d))
    c = rng.normal(0, 0.1, size=d)
    y = 1.0 + Xs @ c
    Xts = rng.uniform(0, 1, size=(16, d))
    ex, coef = oracle.fit_predict(Xs, y, Xts, ridge=0.0, precision="ld")
    np.testing.assert_allclose(coef, np.r_[1.0, c], rtol=0, atol=1e-11)
    yn = y + rng.normal(0, 0.01, size=n)
    exl, _, kl = oracle.fit_predict(Xs, yn, Xts, precision="ld", want_kappa=True)
    exq, _, kq = oracle.fit_predict(Xs, yn, Xts, precision="quad", want_kappa=True)
    np.testing.assert_allclose(exl, exq, rtol=1e-14, atol=0)
    assert abs(kl - kq) <= 1e-10 * kq


def test_precision_policy_by_regime():
    # C3 fits (p <= 65 / underdetermined) stay in quad; C4 fits (n ~ 8192, p =
    # 129, kappa^ ~ 1e3-1e4) run in long double with kappa^ * 2^-64 < 1e-12.
    c3 = gen.make_config("C3", n_splits=4)
    r = oracle.evaluate(c3.dataset, c3.scenarios, 0, 4, want_kappa=True)
    assert (r["fit_ld"] == 0).all() and np.isfinite(r["kappa"]).all()
    c4 = gen.make_config("C4", n_splits=1, n_programs=128)
    r = oracle.evaluate(c4.dataset, c4.scenarios, 0, 1, want_kappa=True)
    assert (r["fit_ld"] == 1).all()
    assert (r["kappa"] * 2.0 ** -64 < 1e-12).all() and (r["kappa"] >= 1).all()
