"""Shared comparison of CUDA-path outputs against oracle outputs.

Bar, the north star's: integer fields bit-exact, FP64 fields
(EX, Σ AC/EX, min, max) within 1e-9 RELATIVE error, |a - b| <= 1e-9 |b|.

Guard cases (reading R21): a decision whose deciding value lies within 1e-9
of its boundary.  Both sides count them by the same rule and `n_guard` must
agree exactly.  Only the decision-dependent fields of a guarded scenario are
exempt (n_correct, n_clamped, the recommendation fields); EX is continuous and
is compared everywhere -- except a test case one side clamped (EX := 0.01,
S:327) while the other did not, which needs the oracle's EX within the guard
band of 0.  Ratio fields are compared wherever the clamp decisions agree.
"""
import numpy as np

TOL = 1e-9
ALWAYS_EXACT = ("n_train", "n_test", "fp_train", "fp_test")
DECISION_EXACT = ("n_correct", "n_clamped")
CLAMP_FLOOR = 0.01


def rel_err(a, b):
    """|a - b| / |b| elementwise (0 where both are 0, inf where only b is 0)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.abs(a - b)
    with np.errstate(divide="ignore", invalid="ignore"):
        e = d / np.abs(b)
    return np.where(b == 0.0, np.where(d == 0.0, 0.0, np.inf), e)


def compare(got, ref, tol=TOL, max_guard_frac=0.0, exact_guard=True):
    """Returns a dict of statistics; raises AssertionError on a parity failure.
    exact_guard: n_guard must agree exactly (always for the LS / IBK learners)."""
    go, ro = got["opt"], ref["opt"]
    gs, rs = got["scn"], ref["scn"]
    assert go.shape == ro.shape and gs.shape == rs.shape
    for f in ALWAYS_EXACT:
        bad = np.argwhere(go[f] != ro[f])
        assert bad.size == 0, f"{f} differs at {bad[:5].tolist()}"
    assert (gs["n_guard"] < 1000000).all(), "GPU factorisation failure (non-positive pivot)"
    if exact_guard:
        bad = np.argwhere(gs["n_guard"] != rs["n_guard"])
        assert bad.size == 0, (f"n_guard differs at {bad[:5].ravel().tolist()}: "
                               f"{gs['n_guard'][bad[:5].ravel()]} vs {rs['n_guard'][bad[:5].ravel()]}")
    guarded = (rs["n_guard"] != 0) | (gs["n_guard"] != 0)
    ok = ~guarded
    for f in DECISION_EXACT:
        bad = np.argwhere((go[f] != ro[f]) & ok[:, None])
        assert bad.size == 0, f"{f} differs at {bad[:5].tolist()}: {go[f][tuple(bad[0])]} vs {ro[f][tuple(bad[0])]}"
    for f in ("n_rec", "n_rec_hit", "n_untrained"):
        bad = np.argwhere((gs[f] != rs[f]) & ok)
        assert bad.size == 0, f"{f} differs at {bad[:5].tolist()}"
    # n_untrained is no decision (n == 0 is integer): exact everywhere
    assert np.array_equal(gs["n_untrained"], rs["n_untrained"]), "n_untrained differs"
    worst = 0.0
    same_clamp = go["n_clamped"] == ro["n_clamped"]
    for f in ("sum_ratio", "min_ratio", "max_ratio"):
        e = rel_err(go[f], ro[f])[same_clamp]
        if e.size:
            worst = max(worst, float(e.max()))
            assert e.max() <= tol, f"{f} rel err {e.max():.3e}"
    if got.get("ex") is not None and ref.get("ex") is not None:
        ge, re_ = np.asarray(got["ex"]), np.asarray(ref["ex"])
        e = rel_err(ge, re_)
        one_clamped = ((ge == CLAMP_FLOOR) ^ (re_ == CLAMP_FLOOR)) & (np.minimum(np.abs(ge), np.abs(re_)) <= tol)
        e = np.where(one_clamped, 0.0, e)
        if e.size:
            worst = max(worst, float(e.max()))
            assert e.max() <= tol, f"EX rel err {e.max():.3e} at {np.unravel_index(e.argmax(), e.shape)}"
        if one_clamped.any():   # only where the scenario is a guard case
            sc = np.unique(np.argwhere(one_clamped)[:, 0])
            assert guarded[sc].all(), f"clamp decision differs outside a guard case: scenarios {sc[:5]}"
    if got.get("recs") is not None and ref.get("recs") is not None:
        bad = np.argwhere((got["recs"] != ref["recs"]).any(axis=(1, 2)) & ok)
        assert bad.size == 0, f"recommendations differ in scenarios {bad[:5].ravel().tolist()}"
    assert guarded.mean() <= max_guard_frac, f"{guarded.sum()} guarded scenarios"
    return dict(n=len(gs), guarded=int(guarded.sum()), worst_rel=worst)
