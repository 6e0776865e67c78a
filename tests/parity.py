"""Shared comparison of CUDA-path outputs against oracle outputs.

Bar: integer fields bit-exact, FP64 fields within 1e-9
relative (|a-b| <= 1e-9 * max(1, |b|)); scenarios the oracle marks as guard
cases (a decision within 1e-9 of its boundary, reading R21) are exempt from
the decision-dependent fields and reported.
"""
import numpy as np

TOL = 1e-9
ALWAYS_EXACT = ("n_train", "n_test", "fp_train", "fp_test")
DECISION_EXACT = ("n_correct", "n_clamped")


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.maximum(1.0, np.abs(b))


def compare(got, ref, tol=TOL, max_guard_frac=1e-3):
    """Returns a dict of statistics; raises AssertionError on a parity failure."""
    go, ro = got["opt"], ref["opt"]
    gs, rs = got["scn"], ref["scn"]
    assert go.shape == ro.shape and gs.shape == rs.shape
    for f in ALWAYS_EXACT:
        bad = np.argwhere(go[f] != ro[f])
        assert bad.size == 0, f"{f} differs at {bad[:5].tolist()}"
    guarded = rs["n_guard"] != 0
    ok = ~guarded
    for f in DECISION_EXACT:
        bad = np.argwhere((go[f] != ro[f]) & ok[:, None])
        assert bad.size == 0, f"{f} differs at {bad[:5].tolist()}: {go[f][tuple(bad[0])]} vs {ro[f][tuple(bad[0])]}"
    for f in ("n_rec", "n_rec_hit", "n_untrained"):
        bad = np.argwhere((gs[f] != rs[f]) & ok)
        assert bad.size == 0, f"{f} differs at {bad[:5].tolist()}"
    worst = 0.0
    for f in ("sum_ratio", "min_ratio", "max_ratio"):
        e = rel_err(go[f], ro[f])[ok]
        if e.size:
            worst = max(worst, float(e.max()))
            assert e.max() <= tol, f"{f} rel err {e.max():.3e}"
    if got.get("ex") is not None and ref.get("ex") is not None:
        e = rel_err(got["ex"], ref["ex"])[ok]
        if e.size:
            worst = max(worst, float(e.max()))
            assert e.max() <= tol, f"EX rel err {e.max():.3e} at {np.unravel_index(e.argmax(), e.shape)}"
    if got.get("recs") is not None and ref.get("recs") is not None:
        bad = np.argwhere((got["recs"] != ref["recs"]).any(axis=(1, 2)) & ok)
        assert bad.size == 0, f"recommendations differ in scenarios {bad[:5].ravel().tolist()}"
    assert guarded.mean() <= max_guard_frac, f"{guarded.sum()} guarded scenarios"
    return dict(n=len(gs), guarded=int(guarded.sum()), worst_rel=worst)
