"""GPU parity of the NEXT-1 learner (IBk, reading R22) vs the oracle.

IBk's EX is the mean of k training labels picked by distances computed with
the same operations in the same order on both sides (oracle or_knn_predict,
kernel knn_ex), so the bar is BIT-EXACT: every EX, every integer field and
every recommendation identical, no guard exemption.  Only the FP64 ratio
sums (a quad sum in the oracle, a warp tree on the GPU) keep the 1e-9
relative bar.
"""
import numpy as np
import pytest

import gen
import oracle
from tests.parity import compare

pytestmark = pytest.mark.gpu


def _run(cfg, first, count, k=10):
    from paper_1910_07776_b200 import Context, default_params
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    got = ctx.evaluate(first, count, params=default_params(learner=1, k_nn=k), want_ex=True, want_recs=True)
    ctx.close()
    ref = oracle.evaluate(cfg.dataset, cfg.scenarios, first, count, want_ex=True, want_recs=True,
                          learner=1, k_nn=k)
    return got, ref


def _exact(got, ref):
    assert np.array_equal(got["ex"], ref["ex"], equal_nan=True), "IBK EX not bit-exact"
    go, ro, gs, rs = got["opt"], ref["opt"], got["scn"], ref["scn"]
    for f in ("n_train", "n_test", "n_correct", "n_clamped", "fp_train", "fp_test", "min_ratio", "max_ratio"):
        assert np.array_equal(go[f], ro[f]), f
    for f in ("n_rec", "n_rec_hit", "n_untrained", "n_guard"):
        assert np.array_equal(gs[f], rs[f]), f
    assert np.array_equal(got["recs"], ref["recs"])
    return compare(got, ref, max_guard_frac=1.0)


@pytest.mark.parametrize("k", [1, 3, 10, 16])
def test_ibk_c1_all_k(k):
    cfg = gen.make_config("C1")
    got, ref = _run(cfg, 0, 64, k)
    print("IBK C1 k", k, _exact(got, ref))


def test_ibk_c2_table2():
    cfg = gen.make_config("C2")
    got, ref = _run(cfg, 0, 240)
    print("IBK C2", _exact(got, ref))


def test_ibk_c3_ragged():
    cfg = gen.make_config("C3", n_splits=2001)
    got, ref = _run(cfg, 0, 2001)
    print("IBK C3", _exact(got, ref))
    got, ref = _run(cfg, 999, 77)
    _exact(got, ref)


def test_ibk_c5_masks():
    cfg = gen.make_config("C5", n_masks_k=5)
    n = cfg.scenarios.n_scenarios
    got, ref = _run(cfg, 0, n)
    print("IBK C5k5", _exact(got, ref))


def test_ibk_degenerate():
    # constant / zero features (d_eff = 0: every distance 0 -> the first k
    # training pairs by index) and feature masks selecting nothing
    cfg = gen.make_config("C1")
    ds = cfg.dataset
    ds.counters[:, :8] = ds.cycles[:, None] * 0.25
    ds.counters[:, 8:16] = 0.0
    cfg.scenarios.feature_masks = np.array([[0, 0], [1 << 20, 0], [0xFFFF0000, 0], [~0 & 0xFFFFFFFF, 0]],
                                           dtype=np.uint64)
    cfg.scenarios.n_masks = 4
    got, ref = _run(cfg, 0, 64 * 4)
    _exact(got, ref)


def test_ibk_rejects_bad_k():
    from paper_1910_07776_b200 import Context, SpeedrecError, default_params
    for name, kw in (("C1", {}), ("C4", dict(n_splits=2, n_programs=96))):
        cfg = gen.make_config(name, **kw)
        ctx = Context(0)
        ctx.load(cfg.dataset)
        ctx.define_scenarios(cfg.scenarios)
        for k in (0, 17):
            with pytest.raises(SpeedrecError, match="k_nn"):
                ctx.evaluate(0, 1, params=default_params(learner=1, k_nn=k))
        ctx.close()


@pytest.mark.parametrize("k", [10, 3])
def test_ibk_large_batch_path(k):
    """IBK on the > 64-group path (k_ibk_prep / k_ibk_dist / k_ibk_score +
    k_rank_warp): 96 programs x 64 variants x 128 counters (n ~ 770 training
    rows, t ~ 1,540 test rows per fit, several 64-test x 32-row tiles and
    ragged tails), 20 splits and a ragged sub-range: bit-exact."""
    cfg = gen.make_config("C4", n_splits=20, n_programs=96)
    got, ref = _run(cfg, 0, 20, k=k)
    print("IBK C4 P=96 k", k, _exact(got, ref))
    got, ref = _run(cfg, 3, 5, k=k)
    _exact(got, ref)


def test_ibk_large_batch_feature_mask():
    """IBK on the large-batch path with a feature mask (d = 37 of 128, odd:
    the last 16-byte staging pair is zero-filled) and an inactive counter."""
    cfg = gen.make_config("C4", n_splits=6, n_programs=80)
    ds = cfg.dataset
    ds.counters[:, 5] = ds.cycles * 0.25                # inactive (constant rate)
    rng = np.random.default_rng(5)
    bits = sorted(rng.choice(128, size=36, replace=False).tolist()) + [5]
    m0 = sum(1 << b for b in bits if b < 64)
    m1 = sum(1 << (b - 64) for b in bits if b >= 64)
    sc = cfg.scenarios
    sc.feature_masks = np.array([[m0, m1]], dtype=np.uint64)
    sc.n_masks = 1
    got, ref = _run(cfg, 0, 6)
    print("IBK C4 masked", _exact(got, ref))


def test_ibk_large_batch_full_size_sampled():
    """IBK at the full C4 lattice (1024 programs, n ~ 8,192 training rows and
    t ~ 16,384 test rows per fit: 256 test tiles x 256 row tiles) in the
    bench's launch shape: a sampled scenario is bit-exact against the oracle."""
    from paper_1910_07776_b200 import Context, default_params
    cfg = gen.make_config("C4", n_splits=16)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    got = ctx.evaluate(0, 16, params=default_params(learner=1), want_ex=True, want_recs=True)
    ctx.close()
    s = 11
    ref = oracle.evaluate(cfg.dataset, cfg.scenarios, s, 1, want_ex=True, want_recs=True, learner=1, k_nn=10,
                          n_threads=16)
    one = {k: (v[s:s + 1] if v is not None else None) for k, v in got.items() if k in ("opt", "scn", "ex", "recs")}
    print("IBK C4 full, scenario", s, _exact(one, ref))
