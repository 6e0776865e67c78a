"""GPU parity: the CUDA path through the C-ABI vs the oracle, element by element.

Sizes: the small configs completely (C1 64, C2 240 scenarios), C3/C5 at sizes
the oracle finishes in seconds that still span many warps/CTAs and a ragged
tail, and the FULL bench configuration (C3, 1e6 splits, the same launch as
bench.py) on sampled scenarios the oracle computes one by one.
"""
import numpy as np
import pytest

import gen
import oracle
from tests.parity import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Context():
    from paper_1910_07776_b200 import Context as C
    return C


def _run(Context, cfg, first, count, params=None, **kw):
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    from paper_1910_07776_b200 import default_params
    p = default_params(**(params or {}))
    got = ctx.evaluate(first, count, params=p, want_ex=True, want_recs=True)
    ctx.close()
    ref = oracle.evaluate(cfg.dataset, cfg.scenarios, first, count, want_ex=True, want_recs=True, **kw)
    return got, ref


def test_rates_bit_exact(Context):
    for name in ("C1", "C2", "C3"):
        cfg = gen.make_config(name, n_splits=8)
        ctx = Context(0)
        ctx.load(cfg.dataset)
        x = ctx.rates()
        ctx.close()
        assert np.array_equal(x, oracle.rates(cfg.dataset.counters, cfg.dataset.cycles))


def test_c1_all(Context):
    cfg = gen.make_config("C1")
    got, ref = _run(Context, cfg, 0, 64)
    st = compare(got, ref, max_guard_frac=0.05)
    print("C1", st)


def test_c2_all_table2(Context):
    cfg = gen.make_config("C2")
    got, ref = _run(Context, cfg, 0, 240)
    st = compare(got, ref, max_guard_frac=0.05)
    from tests.parity import rel_err
    e = rel_err(got["ex"], ref["ex"]).reshape(240, -1).max(axis=1)
    per_exp = {int(x): float(e[cfg.scenarios.experiment == x].max()) for x in range(1, 7)}
    print("C2", st, "worst EX rel err per experiment", per_exp)


def test_c3_small_ragged(Context):
    cfg = gen.make_config("C3", n_splits=3001)
    got, ref = _run(Context, cfg, 0, 3001)
    print("C3", compare(got, ref))
    got, ref = _run(Context, cfg, 1234, 77)         # ragged sub-range
    compare(got, ref)


def test_fused_ranking_opt_in(Context, monkeypatch):
    """SPEEDREC_FUSE_RANK=1: A6 run by the warp that finishes a scenario's
    last fit (cross-SM counter + fences) instead of k_rank_warp: same rows."""
    monkeypatch.setenv("SPEEDREC_FUSE_RANK", "1")
    cfg = gen.make_config("C3", n_splits=1500)
    got, ref = _run(Context, cfg, 0, 1500)
    compare(got, ref)
    cfg = gen.make_config("C2")
    got, ref = _run(Context, cfg, 0, 240)
    compare(got, ref, max_guard_frac=0.05)


def test_c5_small_masks(Context):
    cfg = gen.make_config("C5", n_masks_k=5)        # 32 masks x 128 folds
    n = cfg.scenarios.n_scenarios
    got, ref = _run(Context, cfg, 0, n)
    print("C5k5", compare(got, ref))


@pytest.mark.parametrize("mask_path", ["2", "1"])
def test_c5_prefix_shared_path_explicit_masks(Context, mask_path, monkeypatch):
    """The mask paths with masks spanning all 20 counters (prefix [0, 10) and
    suffix [10, 20) of the prefix-shared path; "1" = the
    per-mask k_mask_fit), an inactive counter in each half (constant rates,
    reading D3), shared and unshared prefixes, the empty and the full mask:
    every per-scenario field vs the oracle."""
    monkeypatch.setenv("SPEEDREC_MASK_PATH", mask_path)
    cfg = gen.make_config("C5", n_masks_k=1)
    ds = cfg.dataset
    ds.counters[:, 3] = ds.cycles * 0.125        # inactive in the prefix half
    ds.counters[:, 14] = ds.cycles * 0.5         # inactive in the suffix half
    rng = np.random.default_rng(11)
    masks = [0, (1 << 20) - 1, 0x3FF, 0xFFC00, 1 << 3, 1 << 14, (1 << 14) | 1, 0x5555, 0xAAAAA]
    masks += [int(m) for m in rng.integers(0, 1 << 20, size=24)]
    masks += [0x155 | (int(m) << 10) for m in rng.integers(0, 1 << 10, size=8)]   # one shared prefix
    sc = cfg.scenarios
    sc.all_subsets_k = 0
    sc.feature_masks = np.stack([np.array(masks, np.uint64), np.zeros(len(masks), np.uint64)], 1)
    sc.n_masks = len(masks)
    n = sc.n_splits * sc.n_masks
    got, ref = _run(Context, cfg, 0, n)
    print("C5 explicit masks path", mask_path, compare(got, ref))


def test_c5_mask_aggregation_and_top_k(Context):
    """A7 for C5: per-mask sums over the 128 LOO folds and the mask ranking
    (sum correct desc, id asc), fused in the kernel, per-scenario rows not
    materialised; exact integers vs the oracle's aggregation."""
    from paper_1910_07776_b200 import default_params
    cfg = gen.make_config("C5", n_masks_k=7)        # 128 masks x 128 folds
    folds = cfg.scenarios.n_splits
    n = cfg.scenarios.n_scenarios
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    for k in (5, 64, 200):
        p = default_params(top_k=k)
        got = ctx.evaluate(0, n, params=p, want_masks=True, per_scenario=False, n_folds=folds)
        ref = oracle.evaluate(cfg.dataset, cfg.scenarios, 0, n)
        assert ref["scn"]["n_guard"].sum() == 0
        rows, top = oracle.aggregate_masks(ref["opt"], ref["scn"], folds, top_k=k)
        for f in rows.dtype.names:
            assert np.array_equal(got["masks"][f], rows[f]), f
        assert list(got["top"][:len(top)]) == list(top)
        assert (got["top"][len(top):] == -1).all()
        assert got["totals"][1] == rows["n_test"].sum()
    # sub-range of whole masks, plus per-scenario rows in the same call
    got = ctx.evaluate(32 * folds, 16 * folds, params=default_params(top_k=4), want_masks=True, n_folds=folds)
    ref = oracle.evaluate(cfg.dataset, cfg.scenarios, 32 * folds, 16 * folds)
    rows, top = oracle.aggregate_masks(ref["opt"], ref["scn"], folds, first_mask=32, top_k=4)
    assert np.array_equal(got["masks"]["n_correct"], rows["n_correct"])
    assert list(got["top"]) == list(top)
    compare(got, ref)
    ctx.close()


def test_c5_full_2pow20_masks_sampled(Context):
    """Full C5 (all 2^20 masks x 128 LOO folds = 1.34e8 scenarios) through the
    feature-mask path in the bench's launch: the mask rows of sampled masks
    (each popcount, the extremes, the reported top 8) equal the oracle's sums
    over their 128 folds exactly; the top-64 keys are ordered by the rule and
    dominate every sampled mask."""
    from paper_1910_07776_b200 import default_params
    cfg = gen.make_config("C5", n_masks_k=20)
    folds = cfg.scenarios.n_splits
    n = cfg.scenarios.n_scenarios
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    got = ctx.evaluate(0, n, params=default_params(top_k=64), want_masks=True, per_scenario=False, n_folds=folds)
    ctx.close()
    rows, top = got["masks"], got["top"]
    rng = np.random.default_rng(3)
    sample = {0, 1, (1 << 20) - 1, 0b1010101010, *top[:8].tolist()}
    for d in range(21):            # one mask of each popcount
        bits = rng.choice(20, size=d, replace=False)
        sample.add(int(sum(1 << int(b) for b in bits)))
    sample |= set(rng.integers(0, 1 << 20, size=12).tolist())
    from concurrent.futures import ThreadPoolExecutor
    def one(m):
        r = oracle.evaluate(cfg.dataset, cfg.scenarios, m * folds, folds, n_threads=1)
        assert r["scn"]["n_guard"].sum() == 0
        return oracle.aggregate_masks(r["opt"], r["scn"], folds, first_mask=m, top_k=1)[0][0]
    with ThreadPoolExecutor(8) as pool:
        refs = dict(zip(sorted(sample), pool.map(one, sorted(sample))))
    for m, ref in refs.items():
        for f in ref.dtype.names:
            assert rows[f][m] == ref[f], (m, f, rows[f][m], ref[f])
    keys = [(int(rows["n_correct"][m]), -int(m)) for m in top]
    assert keys == sorted(keys, reverse=True)
    kth = keys[-1]
    for m in refs:
        assert m in set(top.tolist()) or (int(refs[m]["n_correct"]), -m) < kth


def test_c4_large_batch_path_small(Context):
    """> 64 groups -> the CTA-per-fit DMMA path (k_fit_big + k_rank_big):
    96 programs x 64 variants x 128 counters (n ~ 770 training pairs, d = 128)."""
    cfg = gen.make_config("C4", n_splits=24, n_programs=96)
    got, ref = _run(Context, cfg, 0, 24)
    print("C4 P=96", compare(got, ref))
    got, ref = _run(Context, cfg, 5, 7)             # ragged sub-range
    compare(got, ref)


def test_c4_full_size_sampled(Context):
    """Full C4 lattice (1024 programs, 65,536 slots, n ~ 8,192 pairs per fit,
    p = 129) in the bench launch; sampled scenarios vs the oracle."""
    cfg = gen.make_config("C4", n_splits=10_000_000)
    S = 148
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    got = ctx.evaluate(0, S)
    ctx.close()
    idx = [0, 77, 147]
    from concurrent.futures import ThreadPoolExecutor   # ctypes releases the GIL
    with ThreadPoolExecutor(len(idx)) as pool:
        refs = list(pool.map(lambda s: oracle.evaluate(cfg.dataset, cfg.scenarios, s, 1, n_threads=1), idx))
    st = compare(dict(opt=got["opt"][idx], scn=got["scn"][idx]),
                 dict(opt=np.concatenate([r["opt"] for r in refs]), scn=np.concatenate([r["scn"] for r in refs])))
    print("C4 full sampled", st, "n_train", got["opt"]["n_train"][idx].tolist())


def test_global_scratch_path(Context):
    # Force the Cholesky factor out of shared memory (debug_mcap=8): same results.
    for name, n in (("C3", 500), ("C2", 240), ("C1", 64)):
        cfg = gen.make_config(name, n_splits=n)
        got, ref = _run(Context, cfg, 0, min(n, cfg.scenarios.n_scenarios), params=dict(debug_mcap=8))
        compare(got, ref, max_guard_frac=0.05)


def test_degenerate_inputs(Context):
    # constant counters (d_eff = 0 -> EX = mean label), zero counters, a
    # single feature, and feature masks selecting nothing
    cfg = gen.make_config("C1")
    ds = cfg.dataset
    ds.counters[:, :8] = ds.cycles[:, None] * 0.25   # constant rates -> inactive features
    ds.counters[:, 8:16] = 0.0                       # all-zero features -> inactive
    sc = cfg.scenarios
    got, ref = _run(Context, cfg, 0, 64)
    compare(got, ref, max_guard_frac=0.05)
    sc.feature_masks = np.array([[0, 0], [1 << 20, 0], [0xFFFF0000, 0]], dtype=np.uint64)
    sc.n_masks = 3
    got, ref = _run(Context, cfg, 0, 64 * 3)
    compare(got, ref, max_guard_frac=0.05)


def test_determinism_and_sharding_invariance(Context):
    cfg = gen.make_config("C3", n_splits=4000)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    a = ctx.evaluate(0, 4000)
    b = ctx.evaluate(0, 4000)
    parts = [ctx.evaluate(k * 1000, 1000) for k in range(4)]
    ctx.close()
    assert a["opt"].tobytes() == b["opt"].tobytes() and a["scn"].tobytes() == b["scn"].tobytes()
    assert np.concatenate([p["opt"] for p in parts]).tobytes() == a["opt"].tobytes()
    assert np.concatenate([p["scn"] for p in parts]).tobytes() == a["scn"].tobytes()


def test_c3_full_size_sampled(Context):
    """Full bench workload (C3, 1e6 splits) in the bench's launch; sampled rows
    checked against the oracle one by one."""
    import torch
    from paper_1910_07776_b200.speedrec import OPT_SCORE_DTYPE, SCN_SCORE_DTYPE
    cfg = gen.make_config("C3")
    S = cfg.scenarios.n_scenarios
    ctx = Context(0, stream=torch.cuda.current_stream().cuda_stream)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    O = cfg.dataset.n_opt_ids
    dopt = torch.empty(S * O * OPT_SCORE_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    dscn = torch.empty(S * SCN_SCORE_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    ctx.evaluate(0, S, out=dict(opt=dopt, scn=dscn))
    torch.cuda.synchronize()
    opt = dopt.cpu().numpy().view(OPT_SCORE_DTYPE).reshape(S, O)
    scn = dscn.cpu().numpy().view(SCN_SCORE_DTYPE)
    ctx.close()
    rng = np.random.default_rng(0)
    idx = np.unique(np.r_[0, S - 1, rng.integers(0, S, size=300)])
    ref_opt, ref_scn = [], []
    for s in idx:
        r = oracle.evaluate(cfg.dataset, cfg.scenarios, int(s), 1, n_threads=1)
        ref_opt.append(r["opt"])
        ref_scn.append(r["scn"])
    st = compare(dict(opt=opt[idx], scn=scn[idx]),
                 dict(opt=np.concatenate(ref_opt), scn=np.concatenate(ref_scn)))
    print("C3 full sampled", st)
    # properties at full size: counts conservation of the 2^6 lattice
    assert (opt["n_test"].sum(1) <= 6 * 64).all()
    assert (scn["n_rec"] <= 3 * 128).all()


def test_errors_name_the_entity(Context):
    from paper_1910_07776_b200 import SpeedrecError, default_params
    from paper_1910_07776_b200 import speedrec as S
    cfg = gen.make_config("C1")
    ctx = Context(0)
    with pytest.raises(SpeedrecError) as e:
        ctx.evaluate(0, 1)
    assert e.value.status == S.SR_E_STATE or ctx.shape is None
    ds = cfg.dataset
    bad = ds.cycles.copy()
    bad[17] = 0.0
    with pytest.raises(SpeedrecError) as e:
        ctx.load_dataset(1, 1, 1, ds.n_counters, ds.n_opt_ids, ds.counters, bad, ds.runtime_ms, ds.opt_bit)
    assert e.value.status == S.SR_E_DATA and "slot 17" in str(e.value)
    ob = ds.opt_bit.copy()
    ob[0, 1] = ob[0, 0]
    with pytest.raises(SpeedrecError) as e:
        ctx.load_dataset(1, 1, 1, ds.n_counters, ds.n_opt_ids, ds.counters, ds.cycles, ds.runtime_ms, ob)
    assert e.value.status == S.SR_E_LATTICE
    ctx.load(ds)
    ctx.define_scenarios(cfg.scenarios)
    with pytest.raises(SpeedrecError) as e:
        ctx.evaluate(60, 10)
    assert e.value.status == S.SR_E_ARG
    with pytest.raises(SpeedrecError) as e:
        ctx.evaluate(0, 1, params=default_params(learner=7))
    assert e.value.status == S.SR_E_ARG and "learner" in str(e.value)
    r = ctx.evaluate(0, 0)                           # empty batch is valid
    assert r["opt"].shape[0] == 0
    ctx.close()


def test_bh6_all_table2_and_strip_chart(Context):
    """NEXT-3: Barnes-Hut with all six Table-1 inputs (144 Exp 1-4
    scenarios) vs the oracle, and the strip-chart rows (report.ratio_rows)
    of the GPU result against the oracle's, case by case."""
    from paper_1910_07776_b200 import report
    from tests.parity import rel_err
    cfg = gen.make_config("BH6")
    got, ref = _run(Context, cfg, 0, 144)
    print("BH6", compare(got, ref, max_guard_frac=0.05))
    guarded = ref["scn"]["n_guard"] != 0
    exp = cfg.scenarios.experiment
    g_rows = report.ratio_rows(cfg.dataset, got, exp)
    r_rows = report.ratio_rows(cfg.dataset, ref, exp)
    assert len(g_rows) == len(r_rows)
    for a, b in zip(g_rows, r_rows):
        assert {k: a[k] for k in a if k != "ratio"} == {k: b[k] for k in b if k != "ratio"}
    e = rel_err(np.array([a["ratio"] for a in g_rows]), np.array([b["ratio"] for b in r_rows]))
    assert guarded.any() or e.max() <= 1e-9
