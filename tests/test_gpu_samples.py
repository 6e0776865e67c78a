"""GPU parity on the oracle samples SURVEY §8(d) plans ("Oracle timing"
table), each also the oracle's timing sample:

  C3  first 20,000 splits + 1,000 splits at stride 1e3 of the full 1e6 batch
  C4  64 splits at stride 1e7/64 of the full 1024-program lattice, with EX
  C5  8,192 masks (all |S| <= 1, the full mask, 8,170 hashed masks) x 128 folds

Every scenario is compared element by element (tests/parity.py bar).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import gen
import oracle
from tests.parity import compare

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _cat(rs, keys=("opt", "scn", "ex", "recs")):
    return {k: (np.concatenate([r[k] for r in rs]) if rs[0].get(k) is not None else None) for k in keys}


def test_c3_first_20000_and_stride_1000():
    import torch
    from paper_1910_07776_b200 import Context
    from paper_1910_07776_b200.speedrec import OPT_SCORE_DTYPE, SCN_SCORE_DTYPE
    cfg = gen.make_config("C3")
    S, O = cfg.scenarios.n_scenarios, cfg.dataset.n_opt_ids
    ctx = Context(0, stream=torch.cuda.current_stream().cuda_stream)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    # (a) the bench launch: all 1e6 splits, device rows
    dopt = torch.empty(S * O * OPT_SCORE_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    dscn = torch.empty(S * SCN_SCORE_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    ctx.evaluate(0, S, out=dict(opt=dopt, scn=dscn))
    torch.cuda.synchronize()
    opt = dopt.cpu().numpy().view(OPT_SCORE_DTYPE).reshape(S, O)
    scn = dscn.cpu().numpy().view(SCN_SCORE_DTYPE)
    # (b) EX and recommendations of the first 20,000 splits
    head = ctx.evaluate(0, 20000, want_ex=True, want_recs=True)
    stride = np.arange(0, S, 1000)
    ctx.close()
    ref = oracle.evaluate(cfg.dataset, cfg.scenarios, 0, 20000, want_ex=True, want_recs=True)
    print("C3 first 20000 (EX, recs)", compare(head, ref))
    print("C3 first 20000 (bench launch rows)", compare(dict(opt=opt[:20000], scn=scn[:20000]), ref))
    with ThreadPoolExecutor(8) as pool:
        refs = list(pool.map(lambda s: oracle.evaluate(cfg.dataset, cfg.scenarios, int(s), 1, n_threads=1), stride))
    print("C3 stride 1000 (bench launch rows)",
          compare(dict(opt=opt[stride], scn=scn[stride]), _cat(refs, ("opt", "scn"))))


def test_c4_64_splits_at_stride():
    from paper_1910_07776_b200 import Context
    cfg = gen.make_config("C4", n_splits=10_000_000)
    idx = [k * (10_000_000 // 64) for k in range(64)]
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    got = _cat([ctx.evaluate(s, 1, want_ex=True) for s in idx], ("opt", "scn", "ex"))
    ctx.close()
    with ThreadPoolExecutor(8) as pool:
        refs = list(pool.map(lambda s: oracle.evaluate(cfg.dataset, cfg.scenarios, s, 1, want_ex=True, n_threads=1,
                                                        want_kappa=True), idx))
    ref = _cat(refs, ("opt", "scn", "ex"))
    kap = np.concatenate([r["kappa"] for r in refs])
    assert (np.concatenate([r["fit_ld"] for r in refs]) == 1).all()    # long-double policy
    print("C4 64 at stride (EX)", compare(got, ref), "kappa^ range", float(np.nanmin(kap)), float(np.nanmax(kap)))


def c5_plan_masks(k: int = 20, n: int = 8192, seed: int = 8192) -> np.ndarray:
    """All masks with |S| <= 1, the full mask, then distinct hashed masks."""
    base = [0] + [1 << b for b in range(k)] + [(1 << k) - 1]
    rng = np.random.default_rng(seed)
    seen = set(base)
    out = list(base)
    while len(out) < n:
        m = int(rng.integers(0, 1 << k))
        if m not in seen:
            seen.add(m)
            out.append(m)
    return np.array(sorted(out), dtype=np.uint64)


def test_c5_8192_masks_x_128_folds():
    from paper_1910_07776_b200 import Context, default_params
    cfg = gen.make_config("C5", n_masks_k=20)
    masks = c5_plan_masks()
    sc = cfg.scenarios
    sc.all_subsets_k = 0
    sc.feature_masks = np.stack([masks, np.zeros(len(masks), np.uint64)], 1)
    sc.n_masks = len(masks)
    folds = sc.n_splits
    n = sc.n_scenarios
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(sc)
    got = ctx.evaluate(0, n, params=default_params(top_k=64), want_masks=True)
    head = ctx.evaluate(0, 64 * folds, want_ex=True, want_recs=True)
    ctx.close()
    ref = oracle.evaluate(cfg.dataset, sc, 0, n)
    print("C5 8192 masks x 128 folds", compare(got, ref))
    rows, top = oracle.aggregate_masks(ref["opt"], ref["scn"], folds, top_k=64)
    for f in rows.dtype.names:
        assert np.array_equal(got["masks"][f], rows[f]), f
    assert list(got["top"]) == list(top)
    refh = oracle.evaluate(cfg.dataset, sc, 0, 64 * folds, want_ex=True, want_recs=True)
    print("C5 first 64 masks (EX, recs)", compare(head, refh))
