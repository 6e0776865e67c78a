"""ORACLE -- test infrastructure, not part of the product path.

Python face of `oracle/oracle.c`, the plain CPU implementation of the
paper's Tier-2/Tier-3 path (see the C file's header for the step list and
citations).  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import this module.  It never
imports, links or calls anything from `paper_1910_07776_b200/`.

Parity status: every function is pinned by `tests/test_oracle_pins.py`
(worked examples from SPEC, exact rational brute force, closed forms and
invariants); see DESIGN.md §4 for the pin table.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C11 + libquadmath)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=gnu11", "-o", _LIB, _SRC,
                               "-lquadmath", "-lpthread", "-lm"])
    return _LIB


class OrDataset(ct.Structure):
    _fields_ = [("P", ct.c_int32), ("I", ct.c_int32), ("R", ct.c_int32), ("m", ct.c_int32),
                ("C", ct.c_int32), ("O", ct.c_int32),
                ("counters", ct.c_void_p), ("cycles", ct.c_void_p), ("runtime_ms", ct.c_void_p),
                ("opt_bit", ct.c_void_p)]


class OrScenarios(ct.Structure):
    _fields_ = [("kind", ct.c_int32), ("group_words", ct.c_int32), ("n_splits", ct.c_int64),
                ("train_groups", ct.c_void_p), ("test_groups", ct.c_void_p),
                ("split_opt_masks", ct.c_void_p), ("pool_groups", ct.c_void_p),
                ("seed", ct.c_uint64), ("opt_mask", ct.c_uint32), ("all_subsets_k", ct.c_int32),
                ("n_masks", ct.c_int64), ("feature_masks", ct.c_void_p)]


class OrParams(ct.Structure):
    _fields_ = [("ridge", ct.c_double), ("threshold", ct.c_double), ("clamp_floor", ct.c_double),
                ("guard_tol", ct.c_double), ("max_count", ct.c_int32), ("learner", ct.c_int32),
                ("k_nn", ct.c_int32), ("force_quad", ct.c_int32)]


OPT_SCORE_DTYPE = np.dtype([("n_train", "<i4"), ("n_test", "<i4"), ("n_correct", "<i4"),
                            ("n_clamped", "<i4"), ("sum_ratio", "<f8"), ("min_ratio", "<f8"),
                            ("max_ratio", "<f8"), ("fp_train", "<u8"), ("fp_test", "<u8")])
SCN_SCORE_DTYPE = np.dtype([("n_rec", "<i4"), ("n_rec_hit", "<i4"), ("n_untrained", "<i4"),
                            ("n_guard", "<i4")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ct.CDLL(build())
        _lib.or_mix64.restype = ct.c_uint64
        _lib.or_mix64.argtypes = [ct.c_uint64]
        _lib.or_split_word.restype = ct.c_uint64
        _lib.or_split_word.argtypes = [ct.c_uint64, ct.c_int64, ct.c_int64]
        _lib.or_rates.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_void_p]
        _lib.or_scale.restype = ct.c_int32
        _lib.or_scale.argtypes = [ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_int32, ct.c_void_p,
                                  ct.c_void_p, ct.c_void_p, ct.c_void_p]
        for fn in (_lib.or_fit_predict, _lib.or_fit_predict_ld):
            fn.restype = ct.c_int32
            fn.argtypes = [ct.c_int32, ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_void_p,
                           ct.c_int32, ct.c_void_p, ct.c_double, ct.c_void_p, ct.c_void_p, ct.c_void_p]
        _lib.or_rank.restype = ct.c_int32
        _lib.or_knn_predict.restype = None
        _lib.or_knn_predict.argtypes = [ct.c_int32, ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_void_p,
                                        ct.c_int32, ct.c_void_p, ct.c_int32, ct.c_void_p]
        _lib.or_rank.argtypes = [ct.c_int32, ct.c_void_p, ct.c_void_p, ct.c_double, ct.c_int32,
                                 ct.c_void_p, ct.c_void_p]
        _lib.or_sign_correct.restype = ct.c_int32
        _lib.or_sign_correct.argtypes = [ct.c_double, ct.c_double]
        _lib.or_evaluate.restype = ct.c_int32
        _lib.or_evaluate.argtypes = [ct.POINTER(OrDataset), ct.POINTER(OrScenarios),
                                     ct.POINTER(OrParams), ct.c_int64, ct.c_int64, ct.c_void_p,
                                     ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                     ct.c_int32]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------- steps
def mix64(x: int) -> int:
    return int(lib().or_mix64(int(x) & (2**64 - 1)))


def split_word(seed: int, split: int, word: int) -> int:
    return int(lib().or_split_word(seed, split, word))


def rates(counters: np.ndarray, cycles: np.ndarray) -> np.ndarray:
    counters = np.ascontiguousarray(counters, dtype=np.float64)
    cycles = np.ascontiguousarray(cycles, dtype=np.float64)
    out = np.empty_like(counters)
    lib().or_rates(_p(counters), _p(cycles), counters.shape[0], counters.shape[1], _p(out))
    return out


def scale(X: np.ndarray, Xt: np.ndarray):
    """Min-max scaling over training rows X; returns (Xs, Xts, active_cols)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Xt = np.ascontiguousarray(Xt, dtype=np.float64).reshape(-1, X.shape[1])
    n, d = X.shape
    Xs = np.zeros((n, d))
    Xts = np.zeros((Xt.shape[0], d))
    act = np.zeros(d, dtype=np.int32)
    de = lib().or_scale(n, d, _p(X), Xt.shape[0], _p(Xt), _p(Xs), _p(Xts), _p(act))
    return Xs[:, :de].copy(), Xts[:, :de].copy(), act[:de].copy()


def fit_predict(Xs: np.ndarray, y: np.ndarray, Xts: np.ndarray, ridge: float = 1e-8, precision: str = "quad",
                want_kappa: bool = False):
    """Ridge fit on already-scaled features; returns (EX [t], coef [1+d])
    (+ kappa^ = (max L_ii / min L_ii)^2 with want_kappa).  precision: "quad"
    (__float128) or "ld" (x87 long double, SURVEY 8(c)'s C4 allowance)."""
    Xs = np.ascontiguousarray(Xs, dtype=np.float64)
    n, d = Xs.shape
    y = np.ascontiguousarray(y, dtype=np.float64)
    Xts = np.ascontiguousarray(Xts, dtype=np.float64)
    Xts = Xts.reshape(-1, d) if d else Xts.reshape(Xts.shape[0], 0)
    t = Xts.shape[0]
    ex = np.zeros(t)
    coef = np.zeros(1 + d)
    kap = ct.c_double(1.0)
    fn = lib().or_fit_predict if precision == "quad" else lib().or_fit_predict_ld
    rc = fn(n, d, max(d, 1), _p(Xs) if d else _p(np.zeros(max(n, 1))), _p(y), t,
            _p(Xts) if d else _p(np.zeros(max(t, 1))), ridge, _p(ex), _p(coef), ct.byref(kap))
    if rc != 0:
        raise FloatingPointError("oracle Cholesky failed")
    return (ex, coef, kap.value) if want_kappa else (ex, coef)


def knn_predict(Xs: np.ndarray, y: np.ndarray, Xts: np.ndarray, k: int = 10) -> np.ndarray:
    """IBK on already-scaled features (see or_knn_predict for the exact form)."""
    Xs = np.ascontiguousarray(Xs, dtype=np.float64)
    n, d = Xs.shape
    y = np.ascontiguousarray(y, dtype=np.float64)
    Xts = np.ascontiguousarray(Xts, dtype=np.float64).reshape(-1, d) if d else np.zeros((len(Xts), 0))
    ex = np.zeros(Xts.shape[0])
    lib().or_knn_predict(n, d, max(d, 1), _p(Xs) if d else _p(np.zeros(max(n, 1))), _p(y), Xts.shape[0],
                         _p(Xts) if d else _p(np.zeros(max(len(ex), 1))), k, _p(ex))
    return ex


def rank(ex, ids, threshold: float = 1.05, max_count: int = 3):
    """Tier-3 rank-and-filter; returns (full order of ids, recommended ids)."""
    ex = np.ascontiguousarray(ex, dtype=np.float64)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    order = np.zeros(len(ex), dtype=np.int32)
    rec = np.zeros(max(len(ex), 1), dtype=np.int32)
    nr = lib().or_rank(len(ex), _p(ex), _p(ids), threshold, max_count, _p(order), _p(rec))
    return order.tolist(), rec[:nr].tolist()


def sign_correct(ex: float, ac: float) -> bool:
    return bool(lib().or_sign_correct(ex, ac))


MASK_SCORE_DTYPE = np.dtype([("n_correct", "<i4"), ("n_test", "<i4"), ("n_rec", "<i4"),
                             ("n_rec_hit", "<i4")])


def aggregate_masks(opt, scn, n_folds: int, first_mask: int = 0, top_k: int = 64):
    """C5 scoring (SURVEY §8(a) A7 "C5: per mask, sum over folds; rank masks by
    (sum correct desc, mask asc) and keep the top-K").

    opt/scn: per-scenario rows of whole masks (scenario s = mask*n_folds + fold).
    Returns (rows [n_masks] MASK_SCORE_DTYPE, top [<=top_k] int64 mask ids).
    """
    n_masks = len(scn) // n_folds
    assert n_masks * n_folds == len(scn)
    rows = np.zeros(n_masks, dtype=MASK_SCORE_DTYPE)
    o = opt.reshape(n_masks, n_folds, -1)
    s = scn.reshape(n_masks, n_folds)
    rows["n_correct"] = o["n_correct"].astype(np.int64).sum(axis=(1, 2))
    rows["n_test"] = o["n_test"].astype(np.int64).sum(axis=(1, 2))
    rows["n_rec"] = s["n_rec"].astype(np.int64).sum(axis=1)
    rows["n_rec_hit"] = s["n_rec_hit"].astype(np.int64).sum(axis=1)
    ids = np.arange(first_mask, first_mask + n_masks, dtype=np.int64)
    order = np.lexsort((ids, -rows["n_correct"].astype(np.int64)))   # primary: correct desc; then id asc
    return rows, ids[order[:top_k]]


# ---------------------------------------------------------------- batch
DEFAULT_PARAMS = dict(ridge=1e-8, threshold=1.05, clamp_floor=0.01, guard_tol=1e-9, max_count=3, learner=0,
                      k_nn=10, force_quad=0)
# learner ids: 0 ridge LS, 1 IBK; test-only scoring stubs: 100 EX := AC, 101 EX := 1
LEARNER_PERFECT_STUB, LEARNER_CONSTANT_STUB = 100, 101


def evaluate(ds, sc, first: int = 0, count: int | None = None, want_ex: bool = False,
             want_recs: bool = False, n_threads: int | None = None, want_kappa: bool = False, **params):
    """Run the oracle over scenarios [first, first+count) of (ds, sc).

    ds: gen.synth.Dataset; sc: gen.configs.Scenarios.
    Returns dict(opt=structured [count][O], scn=structured [count],
                 ex=[count][O][G*32] or None, recs=[count][N][K] or None,
                 kappa=[count][O] kappa^ per ridge fit (NaN: no fit) or None,
                 fit_ld=[count][O] 1 where the fit ran in long double, or None).
    """
    prm = dict(DEFAULT_PARAMS)
    prm.update(params)
    if count is None:
        count = sc.n_scenarios - first
    keep = []

    def arr(a, dt):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a

    counters = arr(ds.counters, np.float64)
    cycles = arr(ds.cycles, np.float64)
    rt = arr(ds.runtime_ms, np.float64)
    ob = arr(ds.opt_bit, np.int8)
    d = OrDataset(ds.n_programs, ds.n_inputs, ds.n_runs, ds.n_opt_bits, ds.n_counters, ds.n_opt_ids,
                  _p(counters), _p(cycles), _p(rt), _p(ob))
    kind = {"groups": 0, "loo": 1, "random": 2}[sc.kind]
    tg = arr(sc.train_groups, np.uint64)
    eg = arr(sc.test_groups, np.uint64)
    om = arr(sc.split_opt_masks, np.uint32)
    pg = arr(sc.pool_groups, np.uint64)
    fm = arr(sc.feature_masks, np.uint64)
    s = OrScenarios(kind, sc.group_words, sc.n_splits, _p(tg), _p(eg), _p(om), _p(pg),
                    sc.seed, sc.opt_mask, sc.all_subsets_k, sc.n_masks, _p(fm))
    p = OrParams(prm["ridge"], prm["threshold"], prm["clamp_floor"], prm["guard_tol"],
                 prm["max_count"], prm["learner"], prm["k_nn"], prm["force_quad"])
    O = ds.n_opt_ids
    G = ds.n_programs * ds.n_inputs * ds.n_runs
    V = 1 << ds.n_opt_bits
    opt = np.zeros((count, O), dtype=OPT_SCORE_DTYPE)
    scn = np.zeros(count, dtype=SCN_SCORE_DTYPE)
    ex = np.zeros((count, O, G * V // 2)) if want_ex else None
    recs = np.zeros((count, G * V, prm["max_count"]), dtype=np.int8) if want_recs else None
    kappa = np.full((count, O), np.nan) if want_kappa else None
    fit_ld = np.zeros((count, O), dtype=np.int32) if want_kappa else None
    if n_threads is None:
        n_threads = os.cpu_count() or 1
    rc = lib().or_evaluate(ct.byref(d), ct.byref(s), ct.byref(p), first, count, _p(opt), _p(scn),
                           _p(ex), _p(recs), _p(kappa), _p(fit_ld), n_threads)
    assert rc == 0
    return dict(opt=opt, scn=scn, ex=ex, recs=recs, kappa=kappa, fit_ld=fit_ld)
