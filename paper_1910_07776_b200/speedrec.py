"""Thin ctypes binding of libspeedrec.so (include/speedrec.h).

Argument marshalling only: every step of the path (rates, pairs, scaling,
fits, prediction, ranking, scoring) runs in the library's CUDA kernels.
There is no CPU fallback: if the shared library is missing or no sm_100
GPU is present, the calls raise.

Host buffers are numpy arrays; device buffers are torch CUDA tensors (used
only for their data pointers -- torch is plumbing here).
"""
from __future__ import annotations

import ctypes as ct
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPEEDREC_LIB") or os.path.join(_HERE, "libspeedrec.so")  # env: A/B kernel variants

SR_OK, SR_E_ARG, SR_E_DATA, SR_E_LATTICE, SR_E_EMPTY, SR_E_STATE, SR_E_OOM, SR_E_CUDA, SR_E_UNSUPPORTED = \
    0, -1, -2, -3, -4, -5, -6, -7, -8
SPLIT_KIND = {"groups": 0, "loo": 1, "random": 2}

OPT_SCORE_DTYPE = np.dtype([("n_train", "<i4"), ("n_test", "<i4"), ("n_correct", "<i4"),
                            ("n_clamped", "<i4"), ("sum_ratio", "<f8"), ("min_ratio", "<f8"),
                            ("max_ratio", "<f8"), ("fp_train", "<u8"), ("fp_test", "<u8")])
SCN_SCORE_DTYPE = np.dtype([("n_rec", "<i4"), ("n_rec_hit", "<i4"), ("n_untrained", "<i4"),
                            ("n_guard", "<i4")])


class SpeedrecError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{status}] {message}")
        self.status = status


class sr_dataset(ct.Structure):
    _fields_ = [("n_programs", ct.c_int32), ("n_inputs", ct.c_int32), ("n_runs", ct.c_int32),
                ("n_opt_bits", ct.c_int32), ("n_counters", ct.c_int32), ("n_opt_ids", ct.c_int32),
                ("counters", ct.c_void_p), ("cycles", ct.c_void_p), ("runtime_ms", ct.c_void_p),
                ("opt_bit", ct.c_void_p), ("on_device", ct.c_int32)]


class sr_scenarios(ct.Structure):
    _fields_ = [("kind", ct.c_int32), ("group_words", ct.c_int32), ("n_splits", ct.c_int64),
                ("train_groups", ct.c_void_p), ("test_groups", ct.c_void_p),
                ("split_opt_masks", ct.c_void_p), ("pool_groups", ct.c_void_p),
                ("seed", ct.c_uint64), ("opt_mask", ct.c_uint32), ("all_subsets_k", ct.c_int32),
                ("n_masks", ct.c_int64), ("feature_masks", ct.c_void_p)]


class sr_params(ct.Structure):
    _fields_ = [("learner", ct.c_int32), ("max_count", ct.c_int32), ("refine_steps", ct.c_int32),
                ("debug_mcap", ct.c_int32), ("ridge", ct.c_double), ("threshold", ct.c_double),
                ("clamp_floor", ct.c_double), ("guard_tol", ct.c_double), ("top_k", ct.c_int32),
                ("k_nn", ct.c_int32)]


class sr_outputs(ct.Structure):
    _fields_ = [("opt_scores", ct.c_void_p), ("scn_scores", ct.c_void_p), ("ex", ct.c_void_p),
                ("recs", ct.c_void_p), ("totals", ct.c_void_p), ("mask_scores", ct.c_void_p),
                ("top_masks", ct.c_void_p), ("on_device", ct.c_int32)]


MASK_SCORE_DTYPE = np.dtype([("n_correct", "<i4"), ("n_test", "<i4"), ("n_rec", "<i4"),
                             ("n_rec_hit", "<i4")])


# Every symbol include/speedrec.h declares (checked by tests/test_boundary.py).
EXPORTS = ["sr_create", "sr_destroy", "sr_last_error", "sr_version", "sr_load_dataset",
           "sr_define_scenarios", "sr_default_params", "sr_evaluate", "sr_rates", "sr_synchronize",
           "sr_set_timing", "sr_kernel_stats", "sr_reset_kernel_stats", "sr_last_launch_count",
           "sr_fit", "sr_predict", "sr_recommend", "sr_sweep", "sr_last_work"]

_lib = None


def lib() -> ct.CDLL:
    """Load libspeedrec.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ct.CDLL(LIB_PATH)
        L.sr_create.argtypes = [ct.c_int32, ct.c_void_p, ct.POINTER(ct.c_void_p)]
        L.sr_create.restype = ct.c_int32
        L.sr_destroy.argtypes = [ct.c_void_p]
        L.sr_destroy.restype = None
        L.sr_last_error.argtypes = [ct.c_void_p]
        L.sr_last_error.restype = ct.c_char_p
        L.sr_version.restype = ct.c_char_p
        L.sr_load_dataset.argtypes = [ct.c_void_p, ct.POINTER(sr_dataset)]
        L.sr_load_dataset.restype = ct.c_int32
        L.sr_define_scenarios.argtypes = [ct.c_void_p, ct.POINTER(sr_scenarios), ct.POINTER(ct.c_int64)]
        L.sr_define_scenarios.restype = ct.c_int32
        L.sr_default_params.argtypes = [ct.POINTER(sr_params)]
        L.sr_default_params.restype = None
        L.sr_evaluate.argtypes = [ct.c_void_p, ct.POINTER(sr_params), ct.c_int64, ct.c_int64,
                                  ct.POINTER(sr_outputs)]
        L.sr_evaluate.restype = ct.c_int32
        L.sr_rates.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_int32]
        L.sr_rates.restype = ct.c_int32
        L.sr_synchronize.argtypes = [ct.c_void_p]
        L.sr_synchronize.restype = ct.c_int32
        L.sr_set_timing.argtypes = [ct.c_void_p, ct.c_int32]
        L.sr_set_timing.restype = ct.c_int32
        L.sr_kernel_stats.argtypes = [ct.c_void_p, ct.c_int32, ct.POINTER(ct.c_char_p),
                                      ct.POINTER(ct.c_int32), ct.POINTER(ct.c_double)]
        L.sr_kernel_stats.restype = ct.c_int32
        L.sr_reset_kernel_stats.argtypes = [ct.c_void_p]
        L.sr_reset_kernel_stats.restype = ct.c_int32
        L.sr_last_launch_count.argtypes = [ct.c_void_p]
        L.sr_last_launch_count.restype = ct.c_int32
        L.sr_last_work.argtypes = [ct.c_void_p]
        L.sr_last_work.restype = ct.c_int64
        L.sr_fit.argtypes = [ct.c_void_p, ct.POINTER(sr_params), ct.c_int64, ct.c_void_p]
        L.sr_sweep.argtypes = [ct.c_void_p, ct.POINTER(sr_params), ct.c_int64, ct.c_int64, ct.c_int32, ct.c_void_p,
                               ct.c_int32, ct.c_void_p, ct.c_void_p, ct.c_void_p]
        L.sr_sweep.restype = ct.c_int32
        L.sr_fit.restype = ct.c_int32
        L.sr_predict.argtypes = [ct.POINTER(sr_params), ct.c_void_p, ct.c_int32, ct.c_int32, ct.c_void_p,
                                 ct.c_double, ct.c_void_p]
        L.sr_predict.restype = ct.c_int32
        L.sr_recommend.argtypes = [ct.POINTER(sr_params), ct.c_void_p, ct.c_void_p, ct.c_int32, ct.c_void_p,
                                   ct.POINTER(ct.c_int32)]
        L.sr_recommend.restype = ct.c_int32
        _lib = L
    return _lib


SR_LINREG, SR_IBK, SR_M5P = 0, 1, 2          # sr_learner (include/speedrec.h)
LEARNERS = {"linreg": SR_LINREG, "ibk": SR_IBK, "m5": SR_M5P}


def default_params(**overrides) -> sr_params:
    """sr_default_params + overrides; learner may be given by name
    ("linreg" | "ibk" | "m5") or by its sr_learner value."""
    if isinstance(overrides.get("learner"), str):
        overrides["learner"] = LEARNERS[overrides["learner"]]
    p = sr_params()
    lib().sr_default_params(ct.byref(p))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


def _is_dev(a) -> bool:
    return not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)


class Context:
    """One sr_ctx on one GPU (one process per GPU for multi-GPU runs)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self._h = ct.c_void_p()
        st = lib().sr_create(device, ct.c_void_p(stream) if stream else None, ct.byref(self._h))
        if st != SR_OK:
            raise SpeedrecError(st, f"sr_create(device={device}) failed (needs an sm_100 GPU)")
        self._keep = []
        self.n_scenarios = 0
        self.n_splits = None
        self.shape = None

    def close(self):
        if self._h:
            lib().sr_destroy(self._h)
            self._h = ct.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != SR_OK:
            raise SpeedrecError(st, lib().sr_last_error(self._h).decode())

    # ------------------------------------------------------------ inputs
    def load_dataset(self, n_programs, n_inputs, n_runs, n_counters, n_opt_ids, counters, cycles,
                     runtime_ms, opt_bit, n_opt_bits: int = 6):
        """counters/cycles/runtime_ms/opt_bit: all numpy (host) or all torch CUDA tensors."""
        dev = _is_dev(counters)
        if not dev:
            counters = np.ascontiguousarray(counters, dtype=np.float64)
            cycles = np.ascontiguousarray(cycles, dtype=np.float64)
            runtime_ms = np.ascontiguousarray(runtime_ms, dtype=np.float64)
            opt_bit = np.ascontiguousarray(opt_bit, dtype=np.int8)
        d = sr_dataset(n_programs, n_inputs, n_runs, n_opt_bits, n_counters, n_opt_ids,
                       _ptr(counters), _ptr(cycles), _ptr(runtime_ms), _ptr(opt_bit), int(dev))
        self.shape = None             # the library drops the previous dataset on any failure
        self.n_scenarios = 0
        self._check(lib().sr_load_dataset(self._h, ct.byref(d)))
        self.shape = dict(P=n_programs, I=n_inputs, R=n_runs, C=n_counters, O=n_opt_ids,
                          G=n_programs * n_inputs * n_runs)

    def load(self, ds):
        """Load a gen.synth.Dataset-like object (host arrays)."""
        self.load_dataset(ds.n_programs, ds.n_inputs, ds.n_runs, ds.n_counters, ds.n_opt_ids,
                          ds.counters, ds.cycles, ds.runtime_ms, ds.opt_bit, ds.n_opt_bits)

    def define_scenarios(self, sc) -> int:
        """sc: an object with the sr_scenarios fields (e.g. gen.configs.Scenarios)."""
        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a
        tg, eg = arr(sc.train_groups, np.uint64), arr(sc.test_groups, np.uint64)
        om, pg = arr(sc.split_opt_masks, np.uint32), arr(sc.pool_groups, np.uint64)
        fm = arr(sc.feature_masks, np.uint64)
        s = sr_scenarios(SPLIT_KIND[sc.kind], sc.group_words, sc.n_splits, _ptr(tg), _ptr(eg), _ptr(om),
                         _ptr(pg), sc.seed, sc.opt_mask, sc.all_subsets_k, sc.n_masks, _ptr(fm))
        n = ct.c_int64()
        self.n_scenarios = 0          # the library drops the previous definition on any failure
        self.n_splits = None
        self._check(lib().sr_define_scenarios(self._h, ct.byref(s), ct.byref(n)))
        self._keep = []
        self.n_scenarios = n.value
        self.n_splits = int(sc.n_splits)
        return n.value

    # ------------------------------------------------------------ compute
    def evaluate(self, first: int = 0, count: Optional[int] = None, params: Optional[sr_params] = None,
                 want_ex: bool = False, want_recs: bool = False, out: Optional[dict] = None,
                 want_masks: bool = False, per_scenario: bool = True, n_folds: Optional[int] = None):
        """Run the fused path on scenarios [first, first+count).

        out=None: host numpy outputs (synchronous).  out=dict of torch CUDA
        tensors {opt, scn[, ex, recs, totals, masks, top]}: device outputs,
        asynchronous on the context stream.  want_masks: per-mask sums over
        the folds + top-k mask ids (C5); per_scenario=False skips the rows.
        """
        if count is None:
            count = self.n_scenarios - first
        p = params or default_params()
        if self.shape is None:      # let the library report the call-order error
            o = sr_outputs()
            self._check(lib().sr_evaluate(self._h, ct.byref(p), first, count, ct.byref(o)))
        O, G = self.shape["O"], self.shape["G"]
        if out is None:
            opt = np.zeros((count, O), dtype=OPT_SCORE_DTYPE) if per_scenario else None
            scn = np.zeros(count, dtype=SCN_SCORE_DTYPE) if per_scenario else None
            ex = np.zeros((count, O, G * 32)) if want_ex else None
            recs = np.zeros((count, G * 64, p.max_count), dtype=np.int8) if want_recs else None
            tot = np.zeros(4, dtype=np.int64)
            masks = top = None
            if want_masks:
                folds = n_folds if n_folds is not None else getattr(self, "n_splits", None)
                if not folds:
                    raise ValueError("evaluate(want_masks=True): define_scenarios first (mask rows sum its n_splits folds)")
                masks = np.zeros(count // folds, dtype=MASK_SCORE_DTYPE)
                top = np.zeros(p.top_k, dtype=np.int64)
            o = sr_outputs(_ptr(opt), _ptr(scn), _ptr(ex), _ptr(recs), _ptr(tot), _ptr(masks), _ptr(top), 0)
            self._check(lib().sr_evaluate(self._h, ct.byref(p), first, count, ct.byref(o)))
            return dict(opt=opt, scn=scn, ex=ex, recs=recs, totals=tot, masks=masks, top=top)
        o = sr_outputs(_ptr(out.get("opt")), _ptr(out.get("scn")), _ptr(out.get("ex")), _ptr(out.get("recs")),
                       _ptr(out.get("totals")), _ptr(out.get("masks")), _ptr(out.get("top")), 1)
        self._check(lib().sr_evaluate(self._h, ct.byref(p), first, count, ct.byref(o)))
        return out

    def sweep(self, thresholds, max_counts, first: int = 0, count: Optional[int] = None,
              params: Optional[sr_params] = None):
        """sr_sweep (NEXT-3): pooled (recommendations, hits) [n_thr][n_cnt] of the
        Tier-3 rule for every (threshold, list length) over scenarios [first, first+count)."""
        thr = np.ascontiguousarray(thresholds, dtype=np.float64)
        cnt = np.ascontiguousarray(max_counts, dtype=np.int32)
        if count is None:
            count = self.n_scenarios - first
        rec = np.zeros((len(thr), len(cnt)), dtype=np.int64)
        hit = np.zeros_like(rec)
        p = params or default_params()
        self._check(lib().sr_sweep(self._h, ct.byref(p), int(first), int(count), len(thr), _ptr(thr), len(cnt),
                                   _ptr(cnt), _ptr(rec), _ptr(hit)))
        return rec, hit

    def fit(self, scenario: int, params: Optional[sr_params] = None) -> np.ndarray:
        """sr_fit: [O][1 + C] raw-counter models (c0, u) of one scenario; NaN c0 = no model."""
        coef = np.zeros((self.shape["O"], self.shape["C"] + 1) if self.shape else 1)
        p = params or default_params()
        self._check(lib().sr_fit(self._h, ct.byref(p), int(scenario), _ptr(coef)))
        return coef

    def rates(self) -> np.ndarray:
        N = self.shape["G"] * 64
        x = np.zeros((N, self.shape["C"]))
        self._check(lib().sr_rates(self._h, _ptr(x), 0))
        return x

    def synchronize(self):
        self._check(lib().sr_synchronize(self._h))

    # ------------------------------------------------------------ accounting
    def set_timing(self, on: bool):
        self._check(lib().sr_set_timing(self._h, int(on)))

    def reset_kernel_stats(self):
        self._check(lib().sr_reset_kernel_stats(self._h))

    def kernel_stats(self) -> dict:
        cap = 32
        names = (ct.c_char_p * cap)()
        launches = (ct.c_int32 * cap)()
        ms = (ct.c_double * cap)()
        n = lib().sr_kernel_stats(self._h, cap, names, launches, ms)
        return {names[i].decode(): (int(launches[i]), float(ms[i])) for i in range(min(n, cap))}

    def last_launch_count(self) -> int:
        return int(lib().sr_last_launch_count(self._h))

    def last_work(self) -> int:
        """sr_last_work: executed M5P split-search FP64 operations of the last evaluate."""
        return int(lib().sr_last_work(self._h))


def predict(coef: np.ndarray, counters: np.ndarray, cycles: float, params: Optional[sr_params] = None) -> np.ndarray:
    """sr_predict: Tier-2 EX of one user profile from sr_fit's models."""
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    counters = np.ascontiguousarray(counters, dtype=np.float64)
    O, C1 = coef.shape
    ex = np.zeros(O)
    st = lib().sr_predict(ct.byref(params or default_params()), _ptr(coef), O, C1 - 1, _ptr(counters),
                          float(cycles), _ptr(ex))
    if st:
        raise SpeedrecError(st, f"predict: status {st}")
    return ex


def recommend(ex: np.ndarray, candidate: Optional[np.ndarray] = None,
              params: Optional[sr_params] = None) -> list:
    """sr_recommend: Tier-3 list: ids with EX >= threshold, (EX desc, id asc), first max_count."""
    p = params or default_params()
    ex = np.ascontiguousarray(ex, dtype=np.float64)
    cand = None if candidate is None else np.ascontiguousarray(candidate, dtype=np.uint8)
    rec = np.zeros(p.max_count, dtype=np.int8)
    n = ct.c_int32(0)
    st = lib().sr_recommend(ct.byref(p), _ptr(ex), _ptr(cand), len(ex), _ptr(rec), ct.byref(n))
    if st:
        raise SpeedrecError(st, f"recommend: status {st}")
    return [int(r) for r in rec[:n.value]]
