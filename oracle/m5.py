"""M5P model tree (NEXT-2) -- ORACLE, test infrastructure only.

Plain, slow, obviously-correct Python following the paper's description
("an induction algorithm is used to construct a standard decision
tree.  Then a multivariate regression model is constructed for each node in
the tree ... only the features that appear in the subtree that contains the
node are used.  Finally, the leaf nodes ... are replaced with the newly
constructed regression models ... standard pruning and smoothing techniques
are applied", citing Quinlan's M5 [10]) and SPEC's m5_build / m5_predict
 for the constants.  Readings (M1-M6):

  M1 splits: standard-deviation reduction SDR = sd(T) - sum_i |T_i|/|T| sd(T_i)
     with the population sd (two-pass), candidates = midpoints between
     adjacent distinct sorted values of each feature; max SDR, ties to the
     lower feature index, then the lower threshold; x <= threshold goes left.
  M2 stop: |T| < 4, or sd(T) < 0.05 sd(root), or no candidate with SDR > 0.
  M3 node models: ridge least squares (reading D1: lambda = 1e-8 on the
     weights, intercept unpenalised) over the features split on in the
     node's subtree; leaves: intercept only (the mean).  Solved in exact
     rational arithmetic, rounded once.
  M4 pruning (bottom-up): node error = mean absolute training residual of
     its model times (n+v)/(n-v) (v = model parameters incl. intercept;
     factor 10 when n <= v); subtree error = size-weighted mean of the
     children's (final) errors; prune to the node's model when its error is
     <= the subtree's.
  M5 smoothing (Quinlan): from the leaf up, p <- (n p + k q)/(n + k), q the
     model value of the ancestor, n the training count of the node p came
     from, k = 15.
  M6 features are the fit's min-max scaled counters (reading D3), as for the
     other learners.

Pinned by tests/test_m5_oracle.py (SPEC examples, closed forms, invariants).
"""
from __future__ import annotations

import math
from fractions import Fraction

SMOOTH_K = 15.0
MIN_SPLIT = 4
SD_FRAC = 0.05
RIDGE = 1e-8


def sd_pop(y) -> float:
    """Population standard deviation, two-pass, sums accumulated left to right
    in FP64 (M1; explicit loops, since builtin sum() compensates on 3.12+)."""
    n = len(y)
    if n == 0:
        return 0.0
    s = 0.0
    for v in y:
        s += v
    m = s / n
    q = 0.0
    for v in y:
        dv = v - m
        q += dv * dv
    return math.sqrt(q / n)


def sdr(y, left) -> float:
    """SDR of splitting y into left (bool list) / right."""
    yl = [v for v, l in zip(y, left) if l]
    yr = [v for v, l in zip(y, left) if not l]
    n = len(y)
    return sd_pop(y) - len(yl) / n * sd_pop(yl) - len(yr) / n * sd_pop(yr)


def best_split(X, y, idx):
    """(feature, threshold, sdr) of the best candidate over rows idx, or None (M1)."""
    best = None
    ys = [y[i] for i in idx]
    for a in range(len(X[0]) if X else 0):
        vals = sorted({X[i][a] for i in idx})
        for lo, hi in zip(vals, vals[1:]):
            thr = (lo + hi) / 2.0
            s = sdr(ys, [X[i][a] <= thr for i in idx])
            if best is None or s > best[2]:        # strict: ties keep lower feature, lower threshold
                best = (a, thr, s)
    return best


def ridge_fit(X, y, idx, feats, lam=RIDGE):
    """Exact-rational ridge LS (M3): minimise sum (y - b - w.x)^2 + lam |w|^2
    over the features `feats`; returns (b, {a: w_a}) as floats."""
    p = len(feats) + 1
    rows = [[Fraction(1)] + [Fraction(X[i][a]) for a in feats] for i in idx]
    yv = [Fraction(y[i]) for i in idx]
    lamf = Fraction(lam)
    A = [[sum(r[j] * r[k] for r in rows) + (lamf if (j == k and j > 0) else 0) for k in range(p)] for j in range(p)]
    rhs = [sum(r[j] * t for r, t in zip(rows, yv)) for j in range(p)]
    # Gauss-Jordan with exact arithmetic (A is SPD for lam > 0 and n >= 1)
    for c in range(p):
        piv = next(r for r in range(c, p) if A[r][c] != 0)
        A[c], A[piv] = A[piv], A[c]
        rhs[c], rhs[piv] = rhs[piv], rhs[c]
        inv = 1 / A[c][c]
        for r in range(p):
            if r != c and A[r][c] != 0:
                f = A[r][c] * inv
                for k in range(c, p):
                    A[r][k] -= f * A[c][k]
                rhs[r] -= f * rhs[c]
    sol = [rhs[j] / A[j][j] for j in range(p)]
    return float(sol[0]), {a: float(sol[1 + k]) for k, a in enumerate(feats)}


def model_value(model, x) -> float:
    b, w = model
    s = 0.0
    for a, wa in w.items():                        # ascending feature order
        s += wa * x[a]
    return b + s


class Node:
    __slots__ = ("idx", "n", "feature", "thr", "left", "right", "model", "allowed", "err")

    def __init__(self, idx):
        self.idx, self.n = idx, len(idx)
        self.feature = self.thr = self.left = self.right = None
        self.model = None
        self.allowed = []
        self.err = 0.0

    @property
    def leaf(self) -> bool:
        return self.left is None


def _grow(X, y, idx, sd_root):
    node = Node(idx)
    ys = [y[i] for i in idx]
    if len(idx) < MIN_SPLIT or sd_pop(ys) < SD_FRAC * sd_root:
        return node
    best = best_split(X, y, idx)
    if best is None or not best[2] > 0.0:
        return node
    a, thr, _ = best
    node.feature, node.thr = a, thr
    node.left = _grow(X, y, [i for i in idx if X[i][a] <= thr], sd_root)
    node.right = _grow(X, y, [i for i in idx if X[i][a] > thr], sd_root)
    return node


def _models(node, X, y, tol):
    """Post-order: allowed features = splits in the subtree (M3), models, M4
    pruning.  Returns the number of pruning decisions within tol of their
    boundary (guard cases, reading R21)."""
    guard = 0
    if node.leaf:
        node.allowed = []
    else:
        guard += _models(node.left, X, y, tol)
        guard += _models(node.right, X, y, tol)
        node.allowed = sorted({node.feature, *node.left.allowed, *node.right.allowed})
    node.model = ridge_fit(X, y, node.idx, node.allowed)
    rs = 0.0
    for i in node.idx:
        rs += abs(y[i] - model_value(node.model, X[i]))
    resid = rs / node.n
    v = len(node.allowed) + 1
    f = (node.n + v) / (node.n - v) if node.n > v else 10.0
    own = resid * f
    if node.leaf:
        node.err = own
        return guard
    sub = (node.left.n * node.left.err + node.right.n * node.right.err) / node.n
    if abs(own - sub) <= tol * max(1.0, abs(own)):
        guard += 1
    if own <= sub:                                  # prune to the node's model
        node.left = node.right = None
        node.feature = node.thr = None
        node.err = own
    else:
        node.err = sub
    return guard


def m5_build(X, y, guard_tol=1e-9, counted=False):
    """X: list of feature rows (floats), y: labels.  Returns the root Node
    (counted=True: (root, number of pruning guard cases))."""
    if not y:
        raise ValueError("m5_build: empty dataset")
    if not all(math.isfinite(v) for v in y):
        raise ValueError("m5_build: non-finite labels")
    idx = list(range(len(y)))
    root = _grow(X, y, idx, sd_pop(list(y)))
    guard = _models(root, X, y, guard_tol)
    return (root, guard) if counted else root


def m5_predict(root, x, k: float = SMOOTH_K) -> float:
    """Route x (x[a] <= thr -> left) to a leaf, then smooth root-ward (M5)."""
    path = []
    node = root
    while not node.leaf:
        path.append(node)
        node = node.left if x[node.feature] <= node.thr else node.right
    p, n_below = model_value(node.model, x), node.n
    for anc in reversed(path):
        q = model_value(anc.model, x)
        p = (n_below * p + k * q) / (n_below + k)
        n_below = anc.n
    return p


def walk(root):
    out, stack = [], [root]
    while stack:
        nd = stack.pop()
        out.append(nd)
        if not nd.leaf:
            stack += [nd.left, nd.right]
    return out


# ---------------------------------------------------------------- scenarios
def _membership(ds, sc, split):
    """Train / test flags of every slot under split (reading R17)."""
    from . import split_word
    G, V = ds.n_programs * ds.n_inputs * ds.n_runs, 1 << ds.n_opt_bits
    N = G * V
    tr, te = [False] * N, [False] * N
    if sc.kind == "groups":
        trw, tew = sc.train_groups[split], sc.test_groups[split]
        for t in range(N):
            g = t // V
            tr[t] = bool((int(trw[g >> 6]) >> (g & 63)) & 1)
            te[t] = bool((int(tew[g >> 6]) >> (g & 63)) & 1)
    elif sc.kind == "loo":
        k = 0
        for t in range(N):
            g = t // V
            if not (int(sc.pool_groups[g >> 6]) >> (g & 63)) & 1:
                continue
            if k == split:
                te[t] = True
            else:
                tr[t] = True
            k += 1
    else:
        for t in range(N):
            w = split_word(sc.seed, split, t // 64)
            tr[t] = bool((w >> (t % 64)) & 1)
            te[t] = not tr[t]
    return tr, te


def _features(ds, sc, fidx):
    C = ds.n_counters
    if sc.all_subsets_k:
        return [c for c in range(C) if c < sc.all_subsets_k and (fidx >> c) & 1]
    if sc.feature_masks is not None and sc.n_masks > 0 and sc.feature_masks is not None:
        m = sc.feature_masks[fidx]
        return [c for c in range(C) if (int(m[c >> 6]) >> (c & 63)) & 1]
    return list(range(C))


def evaluate(ds, sc, first=0, count=None, learner="m5", threshold=1.05, max_count=3, clamp_floor=0.01,
             guard_tol=1e-9, ridge=RIDGE):
    """The whole path (A1-A7) for scenarios [first, first+count) with the M5P
    learner (learner="ridge": ridge LS on every active feature instead -- the
    plumbing's pin against the C oracle).  Returns dict(opt, scn, ex) laid out
    like oracle.evaluate(want_ex=True)."""
    from . import OPT_SCORE_DTYPE, SCN_SCORE_DTYPE, mix64, rank, rates, scale
    import numpy as np
    if count is None:
        count = sc.n_scenarios - first
    G, V, O = ds.n_programs * ds.n_inputs * ds.n_runs, 1 << ds.n_opt_bits, ds.n_opt_ids
    IR = ds.n_inputs * ds.n_runs
    half = V // 2
    x = rates(ds.counters, ds.cycles)
    rt = ds.runtime_ms
    opt = np.zeros((count, O), dtype=OPT_SCORE_DTYPE)
    scn = np.zeros(count, dtype=SCN_SCORE_DTYPE)
    ex = np.zeros((count, O, G * half))
    near = lambda a, b: abs(a - b) <= guard_tol * max(1.0, abs(a))
    for si in range(count):
        s = first + si
        split, fidx = s % sc.n_splits, s // sc.n_splits
        F = _features(ds, sc, fidx)
        tr, te = _membership(ds, sc, split)
        om = int(sc.split_opt_masks[split]) if sc.split_opt_masks is not None else int(sc.opt_mask)
        trained = [False] * O
        exo, clo = {}, {}
        guard = 0
        untrained = 0
        for o in range(O):
            if not (om >> o) & 1:
                continue
            rows, ys, tests = [], [], []
            fptr = fpte = 0
            for g in range(G):
                b = int(ds.opt_bit[g // IR, o])
                if b < 0:
                    continue
                k = 0
                for v in range(V):
                    if (v >> b) & 1:
                        continue
                    bef, aft = g * V + v, g * V + (v | (1 << b))
                    pid = (g * O + o) * half + k
                    y = rt[bef] / rt[aft]
                    if tr[bef] and tr[aft]:
                        rows.append(bef)
                        ys.append(y)
                        fptr ^= mix64(pid)
                    if te[bef]:
                        tests.append((bef, g * half + k, y))
                        fpte ^= mix64(pid)
                    k += 1
            row = opt[si, o]
            row["n_train"], row["n_test"], row["fp_train"], row["fp_test"] = len(rows), len(tests), fptr, fpte
            if not rows:
                untrained += len(tests)
                continue
            trained[o] = True
            if not tests:
                continue
            Xr = x[rows][:, F] if F else np.zeros((len(rows), 0))
            Xt = x[[t[0] for t in tests]][:, F] if F else np.zeros((len(tests), 0))
            if F:
                Xs, Xts, _ = scale(Xr, Xt)
            else:
                Xs, Xts = np.zeros((len(rows), 0)), np.zeros((len(tests), 0))
            Xs_l, Xts_l = Xs.tolist(), Xts.tolist()
            if learner == "m5":
                root, gd = m5_build(Xs_l, ys, guard_tol, counted=True)
                guard += gd
                pred = [m5_predict(root, xt) for xt in Xts_l]
            else:
                mdl = ridge_fit(Xs_l, ys, list(range(len(ys))), list(range(Xs.shape[1])), lam=ridge)
                pred = [model_value(mdl, xt) for xt in Xts_l]
            ncorr = ncl = 0
            rs, rmn, rmx = 0.0, math.inf, -math.inf
            for (bef, pk, ac), e in zip(tests, pred):
                if near(e, 0.0) or near(e, 1.0):
                    guard += 1
                cl = e <= 0.0
                if cl:
                    e = clamp_floor
                    ncl += 1
                ncorr += 1 if ((e > 1.0 and ac > 1.0) or (e <= 1.0 and ac <= 1.0)) else 0
                r = ac / e
                rs += r
                rmn, rmx = min(rmn, r), max(rmx, r)
                ex[si, o, pk] = e
                exo[(o, pk)] = e
                clo[(o, pk)] = cl
            row["n_correct"], row["n_clamped"] = ncorr, ncl
            row["sum_ratio"], row["min_ratio"], row["max_ratio"] = rs, rmn, rmx
        # A6: per test version, candidates = scored, trained, bit clear (R13)
        nrec = nhit = 0
        for g in range(G):
            p = g // IR
            for v in range(V):
                if not te[g * V + v]:
                    continue
                ids, exs, cls, acs = [], [], [], []
                for o in range(O):
                    b = int(ds.opt_bit[p, o])
                    if not (om >> o) & 1 or b < 0 or (v >> b) & 1:
                        continue
                    if not trained[o]:
                        continue
                    kk = (v & ((1 << b) - 1)) | ((v >> (b + 1)) << b)
                    ids.append(o)
                    exs.append(exo[(o, g * half + kk)])
                    cls.append(clo[(o, g * half + kk)])
                    acs.append(rt[g * V + v] / rt[g * V + (v | (1 << b))])
                for i in range(len(ids)):
                    if near(exs[i], threshold):
                        guard += 1
                    for j in range(i + 1, len(ids)):
                        if not (cls[i] and cls[j]) and near(exs[i], exs[j]):
                            guard += 1
                if ids:
                    _, r = rank(np.array(exs), np.array(ids), threshold, max_count)
                    nrec += len(r)
                    nhit += sum(acs[ids.index(o)] > 1.0 for o in r)
        scn[si] = (nrec, nhit, untrained, guard)
    return dict(opt=opt, scn=scn, ex=ex)
