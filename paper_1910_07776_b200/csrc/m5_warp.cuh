// m5_warp.cuh -- the M5P model-tree learner (NEXT-2) on the warp path:
// one warp grows, fits, prunes and evaluates the tree of one (scenario,
// optimization) fit.  DESIGN.md §5.11; readings M1-M6.
//
// "an induction algorithm is used to construct a standard decision
// tree.  Then a multivariate regression model is constructed for each node
// ... only the features that appear in the subtree that contains the node are
// used ... the leaf nodes ... are replaced with the newly constructed
// regression models ... standard pruning and smoothing techniques are applied"
// (Quinlan's M5, [10]); constants S:219-228.
//
// Tree growth is decided by floating point (the SDR argmax, the sd stop rule):
// both sides take those decisions with the same IEEE operations in the same
// order (__d*_rn: no FMA contraction), over the same bit-identical scaled
// features and labels, so the grown tree is identical to the oracle's.  The
// node models are ridge LS (FP64 here, exact rationals in the oracle); the one
// decision they feed (pruning, M4) is counted as a guard case when it falls
// within guard_tol of its boundary (reading R21).
//
// Workspace: a per-warp slab of global scratch (L1/L2 resident), carved by
// M5Work.  Nodes are numbered in creation order; children have larger ids
// than their parent, so one ascending pass grows the tree (the order in which
// nodes are split does not change any node's result) and one descending pass
// is a valid post-order for the models and pruning.
#pragma once
#include "kernels.cuh"

namespace speedrec {

constexpr int kM5MinSplit = 4;        // M2: |T| < 4 -> leaf
constexpr double kM5SdFrac = 0.05;    // M2: sd(T) < 5 % of sd(root) -> leaf
constexpr double kM5SmoothK = 15.0;   // M5: Quinlan's smoothing constant
constexpr int kM5MaxFeatures = 64;    // allowed-feature sets are 64-bit masks
#ifndef SR_M5_UNROLL
#define SR_M5_UNROLL 2                // split-search row loops (A/B knob)
#endif

// Scratch doubles one warp needs for fits of <= np training pairs, <= d features.
__host__ __device__ inline long long m5_scratch_doubles(int np, int d) {
  const long long nn = np > 0 ? 2LL * np - 1 : 1;
  const long long pm = (d < np ? d : np) + 1;
  long long t = 2LL * np * d + np;                 // Xs, Xt, yt
  t += (2LL * np + 8 * nn + 1 + 64) / 2 + 1;       // perm, tmp, 8 node ints, feature list
  t += 3 * nn;                                     // thr, err, allowed
  t += nn * pm;                                    // model pool
  t += pm * (pm + 1) / 2 + 4 * pm + np;            // factor, invd, xbar, c, delta, residuals
  return t + 8;
}

struct M5Work {
  double* Xs;       // [n][ld] scaled training rows, kept in node-segment order
  double* Xt;       // [n][ld] partition staging
  double* yt;       // [n]
  int ld;
  double* thr;      // [nn]
  double* err;      // [nn]
  unsigned long long* allow;  // [nn] features split on in the (grown) subtree
  double* pool;     // models: b, w[popc(allow)]
  double* M;        // packed Cholesky factor
  double* invd;
  double* xbar;
  double* cv;
  double* dv;
  double* ev;       // [n]
  int *perm, *tmp, *nlo, *nhi, *feat, *left, *right, *par, *leaf, *moff, *fl;
};

__device__ __forceinline__ M5Work m5_carve(double* base, int np, int d) {
  M5Work W;
  const int nn = np > 0 ? 2 * np - 1 : 1;
  const int pm = (d < np ? d : np) + 1;
  double* p = base;
  W.Xs = p;
  W.ld = d;
  p += (long long)np * d;
  W.Xt = p;
  p += (long long)np * d;
  W.yt = p;
  p += np;
  W.thr = p;
  p += nn;
  W.err = p;
  p += nn;
  W.allow = reinterpret_cast<unsigned long long*>(p);
  p += nn;
  W.pool = p;
  p += (long long)nn * pm;
  W.M = p;
  p += (long long)pm * (pm + 1) / 2;
  W.invd = p;
  p += pm;
  W.xbar = p;
  p += pm;
  W.cv = p;
  p += pm;
  W.dv = p;
  p += pm;
  W.ev = p;
  p += np;
  int* q = reinterpret_cast<int*>(p);
  W.perm = q;
  q += np;
  W.tmp = q;
  q += np;
  W.nlo = q;
  q += nn;
  W.nhi = q;
  q += nn;
  W.feat = q;
  q += nn;
  W.left = q;
  q += nn;
  W.right = q;
  q += nn;
  W.par = q;
  q += nn;
  W.leaf = q;
  q += nn;
  W.moff = q;
  q += nn;
  W.fl = q;
  return W;
}

// Population sd of the labels y[lo, hi), two passes, left to right (M1).
__device__ __forceinline__ double m5_sd(int lo, int hi, const double* y) {
  double s = 0.0;
  for (int k = lo; k < hi; ++k) s = __dadd_rn(s, y[k]);
  const double cnt = (double)(hi - lo);
  const double m = __ddiv_rn(s, cnt);
  double q = 0.0;
  for (int k = lo; k < hi; ++k) {
    const double dv = __dsub_rn(y[k], m);
    q = __dadd_rn(q, __dmul_rn(dv, dv));
  }
  return __dsqrt_rn(__ddiv_rn(q, cnt));
}

__device__ __forceinline__ bool m5_better(double s, int a, double t, double bs, int ba, double bt) {
  return s > bs || (s == bs && (a < ba || (a == ba && t < bt)));
}

// Best split of node segment [lo, hi) (M1): lanes over features, candidates =
// midpoints between adjacent distinct values, key (SDR desc, feature asc,
// threshold asc) -- the oracle's first strict maximum in (feature, threshold)
// order.  Returns the SDR (-inf: no candidate); ba / bt the split.
//
// Row j's value u is a candidate's lower end iff it is its value's first
// occurrence and some value exceeds it; the threshold is (u + next)/2.  No
// value lies strictly between u and next, so "x <= u" is the same partition
// as "x <= threshold" whenever the rounded threshold is below next (always,
// unless u and next are adjacent doubles: then the pass is redone with the
// threshold itself, as the oracle compares): the first SDR pass (left/right label sums in segment
// order) runs fused with the distinct / next-greater scan, and the second
// (squared deviations) only for real candidates -- two O(m) passes per row
// instead of three, the same IEEE operations in the same order as the
// oracle's sd_pop over the filtered lists.
// Second SDR pass and score of one candidate (left sums sL, sR, count nL of
// the partition x <= cut), as the oracle's sd_pop of the two filtered lists.
__device__ __forceinline__ double m5_score(const double* xa, int ld, const double* yv, int m, double cut, double sL,
                                           double sR, int nL, const double* frac, double sdT) {
  const int nR = m - nL;
  const double mL = __ddiv_rn(sL, (double)nL), mR = __ddiv_rn(sR, (double)nR);
  double qL = 0.0, qR = 0.0;
SR_UNROLL(SR_M5_UNROLL)
  for (int k = 0; k < m; ++k) {
    const double v = xa[k * ld];
    const bool l = v <= cut;
    const double dv = __dsub_rn(yv[k], l ? mL : mR);
    const double t = __dadd_rn(l ? qL : qR, __dmul_rn(dv, dv));
    qL = l ? t : qL;
    qR = l ? qR : t;
  }
  const double sdL = __dsqrt_rn(__ddiv_rn(qL, (double)nL)), sdR = __dsqrt_rn(__ddiv_rn(qR, (double)nR));
  return __dsub_rn(__dsub_rn(sdT, __dmul_rn(frac[nL], sdL)), __dmul_rn(frac[nR], sdR));
}

// Candidate at row j (see m5_best_split): false if none; else its SDR and threshold.
__device__ __forceinline__ bool m5_candidate(const double* xa, int ld, const double* yv, int m, int j,
                                             const double* frac, double sdT, double& sdr, double& thr) {
  const double u = xa[j * ld];
  bool dup = false;
  double nx = INFINITY, sL = 0.0, sR = 0.0;
  int nL = 0;
SR_UNROLL(SR_M5_UNROLL)
  for (int k = 0; k < m; ++k) {
    const double v = xa[k * ld], yk = yv[k];
    dup |= (k < j) & (v == u);
    nx = (v > u && v < nx) ? v : nx;
    const bool l = v <= u;
    const double t = __dadd_rn(l ? sL : sR, yk);
    sL = l ? t : sL;
    sR = l ? sR : t;
    nL += l;
  }
  if (dup || nx == INFINITY) return false;
  thr = __dmul_rn(__dadd_rn(u, nx), 0.5);   // (lo + hi) / 2
  double cut = u;
  if (!(thr < nx)) {   // u, nx adjacent doubles and the midpoint rounded up: x <= thr takes nx too
    cut = thr;
    sL = sR = 0.0;
    nL = 0;
    for (int k = 0; k < m; ++k) {
      const bool l = xa[k * ld] <= cut;
      const double t = __dadd_rn(l ? sL : sR, yv[k]);
      sL = l ? t : sL;
      sR = l ? sR : t;
      nL += l;
    }
    if (nL == m) return false;   // unreachable for distinct finite values; keeps the sds defined
  }
  sdr = m5_score(xa, ld, yv, m, cut, sL, sR, nL, frac, sdT);
  return true;
}

// Large nodes (m > kM5WideRows): rows j and j + 1 share one fused first pass
// (two independent sum chains per row load); the second passes stay per
// candidate.  A candidate whose midpoint rounds up (adjacent doubles) is
// rescored by m5_candidate.
#ifndef SR_M5_WIDE_ROWS
#define SR_M5_WIDE_ROWS 32
#endif
constexpr int kM5WideRows = SR_M5_WIDE_ROWS;   // A/B knob

// A team of tw warps fitting the same tree (identical data in each warp's
// slab): the split search's candidates are dealt round-robin over the team and
// the best one is agreed through shared memory (xch: 3 doubles per warp of the
// CTA, team members contiguous; named barrier bar_id over the team's threads).
struct M5Team {
  int tw, trank, bar_id;
  double* xch;       // the team's first warp's slot
  unsigned long long* ops;   // this lane's count of executed split-search FP64 operations
};

__device__ __forceinline__ void m5_team_sync(const M5Team& T) {
  if (T.tw > 1) asm volatile("bar.sync %0, %1;" ::"r"(T.bar_id), "r"(T.tw * 32) : "memory");
}

// SOLO: a one-warp fit (stride-1 candidate loops, no team exchange).
template <bool SOLO>
__device__ double m5_best_split(const M5Work& W, int lo, int hi, int deff, const double* y, double sdT, int lane,
                                int& ba, double& bt, const M5Team& T) {
  const int tr = SOLO ? 0 : T.trank, ts = SOLO ? 1 : T.tw;
  double bs = -INFINITY;
  ba = 0x7fffffff;
  bt = INFINITY;
  const int m = hi - lo;
  const double* yv = y + lo;
  double* frac = W.ev;      // |L|/|T| = k/m for k < m (W.ev is free while the tree grows)
  for (int k = lane; k < m; k += 32) frac[k] = __ddiv_rn((double)k, (double)m);
  __syncwarp();
  for (int a = lane; a < deff; a += 32) {
    const double* xa = W.Xs + lo * W.ld + a;
    const int ld = W.ld;
    if (m <= kM5WideRows) {
      #pragma unroll 1
      for (int j = tr; j < m; j += ts) {
        double sdr, thr;
        const bool cand = m5_candidate(xa, ld, yv, m, j, frac, sdT, sdr, thr);
        *T.ops += (unsigned long long)(cand ? 4 * m : m);   // first pass m adds; a candidate's second 3m
        if (cand && m5_better(sdr, a, thr, bs, ba, bt)) {
          bs = sdr;
          ba = a;
          bt = thr;
        }
      }
      continue;
    }
    #pragma unroll 1
    for (int j = 2 * tr; j < m; j += 2 * ts) {
      const bool two = j + 1 < m;
      *T.ops += (unsigned long long)(2 * m);       // the fused first pass of rows j, j + 1
      const double u0 = xa[j * ld], u1 = two ? xa[(j + 1) * ld] : INFINITY;
      bool d0 = false, d1 = false;
      double n0 = INFINITY, n1 = INFINITY, sL0 = 0.0, sR0 = 0.0, sL1 = 0.0, sR1 = 0.0;
      int nL0 = 0, nL1 = 0;
SR_UNROLL(SR_M5_UNROLL)
      for (int k = 0; k < m; ++k) {
        const double v = xa[k * ld], yk = yv[k];
        d0 |= (k < j) & (v == u0);
        d1 |= (k < j + 1) & (v == u1);
        n0 = (v > u0 && v < n0) ? v : n0;
        n1 = (v > u1 && v < n1) ? v : n1;
        const bool l0 = v <= u0, l1 = v <= u1;
        const double t0 = __dadd_rn(l0 ? sL0 : sR0, yk), t1 = __dadd_rn(l1 ? sL1 : sR1, yk);
        sL0 = l0 ? t0 : sL0;
        sR0 = l0 ? sR0 : t0;
        sL1 = l1 ? t1 : sL1;
        sR1 = l1 ? sR1 : t1;
        nL0 += l0;
        nL1 += l1;
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double u = c ? u1 : u0, nx = c ? n1 : n0;
        if ((c ? d1 : d0) || nx == INFINITY) continue;
        double thr = __dmul_rn(__dadd_rn(u, nx), 0.5), sdr;
        if (thr < nx) {
          sdr = m5_score(xa, ld, yv, m, u, c ? sL1 : sL0, c ? sR1 : sR0, c ? nL1 : nL0, frac, sdT);
          *T.ops += (unsigned long long)(3 * m);
        } else if (!m5_candidate(xa, ld, yv, m, j + c, frac, sdT, sdr, thr)) {
          continue;
        } else {
          *T.ops += (unsigned long long)(5 * m);   // redo pass (m) + first (m) + second (3m)
        }
        if (m5_better(sdr, a, thr, bs, ba, bt)) {
          bs = sdr;
          ba = a;
          bt = thr;
        }
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double os = __shfl_xor_sync(FULL, bs, off), ot = __shfl_xor_sync(FULL, bt, off);
    const int oa = __shfl_xor_sync(FULL, ba, off);
    if (m5_better(os, oa, ot, bs, ba, bt)) {
      bs = os;
      ba = oa;
      bt = ot;
    }
  }
  if (!SOLO) {      // agree on the team's best candidate (same total order: any split of the work)
    if (lane == 0) {
      T.xch[3 * T.trank + 0] = bs;
      T.xch[3 * T.trank + 1] = (double)ba;
      T.xch[3 * T.trank + 2] = bt;
    }
    m5_team_sync(T);
    for (int r = 0; r < T.tw; ++r) {
      const double os = T.xch[3 * r + 0], ot = T.xch[3 * r + 2];
      const int oa = (int)T.xch[3 * r + 1];
      if (m5_better(os, oa, ot, bs, ba, bt)) {
        bs = os;
        ba = oa;
        bt = ot;
      }
    }
    m5_team_sync(T);   // the slots are free again
  }
  return bs;
}

// Stable partition of rows [lo, hi) by Xs[.][a] <= thr (left first, both
// halves in their original order, as the oracle's filtered index lists):
// the rows and labels move, so every node's rows stay contiguous.
__device__ int m5_partition(const M5Work& W, int lo, int hi, int a, double thr, double* y, int lane) {
  const unsigned lt = (1u << lane) - 1u;
  int nL = 0;
  for (int k0 = lo; k0 < hi; k0 += 32) {
    const int k = k0 + lane;
    const bool l = k < hi && W.Xs[k * W.ld + a] <= thr;
    nL += __popc(__ballot_sync(FULL, l));
  }
  int cl = 0, cr = 0;
  for (int k0 = lo; k0 < hi; k0 += 32) {
    const int k = k0 + lane;
    const bool in = k < hi;
    const bool l = in && W.Xs[k * W.ld + a] <= thr;
    const unsigned bl = __ballot_sync(FULL, l), br = __ballot_sync(FULL, in && !l);
    if (l) W.tmp[k] = lo + cl + __popc(bl & lt);
    else if (in) W.tmp[k] = lo + nL + cr + __popc(br & lt);
    cl += __popc(bl);
    cr += __popc(br);
  }
  __syncwarp();
  const int m = hi - lo, d = W.ld;
  for (int e = lane; e < m * d; e += 32) {
    const int r = e / d, c = e - r * d;
    W.Xt[W.tmp[lo + r] * d + c] = W.Xs[(lo + r) * d + c];
  }
  for (int k = lo + lane; k < hi; k += 32) W.yt[W.tmp[k]] = y[k];
  __syncwarp();
  for (int e = lane; e < m * d; e += 32) W.Xs[lo * d + e] = W.Xt[lo * d + e];
  for (int k = lo + lane; k < hi; k += 32) y[k] = W.yt[k];
  __syncwarp();
  return nL;
}

// Model value b + sum_j w_j x_fl[j] (ascending feature order, M3) on a scaled
// training row.
__device__ __forceinline__ double m5_row_value(const M5Work& W, const double* mdl, unsigned long long al,
                                               const double* xs) {
  double s = 0.0;
  int j = 0;
  while (al) {
    const int a = __ffsll((long long)al) - 1;
    al &= al - 1;
    s = fma(mdl[1 + j], xs[a], s);
    ++j;
  }
  return mdl[0] + s;
}

// Node model (M3): ridge LS over rows [lo, hi) on the features of `al`,
// intercept unpenalised: centred normal equations (X_c'X_c + lambda I) w =
// X_c'y_c by Cholesky, nref refinement steps from the rows, b = ybar - w.xbar.
// Writes b, w into mdl; returns false if the factorisation broke down.
__device__ bool m5_node_fit(const M5Work& W, int lo, int hi, unsigned long long al, const double* y, double lambda,
                            int nref, double* mdl, int lane) {
  const int m = hi - lo;
  const int p = __popcll(al);
  if (lane == 0) {
    unsigned long long t = al;
    for (int j = 0; j < p; ++j) {
      W.fl[j] = __ffsll((long long)t) - 1;
      t &= t - 1;
    }
  }
  double ys = 0.0;
  for (int k = lo + lane; k < hi; k += 32) ys += y[k];
  const double ybar = warp_sum(ys) / (double)m;
  __syncwarp();
  if (p == 0) {
    if (lane == 0) mdl[0] = ybar;
    __syncwarp();
    return true;
  }
  for (int j = lane; j < p; j += 32) {
    const int a = W.fl[j];
    double s = 0.0;
    for (int k = lo; k < hi; ++k) s += W.Xs[k * W.ld + a];
    W.xbar[j] = s / (double)m;
  }
  __syncwarp();
  const int ne = p * (p + 1) / 2;
  auto tri = [](int e, int& i, int& j) {     // packed lower-triangle index -> (i, j)
    i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    while (i * (i + 1) / 2 > e) --i;
    j = e - i * (i + 1) / 2;
  };
  // two entries per lane pass (e, e + 32): two independent FMA chains over the
  // rows, each entry's own chain in row order as before (same rounding)
  for (int e0 = lane; e0 < ne; e0 += 64) {
    const int e1 = e0 + 32;
    const bool two = e1 < ne;
    int i0, j0, i1, j1;
    tri(e0, i0, j0);
    if (two) tri(e1, i1, j1);
    else i1 = i0, j1 = j0;
    const int a0 = W.fl[i0], b0 = W.fl[j0], a1 = W.fl[two ? i1 : i0], b1 = W.fl[two ? j1 : j0];
    const double x0 = W.xbar[i0], y0 = W.xbar[j0], x1 = W.xbar[two ? i1 : i0], y1 = W.xbar[two ? j1 : j0];
    double s0 = 0.0, s1 = 0.0;
    for (int k = lo; k < hi; ++k) {
      const double* xr = W.Xs + k * W.ld;
      s0 = fma(xr[a0] - x0, xr[b0] - y0, s0);
      s1 = fma(xr[a1] - x1, xr[b1] - y1, s1);
    }
    W.M[e0] = s0 + (i0 == j0 ? lambda : 0.0);
    if (two) W.M[e1] = s1 + (i1 == j1 ? lambda : 0.0);
  }
  for (int j = lane; j < p; j += 32) {
    const int a = W.fl[j];
    const double xj = W.xbar[j];
    double s = 0.0;
    for (int k = lo; k < hi; ++k) {
      const int r = k;
      s = fma(W.Xs[r * W.ld + a] - xj, y[r] - ybar, s);
    }
    W.cv[j] = s;
  }
  __syncwarp();
  if (!chol_packed(W.M, W.invd, p, lane)) return false;
  chol_solve(W.M, W.invd, W.cv, p, lane);     // cv <- w
  for (int it = 0; it < nref; ++it) {
    for (int k = lo + lane; k < hi; k += 32) {   // residual of the centred system
      const int r = k;
      const double* xr = W.Xs + r * W.ld;
      double s = y[r] - ybar;
      for (int j = 0; j < p; ++j) s = fma(-(xr[W.fl[j]] - W.xbar[j]), W.cv[j], s);
      W.ev[k - lo] = s;
    }
    __syncwarp();
    for (int j = lane; j < p; j += 32) {
      const int a = W.fl[j];
      const double xj = W.xbar[j];
      double s = -lambda * W.cv[j];
      for (int k = lo; k < hi; ++k) s = fma(W.Xs[k * W.ld + a] - xj, W.ev[k - lo], s);
      W.dv[j] = s;
    }
    __syncwarp();
    chol_solve(W.M, W.invd, W.dv, p, lane);
    for (int j = lane; j < p; j += 32) W.cv[j] += W.dv[j];
    __syncwarp();
  }
  double bp = 0.0;
  for (int j = lane; j < p; j += 32) bp = fma(W.cv[j], W.xbar[j], bp);
  const double b = ybar - warp_sum(bp);
  for (int j = lane; j < p; j += 32) mdl[1 + j] = W.cv[j];
  if (lane == 0) mdl[0] = b;
  __syncwarp();
  return true;
}

// Grow (M1, M2), fit + prune (M3, M4) the tree of one fit: n training rows
// (scaled in W.Xs, labels y), deff features.  Returns the node count; *guard
// gets the pruning decisions within tol of their boundary; *ok false if a
// node factorisation broke down.
__device__ int m5_build(const M5Work& W, int n, int deff, double* y, double lambda, int nref, double tol,
                        int lane, int* guard, bool* ok, const M5Team& T) {
  if (lane == 0) {
    W.nlo[0] = 0;
    W.nhi[0] = n;
    W.par[0] = -1;
  }
  __syncwarp();
  const double sd_root = m5_sd(0, n, y);
  const double sd_min = __dmul_rn(kM5SdFrac, sd_root);
  int nn = 1;
  SR_M5T(-1);
  #pragma unroll 1
  for (int i = 0; i < nn; ++i) {
    const int lo = W.nlo[i], hi = W.nhi[i];
    bool split = false;
    int ba = 0;
    double bt = 0.0;
    if (hi - lo >= kM5MinSplit) {
      const double sdT = m5_sd(lo, hi, y);
      if (!(sdT < sd_min))
        split = (T.tw == 1 ? m5_best_split<true>(W, lo, hi, deff, y, sdT, lane, ba, bt, T)
                           : m5_best_split<false>(W, lo, hi, deff, y, sdT, lane, ba, bt, T)) > 0.0;
    }
    SR_M5T(0);
    if (split) {
      const int nL = m5_partition(W, lo, hi, ba, bt, y, lane);
      SR_M5T(1);
      if (lane == 0) {
        W.feat[i] = ba;
        W.thr[i] = bt;
        W.left[i] = nn;
        W.right[i] = nn + 1;
        W.nlo[nn] = lo;
        W.nhi[nn] = lo + nL;
        W.par[nn] = i;
        W.nlo[nn + 1] = lo + nL;
        W.nhi[nn + 1] = hi;
        W.par[nn + 1] = i;
      }
      nn += 2;
    }
    if (lane == 0) W.leaf[i] = split ? 0 : 1;
    __syncwarp();
  }
  // allowed features (M3: split features of the grown subtree), pool offsets
  if (lane == 0) {
    for (int i = nn - 1; i >= 0; --i)
      W.allow[i] = W.leaf[i] ? 0ull : (1ull << W.feat[i]) | W.allow[W.left[i]] | W.allow[W.right[i]];
    int off = 0;
    for (int i = 0; i < nn; ++i) {
      W.moff[i] = off;
      off += 1 + __popcll(W.allow[i]);
    }
  }
  __syncwarp();
  // models + pruning, post-order (M3, M4)
  int g = 0;
  bool good = true;
  #pragma unroll 1
  for (int i = nn - 1; i >= 0; --i) {
    const int lo = W.nlo[i], hi = W.nhi[i], m = hi - lo;
    const unsigned long long al = W.allow[i];
    double* mdl = W.pool + W.moff[i];
    SR_M5T(-1);
    good &= m5_node_fit(W, lo, hi, al, y, lambda, nref, mdl, lane);
    SR_M5T(2);
    double rs = 0.0;
    for (int k = lo + lane; k < hi; k += 32) {
      const int r = k;
      rs += fabs(y[r] - m5_row_value(W, mdl, al, W.Xs + r * W.ld));
    }
    const double resid = warp_sum(rs) / (double)m;
    const int v = __popcll(al) + 1;
    const double f = m > v ? (double)(m + v) / (double)(m - v) : 10.0;
    const double own = resid * f;
    if (lane == 0) {
      if (W.leaf[i]) {
        W.err[i] = own;
      } else {
        const int L = W.left[i], R = W.right[i];
        const double sub = ((double)(W.nhi[L] - W.nlo[L]) * W.err[L] + (double)(W.nhi[R] - W.nlo[R]) * W.err[R]) /
                           (double)m;
        if (near_tol(own, sub, tol)) ++g;
        if (own <= sub) {
          W.leaf[i] = 1;     // prune to the node's model
          W.err[i] = own;
        } else {
          W.err[i] = sub;
        }
      }
    }
    __syncwarp();
    SR_M5T(3);
  }
  *guard = __shfl_sync(FULL, g, 0);
  *ok = good;
  return nn;
}

// Value of node i's model at a raw test row xq (scaled on the fly exactly as
// the training rows: (x - mn) / rg, reading D3).
__device__ __forceinline__ double m5_test_value(const M5Work& W, int i, const double* xq, const int16_t* col,
                                                const double* mnv, const double* rgv) {
  const double* mdl = W.pool + W.moff[i];
  unsigned long long al = W.allow[i];
  double s = 0.0;
  int j = 0;
  while (al) {
    const int a = __ffsll((long long)al) - 1;
    al &= al - 1;
    s = fma(mdl[1 + j], (xq[col[a]] - mnv[a]) / rgv[a], s);
    ++j;
  }
  return mdl[0] + s;
}

// M5P prediction (M5): route x (x' <= thr left) to a leaf of the
// pruned tree, then smooth root-ward p <- (n p + k q)/(n + k), n the count of
// the node p came from, k = 15.
__device__ double m5_predict(const M5Work& W, const double* xq, const int16_t* col, const double* mnv,
                             const double* rgv) {
  int i = 0;
  while (!W.leaf[i]) {
    const int a = W.feat[i];
    const double xs = (xq[col[a]] - mnv[a]) / rgv[a];
    i = xs <= W.thr[i] ? W.left[i] : W.right[i];
  }
  double p = m5_test_value(W, i, xq, col, mnv, rgv);
  int nb = W.nhi[i] - W.nlo[i];
  for (int a = W.par[i]; a >= 0; a = W.par[a]) {
    const double q = m5_test_value(W, a, xq, col, mnv, rgv);
    p = ((double)nb * p + kM5SmoothK * q) / ((double)nb + kM5SmoothK);
    nb = W.nhi[a] - W.nlo[a];
  }
  return p;
}

}  // namespace speedrec
