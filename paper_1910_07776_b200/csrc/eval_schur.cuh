// eval_schur.cuh -- prefix-shared feature-mask path (config C5 at scale).
// DESIGN.md §5.8.
//
// The fit of (mask M, fold, opt) is the Cholesky of the principal submatrix
// G_MM + lambda I of the fold's full-feature Gram (eval_masks.cuh), in
// increasing counter order.  Split the counters [0, K) used by the batch into
// a prefix [0, T) and a suffix [T, K) of U <= 10 counters; M = P u S.  In that
// elimination order the prefix block is factored first, and block elimination
// gives, exactly in real arithmetic,
//   EX - ybar = y_P.u_P + y~_S.u~_S,
//   y_P = L_P^-1 r_P, u_P = L_P^-1 z_P, V = L_P^-1 G_P,suffix,
//   Schur  Q = G_suffix,suffix + lambda I - V^T V,
//   r~ = r_suffix - V^T y_P, z~ = z_suffix - V^T u_P,
// and (y~_S, u~_S) are the same forward solves on the principal submatrix
// Q_SS.  So one record per (prefix, fold, opt) -- Q (U x U), r~, z~, y_P.u_P
// -- serves the 2^U masks that share the prefix; each of them then needs only
// a |S| <= 10 factorisation (SURVEY §8(d) "allowed shortcuts": mask-
// independent precomputation, per-fold ranges respected, reported as an
// effective fraction).
//
//  k_mask_sprep  thread per (prefix group, fold, opt): prefix factor with the
//                r, z and suffix columns carried as augmented rows, Schur
//                complement -> record.
//  k_mask_sfit<D> thread per mask (and fold range when the launch has few
//                masks), one launch per suffix size D: the D x D system in
//                registers, records through L1 (a CTA's masks share the
//                prefix), EX, clamp, score, rank / recommend, per-scenario
//                rows when asked, per-mask sums.
#pragma once
#include <type_traits>

#include "eval_masks.cuh"

namespace speedrec {

constexpr int kSchurU = 10;                 // suffix counters (register system size)
constexpr int kSfitMaxO = 6;                // optimization ids of the prefix-shared path (the paper's six)
constexpr int kSchurT = 12;                 // largest prefix (counters before the suffix)
constexpr int kSchurQ = kSchurU * (kSchurU + 1) / 2;
constexpr int kRec = 80;                    // doubles per record: Q[55] r~[10] z~[10] base flags pad
constexpr int kRecR = kSchurQ, kRecZ = kSchurQ + kSchurU, kRecBase = kSchurQ + 2 * kSchurU, kRecFlag = kRecBase + 1;
#ifndef SPEEDREC_SFIT_THREADS
#define SPEEDREC_SFIT_THREADS 256
#endif
constexpr int kSfitThreads = SPEEDREC_SFIT_THREADS;
#ifndef SPEEDREC_SFIT_PROBE        // timing probes (1 no factorization, 2 no ranking): wrong results
#define SPEEDREC_SFIT_PROBE 0
#endif
#ifndef SPEEDREC_SFIT_NBUF         // record buffers of the staged fold loop
#define SPEEDREC_SFIT_NBUF 3
#endif
#ifndef SPEEDREC_SFIT_ILP_D        // suffix sizes below this let the compiler interleave optimisations
#define SPEEDREC_SFIT_ILP_D 0
#endif
#ifndef SPEEDREC_SFIT_SCHED        // A/B knob: register budget schedule of k_mask_sfit<D>
#define SPEEDREC_SFIT_SCHED 0
#endif
#ifndef SPEEDREC_SFIT_MINB        // CTAs per SM the register budget of k_mask_sfit<D> targets
#if SPEEDREC_SFIT_SCHED == 1
#define SPEEDREC_SFIT_MINB(D) ((D) <= 2 ? 4 : (D) <= 8 ? 2 : 1)
#elif SPEEDREC_SFIT_SCHED == 2
#define SPEEDREC_SFIT_MINB(D) ((D) <= 1 ? 4 : (D) <= 8 ? 2 : 1)
#else
#define SPEEDREC_SFIT_MINB(D) ((D) <= 3 ? 4 : (D) <= 8 ? 2 : 1)
#endif
#endif

struct SchurArgs {
  MaskArgs M;
  int T, U;
  const uint32_t* pfx;      // [n_groups] prefix bits of each group
  int n_groups;
  double* rec;              // [n_groups][S][O][kRec]
  const int32_t* order;     // local mask indices sorted by (suffix popcount, prefix, suffix)
  const int32_t* group;     // prefix group of each sorted item
};

// ------------------------------------------------------------------ prep
static __global__ void __launch_bounds__(128) k_mask_sprep(const SchurArgs SA) {
  const MaskArgs& M = SA.M;
  const long long S = M.sd.n_splits;
  const int O = M.O, C = M.C, T = SA.T, U = SA.U;
  const long long item = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= (long long)SA.n_groups * S * O) return;
  const int o = (int)(item % O);
  const long long split = (item / O) % S;
  const int j = (int)(item / (O * S));
  double* R = SA.rec + item * kRec;
  const PrepMeta pm = M.pm[split * O + o];
  if (pm.n <= 0) {
    R[kRecFlag] = 0.0;
    return;
  }
  const long long it = split * O + o;
  const double* Gm = M.pG + it * C * C;
  const double* rv = M.pr + it * C;
  const double* zv = M.pz + it * C;
  const uint32_t act = (uint32_t)pm.active;
  // prefix features (counter order), active only
  int pf[kSchurT];
  int p = 0;
  {
    uint32_t mm = SA.pfx[j] & act & ((1u << T) - 1u);
    while (mm) {
      pf[p++] = __ffs(mm) - 1;
      mm &= mm - 1u;
    }
  }
  double L[kSchurT * (kSchurT + 1) / 2], V[kSchurU][kSchurT], yv[kSchurT], uv[kSchurT];
  for (int i = 0; i < p; ++i) {
    for (int k = 0; k <= i; ++k) L[i * (i + 1) / 2 + k] = Gm[pf[i] * C + pf[k]] + (i == k ? M.lambda : 0.0);
    yv[i] = rv[pf[i]];
    uv[i] = zv[pf[i]];
    for (int b = 0; b < U; ++b) V[b][i] = Gm[(T + b) * C + pf[i]];
  }
  // left-looking column steps; rows of r, z and the suffix columns ride along
  bool ok = true;
  for (int c = 0; c < p; ++c) {
    const int jc = c * (c + 1) / 2;
    double d = L[jc + c];
    for (int k = 0; k < c; ++k) d = fma(-L[jc + k], L[jc + k], d);
    ok &= d > 0.0;
    const double r = rsqrt_nr(d);
    L[jc + c] = r;                                   // diagonal holds 1/L_cc
    for (int i = c + 1; i < p; ++i) {
      const int ji = i * (i + 1) / 2;
      double a = L[ji + c];
      for (int k = 0; k < c; ++k) a = fma(-L[ji + k], L[jc + k], a);
      L[ji + c] = a * r;
    }
    double a = yv[c], e = uv[c];
    for (int k = 0; k < c; ++k) {
      a = fma(-yv[k], L[jc + k], a);
      e = fma(-uv[k], L[jc + k], e);
    }
    yv[c] = a * r;
    uv[c] = e * r;
    for (int b = 0; b < U; ++b) {
      double v = V[b][c];
      for (int k = 0; k < c; ++k) v = fma(-V[b][k], L[jc + k], v);
      V[b][c] = v * r;
    }
  }
  double base = 0.0;
  for (int k = 0; k < p; ++k) base = fma(yv[k], uv[k], base);
  for (int b = 0; b < U; ++b) {
    for (int c = 0; c <= b; ++c) {
      double q = Gm[(T + b) * C + (T + c)] + (b == c ? M.lambda : 0.0);
      for (int k = 0; k < p; ++k) q = fma(-V[b][k], V[c][k], q);
      R[b * (b + 1) / 2 + c] = q;
    }
    double a = rv[T + b], e = zv[T + b];
    for (int k = 0; k < p; ++k) {
      a = fma(-V[b][k], yv[k], a);
      e = fma(-V[b][k], uv[k], e);
    }
    R[kRecR + b] = a;
    R[kRecZ + b] = e;
  }
  R[kRecBase] = base;
  const unsigned long long flags = 1ull | ((unsigned long long)((act >> T) & ((1u << U) - 1u)) << 8) |
                                   (ok ? 0ull : 2ull);
  R[kRecFlag] = __longlong_as_double((long long)flags);
}

// k_mask_sprep_p<P>: the same record for groups whose prefix has P counters,
// everything in registers (compile-time sizes).  Inactive prefix counters
// stay in the factor: their G row and column, r and z are exactly zero, so
// their pivot is lambda and every quantity they touch gets exact zeros --
// the record equals the one without them (D3).  glist: the launch's groups.
template <int P>
__global__ void __launch_bounds__(128) k_mask_sprep_p(const SchurArgs SA, const int32_t* glist, int ng) {
  const MaskArgs& M = SA.M;
  const long long S = M.sd.n_splits;
  const int O = M.O, C = M.C, T = SA.T, U = SA.U;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)ng * S * O) return;
  const int o = (int)(idx % O);
  const long long split = (idx / O) % S;
  const int j = glist[idx / (O * S)];
  const long long item = ((long long)j * S + split) * O + o;
  double* R = SA.rec + item * kRec;
  const PrepMeta pm = M.pm[split * O + o];
  if (pm.n <= 0) {
    R[kRecFlag] = 0.0;
    return;
  }
  const double* Gm = M.pG + (split * O + o) * C * C;
  const double* rv = M.pr + (split * O + o) * C;
  const double* zv = M.pz + (split * O + o) * C;
  const uint32_t act = (uint32_t)pm.active;
  int pf[P > 0 ? P : 1];
  {
    uint32_t mm = SA.pfx[j] & ((1u << T) - 1u);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      pf[i] = __ffs(mm) - 1;
      mm &= mm - 1u;
    }
  }
  double L[P * (P + 1) / 2 + 1], V[kSchurU][P > 0 ? P : 1], yv[P > 0 ? P : 1], uv[P > 0 ? P : 1];
#pragma unroll
  for (int i = 0; i < P; ++i) {
#pragma unroll
    for (int k = 0; k <= i; ++k) L[i * (i + 1) / 2 + k] = Gm[pf[i] * C + pf[k]] + (i == k ? M.lambda : 0.0);
    yv[i] = rv[pf[i]];
    uv[i] = zv[pf[i]];
#pragma unroll
    for (int b = 0; b < kSchurU; ++b) V[b][i] = b < U ? Gm[(T + b) * C + pf[i]] : 0.0;
  }
  bool ok = true;
#pragma unroll
  for (int c = 0; c < P; ++c) {
    constexpr int dummy = 0;
    (void)dummy;
    const int jc = c * (c + 1) / 2;
    double d = L[jc + c];
#pragma unroll
    for (int k = 0; k < c; ++k) d = fma(-L[jc + k], L[jc + k], d);
    ok &= d > 0.0;
    const double r = rsqrt_nr(d);
    L[jc + c] = r;
#pragma unroll
    for (int i = c + 1; i < P; ++i) {
      const int ji = i * (i + 1) / 2;
      double a = L[ji + c];
#pragma unroll
      for (int k = 0; k < c; ++k) a = fma(-L[ji + k], L[jc + k], a);
      L[ji + c] = a * r;
    }
    double a = yv[c], e = uv[c];
#pragma unroll
    for (int k = 0; k < c; ++k) {
      a = fma(-yv[k], L[jc + k], a);
      e = fma(-uv[k], L[jc + k], e);
    }
    yv[c] = a * r;
    uv[c] = e * r;
#pragma unroll
    for (int b = 0; b < kSchurU; ++b) {
      double v = V[b][c];
#pragma unroll
      for (int k = 0; k < c; ++k) v = fma(-V[b][k], L[jc + k], v);
      V[b][c] = v * r;
    }
  }
  double base = 0.0;
#pragma unroll
  for (int k = 0; k < P; ++k) base = fma(yv[k], uv[k], base);
#pragma unroll
  for (int b = 0; b < kSchurU; ++b) {
    if (b >= U) break;
#pragma unroll
    for (int c = 0; c <= b; ++c) {
      double q = Gm[(T + b) * C + (T + c)] + (b == c ? M.lambda : 0.0);
#pragma unroll
      for (int k = 0; k < P; ++k) q = fma(-V[b][k], V[c][k], q);
      R[b * (b + 1) / 2 + c] = q;
    }
    double a = rv[T + b], e = zv[T + b];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      a = fma(-V[b][k], yv[k], a);
      e = fma(-V[b][k], uv[k], e);
    }
    R[kRecR + b] = a;
    R[kRecZ + b] = e;
  }
  R[kRecBase] = base;
  const unsigned long long flags = 1ull | ((unsigned long long)((act >> T) & ((1u << U) - 1u)) << 8) |
                                   (ok ? 0ull : 2ull);
  R[kRecFlag] = __longlong_as_double((long long)flags);
}

// EX - ybar - base of one suffix system of compile-time size D from a staged
// record: gather Q_SS (f ascending, so the packed lower layout is preserved),
// factor with r~ and z~ carried as augmented rows, y~.u~.
// SM: the record is staged in shared memory (plain loads), else read through
// the read-only path (__ldg).
template <bool SM>
__device__ __forceinline__ double rec_ld(const double* p) { return SM ? *p : __ldg(p); }

template <int D, bool SM = false>
__device__ __forceinline__ double schur_fit(const double* R, const int* f, bool& ok) {
  if (D == 0) return 0.0;
  constexpr int TT = D * (D + 1) / 2;
  double L[TT + 2 * D + 1];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const int fi = f[i], bi = fi * (fi + 1) / 2;
#pragma unroll
    for (int k = 0; k <= i; ++k) L[i * (i + 1) / 2 + k] = rec_ld<SM>(R + bi + f[k]);
    L[TT + i] = rec_ld<SM>(R + kRecR + fi);
    L[TT + D + i] = rec_ld<SM>(R + kRecZ + fi);
  }
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double djj = L[j * (j + 1) / 2 + j];
#pragma unroll
    for (int k = 0; k < j; ++k) djj = fma(-L[j * (j + 1) / 2 + k], L[j * (j + 1) / 2 + k], djj);
    ok &= djj > 0.0;
    const double r = rsqrt_nr(djj);
#pragma unroll
    for (int i = j + 1; i < D + 2; ++i) {
      const int ri = i < D ? i * (i + 1) / 2 : TT + (i - D) * D;
      double a = L[ri + j];
#pragma unroll
      for (int k = 0; k < j; ++k) a = fma(-L[ri + k], L[j * (j + 1) / 2 + k], a);
      L[ri + j] = a * r;
    }
  }
  double e = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) e = fma(L[TT + i], L[TT + D + i], e);
  return e;
}

// ------------------------------------------------------------------ fit
// k_mask_sfit<D>: thread per mask (times fold chunk) for the masks whose
// active suffix has D counters; records read through L1 (the threads of a
// CTA mostly share the prefix, so a fold's O records stay cache-resident).
template <int D>
__global__ void __launch_bounds__(kSfitThreads, SPEEDREC_SFIT_MINB(D)) k_mask_sfit(const SchurArgs SA, int off, int n_items, int fold_chunks) {
  const MaskArgs& M = SA.M;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int O = M.O, G = M.G, T = SA.T;
  const long long S = M.sd.n_splits;
  unsigned long long t_corr = 0, t_test = 0, t_rec = 0, t_hit = 0;
  const int item = tid % n_items, chunk = tid / n_items;
  const bool active = chunk < fold_chunks;
  // Records through shared memory (CTA-uniform decision): when every thread of
  // the CTA evaluates all folds of masks sharing ONE prefix group, a fold's O
  // records (contiguous, O x 640 B) arrive by one TMA bulk copy, double
  // buffered one fold ahead on an mbarrier; otherwise they are gathered
  // through L1 (__ldg).
  // up to two prefix groups per CTA (a CTA of 256 sorted masks spans at most
  // two groups for suffix sizes 3..7, the large launches)
  constexpr int NB = SPEEDREC_SFIT_NBUF;            // fold buffers (prefetch distance NB - 1)
  __shared__ __align__(16) double srec[NB][2][kSfitMaxO * kRec];
  __shared__ __align__(8) uint64_t sbar[NB];
  const int i0 = blockIdx.x * blockDim.x, ilast = min(i0 + (int)blockDim.x, n_items) - 1;
  const int g0 = i0 < n_items ? SA.group[off + i0] : 0, g1 = i0 < n_items ? SA.group[off + ilast] : 0;
  const bool staged = fold_chunks == 1 && i0 < n_items && g1 - g0 <= 1;
  const int ml = active ? SA.order[off + item] : 0;
  const int grp = active ? SA.group[off + item] : 0;
  const long long fidx = M.mask0 + ml;
  const uint32_t sfx = active ? (mask_bits(M.sd, fidx) >> T) & ((1u << SA.U) - 1u) : 0u;
  int f[D > 0 ? D : 1];
  {
    uint32_t mm = sfx;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      f[i] = mm ? __ffs(mm) - 1 : 0;
      mm &= mm - 1u;
    }
  }
  int s_corr = 0, s_test = 0, s_rec = 0, s_hit = 0;
  const double* recg = SA.rec + (long long)grp * S * O * kRec;
  // one fold of this thread's mask; SM: the fold's records are in shared memory at Rb
  // (one code path: generic loads serve both shared and global records)
  auto fold = [&](int split, const double* Rb) {
    constexpr bool SM = true;
    const long long sl = fidx * S + split - M.first;
    const uint32_t om = scored_mask(M.sd, split, O);
    const int g = M.sd.pool_list[split >> 6], v = split & 63;
    double ce[kSfitMaxO];
    bool cv[kSfitMaxO], cc[kSfitMaxO], hit[kSfitMaxO];   // hit: AC > 1 (the held-out case's own label)
    int guard = 0, untrained = 0;
#pragma unroll
    for (int o = 0; o < kSfitMaxO; ++o) {
      cv[o] = cc[o] = hit[o] = false;
      ce[o] = 0.0;
      if (o >= O) continue;
      // one optimisation at a time (no load hoisting across them) for the larger
      // systems; the small ones may interleave two fits' pivot chains
      if (D >= SPEEDREC_SFIT_ILP_D) asm volatile("" ::: "memory");
      const PrepMeta& pm = M.pm[split * O + o];
      OptScore row;
      row.n_train = row.n_test = row.n_correct = row.n_clamped = 0;
      row.sum_ratio = row.min_ratio = row.max_ratio = 0.0;
      row.fp_train = row.fp_test = 0ull;
      const int n = pm.n;
      if (n >= 0 && ((om >> o) & 1u)) {
        row.n_train = n;
        row.n_test = pm.nt;
        row.fp_train = pm.fp_tr;
        row.fp_test = pm.fp_te;
        s_test += pm.nt;
        if (n == 0 && pm.nt > 0) ++untrained;
        if (n > 0 && pm.nt > 0) {
          const double* R = Rb + o * kRec;
          const unsigned long long flags = (unsigned long long)__double_as_longlong(rec_ld<SM>(R + kRecFlag));
          bool ok = (flags & 2ull) == 0ull;
          // an inactive suffix counter (rg = 0 in this fold) has a zero row and
          // column in Q and zero r~, z~: its pivot is lambda and it adds exact
          // zeros, so the fit equals the one without it (reading D3)
#if SPEEDREC_SFIT_PROBE == 1   // timing probe only (wrong results): no suffix factorization
          double e = pm.ybar + rec_ld<SM>(R + kRecBase) + rec_ld<SM>(R + f[0]);
#else
          double e = pm.ybar + rec_ld<SM>(R + kRecBase) + schur_fit<D, SM>(R, f, ok);
#endif
          if (!ok) {
            e = pm.ybar;
            guard += 1000000;
          }
          if (near_tol(e, 0.0, M.guard_tol) || near_tol(e, 1.0, M.guard_tol)) ++guard;
          bool cl = false;
          if (e <= 0.0) {
            e = M.clamp_floor;
            cl = true;
          }
          const double ac = pm.ac;
          const int corr = ((e > 1.0 && ac > 1.0) || (e <= 1.0 && ac <= 1.0)) ? 1 : 0;
          const double ratio = ac / e;
          row.n_correct = corr;
          row.n_clamped = cl ? 1 : 0;
          row.sum_ratio = row.min_ratio = row.max_ratio = ratio;
          s_corr += corr;
          t_corr += corr;
          t_test += 1;
          cv[o] = true;
          hit[o] = ac > 1.0;
          cc[o] = cl;
          ce[o] = e;
          if (M.ex_out) M.ex_out[(sl * O + o) * (long long)G * 32 + pm.tek] = e;
        }
      }
      if (M.opt_out) M.opt_out[sl * O + o] = row;
    }
#if SPEEDREC_SFIT_PROBE == 2   // timing probe only (wrong results): no guard / ranking rules
    int nrec = cv[0] ? 1 : 0, nhit = cc[1] ? 1 : 0;
    (void)ce;
    (void)hit;
#else
    // A6: rank the held-out version's candidates (R13, R21), one pass
    // over the 15 candidate pairs: the guard band of R21 (near_tol with the
    // first one's scale, as k_rank_warp) and the rank order (EX desc, id asc:
    // for a < b, b outranks a iff EX_b > EX_a) of those at or above the
    // threshold.  A recommendation's hit is its own held-out label AC > 1.
    double ta[kSfitMaxO];
    unsigned left = 0u;
    int rk[kSfitMaxO];
#pragma unroll
    for (int a = 0; a < kSfitMaxO; ++a) {
      rk[a] = 0;
      ta[a] = M.guard_tol * (fabs(ce[a]) > 1.0 ? fabs(ce[a]) : 1.0);   // near_tol(ce[a], .)
      if (!cv[a]) continue;
      if (fabs(ce[a] - M.threshold) <= ta[a]) ++guard;
      if (ce[a] >= M.threshold) left |= 1u << a;
    }
#pragma unroll
    for (int a = 0; a < kSfitMaxO; ++a) {
#pragma unroll
      for (int b = a + 1; b < kSfitMaxO; ++b) {
        if (!(cv[a] && cv[b])) continue;
        if (!(cc[a] && cc[b]) && fabs(ce[a] - ce[b]) <= ta[a]) ++guard;
        if (((left >> a) & (left >> b) & 1u) != 0u) {
          if (ce[b] > ce[a]) ++rk[a];
          else ++rk[b];
        }
      }
    }
    int nrec = 0, nhit = 0;
#pragma unroll
    for (int a = 0; a < kSfitMaxO; ++a) {
      if (!((left >> a) & 1u) || rk[a] >= M.max_count) continue;
      ++nrec;
      if (hit[a]) ++nhit;
      if (M.rec_out) M.rec_out[(sl * G * 64 + g * 64 + v) * M.max_count + rk[a]] = (int8_t)a;
    }
#endif
    s_rec += nrec;
    s_hit += nhit;
    t_rec += nrec;
    t_hit += nhit;
    if (M.scn_out) {
      ScnScore sr;
      sr.n_rec = nrec;
      sr.n_rec_hit = nhit;
      sr.n_untrained = untrained;
      sr.n_guard = guard;
      M.scn_out[sl] = sr;
    }
  };
  if (staged) {
    const unsigned bytes = (unsigned)(O * kRec * 8);
    const int ng = g1 - g0 + 1;                      // 1 or 2 groups
    const double* gsrc = SA.rec + (long long)g0 * S * O * kRec;
    const long long gstride = S * O * kRec;
    auto issue = [&](int split, int b) {            // the fold's records of the CTA's groups -> buffer b
      mbar_expect_tx(&sbar[b], ng * bytes);
      for (int q = 0; q < ng; ++q) bulk_g2s_tx(srec[b][q], gsrc + q * gstride + (long long)split * O * kRec, bytes, &sbar[b]);
    };
    if (threadIdx.x == 0) {
      for (int q = 0; q < NB; ++q) mbar_init(&sbar[q], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < NB - 1 && q < S; ++q) issue(q, q);
    unsigned phase = 0u;
    const int mine = grp - g0;
    #pragma unroll 1
    for (int split = 0; split < (int)S; ++split) {
      const int b = split % NB;
      if (threadIdx.x == 0 && split + NB - 1 < S) {  // fold split+NB-1 (its buffer was freed by the last barrier)
        fence_proxy_async();
        issue(split + NB - 1, (split + NB - 1) % NB);
      }
      mbar_wait(&sbar[b], (phase >> b) & 1u);
      phase ^= 1u << b;
      if (active) fold(split, srec[b][mine]);
      __syncthreads();                               // every thread is done with buffer b
    }
  } else if (active) {
    const int s0 = (int)(S * chunk / fold_chunks), s1 = (int)(S * (chunk + 1) / fold_chunks);
    #pragma unroll 1
    for (int split = s0; split < s1; ++split) fold(split, recg + (long long)split * O * kRec);
  }
  if (active && M.mask_acc) {
    int* acc = M.mask_acc + (long long)ml * 4;
    if (fold_chunks == 1) {
      acc[0] = s_corr;
      acc[1] = s_test;
      acc[2] = s_rec;
      acc[3] = s_hit;
    } else {
      atomicAdd(acc + 0, s_corr);
      atomicAdd(acc + 1, s_test);
      atomicAdd(acc + 2, s_rec);
      atomicAdd(acc + 3, s_hit);
    }
  }
  if (M.totals) {
    const unsigned long long a = warp_usum(t_corr), b = warp_usum(t_test), c2 = warp_usum(t_rec),
                             d = warp_usum(t_hit);
    if ((threadIdx.x & 31) == 0 && (a | b | c2 | d)) {
      atomicAdd(&M.totals[0], a);
      atomicAdd(&M.totals[1], b);
      atomicAdd(&M.totals[2], c2);
      atomicAdd(&M.totals[3], d);
    }
  }
}

cudaError_t mask_sfit_launch(int D, unsigned grid, cudaStream_t st, const SchurArgs& SA, int off, int n_items,
                             int fold_chunks);
cudaError_t mask_sprep_launch(int P, unsigned grid, cudaStream_t st, const SchurArgs& SA, const int32_t* glist, int ng);

}  // namespace speedrec
