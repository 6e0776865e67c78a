// eval_masks.cuh -- the feature-mask path for LOO batches (config C5).
// DESIGN.md §5.7.
//
// Every mask of a C5 batch shares the 128 LOO folds, and everything a fit
// needs except the choice of features is mask-independent: the pairs, the
// per-feature min/max/mean of D3 (computed per feature over the fold's
// training befores), and therefore every entry of the centred, scaled Gram
// G_ab = sum_i z_ia z_ib, of the right-hand side r_a = sum_i z_ia (y_i - ybar)
// and of the test row.  The fit of (mask, fold, opt) is the ridge solve on
// the principal submatrix of the fold's full-feature Gram (SURVEY §8(d)
// "allowed shortcuts": the mask-independent per-(o, fold) scaled Gram).
//
//  k_mask_prep  one warp per (fold, opt): pairs, statistics, full Gram,
//               rhs, test row, fingerprints -> a per-(fold, opt) record.
//  k_mask_fit<D> one thread per mask (all masks of the launch have <= D
//               features, D a compile-time size so the d x d system lives in
//               registers): for every fold, gather the submatrix, Cholesky,
//               solve, predict the held-out case, clamp, score, rank and
//               recommend (A4-A7), and the mask's sums over the folds.
//               Masks are ordered by popcount so a warp's threads do equal
//               work; features of a smaller mask are padded with identity
//               rows after the real ones, which leaves the real solution
//               bit-for-bit unchanged.
#pragma once
#include "kernels.cuh"

namespace speedrec {

constexpr int kMaskMaxC = 32;   // counters the path handles (feature word 0)
constexpr int kMaskMaxD = 20;   // largest mask popcount (register-resident system)
constexpr int kMaskMaxO = 8;    // optimization ids

struct PrepMeta {
  double ybar, ac;                      // mean training label; label of the held-out case
  unsigned long long fp_tr, fp_te;      // pair fingerprints (A1)
  int n, nt, tek, active;               // n = -1: opt not scored in the fold; active = feature bits
};

struct MaskArgs {
  ScenDesc sd;
  const double* x;
  const double* ylab;
  const int8_t* opt_bit;
  int P, IR, C, O, G;
  double lambda, threshold, clamp_floor, guard_tol;
  int max_count;
  long long first;       // first scenario (multiple of n_splits)
  long long mask0;       // = first / n_splits
  // per-(fold, opt) records
  double* pG;            // [S*O][C][C] full symmetric centred scaled Gram
  double* pr;            // [S*O][C] rhs
  double* pz;            // [S*O][C] centred scaled held-out row
  PrepMeta* pm;          // [S*O]
  int np_tr;             // max training pairs of a fit (smem lists of k_mask_prep)
  // k_mask_fit launch: local mask indices (into [mask0, mask0 + n_masks_call))
  const int32_t* perm;
  int n_items;
  int fold_chunks;       // threads per mask: folds split into this many ranges (mask sums by atomics)
  // outputs (any may be null)
  OptScore* opt_out;
  ScnScore* scn_out;
  double* ex_out;
  int8_t* rec_out;
  unsigned long long* totals;
  int* mask_acc;         // [n_masks_call][4]: correct, test, rec, hit
};

__device__ __forceinline__ uint32_t mask_bits(const ScenDesc& D, long long fidx) {
  if (D.subsets_k > 0) return (uint32_t)fidx;
  if (D.fmasks) return (uint32_t)D.fmasks[fidx * 2];
  return 0xFFFFFFFFu;
}

// ------------------------------------------------------------------ prep
static __global__ void __launch_bounds__(128) k_mask_prep(const MaskArgs M) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int nw = blockDim.x >> 5;
  double* yv = reinterpret_cast<double*>(smem) + (long long)warp * M.np_tr;           // [nw][np_tr]
  int32_t* trs = reinterpret_cast<int32_t*>(smem + (size_t)nw * M.np_tr * 8) + (long long)warp * M.np_tr;
  const long long S = M.sd.n_splits;
  const int O = M.O, C = M.C, G = M.G;
  const long long item = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= S * O) return;
  const long long split = item / O;
  const int o = (int)(item - split * O);
  PrepMeta meta{};
  double* Gm = M.pG + item * C * C;
  double* rv = M.pr + item * C;
  double* zt = M.pz + item * C;
  if (!((scored_mask(M.sd, split, O) >> o) & 1u)) {
    if (lane == 0) {
      meta.n = -1;
      M.pm[item] = meta;
    }
    return;
  }
  // A1: pairs of the fold, LOO membership (R17)
  int n = 0, nt = 0, tslot = 0, tek = 0;
  uint64_t fptr = 0, fpte = 0;
  for (int g = 0; g < G; ++g) {
    const int b = M.opt_bit[(g / M.IR) * O + o];
    uint64_t tr, te;
    member_words(M.sd, split, g, tr, te);
    if (b < 0 || (tr == 0ull && te == 0ull)) continue;
    const int v = ins0(lane, b);
    const bool istr = ((tr >> v) & 1ull) && ((tr >> (v | (1 << b))) & 1ull);
    const bool iste = (te >> v) & 1ull;
    const unsigned mtr = __ballot_sync(FULL, istr), mte = __ballot_sync(FULL, iste);
    const int lab = (g * O + o) * 32 + lane;
    const uint64_t h = mix64((uint64_t)lab);
    if (istr) {
      const int p = n + __popc(mtr & lt);
      trs[p] = g * 64 + v;
      yv[p] = M.ylab[lab];
      fptr ^= h;
    }
    if (iste) {
      fpte ^= h;
      tslot = g * 64 + v;
      tek = g * 32 + lane;
    }
    if (mte) {
      const int src = __ffs(mte) - 1;   // LOO: at most one held-out case
      tslot = __shfl_sync(FULL, tslot, src);
      tek = __shfl_sync(FULL, tek, src);
    }
    n += __popc(mtr);
    nt += __popc(mte);
  }
  __syncwarp();
  meta.n = n;
  meta.nt = nt;
  meta.fp_tr = warp_xor(fptr);
  meta.fp_te = warp_xor(fpte);
  meta.tek = tek;
  if (nt > 0) meta.ac = M.ylab[((tek >> 5) * O + o) * 32 + (tek & 31)];
  // A2: per-feature min/max/mean over the training befores (D3), all counters
  double xb = 0.0, sc = 0.0;
  bool act = false;
  if (n > 0 && lane < C) {
    double mn = M.x[(long long)trs[0] * C + lane], mx = mn, sm = mn;
    for (int i = 1; i < n; ++i) {
      const double v = M.x[(long long)trs[i] * C + lane];
      mn = fmin(mn, v);
      mx = fmax(mx, v);
      sm += v;
    }
    act = mx > mn;
    if (act) {
      xb = sm / (double)n;
      sc = 1.0 / (mx - mn);
    }
  }
  meta.active = (int)__ballot_sync(FULL, act);
  double ys = 0.0;
  for (int i = lane; i < n; i += 32) ys += yv[i];
  const double ybar = n > 0 ? warp_sum(ys) / (double)n : 0.0;
  meta.ybar = ybar;
  // A3: full-feature centred Gram, rhs, held-out row (z = (x - xbar) * s, 0 if inactive);
  // lanes over the column b <= a of row a, every entry written (symmetric)
  for (int a = 0; a < C; ++a) {
    const double xba = __shfl_sync(FULL, xb, a), sa = __shfl_sync(FULL, sc, a);
    double acc = 0.0;
    if (((meta.active >> a) & 1) && act && lane <= a) {
      for (int i = 0; i < n; ++i) {
        const double* xr = M.x + (long long)trs[i] * C;
        acc = fma((xr[a] - xba) * sa, (xr[lane] - xb) * sc, acc);
      }
    }
    if (lane <= a) {
      Gm[a * C + lane] = acc;
      Gm[lane * C + a] = acc;
    }
  }
  if (lane < C) {
    double r = 0.0;
    if (act)
      for (int i = 0; i < n; ++i) r = fma((M.x[(long long)trs[i] * C + lane] - xb) * sc, yv[i] - ybar, r);
    rv[lane] = r;
    zt[lane] = (act && nt > 0) ? (M.x[(long long)tslot * C + lane] - xb) * sc : 0.0;
  }
  if (lane == 0) M.pm[item] = meta;
}

// ------------------------------------------------------------------ fit
template <int D>
__global__ void __launch_bounds__(128) k_mask_fit(const MaskArgs M) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int O = M.O, C = M.C, G = M.G;
  const long long S = M.sd.n_splits;
  unsigned long long t_corr = 0, t_test = 0, t_rec = 0, t_hit = 0;
  const int item = tid % M.n_items, chunk = tid / M.n_items;   // neighbours share the fold range
  if (chunk < M.fold_chunks) {
    const int ml = M.perm[item];
    const long long fidx = M.mask0 + ml;
    const uint32_t fm = mask_bits(M.sd, fidx) & (C >= 32 ? 0xFFFFFFFFu : ((1u << C) - 1u));
    int s_corr = 0, s_test = 0, s_rec = 0, s_hit = 0;
    const long long s0 = S * chunk / M.fold_chunks, s1 = S * (chunk + 1) / M.fold_chunks;
    #pragma unroll 1
    for (long long split = s0; split < s1; ++split) {
      const long long sl = fidx * S + split - M.first;
      const uint32_t om = scored_mask(M.sd, split, O);
      // held-out slot of the LOO fold (R17)
      const int g = M.sd.pool_list[split >> 6], v = (int)(split & 63), p = g / M.IR;
      double ce[kMaskMaxO];
      bool cv[kMaskMaxO], cc[kMaskMaxO];
      int guard = 0, untrained = 0;
#pragma unroll
      for (int o = 0; o < kMaskMaxO; ++o) {
        cv[o] = false;
        cc[o] = false;
        ce[o] = 0.0;
        if (o >= O) continue;
        OptScore row;
        row.n_train = row.n_test = row.n_correct = row.n_clamped = 0;
        row.sum_ratio = row.min_ratio = row.max_ratio = 0.0;
        row.fp_train = row.fp_test = 0ull;
        const PrepMeta& pm = M.pm[split * O + o];
        const int n = pm.n;
        if (n >= 0 && ((om >> o) & 1u)) {
          row.n_train = n;
          row.n_test = pm.nt;
          row.fp_train = pm.fp_tr;
          row.fp_test = pm.fp_te;
          s_test += pm.nt;
          if (n == 0 && pm.nt > 0) ++untrained;
          if (n > 0 && pm.nt > 0) {
            // ---- A4 on the principal submatrix of the fold's Gram ----
            const long long it = split * O + o;
            const double* Gm = M.pG + it * C * C;
            const double* rv = M.pr + it * C;
            const double* zv = M.pz + it * C;
            const uint32_t am = fm & (uint32_t)pm.active;
            const int de = __popc(am);
            int f[D > 0 ? D : 1];
            {
              uint32_t mm = am;
#pragma unroll
              for (int i = 0; i < D; ++i) {
                f[i] = mm ? __ffs(mm) - 1 : 0;
                mm &= mm - 1u;
              }
            }
            // Augmented factor: rows 0..D-1 = L (diagonal holds 1/L_jj), row D =
            // r and row D+1 = z_t carried through the same column steps, which
            // leaves them as y = L^-1 r and u = L^-1 z, so EX - ybar = w.z =
            // (L^-T y).z = y.u -- no back substitution.
            constexpr int T = D * (D + 1) / 2;
            double L[T + 2 * D + 1];
#pragma unroll
            for (int i = 0; i < D; ++i) {
#pragma unroll
              for (int j = 0; j <= i; ++j)
                L[i * (i + 1) / 2 + j] = (i < de) ? Gm[f[i] * C + f[j]] + (i == j ? M.lambda : 0.0)
                                                  : (i == j ? 1.0 : 0.0);
              L[T + i] = i < de ? rv[f[i]] : 0.0;
              L[T + D + i] = i < de ? zv[f[i]] : 0.0;
            }
            bool ok = true;
#pragma unroll
            for (int j = 0; j < D; ++j) {         // left-looking column step j
              double djj = L[j * (j + 1) / 2 + j];
#pragma unroll
              for (int k = 0; k < j; ++k) djj = fma(-L[j * (j + 1) / 2 + k], L[j * (j + 1) / 2 + k], djj);
              ok &= djj > 0.0;
              const double r = rsqrt_nr(djj);
              L[j * (j + 1) / 2 + j] = r;
#pragma unroll
              for (int i = j + 1; i < D + 2; ++i) {
                const int ri = i < D ? i * (i + 1) / 2 : T + (i - D) * D;   // row start
                double a = L[ri + j];
#pragma unroll
                for (int k = 0; k < j; ++k) a = fma(-L[ri + k], L[j * (j + 1) / 2 + k], a);
                L[ri + j] = a * r;
              }
            }
            double e = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) e = fma(L[T + i], L[T + D + i], e);
            e += pm.ybar;
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
            cc[o] = cl;
            ce[o] = e;
            if (M.ex_out) M.ex_out[(sl * O + o) * (long long)G * 32 + pm.tek] = e;
          }
        }
        if (M.opt_out) M.opt_out[sl * O + o] = row;
      }
      // ---- A6: rank the held-out version's candidates (R13, R21) ----
#pragma unroll
      for (int q = 0; q < kMaskMaxO; ++q) {
        if (!cv[q]) continue;
        if (near_tol(ce[q], M.threshold, M.guard_tol)) ++guard;
#pragma unroll
        for (int r = q + 1; r < kMaskMaxO; ++r)
          if (cv[r] && !(cc[q] && cc[r]) && near_tol(ce[q], ce[r], M.guard_tol)) ++guard;
      }
      int nrec = 0, nhit = 0;
#pragma unroll
      for (int q = 0; q < kMaskMaxO; ++q) {
        if (!cv[q] || !(ce[q] >= M.threshold)) continue;
        int rk = 0;
#pragma unroll
        for (int r = 0; r < kMaskMaxO; ++r)
          if (r != q && cv[r] && ce[r] >= M.threshold && (ce[r] > ce[q] || (ce[r] == ce[q] && r < q))) ++rk;
        if (rk < M.max_count) {
          ++nrec;
          const int b = M.opt_bit[p * O + q];
          if (M.ylab[(g * O + q) * 32 + rmv(v, b)] > 1.0) ++nhit;
          if (M.rec_out) M.rec_out[(sl * G * 64 + g * 64 + v) * M.max_count + rk] = (int8_t)q;
        }
      }
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
    }
    if (M.mask_acc) {
      int* acc = M.mask_acc + (long long)ml * 4;
      if (M.fold_chunks == 1) {   // the thread owns the mask: plain stores
        acc[0] = s_corr;
        acc[1] = s_test;
        acc[2] = s_rec;
        acc[3] = s_hit;
      } else {                    // integer sums: order-independent, exact
        atomicAdd(acc + 0, s_corr);
        atomicAdd(acc + 1, s_test);
        atomicAdd(acc + 2, s_rec);
        atomicAdd(acc + 3, s_hit);
      }
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

// Host launchers of k_mask_fit<D>, one translation unit per D range so the
// unrolled instantiations compile in parallel (mask_fit_*.cu).  Each returns
// cudaErrorInvalidValue for a D outside its range.
cudaError_t mask_fit_launch_a(int D, unsigned grid, cudaStream_t st, const MaskArgs& M);   // 0..9
cudaError_t mask_fit_launch_b(int D, unsigned grid, cudaStream_t st, const MaskArgs& M);   // 10..13
cudaError_t mask_fit_launch_c(int D, unsigned grid, cudaStream_t st, const MaskArgs& M);   // 14..16
cudaError_t mask_fit_launch_d(int D, unsigned grid, cudaStream_t st, const MaskArgs& M);   // 17..20

#define SR_MASK_FIT_CASE(K)                              \
  case K:                                                \
    k_mask_fit<K><<<grid, 128, 0, st>>>(M);              \
    return cudaGetLastError();

}  // namespace speedrec
