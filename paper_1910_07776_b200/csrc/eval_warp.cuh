// eval_warp.cuh -- the warp-per-fit path (<= 64 groups: configs C1, C2, C3, C5).
// DESIGN.md §5.2.
//
//  k_fit_warp  one warp = one (scenario, optimization) fit, A1-A5 + the
//              per-(scenario, optimization) scores of A7.  Persistent grid of
//              warps over the fits of a scenario chunk; the rate matrix is
//              staged once per CTA in shared memory when it fits.  EX of every
//              test case goes to a per-chunk table (clamped values negated).
//  k_rank_warp one warp = one scenario: A6 rank + thresholded recommendation
//              per test slot from the EX table, per-scenario scores (A7).
//  k_mask_final C5: per-mask rows and ranking keys from the atomically summed
//              integer accumulators.
// Splitting fit and rank keeps each kernel's hot code small (instruction
// cache) and balances the fits (warp per fit, not per scenario).
#pragma once
#include "fit_fast.cuh"
#include "kernels.cuh"

namespace speedrec {

// ---------------------------------------------------------------- generic
// (m > 32: rare on C3, never on C1/C2/C5) -- packed factor and two vectors
// in the warp's global scratch slab.
struct FitView {
  const double* X;   // rates, row stride ldx (staged smem or global)
  int ldx;
  const int32_t* trs;
  int n;
  const int16_t* col;
  const double* xb;
  const double* s;
  int deff;
};

template <bool DUAL>
__device__ __forceinline__ double zval(const FitView& f, int r, int k) {
  int i = DUAL ? r : k, a = DUAL ? k : r;
  if (i < f.n && a < f.deff) return (f.X[(long long)f.trs[i] * f.ldx + f.col[a]] - f.xb[a]) * f.s[a];
  return 0.0;
}

template <bool DUAL>
__device__ void build_gram(double* M, int m, int Lk, const FitView& f, double lambda, int lane) {
  const int nb = (m + 7) >> 3;
  const int rl = lane >> 2, kl = lane & 3;
  for (int I = 0; I < nb; ++I) {
    for (int J0 = 0; J0 <= I; J0 += 4) {
      double acc[4][2];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[jj][0] = acc[jj][1] = 0.0;
      for (int k0 = 0; k0 < Lk; k0 += 4) {
        const int kk = k0 + kl;
        const double a = zval<DUAL>(f, I * 8 + rl, kk);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int J = J0 + jj;
          if (J <= I) {
            const double b = (J == I) ? a : zval<DUAL>(f, J * 8 + rl, kk);
            dmma(acc[jj][0], acc[jj][1], a, b);
          }
        }
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int J = J0 + jj;
        if (J <= I) {
          const int row = I * 8 + rl;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = J * 8 + 2 * kl + e;
            if (row < m && c <= row) M[pk(row, c)] = acc[jj][e] + (row == c ? lambda : 0.0);
          }
        }
      }
    }
  }
  __syncwarp();
}

__device__ bool chol_packed(double* M, double* invd, int m, int lane) {
  for (int j = 0; j < m; ++j) {
    const double djj = M[pk(j, j)];
    __syncwarp();
    if (!(djj > 0.0)) return false;
    const double r = rsqrt_nr(djj);
    for (int i = j + 1 + lane; i < m; i += 32) M[pk(i, j)] *= r;
    if (lane == 0) {
      M[pk(j, j)] = djj * r;
      invd[j] = r;
    }
    __syncwarp();
    for (int i = j + 1 + lane; i < m; i += 32) {
      const double lij = M[pk(i, j)];
      double* Mi = M + pk(i, 0);
      for (int k = j + 1; k <= i; ++k) Mi[k] -= lij * M[pk(k, j)];
    }
    __syncwarp();
  }
  return true;
}

__device__ void chol_solve(const double* M, const double* invd, double* z, int m, int lane) {
  for (int j = 0; j < m; ++j) {
    const double yj = z[j] * invd[j];
    __syncwarp();
    if (lane == 0) z[j] = yj;
    for (int i = j + 1 + lane; i < m; i += 32) z[i] -= M[pk(i, j)] * yj;
    __syncwarp();
  }
  for (int j = m - 1; j >= 0; --j) {
    const double xj = z[j] * invd[j];
    __syncwarp();
    if (lane == 0) z[j] = xj;
    for (int i = lane; i < j; i += 32) z[i] -= M[pk(j, i)] * xj;
    __syncwarp();
  }
}

__device__ void xt_times(const FitView& f, const double* v, double* out, int lane) {
  for (int a = lane; a < f.deff; a += 32) {
    const int c = f.col[a];
    const double xb = f.xb[a];
    double acc = 0.0;
    for (int i = 0; i < f.n; ++i) acc = fma(f.X[(long long)f.trs[i] * f.ldx + c] - xb, v[i], acc);
    out[a] = acc * f.s[a];
  }
  __syncwarp();
}

__device__ __forceinline__ double row_dot_u(const FitView& f, const double* xrow, const double* u) {
  double acc = 0.0;
  for (int a = 0; a < f.deff; ++a) acc = fma(xrow[f.col[a]] - f.xb[a], u[a], acc);
  return acc;
}

// Generic fit (any m): yc [n] smem, scratch slab: M packed + v1 [vmax] + invd [vmax].
// Output w' in wv[0..deff).
__device__ __noinline__ bool fit_generic(const FitView& f, const double* yc, double lambda, int nref, bool dual,
                                         double* scr, int vmax, double* uv, double* v2, double* wv, int lane) {
  const int m = dual ? f.n : f.deff;
  double* M = scr;
  double* v1 = scr + (long long)m * (m + 1) / 2;
  double* invd = v1 + vmax;
  if (dual) build_gram<true>(M, m, f.deff, f, lambda, lane);
  else build_gram<false>(M, m, f.n, f, lambda, lane);
  if (!chol_packed(M, invd, m, lane)) return false;
  if (dual) {
    for (int i = lane; i < f.n; i += 32) v1[i] = yc[i];
    __syncwarp();
    chol_solve(M, invd, v1, m, lane);
    for (int it = 0; it < nref; ++it) {
      xt_times(f, v1, wv, lane);
      for (int a = lane; a < f.deff; a += 32) uv[a] = wv[a] * f.s[a];
      __syncwarp();
      for (int i = lane; i < f.n; i += 32)
        v2[i] = yc[i] - row_dot_u(f, f.X + (long long)f.trs[i] * f.ldx, uv) - lambda * v1[i];
      __syncwarp();
      chol_solve(M, invd, v2, m, lane);
      for (int i = lane; i < f.n; i += 32) v1[i] += v2[i];
      __syncwarp();
    }
    xt_times(f, v1, wv, lane);
  } else {
    xt_times(f, yc, wv, lane);
    chol_solve(M, invd, wv, m, lane);
    for (int it = 0; it < nref; ++it) {
      for (int a = lane; a < f.deff; a += 32) uv[a] = wv[a] * f.s[a];
      __syncwarp();
      for (int i = lane; i < f.n; i += 32) v2[i] = yc[i] - row_dot_u(f, f.X + (long long)f.trs[i] * f.ldx, uv);
      __syncwarp();
      xt_times(f, v2, v1, lane);
      for (int a = lane; a < f.deff; a += 32) v1[a] -= lambda * wv[a];
      __syncwarp();
      chol_solve(M, invd, v1, m, lane);
      for (int a = lane; a < f.deff; a += 32) wv[a] += v1[a];
      __syncwarp();
    }
  }
  return true;
}

}  // namespace speedrec
#include "m5_warp.cuh"
namespace speedrec {

// ------------------------------------------------------------- IBK (NEXT-1)
// EX of one test case under IBk (reading R22): the mean training
// label of the min(k, n) training befores nearest in min-max scaled counter
// space, x' = (x - mn) / rg over the active features (D3), squared Euclidean
// distance accumulated with fma in active-feature order, neighbours ordered by
// (distance, training index), labels summed in that order and divided by k'.
// Every operation is the definition's, in its order, so EX is bit-exact.
// Warp-collective: each sweep stages kKnnRows scaled training rows in S
// (shared) and every lane scans them against its own test row xq (null for an
// idle lane).  The lane's k-best list lives in registers (kKnnMax slots,
// sorted; a new candidate has the largest index so far, so strict > keeps
// (distance, index) order).
__device__ __forceinline__ double knn_ex(const double* __restrict__ X, int ldx, const int32_t* trs,
                                         const double* y, int n, const int16_t* col, const double* mnv,
                                         const double* rgv, int deff, int kk, const double* xq,
                                         double* S, int lane) {
  double bd[kKnnMax];
  int bi[kKnnMax];
#pragma unroll
  for (int q = 0; q < kKnnMax; ++q) {
    bd[q] = INFINITY;
    bi[q] = 0;
  }
  double thr = INFINITY;  // distance of the current kk-th neighbour
  #pragma unroll 1
  for (int i0 = 0; i0 < n; i0 += kKnnRows) {
    const int rows = min(kKnnRows, n - i0);
    __syncwarp();
    for (int e = lane; e < rows * deff; e += 32) {
      const int r = e / deff, a = e - r * deff;
      S[r * deff + a] = (X[(long long)trs[i0 + r] * ldx + col[a]] - mnv[a]) / rgv[a];
    }
    __syncwarp();
    if (xq) {
      double acc[kKnnRows];
#pragma unroll
      for (int r = 0; r < kKnnRows; ++r) acc[r] = 0.0;
      #pragma unroll 1
      for (int a = 0; a < deff; ++a) {
        const double v = (xq[col[a]] - mnv[a]) / rgv[a];
#pragma unroll
        for (int r = 0; r < kKnnRows; ++r) {   // rows >= `rows` read stale values, dropped below
          const double dl = v - S[r * deff + a];
          acc[r] = fma(dl, dl, acc[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < kKnnRows; ++r) {
        const double D = acc[r];
        if (r < rows && D < thr) {
          const int id = i0 + r;
#pragma unroll
          for (int q = kKnnMax - 1; q > 0; --q) {
            const bool sh = bd[q - 1] > D, put = !sh && bd[q] > D;
            if (sh) {
              bd[q] = bd[q - 1];
              bi[q] = bi[q - 1];
            } else if (put) {
              bd[q] = D;
              bi[q] = id;
            }
          }
          if (bd[0] > D) {
            bd[0] = D;
            bi[0] = id;
          }
#pragma unroll
          for (int q = 0; q < kKnnMax; ++q)
            if (q == kk - 1) thr = bd[q];
        }
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kKnnMax; ++q)
    if (q < kk) s += y[bi[q]];
  return s / (double)kk;
}

template <int CMAX>
__device__ __forceinline__ void rank_scenario(const EvalArgs& A, long long sl, int lane, bool ext_cg,
                                              unsigned long long& tot_rec, unsigned long long& tot_hit);

// ---------------------------------------------------------------- fit kernel
// MODE 0: ridge LS (the paper's model); 1: IBK (NEXT-1); 2: ridge LS + the
// sr_fit coefficient store; 3: M5P model tree (NEXT-2, m5_warp.cuh); 4: ridge
// LS writing each fit's model (u, c0) and counts to the model table, with A5-A7
// in k_pred_rank (pred_rank.cuh).  Separate instantiations
// keep the hot code lean.
// STAGED: x staged in shared memory (compile-time, so every x access is an
// LDS rather than a generic load).
template <int WMAX, int MODE, bool STAGED>
#ifndef SR_M5_MINB
#define SR_M5_MINB 1      // M5P: resident CTAs per SM the register budget is cut for (A/B knob)
#endif
#ifndef SR_M5_WMAX
#define SR_M5_WMAX 16     // M5P: warps per CTA
#endif
__global__ void __launch_bounds__(WMAX * 32, MODE == 3 ? SR_M5_MINB : 1) k_fit_warp(const EvalArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const WarpLayout& L = A.L;
  int8_t* obit = reinterpret_cast<int8_t*>(smem);
  const int tid = threadIdx.x, nthr = blockDim.x;
  // per-GROUP optimization bits (no division by I*R in the pair loop)
  for (int i = tid; i < A.G * A.O; i += nthr) obit[i] = A.opt_bit[(i / A.O / A.IR) * A.O + i % A.O];
  const double* X = A.x;
  int ldx = A.C;
  if (STAGED) {
    double* xs = reinterpret_cast<double*>(smem + A.off_stage);
    const int tot = A.G * 64 * A.C;
    for (int i = tid; i < tot; i += nthr) xs[(i / A.C) * A.ldxs + (i % A.C)] = A.x[i];
    X = xs;
    ldx = A.ldxs;
  }
  const double* ylab = A.ylab;          // the labels, staged when small (C1, C3: 1-3 KB)
  if (A.stage_y) {
    double* ys = reinterpret_cast<double*>(smem + A.off_y);
    for (int i = tid; i < A.G * A.O * 32; i += nthr) ys[i] = A.ylab[i];
    ylab = ys;
  }
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned char* slab = smem + A.off_warps + warp * L.bytes;
  uint64_t* trw = reinterpret_cast<uint64_t*>(slab + L.off_trw);
  uint64_t* tew = reinterpret_cast<uint64_t*>(slab + L.off_tew);
  int16_t* F = reinterpret_cast<int16_t*>(slab + L.off_F);
  int32_t* trs = reinterpret_cast<int32_t*>(slab + L.off_trs);
  double* yc = reinterpret_cast<double*>(slab + L.off_yc);
  int32_t* tes = reinterpret_cast<int32_t*>(slab + L.off_tes);
  int32_t* tek = reinterpret_cast<int32_t*>(slab + L.off_tek);
  int16_t* col = reinterpret_cast<int16_t*>(slab + L.off_col);
  double* xb = reinterpret_cast<double*>(slab + L.off_xb);
  double* sv = reinterpret_cast<double*>(slab + L.off_s);
  double* wv = reinterpret_cast<double*>(slab + L.off_w);
  double* uv = reinterpret_cast<double*>(slab + L.off_u);
  double* v2 = reinterpret_cast<double*>(slab + L.off_v2);
  double* Msm = reinterpret_cast<double*>(slab + L.off_M);
  double* ufull = reinterpret_cast<double*>(slab + L.off_ufull);

  const long long gwarp = (long long)blockIdx.x * A.warps_per_block + warp;
  const long long nwarps = (long long)gridDim.x * A.warps_per_block;
  double* scr = A.gscratch ? A.gscratch + gwarp * A.mscratch : nullptr;
  // M5P teams (A.m5_team warps per fit): every member fits
  // the same tree in its own slab, the split search is shared; only the lead
  // warp writes outputs
  const int tw = MODE == 3 ? A.m5_team : 1;
  const int trank = warp % tw;
  const bool lead = trank == 0;
  const long long team = gwarp / tw, nteams = nwarps / tw;
  __shared__ double m5x[3 * kMaxWarpsPerBlock];
  unsigned long long m5ops = 0;           // executed split-search FP64 operations (this lane)
  const M5Team m5t{tw, trank, 1 + warp / tw, m5x + 3 * (warp - trank), &m5ops};
  const int G = A.G, O = A.O, C = A.C;
  unsigned long long tot_corr = 0, tot_test = 0, tot_rec = 0, tot_hit = 0;
  // fused A6 (A.fuse_rank): the warp finishing the last scored fit of a
  // scenario ranks it at once, from the L2-hot EX table
  auto finish = [&](long long sl, uint32_t om) {
    if (MODE != 0 || !A.fuse_rank) return;
    __threadfence();                      // this warp's EX / trained / guard writes before the count
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicAdd(&A.done[sl], 1) == __popc(om) - 1;
    if (__shfl_sync(FULL, last, 0)) {
      __threadfence();
      rank_scenario<8>(A, sl, lane, true, tot_rec, tot_hit);
    }
  };

  // scenario-major (A.scn_major, large batches): a warp fits all O
  // optimizations of one scenario in turn, so the split words and the feature
  // list are formed once per scenario; fit-major (small, latency-bound
  // batches): one fit per work unit, spreading a scenario over warps
  const long long units = A.scn_major ? A.count : A.count * O;
  // work units: the first nteams by warp index, then (A.queue) one at a time
  // from a launch-wide counter, so warps that drew cheap scenarios keep
  // working instead of waiting out the last warps of a static stride (the
  // outputs are per unit, the totals integer: the order changes nothing)
  // (M5P teams: the lead warp draws, its team reads the unit from a shared slot)
  __shared__ long long m5q[kMaxWarpsPerBlock];
  auto next_unit = [&](long long u) -> long long {
    if (A.queue == nullptr) return u + nteams;
    if (MODE == 3) {
      if (lead && lane == 0) m5q[warp - trank] = (long long)atomicAdd(A.queue, 1ull) + nteams;
      if (tw > 1) m5_team_sync(m5t);
      else __syncwarp();
      const long long nu = m5q[warp - trank];
      if (tw > 1) m5_team_sync(m5t);   // every member has read the slot before the next draw
      else __syncwarp();
      return nu;
    }
    unsigned long long v = 0ull;
    if (lane == 0) v = atomicAdd(A.queue, 1ull);
    return (long long)__shfl_sync(FULL, v, 0) + nteams;
  };
  if (MODE == 4) SR_WT(-1);
  for (long long u = team; u < units; u = next_unit(u)) {
  const long long sl = A.scn_major ? u : u / O;
  const int o_lo = A.scn_major ? 0 : (int)(u - sl * O), o_hi = A.scn_major ? O : o_lo + 1;
  const long long s = A.first + sl, so = A.out0 + sl;
  const long long split = s % A.sd.n_splits, fidx = s / A.sd.n_splits;
  const uint32_t om = scored_mask(A.sd, split, O);
  // ---- A1: split membership (Table 2; R17), features ----
  for (int g = lane; g < G; g += 32) {
    uint64_t tr, te;
    member_words(A.sd, split, g, tr, te);
    trw[g] = tr;
    tew[g] = te;
  }
  int d = 0;
  for (int c0 = 0; c0 < C; c0 += 32) {
    const int c = c0 + lane;
    const bool in = c < C && feature_in(A.sd, fidx, c);
    const unsigned bm = __ballot_sync(FULL, in);
    if (in) F[d + __popc(bm & lt)] = (int16_t)c;
    d += __popc(bm);
  }
  __syncwarp();
  if (MODE == 4) SR_WT(0);
  for (int o = o_lo; o < o_hi; ++o) {
    OptScore row;
    row.n_train = row.n_test = row.n_correct = row.n_clamped = 0;
    row.sum_ratio = row.min_ratio = row.max_ratio = 0.0;
    row.fp_train = row.fp_test = 0ull;
    if (!((om >> o) & 1u)) {
      if (lane == 0 && lead && A.opt_out) A.opt_out[so * O + o] = row;
      // no scored optimization at all: nothing will finish, rank (empty row) here
      if (MODE == 0 && A.fuse_rank && om == 0u && o == 0) rank_scenario<8>(A, sl, lane, true, tot_rec, tot_hit);
      continue;
    }
    const int q = __popc(om & ((1u << o) - 1u));  // scored-optimization slot in the EX table
    double* urow = MODE == 4 ? A.utab + (sl * (long long)A.n_os + q) * A.ldu : nullptr;

    // ---- A1: pairs ----
    int n = 0, nt = 0;
    uint64_t fptr = 0, fpte = 0;
    #pragma unroll 1
    for (int g = 0; g < G; ++g) {
      const int b = obit[g * O + o];
      const uint64_t tr = trw[g], te = tew[g];
      if (b < 0 || (tr == 0ull && te == 0ull)) continue;
      const int v = ins0(lane, b);
      const bool istr = ((tr >> v) & 1ull) && ((tr >> (v | (1 << b))) & 1ull);
      const bool iste = (te >> v) & 1ull;
      const unsigned mtr = __ballot_sync(FULL, istr), mte = __ballot_sync(FULL, iste);
      const int lab = (g * O + o) * 32 + lane;
      if (istr | iste) {
        const uint64_t h = mix64((uint64_t)lab);
        if (istr) {
          const int p = n + __popc(mtr & lt);
          trs[p] = g * 64 + v;
          yc[p] = ylab[lab];
          fptr ^= h;
        }
        if (iste) {
          if (MODE != 4) {              // MODE 4 predicts in k_pred_rank: counts only
            const int p = nt + __popc(mte & lt);
            tes[p] = g * 64 + v;
            tek[p] = g * 32 + lane;
          }
          fpte ^= h;
        }
      }
      n += __popc(mtr);
      nt += __popc(mte);
    }
    row.n_train = n;
    row.n_test = nt;
    row.fp_train = warp_xor(fptr);
    row.fp_test = warp_xor(fpte);
    __syncwarp();
    if (MODE == 4) SR_WT(1);
    if (n > 0 && lane == 0 && lead && MODE != 4) atomicOr(&A.trained[sl], 1u << o);
    auto put_counts = [&](double flag) {   // MODE 4: the model-table row's fields after u, c0
      if (lane == 0) {
        double* e = urow + ((A.C + 3) & ~3);   // fields after the k-step-padded weights
        e[kUflag] = flag;
        e[kUntr] = (double)n;
        e[kUnte] = (double)nt;
        e[kUfptr] = __longlong_as_double((long long)row.fp_train);
        e[kUfpte] = __longlong_as_double((long long)row.fp_test);
      }
    };
    // untrained (reading R18) or nothing to predict; sr_fit (MODE 2) fits every
    // trained optimization, tested or not (its model is the call's output)
    if (n == 0 || (nt == 0 && MODE != 2)) {
      if (MODE == 4) {
        put_counts(n > 0 ? 1.0 : 0.0);
        SR_WT(7);
        continue;
      }
      if (lane == 0 && lead && A.opt_out) A.opt_out[so * O + o] = row;
      if (A.agg && lane == 0 && lead && nt > 0) atomicAdd(&A.mask_acc[(fidx - A.mask0) * 4 + 1], nt);
      finish(sl, om);
      continue;
    }

    // ---- A2: per-fit min-max statistics over the training befores (D3) ----
    constexpr bool ibk = MODE == 1, m5 = MODE == 3;
    int deff = 0;
    // rates are finite and >= 0 (sr_load_dataset validates them), so min/max
    // need no NaN handling: one compare + select each (dmin/dmax)
    const unsigned xs32 = STAGED ? (unsigned)__cvta_generic_to_shared(X) : 0u;
    const int ldx8 = ldx * 8;
    for (int a0 = 0; a0 < d; a0 += 64) {       // two features per lane per row pass
      const int a1 = a0 + lane, a2 = a0 + 32 + lane;
      const int c1 = a1 < d ? F[a1] : 0, c2 = a2 < d ? F[a2] : 0;
      const int o1 = c1 * 8, o2 = c2 * 8;
      const int r0 = trs[0] * ldx8;
      double mn1 = xload<STAGED>(X, xs32, r0 + o1), mx1 = mn1, sm1 = mn1;
      double mn2 = xload<STAGED>(X, xs32, r0 + o2), mx2 = mn2, sm2 = mn2;
      // two rows per pass into separate accumulators (independent min/max chains)
      double nb1 = mn1, xb1 = mx1, tb1 = 0.0, nb2 = mn2, xb2 = mx2, tb2 = 0.0;
      int i = 1;
      SR_UNROLL(SR_UNROLL_STATS)
      for (; i + 1 < n; i += 2) {
        const int ri = trs[i] * ldx8, rq = trs[i + 1] * ldx8;
        const double v1 = xload<STAGED>(X, xs32, ri + o1), v2 = xload<STAGED>(X, xs32, ri + o2);
        const double w1 = xload<STAGED>(X, xs32, rq + o1), w2 = xload<STAGED>(X, xs32, rq + o2);
        mn1 = dmin(mn1, v1);
        nb1 = dmin(nb1, w1);
        mx1 = dmax(mx1, v1);
        xb1 = dmax(xb1, w1);
        sm1 += v1;
        tb1 += w1;
        mn2 = dmin(mn2, v2);
        nb2 = dmin(nb2, w2);
        mx2 = dmax(mx2, v2);
        xb2 = dmax(xb2, w2);
        sm2 += v2;
        tb2 += w2;
      }
      if (i < n) {
        const int ri = trs[i] * ldx8;
        const double v1 = xload<STAGED>(X, xs32, ri + o1), v2 = xload<STAGED>(X, xs32, ri + o2);
        mn1 = dmin(mn1, v1);
        mx1 = dmax(mx1, v1);
        sm1 += v1;
        mn2 = dmin(mn2, v2);
        mx2 = dmax(mx2, v2);
        sm2 += v2;
      }
      mn1 = dmin(mn1, nb1);
      mx1 = dmax(mx1, xb1);
      sm1 += tb1;
      mn2 = dmin(mn2, nb2);
      mx2 = dmax(mx2, xb2);
      sm2 += tb2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = h ? a2 : a1;
        const double mn = h ? mn2 : mn1, mx = h ? mx2 : mx1, sm = h ? sm2 : sm1;
        const bool act = a < d && mx > mn;
        const unsigned bm = __ballot_sync(FULL, act);
        if (act) {
          const int p = deff + __popc(bm & lt);
          col[p] = (int16_t)(h ? c2 : c1);
          xb[p] = sm / (double)n;
          sv[p] = 1.0 / (mx - mn);
          if (ibk || m5) {
            uv[p] = mn;
            wv[p] = mx - mn;
          }
        }
        deff += __popc(bm);
      }
    }
    {  // zero padding read by the fast-path fragment loads
      const int pad_end = max(32, (deff + 3) & ~3);
      for (int p = deff + lane; p < pad_end; p += 32) {
        col[p] = 0;
        xb[p] = 0.0;
        sv[p] = 0.0;
      }
    }
    if (MODE == 4) SR_WT(2);
    double c0 = 0.0;
    bool ok = true;
    if (!ibk && !m5) {
      double ysum = 0.0;
      #pragma unroll 1
      for (int i = lane; i < n; i += 32) ysum += yc[i];
      const double ybar = warp_sum(ysum) / (double)n;
      for (int i = lane; i < n; i += 32) yc[i] -= ybar;
      __syncwarp();

      // ---- A3/A4: centred normal equations, dual or primal ----
      const bool dual = (n - 1) < deff;
      const int m = dual ? n : deff;
      // refine where conditioning or the O(n eps) Gram accumulation error needs it
      const int nref = (dual ? 2 * (n - 1) >= deff : ((n - 1) < 2 * deff || n > 64)) ? A.refine : 0;
      if (m > 0 && m <= (L.mcap < 32 ? L.mcap : 32)) {
        const FastView fv{X, ldx, trs, n, col, xb, sv, deff, xs32};
        ok = dual ? fit_fast<true, STAGED>(fv, yc, A.lambda, nref, Msm, v2, uv, wv, lane, L.mcap)
                  : fit_fast<false, STAGED>(fv, yc, A.lambda, nref, Msm, v2, uv, wv, lane, L.mcap);
      } else if (m > 0) {
        const FitView fv{X, ldx, trs, n, col, xb, sv, deff};
        ok = fit_generic(fv, yc, A.lambda, nref, dual, scr, L.vmax, uv, v2, wv, lane);
      }
      // weights on raw counters: EX = c0 + sum_c x_c * ufull[c]
      for (int c = lane; c < C; c += 32) ufull[c] = 0.0;
      __syncwarp();
      double cpart = 0.0;
      if (m > 0 && ok)
        for (int a = lane; a < deff; a += 32) {
          const double u = wv[a] * sv[a];
          ufull[col[a]] = u;
          cpart = fma(xb[a], u, cpart);
        }
      c0 = ybar - warp_sum(cpart);
      __syncwarp();
      if (MODE == 2) {   // sr_fit: the model in raw-counter form, EX = c0 + sum_c u_c x_c
        double* cf = A.coef_out + (sl * O + o) * (long long)(C + 1);
        for (int c = lane; c < C; c += 32) cf[1 + c] = ufull[c];
        if (lane == 0) cf[0] = c0;
      }
      if (MODE == 4) {   // the model for k_pred_rank (A5-A7 there)
        const int Cp = (C + 3) & ~3;       // weights padded with zeros to whole DMMA k-steps
        for (int c = lane; c < Cp; c += 32) urow[c] = c < C ? ufull[c] : 0.0;
        if (lane == 0) urow[Cp + kUc0] = c0;
        put_counts(ok ? 1.0 : 2.0);
        SR_WT(7);
        continue;
      }
    }

    // ---- A5: predict + clamp; A7 per-(s,o) scores ----
    double* ext = A.extab + sl * A.ex_stride + q * A.tg_stride;
    int ncorr = 0, ncl = 0, guard = (ok || lane != 0) ? 0 : 1000000;   // per lane, summed below
    double rsum = 0.0, rmin = INFINITY, rmax = -INFINITY;
    auto score = [&](const int j, double e) {
      if (near_tol(e, 0.0, A.guard_tol) || near_tol(e, 1.0, A.guard_tol)) ++guard;
      bool cl = false;
      if (e <= 0.0) {
        e = A.clamp_floor;
        cl = true;
        ++ncl;
      }
      const int gk = tek[j];
      const double ac = ylab[((gk >> 5) * O + o) * 32 + (gk & 31)];
      ncorr += ((e > 1.0 && ac > 1.0) || (e <= 1.0 && ac <= 1.0)) ? 1 : 0;
      const double ratio = ac / e;
      rsum += ratio;
      rmin = fmin(rmin, ratio);
      rmax = fmax(rmax, ratio);
      if (lead) {
        ext[test_group_index(A.sd, split, gk >> 5) * 32 + (gk & 31)] = cl ? -e : e;
        if (A.ex_out) A.ex_out[(so * O + o) * (long long)G * 32 + gk] = e;
      }
    };
    if (m5) {    // NEXT-2: grow + prune the tree in the warp's scratch slab, then lanes over tests
      SR_M5T(-1);
      M5Work W = m5_carve(scr, L.np_tr, A.C);
      W.ld = deff > 0 ? deff : 1;    // rows of the active features only
      for (int e = lane; e < n * deff; e += 32) {
        const int r = e / deff, a = e - r * deff;
        W.Xs[r * W.ld + a] = (X[(long long)trs[r] * ldx + col[a]] - uv[a]) / wv[a];
      }
      __syncwarp();
      SR_M5T(4);
      int tg = 0;
      bool tok = true;
      m5_build(W, n, deff, yc, A.lambda, A.refine, A.guard_tol, lane, &tg, &tok, m5t);
      if (lane == 0) guard += tg + (tok ? 0 : 1000000);   // warp-uniform counts: once, not per lane
      SR_M5T(-1);
      for (int j = lane; j < nt; j += 32) score(j, m5_predict(W, X + (long long)tes[j] * ldx, col, uv, wv));
      SR_M5T(5);
    } else if (ibk) {   // NEXT-1: IBk prediction, all lanes sweep together (knn_ex)
      const int kk = min(A.k_nn, n);
      #pragma unroll 1
      for (int j0 = 0; j0 < nt; j0 += 32) {
        const int j = j0 + lane;
        const double* xq = j < nt ? X + (long long)tes[j] * ldx : nullptr;
        const double e = knn_ex(X, ldx, trs, yc, n, col, uv, wv, deff, kk, xq, Msm, lane);
        if (j < nt) score(j, e);
      }
    } else {
      for (int j = lane; j < nt; j += 32) {
        const double* xr = X + (long long)tes[j] * ldx;
        double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;   // 4 independent chains
        int c = 0;
        SR_UNROLL(SR_UNROLL_PRED)
        for (; c + 3 < C; c += 4) {
          const double2 u01 = *reinterpret_cast<const double2*>(ufull + c);
          const double2 u23 = *reinterpret_cast<const double2*>(ufull + c + 2);
          e0 = fma(xr[c], u01.x, e0);
          e1 = fma(xr[c + 1], u01.y, e1);
          e2 = fma(xr[c + 2], u23.x, e2);
          e3 = fma(xr[c + 3], u23.y, e3);
        }
        for (; c < C; ++c) e0 = fma(xr[c], ufull[c], e0);
        double e = c0 + ((e0 + e1) + (e2 + e3));
        score(j, e);
      }
    }
    row.n_correct = warp_isum(ncorr);
    row.n_clamped = warp_isum(ncl);
    row.sum_ratio = warp_sum(rsum);
    row.min_ratio = warp_min(rmin);
    row.max_ratio = warp_max(rmax);
    if (MODE == 2 && nt == 0) row.min_ratio = row.max_ratio = 0.0;   // fitted, nothing tested
    guard = warp_isum(guard);
    if (lead) {
      tot_corr += row.n_correct;
      tot_test += nt;
    }
    if (lane == 0 && lead) {
      if (A.opt_out) A.opt_out[so * O + o] = row;
      if (guard) atomicAdd(&A.guard_acc[sl], guard);
      if (A.agg) {
        atomicAdd(&A.mask_acc[(fidx - A.mask0) * 4 + 0], row.n_correct);
        atomicAdd(&A.mask_acc[(fidx - A.mask0) * 4 + 1], nt);
      }
    }
    __syncwarp();
    finish(sl, om);
  }
  }
  if (A.totals && lane == 0 && tot_test) {
    atomicAdd(&A.totals[0], tot_corr);
    atomicAdd(&A.totals[1], tot_test);
  }
#if SR_WARP_TIMING && SR_M5_TIMING
  if (MODE == 3 && blockIdx.x < 4 && lane == 0) {
    const long long* a = sr_wt_acc[blockIdx.x * A.warps_per_block + warp];
    printf("SR_M5T cta %d warp %d: search %lld partition %lld models %lld prune %lld rows %lld predict %lld\n",
           blockIdx.x, warp, a[0], a[1], a[2], a[3], a[4], a[5]);
  }
#endif
#if SR_WARP_TIMING
  if (MODE == 4 && blockIdx.x == 0 && lane == 0) {
    const long long* a = sr_wt_acc[warp];
    printf("SR_WT warp %d: setup %lld pairs %lld stats %lld gram %lld chol %lld solve %lld xta %lld out %lld\n", warp,
           a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7]);
  }
#endif
  if (MODE == 3 && A.work) {                // every team member adds its own share of the search
    const unsigned long long w = warp_usum(m5ops);
    if (lane == 0 && w) atomicAdd(A.work, w);
  }
  if (A.totals && lane == 0 && (tot_rec | tot_hit)) {
    atomicAdd(&A.totals[2], tot_rec);
    atomicAdd(&A.totals[3], tot_hit);
  }
}

// ---------------------------------------------------------------- rank kernel
// A6: per test slot, candidates = scored, trained optimizations whose bit is
// clear (reading R13); sort by (EX desc, id asc), keep EX >= threshold, first
// max_count.  One warp per scenario, lanes over the slot's versions.
// A6 + A7 (per scenario) for scenario sl of the chunk, one warp.  ext_cg:
// the EX table, trained masks and guard counts were written by other SMs in
// this launch (the fused path): read them from L2 (ld.global.cg).
template <int CMAX>
__device__ __forceinline__ void rank_scenario(const EvalArgs& A, long long sl, int lane, bool ext_cg,
                                              unsigned long long& tot_rec, unsigned long long& tot_hit) {
  const int G = A.G, O = A.O;
  const long long s = A.first + sl, so = A.out0 + sl;
  const long long split = s % A.sd.n_splits, fidx = s / A.sd.n_splits;
  const uint32_t om = scored_mask(A.sd, split, O);
  const uint32_t trained = ext_cg ? __ldcg(A.trained + sl) : A.trained[sl];
  int olist[CMAX];
  int n_os = 0;
#pragma unroll
  for (int q = 0; q < CMAX; ++q) olist[q] = -1;
  {
    uint32_t mm = om;
#pragma unroll
    for (int q = 0; q < CMAX; ++q) {
      if (mm) {
        olist[q] = __ffs(mm) - 1;
        mm &= mm - 1;
        ++n_os;
      }
    }
  }
  const double* ext = A.extab + sl * A.ex_stride;
  int nrec = 0, nhit = 0, guard = 0, untrained = 0;
  #pragma unroll 1
  for (int g = 0; g < G; ++g) {
    uint64_t tr, te;
    member_words(A.sd, split, g, tr, te);
    if (te == 0ull) continue;
    const int gi = test_group_index(A.sd, split, g);
    const int p = g / A.IR;
    for (int h = 0; h < 2; ++h) {
      const int v = h * 32 + lane;
      if (!((te >> v) & 1ull)) continue;
      double ce[CMAX];
      bool cv[CMAX], cc[CMAX];
      int ck[CMAX];
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        const int o = olist[q];
        int b = -1;
        if (o >= 0) b = A.opt_bit[p * O + o];
        bool cand = o >= 0 && b >= 0 && !((v >> b) & 1);
        if (cand && !((trained >> o) & 1u)) {
          ++untrained;
          cand = false;
        }
        cv[q] = cand;
        ck[q] = cand ? rmv(v, b) : 0;
        const double* ep = ext + q * A.tg_stride + gi * 32 + ck[q];
        const double raw = cand ? (ext_cg ? __ldcg(ep) : *ep) : 0.0;
        cc[q] = raw < 0.0;
        ce[q] = fabs(raw);
      }
      // guard band (reading R21)
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        if (!cv[q]) continue;
        if (near_tol(ce[q], A.threshold, A.guard_tol)) ++guard;
#pragma unroll
        for (int r = q + 1; r < CMAX; ++r)
          if (cv[r] && !(cc[q] && cc[r]) && near_tol(ce[q], ce[r], A.guard_tol)) ++guard;
      }
      // rank among candidates with EX >= threshold: (EX desc, id asc) by
      // selection -- round rk takes the best remaining candidate, whose rank
      // is rk; only the first max_count rounds recommend
      unsigned left = 0u;
#pragma unroll
      for (int q = 0; q < CMAX; ++q)
        if (cv[q] && ce[q] >= A.threshold) left |= 1u << q;
      for (int rk = 0; rk < A.max_count && left; ++rk) {
        int best = -1;
        double be = -INFINITY;
#pragma unroll
        for (int q = 0; q < CMAX; ++q)
          if (((left >> q) & 1u) && ce[q] > be) {     // strict: ties keep the lower id
            be = ce[q];
            best = q;
          }
        left &= ~(1u << best);
        ++nrec;
        int kb = 0, ob = 0;
#pragma unroll
        for (int q = 0; q < CMAX; ++q)
          if (q == best) {
            kb = ck[q];
            ob = olist[q];
          }
        if (A.ylab[(g * O + ob) * 32 + kb] > 1.0) ++nhit;
        if (A.rec_out) A.rec_out[(so * G * 64 + g * 64 + v) * A.max_count + rk] = (int8_t)ob;
      }
    }
  }
  ScnScore sr;
  sr.n_rec = warp_isum(nrec);
  sr.n_rec_hit = warp_isum(nhit);
  sr.n_untrained = warp_isum(untrained);
  sr.n_guard = warp_isum(guard) + (ext_cg ? __ldcg(A.guard_acc + sl) : A.guard_acc[sl]);
  tot_rec += sr.n_rec;
  tot_hit += sr.n_rec_hit;
  if (lane == 0) {
    if (A.scn_out) A.scn_out[so] = sr;
    if (A.agg) {
      atomicAdd(&A.mask_acc[(fidx - A.mask0) * 4 + 2], sr.n_rec);
      atomicAdd(&A.mask_acc[(fidx - A.mask0) * 4 + 3], sr.n_rec_hit);
    }
  }

}

template <int CMAX>
__global__ void __launch_bounds__(256) k_rank_warp(const EvalArgs A) {
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned long long tot_rec = 0, tot_hit = 0;
  for (long long sl = gwarp; sl < A.count; sl += nwarps) rank_scenario<CMAX>(A, sl, lane, false, tot_rec, tot_hit);
  if (A.totals && lane == 0 && (tot_rec | tot_hit)) {
    atomicAdd(&A.totals[2], tot_rec);
    atomicAdd(&A.totals[3], tot_hit);
  }
}

// ---------------------------------------------------------------- sweep
// NEXT-3 (sr_sweep): per test version the candidates of rank_scenario,
// sorted by (EX desc, id asc); candidate at position p with EX e is
// recommended for (theta_i, K_j) iff p < K_j and theta_i <= e.  With u =
// #{theta_i <= e} (thresholds ascending) that is i < u: a difference array per
// list length, D_j[0] += 1, D_j[u] -= 1, accumulated in shared memory (integer
// atomics: exact, order-free) and prefix-summed into the int64 totals.
struct SweepArgs {
  const double* thr;     // [n_thr] ascending
  const int* cnt;        // [n_cnt]
  int n_thr, n_cnt;
  unsigned long long* out;   // [2][n_thr][n_cnt]: recommendations, hits
};

template <int CMAX>
__global__ void __launch_bounds__(256) k_sweep_warp(const EvalArgs A, const SweepArgs W) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* thr = reinterpret_cast<double*>(smem);                          // [n_thr]
  int* cnt = reinterpret_cast<int*>(thr + W.n_thr);                       // [n_cnt]
  int* D = cnt + W.n_cnt;                                                 // [2][n_cnt][n_thr + 1]
  const int nd = 2 * W.n_cnt * (W.n_thr + 1);
  for (int i = threadIdx.x; i < W.n_thr; i += blockDim.x) thr[i] = W.thr[i];
  for (int i = threadIdx.x; i < W.n_cnt; i += blockDim.x) cnt[i] = W.cnt[i];
  for (int i = threadIdx.x; i < nd; i += blockDim.x) D[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int G = A.G, O = A.O;
  for (long long sl = gwarp; sl < A.count; sl += nwarps) {
    const long long s = A.first + sl;
    const long long split = s % A.sd.n_splits;
    const uint32_t om = scored_mask(A.sd, split, O);
    const uint32_t trained = A.trained[sl];
    int olist[CMAX];
#pragma unroll
    for (int q = 0; q < CMAX; ++q) olist[q] = -1;
    {
      uint32_t mm = om;
#pragma unroll
      for (int q = 0; q < CMAX; ++q)
        if (mm) {
          olist[q] = __ffs(mm) - 1;
          mm &= mm - 1;
        }
    }
    const double* ext = A.extab + sl * A.ex_stride;
    #pragma unroll 1
    for (int g = 0; g < G; ++g) {
      uint64_t tr, te;
      member_words(A.sd, split, g, tr, te);
      if (te == 0ull) continue;
      const int gi = test_group_index(A.sd, split, g);
      const int p = g / A.IR;
      for (int h = 0; h < 2; ++h) {
        const int v = h * 32 + lane;
        if (!((te >> v) & 1ull)) continue;
        // candidates in id order, then a stable insertion sort on EX desc
        double ce[CMAX];
        int hit[CMAX];
        int nc = 0;
#pragma unroll
        for (int q = 0; q < CMAX; ++q) {
          const int o = olist[q];
          const int b = o >= 0 ? A.opt_bit[p * O + o] : -1;
          if (o >= 0 && b >= 0 && !((v >> b) & 1) && ((trained >> o) & 1u)) {
            const int k = rmv(v, b);
            ce[nc] = fabs(ext[q * A.tg_stride + gi * 32 + k]);
            hit[nc] = A.ylab[(g * O + o) * 32 + k] > 1.0 ? 1 : 0;
            ++nc;
          }
        }
        for (int a = 1; a < nc; ++a) {
          const double e = ce[a];
          const int hh = hit[a];
          int z = a;
          while (z > 0 && ce[z - 1] < e) {     // strict: equal EX keep id order
            ce[z] = ce[z - 1];
            hit[z] = hit[z - 1];
            --z;
          }
          ce[z] = e;
          hit[z] = hh;
        }
        for (int pos = 0; pos < nc; ++pos) {
          int lo = 0, hi = W.n_thr;               // u = #{theta <= e}
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (thr[mid] <= ce[pos]) lo = mid + 1;
            else hi = mid;
          }
          if (lo == 0) break;                     // below every threshold, and so is the rest
          for (int j = 0; j < W.n_cnt; ++j) {
            if (pos >= cnt[j]) continue;
            int* Dr = D + j * (W.n_thr + 1);
            atomicAdd(Dr, 1);
            atomicAdd(Dr + lo, -1);
            if (hit[pos]) {
              int* Dh = D + (W.n_cnt + j) * (W.n_thr + 1);
              atomicAdd(Dh, 1);
              atomicAdd(Dh + lo, -1);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // prefix sums over thresholds -> totals
  for (int r = threadIdx.x; r < 2 * W.n_cnt; r += blockDim.x) {
    const int* Dr = D + r * (W.n_thr + 1);
    const int kind = r / W.n_cnt, j = r % W.n_cnt;
    long long run = 0;
    for (int i = 0; i < W.n_thr; ++i) {
      run += Dr[i];
      if (run) atomicAdd(&W.out[((long long)kind * W.n_thr + i) * W.n_cnt + j], (unsigned long long)run);
    }
  }
}

// C5: per-mask rows + ranking keys (O8) from the integer accumulators.
__global__ void k_mask_final(const EvalArgs A) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < A.n_mask_range;
       i += (long long)gridDim.x * blockDim.x) {
    const int* a = A.mask_acc + i * 4;
    MaskScore ms{a[0], a[1], a[2], a[3]};
    if (A.mask_out) A.mask_out[i] = ms;
    const long long mask_id = A.mask0 + i;
    A.keys_out[i] = ((unsigned long long)(unsigned)a[0] << 32) | (0xFFFFFFFFull - (unsigned long long)mask_id);
  }
}

}  // namespace speedrec
