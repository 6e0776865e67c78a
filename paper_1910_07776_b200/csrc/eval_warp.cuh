// eval_warp.cuh -- k_eval_warp: one warp = one scenario, A1..A7 fused.
// Paper passages per step are cited inline; the numerics (dual/primal choice,
// refinement) are argued in DESIGN.md §5.3.
#pragma once
#include "kernels.cuh"
#include "fit_fast.cuh"

namespace speedrec {

// View of one fit's operands: training rows are tr_slot[0..n), active
// features col[0..deff) with centring xb and scale s (1/range).
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

// Element (r, k) of the contraction operand Z (m x L).  Dual (kernel) form:
// Z = Xtilde (rows = training rows, k = features).  Primal form: Z = Xtilde^T.
// Xtilde_ia = (x_ia - xbar_a) * s_a: the min-max scaled, centred feature
// (the min cancels under centring; reading D3).
template <bool DUAL>
__device__ __forceinline__ double zval(const FitView& f, int r, int k) {
  int i = DUAL ? r : k, a = DUAL ? k : r;
  if (i < f.n && a < f.deff) return (f.X[(long long)f.trs[i] * f.ldx + f.col[a]] - f.xb[a]) * f.s[a];
  return 0.0;
}

// Packed lower triangle of Z Z^T + lambda I (m x m), 8x8 tiles on DMMA.
// All 32 lanes execute every mma (warp-uniform loops).
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

// In-place Cholesky of the packed lower triangle, rsqrt pivots.
// invd[j] = 1 / L_jj.  Returns false if a pivot is not positive.
__device__ bool chol_packed(double* M, double* invd, int m, int lane) {
  for (int j = 0; j < m; ++j) {
    const double djj = M[pk(j, j)];
    __syncwarp();
    if (!(djj > 0.0)) return false;
    const double r = rsqrt(djj);
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

// z <- (L L^T)^{-1} z, z in shared memory.
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

// out_a = s_a * sum_i (x_ia - xb_a) * v_i   (= Xtilde^T v), lanes over features.
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

// out_i = sum_a (x_ia - xb_a) * u_a   (= Xtilde w with u = s .* w), lanes over rows.
__device__ __forceinline__ double row_dot_u(const FitView& f, const double* xrow, const double* u) {
  double acc = 0.0;
  for (int a = 0; a < f.deff; ++a) acc = fma(xrow[f.col[a]] - f.xb[a], u[a], acc);
  return acc;
}

template <int CMAX>
__global__ void __launch_bounds__(kMaxWarpsPerBlock * 32, 1) k_eval_warp(const EvalArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const WarpLayout& L = A.L;
  int8_t* obit = reinterpret_cast<int8_t*>(smem);
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int i = tid; i < A.P * A.O; i += nthr) obit[i] = A.opt_bit[i];
  const double* X = A.x;
  int ldx = A.C;
  if (A.stage_x) {
    double* xs = reinterpret_cast<double*>(smem + A.off_stage);
    const long long tot = (long long)A.G * 64 * A.C;
    for (long long i = tid; i < tot; i += nthr) xs[(i / A.C) * A.ldxs + (i % A.C)] = A.x[i];
    X = xs;
    ldx = A.ldxs;
  }
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned char* slab = smem + A.off_warps + warp * L.bytes;
  uint64_t* trw = reinterpret_cast<uint64_t*>(slab + L.off_trw);
  uint64_t* tew = reinterpret_cast<uint64_t*>(slab + L.off_tew);
  int16_t* gidx = reinterpret_cast<int16_t*>(slab + L.off_gidx);
  int16_t* F = reinterpret_cast<int16_t*>(slab + L.off_F);
  double* extab = reinterpret_cast<double*>(slab + L.off_ex);
  uint8_t* excl = reinterpret_cast<uint8_t*>(slab + L.off_excl);
  int32_t* trs = reinterpret_cast<int32_t*>(slab + L.off_trs);
  double* tr_y = reinterpret_cast<double*>(slab + L.off_try);
  int32_t* tes = reinterpret_cast<int32_t*>(slab + L.off_tes);
  int32_t* tek = reinterpret_cast<int32_t*>(slab + L.off_tek);
  double* te_y = reinterpret_cast<double*>(slab + L.off_tey);
  int16_t* col = reinterpret_cast<int16_t*>(slab + L.off_col);
  double* xb = reinterpret_cast<double*>(slab + L.off_xb);
  double* sv = reinterpret_cast<double*>(slab + L.off_s);
  double* wv = reinterpret_cast<double*>(slab + L.off_w);
  double* uv = reinterpret_cast<double*>(slab + L.off_u);
  double* v1 = reinterpret_cast<double*>(slab + L.off_v1);
  double* v2 = reinterpret_cast<double*>(slab + L.off_v2);
  double* v3 = reinterpret_cast<double*>(slab + L.off_v3);
  double* invd = reinterpret_cast<double*>(slab + L.off_invd);
  double* Msm = reinterpret_cast<double*>(slab + L.off_M);
  double* ufull = reinterpret_cast<double*>(slab + L.off_ufull);

  const long long gwarp = (long long)blockIdx.x * A.warps_per_block + warp;
  const long long nwarps = (long long)gridDim.x * A.warps_per_block;
  double* Mgl = A.gscratch ? A.gscratch + gwarp * A.mscratch : nullptr;
  const int G = A.G, O = A.O, C = A.C;
  unsigned long long tot_corr = 0, tot_test = 0, tot_rec = 0, tot_hit = 0;  // lane 0

  // Work item = one scenario, or (C5 aggregation) one feature mask with all
  // its folds, whose per-mask sums are reduced in registers (A7).
  const long long n_items = A.agg ? A.count / A.n_splits : A.count;
  const long long n_inner = A.agg ? A.n_splits : 1;
  for (long long item = gwarp; item < n_items; item += nwarps) {
  int m_corr = 0, m_test = 0, m_rec = 0, m_hit = 0;
  for (long long inner = 0; inner < n_inner; ++inner) {
    const long long sl = A.agg ? item * A.n_splits + inner : item;
    const long long s = A.first + sl;
    const long long split = s % A.n_splits, fidx = s / A.n_splits;

    // ---- A1: split membership words per group (Table 2; R17) ----
    for (int g = lane; g < G; g += 32) {
      uint64_t tr = 0, te = 0;
      if (A.kind == 0) {
        tr = ((A.train_g[split * A.gw + (g >> 6)] >> (g & 63)) & 1ull) ? ~0ull : 0ull;
        te = ((A.test_g[split * A.gw + (g >> 6)] >> (g & 63)) & 1ull) ? ~0ull : 0ull;
      } else if (A.kind == 1) {
        bool inpool = false;
        for (int q = 0; q < A.n_pool; ++q) inpool |= (A.pool_list[q] == g);
        tr = inpool ? ~0ull : 0ull;
        const int gh = A.pool_list[split >> 6];
        const int vh = (int)(split & 63);
        if (g == gh) {
          tr &= ~(1ull << vh);
          te = 1ull << vh;
        }
      } else {
        tr = mix64(mix64(A.seed ^ mix64((uint64_t)split)) + (uint64_t)g);
        te = ~tr;
      }
      trw[g] = tr;
      tew[g] = te;
    }
    // feature set F, counter-index order
    int d = 0;
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      bool in = false;
      if (c < C) {
        if (A.subsets_k > 0) in = c < A.subsets_k && ((fidx >> c) & 1);
        else if (A.fmasks) in = (A.fmasks[fidx * 2 + (c >> 6)] >> (c & 63)) & 1ull;
        else in = true;
      }
      const unsigned bm = __ballot_sync(FULL, in);
      if (in) F[d + __popc(bm & lt)] = (int16_t)c;
      d += __popc(bm);
    }
    __syncwarp();
    // test-group index
    int n_tg = 0;
    for (int g0 = 0; g0 < G; g0 += 32) {
      const int g = g0 + lane;
      const bool has = g < G && tew[g] != 0ull;
      const unsigned bm = __ballot_sync(FULL, has);
      if (g < G) gidx[g] = has ? (int16_t)(n_tg + __popc(bm & lt)) : (int16_t)-1;
      n_tg += __popc(bm);
    }
    const uint32_t om = (A.split_om ? A.split_om[split] : A.opt_mask) & ((1u << O) - 1u);
    const int exs = n_tg * 32;  // EX table stride per optimization
    // zero the optional debug slabs
    if (A.ex_out) {
      double* e = A.ex_out + sl * (long long)O * G * 32;
      for (int i = lane; i < O * G * 32; i += 32) e[i] = 0.0;
    }
    if (A.rec_out) {
      int8_t* r = A.rec_out + sl * (long long)G * 64 * A.max_count;
      for (int i = lane; i < G * 64 * A.max_count; i += 32) r[i] = -1;
    }
    __syncwarp();

    int guard = 0;        // lane-partial guard count
    int untrained = 0;    // lane 0 only
    uint32_t trained = 0;
    int oi = 0;
    int8_t olist[kMaxOpt];
#pragma unroll
    for (int q = 0; q < kMaxOpt; ++q) olist[q] = -1;

    for (int o = 0; o < O; ++o) {
      OptScore row;
      row.n_train = row.n_test = row.n_correct = row.n_clamped = 0;
      row.sum_ratio = row.min_ratio = row.max_ratio = 0.0;
      row.fp_train = row.fp_test = 0ull;
      if (!((om >> o) & 1u)) {
        if (lane == 0 && A.opt_out) A.opt_out[sl * O + o] = row;
        continue;
      }
      const int my_oi = oi++;
#pragma unroll
      for (int q = 0; q < kMaxOpt; ++q)
        if (q == my_oi) olist[q] = (int8_t)o;

      // ---- A1: before/after pairs by ballot compaction ----
      int n = 0, nt = 0;
      uint64_t fptr = 0, fpte = 0;
      for (int g = 0; g < G; ++g) {
        const int b = obit[(g / A.IR) * O + o];
        const uint64_t tr = trw[g], te = tew[g];
        if (b < 0 || (tr == 0ull && te == 0ull)) continue;
        const int k = lane, v = ins0(k, b);
        const bool istr = ((tr >> v) & 1ull) && ((tr >> (v | (1 << b))) & 1ull);
        const bool iste = (te >> v) & 1ull;
        const unsigned mtr = __ballot_sync(FULL, istr), mte = __ballot_sync(FULL, iste);
        const int lab = (g * O + o) * 32 + k;
        if (istr | iste) {
          const uint64_t h = mix64((uint64_t)lab);
          const double y = A.ylab[lab];
          if (istr) {
            const int p = n + __popc(mtr & lt);
            trs[p] = g * 64 + v;
            tr_y[p] = y;
            fptr ^= h;
          }
          if (iste) {
            const int p = nt + __popc(mte & lt);
            tes[p] = g * 64 + v;
            tek[p] = g * 32 + k;
            te_y[p] = y;
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
      if (n == 0) {                      // untrained (reading R18)
        untrained += nt;
        if (lane == 0 && A.opt_out) A.opt_out[sl * O + o] = row;
        continue;
      }
      trained |= 1u << o;
      if (nt == 0) {
        if (lane == 0 && A.opt_out) A.opt_out[sl * O + o] = row;
        continue;
      }

      // ---- A2: per-fit min-max statistics over the training befores ----
      int deff = 0;
      for (int a0 = 0; a0 < d; a0 += 32) {
        const int a = a0 + lane;
        double mn = 0.0, mx = 0.0, sm = 0.0;
        int c = 0;
        if (a < d) {
          c = F[a];
          mn = mx = X[(long long)trs[0] * ldx + c];
          sm = mn;
          for (int i = 1; i < n; ++i) {
            const double vv = X[(long long)trs[i] * ldx + c];
            mn = fmin(mn, vv);
            mx = fmax(mx, vv);
            sm += vv;
          }
        }
        const bool act = a < d && mx > mn;
        const unsigned bm = __ballot_sync(FULL, act);
        if (act) {
          const int p = deff + __popc(bm & lt);
          col[p] = (int16_t)c;
          xb[p] = sm / (double)n;
          sv[p] = 1.0 / (mx - mn);
        }
        deff += __popc(bm);
      }
      {  // zero padding read by the fast-path fragment loads
        const int pad_end = max(32, (deff + 3) & ~3);
        for (int p = deff + lane; p < pad_end; p += 32) {
          col[p] = 0;
          xb[p] = 0.0;
          sv[p] = 0.0;
        }
      }
      double ysum = 0.0;
      for (int i = lane; i < n; i += 32) ysum += tr_y[i];
      const double ybar = warp_sum(ysum) / (double)n;
      for (int i = lane; i < n; i += 32) v3[i] = tr_y[i] - ybar;
      __syncwarp();

      // ---- A3/A4: centred normal equations, dual or primal ----
      const bool dual = (n - 1) < deff;
      const int m = dual ? n : deff;
      // refinement only where the conditioning needs it
      const int nref = (dual ? 2 * (n - 1) >= deff : (n - 1) < 2 * deff) ? A.refine : 0;
      bool ok = true;
      if (m > 0 && m <= (L.mcap < 32 ? L.mcap : 32)) {
        const FastView fv{X, ldx, trs, n, col, xb, sv, deff};
        ok = dual ? fit_fast<true>(fv, v3, A.lambda, nref, Msm, v2, uv, wv, lane)
                  : fit_fast<false>(fv, v3, A.lambda, nref, Msm, v2, uv, wv, lane);
      } else if (m > 0) {
        FitView f{X, ldx, trs, n, col, xb, sv, deff};
        double* M = (m <= L.mcap) ? Msm : Mgl;
        if (dual) build_gram<true>(M, m, deff, f, A.lambda, lane);
        else build_gram<false>(M, m, n, f, A.lambda, lane);
        ok = chol_packed(M, invd, m, lane);
        if (ok && dual) {
          // alpha = (K + lambda I)^{-1} yc ;  w' = Xtilde^T alpha
          for (int i = lane; i < n; i += 32) v1[i] = v3[i];
          __syncwarp();
          chol_solve(M, invd, v1, m, lane);
          for (int it = 0; it < nref; ++it) {
            xt_times(f, v1, wv, lane);
            for (int a = lane; a < deff; a += 32) uv[a] = wv[a] * sv[a];
            __syncwarp();
            for (int i = lane; i < n; i += 32) {
              const double* xr = X + (long long)trs[i] * ldx;
              v2[i] = v3[i] - row_dot_u(f, xr, uv) - A.lambda * v1[i];
            }
            __syncwarp();
            chol_solve(M, invd, v2, m, lane);
            for (int i = lane; i < n; i += 32) v1[i] += v2[i];
            __syncwarp();
          }
          xt_times(f, v1, wv, lane);
        } else if (ok) {
          // w' = (G + lambda I)^{-1} Xtilde^T yc
          xt_times(f, v3, wv, lane);
          chol_solve(M, invd, wv, m, lane);
          for (int it = 0; it < nref; ++it) {
            for (int a = lane; a < deff; a += 32) uv[a] = wv[a] * sv[a];
            __syncwarp();
            for (int i = lane; i < n; i += 32) {
              const double* xr = X + (long long)trs[i] * ldx;
              v2[i] = v3[i] - row_dot_u(f, xr, uv);
            }
            __syncwarp();
            xt_times(f, v2, v1, lane);
            for (int a = lane; a < deff; a += 32) v1[a] -= A.lambda * wv[a];
            __syncwarp();
            chol_solve(M, invd, v1, m, lane);
            for (int a = lane; a < deff; a += 32) wv[a] += v1[a];
            __syncwarp();
          }
        }
      }
      if (!ok) guard += 1000000;  // unreachable for lambda > 0; poisons the row
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
      const double c0 = ybar - warp_sum(cpart);
      __syncwarp();

      // ---- A5: predict + clamp; A7 per-(s,o) scores ----
      const int oiex = my_oi * exs;
      int ncorr = 0, ncl = 0;
      double rsum = 0.0, rmin = INFINITY, rmax = -INFINITY;
      for (int j = lane; j < nt; j += 32) {
        const double* xr = X + (long long)tes[j] * ldx;
        double e0 = 0.0, e1 = 0.0;
        int c = 0;
        for (; c + 1 < C; c += 2) {
          e0 = fma(xr[c], ufull[c], e0);
          e1 = fma(xr[c + 1], ufull[c + 1], e1);
        }
        if (c < C) e0 = fma(xr[c], ufull[c], e0);
        double e = c0 + (e0 + e1);
        if (near_tol(e, 0.0, A.guard_tol) || near_tol(e, 1.0, A.guard_tol)) ++guard;
        uint8_t cl = 0;
        if (e <= 0.0) { e = A.clamp_floor; cl = 1; ++ncl; }
        const double ac = te_y[j];
        ncorr += ((e > 1.0 && ac > 1.0) || (e <= 1.0 && ac <= 1.0)) ? 1 : 0;
        const double ratio = ac / e;
        rsum += ratio;
        rmin = fmin(rmin, ratio);
        rmax = fmax(rmax, ratio);
        const int gk = tek[j];
        const int gi = gidx[gk >> 5];
        extab[oiex + gi * 32 + (gk & 31)] = e;
        excl[oiex + gi * 32 + (gk & 31)] = cl;
        if (A.ex_out) A.ex_out[(sl * O + o) * (long long)G * 32 + gk] = e;
      }
      row.n_correct = warp_isum(ncorr);
      row.n_clamped = warp_isum(ncl);
      row.sum_ratio = warp_sum(rsum);
      row.min_ratio = warp_min(rmin);
      row.max_ratio = warp_max(rmax);
      tot_corr += row.n_correct;
      tot_test += nt;
      m_corr += row.n_correct;
      m_test += nt;
      if (lane == 0 && A.opt_out) A.opt_out[sl * O + o] = row;
      __syncwarp();
    }

    // ---- A6: rank + thresholded recommendation per test slot ----
    int nrec = 0, nhit = 0;
    const int n_os = oi;
    for (int g = 0; g < G; ++g) {
      const uint64_t te = tew[g];
      if (te == 0ull) continue;
      const int gi = gidx[g];
      const int p = g / A.IR;
      for (int h = 0; h < 2; ++h) {
        const int v = h * 32 + lane;
        if (!((te >> v) & 1ull)) continue;
        double ce[CMAX];
        bool cv[CMAX], cc[CMAX];
        int co[CMAX], ck[CMAX];
#pragma unroll
        for (int q = 0; q < CMAX; ++q) {
          const int o = (q < kMaxOpt) ? olist[q] : -1;
          bool valid = q < n_os && o >= 0 && ((trained >> o) & 1u);
          int b = -1;
          if (valid) {
            b = obit[p * O + o];
            valid = b >= 0 && !((v >> b) & 1);
          }
          cv[q] = valid;
          co[q] = o;
          ck[q] = valid ? rmv(v, b) : 0;
          ce[q] = valid ? extab[q * exs + gi * 32 + ck[q]] : 0.0;
          cc[q] = valid ? excl[q * exs + gi * 32 + ck[q]] != 0 : false;
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
        // rank among candidates with EX >= threshold: (EX desc, id asc)
#pragma unroll
        for (int q = 0; q < CMAX; ++q) {
          if (!cv[q] || !(ce[q] >= A.threshold)) continue;
          int rk = 0;
#pragma unroll
          for (int r = 0; r < CMAX; ++r)
            if (r != q && cv[r] && ce[r] >= A.threshold && (ce[r] > ce[q] || (ce[r] == ce[q] && r < q))) ++rk;
          if (rk < A.max_count) {
            ++nrec;
            const int o = co[q];
            if (A.ylab[(g * O + o) * 32 + ck[q]] > 1.0) ++nhit;
            if (A.rec_out)
              A.rec_out[(sl * G * 64 + g * 64 + v) * A.max_count + rk] = (int8_t)o;
          }
        }
      }
    }
    ScnScore sr;
    sr.n_rec = warp_isum(nrec);
    sr.n_rec_hit = warp_isum(nhit);
    sr.n_untrained = untrained;
    sr.n_guard = warp_isum(guard);
    tot_rec += sr.n_rec;
    tot_hit += sr.n_rec_hit;
    m_rec += sr.n_rec;
    m_hit += sr.n_rec_hit;
    if (lane == 0 && A.scn_out) A.scn_out[sl] = sr;
    __syncwarp();
  }  // inner (folds)
  if (A.agg && lane == 0) {
    const long long mask_id = A.first / A.n_splits + item;
    MaskScore ms{m_corr, m_test, m_rec, m_hit};
    if (A.mask_out) A.mask_out[item] = ms;
    // top-K key: more correct first, then smaller mask id (O8)
    A.keys_out[item] = ((unsigned long long)(unsigned)m_corr << 32) | (0xFFFFFFFFull - (unsigned long long)mask_id);
  }
  }  // items
  if (A.totals && lane == 0 && (tot_test | tot_rec)) {
    atomicAdd(&A.totals[0], tot_corr);
    atomicAdd(&A.totals[1], tot_test);
    atomicAdd(&A.totals[2], tot_rec);
    atomicAdd(&A.totals[3], tot_hit);
  }
}

}  // namespace speedrec
