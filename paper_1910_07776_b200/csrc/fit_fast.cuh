// fit_fast.cuh -- fast path of one ridge fit (A3-A4) for systems of size
// m <= 32 (dual m = n training pairs, primal m = d_eff active features),
// one warp per fit.  DESIGN.md §5.3.
//
//  * Gram: all NB = ceil(m/8) row-block fragments of the centred, scaled
//    operand are formed once per k-step (x from shared memory, index math
//    hoisted) and every lower 8x8 tile is accumulated on DMMA.8x8x4 in
//    registers (templated on NB only -- the rest is compact loop code, the
//    kernel must stay inside the instruction cache).
//  * Factorisation: right-looking LDL^T-form Cholesky in shared memory with
//    unscaled columns: step j only reads column j (final) and rewrites the
//    lane's own row, so one __syncwarp per pivot; rsqrt pivots.
//  * Solves: vectors lane-owned (lane i holds element i), pivots broadcast by
//    shuffle, factor entries read from shared memory.
//  * Refinement (adaptive): residual from the data rows.
#pragma once
#include "kernels.cuh"

namespace speedrec {

struct FastView {
  const double* X;   // rates (row stride ldx), staged in smem when small
  int ldx;
  const int32_t* trs;
  int n;
  const int16_t* col;  // [>= max(32, round4(deff))], zero padded
  const double* xb;
  const double* s;
  int deff;
};

// Packed lower triangle of Z Z^T + lambda I; Z = Xtilde (dual) or Xtilde^T.
template <int NB, bool DUAL>
__device__ __forceinline__ void gram_fast(const FastView& f, int m, double lambda, double* Mpk, int lane) {
  constexpr int NT = NB * (NB + 1) / 2;
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int rl = lane >> 2, kl = lane & 3;
  if (DUAL) {
    int so[NB];
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      const int r = I * 8 + rl;
      so[I] = r < f.n ? f.trs[r] * f.ldx : -1;
    }
#pragma unroll 2
    for (int k0 = 0; k0 < f.deff; k0 += 4) {
      const int ka = k0 + kl;
      const int c = f.col[ka];
      const double xbv = f.xb[ka], sv = f.s[ka];
      double fr[NB];
#pragma unroll
      for (int I = 0; I < NB; ++I) fr[I] = so[I] >= 0 ? (f.X[so[I] + c] - xbv) * sv : 0.0;
      int t = 0;
#pragma unroll
      for (int I = 0; I < NB; ++I)
#pragma unroll
        for (int J = 0; J <= I; ++J, ++t) dmma(acc[t][0], acc[t][1], fr[I], fr[J]);
    }
  } else {
    int ca[NB];
    double xba[NB], sa[NB];
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      const int a = I * 8 + rl;
      ca[I] = f.col[a];
      xba[I] = f.xb[a];
      sa[I] = f.s[a];
    }
#pragma unroll 2
    for (int i0 = 0; i0 < f.n; i0 += 4) {
      const int ri = i0 + kl;
      const int so = ri < f.n ? f.trs[ri] * f.ldx : -1;
      double fr[NB];
#pragma unroll
      for (int I = 0; I < NB; ++I) fr[I] = so >= 0 ? (f.X[so + ca[I]] - xba[I]) * sa[I] : 0.0;
      int t = 0;
#pragma unroll
      for (int I = 0; I < NB; ++I)
#pragma unroll
        for (int J = 0; J <= I; ++J, ++t) dmma(acc[t][0], acc[t][1], fr[I], fr[J]);
    }
  }
  int t = 0;
#pragma unroll
  for (int I = 0; I < NB; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J, ++t) {
      const int r = I * 8 + rl;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = J * 8 + 2 * kl + e;
        if (r < m && c <= r) Mpk[pk(r, c)] = acc[t][e] + (r == c ? lambda : 0.0);
      }
    }
  __syncwarp();
}

template <bool DUAL>
__device__ __noinline__ void gram_fast_dispatch(const FastView& f, int m, double lambda, double* Mpk, int lane) {
  if (m <= 8) gram_fast<1, DUAL>(f, m, lambda, Mpk, lane);
  else if (m <= 16) gram_fast<2, DUAL>(f, m, lambda, Mpk, lane);
  else if (m <= 24) gram_fast<3, DUAL>(f, m, lambda, Mpk, lane);
  else gram_fast<4, DUAL>(f, m, lambda, Mpk, lane);
}

// LDL^T-form Cholesky of the packed lower triangle, m <= 32, unscaled columns:
// on exit M[i][j] (i > j) = L_ij * L_jj, and the lane's 1/L_ii is returned in
// myinv (lane i < m).  Lane i owns row i.  Returns false on a non-positive pivot.
__device__ __noinline__ bool chol_ldl(double* M, int m, int lane, double& myinv) {
  bool ok = true;
  myinv = 0.0;
  const int rb = (lane * (lane + 1)) >> 1;
  for (int j = 0; j < m; ++j) {
    const double djj = M[((j * (j + 1)) >> 1) + j];
    ok = ok && djj > 0.0;
    const double r = rsqrt(djj);
    if (lane == j) myinv = r;
    if (lane > j && lane < m) {
      const double sij = M[rb + j] * (r * r);
      int k = j + 1;
      for (; k + 1 <= lane; k += 2) {
        const double a0 = M[((k * (k + 1)) >> 1) + j], a1 = M[(((k + 1) * (k + 2)) >> 1) + j];
        M[rb + k] = fma(-sij, a0, M[rb + k]);
        M[rb + k + 1] = fma(-sij, a1, M[rb + k + 1]);
      }
      if (k <= lane) M[rb + k] = fma(-sij, M[((k * (k + 1)) >> 1) + j], M[rb + k]);
    }
    __syncwarp();
  }
  return ok;
}

// z <- (L L^T)^{-1} z for the chol_ldl factor; z lane-owned, m <= 32.
__device__ __noinline__ double solve_ldl(const double* M, int m, int lane, double myinv, double z) {
  const int rb = (lane * (lane + 1)) >> 1;
  for (int j = 0; j < m; ++j) {                     // forward: L y = z
    if (lane == j) z *= myinv;
    const double t = __shfl_sync(FULL, z * myinv, j);  // y_j / L_jj
    if (lane > j && lane < m) z = fma(-M[rb + j], t, z);
  }
  double acc = 0.0;
  for (int j = m - 1; j >= 0; --j) {                // backward: L^T x = y
    if (lane == j) z = (z - myinv * acc) * myinv;
    const double xj = __shfl_sync(FULL, z, j);
    if (lane < j) acc = fma(M[((j * (j + 1)) >> 1) + lane], xj, acc);
  }
  return z;
}

// w'_a = s_a * sum_i (x_ia - xb_a) * alpha_i, alpha lane-owned (n <= 32);
// lanes over features, written to wout[0..deff).
__device__ __noinline__ void xt_alpha_lanes(const FastView& f, double alpha, double* wout, int lane) {
  for (int a0 = 0; a0 < f.deff; a0 += 64) {
    const int a1 = a0 + lane, a2 = a0 + 32 + lane;
    const int c1 = f.col[a1 < f.deff ? a1 : 0], c2 = f.col[a2 < f.deff ? a2 : 0];
    const double x1 = f.xb[a1 < f.deff ? a1 : 0], x2 = f.xb[a2 < f.deff ? a2 : 0];
    double acc1 = 0.0, acc2 = 0.0;
    for (int i = 0; i < f.n; ++i) {
      const double ai = __shfl_sync(FULL, alpha, i);
      const double* xr = f.X + f.trs[i] * f.ldx;
      acc1 = fma(xr[c1] - x1, ai, acc1);
      acc2 = fma(xr[c2] - x2, ai, acc2);
    }
    if (a1 < f.deff) wout[a1] = acc1 * f.s[a1];
    if (a2 < f.deff) wout[a2] = acc2 * f.s[a2];
  }
  __syncwarp();
}

// sum_a (x_ra - xb_a) * u_a for the row at xr (u = s .* w'), serial over features.
__device__ __forceinline__ double xrow_dot(const FastView& f, const double* xr, const double* u) {
  double acc = 0.0;
  for (int a = 0; a < f.deff; ++a) acc = fma(xr[f.col[a]] - f.xb[a], u[a], acc);
  return acc;
}

// One fit on the fast path (m <= 32).  yc: y - ybar per training row (smem [n]).
// Output: w' (weights on the scaled features) in wout[0..deff).
// scratch: [n] doubles for the primal residual; uwork: [deff].
template <bool DUAL>
__device__ bool fit_fast(const FastView& f, const double* yc, double lambda, int refine, double* Mpk,
                         double* scratch, double* uwork, double* wout, int lane) {
  const int m = DUAL ? f.n : f.deff;
  gram_fast_dispatch<DUAL>(f, m, lambda, Mpk, lane);
  double myinv;
  const bool ok = chol_ldl(Mpk, m, lane, myinv);
  if (DUAL) {
    double alpha = lane < f.n ? yc[lane] : 0.0;
    alpha = solve_ldl(Mpk, m, lane, myinv, alpha);
    for (int it = 0; it < refine; ++it) {
      xt_alpha_lanes(f, alpha, wout, lane);
      for (int a = lane; a < f.deff; a += 32) uwork[a] = wout[a] * f.s[a];
      __syncwarp();
      double e = 0.0;
      if (lane < f.n) e = yc[lane] - xrow_dot(f, f.X + f.trs[lane] * f.ldx, uwork) - lambda * alpha;
      alpha += solve_ldl(Mpk, m, lane, myinv, e);
      __syncwarp();
    }
    xt_alpha_lanes(f, alpha, wout, lane);
  } else {
    // rhs_a = s_a * sum_i (x_ia - xb_a) * yc_i, lane a < deff <= 32
    double w = 0.0;
    if (lane < f.deff) {
      const int c = f.col[lane];
      const double x0 = f.xb[lane];
      for (int i = 0; i < f.n; ++i) w = fma(f.X[f.trs[i] * f.ldx + c] - x0, yc[i], w);
      w *= f.s[lane];
    }
    w = solve_ldl(Mpk, m, lane, myinv, w);
    for (int it = 0; it < refine; ++it) {
      if (lane < f.deff) uwork[lane] = w * f.s[lane];
      __syncwarp();
      for (int i = lane; i < f.n; i += 32) scratch[i] = yc[i] - xrow_dot(f, f.X + f.trs[i] * f.ldx, uwork);
      __syncwarp();
      double r = 0.0;
      if (lane < f.deff) {
        const int c = f.col[lane];
        const double x0 = f.xb[lane];
        for (int i = 0; i < f.n; ++i) r = fma(f.X[f.trs[i] * f.ldx + c] - x0, scratch[i], r);
        r = r * f.s[lane] - lambda * w;
      }
      w += solve_ldl(Mpk, m, lane, myinv, r);
      __syncwarp();
    }
    if (lane < f.deff) wout[lane] = w;
    __syncwarp();
  }
  return ok;
}

}  // namespace speedrec
