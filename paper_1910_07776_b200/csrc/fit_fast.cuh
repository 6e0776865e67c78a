// fit_fast.cuh -- fast path of one ridge fit (A3-A4) for systems of size
// m <= 32 (dual m = n training pairs, primal m = d_eff active features),
// one warp per fit.  DESIGN.md §5.3.
//
//  * Gram: all NB = ceil(m/8) row-block fragments of the centred, scaled
//    operand are formed once per k-step (x from shared memory, index math
//    hoisted) and every lower 8x8 tile is accumulated on DMMA.8x8x4 in
//    registers (templated on NB only -- the rest is compact loop code, the
//    kernel must stay inside the instruction cache).
//  * Factorisation: left-looking (Crout) Cholesky in shared memory, rows
//    16-byte aligned (rb2 layout) so the row-prefix dot products use 128-bit
//    loads; one __syncwarp per pivot; rsqrt pivots.
//  * Solves: vectors lane-owned (lane i holds element i), pivots broadcast by
//    shuffle, factor entries read from shared memory.
//  * Refinement (adaptive): residual from the data rows.
#pragma once
#include "kernels.cuh"

// Fast-path helpers are inlined by default; -DSPEEDREC_NOINLINE_FAST=1 keeps
// them out of line (A/B of code size vs call overhead, tools/ab_variants.sh).
#if SPEEDREC_NOINLINE_FAST
#define SR_FAST_FN __noinline__
#else
#define SR_FAST_FN __forceinline__
#endif

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
  unsigned xs32;     // staged rates: 32-bit shared-window address of X (SX instantiations)
};

// Rate at byte offset `off` of X: a 32-bit ld.shared when the rates are staged
// (SX), else a generic load.  The staged rates are read-only after the
// kernel's staging barrier, so the asm needs no memory clobber.
template <bool SX>
__device__ __forceinline__ double xload(const double* X, unsigned xs32, int off) {
  if (SX) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(xs32 + (unsigned)off));
    return v;
  }
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(X) + off);
}
template <bool SX>
__device__ __forceinline__ double xat(const FastView& f, int off) { return xload<SX>(f.X, f.xs32, off); }

// Lower triangle (rb2 row layout) of Z Z^T + lambda I; Z = Xtilde (dual) or
// Xtilde^T (primal), NB = ceil(m/8) row-blocks (one compact k-loop per NB,
// chosen outside the loop: no warp-uniform branches or address rebuilds inside).
// Fragments: lane (rl, kl) forms Z[I*8 + rl][k0 + kl] = (x - xbar) * s.
template <bool DUAL, bool SX, int NB>
__device__ __forceinline__ void gram_acc(const FastView& f, double (&acc)[10][2], int lane) {
  const int rl = lane >> 2, kl = lane & 3;
  const int ldx8 = f.ldx * 8;
  int ro[NB];                        // DUAL: byte offset of row I*8+rl
  int co[NB];                        // primal: byte offset of column (feature) I*8+rl
  double xba[NB], sa[NB];
#pragma unroll
  for (int I = 0; I < NB; ++I) {
    const int r = I * 8 + rl;
    if (DUAL) {
      // rows >= n only reach Gram rows/columns >= m, never stored or read
      ro[I] = f.trs[r < f.n ? r : 0] * ldx8;
    } else {
      co[I] = f.col[r] * 8;
      xba[I] = f.xb[r];
      sa[I] = f.s[r];
    }
  }
  const int kend = DUAL ? f.deff : f.n;
  #pragma unroll 1
  for (int k0 = 0; k0 < kend; k0 += 4) {
    double fr[NB];
    if (DUAL) {
      const int ka = k0 + kl;
      const int c8 = f.col[ka] * 8;
      const double xbv = f.xb[ka], sv = f.s[ka];
#pragma unroll
      for (int I = 0; I < NB; ++I) fr[I] = (xat<SX>(f, ro[I] + c8) - xbv) * sv;
    } else {
      const int ri = k0 + kl;
      const bool live = ri < f.n;
      const int sr = f.trs[live ? ri : 0] * ldx8;
#pragma unroll
      for (int I = 0; I < NB; ++I) fr[I] = live ? (xat<SX>(f, sr + co[I]) - xba[I]) * sa[I] : 0.0;
    }
    int t = 0;
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int J = 0; J <= I; ++J, ++t) dmma(acc[t][0], acc[t][1], fr[I], fr[J]);
  }
}

template <bool DUAL, bool SX>
__device__ SR_FAST_FN void gram_fast(const FastView& f, int m, double lambda, double* Mpk, int lane) {
  constexpr int NB = 4, NT = 10;
  const int nb = (m + 7) >> 3;
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  if (nb == 1) gram_acc<DUAL, SX, 1>(f, acc, lane);
  else if (nb == 2) gram_acc<DUAL, SX, 2>(f, acc, lane);
  else if (nb == 3) gram_acc<DUAL, SX, 3>(f, acc, lane);
  else gram_acc<DUAL, SX, 4>(f, acc, lane);
  const int rl = lane >> 2, kl = lane & 3;
  int t = 0;
#pragma unroll
  for (int I = 0; I < NB; ++I) {
    if (I < nb) {
      const int r = I * 8 + rl;
      double* Mr = Mpk + rb2(r);
#pragma unroll
      for (int J = 0; J <= I; ++J) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = J * 8 + 2 * kl + e;
          if (r < m && c <= r) Mr[c] = acc[t + J][e] + (r == c ? lambda : 0.0);
        }
      }
    }
    t += I + 1;
  }
  __syncwarp();
}

#if SPEEDREC_CHOL_RL
// A/B variant (compile with -DSPEEDREC_CHOL_RL=1): right-looking LDL^T form in
// the same rb2 layout, unscaled columns; M[i][j] (i > j) = L_ij * L_jj.
__device__ SR_FAST_FN bool chol_rl(double* M, int m, int lane, double& myinv) {
  bool ok = true;
  myinv = 0.0;
  double* ri = M + rb2(lane < m ? lane : 0);
  #pragma unroll 1
  for (int j = 0; j < m; ++j) {
    const double djj = M[rb2(j) + j];
    ok = ok && djj > 0.0;
    const double r = rsqrt_nr(djj);
    if (lane == j) myinv = r;
    if (lane > j && lane < m) {
      const double sij = ri[j] * (r * r);
      for (int k = j + 1; k <= lane; ++k) ri[k] = fma(-sij, M[rb2(k) + j], ri[k]);
    }
    __syncwarp();
  }
  return ok;
}
__device__ SR_FAST_FN double solve_rl(const double* M, int m, int lane, double myinv, double z) {
  const double* ri = M + rb2(lane < m ? lane : 0);
  #pragma unroll 1
  for (int j = 0; j < m; ++j) {
    if (lane == j) z *= myinv;
    const double t = __shfl_sync(FULL, z * myinv, j);
    if (lane > j && lane < m) z = fma(-ri[j], t, z);
  }
  double acc = 0.0;
  #pragma unroll 1
  for (int j = m - 1; j >= 0; --j) {
    if (lane == j) z = (z - myinv * acc) * myinv;
    const double xj = __shfl_sync(FULL, z, j);
    if (lane < j) acc = fma(M[rb2(j) + lane], xj, acc);
  }
  return z;
}
#define chol_ll chol_rl
#define solve_ll solve_rl
#else
// Left-looking (Crout) Cholesky in the 16-byte-aligned row layout rb2(), m <= 32.
// Step j: every lane i >= j forms sum_{k<j} L_ik L_jk from final row prefixes
// (vectorised 16-byte loads, row j broadcast), lane j takes the rsqrt pivot,
// lanes i > j scale.  One __syncwarp per pivot, no stores of partial updates.
// On exit M holds L (scaled); myinv = 1/L_{lane,lane}.
// aug: row m holds a right-hand side b (m < 32); the same column steps turn it
// into y = L^-1 b (forward substitution fused into the factorisation).
#ifndef SPEEDREC_CHOL_BLK
#define SPEEDREC_CHOL_BLK 1
#endif
#ifndef SPEEDREC_CHOL_PAR
#define SPEEDREC_CHOL_PAR 0
#endif
#ifndef SPEEDREC_SOLVE_PAR
#define SPEEDREC_SOLVE_PAR 0
#endif
// Trailing update of chol_ll's blocked form after the 8-column panel
// [P-8, P): M[r][c] -= sum_{k in panel} L_rk L_ck for P <= c <= r, r < mr,
// c < m, as 8x8 DMMA tiles (two k-steps of 4; the B fragment of tile (I, J)
// is block-row J's A fragment, L L^T being symmetric).  Replaces the panel's
// terms in every later column's row-prefix sum.
__device__ SR_FAST_FN void chol_trail(double* M, int P, int m, int mr, int lane) {
  const int rl = lane >> 2, kl = lane & 3;
  const int I0 = P >> 3, nbr = (mr + 7) >> 3, nbc = (m + 7) >> 3;
  double f0[4], f1[4];
#pragma unroll
  for (int I = 0; I < 4; ++I) {
    const int r = I * 8 + rl;
    f0[I] = f1[I] = 0.0;
    if (I >= I0 && I < nbr && r < mr) {
      const double* rp = M + rb2(r) + P - 8 + kl;
      f0[I] = rp[0];
      f1[I] = rp[4];
    }
  }
#pragma unroll
  for (int I = 1; I < 4; ++I) {
    if (I < I0 || I >= nbr) continue;
    const int r = I * 8 + rl;
    double* rowp = M + rb2(r < mr ? r : 0);
#pragma unroll
    for (int J = 1; J <= I; ++J) {
      if (J < I0 || J >= nbc) continue;
      const int c = J * 8 + 2 * kl;
      const bool in = r < mr && c <= r;           // then c + 1 is inside row r's padded length
      const double2 cv = in ? *reinterpret_cast<const double2*>(rowp + c) : make_double2(0.0, 0.0);
      double d0 = cv.x, d1 = cv.y;
      dmma(d0, d1, -f0[I], f0[J]);
      dmma(d0, d1, -f1[I], f1[J]);
      if (in && c < m) rowp[c] = d0;
      if (in && c + 1 <= r && c + 1 < m) rowp[c + 1] = d1;
    }
  }
  __syncwarp();
}

__device__ SR_FAST_FN bool chol_ll(double* M, int m, int lane, double& myinv, bool aug = false) {
  myinv = 0.0;
  const int mr = m + (aug ? 1 : 0);               // rows carried through the column steps
  double* ri = M + rb2(lane < mr ? lane : 0);
  const double* rj = M;                           // row j (j even), advanced two rows per step
  // two columns per step: the row-prefix sums over k < j for columns j and
  // j+1 share the loads of row i; column j+1 then takes the k = j term with
  // L_{j+1,j} from lane j+1.  One __syncwarp per two pivots.  Blocked form
  // (SPEEDREC_CHOL_BLK): at every 8-column boundary the finished panel is
  // subtracted from the trailing matrix on DMMA (chol_trail), so the prefix
  // sums run over the current panel's columns only (<= 6 terms).
  #pragma unroll 1
  for (int j = 0; j < m; j += 2) {
    const double* rj1 = j + 1 < m ? rj + j + 2 : rj;   // row j+1 (row j has padded length j+2)
    double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
#if SPEEDREC_CHOL_BLK
    const int kb = j & ~7;
    if (kb == j && j > 0) chol_trail(M, j, m, mr, lane);
#else
    const int kb = 0;
#endif
    SR_UNROLL(SR_UNROLL_CHOL)
    for (int k = kb; k < j; k += 2) {              // j even: pairs cover [kb, j) exactly
      const double2 a = *reinterpret_cast<const double2*>(ri + k);
      const double2 b = *reinterpret_cast<const double2*>(rj + k);
      const double2 c = *reinterpret_cast<const double2*>(rj1 + k);
      s0 = fma(a.x, b.x, s0);
      s1 = fma(a.y, b.y, s1);
      t0 = fma(a.x, c.x, t0);
      t1 = fma(a.y, c.y, t1);
    }
    // K_ij, K_i,j+1 (row i >= j+1); lanes past the rows (whose ri aliases row
    // 0) read nothing: lane 0 writes row 0 in this step (racecheck-clean)
    const double2 kij = lane < mr ? *reinterpret_cast<const double2*>(ri + j) : make_double2(0.0, 0.0);
    const double v = kij.x - (s0 + s1);           // lane j: pivot; lanes i > j: unscaled L_ij
#if SPEEDREC_CHOL_PAR
    // both pivots of the step from one round of broadcasts: with p_j = v_j,
    // w = v_{j+1,j} and K' = K'_{j+1,j+1} (row-prefix sums applied), the next
    // pivot is p_{j+1} = K' - w^2 / p_j, so 1/L_{j+1,j+1} = rsqrt(K' p_j - w^2)
    // * sqrt(p_j) = rsqrt(K' p_j - w^2) * p_j / L_jj: the two rsqrt chains
    // run side by side instead of one after the other
    const double vj = __shfl_sync(FULL, v, j);
    const double r = rsqrt_nr(vj);                // 1/L_jj in every lane (NaN/inf iff p_j is not > 0)
    const double lij = v * r;
    if (lane >= j && lane < mr) ri[j] = lij;
    if (lane == j) myinv = r;
    if (j + 1 < m) {
      const double kp = kij.y - (t0 + t1);        // lane i: K'_{i,j+1}
      const double w = __shfl_sync(FULL, v, j + 1);
      const double kp1 = __shfl_sync(FULL, kp, j + 1);
      const double r1 = rsqrt_nr(fma(kp1, vj, -(w * w))) * (vj * r);
      const double v1 = kp - lij * (w * r);       // lane j+1: pivot; lanes i > j+1: unscaled L_i,j+1
      if (lane > j && lane < mr) ri[j + 1] = v1 * r1;
      if (lane == j + 1) myinv = r1;
    }
#else
    const double r = __shfl_sync(FULL, rsqrt_nr(v), j);  // 1/L_jj (NaN/inf iff the pivot is not > 0)
    const double lij = v * r;
    if (lane >= j && lane < mr) ri[j] = lij;
    if (lane == j) myinv = r;
    if (j + 1 < m) {
      const double l1 = __shfl_sync(FULL, lij, j + 1);              // L_{j+1,j}
      const double v1 = kij.y - (t0 + t1) - lij * l1;              // lane j+1: pivot
      const double r1 = __shfl_sync(FULL, rsqrt_nr(v1), j + 1);
      if (lane > j && lane < mr) ri[j + 1] = v1 * r1;
      if (lane == j + 1) myinv = r1;
    }
#endif
    rj += 2 * j + 4;                              // row j+2 (rows j, j+1 have padded length j+2)
    __syncwarp();
  }
  // a non-positive pivot makes its 1/L_jj NaN or inf (and NaN propagates to
  // later pivots): one vote at the end instead of a test per step
  return __all_sync(FULL, lane >= m || (myinv > 0.0 && myinv < INFINITY));
}

// z <- L^{-T} z for the chol_ll factor; z lane-owned, m <= 32.
__device__ SR_FAST_FN double solve_bwd(const double* M, int m, int lane, double myinv, double z) {
#if SPEEDREC_SOLVE_PAR
  // two unknowns per step from one round of broadcasts: x_j = z_j / L_jj and
  // x_{j-1} = (z_{j-1} - L_{j,j-1} x_j) / L_{j-1,j-1} in every lane, then
  // lanes i < j-1 take both updates (the 1/L_jj broadcasts and L_{j,j-1}
  // do not depend on z, so they leave the dependency chain)
  int j = m - 1;
  #pragma unroll 1
  for (; j >= 1; j -= 2) {
    const double* rj = M + rb2(j);
    const double* rj1 = M + rb2(j - 1);
    const double ij = __shfl_sync(FULL, myinv, j), ij1 = __shfl_sync(FULL, myinv, j - 1);
    const double ljj1 = rj[j - 1];
    const double lji = lane < j - 1 ? rj[lane] : 0.0, lj1i = lane < j - 1 ? rj1[lane] : 0.0;
    const double zj = __shfl_sync(FULL, z, j), zj1 = __shfl_sync(FULL, z, j - 1);
    const double xj = zj * ij;
    const double xj1 = fma(-ljj1, xj, zj1) * ij1;
    if (lane < j - 1) z = fma(-lj1i, xj1, fma(-lji, xj, z));
    if (lane == j) z = xj;
    if (lane == j - 1) z = xj1;
  }
  if (j == 0 && lane == 0) z *= myinv;
  return z;
#endif
  const double* rj = M + rb2(m - 1) + lane;         // row j, column `lane`
  #pragma unroll 1
  for (int j = m - 1; j >= 0; --j) {                // backward: L^T x = y
    if (lane == j) z *= myinv;
    const double xj = __shfl_sync(FULL, z, j);
    if (lane < j) z = fma(-*rj, xj, z);
    rj -= (j + 1) & ~1;                             // padded length of row j-1
  }
  return z;
}

// z <- (L L^T)^{-1} z for the chol_ll factor; z lane-owned, m <= 32.
__device__ SR_FAST_FN double solve_ll(const double* M, int m, int lane, double myinv, double z) {
  const double* ri = M + rb2(lane < m ? lane : 0);
  #pragma unroll 1
  for (int j = 0; j < m; ++j) {                     // forward: L y = z
    if (lane == j) z *= myinv;
    const double yj = __shfl_sync(FULL, z, j);
    if (lane > j && lane < m) z = fma(-ri[j], yj, z);
  }
  return solve_bwd(M, m, lane, myinv, z);
}
#endif

// w'_a = s_a * sum_i (x_ia - xb_a) * alpha_i, alpha lane-owned (n <= 32);
// lanes over features, written to wout[0..deff).
template <bool SX>
__device__ SR_FAST_FN void xt_alpha_lanes(const FastView& f, double alpha, double* wout, int lane,
                                           double* abuf) {
  if (lane < f.n) abuf[lane] = alpha;   // broadcast through shared memory (1 LDS per row, no shuffles)
  __syncwarp();
  const int ldx8 = f.ldx * 8;
  for (int a0 = 0; a0 < f.deff; a0 += 64) {
    const int a1 = a0 + lane, a2 = a0 + 32 + lane;
    const int o1 = f.col[a1 < f.deff ? a1 : 0] * 8, o2 = f.col[a2 < f.deff ? a2 : 0] * 8;
    const double x1 = f.xb[a1 < f.deff ? a1 : 0], x2 = f.xb[a2 < f.deff ? a2 : 0];
    double acc1 = 0.0, acc2 = 0.0;
    SR_UNROLL(SR_UNROLL_XTA)
    for (int i = 0; i < f.n; ++i) {
      const double ai = abuf[i];
      const int ro = f.trs[i] * ldx8;
      acc1 = fma(xat<SX>(f, ro + o1) - x1, ai, acc1);
      acc2 = fma(xat<SX>(f, ro + o2) - x2, ai, acc2);
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
// mcap: rows the factor buffer holds (the dual fuses the forward solve as row m when m < mcap).
template <bool DUAL, bool SX>
__device__ SR_FAST_FN bool fit_fast(const FastView& f, const double* yc, double lambda, int refine, double* Mpk,
                         double* scratch, double* uwork, double* wout, int lane, int mcap) {
  const int m = DUAL ? f.n : f.deff;
  gram_fast<DUAL, SX>(f, m, lambda, Mpk, lane);
  SR_WT(3);
  double myinv;
#if SPEEDREC_CHOL_RL
  const bool aug = false;
#else
  const bool aug = DUAL && m < mcap;
#endif
  if (aug) {
    if (lane < m) Mpk[rb2(m) + lane] = yc[lane];
    __syncwarp();
  }
  const bool ok = chol_ll(Mpk, m, lane, myinv, aug);
  SR_WT(4);
  if (DUAL) {
    double alpha = lane < f.n ? (aug ? Mpk[rb2(m) + lane] : yc[lane]) : 0.0;
    alpha = aug ? solve_bwd(Mpk, m, lane, myinv, alpha) : solve_ll(Mpk, m, lane, myinv, alpha);
    for (int it = 0; it < refine; ++it) {
      xt_alpha_lanes<SX>(f, alpha, wout, lane, scratch);
      for (int a = lane; a < f.deff; a += 32) uwork[a] = wout[a] * f.s[a];
      __syncwarp();
      double e = 0.0;
      if (lane < f.n) e = yc[lane] - xrow_dot(f, f.X + f.trs[lane] * f.ldx, uwork) - lambda * alpha;
      alpha += solve_ll(Mpk, m, lane, myinv, e);
      __syncwarp();
    }
    SR_WT(5);
    xt_alpha_lanes<SX>(f, alpha, wout, lane, scratch);
    SR_WT(6);
  } else {
    // rhs_a = s_a * sum_i (x_ia - xb_a) * yc_i, lane a < deff <= 32
    double w = 0.0;
    if (lane < f.deff) {
      const int c = f.col[lane];
      const double x0 = f.xb[lane];
      for (int i = 0; i < f.n; ++i) w = fma(f.X[f.trs[i] * f.ldx + c] - x0, yc[i], w);
      w *= f.s[lane];
    }
    w = solve_ll(Mpk, m, lane, myinv, w);
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
      w += solve_ll(Mpk, m, lane, myinv, r);
      __syncwarp();
    }
    if (lane < f.deff) wout[lane] = w;
    __syncwarp();
  }
  return ok;
}

}  // namespace speedrec
