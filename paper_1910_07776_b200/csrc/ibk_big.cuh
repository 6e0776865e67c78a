// ibk_big.cuh -- IBK (NEXT-1) on the large-batch path (> 64 groups: C4).
// DESIGN.md §5.9.
//
// The k-nearest-neighbour predictor of DESIGN.md §3 (R19/R22): per fit, the
// training befores and test befores scaled by the fit's min-max map
// x' = (x - mn) / rg over the active counters (D3), D_i = sum_a fma(d_a, d_a,
// acc) in active-counter order with d_a = x'_test,a - x'_i,a, neighbours = the
// min(k, n) smallest (D_i, i), EX = (labels summed in neighbour order) /
// min(k, n).  Every step is an IEEE operation in a fixed order, so EX is
// bit-exact against the oracle.  At C4 size a fit is n ~ 8,192 training rows
// x t ~ 16,384 test rows x d = 128: 1.7e10 subtract + FMA pairs, pure FP64
// pipe work (the distance definition forbids the GEMM form |a|^2+|b|^2-2ab).
//
//  k_ibk_prep  CTA per fit: pair and test lists (A1), exact min / max (A2),
//              the scaled training rows -> global scratch [n][kIbkLd].
//  k_ibk_dist  CTA per (fit, test-tile chunk): 64-test tile scaled into
//              shared memory (counter-major), 32-row training tiles
//              double-buffered by cp.async; thread = 4 tests x 2 rows
//              register block; per tile the 64 x 32 distances go through
//              shared memory to 4 partial sorted top-k lists per test (each
//              thread takes 8 rows of every tile; strict <, rows in index
//              order => ties keep the lower index), merged in (D, index)
//              order at the end of the test tile.
//              EX -> the warp path's EX table.
//  k_ibk_score warp per fit: per-(scenario, opt) scores (A7) in test order.
// A6 then runs in k_rank_warp on the same EX table.
#pragma once
#include "eval_warp.cuh"
#include "fit_big.cuh"

namespace speedrec {

constexpr int kIbkLd = kBigMaxD + 1;   // scaled row stride (odd: conflict-free row-parallel reads)
constexpr int kIbkTT = 64;             // test rows per tile
constexpr int kIbkTR = 32;             // training rows per tile

struct IbkMeta {
  int n, nt, deff, scored;             // scored = 0: optimization not scored in the scenario
  unsigned long long fp_tr, fp_te;
  int col[kBigMaxD];
  double mn[kBigMaxD], rg[kBigMaxD];
};

struct IbkArgs {
  BigArgs B;            // dataset, scenario description (member_words, features)
  EvalArgs E;           // EX-table exchange with k_rank_warp, outputs
  int k_nn;
  long long np;         // list capacity per fit (32 G)
  int32_t* trs;         // [fits][np] training before slots
  double* yl;           // [fits][np] training labels (raw)
  int32_t* tes;         // [fits][np] test before slots
  int32_t* tek;         // [fits][np] g*32 + pair rank of each test case
  double* xs;           // [fits][np][kIbkLd] scaled training rows
  IbkMeta* meta;        // [fits]
  int chunks;           // test-tile chunks (CTAs) per fit
};

// ------------------------------------------------------------------ prep
static __global__ void __launch_bounds__(kBigThreads) k_ibk_prep(const IbkArgs I) {
  __shared__ int ctr[1024 + 8], cte[1024 + 8], Fl[kBigMaxD], wsum[16], misc[4];
  __shared__ uint64_t xred[8];
  __shared__ double zmn[kBigMaxD], zmx[kBigMaxD];
  const BigArgs& A = I.B;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const unsigned ltm = (1u << lane) - 1u;
  const int G = A.G, O = A.O, C = A.C;
  const long long fit = blockIdx.x;
  const long long sl = fit / O;
  const int o = (int)(fit % O);
  const long long s = A.first + sl;
  const long long split = s % A.n_splits, fidx = s / A.n_splits;
  const uint32_t om = (A.split_om ? A.split_om[split] : A.opt_mask) & ((1u << O) - 1u);
  IbkMeta& M = I.meta[fit];
  if (!((om >> o) & 1u)) {
    if (t == 0) {
      M.scored = 0;
      M.n = M.nt = M.deff = 0;
    }
    return;
  }
  int32_t* trs = I.trs + fit * I.np;
  double* yl = I.yl + fit * I.np;
  int32_t* tes = I.tes + fit * I.np;
  int32_t* tek = I.tek + fit * I.np;
  // ---- A1: pair counts per group, CTA scans, lists in (group, pair rank) order ----
  uint64_t fptr = 0, fpte = 0;
  for (int g = warp; g < G; g += kBigThreads / 32) {
    const int b = A.opt_bit[(g / A.IR) * O + o];
    int ntr = 0, nte = 0;
    if (b >= 0) {
      uint64_t tr, te;
      member_words(A, split, g, tr, te);
      const int v = ins0(lane, b);
      const bool istr = ((tr >> v) & 1ull) && ((tr >> (v | (1 << b))) & 1ull);
      const bool iste = (te >> v) & 1ull;
      const uint64_t h = mix64((uint64_t)((g * O + o) * 32 + lane));
      if (istr) fptr ^= h;
      if (iste) fpte ^= h;
      ntr = __popc(__ballot_sync(FULL, istr));
      nte = __popc(__ballot_sync(FULL, iste));
    }
    if (lane == 0) {
      ctr[g] = ntr;
      cte[g] = nte;
    }
  }
  const uint64_t fp_tr = cta_xor(fptr, xred), fp_te = cta_xor(fpte, xred);
  const int n = cta_scan(ctr, G, wsum);
  const int nt = cta_scan(cte, G, wsum);
  for (int g = warp; g < G; g += kBigThreads / 32) {
    const int b = A.opt_bit[(g / A.IR) * O + o];
    if (b < 0) continue;
    uint64_t tr, te;
    member_words(A, split, g, tr, te);
    const int v = ins0(lane, b);
    const bool istr = ((tr >> v) & 1ull) && ((tr >> (v | (1 << b))) & 1ull);
    const bool iste = (te >> v) & 1ull;
    const unsigned mtr = __ballot_sync(FULL, istr), mte = __ballot_sync(FULL, iste);
    if (istr) {
      const int p = ctr[g] + __popc(mtr & ltm);
      trs[p] = g * 64 + v;
      yl[p] = A.ylab[(g * O + o) * 32 + lane];
    }
    if (iste) {
      const int p = cte[g] + __popc(mte & ltm);
      tes[p] = g * 64 + v;
      tek[p] = g * 32 + lane;
    }
  }
  // ---- feature set F (counter-index order) ----
  {
    const int c = t;
    bool in = false;
    if (c < C && c < kBigMaxD) {
      if (A.subsets_k > 0) in = c < A.subsets_k && ((fidx >> c) & 1);
      else if (A.fmasks) in = (A.fmasks[fidx * 2 + (c >> 6)] >> (c & 63)) & 1ull;
      else in = true;
    }
    const unsigned bm = __ballot_sync(FULL, in);
    if (lane == 0) wsum[warp] = __popc(bm);
    __syncthreads();
    int base = 0;
    for (int q = 0; q < warp; ++q) base += wsum[q];
    if (in) Fl[base + __popc(bm & ltm)] = c;
    if (t == 0) {
      int dd = 0;
      for (int q = 0; q < kBigThreads / 32; ++q) dd += wsum[q];
      misc[0] = dd;
    }
    __syncthreads();
  }
  const int d = misc[0];
  // ---- A2: exact min / max per feature (two row halves), active compaction ----
  {
    const int a = t & (kBigMaxD - 1), h = t >> 7;
    double mn = INFINITY, mx = -INFINITY;
    if (a < d && n > 0) {
      const int c = Fl[a];
      for (int i = h; i < n; i += 2) {
        const double vv = A.x[(long long)trs[i] * C + c];
        mn = fmin(mn, vv);
        mx = fmax(mx, vv);
      }
    }
    if (h == 1) {
      zmn[a] = mn;
      zmx[a] = mx;
    }
    __syncthreads();
    bool act = false;
    if (h == 0) {
      mn = fmin(mn, zmn[a]);
      mx = fmax(mx, zmx[a]);
      act = a < d && n > 0 && mx > mn;
    }
    const unsigned bm = __ballot_sync(FULL, act);
    if (h == 0 && lane == 0) wsum[warp] = __popc(bm);
    __syncthreads();
    if (h == 0) {
      int base = 0;
      for (int q = 0; q < warp; ++q) base += wsum[q];
      if (act) {
        const int p = base + __popc(bm & ltm);
        M.col[p] = Fl[a];
        M.mn[p] = mn;
        M.rg[p] = mx - mn;
      }
      if (t == 0) {
        int de = 0;
        for (int q = 0; q < kBigMaxD / 32; ++q) de += wsum[q];
        misc[1] = de;
      }
    }
    __syncthreads();
  }
  const int deff = misc[1];
  if (t == 0) {
    M.scored = 1;
    M.n = n;
    M.nt = nt;
    M.deff = deff;
    M.fp_tr = fp_tr;
    M.fp_te = fp_te;
  }
  __syncthreads();
  // ---- scaled training rows (IEEE (x - mn) / rg, the oracle's order) ----
  double* xs = I.xs + fit * I.np * kIbkLd;
  const long long tot = (long long)n * deff;
  for (long long e = t; e < tot; e += kBigThreads) {
    const int i = (int)(e / deff), a = (int)(e - (long long)i * deff);
    xs[(long long)i * kIbkLd + a] = (A.x[(long long)trs[i] * C + M.col[a]] - M.mn[a]) / M.rg[a];
  }
}

// ------------------------------------------------------------------ distances
static __global__ void __launch_bounds__(kBigThreads, 1) k_ibk_dist(const IbkArgs I) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* Ts = reinterpret_cast<double*>(smem);                 // [kBigMaxD][kIbkTT] test tile, counter-major
  double* Rs = Ts + kBigMaxD * kIbkTT;                          // [2][kIbkTR][kIbkLd] training tiles
  double* Dt = Rs + 2 * kIbkTR * kIbkLd;                        // [kIbkTT][kIbkTR + 1]
  const BigArgs& A = I.B;
  const EvalArgs& E = I.E;
  const int t = threadIdx.x;
  const long long fit = blockIdx.x / I.chunks;
  const int chunk = blockIdx.x % I.chunks;
  const IbkMeta& M = I.meta[fit];
  if (!M.scored) return;
  const int n = M.n, nt = M.nt, deff = M.deff;
  if (n == 0 || nt == 0) return;
  const int O = A.O, C = A.C;
  const long long sl = fit / O;
  const int o = (int)(fit % O);
  const long long s = A.first + sl, split = s % A.n_splits;
  const uint32_t om = (A.split_om ? A.split_om[split] : A.opt_mask) & ((1u << O) - 1u);
  const int q = __popc(om & ((1u << o) - 1u));
  const int32_t* tes = I.tes + fit * I.np;
  const int32_t* tek = I.tek + fit * I.np;
  const double* yl = I.yl + fit * I.np;
  const double* xs = I.xs + fit * I.np * kIbkLd;
  const int kk = I.k_nn < n ? I.k_nn : n;
  const int tx = t & 15, ty = t >> 4;         // rows 2tx, 2tx+1; tests 4ty .. 4ty+3
  const int ntile_r = (n + kIbkTR - 1) / kIbkTR;
  auto stage_rows = [&](int rt, int buf) {    // 32 scaled rows, 16-byte copies (deff rounded up to even)
    const int r0 = rt * kIbkTR, rows = min(kIbkTR, n - r0), w = (deff + 1) >> 1;
    double* dst = Rs + buf * kIbkTR * kIbkLd;
    for (int e = t; e < rows * w; e += kBigThreads) {
      const int r = e / w, a2 = (e - r * w) * 2;
      const double* src = xs + (long long)(r0 + r) * kIbkLd + a2;
      double* dd = dst + r * kIbkLd + a2;
      // kIbkLd is odd: rows alternate 16-byte alignment -> two 8-byte copies
      cp_async8(dd, src, true);
      cp_async8(dd + 1, src + 1, a2 + 1 < deff);
    }
    cp_commit();
  };
  for (int j0 = chunk * kIbkTT; j0 < nt; j0 += I.chunks * kIbkTT) {
    // ---- test tile, scaled exactly as the training rows ----
    for (int e = t; e < kIbkTT * deff; e += kBigThreads) {
      const int j = e / deff, a = e - j * deff;
      double v = 0.0;
      if (j0 + j < nt) v = (A.x[(long long)tes[j0 + j] * C + M.col[a]] - M.mn[a]) / M.rg[a];
      Ts[a * kIbkTT + j] = v;
    }
    // partial top-k of test (t >> 2) over the rows r = 8 (t & 3) .. +7 of every
    // tile (four lists per test, merged in (D, index) order at the end)
    double bd[kKnnMax];
    int bi[kKnnMax];
    int cnt = 0;
    double thr = INFINITY;                     // current k-th best distance of this list
#pragma unroll
    for (int z = 0; z < kKnnMax; ++z) {
      bd[z] = INFINITY;
      bi[z] = 0x7FFFFFFF;
    }
    stage_rows(0, 0);
    for (int rt = 0; rt < ntile_r; ++rt) {
      if (rt + 1 < ntile_r) {
        stage_rows(rt + 1, (rt + 1) & 1);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();                         // tile rt landed (and the test tile written)
      const double* R = Rs + (rt & 1) * kIbkTR * kIbkLd;
      const double* r0p = R + (2 * tx) * kIbkLd;
      const double* r1p = r0p + kIbkLd;
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
      for (int a = 0; a < deff; ++a) {
        const double2 t01 = *reinterpret_cast<const double2*>(Ts + a * kIbkTT + 4 * ty);
        const double2 t23 = *reinterpret_cast<const double2*>(Ts + a * kIbkTT + 4 * ty + 2);
        const double u0 = r0p[a], u1 = r1p[a];
        const double tv[4] = {t01.x, t01.y, t23.x, t23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double d0 = tv[i] - u0, d1 = tv[i] - u1;
          acc[i][0] = fma(d0, d0, acc[i][0]);
          acc[i][1] = fma(d1, d1, acc[i][1]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        Dt[(4 * ty + i) * (kIbkTR + 1) + 2 * tx] = acc[i][0];
        Dt[(4 * ty + i) * (kIbkTR + 1) + 2 * tx + 1] = acc[i][1];
      }
      __syncthreads();
      {                                        // 4 threads per test, 8 rows each, in index order
        const int tt = t >> 2, r0 = 8 * (t & 3);
        const int rows = min(kIbkTR, n - rt * kIbkTR);
#pragma unroll
        for (int r = r0; r < r0 + 8; ++r) {
          const double D = Dt[tt * (kIbkTR + 1) + r];
          if (r < rows && (cnt < kk || D < thr)) {
            int p = cnt < kk ? cnt++ : kk - 1;
            // sorted insert (registers: compile-time indices, predicated shifts)
#pragma unroll
            for (int z = kKnnMax - 1; z > 0; --z) {
              if (z <= p && bd[z - 1] > D) {
                bd[z] = bd[z - 1];
                bi[z] = bi[z - 1];
                p = z - 1;
              }
            }
#pragma unroll
            for (int z = 0; z < kKnnMax; ++z)
              if (z == p) {
                bd[z] = D;
                bi[z] = rt * kIbkTR + r;
              }
#pragma unroll
            for (int z = 0; z < kKnnMax; ++z)
              if (z == kk - 1) thr = cnt < kk ? INFINITY : bd[z];
          }
        }
      }
      // (the next iteration's barrier protects Dt and the refilled buffer)
    }
    // merge the 4 partial lists of each test in (D, index) order (Ts / Rs are free)
    __syncthreads();
    double* MD = Ts;                                            // [256][kKnnMax] distances
    int* MI = reinterpret_cast<int*>(Rs);                       // [256][kKnnMax] indices
#pragma unroll
    for (int z = 0; z < kKnnMax; ++z) {
      MD[t * kKnnMax + z] = bd[z];
      MI[t * kKnnMax + z] = bi[z];
    }
    __syncthreads();
    if (t < kIbkTT && j0 + t < nt) {
      int h[4] = {0, 0, 0, 0};
      double ssum = 0.0;
      for (int z = 0; z < kk; ++z) {           // k smallest of the 4 sorted lists
        int best = 0;
        double bdv = INFINITY;
        int biv = 0x7FFFFFFF;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int row = 4 * t + w;
          const double dv = h[w] < kKnnMax ? MD[row * kKnnMax + h[w]] : INFINITY;
          const int iv = h[w] < kKnnMax ? MI[row * kKnnMax + h[w]] : 0x7FFFFFFF;
          if (dv < bdv || (dv == bdv && iv < biv)) {
            bdv = dv;
            biv = iv;
            best = w;
          }
        }
#pragma unroll
        for (int w = 0; w < 4; ++w) h[w] += (w == best) ? 1 : 0;
        ssum += yl[biv];
      }
      const double e = ssum / (double)kk;
      const int gk = tek[j0 + t];
      const int g = gk >> 5;
      E.extab[sl * E.ex_stride + q * E.tg_stride + test_group_index(E.sd, split, g) * 32 + (gk & 31)] = e;
    }
    __syncthreads();                           // Ts / Dt / Rs reused by the next test tile
  }
}

// ------------------------------------------------------------------ scores
// Warp per fit: the A7 row in test order (lane-strided partials, butterfly),
// trained flags and guard counts for k_rank_warp, pooled totals.
static __global__ void __launch_bounds__(256) k_ibk_score(const IbkArgs I, long long n_fits) {
  const BigArgs& A = I.B;
  const EvalArgs& E = I.E;
  const int lane = threadIdx.x & 31;
  const long long fit = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (fit >= n_fits) return;
  const IbkMeta& M = I.meta[fit];
  const int O = A.O, G = A.G;
  const long long sl = fit / O;
  const int o = (int)(fit % O);
  OptScore row;
  row.n_train = row.n_test = row.n_correct = row.n_clamped = 0;
  row.sum_ratio = row.min_ratio = row.max_ratio = 0.0;
  row.fp_train = row.fp_test = 0ull;
  if (!M.scored) {
    if (lane == 0) E.opt_out[sl * O + o] = row;
    return;
  }
  const int n = M.n, nt = M.nt;
  row.n_train = n;
  row.n_test = nt;
  row.fp_train = M.fp_tr;
  row.fp_test = M.fp_te;
  if (n > 0 && lane == 0) atomicOr(&E.trained[sl], 1u << o);
  if (n == 0 || nt == 0) {
    if (lane == 0) E.opt_out[sl * O + o] = row;
    return;
  }
  const long long s = A.first + sl, split = s % A.n_splits;
  const uint32_t om = (A.split_om ? A.split_om[split] : A.opt_mask) & ((1u << O) - 1u);
  const int q = __popc(om & ((1u << o) - 1u));
  const int32_t* tek = I.tek + fit * I.np;
  int ncorr = 0, guard = 0;
  double rsum = 0.0, rmin = INFINITY, rmax = -INFINITY;
  for (int j = lane; j < nt; j += 32) {
    const int gk = tek[j], g = gk >> 5, k = gk & 31;
    const double e = E.extab[sl * E.ex_stride + q * E.tg_stride + test_group_index(E.sd, split, g) * 32 + k];
    if (near_tol(e, 0.0, E.guard_tol) || near_tol(e, 1.0, E.guard_tol)) ++guard;
    const double ac = A.ylab[(g * O + o) * 32 + k];
    ncorr += ((e > 1.0 && ac > 1.0) || (e <= 1.0 && ac <= 1.0)) ? 1 : 0;
    const double ratio = ac / e;
    rsum += ratio;
    rmin = fmin(rmin, ratio);
    rmax = fmax(rmax, ratio);
    if (E.ex_out) E.ex_out[(sl * O + o) * (long long)G * 32 + gk] = e;
  }
  row.n_correct = warp_isum(ncorr);
  row.sum_ratio = warp_sum(rsum);
  row.min_ratio = warp_min(rmin);
  row.max_ratio = warp_max(rmax);
  guard = warp_isum(guard);
  if (lane == 0) {
    E.opt_out[sl * O + o] = row;
    if (guard) atomicAdd(&E.guard_acc[sl], guard);
    if (E.totals) {
      atomicAdd(&E.totals[0], (unsigned long long)row.n_correct);
      atomicAdd(&E.totals[1], (unsigned long long)nt);
    }
  }
}

constexpr int kIbkDistSmem = (kBigMaxD * kIbkTT + 2 * kIbkTR * kIbkLd + kIbkTT * (kIbkTR + 1)) * 8;

}  // namespace speedrec
