// pred_rank.cuh -- A5-A7 of the split LS path.
//
// k_fit_warp<., 4, true> leaves one row per (scenario, scored optimization)
// in the model table: u (weights on raw counters, EX = c0 + sum_c x_c u_c),
// c0, a flag and the A1 counts.  k_pred_rank then finishes each scenario with
// one warp:
//  * A5: EX for every test version of the scenario x every scored
//    optimization as one FP64 tensor-core product (mma.sync m8n8k4 -> DMMA):
//    rows = the scenario's test versions (rate rows staged once per CTA in
//    shared memory, row stride = 4 mod 16 doubles: conflict-free fragment
//    loads), columns = the scored optimizations (the table's u rows, staged
//    per warp in shared memory with the same stride);
//  * clamp EX <= 0 -> 0.01, sign accuracy and AC/EX per test case,
//    guard band (R21), rank + threshold + top-K per test version (R13),
//    recommendation hits;
//  * A7 rows per (scenario, optimization) and per scenario, pooled totals.
// No EX table in HBM and no separate ranking kernel: the scenario's EX lives in
// registers / a per-warp shared-memory tile only.
#pragma once
#include "kernels.cuh"

namespace speedrec {

constexpr int kPrWarps = 16;    // most warps per CTA (one CTA per SM: the staged rates are shared)
constexpr int kPrChunk = 32;    // test versions per scoring pass (4 DMMA row-blocks)
constexpr int kPrMaxC = 64;     // counters covered (16 unrolled k-steps)

// Shared-memory plan (byte offsets) of k_pred_rank.
struct PredLayout {
  int ldxp;        // row stride of the staged rates (doubles, = 4 mod 16)
  int off_x;       // [N][ldxp] doubles
  int off_y;       // [G][O][32] labels
  int off_w;       // first per-warp slab: 2 x model rows [CMAX][ldut] + EX tile [kPrChunk][CMAX + 1]
                   // + slot list [N] int16
  int ldut;        // model-row stride in shared memory (>= ldu, = 4 mod 16 doubles)
  int wbytes;
  int warps;       // warps per CTA
  int bytes;
};

// Reduce-scatter of 8 values per lane over the warp: returns, in lane l, the
// total (OP 0 sum, 1 min, 2 max) of column (l >> 2) & 7 over all 32 lanes --
// 9 double shuffles instead of 8 full butterflies (40).
template <int OP>
__device__ __forceinline__ double scatter_reduce8(double (&v)[8], int lane) {
  auto op = [](double a, double b) { return OP == 0 ? a + b : OP == 1 ? fmin(a, b) : fmax(a, b); };
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
  double a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {     // xor 16: keep columns 0-3 (low lanes) or 4-7
    const double keep = h16 ? v[i + 4] : v[i], give = h16 ? v[i] : v[i + 4];
    a[i] = op(keep, __shfl_xor_sync(FULL, give, 16));
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {     // xor 8: keep 2 of the 4
    const double keep = h8 ? a[i + 2] : a[i], give = h8 ? a[i] : a[i + 2];
    b[i] = op(keep, __shfl_xor_sync(FULL, give, 8));
  }
  const double keep = h4 ? b[1] : b[0], give = h4 ? b[0] : b[1];   // xor 4: keep 1
  double r = op(keep, __shfl_xor_sync(FULL, give, 4));
  r = op(r, __shfl_xor_sync(FULL, r, 2));
  return op(r, __shfl_xor_sync(FULL, r, 1));
}

// Exact guard-band count (reading R21) of one test version, as rank_scenario
// counts it: EX within tol max(1, |EX|) of 0 or 1 (raw EX), of the threshold
// (clamped EX), and every candidate pair (clamped EX; two clamped candidates
// tie by rule).  Called only when the cheap screen fired (essentially never).
template <int CMAX>
__device__ __noinline__ int guard_count(const EvalArgs& A, const double* ut, int ldut, int Cp, const int* ols,
                                        const int8_t* obit, const double* er, int t, int O) {
  const int g = t >> 6, v = t & 63, p = g / A.IR;
  const double tol = A.guard_tol;
  double ce[CMAX];
  unsigned cvm = 0u, ccm = 0u;
  int guard = 0;
  for (int q = 0; q < CMAX; ++q) {
    const int o = ols[q];
    const int b = o >= 0 ? obit[p * O + o] : -1;
    ce[q] = 0.0;
    if (!(o >= 0 && b >= 0 && !((v >> b) & 1)) || ut[q * ldut + Cp + kUflag] == 0.0) continue;
    double e = ut[q * ldut + Cp + kUc0] + er[q];
    if (near_tol(e, 0.0, tol) || near_tol(e, 1.0, tol)) ++guard;
    if (e <= 0.0) {
      e = A.clamp_floor;
      ccm |= 1u << q;
    }
    ce[q] = e;
    cvm |= 1u << q;
  }
  for (int q = 0; q < CMAX; ++q) {
    if (!((cvm >> q) & 1u)) continue;
    if (near_tol(ce[q], A.threshold, tol)) ++guard;
    for (int r = q + 1; r < CMAX; ++r)
      if (((cvm >> r) & 1u) && !((ccm >> q) & (ccm >> r) & 1u) && near_tol(ce[q], ce[r], tol)) ++guard;
  }
  return guard;
}

template <int CMAX, int KS>
__global__ void __launch_bounds__(kPrWarps * 32, 1) k_pred_rank(const EvalArgs A, const PredLayout PL) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = A.G, O = A.O, C = A.C, N = G * 64;
  const int ldx = PL.ldxp, ldut = PL.ldut, wpb = PL.warps;
  const int Cp = 4 * KS;                           // k-steps (KS = ceil(C/4)); model fields start at Cp
  int8_t* obit = reinterpret_cast<int8_t*>(smem);
  double* xs = reinterpret_cast<double*>(smem + PL.off_x);
  double* ys = reinterpret_cast<double*>(smem + PL.off_y);
  double* zrow = ys + G * O * 32;                    // [ldut] zeros: B rows of unused columns
  for (int i = tid; i < A.P * O; i += blockDim.x) obit[i] = A.opt_bit[i];
  for (int r = warp; r < N; r += wpb)
    for (int c = lane; c < ldx; c += 32) xs[r * ldx + c] = c < C ? A.x[(long long)r * C + c] : 0.0;
  for (int i = tid; i < G * O * 32; i += blockDim.x) ys[i] = A.ylab[i];
  for (int i = tid; i < ldut; i += blockDim.x) zrow[i] = 0.0;
  unsigned char* slab = smem + PL.off_w + warp * PL.wbytes;
  double* ubuf = reinterpret_cast<double*>(slab);                                    // [2][CMAX][ldut] model rows
  double* ext = ubuf + 2 * CMAX * ldut;                                              // [kPrChunk][CMAX + 1]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ext + kPrChunk * (CMAX + 1));        // [2] bulk-copy barriers
  int* ols = reinterpret_cast<int*>(bars + 2);                                       // [8] scored ids (-1 pad)
  int16_t* slots = reinterpret_cast<int16_t*>(ols + 8);                              // [N]
  const int rl = lane >> 2, kl = lane & 3;
  const long long gwarp = (long long)blockIdx.x * wpb + warp;
  const long long nwarps = (long long)gridDim.x * wpb;
  unsigned long long tot_corr = 0, tot_test = 0, tot_rec = 0, tot_hit = 0;
  const unsigned lt = (1u << lane) - 1u;
  // model rows of scenario sl -> buffer b: ONE bulk copy (TMA engine) of the
  // scenario's n_os contiguous rows (table stride ldu == ldut), completing on
  // the buffer's mbarrier
  const unsigned row_bytes = (unsigned)(A.n_os * A.ldu * 8);
  auto prefetch = [&](long long sl, int b) {
    if (lane == 0 && sl < A.count) {
      fence_proxy_async();               // this warp's earlier reads of the buffer precede the async write
      bulk_g2s(ubuf + b * CMAX * ldut, A.utab + sl * (long long)A.n_os * A.ldu, row_bytes, bars + b);
    }
  };
  if (lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    fence_mbar_init();
  }
  __syncthreads();
  int buf = 0;
  unsigned phase = 0u;                   // bit b: parity of buffer b's next completion
  prefetch(gwarp, 0);

  for (long long sl = gwarp; sl < A.count; sl += nwarps, buf ^= 1) {
    const long long s = A.first + sl, so = A.out0 + sl;
    const long long split = s % A.sd.n_splits;
    const uint32_t om = scored_mask(A.sd, split, O);
    const int n_os = __popc(om);
    prefetch(sl + nwarps, buf ^ 1);                  // next scenario's rows land while this one runs
    if (lane < 8) {                                  // scored optimizations in id order
      int o = -1;
      if (lane < n_os) {
        uint32_t mm = om;
        for (int q = 0; q < lane; ++q) mm &= mm - 1;
        o = __ffs(mm) - 1;
      }
      ols[lane] = o;
    }
    mbar_wait(bars + buf, (phase >> buf) & 1u);      // this scenario's rows have landed
    phase ^= 1u << buf;
    __syncwarp();
    const double* ut = ubuf + buf * CMAX * ldut;     // row q: u[0..C), then c0, flag, counts (kU*)
    // the scenario's test versions (slot ids), in slot order
    int ns = 0;
    for (int g = 0; g < G; ++g) {
      uint64_t tr, te;
      member_words(A.sd, split, g, tr, te);
      if (te == 0ull) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool in = (te >> (h * 32 + lane)) & 1ull;
        const unsigned bm = __ballot_sync(FULL, in);
        if (in) slots[ns + __popc(bm & lt)] = (int16_t)(g * 64 + h * 32 + lane);
        ns += __popc(bm);
      }
    }
    __syncwarp();
    // per-lane partial scores per scored slot
    int pc[CMAX], pcl[CMAX];
    double ps[CMAX], pmn[CMAX], pmx[CMAX];
#pragma unroll
    for (int q = 0; q < CMAX; ++q) {
      pc[q] = pcl[q] = 0;
      ps[q] = 0.0;
      pmn[q] = INFINITY;
      pmx[q] = -INFINITY;
    }
    int nrec = 0, nhit = 0, guard = 0, untrained = 0;
    #pragma unroll 1
    for (int r0 = 0; r0 < ns; r0 += kPrChunk) {
      // ---- A5: EX tile of up to kPrChunk test versions x CMAX columns on DMMA ----
      #pragma unroll 1
      for (int rb = 0; rb < kPrChunk / 8 && r0 + rb * 8 < ns; ++rb) {
        const int row = r0 + rb * 8 + rl;
        const double* xr = xs + (row < ns ? slots[row] : 0) * ldx + kl;
        const double* br = (rl < n_os ? ut + rl * ldut : zrow) + kl;   // B[k][n] = u of slot n at 4 kstep + k
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int k = 0; k < KS; ++k) dmma(d0, d1, xr[4 * k], br[4 * k]);
        double* er = ext + (rb * 8 + rl) * (CMAX + 1) + 2 * kl;
        if (2 * kl < CMAX) er[0] = d0;
        if (2 * kl + 1 < CMAX) er[1] = d1;
      }
      __syncwarp();
      // ---- clamp, score, rank: lane = test version ----
      const int row = r0 + lane;
      bool scr = false;                  // a guard-band screen fired on this lane (rare)
      if (row < ns) {
        const int t = slots[row], g = t >> 6, v = t & 63, p = g / A.IR;
        const double* er = ext + lane * (CMAX + 1);
        double ce[CMAX];                 // EX (clamped)
        unsigned cvm = 0u;               // candidate bit mask
        const double tol = A.guard_tol;
#pragma unroll
        for (int q = 0; q < CMAX; ++q) {
          const int o = ols[q];
          const int b = o >= 0 ? obit[p * O + o] : -1;
          bool cand = o >= 0 && b >= 0 && !((v >> b) & 1);
          if (cand && ut[q * ldut + Cp + kUflag] == 0.0) {   // untrained (R18): counted, never a candidate
            ++untrained;
            cand = false;
          }
          ce[q] = 0.0;
          if (cand) {
            cvm |= 1u << q;
            const int k = rmv(v, b);
            double e = ut[q * ldut + Cp + kUc0] + er[q];
            // guard band (R21), screened: tol (1 + |e|) >= tol max(1, |e|), so a
            // miss is exact; the rule itself runs (warp-uniformly) only on a hit
            const double te = fma(tol, fabs(e), tol);
            scr |= fabs(e) <= te || fabs(e - 1.0) <= te;
            if (e <= 0.0) {
              e = A.clamp_floor;
              ++pcl[q];
            }
            const double ac = ys[(g * O + o) * 32 + k];
            pc[q] += ((e > 1.0 && ac > 1.0) || (e <= 1.0 && ac <= 1.0)) ? 1 : 0;
            const double ratio = ac * rcp_nr(e);   // AC/EX within 2 ulp (bar: 1e-9)
            ps[q] += ratio;
            pmn[q] = dmin(pmn[q], ratio);
            pmx[q] = dmax(pmx[q], ratio);
            ce[q] = e;
            if (A.ex_out) A.ex_out[(so * O + o) * (long long)G * 32 + g * 32 + k] = e;
          }
        }
#pragma unroll
        for (int q = 0; q < CMAX; ++q) {
          if (!((cvm >> q) & 1u)) continue;
          const double tq = fma(tol, fabs(ce[q]), tol);
          scr |= fabs(ce[q] - A.threshold) <= tq;
#pragma unroll
          for (int r = q + 1; r < CMAX; ++r) scr |= ((cvm >> r) & 1u) && fabs(ce[q] - ce[r]) <= tq;
        }
        // rank (EX desc, id asc) among candidates with EX >= threshold, first max_count
        unsigned left = 0u;
#pragma unroll
        for (int q = 0; q < CMAX; ++q)
          if (((cvm >> q) & 1u) && ce[q] >= A.threshold) left |= 1u << q;
        for (int rk = 0; rk < A.max_count && left; ++rk) {
          int best = -1;
          double be = -INFINITY;
#pragma unroll
          for (int q = 0; q < CMAX; ++q)
            if (((left >> q) & 1u) && ce[q] > be) {    // strict: ties keep the lower id
              be = ce[q];
              best = q;
            }
          left &= ~(1u << best);
          ++nrec;
          const int ob = ols[best];
          const int kb = rmv(v, obit[p * O + ob]);
          if (ys[(g * O + ob) * 32 + kb] > 1.0) ++nhit;
          if (A.rec_out) A.rec_out[(so * G * 64 + t) * A.max_count + rk] = (int8_t)ob;
        }
      }
      if (__any_sync(FULL, scr) && scr)      // cold: the exact guard rule of this lane's version
        guard += guard_count<CMAX>(A, ut, ldut, Cp, ols, obit, ext + lane * (CMAX + 1), slots[row], O);
      __syncwarp();
    }
    // ---- A7 rows ----
    int gsum = warp_isum(guard);
    const int nr = warp_isum(nrec), nh = warp_isum(nhit), nu = warp_isum(untrained);
    // reduce-scatter of the per-slot sums / minima / maxima (8 columns, padded):
    // afterwards lane l holds column (l >> 2) & 7's total over all 32 lanes
    double rs[8], rmn[8], rmx[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      rs[q] = q < CMAX ? ps[q] : 0.0;
      rmn[q] = q < CMAX ? pmn[q] : INFINITY;
      rmx[q] = q < CMAX ? pmx[q] : -INFINITY;
    }
    const double tsum = scatter_reduce8<0>(rs, lane), tmin = scatter_reduce8<1>(rmn, lane),
                 tmax = scatter_reduce8<2>(rmx, lane);
    int mycorr = 0, mycl = 0;
#pragma unroll
    for (int q = 0; q < CMAX; ++q) {
      const int a = warp_isum(pc[q]), b = warp_isum(pcl[q]);
      if (((lane >> 2) & 7) == q) {
        mycorr = a;
        mycl = b;
      }
    }
    {
      const int q = (lane >> 2) & 7;
      if ((lane & 3) == 0 && q < n_os) {
        const double* e = ut + q * ldut + Cp;
        OptScore row;
        row.n_train = (int)e[kUntr];
        row.n_test = (int)e[kUnte];
        row.fp_train = (uint64_t)__double_as_longlong(e[kUfptr]);
        row.fp_test = (uint64_t)__double_as_longlong(e[kUfpte]);
        const int fq = (int)e[kUflag];
        const bool has = fq != 0 && row.n_test > 0;
        row.n_correct = has ? mycorr : 0;
        row.n_clamped = has ? mycl : 0;
        row.sum_ratio = has ? tsum : 0.0;
        row.min_ratio = has ? tmin : 0.0;
        row.max_ratio = has ? tmax : 0.0;
        if (A.opt_out) A.opt_out[so * O + ols[q]] = row;
        if (has) {
          tot_corr += (unsigned long long)mycorr;
          tot_test += (unsigned long long)row.n_test;
        }
      }
      // a non-positive pivot poisons the scenario (guard count, as the EX-table path)
      gsum += 1000000 * __popc(__ballot_sync(FULL, (lane & 3) == 0 && q < n_os && ut[q * ldut + Cp + kUflag] == 2.0));
    }
    if (lane == 0) {
      if (A.opt_out) {
        OptScore z;
        z.n_train = z.n_test = z.n_correct = z.n_clamped = 0;
        z.sum_ratio = z.min_ratio = z.max_ratio = 0.0;
        z.fp_train = z.fp_test = 0ull;
        for (int o = 0; o < O; ++o)
          if (!((om >> o) & 1u)) A.opt_out[so * O + o] = z;
      }
      ScnScore sr{nr, nh, nu, gsum};
      if (A.scn_out) A.scn_out[so] = sr;
    }
    tot_rec += nr;
    tot_hit += nh;
    __syncwarp();            // every lane is done with buffer `buf` before the next prefetch reuses it
  }
  tot_corr = warp_usum(tot_corr);      // accumulated by the row-writing lanes
  tot_test = warp_usum(tot_test);
  if (A.totals && lane == 0 && (tot_test | tot_rec | tot_hit)) {
    atomicAdd(&A.totals[0], tot_corr);
    atomicAdd(&A.totals[1], tot_test);
    atomicAdd(&A.totals[2], tot_rec);
    atomicAdd(&A.totals[3], tot_hit);
  }
}

}  // namespace speedrec
