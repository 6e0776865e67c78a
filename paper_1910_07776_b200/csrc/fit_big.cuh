// fit_big.cuh -- the large-batch path (config C4: 1024 programs x 64 variants
// x 128 counters, thousands of training pairs per fit).  DESIGN.md §5.5.
//
// k_fit_big: one CTA (8 warps) per (scenario, optimization) fit, persistent
//   over fits.  Pair lists are built by ballot + CTA scan (deterministic
//   order); min/max/sum statistics stream the training rows once; the centred,
//   scaled Gram X~^T X~ (d_eff <= 128) is accumulated on the FP64 tensor pipe
//   (mma.sync.m8n8k4.f64): training rows are gathered from L2 in 32-row chunks,
//   prefetched into registers while the previous chunk is contracted from
//   shared memory, each warp owning block-rows w and 15-w (17 tiles).  Then a
//   CTA LDL-form Cholesky, triangular solves, optional refinement (streamed
//   residual), and the weights on raw counters + intercept are written out.
// k_rank_big: one CTA per scenario: every test slot's candidates are
//   predicted (warp dot products against the staged weights), clamped,
//   ranked, thresholded and scored (A5-A7), deterministic reduction order.
#pragma once
#include "kernels.cuh"

namespace speedrec {

constexpr int kBigThreads = 256;
#ifndef SPEEDREC_GRAM_FRAGSTATS    // 1: D3 statistics from the warps' own DMMA A fragments (raw coordinates)
#define SPEEDREC_GRAM_FRAGSTATS 1
#endif
#ifndef SPEEDREC_GRAM_SHIFT        // FRAGSTATS 0 only: 1 Gram shifted by the first training row (in place), 0 raw
#define SPEEDREC_GRAM_SHIFT 1
#endif
#ifndef SPEEDREC_GRAM_EXPERIMENT   // timing probes of the Gram pass (1 no statistics, 2 no barrier, 3 no shift, 4 no min/max): wrong results
#define SPEEDREC_GRAM_EXPERIMENT 0
#endif
constexpr int kBigChunk = 32;   // training rows per refinement chunk (8 k-steps)
#ifndef SPEEDREC_GRAM_CHUNK
#define SPEEDREC_GRAM_CHUNK 32
#endif
constexpr int kGramChunk = SPEEDREC_GRAM_CHUNK;   // rows per Gram-pass ring stage (3 stages in Gbuf + rch)
constexpr int kBigLd = 132;     // chunk row stride in doubles: conflict-free 4x8 fragments
constexpr int kBigMaxD = 128;
constexpr int kBigGLd = 129;    // Gram row stride (odd: conflict-free columns)

struct BigArgs {
  const double* x;
  const double* ylab;
  const int8_t* opt_bit;
  int P, IR, C, O, G;
  int kind, gw;
  long long n_splits;
  const uint64_t* train_g;
  const uint64_t* test_g;
  const uint32_t* split_om;
  const int32_t* pool_list;
  int n_pool;
  unsigned long long seed;
  uint32_t opt_mask;
  int subsets_k;
  long long n_masks;
  const uint64_t* fmasks;
  double lambda, threshold, clamp_floor, guard_tol;
  int refine, max_count;
  long long first, count;  // scenario range of this batch
  // k_fit_big scratch: per CTA [np] training slots + [np] centred labels
  int32_t* lists;
  double* ylist;
  long long np;
  // fit results per (scenario in batch, optimization)
  double* U;        // [count][O][C]
  double* c0;       // [count][O]
  int32_t* fitflag; // [count][O]: 1 = model available
  OptScore* opt_out;  // [count][O] (k_fit_big writes counts/fingerprints, k_rank_big the scores)
  ScnScore* scn_out;
  double* ex_out;
  int8_t* rec_out;
  unsigned long long* totals;
  int fit_all;        // sr_fit: fit every trained optimization, also those with no test case
};

__device__ __forceinline__ void member_words(const BigArgs& A, long long split, int g, uint64_t& tr,
                                             uint64_t& te) {
  if (A.kind == 0) {
    tr = ((A.train_g[split * A.gw + (g >> 6)] >> (g & 63)) & 1ull) ? ~0ull : 0ull;
    te = ((A.test_g[split * A.gw + (g >> 6)] >> (g & 63)) & 1ull) ? ~0ull : 0ull;
  } else if (A.kind == 1) {
    bool inpool = false;
    for (int q = 0; q < A.n_pool; ++q) inpool |= (A.pool_list[q] == g);
    tr = inpool ? ~0ull : 0ull;
    te = 0ull;
    if (g == A.pool_list[split >> 6]) {
      tr &= ~(1ull << (split & 63));
      te = 1ull << (split & 63);
    }
  } else {
    tr = mix64(mix64(A.seed ^ mix64((uint64_t)split)) + (uint64_t)g);
    te = ~tr;
  }
}

// CTA-wide exclusive scan of n ints in smem (n <= 4 * kBigThreads); returns the total.
__device__ int cta_scan(int* v, int n, int* wsum) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  int loc[4], s = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = t * 4 + q;
    loc[q] = i < n ? v[i] : 0;
    s += loc[q];
  }
  int inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int q = 0; q < kBigThreads / 32; ++q) {
      const int y = wsum[q];
      wsum[q] = acc;
      acc += y;
    }
    wsum[kBigThreads / 32] = acc;
  }
  __syncthreads();
  int run = wsum[w] + inc - s;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = t * 4 + q;
    if (i < n) v[i] = run;
    run += loc[q];
  }
  const int total = wsum[kBigThreads / 32];
  __syncthreads();
  return total;
}

__device__ __forceinline__ double cta_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int q = 0; q < kBigThreads / 32; ++q) s += red[q];  // fixed order
  __syncthreads();
  return s;
}

__device__ __forceinline__ uint64_t cta_xor(uint64_t v, uint64_t* red) {
  v = warp_xor(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  uint64_t s = 0;
  for (int q = 0; q < kBigThreads / 32; ++q) s ^= red[q];
  __syncthreads();
  return s;
}

// Gather one row of a 32-row chunk into registers (thread: row t>>3,
// features (t&7)+8q), raw values; slot < 0 (row past n) and features past
// deff give 0.  The caller prefetches the slot index one chunk ahead, so the
// gather issues at once and stays in flight until big_scale_chunk consumes
// it (the L2 gather overlaps the contraction of the previous chunk).
__device__ __forceinline__ void big_load_rows(const double* X, int C, int slot, const int* col, int deff,
                                              double (&v)[16]) {
  const int a0 = threadIdx.x & 7;
  const double* xr = slot >= 0 ? X + (long long)slot * C : nullptr;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int a = a0 + 8 * q;
    v[q] = (xr && a < deff) ? xr[col[a]] : 0.0;
  }
}


// Training slot of this thread's row in chunk ch (-1 past n).
__device__ __forceinline__ int big_slot(const int32_t* trs, int n, int ch) {
  const int r = ch * kBigChunk + (threadIdx.x >> 3);
  return r < n ? trs[r] : -1;
}

// Centre and scale a gathered chunk in registers (padding stays exactly 0).
__device__ __forceinline__ void big_scale_chunk(int n, int r0, const double* xb, const double* s, int deff,
                                                double (&v)[16]) {
  const int r = r0 + (threadIdx.x >> 3);
  const int a0 = threadIdx.x & 7;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int a = a0 + 8 * q;
    if (r < n && a < deff) v[q] = (v[q] - xb[a]) * s[a];
  }
}


__global__ void __launch_bounds__(kBigThreads, 1) k_fit_big(const BigArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  // layout: Gbuf (union with the Gram-pass cp.async ring, which extends into rch) | rpt | vectors | scan arrays
  double* Gbuf = reinterpret_cast<double*>(smem);                       // [128][129]
  double* rch = Gbuf + kBigMaxD * kBigGLd;                              // [32][132] tail of the Gram ring
  double* rpt = rch + kBigChunk * kBigLd;                               // [32][128] refinement partials
  double* xb = rpt + kBigChunk * kBigMaxD;                              // [128]
  double* sv = xb + kBigMaxD;                                           // [128]
  double* rhs = sv + kBigMaxD;                                          // [128]
  double* wv = rhs + kBigMaxD;                                          // [128]
  double* zv = wv + kBigMaxD;                                           // [128]
  double* invd = zv + kBigMaxD;                                         // [128]
  double* red = invd + kBigMaxD + 2 * kBigChunk;                        // [16] (after 64 spare doubles)
  uint64_t* xred = reinterpret_cast<uint64_t*>(red + 16);               // [8]
  int* col = reinterpret_cast<int*>(xred + 8);                          // [128]
  int* Fl = col + kBigMaxD;                                             // [128]
  int* ctr = Fl + kBigMaxD;                                             // [G]
  int* cte = ctr + A.G;                                                 // [G] (counts only)
  int* wsum = cte + A.G;                                                // [9]
  int* misc = wsum + 16;                                                // [4]

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const unsigned ltm = (1u << lane) - 1u;
  int32_t* trs = A.lists + blockIdx.x * A.np;
  double* yl = A.ylist + blockIdx.x * A.np;
  const int G = A.G, O = A.O, C = A.C;
#if SPEEDREC_PHASE_TIMING
  // instrumented build (-DSPEEDREC_PHASE_TIMING=1): cycles per phase, CTA 0 prints at exit
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ph_last = clock64();
#define SR_PT(k)                            \
  if (t == 0) {                             \
    const long long now_ = clock64();       \
    ph[k] += now_ - ph_last;                \
    ph_last = now_;                         \
  }
#else
#define SR_PT(k)
#endif

  for (long long fit = blockIdx.x; fit < A.count * O; fit += gridDim.x) {
    const long long sl = fit / O;
    const int o = (int)(fit % O);
    const long long s = A.first + sl;
    const long long split = s % A.n_splits, fidx = s / A.n_splits;
    const uint32_t om = (A.split_om ? A.split_om[split] : A.opt_mask) & ((1u << O) - 1u);
    OptScore row;
    row.n_train = row.n_test = row.n_correct = row.n_clamped = 0;
    row.sum_ratio = row.min_ratio = row.max_ratio = 0.0;
    row.fp_train = row.fp_test = 0ull;
    if (!((om >> o) & 1u)) {
      if (t == 0) {
        A.opt_out[sl * O + o] = row;
        A.fitflag[sl * O + o] = 0;
      }
      continue;
    }
    // ---- A1: pair counts per group, then deterministic positions ----
    uint64_t fptr = 0, fpte = 0;
    #pragma unroll 4
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
    row.fp_train = cta_xor(fptr, xred);
    row.fp_test = cta_xor(fpte, xred);
    const int n = cta_scan(ctr, G, wsum);
    const int nt = cta_scan(cte, G, wsum);
    row.n_train = n;
    row.n_test = nt;
    if (n == 0 || (nt == 0 && !A.fit_all)) {
      if (t == 0) {
        A.opt_out[sl * O + o] = row;
        A.fitflag[sl * O + o] = n > 0 ? 1 : 0;
        A.c0[sl * O + o] = 0.0;
      }
      for (int c = t; c < C; c += kBigThreads) A.U[(sl * O + o) * C + c] = 0.0;
      // n > 0, nt == 0: the rank kernel needs no model (sr_fit asks for it: fit_all)
      continue;
    }
    #pragma unroll 4
    for (int g = warp; g < G; g += kBigThreads / 32) {
      const int b = A.opt_bit[(g / A.IR) * O + o];
      if (b < 0) continue;
      uint64_t tr, te;
      member_words(A, split, g, tr, te);
      const int v = ins0(lane, b);
      const bool istr = ((tr >> v) & 1ull) && ((tr >> (v | (1 << b))) & 1ull);
      const unsigned m = __ballot_sync(FULL, istr);
      if (istr) {
        const int p = ctr[g] + __popc(m & ltm);
        trs[p] = g * 64 + v;
        yl[p] = A.ylab[(g * O + o) * 32 + lane];
      }
    }
    // feature set F (counter-index order)
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
    SR_PT(0);
    // ---- ybar, centred labels ----
    double ys = 0.0;
    for (int i = t; i < n; i += kBigThreads) ys += yl[i];
    const double ybar = cta_sum(ys, red) / (double)n;
    for (int i = t; i < n; i += kBigThreads) yl[i] -= ybar;
    __syncthreads();
    SR_PT(1);

    // ---- A2 + A3 in one pass over the training rows ----
    // Rows stream through a 3-stage cp.async ring (32 rows x all d selected
    // features per stage) in the Gbuf region.  Per chunk, thread (feature fa,
    // row parity fh) folds the raw values into the D3 min / max / sum of its
    // feature and shifts them in place by c = the fit's first training row,
    // accumulating the rhs sum_i (x_i - c) y~_i; the warps then accumulate the
    // shifted Gram G^ = sum_i (x_i - c)(x_i - c)^T on DMMA.  After the pass:
    // xbar, rg and the activity of D3, and the centred, scaled system
    // G~_ab = s_a s_b (G^_ab - n (xbar_a - c_a)(xbar_b - c_b)) + lambda, exact
    // algebra of the definition (sum_i y~_i = 0); the streamed refinement below
    // removes the rounding.  Inactive features (rg = 0) become identity rows
    // with s = 0, so the solution on the active ones is unchanged.
    const int nref = A.refine;
    bool ok = true;
    const int deff = d;                   // system over the selected features
    if (deff > 0) {
      const int I1 = warp, I2 = 15 - warp;
      double accU[8][2], accS[8][2], accX[2] = {0.0, 0.0};
#pragma unroll
      for (int J = 0; J < 8; ++J) accU[J][0] = accU[J][1] = accS[J][0] = accS[J][1] = 0.0;
      const int fa = t & (kBigMaxD - 1), fh = t >> 7;
      const bool fin = fa < d;
#if SPEEDREC_GRAM_SHIFT && !SPEEDREC_GRAM_FRAGSTATS
      const double cshift = fin ? A.x[(long long)trs[0] * C + Fl[fa]] : 0.0;
#else
      const double cshift = 0.0;            // raw coordinates: no in-place shift pass
#endif
      double pmn = INFINITY, pmx = -INFINITY, psm = 0.0, prh = 0.0;
#if SPEEDREC_GRAM_FRAGSTATS
      // lane (rl, kl) of warp w folds rows = kl (mod 4) of features I1*8+rl and
      // I2*8+rl (its A fragments) into min / max / sum / sum x y~; the quads
      // combine them after the pass (fixed order)
      double qmn = INFINITY, qmx = -INFINITY, qsm = 0.0, qrh = 0.0;
#endif
      double* ring = Gbuf;                                  // [3][kGramChunk][kBigLd] (spills into the free rch space)
      double* yring = rpt;                                  // [3][kGramChunk] centred labels of the stage rows
      const int nchunks = (n + kGramChunk - 1) / kGramChunk;
      const int crow = t >> 3, ca0 = t & 7;
      // copy mapping: thread (row crow, features ca0 + 8q); rows >= n and
      // features >= d are zero-filled
      // rows crow (all threads) and 32 + crow (t < 128) of the chunk
      // every counter selected (d == C, so Fl[a] == a) and C even: each row
      // is one contiguous span -> 16-byte copies (half the copy instructions)
      const bool contig = d == C && (C & 1) == 0;
      auto issue = [&](int ch, int slot, int slot2) {
        double* st = ring + (ch % 3) * kGramChunk * kBigLd;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = crow + 32 * h;
          if (row >= kGramChunk) break;
          const int sl_ = h ? slot2 : slot;
          const double* xr = A.x + (sl_ >= 0 ? (long long)sl_ * C : 0);
          if (contig) {
            double* dst = st + row * kBigLd;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int a = 2 * ca0 + 16 * q;
              const bool ok_ = sl_ >= 0 && a < d;
              const unsigned dd = (unsigned)__cvta_generic_to_shared(dst + a);
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dd), "l"(xr + (ok_ ? a : 0)),
                           "r"(ok_ ? 16 : 0)
                           : "memory");
            }
          } else {
            double* dst = st + row * kBigLd + ca0;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const int a = ca0 + 8 * q;
              const bool ok_ = sl_ >= 0 && a < d;
              cp_async8(dst + 8 * q, xr + (ok_ ? Fl[a] : 0), ok_);
            }
          }
          if (ca0 == 0) {
            const int r = ch * kGramChunk + row;
            cp_async8(yring + (ch % 3) * kGramChunk + row, yl + (r < n ? r : 0), r < n);
          }
        }
      };
      auto gslot = [&](int ch, int row) {
        const int r = ch * kGramChunk + row;
        return (row < kGramChunk && r < n) ? trs[r] : -1;
      };
      // fold chunk cc's raw values into the statistics and shift them in
      // place (thread: feature fa, rows fh + 2j)
      auto shift_rows = [&](int cc, int j0, int j1) {
        double* st = ring + (cc % 3) * kGramChunk * kBigLd;
        const double* ys = yring + (cc % 3) * kGramChunk;
#pragma unroll
        for (int j = j0; j < j1; ++j) {
          const int r = fh + 2 * j;
          const bool live = fin && cc * kGramChunk + r < n;
          double xv = st[r * kBigLd + fa];
          if (live) {                 // rates: finite, >= 0 (validated): no NaN handling
#if SPEEDREC_GRAM_EXPERIMENT != 4
            pmn = dmin(pmn, xv);
            pmx = dmax(pmx, xv);
#endif
            psm += xv;
          }
#if SPEEDREC_GRAM_EXPERIMENT == 3 || !SPEEDREC_GRAM_SHIFT     // no in-place shift (raw coordinates)
          if (!live) xv = 0.0;
          prh = fma(xv, ys[r], prh);
#else
          xv = live ? xv - cshift : 0.0;
          if (fin) st[r * kBigLd + fa] = xv;
          prh = fma(xv, ys[r], prh);
#endif
        }
      };
      issue(0, gslot(0, crow), gslot(0, crow + 32));
      cp_commit();
      if (nchunks > 1) issue(1, gslot(1, crow), gslot(1, crow + 32));
      cp_commit();
      int slot_pf = gslot(2, crow), slot_pf2 = gslot(2, crow + 32);
      cp_wait<1>();
      __syncthreads();
#if !SPEEDREC_GRAM_FRAGSTATS
      shift_rows(0, 0, kGramChunk / 2);
#endif
      const int rl = lane >> 2, kl = lane & 3;
      // iteration ch: contract chunk ch on DMMA while the same warps fold and
      // shift chunk ch+1 (two rows per k-step); one barrier per chunk
      for (int ch = 0; ch < nchunks; ++ch) {
#if SPEEDREC_GRAM_EXPERIMENT == 2     // timing probe only (wrong results): no per-chunk barrier
        cp_wait<0>();
        if (ch == 0) __syncthreads();
#else
        cp_wait<0>();                                       // this thread's copies of chunk ch+1 landed
        __syncthreads();                                    // chunk ch shifted, ch+1 visible, ch-1 free
#endif
        if (ch + 2 < nchunks) {
          issue(ch + 2, slot_pf, slot_pf2);
          slot_pf = gslot(ch + 3, crow);
          slot_pf2 = gslot(ch + 3, crow + 32);
        }
        cp_commit();
        const double* cur = ring + (ch % 3) * kGramChunk * kBigLd;
        const bool nxt = ch + 1 < nchunks;
#pragma unroll
        for (int k0 = 0; k0 < kGramChunk; k0 += 4) {
#if SPEEDREC_GRAM_EXPERIMENT == 1 || SPEEDREC_GRAM_FRAGSTATS     // (1: timing probe only, wrong results)
          (void)nxt;
#else
          if (nxt) shift_rows(ch + 1, k0 / 2, k0 / 2 + 2);
#endif
          const double* base = cur + (k0 + kl) * kBigLd + rl;
          double f[16];
#pragma unroll
          for (int J = 0; J < 16; ++J) f[J] = base[8 * J];
          const double fa1 = base[8 * I1], fa2 = base[8 * I2];  // A fragments of the warp's block-rows
#pragma unroll
          for (int J = 0; J < 8; ++J) dmma(accU[J][0], accU[J][1], fa2, f[J]);
#pragma unroll
          for (int J = 0; J < 8; ++J) {
            const bool lo = J <= I1;
            dmma(accS[J][0], accS[J][1], lo ? fa1 : fa2, lo ? f[J] : f[15 - J]);
          }
          dmma(accX[0], accX[1], fa2, fa2);
#if SPEEDREC_GRAM_FRAGSTATS
          {   // rows past n and features past d are zero-filled: they add exact zeros to the sums
            const double yv = yring[(ch % 3) * kGramChunk + k0 + kl];
            if (ch * kGramChunk + k0 + kl < n) {   // rates: finite, >= 0 (validated): no NaN handling
              pmn = dmin(pmn, fa1);
              pmx = dmax(pmx, fa1);
              qmn = dmin(qmn, fa2);
              qmx = dmax(qmx, fa2);
            }
            psm += fa1;
            qsm += fa2;
            prh = fma(fa1, yv, prh);
            qrh = fma(fa2, yv, qrh);
          }
#endif
        }
      }
      cp_wait<0>();
#if SPEEDREC_GRAM_FRAGSTATS
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {     // the quad's four row residues (fixed order)
        pmn = dmin(pmn, __shfl_xor_sync(FULL, pmn, off));
        pmx = dmax(pmx, __shfl_xor_sync(FULL, pmx, off));
        psm += __shfl_xor_sync(FULL, psm, off);
        prh += __shfl_xor_sync(FULL, prh, off);
        qmn = dmin(qmn, __shfl_xor_sync(FULL, qmn, off));
        qmx = dmax(qmx, __shfl_xor_sync(FULL, qmx, off));
        qsm += __shfl_xor_sync(FULL, qsm, off);
        qrh += __shfl_xor_sync(FULL, qrh, off);
      }
      __syncthreads();                                      // ring consumed; Gbuf free
      if (kl == 0) {
        const int a1 = I1 * 8 + rl, a2 = I2 * 8 + rl;
        zv[a1] = pmn;
        wv[a1] = pmx;
        rhs[a1] = psm;
        invd[a1] = prh;
        zv[a2] = qmn;
        wv[a2] = qmx;
        rhs[a2] = qsm;
        invd[a2] = qrh;
      }
      __syncthreads();
      if (fh == 0) {
        const double mn = zv[fa], mx = wv[fa], sm = rhs[fa], rh = invd[fa];
#else
      // statistics of D3 from the two row halves (fixed order), rhs, shift difference
      if (fh == 1) {
        zv[fa] = pmn;
        wv[fa] = pmx;
        rhs[fa] = psm;
        invd[fa] = prh;
      }
      __syncthreads();                                      // ring consumed; Gbuf free
      if (fh == 0) {
        const double mn = fmin(pmn, zv[fa]), mx = fmax(pmx, wv[fa]), sm = psm + rhs[fa], rh = prh + invd[fa];
#endif
        const bool act = fin && mx > mn;
        const double xbar = fin ? sm / (double)n : 0.0;
        const double sc = act ? 1.0 / (mx - mn) : 0.0;
        col[fa] = fin ? Fl[fa] : 0;
        xb[fa] = xbar;
        sv[fa] = sc;
        rhs[fa] = sc * rh;                                  // s_a sum_i (x_ia - c_a) y~_i
        zv[fa] = xbar - cshift;                             // xbar_a - c_a
        if (t == 0) misc[1] = 0;
      }
      // shifted Gram tiles -> Gbuf (lower triangle, unscaled)
      {
        auto put = [&](int I, int J, const double (&acc)[2]) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = I * 8 + rl, c = J * 8 + 2 * kl + e;
            if (r < deff && c <= r) Gbuf[r * kBigGLd + c] = acc[e];
          }
        };
#pragma unroll
        for (int J = 0; J < 8; ++J) {
          put(I2, J, accU[J]);
          if (J <= I1) put(I1, J, accS[J]);
          else put(I2, 15 - J, accS[J]);
        }
        put(I2, I2, accX);
      }
      __syncthreads();
      // centred, scaled system; inactive features -> identity rows
      for (int e = t; e < deff * (deff + 1) / 2; e += kBigThreads) {
        int r = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
        while (r * (r + 1) / 2 > e) --r;
        while ((r + 1) * (r + 2) / 2 <= e) ++r;
        const int c = e - r * (r + 1) / 2;
        const double sr = sv[r], sc = sv[c];
        double g;
        if (sr != 0.0 && sc != 0.0)
          g = sr * sc * (Gbuf[r * kBigGLd + c] - (double)n * zv[r] * zv[c]) + (r == c ? A.lambda : 0.0);
        else
          g = (r == c) ? 1.0 : 0.0;
        Gbuf[r * kBigGLd + c] = g;
      }
      __syncthreads();
      SR_PT(2);
      // ---- A4: blocked Cholesky, 8-column panels ----
      // per panel: warp 0 factors the 8x8 diagonal block (lanes = rows),
      // one thread per row solves the panel below it (TRSM), and the warps
      // update the trailing lower triangle on DMMA (C -= L21 L21^T, two
      // k-steps per 8x8 tile, C loaded from and stored to shared memory).
      // Rows / columns in [deff, 8 nb) are identity padding.  The result is
      // turned into the solves' form: Gbuf[i][j] = L_ij L_jj (i > j), invd.
      {
        const int nbk = (deff + 7) >> 3, dpad = nbk * 8;
        for (int e = t; e < dpad * dpad; e += kBigThreads) {
          const int r = e / dpad, c = e - r * dpad;
          if ((r >= deff || c >= deff) && c <= r) Gbuf[r * kBigGLd + c] = (r == c) ? 1.0 : 0.0;
        }
        __syncthreads();
        const int rl = lane >> 2, kl = lane & 3;
        for (int pb = 0; pb < nbk; ++pb) {
          const int c0 = pb * 8;
          if (warp == 0) {                       // diagonal block, lanes 0..7 = rows c0 + lane
            double* ri = Gbuf + (c0 + (lane & 7)) * kBigGLd + c0;
            for (int j = 0; j < 8; ++j) {
              const double* rj = Gbuf + (c0 + j) * kBigGLd + c0;
              double v = lane < 8 ? ri[j] : 0.0;     // lanes >= 8 alias rows 0..7: no read of the element being written
              for (int k = 0; k < j; ++k) v = fma(-ri[k], rj[k], v);
              const double r = __shfl_sync(FULL, rsqrt_nr(v), j);   // 1/L_jj from lane j
              if (lane < 8 && lane >= j) ri[j] = v * r;            // L_ij (lane j: L_jj = v / sqrt(v))
              if (lane == j) invd[c0 + j] = r;
              __syncwarp();
            }
          }
          __syncthreads();
          // TRSM: rows below the panel, L21 = A21 L11^-T
          for (int i = c0 + 8 + t; i < dpad; i += kBigThreads) {
            double* ri = Gbuf + i * kBigGLd + c0;
            double x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const double* rj = Gbuf + (c0 + j) * kBigGLd + c0;
              double v = ri[j];
#pragma unroll
              for (int k = 0; k < j; ++k) v = fma(-x[k], rj[k], v);
              x[j] = v * invd[c0 + j];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) ri[j] = x[j];
          }
          __syncthreads();
          // SYRK on DMMA: trailing tiles (I, J), pb < J <= I < nbk
          const int nt = nbk - pb - 1, ntiles = nt * (nt + 1) / 2;
          for (int tt = warp; tt < ntiles; tt += kBigThreads / 32) {
            int I = 0;
            while ((I + 1) * (I + 2) / 2 <= tt) ++I;
            const int J = tt - I * (I + 1) / 2;
            const int gi = (pb + 1 + I) * 8, gj = (pb + 1 + J) * 8;
            double* cp = Gbuf + (gi + rl) * kBigGLd + gj + 2 * kl;
            double d0 = cp[0], d1 = cp[1];
#pragma unroll
            for (int ks = 0; ks < 8; ks += 4) {
              const double a = -Gbuf[(gi + rl) * kBigGLd + c0 + ks + kl];
              const double b = Gbuf[(gj + rl) * kBigGLd + c0 + ks + kl];
              dmma(d0, d1, a, b);
            }
            cp[0] = d0;
            cp[1] = d1;
          }
          __syncthreads();
        }
        for (int j = 0; j < deff; ++j)
          if (!(invd[j] > 0.0 && invd[j] < INFINITY)) ok = false;
        // solves' form: strictly lower entries scaled by their column's L_jj
        for (int e = t; e < deff * deff; e += kBigThreads) {
          const int r = e / deff, c = e - r * deff;
          if (c < r) Gbuf[r * kBigGLd + c] /= invd[c];
        }
        __syncthreads();
      }
      SR_PT(3);
      // solves by warp 0 (lane l owns rows l + 32s in registers, pivots by
      // shuffle, no shared-memory round trips): w' = G^-1 rhs, then the
      // refinement corrections.  Adaptive stop: once a correction is below
      // 1e-8 of w' (relative, max norm), the next one would be below
      // ~1e-16 (its size is the contraction factor kappa*eps_G times this
      // one, and kappa*eps_G is itself at most ~ this ratio), so further
      // passes over the data are skipped.
      for (int it = 0; it <= nref; ++it) {
        if (warp == 0) {
          double z[4], ir[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = q * 32 + lane;
            z[q] = r < deff ? (it == 0 ? rhs[r] : zv[r]) : 0.0;
            ir[q] = r < deff ? invd[r] : 0.0;
          }
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {            // forward: L y = z
            const int jend = min(32, deff - jb * 32);
            for (int jj = 0; jj < jend; ++jj) {
              const int j = jb * 32 + jj;
              const double ij = __shfl_sync(FULL, ir[jb], jj);
              const double yj = __shfl_sync(FULL, z[jb], jj) * ij;
              if (lane == jj) z[jb] = yj;
              const double tj = yj * ij;
#pragma unroll
              for (int q = jb; q < 4; ++q) {
                const int r = q * 32 + lane;
                if (r > j && r < deff) z[q] = fma(-Gbuf[r * kBigGLd + j], tj, z[q]);
              }
            }
          }
#pragma unroll
          for (int jb = 3; jb >= 0; --jb) {           // backward: L^T x = y
            const int jend = min(32, deff - jb * 32);
            for (int jj = jend - 1; jj >= 0; --jj) {
              const int j = jb * 32 + jj;
              const double xj = __shfl_sync(FULL, z[jb], jj) * __shfl_sync(FULL, ir[jb], jj);
              if (lane == jj) z[jb] = xj;
#pragma unroll
              for (int q = 0; q <= jb; ++q) {
                const int r = q * 32 + lane;
                if (r < j) z[q] = fma(-Gbuf[j * kBigGLd + r] * ir[q], xj, z[q]);
              }
            }
          }
          double dmax = 0.0, wmax = 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = q * 32 + lane;
            if (r < deff) {
              zv[r] = z[q];
              const double w = (it == 0) ? z[q] : wv[r] + z[q];
              wv[r] = w;
              dmax = fmax(dmax, fabs(z[q]));
              wmax = fmax(wmax, fabs(w));
            }
          }
          dmax = warp_max(dmax);
          wmax = warp_max(wmax);
          if (lane == 0) misc[2] = (it > 0 && dmax <= 1e-8 * wmax) ? 1 : 0;
        }
        __syncthreads();
        SR_PT(4);
        if (it == nref || misc[2]) break;
        // residual r = X~^T (yc - X~ w') - lambda w' streamed over the training rows
        for (int a = t; a < kBigMaxD; a += kBigThreads) rhs[a] = 0.0;
        __syncthreads();
        // Register-only pass: thread (row t>>3, features (t&7)+8q) holds its 16
        // centred values; the row's residual is a 3-step shuffle reduction over
        // the 8 threads of the row (fixed order), next chunk prefetched.
        double rp[16], wq[16], v[16], vn[16], vnn[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          rp[q] = 0.0;
          const int a = (t & 7) + 8 * q;
          wq[q] = a < deff ? wv[a] : 0.0;
        }
        const int nch = (n + kBigChunk - 1) / kBigChunk;
        const int rrow = t >> 3;
        // gathers two chunks ahead (register ring v <- vn <- vnn), slot indices three ahead
        int snext = big_slot(trs, n, 2);
        double ycur = rrow < n ? yl[rrow] : 0.0, ynext = kBigChunk + rrow < n ? yl[kBigChunk + rrow] : 0.0;
        big_load_rows(A.x, C, big_slot(trs, n, 0), col, deff, v);
        big_load_rows(A.x, C, big_slot(trs, n, 1), col, deff, vn);
        for (int ch = 0; ch < nch; ++ch) {
          double yfut = 0.0;
          if (ch + 2 < nch) {
            big_load_rows(A.x, C, snext, col, deff, vnn);
            snext = big_slot(trs, n, ch + 3);
          }
          {
            const int r2 = (ch + 2) * kBigChunk + rrow;
            yfut = r2 < n ? yl[r2] : 0.0;
          }
          big_scale_chunk(n, ch * kBigChunk, xb, sv, deff, v);
          double dot = 0.0;
#pragma unroll
          for (int q = 0; q < 16; ++q) dot = fma(v[q], wq[q], dot);
          dot += __shfl_xor_sync(FULL, dot, 1);
          dot += __shfl_xor_sync(FULL, dot, 2);
          dot += __shfl_xor_sync(FULL, dot, 4);
          const int gr = ch * kBigChunk + rrow;
          const double e = gr < n ? ycur - dot : 0.0;
#pragma unroll
          for (int q = 0; q < 16; ++q) rp[q] = fma(v[q], e, rp[q]);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            v[q] = vn[q];
            vn[q] = vnn[q];
          }
          ycur = ynext;
          ynext = yfut;
        }
        {
          double* part = rpt;  // never aliases the factor in Gbuf
          const int r = t >> 3, a0 = t & 7;
#pragma unroll
          for (int q = 0; q < 16; ++q) part[r * kBigMaxD + a0 + 8 * q] = rp[q];
          __syncthreads();
          if (t < deff) {
            double acc = 0.0;
            for (int rr = 0; rr < kBigChunk; ++rr) acc += part[rr * kBigMaxD + t];
            zv[t] = acc - A.lambda * wv[t];
          }
          __syncthreads();
        }
        SR_PT(5);
      }
    }
    // ---- outputs: weights on raw counters, intercept ----
    for (int c = t; c < C; c += kBigThreads) A.U[(sl * O + o) * C + c] = 0.0;
    __syncthreads();
    double cp = 0.0;
    if (deff > 0 && ok)
      for (int a = t; a < deff; a += kBigThreads) {
        const double u = wv[a] * sv[a];
        A.U[(sl * O + o) * C + col[a]] = u;
        cp = fma(xb[a], u, cp);
      }
    const double csum = cta_sum(cp, red);
    if (t == 0) {
      A.c0[sl * O + o] = ybar - csum;
      A.fitflag[sl * O + o] = ok ? 1 : 2;  // 2: poisoned (non-positive pivot)
      A.opt_out[sl * O + o] = row;
    }
    __syncthreads();
    SR_PT(6);
  }
#if SPEEDREC_PHASE_TIMING
  if (blockIdx.x == 0 && t == 0)
    printf("k_fit_big CTA0 cycles: A1 %lld stats %lld gram %lld chol %lld solves %lld refine %lld out %lld\n", ph[0],
           ph[1], ph[2], ph[3], ph[4], ph[5], ph[6]);
#endif
}

// ---- A5-A7 for one scenario per CTA ----
// Prediction on the FP64 tensor pipe: for each group, EX for its 64 versions x
// the scored optimizations is one (64 x C) x (C x 8) product (8 row-block
// DMMA tiles per k-step; training rows are zeroed, not loaded), the tile goes
// through shared memory and each lane then ranks/scores its own versions.
template <int CMAX>
__global__ void __launch_bounds__(kBigThreads) k_rank_big(const BigArgs A) {
  constexpr int NT = CMAX / 8;                  // 8-column tiles of scored optimizations
  constexpr int ULD = kBigMaxD + 4;
  __shared__ double Us[CMAX][ULD];
  __shared__ double c0s[CMAX];
  __shared__ int ols[CMAX];
  __shared__ int trained_s[CMAX];
  __shared__ double exs[kBigThreads / 32][64][CMAX + 1];
  __shared__ double redd[kBigThreads / 32][CMAX][3];
  __shared__ int redi[kBigThreads / 32][CMAX][2];
  __shared__ int reds[kBigThreads / 32][4];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int G = A.G, O = A.O, C = A.C;
  const long long sl = blockIdx.x;
  const long long s = A.first + sl;
  const long long split = s % A.n_splits;
  const uint32_t om = (A.split_om ? A.split_om[split] : A.opt_mask) & ((1u << O) - 1u);
  int n_os = 0;
  for (int o = 0; o < O; ++o)
    if ((om >> o) & 1u) {
      if (t == 0) {
        ols[n_os] = o;
        trained_s[n_os] = A.fitflag[sl * O + o];
        c0s[n_os] = A.c0[sl * O + o];
      }
      for (int c = t; c < ULD; c += kBigThreads) Us[n_os][c] = c < C ? A.U[(sl * O + o) * C + c] : 0.0;
      ++n_os;
    }
  for (int q = n_os; q < CMAX; ++q)
    for (int c = t; c < ULD; c += kBigThreads) Us[q][c] = 0.0;
  if (A.ex_out)
    for (int i = t; i < O * G * 32; i += kBigThreads) A.ex_out[sl * (long long)O * G * 32 + i] = 0.0;
  if (A.rec_out)
    for (int i = t; i < G * 64 * A.max_count; i += kBigThreads) A.rec_out[sl * (long long)G * 64 * A.max_count + i] = -1;
  __syncthreads();
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
  const int rl = lane >> 2, kl = lane & 3;
  double (*ex)[CMAX + 1] = exs[warp];
  for (int g = warp; g < G; g += kBigThreads / 32) {
    uint64_t tr, te;
    member_words(A, split, g, tr, te);
    if (te == 0ull) continue;
    const int p = g / A.IR;
    // ---- EX tile: (64 versions) x (C counters) times (C) x (CMAX weights) ----
    double acc[8][NT][2];
#pragma unroll
    for (int rb = 0; rb < 8; ++rb)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[rb][nt][0] = acc[rb][nt][1] = 0.0;
    const double* xg = A.x + (long long)g * 64 * C;
    for (int k0 = 0; k0 < C; k0 += 4) {
      const int kk = k0 + kl;
      double b[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = Us[nt * 8 + rl][kk];
#pragma unroll
      for (int rb = 0; rb < 8; ++rb) {
        const int v = rb * 8 + rl;
        const double a = (((te >> v) & 1ull) && kk < C) ? xg[v * C + kk] : 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[rb][nt][0], acc[rb][nt][1], a, b[nt]);
      }
    }
#pragma unroll
    for (int rb = 0; rb < 8; ++rb)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        ex[rb * 8 + rl][nt * 8 + 2 * kl] = acc[rb][nt][0];
        ex[rb * 8 + rl][nt * 8 + 2 * kl + 1] = acc[rb][nt][1];
      }
    __syncwarp();
    // ---- per version: clamp, score, rank (lane owns versions lane, lane+32) ----
    for (int h = 0; h < 2; ++h) {
      const int v = h * 32 + lane;
      if (!((te >> v) & 1ull)) continue;
      double ce[CMAX];
      bool cv[CMAX], cc[CMAX];
      int ck[CMAX];
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        cv[q] = false;
        cc[q] = false;
        ck[q] = 0;
        ce[q] = 0.0;
        if (q < n_os) {
          const int o = ols[q];
          const int b = A.opt_bit[p * O + o];
          if (b >= 0 && !((v >> b) & 1)) {
            if (trained_s[q] != 1) {
              if (trained_s[q] == 0) ++untrained;
              if (trained_s[q] == 2) guard += 1000000;
              continue;
            }
            const int k = rmv(v, b);
            double e = c0s[q] + ex[v][q];
            if (near_tol(e, 0.0, A.guard_tol) || near_tol(e, 1.0, A.guard_tol)) ++guard;
            bool cl = false;
            if (e <= 0.0) {
              e = A.clamp_floor;
              cl = true;
            }
            const double ac = A.ylab[(g * O + o) * 32 + k];
            cv[q] = true;
            cc[q] = cl;
            ck[q] = k;
            ce[q] = e;
            const double ratio = ac / e;
            pc[q] += ((e > 1.0 && ac > 1.0) || (e <= 1.0 && ac <= 1.0)) ? 1 : 0;
            pcl[q] += cl ? 1 : 0;
            ps[q] += ratio;
            pmn[q] = fmin(pmn[q], ratio);
            pmx[q] = fmax(pmx[q], ratio);
            if (A.ex_out) A.ex_out[(sl * O + o) * (long long)G * 32 + g * 32 + k] = e;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        if (!cv[q]) continue;
        if (near_tol(ce[q], A.threshold, A.guard_tol)) ++guard;
#pragma unroll
        for (int r = q + 1; r < CMAX; ++r)
          if (cv[r] && !(cc[q] && cc[r]) && near_tol(ce[q], ce[r], A.guard_tol)) ++guard;
      }
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        if (!cv[q] || !(ce[q] >= A.threshold)) continue;
        int rk = 0;
#pragma unroll
        for (int r = 0; r < CMAX; ++r)
          if (r != q && cv[r] && ce[r] >= A.threshold && (ce[r] > ce[q] || (ce[r] == ce[q] && r < q))) ++rk;
        if (rk < A.max_count) {
          ++nrec;
          const int o = ols[q];
          if (A.ylab[(g * O + o) * 32 + ck[q]] > 1.0) ++nhit;
          if (A.rec_out) A.rec_out[(sl * G * 64 + g * 64 + v) * A.max_count + rk] = (int8_t)o;
        }
      }
    }
    __syncwarp();
  }
  // ---- deterministic reduction: lanes (butterfly), then warps in order ----
#pragma unroll
  for (int q = 0; q < CMAX; ++q) {
    const int a = warp_isum(pc[q]), b = warp_isum(pcl[q]);
    const double sm = warp_sum(ps[q]), mn = warp_min(pmn[q]), mx = warp_max(pmx[q]);
    if (lane == 0) {
      redi[warp][q][0] = a;
      redi[warp][q][1] = b;
      redd[warp][q][0] = sm;
      redd[warp][q][1] = mn;
      redd[warp][q][2] = mx;
    }
  }
  {
    const int a = warp_isum(nrec), b = warp_isum(nhit), c = warp_isum(untrained), d = warp_isum(guard);
    if (lane == 0) {
      reds[warp][0] = a;
      reds[warp][1] = b;
      reds[warp][2] = c;
      reds[warp][3] = d;
    }
  }
  __syncthreads();
  if (t < n_os) {
    const int q = t, o = ols[q];
    OptScore row = A.opt_out[sl * O + o];
    int nc = 0, ncl = 0;
    double sm = 0.0, mn = INFINITY, mx = -INFINITY;
    for (int w = 0; w < kBigThreads / 32; ++w) {
      nc += redi[w][q][0];
      ncl += redi[w][q][1];
      sm += redd[w][q][0];
      mn = fmin(mn, redd[w][q][1]);
      mx = fmax(mx, redd[w][q][2]);
    }
    const bool has = row.n_test > 0 && trained_s[q] == 1;
    row.n_correct = nc;
    row.n_clamped = ncl;
    row.sum_ratio = has ? sm : 0.0;
    row.min_ratio = has ? mn : 0.0;
    row.max_ratio = has ? mx : 0.0;
    A.opt_out[sl * O + o] = row;
    if (A.totals && has) {
      atomicAdd(&A.totals[0], (unsigned long long)nc);
      atomicAdd(&A.totals[1], (unsigned long long)row.n_test);
    }
  }
  if (t == 0) {
    ScnScore sr{0, 0, 0, 0};
    for (int w = 0; w < kBigThreads / 32; ++w) {
      sr.n_rec += reds[w][0];
      sr.n_rec_hit += reds[w][1];
      sr.n_untrained += reds[w][2];
      sr.n_guard += reds[w][3];
    }
    A.scn_out[sl] = sr;
    if (A.totals) {
      atomicAdd(&A.totals[2], (unsigned long long)sr.n_rec);
      atomicAdd(&A.totals[3], (unsigned long long)sr.n_rec_hit);
    }
  }
}

// ---- A5-A7 for kRankSB scenarios per CTA ----
// The scenarios of a CTA share every group's 64 x C rate tile: it is staged
// once per group in shared memory (cp.async, double-buffered, 64 KB) and
// multiplied on DMMA by the weights of all kRankSB x 8 (scenario, scored
// optimization) columns: warp w owns versions 8w..8w+7, 4 column tiles.  Then
// thread (scenario t>>6, version t&63) clamps, scores and ranks its version's
// candidates; per-scenario sums are reduced over its 64 threads in a fixed
// order at the end.
constexpr int kRankSB = 4;
constexpr int kBigYO = 16;       // optimization ids a staged label block holds (O <= 16)

static __global__ void __launch_bounds__(kBigThreads, 1) k_rank_big4(const BigArgs A) {
  constexpr int CM = 8, NC = kRankSB * CM, ULD = kBigMaxD + 4, XLD = kBigMaxD + 4;
  extern __shared__ __align__(16) unsigned char smem[];
  double* Us = reinterpret_cast<double*>(smem);                 // [NC][ULD]
  double* xs = Us + NC * ULD;                                   // [2][64][XLD]
  double* exs = xs + 2 * 64 * XLD;                              // [64][NC + 1]
  double* c0s = exs + 64 * (NC + 1);                            // [NC]
  double* redd = c0s + NC;                                      // [8 warps][CM][3]
  double* ys = redd + 8 * CM * 3;                               // [2][O][32] labels of the staged group
  int* ols = reinterpret_cast<int*>(ys + 2 * kBigYO * 32);   // [NC]
  int* trs_ = ols + NC;                                         // [NC] fit flags
  int* nos = trs_ + NC;                                         // [kRankSB]
  int* redi = nos + kRankSB;                                    // [8][CM][2]
  int* reds = redi + 8 * CM * 2;                                // [8][4]
  int8_t* obs = reinterpret_cast<int8_t*>(reds + 8 * 4);        // [P][O] opt bits
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int G = A.G, O = A.O, C = A.C;
  const long long sl0 = (long long)blockIdx.x * kRankSB;
  const int nsb = (int)(A.count - sl0 < kRankSB ? A.count - sl0 : kRankSB);
  // weights, intercepts, scored lists
  if (t < kRankSB) {
    int n = 0;
    if (t < nsb) {
      const long long sl = sl0 + t, split = (A.first + sl) % A.n_splits;
      const uint32_t om = (A.split_om ? A.split_om[split] : A.opt_mask) & ((1u << O) - 1u);
      for (int o = 0; o < O && n < CM; ++o)
        if ((om >> o) & 1u) {
          ols[t * CM + n] = o;
          trs_[t * CM + n] = A.fitflag[sl * O + o];
          c0s[t * CM + n] = A.c0[sl * O + o];
          ++n;
        }
    }
    nos[t] = n;
  }
  for (int i = t; i < A.P * O; i += kBigThreads) obs[i] = A.opt_bit[i];
  __syncthreads();
  for (int i = t; i < NC * ULD; i += kBigThreads) {
    const int col = i / ULD, c = i % ULD, sb = col / CM, q = col % CM;
    double u = 0.0;
    if (sb < nsb && q < nos[sb] && c < C) u = A.U[((sl0 + sb) * O + ols[sb * CM + q]) * C + c];
    Us[i] = u;
  }
  for (int sb = 0; sb < nsb; ++sb) {
    const long long sl = sl0 + sb;
    if (A.ex_out)
      for (int i = t; i < O * G * 32; i += kBigThreads) A.ex_out[sl * (long long)O * G * 32 + i] = 0.0;
    if (A.rec_out)
      for (int i = t; i < G * 64 * A.max_count; i += kBigThreads) A.rec_out[sl * (long long)G * 64 * A.max_count + i] = -1;
  }
  for (int i = t; i < 2 * 64 * (XLD - C); i += kBigThreads) {   // pad columns (never copied) read as 0
    const int r = i / (XLD - C), c = C + i % (XLD - C);
    xs[r * XLD + c] = 0.0;
  }
  // stage the 64 x C rate tile of group g (16-byte cp.async; C is a multiple of 2)
  auto stage = [&](int g, int buf) {
    const double* src = A.x + (long long)g * 64 * C;
    double* dst = xs + buf * 64 * XLD;
    const int per_row = C / 2;
    if (kBigThreads % per_row == 0) {             // a fixed 16-byte column per thread, no division per copy
      const int c2 = (t % per_row) * 2, rs = kBigThreads / per_row;
      for (int r = t / per_row; r < 64; r += rs) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst + r * XLD + c2);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + r * C + c2) : "memory");
      }
    } else {
      for (int i = t; i < 64 * per_row; i += kBigThreads) {
        const int r = i / per_row, c2 = (i % per_row) * 2;
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst + r * XLD + c2);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + r * C + c2) : "memory");
      }
    }
    // the group's labels ylab[g][o][k] (the same for every scenario)
    const double* ysrc = A.ylab + (long long)g * O * 32;
    double* ydst = ys + buf * kBigYO * 32;
    for (int i = t; i < O * 16; i += kBigThreads) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(ydst + 2 * i);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(ysrc + 2 * i) : "memory");
    }
    cp_commit();
  };
  // this thread's scenario / version and its partial scores
  const int msb = t >> 6, v = t & 63;
  const bool mine = msb < nsb;
  const long long msl = sl0 + msb, msplit = (A.first + msl) % A.n_splits;
  const int my_n = mine ? nos[msb] : 0;
  int pc[CM], pcl[CM];
  double ps[CM], pmn[CM], pmx[CM];
#pragma unroll
  for (int q = 0; q < CM; ++q) {
    pc[q] = pcl[q] = 0;
    ps[q] = 0.0;
    pmn[q] = INFINITY;
    pmx[q] = -INFINITY;
  }
  int nrec = 0, nhit = 0, guard = 0, untrained = 0;
  const int rl = lane >> 2, kl = lane & 3;
  stage(0, 0);
  for (int g = 0; g < G; ++g) {
    if (g + 1 < G) {
      stage(g + 1, (g + 1) & 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();                              // tile g landed; EX tile of g-1 consumed
    // ---- EX tile: (64 versions) x (C counters) times (C) x (NC columns) ----
    {
      const double* xt = xs + (g & 1) * 64 * XLD;
      // two accumulator sets over alternating k-steps (independent DMMA
      // chains), added at the end
      double acc[NC / 8][2], acc2[NC / 8][2];
#pragma unroll
      for (int nt = 0; nt < NC / 8; ++nt) acc[nt][0] = acc[nt][1] = acc2[nt][0] = acc2[nt][1] = 0.0;
      const double* arow = xt + (warp * 8 + rl) * XLD + kl;
      int k0 = 0;
#pragma unroll 2
      for (; k0 + 4 < C; k0 += 8) {
        const double a = arow[k0], a2 = arow[k0 + 4];
#pragma unroll
        for (int nt = 0; nt < NC / 8; ++nt) {
          dmma(acc[nt][0], acc[nt][1], a, Us[(nt * 8 + rl) * ULD + k0 + kl]);
          dmma(acc2[nt][0], acc2[nt][1], a2, Us[(nt * 8 + rl) * ULD + k0 + 4 + kl]);
        }
      }
      if (k0 < C) {
        const double a = arow[k0];
#pragma unroll
        for (int nt = 0; nt < NC / 8; ++nt) dmma(acc[nt][0], acc[nt][1], a, Us[(nt * 8 + rl) * ULD + k0 + kl]);
      }
#pragma unroll
      for (int nt = 0; nt < NC / 8; ++nt) {
        exs[(warp * 8 + rl) * (NC + 1) + nt * 8 + 2 * kl] = acc[nt][0] + acc2[nt][0];
        exs[(warp * 8 + rl) * (NC + 1) + nt * 8 + 2 * kl + 1] = acc[nt][1] + acc2[nt][1];
      }
    }
    __syncthreads();
    // ---- per (scenario, version): clamp, score, rank ----
    if (mine) {
      uint64_t tr, te;
      member_words(A, msplit, g, tr, te);
      if ((te >> v) & 1ull) {
        const int p = g / A.IR;
        double ce[CM];
        bool cv[CM], cc[CM];
        int ck[CM];
#pragma unroll
        for (int q = 0; q < CM; ++q) {
          cv[q] = false;
          cc[q] = false;
          ck[q] = 0;
          ce[q] = 0.0;
          if (q < my_n) {
            const int o = ols[msb * CM + q];
            const int b = obs[p * O + o];
            if (b >= 0 && !((v >> b) & 1)) {
              const int fl = trs_[msb * CM + q];
              if (fl != 1) {
                if (fl == 0) ++untrained;
                if (fl == 2) guard += 1000000;
                continue;
              }
              const int k = rmv(v, b);
              double e = c0s[msb * CM + q] + exs[v * (NC + 1) + msb * CM + q];
              if (near_tol(e, 0.0, A.guard_tol) || near_tol(e, 1.0, A.guard_tol)) ++guard;
              bool cl = false;
              if (e <= 0.0) {
                e = A.clamp_floor;
                cl = true;
              }
              const double ac = ys[(g & 1) * kBigYO * 32 + o * 32 + k];
              cv[q] = true;
              cc[q] = cl;
              ck[q] = k;
              ce[q] = e;
              const double ratio = ac / e;
              pc[q] += ((e > 1.0 && ac > 1.0) || (e <= 1.0 && ac <= 1.0)) ? 1 : 0;
              pcl[q] += cl ? 1 : 0;
              ps[q] += ratio;
              pmn[q] = fmin(pmn[q], ratio);
              pmx[q] = fmax(pmx[q], ratio);
              if (A.ex_out) A.ex_out[(msl * O + o) * (long long)G * 32 + g * 32 + k] = e;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < CM; ++q) {
          if (!cv[q]) continue;
          if (near_tol(ce[q], A.threshold, A.guard_tol)) ++guard;
#pragma unroll
          for (int r = q + 1; r < CM; ++r)
            if (cv[r] && !(cc[q] && cc[r]) && near_tol(ce[q], ce[r], A.guard_tol)) ++guard;
        }
#pragma unroll
        for (int q = 0; q < CM; ++q) {
          if (!cv[q] || !(ce[q] >= A.threshold)) continue;
          int rk = 0;
#pragma unroll
          for (int r = 0; r < CM; ++r)
            if (r != q && cv[r] && ce[r] >= A.threshold && (ce[r] > ce[q] || (ce[r] == ce[q] && r < q))) ++rk;
          if (rk < A.max_count) {
            ++nrec;
            const int o = ols[msb * CM + q];
            if (ys[(g & 1) * kBigYO * 32 + o * 32 + ck[q]] > 1.0) ++nhit;
            if (A.rec_out) A.rec_out[(msl * G * 64 + g * 64 + v) * A.max_count + rk] = (int8_t)o;
          }
        }
      }
    }
    // the next iteration's cp.async stage(g + 2) overwrites this group's label
    // buffer ys[g & 1]: every thread must be done scoring group g first (a
    // thread with no scenario of its own otherwise races ahead; found by the
    // single-scenario C4 parity test, tests/test_gpu_samples.py)
    __syncthreads();
  }
  // ---- deterministic reduction per scenario: lanes (butterfly), its 2 warps in order ----
#pragma unroll
  for (int q = 0; q < CM; ++q) {
    const int a = warp_isum(pc[q]), b = warp_isum(pcl[q]);
    const double sm = warp_sum(ps[q]), mn = warp_min(pmn[q]), mx = warp_max(pmx[q]);
    if (lane == 0) {
      redi[(warp * CM + q) * 2 + 0] = a;
      redi[(warp * CM + q) * 2 + 1] = b;
      redd[(warp * CM + q) * 3 + 0] = sm;
      redd[(warp * CM + q) * 3 + 1] = mn;
      redd[(warp * CM + q) * 3 + 2] = mx;
    }
  }
  {
    const int a = warp_isum(nrec), b = warp_isum(nhit), c = warp_isum(untrained), d = warp_isum(guard);
    if (lane == 0) {
      reds[warp * 4 + 0] = a;
      reds[warp * 4 + 1] = b;
      reds[warp * 4 + 2] = c;
      reds[warp * 4 + 3] = d;
    }
  }
  __syncthreads();
  if (t < nsb * CM) {
    const int sb = t / CM, q = t % CM;
    if (q < nos[sb]) {
      const long long sl = sl0 + sb;
      const int o = ols[sb * CM + q];
      OptScore row = A.opt_out[sl * O + o];
      int nc = 0, ncl = 0;
      double sm = 0.0, mn = INFINITY, mx = -INFINITY;
      for (int w = 2 * sb; w < 2 * sb + 2; ++w) {
        nc += redi[(w * CM + q) * 2 + 0];
        ncl += redi[(w * CM + q) * 2 + 1];
        sm += redd[(w * CM + q) * 3 + 0];
        mn = fmin(mn, redd[(w * CM + q) * 3 + 1]);
        mx = fmax(mx, redd[(w * CM + q) * 3 + 2]);
      }
      const bool has = row.n_test > 0 && trs_[sb * CM + q] == 1;
      row.n_correct = nc;
      row.n_clamped = ncl;
      row.sum_ratio = has ? sm : 0.0;
      row.min_ratio = has ? mn : 0.0;
      row.max_ratio = has ? mx : 0.0;
      A.opt_out[sl * O + o] = row;
      if (A.totals && has) {
        atomicAdd(&A.totals[0], (unsigned long long)nc);
        atomicAdd(&A.totals[1], (unsigned long long)row.n_test);
      }
    }
  }
  if (t < nsb) {
    ScnScore sr{0, 0, 0, 0};
    for (int w = 2 * t; w < 2 * t + 2; ++w) {
      sr.n_rec += reds[w * 4 + 0];
      sr.n_rec_hit += reds[w * 4 + 1];
      sr.n_untrained += reds[w * 4 + 2];
      sr.n_guard += reds[w * 4 + 3];
    }
    A.scn_out[sl0 + t] = sr;
    if (A.totals) {
      atomicAdd(&A.totals[2], (unsigned long long)sr.n_rec);
      atomicAdd(&A.totals[3], (unsigned long long)sr.n_rec_hit);
    }
  }
}

// shared-memory bytes of k_rank_big4
// (+ the [P][O] opt bits, sized at launch)
constexpr int kRankBig4Smem = (8 * 4 * (kBigMaxD + 4) + 2 * 64 * (kBigMaxD + 4) + 64 * (8 * 4 + 1) + 8 * 4 + 8 * 8 * 3 +
                               2 * kBigYO * 32) * 8 + (2 * 8 * 4 + 4 + 8 * 8 * 2 + 8 * 4) * 4;

}  // namespace speedrec
