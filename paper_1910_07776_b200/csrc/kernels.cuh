// kernels.cuh -- sm_100a kernels of the Tier-2/Tier-3 hot path of
// arXiv 1910.07776 (see include/speedrec.h for the step list A0-A7 and
// DESIGN.md §5-6 for the data layout and the roofline of each kernel).
//
// Design (B200-first):
//  * k_rates / k_labels: elementwise FP64 IEEE divisions (A0, A1 labels),
//    grid-stride, coalesced; bit-exact by construction.
//  * k_eval_warp: one warp owns one scenario end to end (A1-A7): split
//    membership from the counter-based hash, pair compaction by ballot,
//    per-fit min-max statistics, the centred Gram (dual n x n when the fit is
//    underdetermined, primal d x d otherwise) accumulated on the FP64 tensor
//    pipe with mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), a packed warp Cholesky
//    with rsqrt pivots, two refinement steps whose residual is formed from
//    the data rows, prediction, clamping, warp-shuffle top-k ranking and the
//    segmented score reduction.  No inter-warp synchronisation: a persistent
//    grid of warps strides over scenarios.  The scenario's rate matrix is
//    staged once per CTA in shared memory when it fits (C1, C3, C5).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace speedrec {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kMaxOpt = 16;
constexpr int kMaxGroups = 64;       // warp-per-scenario path
constexpr int kMaxGroupsBig = 4096;  // CTA-per-fit path (config C4)
constexpr int kMaxCounters = 128;
constexpr int kMaxRec = 8;
constexpr int kKnnMax = 16;            // largest IBK k (sr_params.k_nn)
constexpr int kKnnRows = 8;            // training rows staged per IBK distance sweep
constexpr int kMaxWarpsPerBlock = 16;  // default warps/CTA of k_fit_warp (tools/tune_launch.sh)

struct OptScore {
  int32_t n_train, n_test, n_correct, n_clamped;
  double sum_ratio, min_ratio, max_ratio;
  uint64_t fp_train, fp_test;
};
struct ScnScore {
  int32_t n_rec, n_rec_hit, n_untrained, n_guard;
};
struct MaskScore {
  int32_t n_correct, n_test, n_rec, n_rec_hit;
};

// Scenario batch as the kernels see it (sr_scenarios after validation).
struct ScenDesc {
  int kind;              // 0 groups, 1 loo, 2 random
  int gw;                // group words
  long long n_splits;
  const uint64_t* train_g;
  const uint64_t* test_g;
  const uint32_t* split_om;
  const int32_t* pool_list;  // pool groups ascending
  int n_pool;
  unsigned long long seed;
  uint32_t opt_mask;
  int subsets_k;
  long long n_masks;
  const uint64_t* fmasks;    // [n_masks][2] or null
};

// Per-warp shared-memory layout of k_fit_warp (byte offsets inside the slab).
struct WarpLayout {
  int bytes;            // slab size (multiple of 16)
  int off_trw, off_tew; // uint64 [G] split words of the fit's scenario
  int off_F;            // int16 [dmax] feature columns of the scenario
  int off_trs;          // int32 [np_tr]  training before-slots
  int off_yc;           // double [np_tr] training labels, centred in place
  int off_tes;          // int32 [np_te]  test before-slots
  int off_tek;          // int32 [np_te]  g*32+k of the test case
  int np_tr, np_te;
  int off_col;          // int16 [dpad] active feature columns (zero padded)
  int off_xb;           // double [dpad]
  int off_s;            // double [dpad]
  int off_w;            // double [dmax]  weights on scaled features
  int off_u;            // double [dmax]  work vector
  int off_v2;           // double [vmax] residual / work vector
  int off_M;            // double [mcap(mcap+1)/2] packed factor
  int mcap;
  int vmax;
  int off_ufull;        // double [C] weights on raw counters
};

// Arguments of the warp-per-fit path (k_fit_warp, k_rank_warp, k_mask_final).
struct EvalArgs {
  // dataset (device)
  const double* x;       // rates [N][C]
  const double* ylab;    // labels [G][O][32]
  const int8_t* opt_bit; // [P][O]
  int P, IR, C, O, G;
  ScenDesc sd;
  // params
  double lambda, threshold, clamp_floor, guard_tol;
  int max_count, refine;
  int learner, k_nn;    // SR_LINREG / SR_IBK and the IBK k
  // scenario range of this launch (a chunk of the sr_evaluate range)
  long long first, count;
  long long out0;        // index of `first` inside the caller's output arrays
  // per-chunk exchange between the fit and rank kernels
  double* extab;         // [count][ex_stride]: EX per (scored-opt slot q, test group, k); clamped -> -EX
  int ex_stride, tg_stride;  // tg_stride = 32 * max test groups; ex_stride = n_os_max * tg_stride
  uint32_t* trained;     // [count] bit o set iff optimization o has >= 1 training pair
  int* guard_acc;        // [count] guard cases counted by the fit kernel
  int* done;             // [count] scored fits finished (fused ranking)
  unsigned long long* queue;   // k_fit_warp work units handed out past the first nteams (nullptr: static stride)
  int fuse_rank;         // 1: k_fit_warp ranks each scenario after its last fit (no k_rank_warp)
  // outputs (device, indexed by out0 + local scenario)
  OptScore* opt_out;     // [.][O] or null
  ScnScore* scn_out;     // or null
  double* ex_out;        // [.][O][G*32] or null (pre-zeroed)
  int8_t* rec_out;       // [.][N][max_count] or null (pre-filled with -1)
  unsigned long long* totals;  // [4] or null
  double* coef_out;            // sr_fit: [count][O][1 + C] raw-counter weights (c0, u), or null
  // mask aggregation (C5)
  int agg;
  int* mask_acc;         // [masks of the evaluate range][4], atomically accumulated
  long long mask0;       // first mask id of the evaluate range
  MaskScore* mask_out;
  unsigned long long* keys_out;
  long long n_mask_range;
  // workspace of k_fit_warp
  WarpLayout L;
  int warps_per_block;
  int stage_x;           // 1: stage x [N][C] in smem with ld = ldxs
  int ldxs;
  int off_stage;         // byte offset of the staged x (after the opt_bit table)
  int off_warps;         // byte offset of the first warp slab
  double* gscratch;      // per global warp: mscratch doubles (large systems: factor + 2 vectors)
  long long mscratch;
  // model table of the split LS path (k_fit_warp MODE 4 -> k_pred_rank):
  // [count][n_os][ldu]: u[0..Cp) raw-counter weights (Cp = C rounded up to 4,
  // zero padded), then c0, flag, n_train, n_test, fp_train bits, fp_test bits
  // (flag 0 untrained, 1 fitted, 2 non-positive pivot)
  double* utab;
  int ldu;
  int n_os;              // scored-optimization slots per scenario (table rows)
  int scn_major;         // k_fit_warp work unit: 1 = a whole scenario, 0 = one fit
  int stage_y;           // 1: the labels ylab [G][O][32] staged in shared memory at off_y
  int off_y;
  int m5_team;           // M5P: warps per fit (1, 2 or 4; divides warps_per_block)
  unsigned long long* work;    // M5P: executed split-search FP64 operations (sr_last_work), or null
};
// model-table row fields after the C weights (k_fit_warp MODE 4 / k_pred_rank)
constexpr int kUc0 = 0, kUflag = 1, kUntr = 2, kUnte = 3, kUfptr = 4, kUfpte = 5, kUextra = 6;

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Train/test words of group g under split k (reading R17).
__device__ __forceinline__ void member_words(const ScenDesc& D, long long split, int g, uint64_t& tr,
                                             uint64_t& te) {
  if (D.kind == 0) {
    tr = ((D.train_g[split * D.gw + (g >> 6)] >> (g & 63)) & 1ull) ? ~0ull : 0ull;
    te = ((D.test_g[split * D.gw + (g >> 6)] >> (g & 63)) & 1ull) ? ~0ull : 0ull;
  } else if (D.kind == 1) {
    bool inpool = false;
    for (int q = 0; q < D.n_pool; ++q) inpool |= (D.pool_list[q] == g);
    tr = inpool ? ~0ull : 0ull;
    te = 0ull;
    if (g == D.pool_list[split >> 6]) {
      tr &= ~(1ull << (split & 63));
      te = 1ull << (split & 63);
    }
  } else {
    tr = mix64(mix64(D.seed ^ mix64((uint64_t)split)) + (uint64_t)g);
    te = ~tr;
  }
}

// Index of group g among the split's test groups (EX-table row).
__device__ __forceinline__ int test_group_index(const ScenDesc& D, long long split, int g) {
  if (D.kind == 2) return g;
  if (D.kind == 1) return 0;
  int gi = 0;
  for (int w = 0; w < (g >> 6); ++w) gi += __popcll(D.test_g[split * D.gw + w]);
  return gi + __popcll(D.test_g[split * D.gw + (g >> 6)] & ((1ull << (g & 63)) - 1ull));
}

__device__ __forceinline__ uint32_t scored_mask(const ScenDesc& D, long long split, int O) {
  return (D.split_om ? D.split_om[split] : D.opt_mask) & ((1u << O) - 1u);
}

__device__ __forceinline__ bool feature_in(const ScenDesc& D, long long fidx, int c) {
  if (D.subsets_k > 0) return c < D.subsets_k && ((fidx >> c) & 1);
  if (D.fmasks) return (D.fmasks[fidx * 2 + (c >> 6)] >> (c & 63)) & 1ull;
  return true;
}
__device__ __forceinline__ int ins0(int k, int b) { return ((k >> b) << (b + 1)) | (k & ((1 << b) - 1)); }
__device__ __forceinline__ int rmv(int v, int b) { return (v & ((1 << b) - 1)) | ((v >> (b + 1)) << b); }
__device__ __forceinline__ int pk(int r, int c) { return ((r * (r + 1)) >> 1) + c; }
// Row offset of a lower-triangular layout whose rows are padded to even
// length (16-byte aligned rows): rb2(2p) = 2p(p+1), rb2(2p+1) = 2(p+1)^2.
__host__ __device__ __forceinline__ int rb2(int i) { const int p = i >> 1; return (i & 1) ? 2 * (p + 1) * (p + 1) : 2 * p * (p + 1); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ int warp_isum(int v) {   // one REDUX (sm_80+)
  return (int)__reduce_add_sync(FULL, (unsigned)v);
}
__device__ __forceinline__ unsigned long long warp_usum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ uint64_t warp_xor(uint64_t v) {   // two REDUX on the halves
  const unsigned lo = __reduce_xor_sync(FULL, (unsigned)v), hi = __reduce_xor_sync(FULL, (unsigned)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}
// 1/sqrt(x) for a Cholesky pivot: MUFU.RSQ64H estimate + two branch-free
// Newton steps (relative error a few ulp).  x <= 0, inf or NaN give NaN or
// inf, which the callers' pivot checks reject; subnormal x is flushed (a
// pivot that small never passes them either).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = fma(y, fma(-h * y, y, 0.5), y);
  y = fma(y, fma(-h * y, y, 0.5), y);
  return y;
}

// Unroll factors of the warp path's hot loops (A/B knobs, -DSR_UNROLL_*=n).
#define SR_PRAGMA_(x) _Pragma(#x)
#define SR_UNROLL(n) SR_PRAGMA_(unroll n)
#ifndef SR_UNROLL_GRAM
#define SR_UNROLL_GRAM 1
#endif
#ifndef SR_UNROLL_STATS
#define SR_UNROLL_STATS 1
#endif
#ifndef SR_UNROLL_PRED
#define SR_UNROLL_PRED 1
#endif
#ifndef SR_UNROLL_CHOL
#define SR_UNROLL_CHOL 2
#endif
#ifndef SR_UNROLL_XTA
#define SR_UNROLL_XTA 2
#endif

// Instrumented build (-DSR_WARP_TIMING=1): k_fit_warp MODE 4 charges the
// cycles between consecutive SR_WT(k) marks to phase k, per warp (lane 0);
// CTA 0 prints its warps' totals at exit.  Timing only, never a bench build.
#if SR_WARP_TIMING
__device__ long long sr_wt_acc[148 * 32][8];
__device__ long long sr_wt_last[148 * 32];
__device__ __forceinline__ void sr_wt(int k) {
  if ((threadIdx.x & 31) == 0) {
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long now = clock64();
    if (k >= 0) sr_wt_acc[w][k] += now - sr_wt_last[w];
    sr_wt_last[w] = now;
  }
}
#define SR_WT(k) sr_wt(k)
#else
#define SR_WT(k)
#endif
// M5P phases (-DSR_M5_TIMING=1, same accumulators): 0 split search, 1
// partition, 2 node models, 3 pruning residuals, 4 scaled rows, 5 prediction
#if SR_M5_TIMING && SR_WARP_TIMING
#define SR_M5T(k) sr_wt(k)
#else
#define SR_M5T(k)
#endif

// min / max of non-NaN doubles: one compare + select (fmin/fmax add NaN handling)
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

__device__ __forceinline__ bool near_tol(double a, double b, double tol) {
  double s = fabs(a) > 1.0 ? fabs(a) : 1.0;
  return fabs(a - b) <= tol * s;
}
// D(8x8) += A(8x4) * B(4x8), FP64 tensor pipe (SASS DMMA.8x8x4).
// Lane l holds A[l>>2][l&3], B[l&3][l>>2], D[l>>2][2(l&3) + {0,1}].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// 8-byte asynchronous global -> shared copy (LDGSTS); zero-fills when !valid.
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(gsrc), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// 16-byte asynchronous global -> shared copy (LDGSTS, bypassing L1).
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}

// 1-D bulk copy global -> shared (TMA engine) completing on an mbarrier, and
// the mbarrier operations it needs (CTA scope; no cluster launch).
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(sdst)),
               "l"(gsrc), "r"(bytes), "r"(b)
               : "memory");
}
// split form: one arrive.expect_tx for the total, then copies that only complete_tx
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_tx(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(sdst)),
               "l"(gsrc), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(b), "r"(phase)
      : "memory");
}
// 1/x for x > 0 finite: MUFU.RCP64H estimate + two Newton steps (<= 2 ulp).
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// ---------------------------------------------------------------- A0 / A1
// x = counters / cycles, IEEE division => bit-exact with any
// correctly rounded implementation.
static __global__ void k_rates(const double* __restrict__ counters, const double* __restrict__ cycles,
                        double* __restrict__ x, long long n_slots, int C) {
  long long total = n_slots * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = counters[i] / cycles[i / C];
}

// ylab[g][o][k] = rt[before] / rt[after] (reading D2), 0 when the
// optimization is absent from the group's program.
static __global__ void k_labels(const double* __restrict__ rt, const int8_t* __restrict__ opt_bit,
                         double* __restrict__ ylab, int G, int O, int IR) {
  int total = G * O * 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    int k = i & 31, o = (i >> 5) % O, g = (i >> 5) / O;
    int b = opt_bit[(g / IR) * O + o];
    double y = 0.0;
    if (b >= 0) {
      int v = ins0(k, b);
      y = rt[g * 64 + v] / rt[g * 64 + (v | (1 << b))];
    }
    ylab[i] = y;
  }
}

// Mask ranking: keys = (sum correct << 32) | (2^32-1 - mask);
// each 1024-thread block bitonic-sorts up to 1024 keys in shared memory
// (descending) and keeps its first K.  Launched repeatedly (n -> n/1024*K)
// until one block remains.  Integer keys => exact and order-independent.
static __global__ void __launch_bounds__(1024) k_topk_keys(const unsigned long long* __restrict__ in, long long n,
                                                    unsigned long long* __restrict__ out, int K) {
  __shared__ unsigned long long sk[1024];
  const long long base = (long long)blockIdx.x * 1024;
  const int t = threadIdx.x;
  sk[t] = (base + t < n) ? in[base + t] : 0ull;
  __syncthreads();
  for (int size = 2; size <= 1024; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int p = t ^ stride;
      if (p > t) {
        const bool desc = (t & size) == 0;
        const unsigned long long a = sk[t], b = sk[p];
        if (desc ? (a < b) : (a > b)) {
          sk[t] = b;
          sk[p] = a;
        }
      }
      __syncthreads();
    }
  }
  if (t < K) out[(long long)blockIdx.x * K + t] = sk[t];
}

// keys -> mask ids (-1 for padding), first K of a descending-sorted list.
static __global__ void k_decode_top(const unsigned long long* __restrict__ keys, long long n, int64_t* __restrict__ ids,
                             int K) {
  for (int t = threadIdx.x; t < K; t += blockDim.x) {
    const unsigned long long k = t < n ? keys[t] : 0ull;
    ids[t] = k ? (int64_t)(0xFFFFFFFFull - (k & 0xFFFFFFFFull)) : (int64_t)-1;
  }
}

// Validation of the Tier-1 input: first offending flat index.
static __global__ void k_validate(const double* __restrict__ counters, const double* __restrict__ cycles,
                           const double* __restrict__ rt, long long n_slots, int C,
                           unsigned long long* __restrict__ bad) {
  long long total = n_slots * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    double c = counters[i];
    if (!(c >= 0.0) || !isfinite(c)) atomicMin(&bad[0], (unsigned long long)i);
    if (i < n_slots) {
      double cy = cycles[i], r = rt[i];
      if (!(cy > 0.0) || !isfinite(cy)) atomicMin(&bad[1], (unsigned long long)i);
      if (!(r > 0.0) || !isfinite(r)) atomicMin(&bad[2], (unsigned long long)i);
    }
  }
}

}  // namespace speedrec
