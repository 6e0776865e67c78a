/*
 * speedrec.h -- C-ABI of the B200-native Tier-2/Tier-3 hot path of
 * arXiv 1910.07776, "A Tool for Automatically Suggesting Source-Code
 * Optimizations for Complex GPU Kernels" (Taheri, Qasem, Burtscher).
 *
 * Citations: P:n = line n of the paper text, S:n = line n of
 * SPEC.md, "reading Rk/Dk" = DESIGN.md §3 (the interpretation adopted where
 * the paper is silent).  Library: paper_1910_07776_b200/libspeedrec.so.
 *
 * What the library computes (one call of sr_evaluate = the whole path for a
 * batch of scenarios, every step in CUDA kernels on the context's stream):
 *   A0  rates x = counters / cycles                    (Tier 1)
 *   A1  before/after pairs per optimization, label
 *       AC = rt_before / rt_after, split membership    (D2)
 *   A2  per-fit min-max feature scaling                (reading D3)
 *   A3  centred Gram / kernel matrix (FP64 DMMA)       (D1)
 *   A4  Cholesky + 2 iterative-refinement steps        (S:253 lambda=1e-8; D1)
 *   A5  predict EX, clamp EX<=0 to 0.01
 *   A6  rank by (EX desc, id asc), keep EX>=threshold,
 *       first max_count
 *   A7  per-(scenario, optimization) and per-scenario
 *       scores: sign accuracy, AC/EX, rec hits
 *
 * Conventions
 *   Errors: every function returns sr_status; no exception crosses the ABI.
 *     sr_last_error(ctx) returns one line "<CODE> <entity>: <text>" naming
 *     the offending slot / group / optimization.
 *   Ownership: input pointers are borrowed for the duration of the call and
 *     copied (host or device); all outputs are caller-allocated.  The context
 *     owns its device memory and its CUDA stream (unless one is passed in)
 *     and frees everything in sr_destroy.
 *   Threading: a context is not re-entrant; separate contexts are independent.
 *   Call order: sr_evaluate before sr_load_dataset and sr_define_scenarios
 *     returns SR_E_STATE.
 *   Determinism: outputs are a pure function of (dataset, scenarios, params,
 *     first, count), independent of launch configuration and GPU count
 *     (FP sums inside one (scenario, optimization) row use a fixed order).
 *   Limits: n_opt_bits == 6 (the paper's lattice), n_counters <= 128,
 *     n_opt_ids <= 16, max_count <= 8.  Up to 64 groups run on the warp path
 *     (all features); more groups on the large-batch path (config C4), which
 *     needs <= 8 scored optimizations and supports neither mask aggregation
 *     nor sr_sweep.  Learner SR_M5P runs on the warp path only, with <= 64
 *     counters.  Violations return SR_E_UNSUPPORTED.
 */
#ifndef SPEEDREC_H_
#define SPEEDREC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sr_ctx sr_ctx; /* opaque */

typedef enum {
  SR_OK = 0,
  SR_E_ARG = -1,         /* usage: NULL pointer, bad size or enum (SPEC exit 2) */
  SR_E_DATA = -2,        /* cycles<=0, runtime<=0, counter<0 or non-finite */
  SR_E_LATTICE = -3,     /* opt_bit / masks inconsistent with the 2^m lattice */
  SR_E_EMPTY = -4,       /* selector matches no group / slot */
  SR_E_STATE = -5,       /* call order */
  SR_E_OOM = -6,         /* device allocation failed */
  SR_E_CUDA = -7,        /* CUDA runtime error (message carries cudaGetErrorString) */
  SR_E_UNSUPPORTED = -8  /* outside the limits above, or learner not built yet */
} sr_status;

/* Create a context on CUDA device `cuda_device`.  cuda_stream: a cudaStream_t
 * to launch on (e.g. torch.cuda.current_stream().cuda_stream) or NULL for a
 * context-owned non-blocking stream. */
sr_status sr_create(int32_t cuda_device, void* cuda_stream, sr_ctx** out);
void sr_destroy(sr_ctx* ctx); /* NULL-safe; frees all device memory */
const char* sr_last_error(const sr_ctx* ctx); /* valid until the next call on ctx */
const char* sr_version(void);

/* ---------------------------------------------------------------------- */
/* Tier-1 input for a whole version lattice (Table 1-2).   */
/* Slot t = ((p*I + i)*R + r) * 2^m + v, v = version mask (bit j set =     */
/* the j-th optimization of program p applied).                            */
/* ---------------------------------------------------------------------- */
typedef struct {
  int32_t n_programs, n_inputs, n_runs; /* P, I, R: groups G = P*I*R */
  int32_t n_opt_bits;                   /* m, must be 6 */
  int32_t n_counters;                   /* C <= 128 */
  int32_t n_opt_ids;                    /* O <= 16: global optimization ids (alphabetical) */
  const double* counters;               /* [N][C] raw counts, >= 0, finite; N = G * 2^m */
  const double* cycles;                 /* [N] > 0 (the normaliser) */
  const double* runtime_ms;             /* [N] > 0 (labels, reading D2) */
  const int8_t* opt_bit;                /* [P][O] bit of optimization o in program p, -1 absent */
  int32_t on_device;                    /* 0: host pointers; 1: device pointers on the ctx device */
} sr_dataset;

/* Validate (host-side checks when on_device == 0; device-side reduction
 * otherwise) and copy into context memory.  Replaces any previous dataset.
 * Errors: SR_E_ARG, SR_E_DATA (names the first bad slot/counter),
 * SR_E_LATTICE (opt_bit out of range or duplicated within a program),
 * SR_E_UNSUPPORTED, SR_E_OOM, SR_E_CUDA. */
sr_status sr_load_dataset(sr_ctx* ctx, const sr_dataset* ds);

/* ---------------------------------------------------------------------- */
/* Scenario batch.  Scenario s = (feature-mask index f, split index k),   */
/* s = f * n_splits + k.  Slot membership per split (reading R17):         */
/*   GROUPS: slot t is train iff its group is in train_groups[k], test iff */
/*           its group is in test_groups[k] (both may hold, Exp 1 P:214);  */
/*   LOO:    the pool = slots of pool_groups in ascending order; split k   */
/*           holds out the k-th pool slot: train = pool minus it, test = it;*/
/*   RANDOM: train iff bit (t mod 64) of                                    */
/*           mix(mix(seed ^ mix(k)) + floor(t/64)) is 1, test otherwise,     */
/*           mix = SplitMix64 finalizer (incl. += 0x9E3779B97F4A7C15).       */
/* Scored optimizations O_s = split_opt_masks[k] (if non-NULL) else         */
/* opt_mask, restricted to ids < O (Exp 5/6: FTZ, RSQRT only).   */
/* Feature set F = all counters; or feature_masks[f] (2 words, <=128       */
/* counters); or, when all_subsets_k > 0, the bits of f over counters       */
/* [0, k) (n_masks = 2^k).  All pointers are HOST pointers, copied.         */
/* ---------------------------------------------------------------------- */
typedef enum { SR_SPLIT_GROUPS = 0, SR_SPLIT_LOO = 1, SR_SPLIT_RANDOM = 2 } sr_split_kind;

typedef struct {
  int32_t kind;                    /* sr_split_kind */
  int32_t group_words;             /* ceil(G/64) */
  int64_t n_splits;
  const uint64_t* train_groups;    /* GROUPS: [n_splits][group_words] */
  const uint64_t* test_groups;     /* GROUPS: [n_splits][group_words] */
  const uint32_t* split_opt_masks; /* GROUPS: [n_splits] or NULL */
  const uint64_t* pool_groups;     /* LOO: [group_words] */
  uint64_t seed;                   /* RANDOM */
  uint32_t opt_mask;               /* O_s when split_opt_masks == NULL */
  int32_t all_subsets_k;           /* 0 or 1..20 */
  int64_t n_masks;                 /* >= 1 */
  const uint64_t* feature_masks;   /* [n_masks][2] or NULL */
} sr_scenarios;

/* Copies the definition; *n_scenarios = n_splits * n_masks.
 * Errors: SR_E_STATE (no dataset), SR_E_ARG, SR_E_EMPTY (LOO pool empty,
 * split k >= pool size, GROUPS split with no test group), SR_E_UNSUPPORTED. */
sr_status sr_define_scenarios(sr_ctx* ctx, const sr_scenarios* sc, int64_t* n_scenarios);

/* ---------------------------------------------------------------------- */
/* Parameters (defaults from sr_default_params).                           */
/* ---------------------------------------------------------------------- */
typedef enum { SR_LINREG = 0, SR_IBK = 1, SR_M5P = 2 } sr_learner;

typedef struct {
  int32_t learner;       /* SR_LINREG (ridge LS, reading D1), SR_IBK (k-nearest neighbours,
                            P:147-149, reading R22; bit-exact, both the <= 64-group and the
                            large-batch path) or SR_M5P (model tree, readings M1-M6;
                            <= 64 groups and <= 64 counters, else SR_E_UNSUPPORTED) */
  int32_t max_count;     /* Tier-3 max recommendations, 3 */
  int32_t refine_steps;  /* iterative-refinement steps of the solve, 2 */
  int32_t debug_mcap;    /* 0 = auto; >0 caps the shared-memory Cholesky size so larger
                            systems take the global-scratch path (tests only) */
  double ridge;          /* lambda, 1e-8 */
  double threshold;      /* recommend iff EX >= threshold, 1.05 (reading R8) */
  double clamp_floor;    /* EX <= 0 -> clamp_floor, 0.01 */
  double guard_tol;      /* guard band for n_guard, 1e-9 (reading R21) */
  int32_t top_k;         /* masks kept by the mask ranking, 64, <= 512 */
  int32_t k_nn;          /* IBK neighbours k, 10 (P:149 IBk default reading R22), 1..16 */
} sr_params;

void sr_default_params(sr_params* out);

/* Per (scenario, optimization id) row (A7).  Rows for ids not in O_s are
 * all-zero.  min/max are 0 when n_test == 0.  fp_* = XOR over the pairs of
 * SplitMix64(pair id), pair id = (g*O + o)*32 + k, k = rank of the before
 * version among the 32 with bit b clear. */
typedef struct {
  int32_t n_train;   /* training pairs: both slots in train (A1) */
  int32_t n_test;    /* test cases: before slot in test */
  int32_t n_correct; /* (EX>1 && AC>1) || (EX<=1 && AC<=1) (R11) */
  int32_t n_clamped; /* EX <= 0 clamped */
  double sum_ratio;  /* sum of AC/EX */
  double min_ratio, max_ratio;
  uint64_t fp_train, fp_test;
} sr_opt_score;      /* 56 bytes */

/* Per scenario row (A6/A7). */
typedef struct {
  int32_t n_rec;       /* recommendations made over all test slots */
  int32_t n_rec_hit;   /* ... whose AC > 1 */
  int32_t n_untrained; /* test cases of scored optimizations with no training pair */
  int32_t n_guard;     /* decisions within guard_tol of a boundary (reading R21) */
} sr_scn_score;      /* 16 bytes */

/* Per feature mask, summed over all folds (splits) of the mask (A7, C5). */
typedef struct {
  int32_t n_correct, n_test, n_rec, n_rec_hit;
} sr_mask_score;     /* 16 bytes */

typedef struct {
  sr_opt_score* opt_scores; /* required: [count][O] */
  sr_scn_score* scn_scores; /* required: [count] */
  double* ex;               /* optional: [count][O][G*32] EX per (optimization, pair), 0 = not a predicted test case */
  int8_t* recs;             /* optional: [count][N][max_count] recommended ids per test slot, -1 padded */
  int64_t* totals;          /* optional: [4] pooled over the range (A7 "per config"):
                               sum n_correct, sum n_test, sum n_rec, sum n_rec_hit;
                               pooled sign accuracy = 100 * totals[0] / totals[1] (Table 3) */
  sr_mask_score* mask_scores; /* optional: [count / n_splits] per feature mask, summed over its folds */
  int64_t* top_masks;       /* optional: [params.top_k] mask ids ranked by (sum n_correct desc, id asc),
                               -1 padded.  Either of these two switches
                               the call to mask aggregation: first and count must then be multiples of
                               n_splits, and opt_scores / scn_scores may be NULL (not materialised). */
  int32_t on_device;        /* 0: host buffers (copied back, call is synchronous); 1: device buffers */
} sr_outputs;

/* Fused fit -> predict -> rank -> recommend -> score for scenarios
 * [first, first + count) -- the sharding unit of multi-GPU runs.
 * Host outputs: synchronous.  Device outputs: asynchronous on the context
 * stream (call sr_synchronize or sync the stream before reading).
 * Errors: SR_E_STATE, SR_E_ARG (range), SR_E_UNSUPPORTED, SR_E_OOM, SR_E_CUDA. */
sr_status sr_evaluate(sr_ctx* ctx, const sr_params* params, int64_t first, int64_t count,
                      sr_outputs* out);

/* Tier-3 rule sweep ("recommend the top choices
 * if their benefit is above a preset threshold ... the user can select how
 * many"): the fits of scenarios [first, first + count) run once (same
 * kernels and learner as sr_evaluate); then for every test version the
 * scored, trained candidates (R13) are ordered by (EX desc, id asc) (R10) and,
 * for each threshold thresholds[i] and list length max_counts[j], the first
 * min(#{EX >= thresholds[i]}, max_counts[j]) are recommended (R8, R9).
 *   thresholds  host [n_thr], strictly ascending, finite, 1 <= n_thr <= 256
 *   max_counts  host [n_cnt], each in [1, 16], 1 <= n_cnt <= 16
 *   out_rec, out_hit  host int64 [n_thr][n_cnt]: recommendations made, and
 *               those whose actual speedup AC > 1 (R11), summed over the range.
 * params->threshold / max_count are ignored.  Warp path only (<= 64 groups;
 * feature-mask batches run their masks on the warp path here).  Caller owns
 * every buffer.  Errors: SR_E_ARG, SR_E_STATE, SR_E_UNSUPPORTED (> 64
 * groups), and sr_evaluate's. */
sr_status sr_sweep(sr_ctx* ctx, const sr_params* params, int64_t first, int64_t count, int32_t n_thr,
                   const double* thresholds, int32_t n_cnt, const int32_t* max_counts, int64_t* out_rec,
                   int64_t* out_hit);

/* ---------------------------------------------------------------------- */
/* Tool path: one scenario, one user profile (SPEC train_all S:282,        */
/* predict_all S:291, rank_and_filter S:300; P:60-62 Tiers 2 and 3).        */
/* ---------------------------------------------------------------------- */

/* Fit the ridge model of every optimization id of one scenario (A1-A4, the
 * same kernels as sr_evaluate) and return it in raw-counter form:
 *   coef_out host [O][1 + C]: row o = (c0, u_0 .. u_{C-1}) with
 *   EX = c0 + sum_c u_c * x_c,  x_c = counters_c / cycles,
 * i.e. the scaled-feature model b + w.x' of reading D1/D3 with the scaling
 * folded in (u_c = w_c / rg_c for active c, 0 otherwise).  Rows of ids not
 * scored in the scenario, or untrained (n = 0, reading R18): c0 = NaN, u = 0.
 * Caller owns coef_out.  Errors: SR_E_ARG, SR_E_STATE, SR_E_UNSUPPORTED
 * (learner IBK: the model is its training set), and sr_evaluate's. */
sr_status sr_fit(sr_ctx* ctx, const sr_params* params, int64_t scenario, double* coef_out);

/* Tier 2 for one user profile (host, no context; O(O*C) work):
 *   ex_out[o] = c0 + sum_c u_c * (counters[c] / cycles), clamped to
 *   params->clamp_floor when <= 0; NaN for rows with c0 = NaN.
 * coef [n_opts][1 + n_counters] as written by sr_fit.  Borrowed pointers.
 * Errors: SR_E_ARG (null/size), SR_E_DATA (cycles <= 0, counter < 0 or
 * non-finite). */
sr_status sr_predict(const sr_params* params, const double* coef, int32_t n_opts, int32_t n_counters,
                     const double* counters, double cycles, double* ex_out);

/* Tier 3: candidates are ids with candidate[o] != 0 (all
 * when candidate is NULL) and a non-NaN EX >= params->threshold (R8); sorted
 * by (EX desc, id asc) (R10); the first params->max_count (1..64) go to
 * rec_out [max_count], -1 padded; *n_rec_out = their number.  An empty list is valid
 * (S:304).  Errors: SR_E_ARG. */
sr_status sr_recommend(const sr_params* params, const double* ex, const uint8_t* candidate, int32_t n_opts,
                       int8_t* rec_out, int32_t* n_rec_out);

/* A0 alone: rates x[N][C] (bit-exact IEEE FP64 division) into x_out
 * (host if on_device == 0).  For parity tests of Tier 1. */
sr_status sr_rates(sr_ctx* ctx, double* x_out, int32_t on_device);

sr_status sr_synchronize(sr_ctx* ctx);

/* Launch accounting / live timing of the last sr_evaluate.
 * sr_set_timing(ctx, 1) records a CUDA event pair on the context stream
 * around every kernel launch; sr_kernel_stats then reports, for up to
 * `cap` kernels, their names, launch counts and summed milliseconds.
 * Returns the number of distinct kernels (or < 0 on error). */
sr_status sr_set_timing(sr_ctx* ctx, int32_t enable);
int32_t sr_kernel_stats(sr_ctx* ctx, int32_t cap, const char** names, int32_t* launches,
                        double* ms);
sr_status sr_reset_kernel_stats(sr_ctx* ctx); /* zero the accumulated counts and times */
/* Kernels launched by the last sr_evaluate call. */
int32_t sr_last_launch_count(const sr_ctx* ctx);
/* Executed work of the last sr_evaluate with learner SR_M5P: the FP64
 * operations of every split search the grown trees ran (P:151 model-tree
 * induction, reading M1): per searched node and feature, m label additions of
 * the first pass for every candidate row, 3m more for every scored candidate
 * (+ 2m for a redone adjacent-double candidate).  0 for the other learners or
 * before any M5P evaluate; synchronizes the context stream; < 0 on error. */
int64_t sr_last_work(sr_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SPEEDREC_H_ */
