// speedrec.cu -- runtime + C-ABI of the B200-native Tier-2/Tier-3 path of
// arXiv 1910.07776.  The ABI is declared (with argument semantics, layout,
// ownership and errors) in include/speedrec.h.  Everything numerical runs in
// the kernels of kernels.cuh / eval_warp.cuh; this file validates arguments,
// owns device memory, plans the launch (shared-memory layout, occupancy) and
// accounts for launches and their live CUDA-event timing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <cstdlib>

#include "../../include/speedrec.h"
#include "eval_masks.cuh"
#include "eval_schur.cuh"
#include "eval_warp.cuh"
#include "fit_big.cuh"
#include "ibk_big.cuh"
#include "kernels.cuh"
#include "pred_rank.cuh"

using namespace speedrec;

static_assert(sizeof(sr_opt_score) == 56, "sr_opt_score layout");
static_assert(sizeof(OptScore) == sizeof(sr_opt_score), "OptScore layout");
static_assert(sizeof(ScnScore) == sizeof(sr_scn_score), "ScnScore layout");
static_assert(sizeof(MaskScore) == sizeof(sr_mask_score), "MaskScore layout");

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct KStat {
  const char* name;
  int launches = 0;
  double ms = 0.0;
};

}  // namespace

struct sr_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t cstream = nullptr;        // copy stream: D2H of finished chunks overlaps later ones
  cudaStream_t fstream[8] = {};          // side streams of a fork-join launch group (launch_group)
  cudaEvent_t fevent[9] = {};            // its fork / join events (no timing)
  std::vector<cudaEvent_t> cp_events;
  std::string err;
  int sm_count = 0;
  int max_smem_optin = 0;
  // dataset
  bool have_ds = false;
  int P = 0, I = 0, R = 0, m = 0, C = 0, O = 0, G = 0;
  long long N = 0;
  DevBuf counters, cycles, runtime, opt_bit, x, ylab, bad;
  std::vector<int8_t> h_opt_bit;
  // scenarios
  bool have_sc = false;
  sr_scenarios sc{};
  DevBuf train_g, test_g, split_om, pool_list, fmasks;
  std::vector<uint64_t> h_train, h_test, h_fmasks;
  std::vector<uint32_t> h_om;
  std::vector<int32_t> h_pool;
  int dmax = 0, np_tr = 0, np_te = 0, n_tg = 0, n_os = 0;
  // scratch + outputs
  DevBuf gscratch, out_opt, out_scn, out_ex, out_rec, out_tot, out_mask, out_top, keys_a, keys_b;
  DevBuf big_lists, big_y, big_U, big_c0, big_flag;  // large-batch path (> 64 groups)
  DevBuf ibk_lists, ibk_xs, ibk_meta;                // IBK on the large-batch path
  DevBuf fit_coef;              // sr_fit: [O][1 + C]
  // feature-mask path (eval_masks.cuh)
  DevBuf mp_G, mp_r, mp_z, mp_meta, mp_perm;
  long long sc_gen = 0, perm_key[3] = {-1, -1, -1};
  std::vector<int> perm_off;     // [kMaskMaxD + 2] start of each popcount group in mp_perm
  unsigned mask_or = 0;          // union of the call's masks (with the perm cache)
  // prefix-shared mask path (eval_schur.cuh): plan cached per (definition, range)
  DevBuf mp_rec, mp_order, mp_units, mp_pfx, mp_glist;
  std::vector<int> splan_goff;   // [kSchurU + 2] groups of each prefix popcount in mp_glist
  long long splan_key[4] = {-1, -1, -1, -1};
  int splan_groups = 0;
  std::vector<int> splan_doff;   // [kSchurU + 2] start of each suffix-size group in mp_order
  double* coef_req = nullptr;   // set by sr_fit for the duration of its evaluate
  const SweepArgs* sweep = nullptr;   // set by sr_sweep for the duration of its evaluate
  DevBuf sw_buf;
  DevBuf extab, trained, guard_acc, mask_acc, done;   // fit -> rank exchange (warp path)
  DevBuf utab;                                        // fit -> k_pred_rank model table (split LS path)
  DevBuf work;                                        // M5P executed split-search operations (sr_last_work)
  DevBuf qctr;                                        // k_fit_warp dynamic work-unit counter
  // accounting
  bool timing = false;
  std::vector<KStat> kstats;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  int last_launches = 0;
};

namespace {

sr_status fail(sr_ctx* c, sr_status st, const char* fmt, ...) {
  static const char* names[] = {"SR_OK", "SR_E_ARG", "SR_E_DATA", "SR_E_LATTICE", "SR_E_EMPTY",
                                "SR_E_STATE", "SR_E_OOM", "SR_E_CUDA", "SR_E_UNSUPPORTED"};
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = std::string(names[-(int)st]) + " " + buf;
  return st;
}

#define CU(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) return fail(c, SR_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

sr_status ensure(sr_ctx* c, DevBuf& b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return SR_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  if (bytes == 0) return SR_OK;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, SR_E_OOM, "device allocation of %zu bytes: %s", bytes, cudaGetErrorString(e));
  }
  b.bytes = bytes;
  return SR_OK;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

int kstat_id(sr_ctx* c, const char* name) {
  for (size_t i = 0; i < c->kstats.size(); ++i)
    if (c->kstats[i].name == name) return (int)i;
  c->kstats.push_back(KStat{name, 0, 0.0});
  return (int)c->kstats.size() - 1;
}

cudaEvent_t take_event(sr_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Bracket a launch with events when timing is on; count it always.
template <typename F>
sr_status launch(sr_ctx* c, const char* name, F&& f) {
  const int id = kstat_id(c, name);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    e0 = take_event(c);
    e1 = take_event(c);
    cudaEventRecord(e0, c->stream);
  }
  f();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, SR_E_CUDA, "launch of %s: %s", name, cudaGetErrorString(e));
  if (c->timing) {
    cudaEventRecord(e1, c->stream);
    c->pending.push_back({id, {e0, e1}});
  }
  c->kstats[id].launches++;
  c->last_launches++;
  return SR_OK;
}

// A group of independent launches of one kernel family (disjoint outputs)
// spread over up to 8 side streams forked from and joined back into the
// context stream, so one launch's tail wave overlaps the next launch's first
// (DESIGN.md §5.8).  f(i, stream) issues launch i.  Timing (when on): one
// event pair on the context stream around the whole group, charged to `name`
// with n launches, so the family's summed time is the group's wall time.
// SPEEDREC_GROUP_STREAMS=1 keeps the launches on the context stream.
template <typename F>
sr_status launch_group(sr_ctx* c, const char* name, int n, F&& f) {
  if (n <= 0) return SR_OK;
  static const int env_k = [] {
    const char* e = getenv("SPEEDREC_GROUP_STREAMS");
    return e ? atoi(e) : 8;
  }();
  const int k = std::max(1, std::min(std::min(env_k, 8), n));
  const int id = kstat_id(c, name);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    e0 = take_event(c);
    e1 = take_event(c);
    cudaEventRecord(e0, c->stream);
  }
  if (k == 1) {
    for (int i = 0; i < n; ++i) {
      const cudaError_t ce = f(i, c->stream);
      if (ce != cudaSuccess) return fail(c, SR_E_CUDA, "launch of %s: %s", name, cudaGetErrorString(ce));
    }
  } else {
    for (int q = 0; q < k; ++q)
      if (!c->fstream[q]) CU(cudaStreamCreateWithFlags(&c->fstream[q], cudaStreamNonBlocking));
    for (int q = 0; q <= k; ++q)
      if (!c->fevent[q]) CU(cudaEventCreateWithFlags(&c->fevent[q], cudaEventDisableTiming));
    CU(cudaEventRecord(c->fevent[k], c->stream));                     // fork
    for (int q = 0; q < k; ++q) CU(cudaStreamWaitEvent(c->fstream[q], c->fevent[k], 0));
    cudaError_t first_err = cudaSuccess;
    for (int i = 0; i < n && first_err == cudaSuccess; ++i) first_err = f(i, c->fstream[i % k]);
    for (int q = 0; q < k; ++q) {                                      // join (also after a failed launch)
      CU(cudaEventRecord(c->fevent[q], c->fstream[q]));
      CU(cudaStreamWaitEvent(c->stream, c->fevent[q], 0));
    }
    if (first_err != cudaSuccess) return fail(c, SR_E_CUDA, "launch of %s: %s", name, cudaGetErrorString(first_err));
  }
  if (c->timing) {
    cudaEventRecord(e1, c->stream);
    c->pending.push_back({id, {e0, e1}});
  }
  c->kstats[id].launches += n;
  c->last_launches += n;
  return SR_OK;
}

void collect_timing(sr_ctx* c) {
  for (auto& pe : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(pe.second.second);
    cudaEventElapsedTime(&ms, pe.second.first, pe.second.second);
    c->kstats[pe.first].ms += ms;
    c->ev_pool.push_back(pe.second.first);
    c->ev_pool.push_back(pe.second.second);
  }
  c->pending.clear();
}

int grid_for(const sr_ctx* c, long long work, int block) {
  long long g = (work + block - 1) / block;
  long long cap = (long long)c->sm_count * 8;
  return (int)std::max(1LL, std::min(g, cap));
}

int align16(int x) { return (x + 15) & ~15; }

ScenDesc scen_desc(const sr_ctx* c) {
  ScenDesc D{};
  D.kind = c->sc.kind;
  D.gw = (c->G + 63) / 64;
  D.n_splits = c->sc.n_splits;
  D.train_g = (const uint64_t*)c->train_g.p;
  D.test_g = (const uint64_t*)c->test_g.p;
  D.split_om = c->sc.split_opt_masks ? (const uint32_t*)c->split_om.p : nullptr;
  D.pool_list = (const int32_t*)c->pool_list.p;
  D.n_pool = (int)c->h_pool.size();
  D.seed = c->sc.seed;
  D.opt_mask = c->sc.opt_mask;
  D.subsets_k = c->sc.all_subsets_k;
  D.n_masks = c->sc.n_masks;
  D.fmasks = (c->sc.feature_masks && c->sc.all_subsets_k == 0) ? (const uint64_t*)c->fmasks.p : nullptr;
  return D;
}

}  // namespace

extern "C" {

const char* sr_version(void) { return "speedrec 0.1 (sm_100a)"; }

sr_status sr_create(int32_t cuda_device, void* cuda_stream, sr_ctx** out) {
  if (!out) return SR_E_ARG;
  *out = nullptr;
  sr_ctx* c = new sr_ctx();
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || cuda_device < 0 || cuda_device >= n) {
    cudaGetLastError();
    delete c;
    return SR_E_CUDA;
  }
  c->device = cuda_device;
  cudaSetDevice(cuda_device);
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, cuda_device);
  cudaDeviceGetAttribute(&c->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cuda_device);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cuda_device);
  if (major != 10) {
    delete c;
    return SR_E_UNSUPPORTED;
  }
  if (cuda_stream) {
    c->stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return SR_E_CUDA;
    }
    c->own_stream = true;
  }
  *out = c;
  return SR_OK;
}

void sr_destroy(sr_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  collect_timing(c);
  for (DevBuf* b : {&c->counters, &c->cycles, &c->runtime, &c->opt_bit, &c->x, &c->ylab, &c->bad,
                    &c->train_g, &c->test_g, &c->split_om, &c->pool_list, &c->fmasks, &c->gscratch,
                    &c->out_opt, &c->out_scn, &c->out_ex, &c->out_rec, &c->out_tot, &c->out_mask,
                    &c->out_top, &c->keys_a, &c->keys_b, &c->big_lists, &c->big_y, &c->big_U, &c->big_c0,
                    &c->big_flag, &c->extab, &c->trained, &c->guard_acc, &c->mask_acc, &c->done, &c->fit_coef,
                    &c->mp_G, &c->mp_r, &c->mp_z, &c->mp_meta, &c->mp_perm, &c->mp_rec, &c->mp_order,
                    &c->mp_units, &c->mp_pfx, &c->mp_glist, &c->sw_buf, &c->ibk_lists, &c->ibk_xs, &c->ibk_meta,
                    &c->utab, &c->work, &c->qctr})
    release(*b);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->cp_events) cudaEventDestroy(e);
  if (c->cstream) {
    cudaStreamSynchronize(c->cstream);
    cudaStreamDestroy(c->cstream);
  }
  for (cudaStream_t fs : c->fstream)
    if (fs) {
      cudaStreamSynchronize(fs);
      cudaStreamDestroy(fs);
    }
  for (cudaEvent_t e : c->fevent)
    if (e) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* sr_last_error(const sr_ctx* c) { return c ? c->err.c_str() : "SR_E_ARG null context"; }

void sr_default_params(sr_params* p) {
  if (!p) return;
  p->learner = SR_LINREG;
  p->max_count = 3;
  p->refine_steps = 2;
  p->debug_mcap = 0;
  p->ridge = 1e-8;
  p->threshold = 1.05;
  p->clamp_floor = 0.01;
  p->guard_tol = 1e-9;
  p->top_k = 64;
  p->k_nn = 10;
}

sr_status sr_load_dataset(sr_ctx* c, const sr_dataset* d) {
  if (!c) return SR_E_ARG;
  c->err.clear();
  if (!d || !d->counters || !d->cycles || !d->runtime_ms || !d->opt_bit)
    return fail(c, SR_E_ARG, "dataset: null pointer");
  if (d->n_programs <= 0 || d->n_inputs <= 0 || d->n_runs <= 0 || d->n_counters <= 0 || d->n_opt_ids <= 0)
    return fail(c, SR_E_ARG, "dataset: non-positive size (P=%d I=%d R=%d C=%d O=%d)", d->n_programs,
                d->n_inputs, d->n_runs, d->n_counters, d->n_opt_ids);
  if (d->n_opt_bits != 6) return fail(c, SR_E_UNSUPPORTED, "dataset: n_opt_bits=%d (only 6)", d->n_opt_bits);
  if (d->n_counters > kMaxCounters) return fail(c, SR_E_UNSUPPORTED, "dataset: n_counters=%d > 128", d->n_counters);
  if (d->n_opt_ids > kMaxOpt) return fail(c, SR_E_UNSUPPORTED, "dataset: n_opt_ids=%d > 16", d->n_opt_ids);
  cudaSetDevice(c->device);
  // the device copies are overwritten below: the old dataset (and the scenario
  // batch defined on it) stop being valid now, whatever the outcome
  c->have_ds = false;
  c->have_sc = false;
  const long long G = (long long)d->n_programs * d->n_inputs * d->n_runs;
  const long long N = G * 64;
  const int C = d->n_counters, O = d->n_opt_ids, P = d->n_programs;
  sr_status st;
  if ((st = ensure(c, c->counters, N * C * 8)) || (st = ensure(c, c->cycles, N * 8)) ||
      (st = ensure(c, c->runtime, N * 8)) || (st = ensure(c, c->opt_bit, (size_t)P * O)) ||
      (st = ensure(c, c->x, N * C * 8)) || (st = ensure(c, c->ylab, G * O * 32 * 8)) ||
      (st = ensure(c, c->bad, 3 * 8)))
    return st;
  // opt_bit is small: validate on host (copy first when it lives on device)
  c->h_opt_bit.assign((size_t)P * O, 0);
  cudaMemcpyKind k = d->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CU(cudaMemcpyAsync(c->counters.p, d->counters, N * C * 8, k, c->stream));
  CU(cudaMemcpyAsync(c->cycles.p, d->cycles, N * 8, k, c->stream));
  CU(cudaMemcpyAsync(c->runtime.p, d->runtime_ms, N * 8, k, c->stream));
  CU(cudaMemcpyAsync(c->h_opt_bit.data(), d->opt_bit, (size_t)P * O,
                     d->on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (int p = 0; p < P; ++p) {
    unsigned seen = 0;
    for (int o = 0; o < O; ++o) {
      int b = c->h_opt_bit[(size_t)p * O + o];
      if (b < -1 || b >= 6) return fail(c, SR_E_LATTICE, "program %d optimization %d: bit %d out of range", p, o, b);
      if (b >= 0) {
        if (seen & (1u << b)) return fail(c, SR_E_LATTICE, "program %d: bit %d used by two optimizations", p, b);
        seen |= 1u << b;
      }
    }
  }
  CU(cudaMemcpyAsync(c->opt_bit.p, c->h_opt_bit.data(), (size_t)P * O, cudaMemcpyHostToDevice, c->stream));
  unsigned long long init[3] = {~0ull, ~0ull, ~0ull};
  CU(cudaMemcpyAsync(c->bad.p, init, sizeof init, cudaMemcpyHostToDevice, c->stream));
  c->have_ds = false;
  c->last_launches = 0;
  sr_status ls = launch(c, "k_validate", [&] {
    k_validate<<<grid_for(c, N * C, 256), 256, 0, c->stream>>>(
        (const double*)c->counters.p, (const double*)c->cycles.p, (const double*)c->runtime.p, N, C,
        (unsigned long long*)c->bad.p);
  });
  if (ls) return ls;
  unsigned long long bad[3];
  CU(cudaMemcpyAsync(bad, c->bad.p, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  collect_timing(c);
  if (bad[0] != ~0ull)
    return fail(c, SR_E_DATA, "slot %llu counter %llu: negative or non-finite count", bad[0] / C, bad[0] % C);
  if (bad[1] != ~0ull) return fail(c, SR_E_DATA, "slot %llu: cycles must be > 0 and finite", bad[1]);
  if (bad[2] != ~0ull) return fail(c, SR_E_DATA, "slot %llu: runtime_ms must be > 0 and finite", bad[2]);
  c->P = P;
  c->I = d->n_inputs;
  c->R = d->n_runs;
  c->m = 6;
  c->C = C;
  c->O = O;
  c->G = (int)G;
  c->N = N;
  c->have_ds = true;
  c->have_sc = false;
  return SR_OK;
}

sr_status sr_define_scenarios(sr_ctx* c, const sr_scenarios* s, int64_t* n_scenarios) {
  if (!c) return SR_E_ARG;
  c->err.clear();
  if (!c->have_ds) return fail(c, SR_E_STATE, "define_scenarios: no dataset loaded");
  if (!s || !n_scenarios) return fail(c, SR_E_ARG, "define_scenarios: null pointer");
  const int G = c->G, gw = (G + 63) / 64;
  if (s->kind < 0 || s->kind > 2) return fail(c, SR_E_ARG, "scenarios: kind %d", s->kind);
  if (s->n_splits <= 0 || s->n_masks <= 0) return fail(c, SR_E_ARG, "scenarios: n_splits/n_masks must be > 0");
  if (s->group_words != gw) return fail(c, SR_E_ARG, "scenarios: group_words=%d, expected %d", s->group_words, gw);
  if (G > kMaxGroupsBig) return fail(c, SR_E_UNSUPPORTED, "scenarios: %d groups > %d", G, kMaxGroupsBig);
  if (s->all_subsets_k < 0 || s->all_subsets_k > 20 || s->all_subsets_k > c->C)
    return fail(c, SR_E_ARG, "scenarios: all_subsets_k=%d", s->all_subsets_k);
  if (s->all_subsets_k > 0 && s->n_masks != (1LL << s->all_subsets_k))
    return fail(c, SR_E_ARG, "scenarios: n_masks must be 2^all_subsets_k");
  if (s->all_subsets_k == 0 && s->n_masks > 1 && !s->feature_masks)
    return fail(c, SR_E_ARG, "scenarios: n_masks > 1 needs feature_masks");
  const uint32_t valid_ids = (c->O >= 32) ? ~0u : ((1u << c->O) - 1u);
  cudaSetDevice(c->device);
  sr_status st;
  // from here on the previous definition is being overwritten: it stops being
  // valid now, so a failure below leaves no half-updated batch behind
  c->have_sc = false;
  ++c->sc_gen;
  c->sc = *s;
  int np_tr = 0, np_te = 0, n_tg = 0, n_os = 0;
  if (s->kind == SR_SPLIT_GROUPS) {
    if (!s->train_groups || !s->test_groups) return fail(c, SR_E_ARG, "scenarios: GROUPS needs train/test group sets");
    const size_t nw = (size_t)s->n_splits * gw;
    c->h_train.assign(s->train_groups, s->train_groups + nw);
    c->h_test.assign(s->test_groups, s->test_groups + nw);
    for (long long k = 0; k < s->n_splits; ++k) {
      int a = 0, b = 0;
      for (int w = 0; w < gw; ++w) {
        uint64_t lim = (w == gw - 1 && G % 64) ? ((1ull << (G % 64)) - 1) : ~0ull;
        if ((c->h_train[k * gw + w] & ~lim) || (c->h_test[k * gw + w] & ~lim))
          return fail(c, SR_E_ARG, "split %lld: group bit beyond G=%d", k, G);
        a += __builtin_popcountll(c->h_train[k * gw + w]);
        b += __builtin_popcountll(c->h_test[k * gw + w]);
      }
      if (b == 0) return fail(c, SR_E_EMPTY, "split %lld: no test group", k);
      np_tr = std::max(np_tr, 32 * a);
      np_te = std::max(np_te, 32 * b);
      n_tg = std::max(n_tg, b);
    }
    if ((st = ensure(c, c->train_g, nw * 8)) || (st = ensure(c, c->test_g, nw * 8))) return st;
    CU(cudaMemcpyAsync(c->train_g.p, c->h_train.data(), nw * 8, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->test_g.p, c->h_test.data(), nw * 8, cudaMemcpyHostToDevice, c->stream));
  } else if (s->kind == SR_SPLIT_LOO) {
    if (!s->pool_groups) return fail(c, SR_E_ARG, "scenarios: LOO needs pool_groups");
    c->h_pool.clear();
    for (int g = 0; g < G; ++g)
      if ((s->pool_groups[g >> 6] >> (g & 63)) & 1ull) c->h_pool.push_back(g);
    if (c->h_pool.empty()) return fail(c, SR_E_EMPTY, "scenarios: LOO pool is empty");
    if (s->n_splits > (long long)c->h_pool.size() * 64)
      return fail(c, SR_E_EMPTY, "scenarios: split %lld beyond the %zu pool slots", (long long)s->n_splits - 1,
                  c->h_pool.size() * 64);
    np_tr = 32 * (int)c->h_pool.size();
    np_te = 32;
    n_tg = 1;
    if ((st = ensure(c, c->pool_list, c->h_pool.size() * 4))) return st;
    CU(cudaMemcpyAsync(c->pool_list.p, c->h_pool.data(), c->h_pool.size() * 4, cudaMemcpyHostToDevice, c->stream));
  } else {
    np_tr = np_te = 32 * G;
    n_tg = G;
  }
  if (s->split_opt_masks) {
    if (s->kind != SR_SPLIT_GROUPS) return fail(c, SR_E_ARG, "scenarios: split_opt_masks only for GROUPS");
    c->h_om.assign(s->split_opt_masks, s->split_opt_masks + s->n_splits);
    for (uint32_t mk : c->h_om) n_os = std::max(n_os, __builtin_popcount(mk & valid_ids));
    if ((st = ensure(c, c->split_om, c->h_om.size() * 4))) return st;
    CU(cudaMemcpyAsync(c->split_om.p, c->h_om.data(), c->h_om.size() * 4, cudaMemcpyHostToDevice, c->stream));
  } else {
    n_os = __builtin_popcount(s->opt_mask & valid_ids);
  }
  int dmax = c->C;
  if (s->all_subsets_k > 0) {
    dmax = s->all_subsets_k;
  } else if (s->feature_masks) {
    c->h_fmasks.assign(s->feature_masks, s->feature_masks + 2 * s->n_masks);
    dmax = 0;
    for (long long f = 0; f < s->n_masks; ++f) {
      uint64_t m0 = c->h_fmasks[2 * f], m1 = c->h_fmasks[2 * f + 1];
      if (c->C < 64) m0 &= (1ull << c->C) - 1;
      if (c->C <= 64) m1 = 0;
      else if (c->C < 128) m1 &= (1ull << (c->C - 64)) - 1;
      dmax = std::max(dmax, __builtin_popcountll(m0) + __builtin_popcountll(m1));
    }
    if ((st = ensure(c, c->fmasks, c->h_fmasks.size() * 8))) return st;
    CU(cudaMemcpyAsync(c->fmasks.p, c->h_fmasks.data(), c->h_fmasks.size() * 8, cudaMemcpyHostToDevice, c->stream));
  }
  CU(cudaStreamSynchronize(c->stream));
  c->dmax = std::max(dmax, 1);
  c->np_tr = std::max(np_tr, 32);
  c->np_te = std::max(np_te, 32);
  c->n_tg = std::max(n_tg, 1);
  c->n_os = std::max(n_os, 1);
  c->have_sc = true;
  ++c->sc_gen;
  *n_scenarios = s->n_splits * s->n_masks;
  return SR_OK;
}

namespace {

// Shared-memory plan of k_eval_warp for the current batch.
// lean (k_fit_warp MODE 4): no test lists (prediction is k_pred_rank's) and the
// raw-counter weights alias the factor buffer (free once the fit is solved).
WarpLayout plan_layout(const sr_ctx* c, int mcap, bool ibk, bool lean = false) {
  WarpLayout L{};
  int off = 0;
  auto take = [&](int bytes) {
    int o = off;
    off = align16(off + bytes);
    return o;
  };
  const int G = c->G, d = c->dmax, vmax = std::max(c->np_tr, d);
  const int dpad = std::max(d, 32) + 4;  // zero-padded for the fast-path fragment loads
  L.off_trw = take(8 * G);
  L.off_tew = take(8 * G);
  L.off_F = take(2 * d);
  L.np_tr = c->np_tr;
  L.np_te = c->np_te;
  L.off_trs = take(4 * c->np_tr);
  L.off_yc = take(8 * c->np_tr);
  L.off_tes = lean ? 0 : take(4 * c->np_te);
  L.off_tek = lean ? 0 : take(4 * c->np_te);
  L.off_col = take(2 * dpad);
  L.off_xb = take(8 * dpad);
  L.off_s = take(8 * dpad);
  L.off_w = take(8 * d);
  L.off_u = take(8 * d);
  L.vmax = vmax;
  L.off_v2 = take(8 * vmax);
  L.mcap = mcap;
  // Cholesky factor, or for IBK the kKnnRows scaled training rows being scanned
  L.off_M = take(8 * std::max({rb2(mcap), mcap * (mcap + 1) / 2, ibk ? kKnnRows * d : 0}));
  L.off_ufull = lean && rb2(mcap) >= c->C ? L.off_M : take(8 * c->C);
  L.bytes = align16(off);
  return L;
}

// Prefix-shared mask path (eval_schur.cuh): masks sorted by
// (suffix popcount, prefix, suffix); one Schur record per (prefix, fold, opt)
// from k_mask_sprep; one k_mask_sfit<D> launch per suffix size D, folds split
// over threads (integer atomics) when a launch has too few masks to fill the GPU.
sr_status run_schur_path(sr_ctx* c, const MaskArgs& M, long long S, int T, int U, long long mask0, long long nm) {
  sr_status st;
  const int O = c->O;
  const uint32_t pmask = (1u << T) - 1u, smask = (1u << U) - 1u;
  if (c->splan_key[0] != c->sc_gen || c->splan_key[1] != mask0 || c->splan_key[2] != nm ||
      c->splan_key[3] != (T << 8 | U)) {
    std::vector<uint32_t> bits(nm);
    for (long long i = 0; i < nm; ++i) {
      const long long f = mask0 + i;
      bits[i] = c->sc.all_subsets_k > 0 ? (uint32_t)f : (uint32_t)c->h_fmasks[2 * f];
    }
    auto key = [&](int32_t i) {
      const uint32_t b = bits[i], sfx = (b >> T) & smask;
      return ((uint64_t)__builtin_popcount(sfx) << 56) | ((uint64_t)(b & pmask) << 24) | sfx;
    };
    std::vector<int32_t> order(nm), group(nm);
    for (long long i = 0; i < nm; ++i) order[i] = (int32_t)i;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return key(a) < key(b); });
    // prefix groups: dense ids in prefix order
    std::vector<uint32_t> pfx;
    for (long long i = 0; i < nm; ++i) pfx.push_back(bits[i] & pmask);
    std::sort(pfx.begin(), pfx.end());
    pfx.erase(std::unique(pfx.begin(), pfx.end()), pfx.end());
    for (long long i = 0; i < nm; ++i)
      group[i] = (int32_t)(std::lower_bound(pfx.begin(), pfx.end(), bits[order[i]] & pmask) - pfx.begin());
    c->splan_doff.assign(kSchurU + 2, 0);
    for (long long i = 0; i < nm; ++i) ++c->splan_doff[__builtin_popcount((bits[i] >> T) & smask) + 1];
    for (int d = 0; d <= kSchurU; ++d) c->splan_doff[d + 1] += c->splan_doff[d];
    if ((st = ensure(c, c->mp_order, (size_t)nm * 4)) || (st = ensure(c, c->mp_units, (size_t)nm * 4)) ||
        (st = ensure(c, c->mp_pfx, pfx.size() * 4)))
      return st;
    CU(cudaMemcpyAsync(c->mp_order.p, order.data(), (size_t)nm * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->mp_units.p, group.data(), (size_t)nm * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->mp_pfx.p, pfx.data(), pfx.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));   // host vectors go out of scope
    c->splan_groups = (int)pfx.size();
    // groups by prefix popcount (k_mask_sprep_p<P> launches)
    {
      std::vector<int32_t> gl;
      c->splan_goff.assign(kSchurU + 2, 0);
      for (int pp = 0; pp <= kSchurU; ++pp) {
        c->splan_goff[pp] = (int)gl.size();
        for (size_t j = 0; j < pfx.size(); ++j)
          if (__builtin_popcount(pfx[j]) == pp) gl.push_back((int32_t)j);
      }
      c->splan_goff[kSchurU + 1] = (int)gl.size();
      if ((st = ensure(c, c->mp_glist, std::max<size_t>(gl.size(), 1) * 4))) return st;
      CU(cudaMemcpyAsync(c->mp_glist.p, gl.data(), gl.size() * 4, cudaMemcpyHostToDevice, c->stream));
      CU(cudaStreamSynchronize(c->stream));
    }
    c->splan_key[0] = c->sc_gen;
    c->splan_key[1] = mask0;
    c->splan_key[2] = nm;
    c->splan_key[3] = T << 8 | U;
  }
  const long long nrec = (long long)c->splan_groups * S * O;
  if ((st = ensure(c, c->mp_rec, (size_t)nrec * kRec * 8))) return st;
  SchurArgs SA{};
  SA.M = M;
  SA.T = T;
  SA.U = U;
  SA.pfx = (const uint32_t*)c->mp_pfx.p;
  SA.n_groups = c->splan_groups;
  SA.rec = (double*)c->mp_rec.p;
  SA.order = (const int32_t*)c->mp_order.p;
  SA.group = (const int32_t*)c->mp_units.p;
  if (T <= kSchurU && (int)c->splan_goff.size() == kSchurU + 2 &&
      c->splan_goff[kSchurU + 1] == c->splan_groups) {   // register records per prefix size
    std::vector<int> pps;                    // prefix sizes present (independent record groups)
    for (int pp = 0; pp <= kSchurU; ++pp)
      if (c->splan_goff[pp + 1] > c->splan_goff[pp]) pps.push_back(pp);
    if ((st = launch_group(c, "k_mask_sprep", (int)pps.size(), [&](int i, cudaStream_t stg) {
          const int pp = pps[i], g0 = c->splan_goff[pp], ng = c->splan_goff[pp + 1] - g0;
          const long long nth = (long long)ng * S * O;
          return mask_sprep_launch(pp, (unsigned)((nth + 127) / 128), stg, SA, (const int32_t*)c->mp_glist.p + g0, ng);
        })))
      return st;
  } else if ((st = launch(c, "k_mask_sprep",
                          [&] { k_mask_sprep<<<(unsigned)((nrec + 127) / 128), 128, 0, c->stream>>>(SA); }))) {
    return st;
  }
  // suffix sizes present, the largest launches first (the smaller ones fill
  // the tail waves of the large ones on the other side streams)
  std::vector<int> ds;
  for (int d = 0; d <= kSchurU; ++d)
    if (c->splan_doff[d + 1] > c->splan_doff[d]) ds.push_back(d);
  std::stable_sort(ds.begin(), ds.end(), [&](int a, int b) {
    return c->splan_doff[a + 1] - c->splan_doff[a] > c->splan_doff[b + 1] - c->splan_doff[b];
  });
  return launch_group(c, "k_mask_sfit", (int)ds.size(), [&](int i, cudaStream_t stg) {
    const int d = ds[i], off = c->splan_doff[d], n_it = c->splan_doff[d + 1] - off;
    const long long want = (long long)c->sm_count * 1024;
    const int fc = (int)std::max(1LL, std::min<long long>(S, want / n_it));
    const unsigned grid = (unsigned)(((long long)n_it * fc + kSfitThreads - 1) / kSfitThreads);
    return mask_sfit_launch(d, grid, stg, SA, off, n_it, fc);
  });
}

// Feature-mask path: LOO batches of whole feature masks
// (config C5).  Sets *used = false, with no side effects on the outputs,
// when the batch is outside its regime; the warp path then runs.
sr_status run_mask_path(sr_ctx* c, const sr_params* prm, long long first, long long count, const EvalArgs& A,
                        bool* used) {
  *used = false;
  const long long S = c->sc.n_splits;
  const int O = c->O, C = c->C;
  if (const char* e = getenv("SPEEDREC_MASK_PATH"))
    if (atoi(e) == 0) return SR_OK;
  if (c->sweep) return SR_OK;   // sr_sweep ranks on the warp path
  if (c->coef_req) return SR_OK;   // sr_fit needs the coefficient store of k_fit_warp<.,2>
  if (c->sc.kind != SR_SPLIT_LOO || C > kMaskMaxC || O > kMaskMaxO || prm->learner != SR_LINREG ||
      prm->debug_mcap > 0 || count <= 0 || first % S || count % S || c->sc.n_masks < 2)
    return SR_OK;
  const long long mask0 = first / S, nm = count / S;
  if (nm > INT32_MAX) return SR_OK;
  sr_status st;
  // popcount groups of the call's masks (cached per scenario definition and range)
  if (c->perm_key[0] != c->sc_gen || c->perm_key[1] != mask0 || c->perm_key[2] != nm) {
    std::vector<int> pc(nm);
    unsigned mor = 0;
    for (long long i = 0; i < nm; ++i) {
      const long long f = mask0 + i;
      int d;
      if (c->sc.all_subsets_k > 0) {
        d = __builtin_popcountll((unsigned long long)f);
        mor |= (unsigned)f;
      } else if (c->sc.feature_masks) {
        if (c->h_fmasks[2 * f + 1] != 0ull) return SR_OK;
        const unsigned long long mm = c->h_fmasks[2 * f] & (C >= 64 ? ~0ull : ((1ull << C) - 1ull));
        d = __builtin_popcountll(mm);
        mor |= (unsigned)mm;
      } else {
        d = C;
        mor |= C >= 32 ? 0xFFFFFFFFu : ((1u << C) - 1u);
      }
      if (d > kMaskMaxD) return SR_OK;
      pc[i] = d;
    }
    std::vector<int> off(kMaskMaxD + 2, 0), perm(nm);
    for (long long i = 0; i < nm; ++i) ++off[pc[i] + 1];
    for (int d = 0; d <= kMaskMaxD; ++d) off[d + 1] += off[d];
    std::vector<int> pos(off.begin(), off.end() - 1);
    for (long long i = 0; i < nm; ++i) perm[pos[pc[i]]++] = (int)i;
    if ((st = ensure(c, c->mp_perm, (size_t)nm * 4))) return st;
    CU(cudaMemcpyAsync(c->mp_perm.p, perm.data(), (size_t)nm * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));   // perm is a stack vector
    c->perm_off = off;
    c->mask_or = mor;
    c->perm_key[0] = c->sc_gen;
    c->perm_key[1] = mask0;
    c->perm_key[2] = nm;
  }
  int dmax = 0;
  for (int d = 0; d <= kMaskMaxD; ++d)
    if (c->perm_off[d + 1] > c->perm_off[d]) dmax = d;
  const long long items = S * O;
  if ((st = ensure(c, c->mp_G, (size_t)items * C * C * 8)) || (st = ensure(c, c->mp_r, (size_t)items * C * 8)) ||
      (st = ensure(c, c->mp_z, (size_t)items * C * 8)) || (st = ensure(c, c->mp_meta, (size_t)items * sizeof(PrepMeta))))
    return st;
  MaskArgs M{};
  M.sd = A.sd;
  M.x = A.x;
  M.ylab = A.ylab;
  M.opt_bit = A.opt_bit;
  M.P = c->P;
  M.IR = c->I * c->R;
  M.C = C;
  M.O = O;
  M.G = c->G;
  M.lambda = prm->ridge;
  M.threshold = prm->threshold;
  M.clamp_floor = prm->clamp_floor;
  M.guard_tol = prm->guard_tol;
  M.max_count = prm->max_count;
  M.first = first;
  M.mask0 = mask0;
  M.pG = (double*)c->mp_G.p;
  M.pr = (double*)c->mp_r.p;
  M.pz = (double*)c->mp_z.p;
  M.pm = (PrepMeta*)c->mp_meta.p;
  M.np_tr = c->np_tr;
  const int prep_smem = 4 * c->np_tr * 12;
  if (prep_smem > 48 * 1024) CU(cudaFuncSetAttribute(k_mask_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, prep_smem));
  if ((st = launch(c, "k_mask_prep", [&] {
         k_mask_prep<<<(unsigned)((items + 3) / 4), 128, prep_smem, c->stream>>>(M);
       })))
    return st;
  // regime check (one small read-back): every fit primal without refinement
  // under the warp path's rule: n <= 64 and n - 1 >= 2 d
  std::vector<PrepMeta> pm(items);
  CU(cudaMemcpyAsync(pm.data(), M.pm, items * sizeof(PrepMeta), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (const PrepMeta& q : pm)
    if (q.n > 0 && (q.n > 64 || q.n - 1 < 2 * dmax || q.nt > 1)) return SR_OK;
  M.opt_out = A.opt_out;
  M.scn_out = A.scn_out;
  M.ex_out = A.ex_out;
  M.rec_out = A.rec_out;
  M.totals = A.totals;
  M.mask_acc = A.agg ? A.mask_acc : nullptr;
  // prefix-shared path unless SPEEDREC_MASK_PATH=1 asks for k_mask_fit
  int mode = 2;
  if (const char* e = getenv("SPEEDREC_MASK_PATH")) mode = atoi(e);
  const int K = c->mask_or ? 32 - __builtin_clz(c->mask_or) : 0;
  const int U = std::min(kSchurU, K), T = K - U;
  if (mode == 2 && T <= kSchurT && K <= C && O <= kSfitMaxO) {
    if ((st = run_schur_path(c, M, S, T, U, mask0, nm))) return st;
    *used = true;
    return SR_OK;
  }
  for (int d = 0; d <= kMaskMaxD; ++d) {
    const int n_it = c->perm_off[d + 1] - c->perm_off[d];
    if (n_it == 0) continue;
    M.perm = (const int32_t*)c->mp_perm.p + c->perm_off[d];
    M.n_items = n_it;
    // enough threads to fill the GPU: split the folds when a group has few masks
    const long long want = (long long)c->sm_count * 1024;
    M.fold_chunks = (int)std::max(1LL, std::min<long long>(S, want / n_it));
    const unsigned grid = (unsigned)(((long long)n_it * M.fold_chunks + 127) / 128);
    auto fn = d < 10 ? mask_fit_launch_a : d < 14 ? mask_fit_launch_b : d < 17 ? mask_fit_launch_c
                                                                         : mask_fit_launch_d;
    cudaError_t ce = cudaSuccess;
    const sr_status s2 = launch(c, "k_mask_fit", [&] { ce = fn(d, grid, c->stream, M); });
    if (ce != cudaSuccess) return fail(c, SR_E_CUDA, "k_mask_fit<%d>: %s", d, cudaGetErrorString(ce));
    if (s2) return s2;
  }
  *used = true;
  return SR_OK;
}

// IBK (NEXT-1) on the large-batch path (ibk_big.cuh): per
// batch of scenarios k_ibk_prep (CTA per fit), k_ibk_dist (CTA per fit and
// test-tile chunk), k_ibk_score (warp per fit), then A6 in k_rank_warp on the
// warp path's EX-table layout.
sr_status evaluate_big_ibk(sr_ctx* c, const sr_params* prm, long long first, long long count, BigArgs B, OptScore* opt,
                           ScnScore* scn, double* ex, int8_t* rec, unsigned long long* tot, sr_outputs* out) {
  const int G = c->G, O = c->O;
  const long long N = c->N;
  sr_status st;
  const long long np = 32LL * G;
  const long long batch = std::min<long long>(count, 16);
  const long long fits = batch * O;
  const int tg_stride = 32 * c->n_tg, ex_stride = c->n_os * tg_stride;
  if ((st = ensure(c, c->ibk_lists, (size_t)fits * np * (4 + 8 + 4 + 4))) ||
      (st = ensure(c, c->ibk_xs, (size_t)fits * np * kIbkLd * 8)) ||
      (st = ensure(c, c->ibk_meta, (size_t)fits * sizeof(IbkMeta))) ||
      (st = ensure(c, c->extab, (size_t)batch * ex_stride * 8)) || (st = ensure(c, c->trained, (size_t)batch * 4)) ||
      (st = ensure(c, c->guard_acc, (size_t)batch * 4)))
    return st;
  IbkArgs I{};
  I.B = B;
  I.k_nn = prm->k_nn;
  I.np = np;
  unsigned char* lp = (unsigned char*)c->ibk_lists.p;
  I.trs = (int32_t*)lp;
  I.yl = (double*)(lp + (size_t)fits * np * 4);
  I.tes = (int32_t*)(lp + (size_t)fits * np * 12);
  I.tek = (int32_t*)(lp + (size_t)fits * np * 16);
  I.xs = (double*)c->ibk_xs.p;
  I.meta = (IbkMeta*)c->ibk_meta.p;
  // test-tile chunks per fit: one test tile per CTA, so the block scheduler
  // balances the ~25k tiles of a batch over the SMs (CTAs past a fit's tiles
  // exit at once); ~8 waves of multi-tile CTAs left a 0.4-wave tail and
  // 19/20-tile imbalance: 361 -> 339 ms per C4-IBK step, profiles/r5d_ab_ibk_chunks.txt
  const long long tiles_max = (np / 2 + kIbkTT - 1) / kIbkTT;
  I.chunks = (int)std::max(1LL, tiles_max);
  if (const char* e = getenv("SPEEDREC_IBK_CHUNKS"))   // A/B knob: test-tile chunks per fit
    I.chunks = (int)std::max(1LL, std::min<long long>(tiles_max, atoll(e)));
  EvalArgs& E = I.E;
  E.x = B.x;
  E.ylab = B.ylab;
  E.opt_bit = B.opt_bit;
  E.P = c->P;
  E.IR = c->I * c->R;
  E.C = c->C;
  E.O = O;
  E.G = G;
  E.sd = scen_desc(c);
  E.threshold = prm->threshold;
  E.clamp_floor = prm->clamp_floor;
  E.guard_tol = prm->guard_tol;
  E.max_count = prm->max_count;
  E.learner = prm->learner;
  E.k_nn = prm->k_nn;
  E.extab = (double*)c->extab.p;
  E.ex_stride = ex_stride;
  E.tg_stride = tg_stride;
  E.trained = (uint32_t*)c->trained.p;
  E.guard_acc = (int*)c->guard_acc.p;
  E.totals = tot;
  E.out0 = 0;
  CU(cudaFuncSetAttribute(k_ibk_dist, cudaFuncAttributeMaxDynamicSharedMemorySize, kIbkDistSmem));
  for (long long b0 = 0; b0 < count; b0 += batch) {
    const long long bc = std::min(batch, count - b0);
    I.B.first = first + b0;
    I.B.count = bc;
    E.first = first + b0;
    E.count = bc;
    E.opt_out = opt + b0 * O;
    E.scn_out = scn + b0;
    E.ex_out = ex ? ex + b0 * O * G * 32 : nullptr;
    E.rec_out = rec ? rec + b0 * N * prm->max_count : nullptr;
    if (E.ex_out) CU(cudaMemsetAsync(E.ex_out, 0, (size_t)bc * O * G * 32 * 8, c->stream));
    if (E.rec_out) CU(cudaMemsetAsync(E.rec_out, 0xFF, (size_t)bc * N * prm->max_count, c->stream));
    CU(cudaMemsetAsync(E.trained, 0, (size_t)bc * 4, c->stream));
    CU(cudaMemsetAsync(E.guard_acc, 0, (size_t)bc * 4, c->stream));
    const long long nf = bc * O;
    if ((st = launch(c, "k_ibk_prep", [&] { k_ibk_prep<<<(unsigned)nf, kBigThreads, 0, c->stream>>>(I); })))
      return st;
    if ((st = launch(c, "k_ibk_dist",
                     [&] { k_ibk_dist<<<(unsigned)(nf * I.chunks), kBigThreads, kIbkDistSmem, c->stream>>>(I); })))
      return st;
    if ((st = launch(c, "k_ibk_score",
                     [&] { k_ibk_score<<<(unsigned)((nf * 32 + 255) / 256), 256, 0, c->stream>>>(I, nf); })))
      return st;
    const long long rblocks = std::max(1LL, std::min<long long>((long long)c->sm_count * 8, (bc + 7) / 8));
    if ((st = launch(c, "k_rank_warp", [&] { k_rank_warp<8><<<(unsigned)rblocks, 256, 0, c->stream>>>(E); })))
      return st;
  }
  if (!out->on_device) {
    const size_t b_opt = (size_t)count * O * sizeof(sr_opt_score), b_scn = (size_t)count * sizeof(sr_scn_score);
    const size_t b_ex = (size_t)count * O * G * 32 * 8, b_rec = (size_t)count * N * prm->max_count;
    CU(cudaMemcpyAsync(out->opt_scores, opt, b_opt, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(out->scn_scores, scn, b_scn, cudaMemcpyDeviceToHost, c->stream));
    if (out->ex) CU(cudaMemcpyAsync(out->ex, ex, b_ex, cudaMemcpyDeviceToHost, c->stream));
    if (out->recs) CU(cudaMemcpyAsync(out->recs, rec, b_rec, cudaMemcpyDeviceToHost, c->stream));
    if (out->totals) CU(cudaMemcpyAsync(out->totals, tot, 32, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  return SR_OK;
}

// Large-batch path (> 64 groups, config C4): k_fit_big per (scenario, opt)
// fit + k_rank_big per scenario, over scenario batches that bound the
// per-batch weight table.
sr_status evaluate_big(sr_ctx* c, const sr_params* prm, long long first, long long count, sr_outputs* out) {
  const int G = c->G, O = c->O, C = c->C;
  const long long N = c->N;
  sr_status st;
  const long long batch = std::min<long long>(count, 4096);
  const long long np = 32LL * G;
  const int fit_grid = (int)std::min<long long>(c->sm_count, batch * O);
  if ((st = ensure(c, c->big_lists, (size_t)fit_grid * np * 4)) ||
      (st = ensure(c, c->big_y, (size_t)fit_grid * np * 8)) ||
      (st = ensure(c, c->big_U, (size_t)batch * O * C * 8)) || (st = ensure(c, c->big_c0, (size_t)batch * O * 8)) ||
      (st = ensure(c, c->big_flag, (size_t)batch * O * 4)))
    return st;
  const size_t b_opt = (size_t)count * O * sizeof(sr_opt_score), b_scn = (size_t)count * sizeof(sr_scn_score);
  const size_t b_ex = (size_t)count * O * G * 32 * 8, b_rec = (size_t)count * N * prm->max_count;
  OptScore* opt = (OptScore*)out->opt_scores;
  ScnScore* scn = (ScnScore*)out->scn_scores;
  double* ex = out->ex;
  int8_t* rec = out->recs;
  unsigned long long* tot = (unsigned long long*)out->totals;
  if (!out->on_device) {
    if ((st = ensure(c, c->out_opt, b_opt)) || (st = ensure(c, c->out_scn, b_scn))) return st;
    opt = (OptScore*)c->out_opt.p;
    scn = (ScnScore*)c->out_scn.p;
    if (ex) {
      if ((st = ensure(c, c->out_ex, b_ex))) return st;
      ex = (double*)c->out_ex.p;
    }
    if (rec) {
      if ((st = ensure(c, c->out_rec, b_rec))) return st;
      rec = (int8_t*)c->out_rec.p;
    }
    if (tot) {
      if ((st = ensure(c, c->out_tot, 32))) return st;
      tot = (unsigned long long*)c->out_tot.p;
    }
  }
  if (tot) CU(cudaMemsetAsync(tot, 0, 32, c->stream));
  BigArgs B{};
  B.x = (const double*)c->x.p;
  B.ylab = (const double*)c->ylab.p;
  B.opt_bit = (const int8_t*)c->opt_bit.p;
  B.P = c->P;
  B.IR = c->I * c->R;
  B.C = C;
  B.O = O;
  B.G = G;
  B.kind = c->sc.kind;
  B.gw = (G + 63) / 64;
  B.n_splits = c->sc.n_splits;
  B.train_g = (const uint64_t*)c->train_g.p;
  B.test_g = (const uint64_t*)c->test_g.p;
  B.split_om = c->sc.split_opt_masks ? (const uint32_t*)c->split_om.p : nullptr;
  B.pool_list = (const int32_t*)c->pool_list.p;
  B.n_pool = (int)c->h_pool.size();
  B.seed = c->sc.seed;
  B.opt_mask = c->sc.opt_mask;
  B.subsets_k = c->sc.all_subsets_k;
  B.n_masks = c->sc.n_masks;
  B.fmasks = (c->sc.feature_masks && c->sc.all_subsets_k == 0) ? (const uint64_t*)c->fmasks.p : nullptr;
  B.lambda = prm->ridge;
  B.threshold = prm->threshold;
  B.clamp_floor = prm->clamp_floor;
  B.guard_tol = prm->guard_tol;
  B.refine = prm->refine_steps;
  B.max_count = prm->max_count;
  B.lists = (int32_t*)c->big_lists.p;
  B.ylist = (double*)c->big_y.p;
  B.np = np;
  B.U = (double*)c->big_U.p;
  B.c0 = (double*)c->big_c0.p;
  B.fitflag = (int32_t*)c->big_flag.p;
  B.totals = tot;
  B.fit_all = c->coef_req ? 1 : 0;
  const int smem = (kBigMaxD * kBigGLd + kBigChunk * kBigLd + kBigChunk * kBigMaxD + 6 * kBigMaxD + 2 * kBigChunk +
                    16 + 8) * 8 + (2 * kBigMaxD + 2 * G + 20) * 4;
  CU(cudaFuncSetAttribute(k_fit_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (c->n_os > 8) return fail(c, SR_E_UNSUPPORTED, "evaluate: > 64 groups supports <= 8 scored optimizations");
  // optional (SPEEDREC_L2_PERSIST=1): an L2 persisting access window over the
  // rates, which every fit gathers from (A/B knob)
  if (const char* e = getenv("SPEEDREC_L2_PERSIST")) {
    if (atoi(e) != 0) {
      const size_t xb = (size_t)N * C * 8;
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, xb);
      cudaStreamAttrValue av{};
      av.accessPolicyWindow.base_ptr = c->x.p;
      av.accessPolicyWindow.num_bytes = xb;
      av.accessPolicyWindow.hitRatio = 1.0f;
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &av);
      cudaGetLastError();
    }
  }
  if (prm->learner == SR_IBK) return evaluate_big_ibk(c, prm, first, count, B, opt, scn, ex, rec, tot, out);
  for (long long b0 = 0; b0 < count; b0 += batch) {
    const long long bc = std::min(batch, count - b0);
    B.first = first + b0;
    B.count = bc;
    B.opt_out = opt + b0 * O;
    B.scn_out = scn + b0;
    B.ex_out = ex ? ex + b0 * O * G * 32 : nullptr;
    B.rec_out = rec ? rec + b0 * N * prm->max_count : nullptr;
    const int grid = (int)std::min<long long>(c->sm_count, bc * O);
    if ((st = launch(c, "k_fit_big", [&] { k_fit_big<<<grid, kBigThreads, smem, c->stream>>>(B); }))) return st;
    // batched ranking (kRankSB scenarios share each staged rate tile) unless
    // C is odd (16-byte staging) or SPEEDREC_RANK_BIG=1 asks for k_rank_big
    bool r4 = (C % 2) == 0;
    if (const char* e = getenv("SPEEDREC_RANK_BIG")) r4 = r4 && atoi(e) != 1;
    if (r4) {
      const int sm4 = kRankBig4Smem + ((c->P * O + 15) & ~15);
      CU(cudaFuncSetAttribute(k_rank_big4, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
      const unsigned g4 = (unsigned)((bc + kRankSB - 1) / kRankSB);
      if ((st = launch(c, "k_rank_big", [&] { k_rank_big4<<<g4, kBigThreads, sm4, c->stream>>>(B); })))
        return st;
    } else if ((st = launch(c, "k_rank_big", [&] { k_rank_big<8><<<(unsigned)bc, kBigThreads, 0, c->stream>>>(B); }))) {
      return st;
    }
  }
  if (!out->on_device) {
    CU(cudaMemcpyAsync(out->opt_scores, opt, b_opt, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(out->scn_scores, scn, b_scn, cudaMemcpyDeviceToHost, c->stream));
    if (out->ex) CU(cudaMemcpyAsync(out->ex, ex, b_ex, cudaMemcpyDeviceToHost, c->stream));
    if (out->recs) CU(cudaMemcpyAsync(out->recs, rec, b_rec, cudaMemcpyDeviceToHost, c->stream));
    if (out->totals) CU(cudaMemcpyAsync(out->totals, tot, 32, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  return SR_OK;
}

}  // namespace

sr_status sr_evaluate(sr_ctx* c, const sr_params* prm, int64_t first, int64_t count, sr_outputs* out) {
  if (!c) return SR_E_ARG;
  c->err.clear();
  if (!c->have_ds || !c->have_sc) return fail(c, SR_E_STATE, "evaluate: dataset and scenarios must be defined first");
  if (!prm || !out) return fail(c, SR_E_ARG, "evaluate: null pointer");
  const bool agg = out->mask_scores || out->top_masks;
  if (!agg && (!out->opt_scores || !out->scn_scores))
    return fail(c, SR_E_ARG, "evaluate: opt_scores and scn_scores are required without mask aggregation");
  const long long total = c->sc.n_splits * c->sc.n_masks;
  if (first < 0 || count < 0 || first + count > total)
    return fail(c, SR_E_ARG, "evaluate: range [%lld, %lld) outside [0, %lld)", (long long)first,
                (long long)(first + count), total);
  if (agg && (first % c->sc.n_splits || count % c->sc.n_splits))
    return fail(c, SR_E_ARG, "evaluate: mask aggregation needs first/count multiples of n_splits=%lld",
                (long long)c->sc.n_splits);
  if (agg && (prm->top_k < 1 || prm->top_k > 512)) return fail(c, SR_E_ARG, "evaluate: top_k=%d", prm->top_k);
  if (prm->learner != SR_LINREG && prm->learner != SR_IBK && prm->learner != SR_M5P)
    return fail(c, SR_E_ARG, "evaluate: learner %d", prm->learner);
  if (prm->learner == SR_IBK && (prm->k_nn < 1 || prm->k_nn > kKnnMax))
    return fail(c, SR_E_ARG, "evaluate: k_nn=%d outside [1, %d]", prm->k_nn, kKnnMax);
  if (prm->max_count < 1 || prm->max_count > kMaxRec) return fail(c, SR_E_ARG, "evaluate: max_count=%d", prm->max_count);
  if (prm->refine_steps < 0 || prm->refine_steps > 8) return fail(c, SR_E_ARG, "evaluate: refine_steps=%d", prm->refine_steps);
  if (!(prm->ridge > 0.0) || !std::isfinite(prm->ridge)) return fail(c, SR_E_ARG, "evaluate: ridge must be finite and > 0");
  // the EX table marks clamped values by sign: the floor must be positive (S:327 uses 0.01)
  if (!(prm->clamp_floor > 0.0) || !std::isfinite(prm->clamp_floor))
    return fail(c, SR_E_ARG, "evaluate: clamp_floor must be finite and > 0");
  if (!std::isfinite(prm->threshold)) return fail(c, SR_E_ARG, "evaluate: threshold must be finite");
  if (!(prm->guard_tol >= 0.0) || !std::isfinite(prm->guard_tol))
    return fail(c, SR_E_ARG, "evaluate: guard_tol must be finite and >= 0");
  cudaSetDevice(c->device);
  c->last_launches = 0;
  const int G = c->G, O = c->O, C = c->C;
  const long long N = c->N;
  sr_status st;

  // ---- A0 + A1 labels (per call: part of the step) ----
  if ((st = launch(c, "k_rates", [&] {
         k_rates<<<grid_for(c, N * C, 256), 256, 0, c->stream>>>((const double*)c->counters.p,
                                                                 (const double*)c->cycles.p,
                                                                 (double*)c->x.p, N, C);
       })))
    return st;
  if ((st = launch(c, "k_labels", [&] {
         k_labels<<<grid_for(c, (long long)G * O * 32, 256), 256, 0, c->stream>>>(
             (const double*)c->runtime.p, (const int8_t*)c->opt_bit.p, (double*)c->ylab.p, G, O,
             c->I * c->R);
       })))
    return st;
  if (count == 0) return SR_OK;
  if (prm->learner == SR_M5P && (G > kMaxGroups || C > kM5MaxFeatures))
    return fail(c, SR_E_UNSUPPORTED, "evaluate: learner M5P needs <= %d groups and <= %d counters (G=%d, C=%d)",
                kMaxGroups, kM5MaxFeatures, G, C);
  if (G > kMaxGroups) {
    if (agg) return fail(c, SR_E_UNSUPPORTED, "evaluate: mask aggregation needs <= %d groups", kMaxGroups);
    return evaluate_big(c, prm, first, count, out);
  }

  // ---- plan k_fit_warp ----
  // Launch-shape knobs (defaults = the tuned configuration): SPEEDREC_STAGE=0/1
  // forces staging of x in shared memory, SPEEDREC_WMAX in {12,16} picks the
  // warps-per-CTA variant, SPEEDREC_SMEM_KB caps shared memory per CTA.
  const int budget = c->max_smem_optin;                  // 232448 on B200
  const int head = align16(G * O);                      // per-group optimization bits
  const int ldxs = C | 1;
  const long long stage_bytes = N * ldxs * 8;
  const int mmax = std::min(c->np_tr, c->dmax + 1);      // largest system any fit can need
  // M5P reads x only to scale its rows and tests; its hot loops run over the
  // per-warp scratch slab, which wants the shared memory as L1 (+11 %, C3)
  int stage = stage_bytes <= 96 * 1024 && prm->learner != SR_M5P ? 1 : 0;
  if (const char* e = getenv("SPEEDREC_STAGE")) stage = atoi(e) && stage_bytes <= 96 * 1024;
  int wmax = kMaxWarpsPerBlock;
  if (const char* e = getenv("SPEEDREC_WMAX")) {
    const int w = atoi(e);
    wmax = w >= 16 ? 16 : 12;   // 20/24 warps with a smaller factor cap: slower (profiles/r2e_ab_occupancy.txt)
  }
  if (prm->learner != SR_LINREG || c->coef_req) wmax = 16;   // the one IBK / M5P / sr_fit instantiation
  if (prm->learner == SR_M5P) wmax = SR_M5_WMAX;
  // split LS path: k_fit_warp<16, 4, true> leaves each fit's
  // model in a table, k_pred_rank predicts (DMMA), scores and ranks per
  // scenario -- no EX table, no k_rank_warp.  SPEEDREC_SPLIT_LS=0 (or the
  // opt-in fused ranking) keeps the EX-table path.
  const int ks_pr = (C + 3) / 4;                        // k_pred_rank instantiations: 1, 5, 8, 16 k-steps
  bool split_ls = prm->learner == SR_LINREG && !c->coef_req && !c->sweep && !agg && stage && C <= kPrMaxC &&
                  c->n_os <= 8 && (ks_pr == 1 || ks_pr == 5 || ks_pr == 8 || ks_pr == 16);
  if (const char* e = getenv("SPEEDREC_SPLIT_LS")) split_ls = split_ls && atoi(e) != 0;
  if (const char* e = getenv("SPEEDREC_FUSE_RANK")) split_ls = split_ls && atoi(e) == 0;
  // k_pred_rank's shared-memory plan: rates staged with a row stride = 4 mod 16
  // doubles (conflict-free DMMA fragment loads), labels, per-warp EX tiles
  PredLayout PL{};
  if (split_ls) {
    int ld = ((C + 3) / 4) * 4;
    while (ld % 16 != 4) ld += 4;
    const int cm = c->n_os <= 6 ? 6 : 8;
    int ldut = ((C + 3) & ~3) + kUextra;             // weights padded to whole k-steps, then the fields
    while (ldut % 16 != 4) ldut += 2;
    PL.ldxp = ld;
    PL.ldut = ldut;
    PL.off_x = align16(c->P * O);
    PL.off_y = PL.off_x + align16((int)(N * ld * 8));
    PL.off_w = PL.off_y + align16((G * O * 32 + ldut) * 8);
    PL.wbytes = align16(2 * cm * ldut * 8 + kPrChunk * (cm + 1) * 8 + 16 + 8 * 4 + (int)N * 2);
    PL.warps = std::min(kPrWarps, (budget - PL.off_w) / PL.wbytes);
    PL.bytes = PL.off_w + PL.warps * PL.wbytes;
    if (PL.warps < 4) split_ls = false;
  }
  int budget_cap = budget;
  if (const char* e = getenv("SPEEDREC_SMEM_KB")) budget_cap = std::min(budget, std::max(16, atoi(e)) * 1024);
  int mcap = std::min(mmax, 32);
  if (prm->debug_mcap > 0) mcap = std::min(mcap, prm->debug_mcap);
  // A/B knob: a smaller shared-memory factor (rare larger systems go to the
  // global-scratch path) frees shared memory for more warps per SM
  if (const char* e = getenv("SPEEDREC_MCAP")) mcap = std::min(mcap, std::max(8, atoi(e)));
  // the split LS fit kernel's lean slab: no test lists, weights aliased into
  // the factor buffer
  // (20 warps: no faster, the register cap spills -- profiles/r2n_ab_wls.txt)
  if (split_ls) wmax = 16;
  WarpLayout L = plan_layout(c, mcap, prm->learner == SR_IBK, split_ls);
  int avail = budget_cap - head - (stage ? align16((int)stage_bytes) : 0);
  int wpb = std::min(wmax, avail / std::max(L.bytes, 1));
  if (wpb < 1 && stage) {
    stage = 0;
    avail = budget_cap - head;
    wpb = std::min(wmax, avail / L.bytes);
  }
  if (wpb < 1) return fail(c, SR_E_UNSUPPORTED, "evaluate: per-warp workspace %d B exceeds shared memory", L.bytes);
  // stage the labels too when they are small and the warps keep their count
  const int ybytes = align16(G * O * 32 * 8);
  const int base_warps = head + (stage ? align16((int)stage_bytes) : 0);
  const int stage_y = (ybytes <= 16384 && base_warps + ybytes + wpb * L.bytes <= budget_cap) ? 1 : 0;
  // global scratch for systems beyond the shared-memory factor: packed factor + 2 vectors
  long long mscr = (mmax > std::min(mcap, 32)) ? (long long)mmax * (mmax + 1) / 2 + 2LL * L.vmax : 0;
  // M5P: the tree workspace (scaled rows, nodes, model pool, node systems) per warp
  if (prm->learner == SR_M5P) mscr = std::max(mscr, m5_scratch_doubles(c->np_tr, C));

  EvalArgs A{};
  A.x = (const double*)c->x.p;
  A.ylab = (const double*)c->ylab.p;
  A.opt_bit = (const int8_t*)c->opt_bit.p;
  A.P = c->P;
  A.IR = c->I * c->R;
  A.C = C;
  A.O = O;
  A.G = G;
  A.sd = scen_desc(c);
  A.lambda = prm->ridge;
  A.threshold = prm->threshold;
  A.clamp_floor = prm->clamp_floor;
  A.guard_tol = prm->guard_tol;
  A.max_count = prm->max_count;
  A.refine = prm->refine_steps;
  A.learner = prm->learner;
  A.k_nn = prm->k_nn;
  A.L = L;
  A.warps_per_block = wpb;
  A.stage_x = stage;
  A.ldxs = ldxs;
  A.off_stage = head;
  A.stage_y = stage_y;
  A.off_y = base_warps;
  A.off_warps = base_warps + (stage_y ? ybytes : 0);
  const int smem = A.off_warps + wpb * L.bytes;
  auto kfit = split_ls ? k_fit_warp<16, 4, true>
              : prm->learner == SR_IBK ? (stage ? k_fit_warp<16, 1, true> : k_fit_warp<16, 1, false>)
              : prm->learner == SR_M5P ? (stage ? k_fit_warp<SR_M5_WMAX, 3, true> : k_fit_warp<SR_M5_WMAX, 3, false>)
              : c->coef_req      ? (stage ? k_fit_warp<16, 2, true> : k_fit_warp<16, 2, false>)
              : wmax == 16       ? (stage ? k_fit_warp<16, 0, true> : k_fit_warp<16, 0, false>)
                                 : (stage ? k_fit_warp<12, 0, true> : k_fit_warp<12, 0, false>);
  CU(cudaFuncSetAttribute(kfit, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfit, wpb * 32, smem));
  per_sm = std::max(per_sm, 1);

  // ---- per-chunk exchange buffers (EX table, trained masks, guard counts) ----
  const int tg_stride = 32 * c->n_tg;
  const int ex_stride = c->n_os * tg_stride;
  // exchange table per launch (SPEEDREC_CHUNK_MB overrides; tools/sweep_c3.sh,
  // tools/ab_chunk.sh): 1 GB; the split LS path with device outputs takes the
  // whole batch in one launch pair (fewer tails: C3 39.6 -> 38.9 ms), with host
  // outputs 1 GB chunks so each chunk's rows copy back under the next one's fits
  long long chunk_bytes = 1024LL << 20;
  if (const char* e = getenv("SPEEDREC_CHUNK_MB")) chunk_bytes = std::max(1LL, atoll(e)) << 20;
  // model-table row (split LS path): k_pred_rank's shared-memory row stride,
  // so one bulk copy moves a scenario's rows
  const int ldu = split_ls ? PL.ldut : ((C + kUextra + 1) / 2) * 2;
  const long long row_bytes = split_ls ? 8LL * c->n_os * ldu : 8LL * ex_stride;
  if (split_ls && out->on_device && !getenv("SPEEDREC_CHUNK_MB")) chunk_bytes = 4096LL << 20;
  const long long chunk = std::max(1LL, std::min<long long>(count, chunk_bytes / row_bytes));
  if (split_ls) {
    if ((st = ensure(c, c->utab, (size_t)(chunk * row_bytes)))) return st;
  } else if ((st = ensure(c, c->extab, (size_t)chunk * ex_stride * 8)) || (st = ensure(c, c->trained, (size_t)chunk * 4)) ||
             (st = ensure(c, c->guard_acc, (size_t)chunk * 4)) || (st = ensure(c, c->done, (size_t)chunk * 4))) {
    return st;
  }
  A.utab = (double*)c->utab.p;
  if (prm->learner == SR_M5P) {
    if ((st = ensure(c, c->work, 8))) return st;
    CU(cudaMemsetAsync(c->work.p, 0, 8, c->stream));
    A.work = (unsigned long long*)c->work.p;
  }
  A.ldu = ldu;
  A.n_os = c->n_os;
  A.extab = (double*)c->extab.p;
  A.ex_stride = ex_stride;
  A.tg_stride = tg_stride;
  A.trained = (uint32_t*)c->trained.p;
  A.guard_acc = (int*)c->guard_acc.p;
  A.done = (int*)c->done.p;
  A.coef_out = c->coef_req;
  const long long max_fit_blocks = (long long)c->sm_count * per_sm;
  if (mscr > 0) {
    if ((st = ensure(c, c->gscratch, (size_t)(max_fit_blocks * wpb * mscr * 8)))) return st;
    A.gscratch = (double*)c->gscratch.p;
    A.mscratch = mscr;
  }

  // ---- outputs ----
  const size_t b_opt = (size_t)count * O * sizeof(sr_opt_score), b_scn = (size_t)count * sizeof(sr_scn_score);
  const size_t b_ex = (size_t)count * O * G * 32 * 8, b_rec = (size_t)count * N * prm->max_count;
  const long long nm = agg ? count / c->sc.n_splits : 0;
  const int K = prm->top_k;
  if (agg) {
    A.agg = 1;
    A.mask0 = first / c->sc.n_splits;
    A.n_mask_range = nm;
    const long long nk2 = (nm + 1023) / 1024 * K;
    if ((st = ensure(c, c->keys_a, (size_t)std::max(nm, 1LL) * 8)) ||
        (st = ensure(c, c->keys_b, (size_t)std::max(nk2, (long long)K) * 8)) ||
        (st = ensure(c, c->mask_acc, (size_t)std::max(nm, 1LL) * 16)))
      return st;
    A.keys_out = (unsigned long long*)c->keys_a.p;
    A.mask_acc = (int*)c->mask_acc.p;
    CU(cudaMemsetAsync(A.mask_acc, 0, (size_t)nm * 16, c->stream));
  }
  if (out->on_device) {
    A.opt_out = (OptScore*)out->opt_scores;
    A.scn_out = (ScnScore*)out->scn_scores;
    A.ex_out = out->ex;
    A.rec_out = out->recs;
    A.totals = (unsigned long long*)out->totals;
    A.mask_out = (MaskScore*)out->mask_scores;
  } else {
    if (out->opt_scores) {
      if ((st = ensure(c, c->out_opt, b_opt))) return st;
      A.opt_out = (OptScore*)c->out_opt.p;
    }
    if (out->scn_scores) {
      if ((st = ensure(c, c->out_scn, b_scn))) return st;
      A.scn_out = (ScnScore*)c->out_scn.p;
    }
    if (out->mask_scores) {
      if ((st = ensure(c, c->out_mask, (size_t)nm * sizeof(sr_mask_score)))) return st;
      A.mask_out = (MaskScore*)c->out_mask.p;
    }
    if (out->ex) {
      if ((st = ensure(c, c->out_ex, b_ex))) return st;
      A.ex_out = (double*)c->out_ex.p;
    }
    if (out->recs) {
      if ((st = ensure(c, c->out_rec, b_rec))) return st;
      A.rec_out = (int8_t*)c->out_rec.p;
    }
    if (out->totals) {
      if ((st = ensure(c, c->out_tot, 32))) return st;
      A.totals = (unsigned long long*)c->out_tot.p;
    }
  }
  if (A.totals) CU(cudaMemsetAsync(A.totals, 0, 32, c->stream));
  if (A.ex_out) CU(cudaMemsetAsync(A.ex_out, 0, b_ex, c->stream));
  if (A.rec_out) CU(cudaMemsetAsync(A.rec_out, 0xFF, b_rec, c->stream));
  const int cmax = c->n_os <= 8 ? 8 : 16;
  bool mask_path = false;
  if ((st = run_mask_path(c, prm, first, count, A, &mask_path))) return st;
  // host rows of the warp path: each chunk's rows are copied on the copy
  // stream as soon as its ranking is done (overlaps the next chunk's fits)
  const bool early_rows = !out->on_device && out->opt_scores && out->scn_scores && !mask_path && !c->sweep;
  if (early_rows && !c->cstream) CU(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
  int n_cp = 0;
  for (long long c0 = 0; c0 < (mask_path ? 0 : count); c0 += chunk) {
    const long long cc = std::min(chunk, count - c0);
    A.first = first + c0;
    A.count = cc;
    A.out0 = c0;
    if (!split_ls) {
      CU(cudaMemsetAsync(A.trained, 0, (size_t)cc * 4, c->stream));
      CU(cudaMemsetAsync(A.guard_acc, 0, (size_t)cc * 4, c->stream));
    }
    // fused ranking in the LS fit kernel: opt-in (SPEEDREC_FUSE_RANK=1).  Its
    // per-fit __threadfence + cross-SM counter made the C3 step 2x slower
    // (108 vs 56 ms), so k_rank_warp stays the default.
    A.fuse_rank = 0;
    if (const char* e = getenv("SPEEDREC_FUSE_RANK"))
      A.fuse_rank = (atoi(e) != 0 && cmax == 8 && prm->learner == SR_LINREG && !c->coef_req) ? 1 : 0;
    if (A.fuse_rank) CU(cudaMemsetAsync(A.done, 0, (size_t)cc * 4, c->stream));
    // whole scenarios per warp once the chunk has >= 4 scenarios per resident warp
    A.scn_major = cc >= 4 * max_fit_blocks * wpb ? 1 : 0;
    const long long units = A.scn_major ? cc : cc * O;
    // M5P teams: when the fits leave warps idle, 2 or 4 warps share each
    // fit's split search; SPEEDREC_M5_TEAM forces 1/2/4
    A.m5_team = 1;
    if (prm->learner == SR_M5P) {
      // teams of 2 once the work units (many of them cheap: unscored or small
      // fits) no longer fill the warps 1.25 times (C2: 9.4 -> 7.8 ms; teams of
      // 4 and teams on C3 are slower, profiles/r3i_ab_m5team.txt)
      if (units * 4 <= 5 * max_fit_blocks * wpb) A.m5_team = 2;
      if (const char* e = getenv("SPEEDREC_M5_TEAM")) A.m5_team = atoi(e) >= 4 ? 4 : atoi(e) >= 2 ? 2 : 1;
      if (wpb % A.m5_team) A.m5_team = 1;
    }
    const long long fblocks = std::max(1LL, std::min(max_fit_blocks, (units * A.m5_team + wpb - 1) / wpb));
    // dynamic work units (SPEEDREC_DYN_UNITS=0: static stride)
    static const bool dyn_units = [] {
      const char* e = getenv("SPEEDREC_DYN_UNITS");
      return e ? atoi(e) != 0 : true;
    }();
    A.queue = nullptr;
    if (dyn_units && units * A.m5_team > fblocks * wpb) {
      if ((st = ensure(c, c->qctr, 8))) return st;
      CU(cudaMemsetAsync(c->qctr.p, 0, 8, c->stream));
      A.queue = (unsigned long long*)c->qctr.p;
    }
    if ((st = launch(c, "k_fit_warp", [&] { kfit<<<(unsigned)fblocks, wpb * 32, smem, c->stream>>>(A); }))) return st;
    if (split_ls) {
      const int ks = (C + 3) / 4;
      auto kpr = c->n_os <= 6 ? (ks == 16 ? k_pred_rank<6, 16> : ks == 8 ? k_pred_rank<6, 8> : ks == 5 ? k_pred_rank<6, 5>
                                                                                            : k_pred_rank<6, 1>)
                              : (ks == 16 ? k_pred_rank<8, 16> : ks == 8 ? k_pred_rank<8, 8> : ks == 5 ? k_pred_rank<8, 5>
                                                                                            : k_pred_rank<8, 1>);
      CU(cudaFuncSetAttribute(kpr, cudaFuncAttributeMaxDynamicSharedMemorySize, PL.bytes));
      const long long pblocks = std::max(1LL, std::min<long long>(c->sm_count, (cc + PL.warps - 1) / PL.warps));
      if ((st = launch(c, "k_pred_rank", [&] { kpr<<<(unsigned)pblocks, PL.warps * 32, PL.bytes, c->stream>>>(A, PL); })))
        return st;
    }
    const long long rblocks = std::max(1LL, std::min<long long>((long long)c->sm_count * 8, (cc + 7) / 8));
    if (c->sweep) {   // NEXT-3 rule sweep instead of the single-rule ranking
      const SweepArgs W = *c->sweep;
      const int sm = W.n_thr * 8 + W.n_cnt * 4 + 2 * W.n_cnt * (W.n_thr + 1) * 4;
      if ((st = launch(c, "k_sweep_warp", [&] { k_sweep_warp<8><<<(unsigned)rblocks, 256, sm, c->stream>>>(A, W); })))
        return st;
      continue;
    }
    if (A.fuse_rank) continue;
    if (split_ls) {
      // (ranking done by k_pred_rank)
    } else if (c->n_os <= 6) {   // the paper's six optimizations: no empty candidate slots
      if ((st = launch(c, "k_rank_warp", [&] { k_rank_warp<6><<<(unsigned)rblocks, 256, 0, c->stream>>>(A); })))
        return st;
    } else if (cmax == 8) {
      if ((st = launch(c, "k_rank_warp", [&] { k_rank_warp<8><<<(unsigned)rblocks, 256, 0, c->stream>>>(A); })))
        return st;
    } else {
      if ((st = launch(c, "k_rank_warp", [&] { k_rank_warp<16><<<(unsigned)rblocks, 256, 0, c->stream>>>(A); })))
        return st;
    }
    if (early_rows && !A.fuse_rank) {
      if ((int)c->cp_events.size() <= n_cp) {
        cudaEvent_t e;
        CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->cp_events.push_back(e);
      }
      cudaEvent_t e = c->cp_events[n_cp++];
      CU(cudaEventRecord(e, c->stream));
      CU(cudaStreamWaitEvent(c->cstream, e, 0));
      CU(cudaMemcpyAsync(out->opt_scores + c0 * O, (const sr_opt_score*)c->out_opt.p + c0 * O,
                         (size_t)cc * O * sizeof(sr_opt_score), cudaMemcpyDeviceToHost, c->cstream));
      CU(cudaMemcpyAsync(out->scn_scores + c0, (const sr_scn_score*)c->out_scn.p + c0, (size_t)cc * sizeof(sr_scn_score),
                         cudaMemcpyDeviceToHost, c->cstream));
    }
  }
  const bool rows_copied = early_rows && n_cp > 0;
  if (agg) {
    if ((st = launch(c, "k_mask_final",
                     [&] { k_mask_final<<<grid_for(c, nm, 256), 256, 0, c->stream>>>(A); })))
      return st;
  }
  if (agg && out->top_masks) {
    // iterated block top-K over the mask keys (O8)
    unsigned long long* src = (unsigned long long*)c->keys_a.p;
    unsigned long long* dst = (unsigned long long*)c->keys_b.p;
    long long n = nm;
    do {
      const long long nb = (n + 1023) / 1024;
      if ((st = launch(c, "k_topk_keys", [&] { k_topk_keys<<<(unsigned)nb, 1024, 0, c->stream>>>(src, n, dst, K); })))
        return st;
      n = nb * K;
      std::swap(src, dst);
    } while (n > K);
    int64_t* tm = out->on_device ? out->top_masks : nullptr;
    if (!tm) {
      if ((st = ensure(c, c->out_top, (size_t)K * 8))) return st;
      tm = (int64_t*)c->out_top.p;
    }
    if ((st = launch(c, "k_decode_top", [&] { k_decode_top<<<1, 512, 0, c->stream>>>(src, n, tm, K); })))
      return st;
    if (!out->on_device)
      CU(cudaMemcpyAsync(out->top_masks, tm, (size_t)K * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if (!out->on_device) {
    if (out->opt_scores && !rows_copied)
      CU(cudaMemcpyAsync(out->opt_scores, c->out_opt.p, b_opt, cudaMemcpyDeviceToHost, c->stream));
    if (out->scn_scores && !rows_copied)
      CU(cudaMemcpyAsync(out->scn_scores, c->out_scn.p, b_scn, cudaMemcpyDeviceToHost, c->stream));
    if (rows_copied) CU(cudaStreamSynchronize(c->cstream));
    if (out->mask_scores)
      CU(cudaMemcpyAsync(out->mask_scores, c->out_mask.p, (size_t)nm * sizeof(sr_mask_score),
                         cudaMemcpyDeviceToHost, c->stream));
    if (out->ex) CU(cudaMemcpyAsync(out->ex, c->out_ex.p, b_ex, cudaMemcpyDeviceToHost, c->stream));
    if (out->recs) CU(cudaMemcpyAsync(out->recs, c->out_rec.p, b_rec, cudaMemcpyDeviceToHost, c->stream));
    if (out->totals) CU(cudaMemcpyAsync(out->totals, c->out_tot.p, 32, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  return SR_OK;
}

sr_status sr_rates(sr_ctx* c, double* x_out, int32_t on_device) {
  if (!c) return SR_E_ARG;
  c->err.clear();
  if (!c->have_ds) return fail(c, SR_E_STATE, "rates: no dataset loaded");
  if (!x_out) return fail(c, SR_E_ARG, "rates: null output");
  cudaSetDevice(c->device);
  c->last_launches = 0;
  const long long N = c->N;
  const int C = c->C;
  sr_status st = launch(c, "k_rates", [&] {
    k_rates<<<grid_for(c, N * C, 256), 256, 0, c->stream>>>((const double*)c->counters.p,
                                                            (const double*)c->cycles.p, (double*)c->x.p, N, C);
  });
  if (st) return st;
  CU(cudaMemcpyAsync(x_out, c->x.p, N * C * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return SR_OK;
}

// ---------------------------------------------------------------- tool path
// SPEC train_all / predict_all / rank_and_filter for
// one scenario and one user profile (include/speedrec.h).
sr_status sr_sweep(sr_ctx* c, const sr_params* prm, int64_t first, int64_t count, int32_t n_thr,
                   const double* thresholds, int32_t n_cnt, const int32_t* max_counts, int64_t* out_rec,
                   int64_t* out_hit) {
  if (!c) return SR_E_ARG;
  c->err.clear();
  if (!prm || !thresholds || !max_counts || !out_rec || !out_hit) return fail(c, SR_E_ARG, "sweep: null pointer");
  if (n_thr < 1 || n_thr > 256 || n_cnt < 1 || n_cnt > 16)
    return fail(c, SR_E_ARG, "sweep: n_thr=%d (1..256), n_cnt=%d (1..16)", n_thr, n_cnt);
  for (int i = 0; i < n_thr; ++i)
    if (!std::isfinite(thresholds[i]) || (i > 0 && !(thresholds[i] > thresholds[i - 1])))
      return fail(c, SR_E_ARG, "sweep: thresholds must be finite and strictly ascending (index %d)", i);
  for (int j = 0; j < n_cnt; ++j)
    if (max_counts[j] < 1 || max_counts[j] > 16) return fail(c, SR_E_ARG, "sweep: max_counts[%d]=%d", j, max_counts[j]);
  if (!c->have_ds || !c->have_sc) return fail(c, SR_E_STATE, "sweep: dataset and scenarios must be defined first");
  if (c->G > kMaxGroups) return fail(c, SR_E_UNSUPPORTED, "sweep: needs <= %d groups", kMaxGroups);
  if (c->n_os > 8) return fail(c, SR_E_UNSUPPORTED, "sweep: needs <= 8 scored optimizations");
  cudaSetDevice(c->device);
  sr_status st;
  const size_t b_out = (size_t)2 * n_thr * n_cnt * 8;
  const size_t b = b_out + (size_t)n_thr * 8 + (size_t)n_cnt * 4;
  if ((st = ensure(c, c->sw_buf, b))) return st;
  unsigned char* base = (unsigned char*)c->sw_buf.p;
  SweepArgs W{};
  W.out = (unsigned long long*)base;
  W.thr = (const double*)(base + b_out);
  W.cnt = (const int*)(base + b_out + (size_t)n_thr * 8);
  W.n_thr = n_thr;
  W.n_cnt = n_cnt;
  CU(cudaMemsetAsync(base, 0, b_out, c->stream));
  CU(cudaMemcpyAsync(base + b_out, thresholds, (size_t)n_thr * 8, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemcpyAsync(base + b_out + (size_t)n_thr * 8, max_counts, (size_t)n_cnt * 4, cudaMemcpyHostToDevice,
                     c->stream));
  // per-scenario rows land in device scratch (not returned)
  const int O = c->O;
  if ((st = ensure(c, c->out_opt, (size_t)count * O * sizeof(sr_opt_score))) ||
      (st = ensure(c, c->out_scn, (size_t)count * sizeof(sr_scn_score))))
    return st;
  sr_outputs o{};
  o.opt_scores = (sr_opt_score*)c->out_opt.p;
  o.scn_scores = (sr_scn_score*)c->out_scn.p;
  o.on_device = 1;
  c->sweep = &W;
  st = sr_evaluate(c, prm, first, count, &o);
  c->sweep = nullptr;
  if (st) return st;
  std::vector<unsigned long long> h((size_t)2 * n_thr * n_cnt);
  CU(cudaMemcpyAsync(h.data(), W.out, b_out, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (size_t i = 0; i < (size_t)n_thr * n_cnt; ++i) {
    out_rec[i] = (int64_t)h[i];
    out_hit[i] = (int64_t)h[(size_t)n_thr * n_cnt + i];
  }
  return SR_OK;
}

sr_status sr_fit(sr_ctx* c, const sr_params* prm, int64_t scenario, double* coef_out) {
  if (!c) return SR_E_ARG;
  c->err.clear();
  if (!prm || !coef_out) return fail(c, SR_E_ARG, "fit: null params or output");
  if (prm->learner != SR_LINREG)
    return fail(c, SR_E_UNSUPPORTED, "fit: learner %d has no coefficient vector (IBK keeps its training set, M5P a tree)", prm->learner);
  if (!c->have_ds) return fail(c, SR_E_STATE, "fit: no dataset loaded");
  if (!c->have_sc) return fail(c, SR_E_STATE, "fit: no scenarios defined");
  const int O = c->O, C = c->C;
  const size_t bytes = (size_t)O * (C + 1) * 8;
  sr_status st;
  if ((st = ensure(c, c->fit_coef, bytes))) return st;
  cudaSetDevice(c->device);
  CU(cudaMemsetAsync(c->fit_coef.p, 0, bytes, c->stream));
  std::vector<sr_opt_score> opt(O);
  sr_scn_score scn;
  sr_outputs o{};
  o.opt_scores = opt.data();
  o.scn_scores = &scn;
  c->coef_req = (double*)c->fit_coef.p;
  st = sr_evaluate(c, prm, scenario, 1, &o);
  c->coef_req = nullptr;
  if (st) return st;
  if (c->G > kMaxGroups) {  // large-batch path: the batch-0 weight table holds the fit
    CU(cudaMemcpy2DAsync((double*)c->fit_coef.p + 1, (C + 1) * 8, c->big_U.p, C * 8, C * 8, O,
                         cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemcpy2DAsync(c->fit_coef.p, (C + 1) * 8, c->big_c0.p, 8, 8, O, cudaMemcpyDeviceToDevice, c->stream));
  }
  CU(cudaMemcpyAsync(coef_out, c->fit_coef.p, bytes, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (int q = 0; q < O; ++q)
    if (opt[q].n_train == 0) {  // not scored or untrained (R18): no model
      coef_out[(size_t)q * (C + 1)] = NAN;
      for (int k = 0; k < C; ++k) coef_out[(size_t)q * (C + 1) + 1 + k] = 0.0;
    }
  return SR_OK;
}

sr_status sr_predict(const sr_params* prm, const double* coef, int32_t n_opts, int32_t n_counters,
                     const double* counters, double cycles, double* ex_out) {
  if (!prm || !coef || !counters || !ex_out || n_opts < 1 || n_opts > 16 || n_counters < 1 || n_counters > 128)
    return SR_E_ARG;
  if (!(prm->clamp_floor > 0.0) || !std::isfinite(prm->clamp_floor)) return SR_E_ARG;
  if (!(cycles > 0.0) || !std::isfinite(cycles)) return SR_E_DATA;
  for (int k = 0; k < n_counters; ++k)
    if (!(counters[k] >= 0.0) || !std::isfinite(counters[k])) return SR_E_DATA;
  for (int q = 0; q < n_opts; ++q) {
    const double* cf = coef + (size_t)q * (n_counters + 1);
    if (std::isnan(cf[0])) {
      ex_out[q] = NAN;
      continue;
    }
    double e = 0.0;
    for (int k = 0; k < n_counters; ++k) e = std::fma(counters[k] / cycles, cf[1 + k], e);  // Tier 1
    e += cf[0];
    ex_out[q] = e <= 0.0 ? prm->clamp_floor : e;
  }
  return SR_OK;
}

sr_status sr_recommend(const sr_params* prm, const double* ex, const uint8_t* candidate, int32_t n_opts,
                       int8_t* rec_out, int32_t* n_rec_out) {
  if (!prm || !ex || !rec_out || !n_rec_out || n_opts < 0 || n_opts > 16 || prm->max_count < 1 ||
      prm->max_count > 64 || !std::isfinite(prm->threshold))
    return SR_E_ARG;
  int ids[16], n = 0;
  for (int q = 0; q < n_opts; ++q)
    if ((!candidate || candidate[q]) && !std::isnan(ex[q]) && ex[q] >= prm->threshold) ids[n++] = q;  // R8
  std::stable_sort(ids, ids + n, [&](int a, int b) { return ex[a] > ex[b]; });  // (EX desc, id asc), R10
  const int k = std::min(n, (int)prm->max_count);
  for (int q = 0; q < prm->max_count; ++q) rec_out[q] = q < k ? (int8_t)ids[q] : (int8_t)-1;
  *n_rec_out = k;
  return SR_OK;
}

sr_status sr_synchronize(sr_ctx* c) {
  if (!c) return SR_E_ARG;
  cudaSetDevice(c->device);
  CU(cudaStreamSynchronize(c->stream));
  return SR_OK;
}

sr_status sr_set_timing(sr_ctx* c, int32_t enable) {
  if (!c) return SR_E_ARG;
  c->timing = enable != 0;
  return SR_OK;
}

int32_t sr_kernel_stats(sr_ctx* c, int32_t cap, const char** names, int32_t* launches, double* ms) {
  if (!c) return (int32_t)SR_E_ARG;
  cudaSetDevice(c->device);
  collect_timing(c);
  const int n = (int)c->kstats.size();
  for (int i = 0; i < n && i < cap; ++i) {
    if (names) names[i] = c->kstats[i].name;
    if (launches) launches[i] = c->kstats[i].launches;
    if (ms) ms[i] = c->kstats[i].ms;
  }
  return n;
}

sr_status sr_reset_kernel_stats(sr_ctx* c) {
  if (!c) return SR_E_ARG;
  cudaSetDevice(c->device);
  collect_timing(c);
  for (auto& k : c->kstats) k.launches = 0, k.ms = 0.0;
  return SR_OK;
}

int32_t sr_last_launch_count(const sr_ctx* c) { return c ? c->last_launches : (int32_t)SR_E_ARG; }

int64_t sr_last_work(sr_ctx* c) {
  if (!c) return (int64_t)SR_E_ARG;
  if (!c->work.p) return 0;
  cudaSetDevice(c->device);
  unsigned long long w = 0;
  if (cudaMemcpyAsync(&w, c->work.p, 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess) {
    cudaGetLastError();
    return (int64_t)SR_E_CUDA;
  }
  return (int64_t)w;
}

}  // extern "C"
