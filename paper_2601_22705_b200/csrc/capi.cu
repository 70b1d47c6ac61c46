// C ABI of the B200 engine: batch lifecycle, HBM workspace layout, launches
// and result transfer (include/kvgpu.h). Host code only; kernels in engine.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "host_internal.h"
#include "kvg_device.h"

namespace kvg {
__global__ void engine_kernel_small(const SimDev* __restrict__ sims);
__global__ void engine_kernel_big(const SimDev* __restrict__ sims);
__global__ void cache_kernel(const CacheDev* __restrict__ cd);
}  // namespace kvg

using kvg::u32;
using kvg::u64;
using kvg_host::set_error;

namespace {

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return (kvg_status)set_error(KVG_ERR_CUDA, std::string(#expr) + ": " +        \
                                                     cudaGetErrorString(_e));       \
  } while (0)

u64 next_pow2(u64 x) {
  u64 p = 1;
  while (p < x) p <<= 1;
  return p;
}

u64 align_up(u64 x, u64 a = 256) { return (x + a - 1) / a * a; }

// Buckets: 4x the worst-case live chunks (capacity/32 resident chunks plus one
// partial tail chunk per chain), so the load factor stays <= 0.25 after a
// rebuild and rebuilds (triggered at 0.5 occupancy incl. dead buckets) are rare.
u64 bucket_count(u64 capacity, u64 agents) {
  u64 live = (capacity + kvg::kChunk - 1) / kvg::kChunk + agents + 2;
  return std::max<u64>(64, next_pow2(4 * live));
}

u64 max_context_pages(const kvg_population* p, u64 ps) {
  u64 best = 0;
  for (u32 a = 0; a < p->agents; ++a) {
    u64 c = p->prompt_tokens;
    for (u32 s = 0; s < p->steps; ++s) {
      const kvg_step_plan& sp = p->plans[static_cast<size_t>(a) * p->steps + s];
      c += sp.gen_tokens + sp.obs_tokens;
    }
    best = std::max(best, c);
  }
  return best / ps;
}

struct Region {
  u64 off = 0, stride = 0;
};

}  // namespace

struct kvg_batch {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evk = nullptr;
  kvg_batch_options opt{};
  size_t n = 0;
  std::vector<kvg_sim_desc> desc;
  std::vector<u32> nw;          // warps per sim
  std::vector<u64> buckets;     // per sim
  std::vector<u64> trace_cap, log_cap;
  std::vector<size_t> order;    // launch position -> user index
  std::vector<size_t> pos;      // user index -> launch position
  size_t n_small = 0;           // first n_small positions use the 32-thread kernel
  // device memory
  char* arena = nullptr;
  size_t arena_bytes = 0;
  u64 tables_off = 0, tables_bytes = 0;
  std::vector<u64> off_plans, off_table, off_alt, off_occ, off_altocc, off_agents, off_pend,
      off_paus, off_ready, off_batch, off_stats, off_trace, off_log, off_heap, off_rbits,
      off_rl1, off_pinh, off_hist;
  kvg::SimDev* d_sims = nullptr;
  kvg_sim_result* d_results = nullptr;
  u64* d_counts = nullptr;
  // host mirrors
  std::vector<kvg_sim_result> h_results;
  std::vector<u64> h_counts;
  bool fetched = false;
  double last_ms = 0, last_kernel_ms = 0;
  bool ran = false;

  ~kvg_batch() { release(); }

  void release() {
    if (arena) cudaFree(arena);
    if (d_sims) cudaFree(d_sims);
    if (d_results) cudaFree(d_results);
    if (d_counts) cudaFree(d_counts);
    arena = nullptr;
    d_sims = nullptr;
    d_results = nullptr;
    d_counts = nullptr;
  }
};

namespace {

kvg_status layout_and_upload(kvg_batch* b) {
  b->release();
  const size_t n = b->n;
  auto resize = [n](std::vector<u64>& v) { v.assign(n, 0); };
  resize(b->off_plans); resize(b->off_table); resize(b->off_alt); resize(b->off_occ);
  resize(b->off_altocc); resize(b->off_agents); resize(b->off_pend); resize(b->off_paus);
  resize(b->off_ready); resize(b->off_batch); resize(b->off_stats); resize(b->off_trace);
  resize(b->off_log); resize(b->off_heap); resize(b->off_rbits); resize(b->off_rl1);
  resize(b->off_pinh); resize(b->off_hist);
  // Region order: primary tables first so one memset initialises them all.
  u64 cur = 0;
  b->tables_off = 0;
  for (size_t p = 0; p < n; ++p) {
    size_t i = b->order[p];
    b->off_table[i] = cur;
    cur += align_up(b->buckets[i] * kvg::kChunk * sizeof(kvg::Slot));
  }
  b->tables_bytes = cur;
  for (size_t p = 0; p < n; ++p) {
    size_t i = b->order[p];
    const kvg_population* pop = b->desc[i].population;
    const u64 na = pop->agents;
    b->off_alt[i] = cur; cur += align_up(b->buckets[i] * kvg::kChunk * sizeof(kvg::Slot));
    b->off_occ[i] = cur; cur += align_up(b->buckets[i] * sizeof(u32));
    b->off_altocc[i] = cur; cur += align_up(b->buckets[i] * sizeof(u32));
    b->off_plans[i] = cur; cur += align_up(std::max<u64>(1, na * pop->steps) * sizeof(kvg_step_plan));
    b->off_agents[i] = cur; cur += align_up(std::max<u64>(1, na) * sizeof(kvg::AgentDev));
    b->off_pend[i] = cur; cur += align_up(std::max<u64>(1, na) * sizeof(u32));
    b->off_paus[i] = cur; cur += align_up(std::max<u64>(1, na) * sizeof(u32));
    b->off_ready[i] = cur; cur += align_up(std::max<u64>(1, na) * sizeof(u32));
    b->off_batch[i] = cur; cur += align_up(std::max<u64>(1, na) * sizeof(kvg::Member));
    b->off_stats[i] = cur; cur += align_up(std::max<u64>(1, na) * sizeof(kvg_agent_stats));
    b->off_trace[i] = cur; cur += align_up(std::max<u64>(1, b->trace_cap[i]) * sizeof(kvg_trace_row));
    b->off_log[i] = cur; cur += align_up(std::max<u64>(1, b->log_cap[i]) * sizeof(kvg_log_record));
    const u64 nwords = (na + 31) / 32;
    b->off_heap[i] = cur; cur += align_up(std::max<u64>(1, na) * sizeof(kvg::HeapEnt));
    b->off_rbits[i] = cur; cur += align_up(std::max<u64>(1, nwords) * sizeof(u32));
    b->off_rl1[i] = cur; cur += align_up(std::max<u64>(1, (nwords + 31) / 32) * sizeof(u32));
    const u64 sp = pop->shared_prompt ? pop->prompt_tokens / b->desc[i].engine.page_size : 0;
    b->off_pinh[i] = cur; cur += align_up((sp + 1) * sizeof(u32) + (sp / 32 + 1) * sizeof(u32));
    b->off_hist[i] = cur; cur += align_up(2 * 512 * sizeof(u32));
  }
  b->arena_bytes = cur;
  CUDA_TRY(cudaSetDevice(b->device));
  CUDA_TRY(cudaMalloc(&b->arena, b->arena_bytes));
  CUDA_TRY(cudaMalloc(&b->d_sims, n * sizeof(kvg::SimDev) + 1));
  CUDA_TRY(cudaMalloc(&b->d_results, n * sizeof(kvg_sim_result) + 1));
  CUDA_TRY(cudaMalloc(&b->d_counts, n * 3 * sizeof(u64) + 8));
  std::vector<kvg::SimDev> hs(n);
  for (size_t p = 0; p < n; ++p) {
    const size_t i = b->order[p];
    const kvg_sim_desc& d = b->desc[i];
    const kvg_population* pop = d.population;
    kvg::SimDev& s = hs[p];
    std::memset(&s, 0, sizeof s);
    char* base = b->arena;
    s.plans = reinterpret_cast<const kvg_step_plan*>(base + b->off_plans[i]);
    s.n_agents = pop->agents;
    s.n_steps = pop->steps;
    s.prompt_tokens = pop->prompt_tokens;
    s.shared_len = pop->shared_prompt_tokens;
    s.shared_pages = pop->shared_prompt ? pop->prompt_tokens / d.engine.page_size : 0;
    s.workload_hash = pop->stream_hash;
    s.policy = d.policy;
    s.cost = d.cost;
    s.engine = d.engine;
    s.table = reinterpret_cast<kvg::Slot*>(base + b->off_table[i]);
    s.alt = reinterpret_cast<kvg::Slot*>(base + b->off_alt[i]);
    s.occ = reinterpret_cast<u32*>(base + b->off_occ[i]);
    s.alt_occ = reinterpret_cast<u32*>(base + b->off_altocc[i]);
    s.bucket_mask = static_cast<u32>(b->buckets[i] - 1);
    s.agents = reinterpret_cast<kvg::AgentDev*>(base + b->off_agents[i]);
    s.pend = reinterpret_cast<u32*>(base + b->off_pend[i]);
    s.paus = reinterpret_cast<u32*>(base + b->off_paus[i]);
    s.ready = reinterpret_cast<u32*>(base + b->off_ready[i]);
    s.batch = reinterpret_cast<kvg::Member*>(base + b->off_batch[i]);
    s.heap = reinterpret_cast<kvg::HeapEnt*>(base + b->off_heap[i]);
    s.rbits = reinterpret_cast<u32*>(base + b->off_rbits[i]);
    s.rl1 = reinterpret_cast<u32*>(base + b->off_rl1[i]);
    s.pin_hist = reinterpret_cast<u32*>(base + b->off_pinh[i]);
    s.pin_lvl = s.pin_hist + (s.shared_pages + 1);
    s.hist = reinterpret_cast<u32*>(base + b->off_hist[i]);
    s.stats = reinterpret_cast<kvg_agent_stats*>(base + b->off_stats[i]);
    s.trace = reinterpret_cast<kvg_trace_row*>(base + b->off_trace[i]);
    s.trace_cap = b->trace_cap[i];
    s.log = b->log_cap[i] ? reinterpret_cast<kvg_log_record*>(base + b->off_log[i]) : nullptr;
    s.log_cap = b->log_cap[i];
    s.result = b->d_results + p;
    s.counts = b->d_counts + 3 * p;
    if (pop->agents > 0)
      CUDA_TRY(cudaMemcpyAsync(base + b->off_plans[i], pop->plans,
                               static_cast<size_t>(pop->agents) * pop->steps * sizeof(kvg_step_plan),
                               cudaMemcpyHostToDevice, b->stream));
  }
  CUDA_TRY(cudaMemcpyAsync(b->d_sims, hs.data(), n * sizeof(kvg::SimDev), cudaMemcpyHostToDevice,
                           b->stream));
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  return KVG_OK;
}

kvg_status launch(kvg_batch* b) {
  CUDA_TRY(cudaSetDevice(b->device));
  CUDA_TRY(cudaEventRecord(b->ev0, b->stream));
  CUDA_TRY(cudaMemsetAsync(b->arena + b->tables_off, 0xff, b->tables_bytes, b->stream));
  CUDA_TRY(cudaMemsetAsync(b->d_counts, 0, b->n * 3 * sizeof(u64), b->stream));
  CUDA_TRY(cudaEventRecord(b->evk, b->stream));
  if (b->n_small > 0)
    kvg::engine_kernel_small<<<static_cast<unsigned>(b->n_small), 32, 0, b->stream>>>(b->d_sims);
  // big sims: one launch per distinct warp count (positions are grouped)
  size_t p = b->n_small;
  while (p < b->n) {
    size_t q = p;
    const u32 w = b->nw[b->order[p]];
    while (q < b->n && b->nw[b->order[q]] == w) ++q;
    kvg::engine_kernel_big<<<static_cast<unsigned>(q - p), w * 32, 0, b->stream>>>(b->d_sims + p);
    p = q;
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(b->ev1, b->stream));
  CUDA_TRY(cudaEventSynchronize(b->ev1));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, b->ev0, b->ev1));
  b->last_ms = ms;
  CUDA_TRY(cudaEventElapsedTime(&ms, b->evk, b->ev1));
  b->last_kernel_ms = ms;
  return KVG_OK;
}

kvg_status fetch_scalars(kvg_batch* b) {
  if (b->fetched) return KVG_OK;
  b->h_results.resize(b->n);
  b->h_counts.resize(3 * b->n);
  CUDA_TRY(cudaMemcpy(b->h_results.data(), b->d_results, b->n * sizeof(kvg_sim_result),
                      cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(b->h_counts.data(), b->d_counts, b->n * 3 * sizeof(u64),
                      cudaMemcpyDeviceToHost));
  b->fetched = true;
  return KVG_OK;
}

}  // namespace

extern "C" {

KVG_API void kvg_batch_options_init(kvg_batch_options* o) {
  if (o == nullptr) return;
  o->warps_per_sim = 0;
  o->log_capacity = 0;
  o->trace_capacity = 0;
}

KVG_API kvg_status kvg_batch_create(int device, const kvg_sim_desc* sims, size_t n,
                                    const kvg_batch_options* opt, kvg_batch** out) {
  if (out == nullptr || (n > 0 && sims == nullptr))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  for (size_t i = 0; i < n; ++i) {
    std::string why;
    if (!kvg_host::validate_sim(sims[i], &why))
      return (kvg_status)set_error(KVG_ERR_CONFIG, "sim " + std::to_string(i) + ": " + why);
    const kvg_population* pop = sims[i].population;
    if (pop->agents >= (1u << kvg::kAgentBits))
      return (kvg_status)set_error(KVG_ERR_CONFIG, "sim " + std::to_string(i) +
                                                       ": more than 2^20-1 agents");
    if (pop->steps > 65535)
      return (kvg_status)set_error(KVG_ERR_CONFIG, "sim " + std::to_string(i) +
                                                       ": more than 65535 steps per agent");
    if (max_context_pages(pop, 1) >= (1ull << 32))
      return (kvg_status)set_error(KVG_ERR_CONFIG, "sim " + std::to_string(i) +
                                                       ": contexts beyond 2^32 tokens");
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return (kvg_status)set_error(KVG_ERR_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  if (device < 0 || device >= count) return (kvg_status)set_error(KVG_ERR_CONFIG, "bad device index");
  kvg_batch* b = new kvg_batch();
  b->device = device;
  if (opt) b->opt = *opt;
  else kvg_batch_options_init(&b->opt);
  b->n = n;
  b->desc.assign(sims, sims + n);
  b->nw.assign(n, 1);
  b->buckets.assign(n, 0);
  b->trace_cap.assign(n, 0);
  b->log_cap.assign(n, b->opt.log_capacity);
  for (size_t i = 0; i < n; ++i) {
    const kvg_population* pop = sims[i].population;
    b->buckets[i] = bucket_count(sims[i].engine.capacity, pop->agents);
    u32 w = b->opt.warps_per_sim;
    if (w == 0) {
      // throughput mode keeps thousands of small sims resident (1 warp each);
      // latency mode gives a lone big sim a full CTA for its page passes
      const u64 chunks = max_context_pages(pop, sims[i].engine.page_size) / kvg::kChunk + 1;
      w = n >= 296 ? 1 : static_cast<u32>(std::min<u64>(32, next_pow2((chunks + 3) / 4)));
    }
    b->nw[i] = std::max<u32>(1, std::min<u32>(32, w));
    b->trace_cap[i] = b->opt.trace_capacity ? b->opt.trace_capacity : 4096;
  }
  // launch order: small (1-warp) sims first, then big sims grouped by warps
  b->order.resize(n);
  for (size_t i = 0; i < n; ++i) b->order[i] = i;
  std::stable_sort(b->order.begin(), b->order.end(),
                   [&](size_t x, size_t y) { return b->nw[x] < b->nw[y]; });
  b->pos.resize(n);
  for (size_t p = 0; p < n; ++p) b->pos[b->order[p]] = p;
  b->n_small = 0;
  while (b->n_small < n && b->nw[b->order[b->n_small]] == 1) ++b->n_small;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&b->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&b->ev1);
  if (e == cudaSuccess) e = cudaEventCreate(&b->evk);
  if (e != cudaSuccess) {
    delete b;
    return (kvg_status)set_error(KVG_ERR_CUDA, cudaGetErrorString(e));
  }
  kvg_status st = layout_and_upload(b);
  if (st != KVG_OK) {
    delete b;
    return st;
  }
  *out = b;
  return KVG_OK;
}

KVG_API kvg_status kvg_batch_run(kvg_batch* b) {
  if (b == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null batch");
  for (int attempt = 0; attempt < 8; ++attempt) {
    b->fetched = false;
    kvg_status st = launch(b);
    if (st != KVG_OK) return st;
    st = fetch_scalars(b);
    if (st != KVG_OK) return st;
    // regrow outputs that overflowed and re-run (simulations are deterministic)
    bool grow = false;
    for (size_t i = 0; i < b->n; ++i) {
      const size_t p = b->pos[i];
      if (b->h_counts[3 * p] > b->trace_cap[i]) {
        b->trace_cap[i] = b->h_counts[3 * p] + 16;
        grow = true;
      }
    }
    if (!grow) break;
    st = layout_and_upload(b);
    if (st != KVG_OK) return st;
  }
  b->ran = true;
  bool horizon = false;
  for (size_t i = 0; i < b->n; ++i) {
    kvg_sim_result& r = b->h_results[b->pos[i]];
    if (r.status == KVG_ERR_STATE)
      return (kvg_status)set_error(KVG_ERR_STATE,
                                   "sim " + std::to_string(i) + ": device invariant violation, code " +
                                       std::to_string(b->h_counts[3 * b->pos[i] + 2]));
    if (r.status == KVG_ERR_HORIZON) horizon = true;
  }
  if (horizon) return (kvg_status)set_error(KVG_ERR_HORIZON, "a simulation exceeded its horizon");
  return KVG_OK;
}

KVG_API kvg_status kvg_batch_last_ms(const kvg_batch* b, double* ms) {
  if (b == nullptr || ms == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  *ms = b->last_ms;
  return KVG_OK;
}

KVG_API kvg_status kvg_batch_timing(const kvg_batch* b, double* step_ms, double* kernel_ms) {
  if (b == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null batch");
  if (step_ms) *step_ms = b->last_ms;
  if (kernel_ms) *kernel_ms = b->last_kernel_ms;
  return KVG_OK;
}

KVG_API kvg_status kvg_batch_result(kvg_batch* b, size_t i, kvg_sim_result* out) {
  if (b == nullptr || out == nullptr || i >= b->n)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "bad argument");
  if (!b->ran) return (kvg_status)set_error(KVG_ERR_STATE, "batch has not run");
  kvg_status st = fetch_scalars(b);
  if (st != KVG_OK) return st;
  *out = b->h_results[b->pos[i]];
  // phases (metrics.cpp:41-81) from the trace, like finish_result (engine.cpp:413)
  const u64 rows = std::min<u64>(b->h_counts[3 * b->pos[i]], b->trace_cap[i]);
  std::vector<kvg_trace_row> tr(rows);
  if (rows)
    CUDA_TRY(cudaMemcpy(tr.data(), b->arena + b->off_trace[i], rows * sizeof(kvg_trace_row),
                        cudaMemcpyDeviceToHost));
  size_t np = 0;
  kvg_classify_phases(tr.data(), rows, out->makespan, &b->desc[i].engine.phases, out->phases, 3,
                      &np);
  out->n_phases = static_cast<uint32_t>(np);
  return KVG_OK;
}

KVG_API kvg_status kvg_batch_trace(kvg_batch* b, size_t i, kvg_trace_row* rows, size_t cap,
                                   size_t* n_rows) {
  if (b == nullptr || i >= b->n) return (kvg_status)set_error(KVG_ERR_CONFIG, "bad argument");
  kvg_status st = fetch_scalars(b);
  if (st != KVG_OK) return st;
  const u64 total = std::min<u64>(b->h_counts[3 * b->pos[i]], b->trace_cap[i]);
  if (n_rows) *n_rows = total;
  const u64 k = std::min<u64>(total, cap);
  if (rows && k)
    CUDA_TRY(cudaMemcpy(rows, b->arena + b->off_trace[i], k * sizeof(kvg_trace_row),
                        cudaMemcpyDeviceToHost));
  return KVG_OK;
}

KVG_API kvg_status kvg_batch_agent_stats(kvg_batch* b, size_t i, kvg_agent_stats* out,
                                         size_t cap, size_t* n_agents) {
  if (b == nullptr || i >= b->n) return (kvg_status)set_error(KVG_ERR_CONFIG, "bad argument");
  const u64 na = b->desc[i].population->agents;
  if (n_agents) *n_agents = na;
  const u64 k = std::min<u64>(na, cap);
  if (out && k)
    CUDA_TRY(cudaMemcpy(out, b->arena + b->off_stats[i], k * sizeof(kvg_agent_stats),
                        cudaMemcpyDeviceToHost));
  return KVG_OK;
}

KVG_API kvg_status kvg_batch_log(kvg_batch* b, size_t i, kvg_log_record* out, size_t cap,
                                 size_t* n_records) {
  if (b == nullptr || i >= b->n) return (kvg_status)set_error(KVG_ERR_CONFIG, "bad argument");
  kvg_status st = fetch_scalars(b);
  if (st != KVG_OK) return st;
  const u64 total = b->h_counts[3 * b->pos[i] + 1];
  if (n_records) *n_records = total;
  const u64 k = std::min<u64>(std::min<u64>(total, b->log_cap[i]), cap);
  if (out && k) {
    CUDA_TRY(cudaMemcpy(out, b->arena + b->off_log[i], k * sizeof(kvg_log_record),
                        cudaMemcpyDeviceToHost));
    // victims are emitted by a parallel scatter: order each run of VICTIM
    // records as the reference evicts them (stamp asc, page index desc)
    size_t s = 0;
    while (s < k) {
      if (out[s].kind != KVG_LOG_VICTIM) { ++s; continue; }
      size_t e = s;
      while (e < k && out[e].kind == KVG_LOG_VICTIM) ++e;
      std::sort(out + s, out + e, [](const kvg_log_record& x, const kvg_log_record& y) {
        if (x.b != y.b) return x.b < y.b;
        return (x.a & 0xffffffffull) > (y.a & 0xffffffffull);
      });
      s = e;
    }
  }
  return KVG_OK;
}

KVG_API void kvg_batch_free(kvg_batch* b) {
  if (b == nullptr) return;
  cudaSetDevice(b->device);
  if (b->ev0) cudaEventDestroy(b->ev0);
  if (b->ev1) cudaEventDestroy(b->ev1);
  if (b->evk) cudaEventDestroy(b->evk);
  b->release();
  if (b->stream) cudaStreamDestroy(b->stream);
  delete b;
}

KVG_API kvg_status kvg_run_batch(int device, const kvg_sim_desc* sims, size_t n,
                                 kvg_sim_result* results) {
  kvg_batch* b = nullptr;
  kvg_status st = kvg_batch_create(device, sims, n, nullptr, &b);
  if (st != KVG_OK) return st;
  st = kvg_batch_run(b);
  if (st == KVG_OK || st == KVG_ERR_HORIZON) {
    for (size_t i = 0; i < n && results; ++i) {
      kvg_status s2 = kvg_batch_result(b, i, &results[i]);
      if (s2 != KVG_OK) {
        st = s2;
        break;
      }
    }
  }
  kvg_batch_free(b);
  return st;
}

}  // extern "C"

// ----------------------------------------------------------------- cache API

struct kvg_cache {
  int device = 0;
  u64 capacity = 0, page_size = 1, shared_pages = 0, buckets = 0;
  char* mem = nullptr;
  kvg::CacheDev h{};
  kvg::CacheDev* d = nullptr;
  kvg::CacheState* d_state = nullptr;
  kvg_victim* d_victims = nullptr;
  u64 victim_cap = 0;
  std::vector<kvg_victim> victims;  // host copy, sorted per op
  double hit_m = 0, hit_r = 0;
};

extern "C" {

KVG_API kvg_status kvg_cache_create(int device, uint64_t capacity, uint64_t page_size,
                                    uint32_t eviction, uint64_t prompt_tokens,
                                    uint32_t shared_prompt, uint32_t max_agents, kvg_cache** out) {
  if (out == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (capacity == 0 || page_size == 0)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "capacity and page size must be > 0");
  if (eviction != KVG_EVICT_DISCARD)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "offload eviction is not implemented on the device");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return (kvg_status)set_error(KVG_ERR_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  CUDA_TRY(cudaSetDevice(device));
  kvg_cache* c = new kvg_cache();
  c->device = device;
  c->capacity = capacity;
  c->page_size = page_size;
  c->shared_pages = shared_prompt ? prompt_tokens / page_size : 0;
  c->buckets = bucket_count(capacity, max_agents);
  const u64 tb = c->buckets * kvg::kChunk * sizeof(kvg::Slot);
  const u64 ob = align_up(c->buckets * sizeof(u32));
  c->victim_cap = 1 << 20;
  const u64 bytes = 2 * tb + 2 * ob + align_up(sizeof(kvg::CacheState)) +
                    align_up(sizeof(kvg::CacheDev)) + 2 * 512 * sizeof(u32) + 256;
  CUDA_TRY(cudaMalloc(&c->mem, bytes));
  CUDA_TRY(cudaMalloc(&c->d_victims, c->victim_cap * sizeof(kvg_victim)));
  CUDA_TRY(cudaMemset(c->mem, 0xff, 2 * tb));
  char* p = c->mem;
  c->h.capacity = capacity;
  c->h.page_size = page_size;
  c->h.shared_pages = c->shared_pages;
  c->h.table = reinterpret_cast<kvg::Slot*>(p);
  c->h.alt = reinterpret_cast<kvg::Slot*>(p + tb);
  c->h.occ = reinterpret_cast<u32*>(p + 2 * tb);
  c->h.alt_occ = reinterpret_cast<u32*>(p + 2 * tb + ob);
  c->d_state = reinterpret_cast<kvg::CacheState*>(p + 2 * tb + 2 * ob);
  c->d = reinterpret_cast<kvg::CacheDev*>(p + 2 * tb + 2 * ob + align_up(sizeof(kvg::CacheState)));
  static_assert(sizeof(kvg::CacheDev) % 8 == 0, "layout");
  c->h.bucket_mask = static_cast<u32>(c->buckets - 1);
  c->h.victims = c->d_victims;
  c->h.victim_cap = c->victim_cap;
  c->h.state = reinterpret_cast<u64*>(c->d_state);
  c->h.hist = reinterpret_cast<u32*>(p + 2 * tb + 2 * ob + align_up(sizeof(kvg::CacheState)) +
                                     align_up(sizeof(kvg::CacheDev)));
  CUDA_TRY(cudaMemset(c->d_state, 0, sizeof(kvg::CacheState)));
  *out = c;
  return KVG_OK;
}

KVG_API kvg_status kvg_cache_exec(kvg_cache* c, const kvg_cache_op* ops, size_t n,
                                  kvg_cache_op_result* results) {
  if (c == nullptr || (n > 0 && (ops == nullptr || results == nullptr)))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (n == 0) return KVG_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  kvg_cache_op* d_ops = nullptr;
  kvg_cache_op_result* d_res = nullptr;
  CUDA_TRY(cudaMalloc(&d_ops, n * sizeof(kvg_cache_op)));
  CUDA_TRY(cudaMalloc(&d_res, n * sizeof(kvg_cache_op_result)));
  CUDA_TRY(cudaMemcpy(d_ops, ops, n * sizeof(kvg_cache_op), cudaMemcpyHostToDevice));
  // victims of this call are appended after the ones already collected
  kvg::CacheState st{};
  CUDA_TRY(cudaMemcpy(&st, c->d_state, sizeof st, cudaMemcpyDeviceToHost));
  const u64 base = st.n_victims;
  kvg::CacheDev h = c->h;
  h.n_ops = static_cast<u32>(n);
  h.ops = d_ops;
  h.results = d_res;
  CUDA_TRY(cudaMemcpy(c->d, &h, sizeof h, cudaMemcpyHostToDevice));
  kvg::cache_kernel<<<1, 256>>>(c->d);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(results, d_res, n * sizeof(kvg_cache_op_result), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&st, c->d_state, sizeof st, cudaMemcpyDeviceToHost));
  cudaFree(d_ops);
  cudaFree(d_res);
  if (st.n_victims > c->victim_cap)
    return (kvg_status)set_error(KVG_ERR_STATE, "victim list overflow");
  c->victims.resize(st.n_victims);
  if (st.n_victims > base)
    CUDA_TRY(cudaMemcpy(c->victims.data() + base, c->d_victims + base,
                        (st.n_victims - base) * sizeof(kvg_victim), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) {
    auto b0 = c->victims.begin() + results[i].victims_begin;
    auto e0 = c->victims.begin() + results[i].victims_end;
    std::sort(b0, e0, [](const kvg_victim& x, const kvg_victim& y) {
      if (x.stamp != y.stamp) return x.stamp < y.stamp;
      return (x.key & 0xffffffffull) > (y.key & 0xffffffffull);
    });
  }
  c->hit_m = st.hit_m;
  c->hit_r = st.hit_r;
  return KVG_OK;
}

KVG_API kvg_status kvg_cache_victims(const kvg_cache* c, size_t begin, size_t end,
                                     kvg_victim* out) {
  if (c == nullptr || begin > end || end > c->victims.size())
    return (kvg_status)set_error(KVG_ERR_CONFIG, "bad victim range");
  if (out) std::copy(c->victims.begin() + begin, c->victims.begin() + end, out);
  return KVG_OK;
}

KVG_API kvg_status kvg_cache_hit_window(const kvg_cache* c, double* matched, double* requested) {
  if (c == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null cache");
  if (matched) *matched = c->hit_m;
  if (requested) *requested = c->hit_r;
  return KVG_OK;
}

KVG_API void kvg_cache_free(kvg_cache* c) {
  if (c == nullptr) return;
  cudaSetDevice(c->device);
  cudaFree(c->mem);
  cudaFree(c->d_victims);
  delete c;
}

}  // extern "C"
