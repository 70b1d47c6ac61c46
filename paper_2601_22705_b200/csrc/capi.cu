// C ABI of the B200 engine: batch lifecycle, HBM workspace layout, launches
// and result transfer (include/kvgpu.h). Host code only; kernels in engine.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "host_internal.h"
#include "kvg_device.h"

namespace kvg {
__global__ void engine_kernel_small(const SimDev* __restrict__ sims);
__global__ void engine_kernel_small_chain(const SimDev* __restrict__ sims);
__global__ void engine_kernel_small_off(const SimDev* __restrict__ sims);
__global__ void engine_kernel_big(const SimDev* __restrict__ sims);
__global__ void engine_kernel_lone(const SimDev* __restrict__ sims);
__global__ void engine_kernel_mid(const SimDev* __restrict__ sims);
__global__ void cache_kernel(const CacheDev* __restrict__ cd);
__global__ void pack_traces(const SimDev* __restrict__ sims, const u64* __restrict__ dst_off,
                            kvg_trace_row* __restrict__ packed);
}  // namespace kvg

using kvg::u32;
using kvg::u64;
using kvg_host::set_error;

namespace kvg_engine_cfg {  // engine.cu
cudaError_t check_ready_next(const unsigned* rbits, const unsigned* rl1, unsigned n,
                             const unsigned* from, unsigned nq, unsigned* out_narrow,
                             unsigned* out_wide);
}

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

// Offload-mode tree sizes (0 in discard mode): nodes partition the pages the
// tree holds (device or host), at most every agent's whole context.
u64 tree_nodes(const kvg_sim_desc& d) {
  if (d.engine.eviction != KVG_EVICT_OFFLOAD) return 0;
  const kvg_population* p = d.population;
  u64 pages = 0;
  for (u32 a = 0; a < p->agents; ++a) {
    u64 c = p->prompt_tokens;
    for (u32 s = 0; s < p->steps; ++s) {
      const kvg_step_plan& sp = p->plans[static_cast<size_t>(a) * p->steps + s];
      c += sp.gen_tokens + sp.obs_tokens;
    }
    pages += c / d.engine.page_size + 1;
  }
  return pages + 2;
}
u64 tree_hash_slots(u64 nodes) { return nodes ? next_pow2(4 * nodes) : 1; }
u64 xfer_ring(const kvg_sim_desc& d) {
  return d.engine.eviction == KVG_EVICT_OFFLOAD ? 4096 + 4ull * d.population->agents : 1;
}

// Dynamic shared memory holding a small simulation's hot agent records,
// event heap and ready bitmaps (leader.cuh engine_body); 0 = keep in HBM.
// The 1-warp kernel keeps up to 128 agents there (28 CTAs share an SM); the
// big-sim kernel runs one CTA per SM and keeps up to ~200 KB of them (2,048
// agents = 160 KB), so a lone C2 / C3 leader never leaves shared memory.
constexpr size_t kBigSmemMax = 200 * 1024;
// per agent: record 64 B + heap entry 16 B + completion-ring slot 4 B, and
// in the big kernel the chain-LRU links 8 B (leader.cuh smem_bytes_for);
// then the two-level ready bitmap
size_t hot_smem_bytes(u64 n, bool big) {
  const u64 nwords = (n + 31) / 32;
  return n * (sizeof(kvg::AgentDev) + sizeof(kvg::HeapEnt) + 4 + (big ? 8 : 0)) +
         (nwords + (nwords + 31) / 32) * 4;
}
size_t hot_smem(u64 n, bool big = false) {
  if (!big) return n > 128 ? 0 : hot_smem_bytes(n, false);
  const size_t b = hot_smem_bytes(n, true);
  if (b <= kBigSmemMax) return b;
  // too big as a whole: the ready bitmaps alone (leader.cuh engine_body)
  const u64 nwords = (n + 31) / 32;
  const size_t bm = (nwords + (nwords + 31) / 32) * 4;
  return bm <= kBigSmemMax ? bm : 0;
}

// Big-kernel offload sims also keep the tree's walk mirror (tree.cuh tw) in
// the shared memory the hot records leave free: node ids [0, k) for the
// largest k that fits (leader.cuh engine_body derives k the same way).
size_t big_smem(const kvg_sim_desc& d) {
  const size_t hot = hot_smem(d.population->agents, true);
  const u64 tn = tree_nodes(d);
  if (tn == 0) return hot;
  const size_t base = (hot + 15) / 16 * 16;
  const size_t room = kBigSmemMax > base ? kBigSmemMax - base : 0;
  return base + std::min<size_t>(room / kvg::kTWalkSmemBytes, tn) * kvg::kTWalkSmemBytes;
}

}  // namespace

#include "capi_batch.inc"

// ----------------------------------------------------------------- cache API

namespace kvg_tree_seam {  // engine.cu
size_t state_bytes();
cudaError_t init(void* d_state, const kvg::SimDev& sim, unsigned long long capacity,
                 unsigned long long page_size, unsigned long long shared_pages);
cudaError_t exec(void* d_state, const kvg_cache_op* d_ops, unsigned n, kvg_cache_op_result* d_res,
                 kvg_victim* d_vic, unsigned long long vic_cap, unsigned long long* d_nvic);
cudaError_t hit_window(const void* d_state, double* m, double* r);
}  // namespace kvg_tree_seam

namespace kvg_grid_seam {  // engine.cu
unsigned match_blocks(int dev);
unsigned evict_blocks(int dev, unsigned occ_n);
cudaError_t match(const kvg::GridMatchArgs& a, unsigned blocks, cudaStream_t s);
cudaError_t evict(const kvg::GridEvictArgs& a, unsigned blocks, cudaStream_t s);
}  // namespace kvg_grid_seam

struct kvg_cache {
  int device = 0;
  bool offload = false;
  void* tree_state = nullptr;      // offload: kvg::TreeCacheDev (engine.cu)
  unsigned long long* d_nvic = nullptr;
  u64 capacity = 0, page_size = 1, shared_pages = 0, buckets = 0;
  char* mem = nullptr;
  kvg::CacheDev h{};
  kvg::CacheDev* d = nullptr;
  kvg::CacheState* d_state = nullptr;
  kvg_victim* d_victims = nullptr;
  u64 victim_cap = 0;
  std::vector<kvg_victim> victims;  // host copy, sorted per op
  double hit_m = 0, hit_r = 0;
  // grid-wide kernels (grid.cuh): scratch, routing mode, last device time
  uint32_t grid_mode = KVG_GRID_AUTO;
  uint32_t record_victims = 1;
  char* gscratch = nullptr;  // [ghist 3*2*2048 u32 | freed | err | work | pad]
  u32* d_best = nullptr;     // [shared_pages + 1]
  char* gq = nullptr;        // match-batch query arrays
  size_t gq_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0;
  unsigned last_blocks = 0;
};

namespace {

constexpr size_t kGHistBytes = 3 * 2 * kvg::kGridBins * sizeof(u32);
constexpr u64 kGridAutoBuckets = 4096;  // claimed buckets from which EVICT goes grid-wide

kvg_status cache_state(kvg_cache* c, kvg::CacheState* st) {
  CUDA_TRY(cudaMemcpy(st, c->d_state, sizeof *st, cudaMemcpyDeviceToHost));
  return KVG_OK;
}

// evict(k) as one cooperative launch over every SM (grid_evict_kernel).
kvg_status grid_evict(kvg_cache* c, const kvg_cache_op& o, kvg_cache_op_result* r) {
  kvg::CacheState st{};
  kvg_status rc = cache_state(c, &st);
  if (rc != KVG_OK) return rc;
  const u64 k = o.arg, e = st.used - st.pinned_pages;
  *r = kvg_cache_op_result{};
  r->status = KVG_OK;
  r->clock = st.clock;
  r->used = st.used;
  r->victims_begin = r->victims_end = st.n_victims;
  if (k == 0 || e == 0) return KVG_OK;  // cache_tree.cpp:272 (and nothing evictable)
  const bool sw = st.swapped & 1;
  kvg::GridEvictArgs a{};
  a.table = sw ? c->h.alt : c->h.table;
  a.summ = sw ? c->h.alt_summ : c->h.summ;
  a.occ = sw ? c->h.alt_occ : c->h.occ;
  a.occ_n = static_cast<u32>(st.occ_n);
  a.mask = c->h.bucket_mask;
  a.S = c->shared_pages;
  a.k = k;
  a.evictable = e;
  a.clock = st.clock;
  a.vic = c->record_victims ? c->d_victims : nullptr;
  a.vic_cap = c->victim_cap;
  a.vic_n = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<char*>(c->d_state) + offsetof(kvg::CacheState, n_victims));
  a.ghist = reinterpret_cast<u32*>(c->gscratch);
  a.freed = reinterpret_cast<unsigned int*>(c->gscratch + kGHistBytes);
  a.err = reinterpret_cast<int*>(c->gscratch + kGHistBytes + 4);
  CUDA_TRY(cudaMemset(c->gscratch, 0, kGHistBytes + 8));
  c->last_blocks = kvg_grid_seam::evict_blocks(c->device, a.occ_n);
  CUDA_TRY(cudaEventRecord(c->ev0));
  CUDA_TRY(kvg_grid_seam::evict(a, c->last_blocks, 0));
  CUDA_TRY(cudaEventRecord(c->ev1));
  CUDA_TRY(cudaEventSynchronize(c->ev1));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->last_ms += ms;
  unsigned int freed = 0;
  int err = 0;
  CUDA_TRY(cudaMemcpy(&freed, a.freed, 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&err, a.err, 4, cudaMemcpyDeviceToHost));
  st.used -= freed;
  st.discarded += static_cast<u64>(freed) * c->page_size;
  kvg::CacheState cur{};
  rc = cache_state(c, &cur);  // n_victims advanced on the device
  if (rc != KVG_OK) return rc;
  st.n_victims = cur.n_victims;
  CUDA_TRY(cudaMemcpy(c->d_state, &st, sizeof st, cudaMemcpyHostToDevice));
  if (st.n_victims > c->victim_cap)
    return (kvg_status)set_error(KVG_ERR_STATE, "victim list overflow");
  const u64 base = r->victims_begin;
  c->victims.resize(st.n_victims);
  if (st.n_victims > base)
    CUDA_TRY(cudaMemcpy(c->victims.data() + base, c->d_victims + base,
                        (st.n_victims - base) * sizeof(kvg_victim), cudaMemcpyDeviceToHost));
  r->status = err ? KVG_ERR_STATE : KVG_OK;
  r->r0 = freed;
  r->used = st.used;
  r->victims_end = st.n_victims;
  return KVG_OK;
}

}  // namespace

namespace {

// Victims of one op in the reference's eviction order: stamp ascending, the
// deeper page of equal stamps first (cache_tree.cpp:270-319).
void sort_victims(kvg_cache* c, const kvg_cache_op_result& r) {
  if (r.victims_end > c->victims.size() || r.victims_begin >= r.victims_end) return;
  std::sort(c->victims.begin() + r.victims_begin, c->victims.begin() + r.victims_end,
            [](const kvg_victim& x, const kvg_victim& y) {
              if (x.stamp != y.stamp) return x.stamp < y.stamp;
              return (x.key & 0xffffffffull) > (y.key & 0xffffffffull);
            });
}

bool use_grid_evict(kvg_cache* c) {
  if (c->grid_mode == KVG_GRID_NEVER) return false;
  if (c->grid_mode == KVG_GRID_ALWAYS) return true;
  kvg::CacheState st{};
  if (cache_state(c, &st) != KVG_OK) return false;
  return st.occ_n >= kGridAutoBuckets;
}

// ops executed in order by the one-CTA executor (cache.cuh).
kvg_status exec_cta(kvg_cache* c, const kvg_cache_op* ops, size_t n,
                    kvg_cache_op_result* results) {
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
  if (!c->record_victims) h.victims = nullptr;
  h.n_ops = static_cast<u32>(n);
  h.ops = d_ops;
  h.results = d_res;
  CUDA_TRY(cudaMemcpy(c->d, &h, sizeof h, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaEventRecord(c->ev0));
  kvg::cache_kernel<<<1, 256>>>(c->d);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(c->ev1));
  CUDA_TRY(cudaEventSynchronize(c->ev1));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->last_ms += ms;
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
  for (size_t i = 0; i < n; ++i) sort_victims(c, results[i]);
  return KVG_OK;
}


}  // namespace

extern "C" {

KVG_API kvg_status kvg_cache_create(int device, uint64_t capacity, uint64_t page_size,
                                    uint32_t eviction, uint64_t prompt_tokens,
                                    uint32_t shared_prompt, uint32_t max_agents, kvg_cache** out) {
  if (out == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (capacity == 0 || page_size == 0)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "capacity and page size must be > 0");
  if (eviction != KVG_EVICT_DISCARD && eviction != KVG_EVICT_OFFLOAD)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "unknown eviction mode");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return (kvg_status)set_error(KVG_ERR_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  CUDA_TRY(cudaSetDevice(device));
  kvg_cache* c = new kvg_cache();
  c->device = device;
  c->capacity = capacity;
  c->page_size = page_size;
  c->shared_pages = shared_prompt ? prompt_tokens / page_size : 0;
  if (eviction == KVG_EVICT_OFFLOAD) {  // node-level tree (tree.cuh), leader-serial seam
    c->offload = true;
    c->victim_cap = 1 << 20;
    // nodes partition the pages the tree holds; host pages are not bounded by
    // the capacity, so size for 64 x capacity plus 4096 pages per agent
    const u64 tcap = 64 * capacity + 4096ull * std::max<u32>(1, max_agents) + 2;
    const u64 hslots = next_pow2(4 * tcap);
    const u64 logcap = 2 * capacity + 64;
    const u64 bytes = align_up(kvg_tree_seam::state_bytes()) + align_up(tcap * sizeof(kvg::TNodeDev)) +
                      align_up(tcap * sizeof(kvg::TWalk)) + 2 * align_up(tcap * 4) +
                      align_up(tcap * sizeof(kvg::FrEnt)) +
                      align_up(hslots * 8) + align_up(hslots * 4) +
                      align_up(logcap * sizeof(kvg_log_record)) + 256;
    CUDA_TRY(cudaMalloc(&c->mem, bytes));
    CUDA_TRY(cudaMalloc(&c->d_victims, c->victim_cap * sizeof(kvg_victim) + 64));
    c->d_nvic = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(c->d_victims) + c->victim_cap * sizeof(kvg_victim));
    CUDA_TRY(cudaMemset(c->d_nvic, 0, 8));
    char* p = c->mem;
    c->tree_state = p;
    p += align_up(kvg_tree_seam::state_bytes());
    kvg::SimDev sim;
    std::memset(&sim, 0, sizeof sim);
    sim.tnodes = reinterpret_cast<kvg::TNodeDev*>(p);
    p += align_up(tcap * sizeof(kvg::TNodeDev));
    sim.twalk = reinterpret_cast<kvg::TWalk*>(p);
    p += align_up(tcap * sizeof(kvg::TWalk));
    sim.tfree = reinterpret_cast<u32*>(p);
    p += align_up(tcap * 4);
    sim.tstack = reinterpret_cast<u32*>(p);
    p += align_up(tcap * 4);
    sim.fr = reinterpret_cast<kvg::FrEnt*>(p);
    p += align_up(tcap * sizeof(kvg::FrEnt));
    sim.hkeys = reinterpret_cast<u64*>(p);
    CUDA_TRY(cudaMemset(p, 0xff, hslots * 8));
    p += align_up(hslots * 8);
    sim.hvals = reinterpret_cast<u32*>(p);
    p += align_up(hslots * 4);
    sim.log = reinterpret_cast<kvg_log_record*>(p);
    sim.log_cap = logcap;
    sim.tcap = static_cast<u32>(tcap);
    sim.hmask = static_cast<u32>(hslots - 1);
    sim.shared_pages = c->shared_pages;
    CUDA_TRY(kvg_tree_seam::init(c->tree_state, sim, capacity, page_size, c->shared_pages));
    *out = c;
    return KVG_OK;
  }
  c->buckets = bucket_count(capacity, max_agents);
  const u64 tb = c->buckets * kvg::kChunk * sizeof(kvg::Slot);
  const u64 ob = align_up(c->buckets * sizeof(u32));
  c->victim_cap = 1 << 20;
  const u64 sb = align_up(c->buckets * sizeof(kvg::Summ));
  const u64 bytes = 2 * tb + 2 * ob + align_up(sizeof(kvg::CacheState)) +
                    align_up(sizeof(kvg::CacheDev)) + align_up(2 * 512 * sizeof(u32)) + 2 * sb + 256;
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
  char* sp = p + 2 * tb + 2 * ob + align_up(sizeof(kvg::CacheState)) +
             align_up(sizeof(kvg::CacheDev)) + align_up(2 * 512 * sizeof(u32));
  c->h.summ = reinterpret_cast<kvg::Summ*>(sp);
  c->h.alt_summ = reinterpret_cast<kvg::Summ*>(sp + sb);
  CUDA_TRY(cudaMemset(c->d_state, 0, sizeof(kvg::CacheState)));
  CUDA_TRY(cudaMalloc(&c->gscratch, kGHistBytes + 64));
  CUDA_TRY(cudaMalloc(&c->d_best, (c->shared_pages + 1) * sizeof(u32)));
  CUDA_TRY(cudaEventCreate(&c->ev0));
  CUDA_TRY(cudaEventCreate(&c->ev1));
  *out = c;
  return KVG_OK;
}

KVG_API kvg_status kvg_cache_exec(kvg_cache* c, const kvg_cache_op* ops, size_t n,
                                  kvg_cache_op_result* results) {
  if (c == nullptr || (n > 0 && (ops == nullptr || results == nullptr)))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (n == 0) return KVG_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->offload) {  // node-level tree: victims already in eviction order
    kvg_cache_op* d_ops = nullptr;
    kvg_cache_op_result* d_res = nullptr;
    CUDA_TRY(cudaMalloc(&d_ops, n * sizeof(kvg_cache_op)));
    CUDA_TRY(cudaMalloc(&d_res, n * sizeof(kvg_cache_op_result)));
    CUDA_TRY(cudaMemcpy(d_ops, ops, n * sizeof(kvg_cache_op), cudaMemcpyHostToDevice));
    unsigned long long base = 0, nv = 0;
    CUDA_TRY(cudaMemcpy(&base, c->d_nvic, 8, cudaMemcpyDeviceToHost));
    CUDA_TRY(kvg_tree_seam::exec(c->tree_state, d_ops, static_cast<unsigned>(n), d_res,
                                 c->d_victims, c->victim_cap, c->d_nvic));
    CUDA_TRY(cudaMemcpy(results, d_res, n * sizeof(kvg_cache_op_result), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(&nv, c->d_nvic, 8, cudaMemcpyDeviceToHost));
    cudaFree(d_ops);
    cudaFree(d_res);
    if (nv > c->victim_cap) return (kvg_status)set_error(KVG_ERR_STATE, "victim list overflow");
    c->victims.resize(nv);
    if (nv > base)
      CUDA_TRY(cudaMemcpy(c->victims.data() + base, c->d_victims + base,
                          (nv - base) * sizeof(kvg_victim), cudaMemcpyDeviceToHost));
    CUDA_TRY(kvg_tree_seam::hit_window(c->tree_state, &c->hit_m, &c->hit_r));
    return KVG_OK;
  }
  c->last_ms = 0;
  // EVICT ops on a big table run grid-wide (grid.cuh); everything between
  // them runs on the one-CTA op executor, in order
  size_t i = 0;
  while (i < n) {
    size_t j = i;
    while (j < n && !(ops[j].kind == KVG_OP_EVICT && use_grid_evict(c))) ++j;
    if (j > i) {
      const kvg_status rc = exec_cta(c, ops + i, j - i, results + i);
      if (rc != KVG_OK) return rc;
    }
    if (j < n) {
      const kvg_status rc = grid_evict(c, ops[j], results + j);
      if (rc != KVG_OK) return rc;
      sort_victims(c, results[j]);
      ++j;
    }
    i = j;
  }
  kvg::CacheState st{};
  const kvg_status rc = cache_state(c, &st);
  if (rc != KVG_OK) return rc;
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

KVG_API kvg_status kvg_cache_configure(kvg_cache* c, uint32_t grid_mode,
                                       uint32_t record_victims) {
  if (c == nullptr || grid_mode > KVG_GRID_ALWAYS)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "bad cache configuration");
  c->grid_mode = grid_mode;
  c->record_victims = record_victims ? 1u : 0u;
  return KVG_OK;
}

KVG_API kvg_status kvg_cache_last_ms(const kvg_cache* c, double* ms, uint32_t* grid_blocks) {
  if (c == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null cache");
  if (ms) *ms = c->last_ms;
  if (grid_blocks) *grid_blocks = c->last_blocks;
  return KVG_OK;
}

KVG_API kvg_status kvg_cache_match_batch(kvg_cache* c, const uint32_t* agents,
                                         const uint64_t* lens, size_t n,
                                         kvg_cache_op_result* results) {
  if (c == nullptr || (n > 0 && (agents == nullptr || lens == nullptr || results == nullptr)))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (c->offload)
    return (kvg_status)set_error(KVG_ERR_CONFIG,
                                 "match_batch: discard-mode caches only (offload matches "
                                 "split nodes, kvg_cache_exec)");
  CUDA_TRY(cudaSetDevice(c->device));
  c->last_ms = 0;
  const u64 S = c->shared_pages, ps = c->page_size;
  size_t i = 0;
  while (i < n) {
    // one sub-batch: no agent twice, so a private chunk has a single writer
    std::unordered_map<u32, char> seen;
    size_t j = i;
    while (j < n && seen.emplace(agents[j], 0).second) ++j;
    const size_t m = j - i;
    u64 max_groups = 0, n_items = 0;
    for (size_t k = 0; k < m; ++k) {
      const u64 np = lens[i + k] / ps;
      if (np > S) {
        const u64 g = (((np - 1) >> 5) - (S >> 5)) / kvg::kGridItemChunks + 1;
        max_groups = std::max<u64>(max_groups, g);
        n_items += g - 1;
      }
    }
    if (n_items >= (1ull << 32))
      return (kvg_status)set_error(KVG_ERR_CONFIG, "match_batch: too many chunk groups");
    const size_t words = S / 32 + 1;
    const size_t need = 16 * (n_items + 1) + m * (8 + 4 + 4 + 4) + words * 4 + 256;
    if (need > c->gq_cap) {
      cudaFree(c->gq);
      c->gq = nullptr;
      c->gq_cap = 0;
      CUDA_TRY(cudaMalloc(&c->gq, need));
      c->gq_cap = need;
    }
    char* p = c->gq;
    ulonglong2* d_items = reinterpret_cast<ulonglong2*>(p);  // 16 B aligned (cudaMalloc)
    u64* d_lens = reinterpret_cast<u64*>(d_items + n_items + 1);
    u32* d_agents = reinterpret_cast<u32*>(d_lens + m);
    u32* d_fm = d_agents + m;
    u32* d_res = d_fm + m;
    u32* d_smask = d_res + m;
    unsigned int* d_ncont = d_smask + words;
    kvg::CacheState st{};
    kvg_status rc = cache_state(c, &st);
    if (rc != KVG_OK) return rc;
    CUDA_TRY(cudaMemcpy(d_lens, lens + i, m * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d_agents, agents + i, m * 4, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemset(d_ncont, 0, 4));
    CUDA_TRY(cudaMemset(d_fm, 0xff, m * 4));
    CUDA_TRY(cudaMemset(d_res, 0, m * 4));
    CUDA_TRY(cudaMemset(d_smask, 0, words * 4));
    CUDA_TRY(cudaMemset(c->d_best, 0, (S + 1) * sizeof(u32)));
    const bool sw = st.swapped & 1;
    kvg::GridMatchArgs a{};
    a.table = sw ? c->h.alt : c->h.table;
    a.summ = sw ? c->h.alt_summ : c->h.summ;
    a.mask = c->h.bucket_mask;
    a.n = static_cast<u32>(m);
    a.S = S;
    a.ps = ps;
    a.clock0 = st.clock;
    a.agents = d_agents;
    a.lens = d_lens;
    a.max_groups = static_cast<u32>(max_groups);
    a.items = d_items;
    a.n_items = d_ncont;
    a.fm = d_fm;
    a.res = d_res;
    a.smask = d_smask;
    a.best = c->d_best;
    const unsigned blocks = kvg_grid_seam::match_blocks(c->device);
    CUDA_TRY(cudaEventRecord(c->ev0));
    CUDA_TRY(kvg_grid_seam::match(a, blocks, 0));
    CUDA_TRY(cudaEventRecord(c->ev1));
    CUDA_TRY(cudaEventSynchronize(c->ev1));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->last_ms += ms;
    std::vector<u32> fm(m), res(m), smask(words);
    CUDA_TRY(cudaMemcpy(fm.data(), d_fm, m * 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(res.data(), d_res, m * 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(smask.data(), d_smask, words * 4, cudaMemcpyDeviceToHost));
    // shared part: first non-resident shared page and resident pages below p
    u64 f_sh = S;
    for (u64 p0 = 0; p0 < S; p0 += 32) {
      const u32 lim = S - p0 >= 32 ? 0xffffffffu : ((1u << (S - p0)) - 1u);
      const u32 miss = ~smask[p0 / 32] & lim;
      if (miss) {
        f_sh = p0 + __builtin_ctz(miss);
        break;
      }
    }
    std::vector<u64> pre(words + 1, 0);
    for (size_t w = 0; w < words; ++w) pre[w + 1] = pre[w] + __builtin_popcount(smask[w]);
    auto res_below = [&](u64 p) -> u64 {  // resident shared pages in [0, p)
      const u64 w = p / 32, r = p % 32;
      return pre[w] + (r ? __builtin_popcount(smask[w] & ((1u << r) - 1u)) : 0);
    };
    // results and the hit window in call order (cache_tree.cpp:139-140)
    for (size_t k = 0; k < m; ++k) {
      const u64 np = lens[i + k] / ps;
      const u64 sh = np < S ? np : S;
      u64 f = np;
      if (f_sh < sh) f = f_sh;
      if (fm[k] != 0xffffffffu && fm[k] < f) f = fm[k];
      const u64 resident = res_below(sh) + res[k];
      const u64 matched = f * ps;
      st.hit_m += static_cast<double>(matched);
      st.hit_r += static_cast<double>(lens[i + k]);
      kvg_cache_op_result& r = results[i + k];
      r = kvg_cache_op_result{};
      r.status = resident == f ? KVG_OK : KVG_ERR_STATE;
      r.r0 = matched;
      r.clock = st.clock + k + 1;
      r.used = st.used;
      r.victims_begin = r.victims_end = st.n_victims;
    }
    st.clock += m;
    CUDA_TRY(cudaMemcpy(c->d_state, &st, sizeof st, cudaMemcpyHostToDevice));
    c->hit_m = st.hit_m;
    c->hit_r = st.hit_r;
    i = j;
  }
  return KVG_OK;
}

KVG_API void kvg_cache_free(kvg_cache* c) {
  if (c == nullptr) return;
  cudaSetDevice(c->device);
  cudaFree(c->mem);
  cudaFree(c->d_victims);
  cudaFree(c->gscratch);
  cudaFree(c->d_best);
  cudaFree(c->gq);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  delete c;
}

}  // extern "C"

extern "C" {
KVG_API kvg_status kvg_check_ready_next(int device, const uint32_t* rbits, const uint32_t* rl1,
                                        uint32_t n, const uint32_t* from, uint32_t nq,
                                        uint32_t* out_narrow, uint32_t* out_wide) {
  if (rbits == nullptr || rl1 == nullptr || from == nullptr || out_narrow == nullptr ||
      out_wide == nullptr || n == 0)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  const size_t nw = (n + 31) / 32, n1 = (nw + 31) / 32;
  unsigned *d = nullptr;
  const size_t words = nw + n1 + 3 * static_cast<size_t>(nq) + 4;
  CUDA_TRY(cudaMalloc(&d, words * 4));
  unsigned* d_rb = d;
  unsigned* d_r1 = d + ((nw + 3) & ~size_t(3));  // 16 B aligned, as in the engine's layouts
  unsigned* d_from = d_r1 + n1;
  unsigned* d_on = d_from + nq;
  unsigned* d_ow = d_on + nq;
  cudaError_t e = cudaMemcpy(d_rb, rbits, nw * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_r1, rl1, n1 * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_from, from, size_t(nq) * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = kvg_engine_cfg::check_ready_next(d_rb, d_r1, n, d_from, nq, d_on, d_ow);
  if (e == cudaSuccess) e = cudaMemcpy(out_narrow, d_on, size_t(nq) * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(out_wide, d_ow, size_t(nq) * 4, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return (kvg_status)set_error(KVG_ERR_CUDA, cudaGetErrorString(e));
  return KVG_OK;
}
}
