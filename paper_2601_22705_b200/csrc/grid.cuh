// Grid-wide page-table kernels for the CacheTree seam (discard mode): the
// bandwidth form of kernels 1 and 2 on C2 / C5-size tables, where one CTA per
// operation (cache_kernel) cannot pull more than a single SM's share of HBM.
//
//  * grid_match_prep_kernel / grid_match_kernel / grid_match_rest_kernel /
//    grid_match_shared_kernel — a BATCH of match_prefix calls
//    (cache_tree.cpp:114-142) that leaves the table exactly as the same calls
//    issued one by one: query i runs at clock0 + i + 1, every resident page a
//    query's range covers is refreshed, so a page's final stamp is the clock
//    of the LAST query covering it (residency never changes inside a match
//    batch). The shared prompt, common to every query, is probed once (prep);
//    each query's first group of 8 private chunks is probed by one warp (all 8
//    bucket loads in flight) and refreshed in place — the host splits batches
//    so an agent appears at most once, making a private chunk single-writer;
//    the remaining groups of queries whose first group was fully resident are
//    flattened over (query, group) across all warps (rest); shared-prompt
//    pages get max{i : query i covers p} through one atomicMax per query and a
//    suffix max, and are rewritten by one small CTA (shared).
//  * grid_evict_kernel — evict(needed) (cache_tree.cpp:270-319, per-page form
//    SURVEY.md A.2) as ONE cooperative launch over every SM: the radix select
//    of coop_evict with 11-bit digits, per-CTA shared-memory histograms
//    (warp-aggregated atomics) merged into a small global histogram once per
//    pass, a grid barrier per pass, then the scatter-free pass. Same victims,
//    same order after the host's per-op sort.
#pragma once

#include <cooperative_groups.h>

namespace kvg {

#ifndef KVG_GRID_MATCH_WARPS
#define KVG_GRID_MATCH_WARPS 8
#endif
constexpr int kGridMatchWarps = KVG_GRID_MATCH_WARPS;
#ifndef KVG_GM_TMA  // bucket loads of the batched lookup as bulk async copies to shared memory
#define KVG_GM_TMA 1   // measured on the C5-size table: 0.29 ms (register form) -> 0.25 ms
#endif
#ifndef KVG_GM_MINB  // resident grid-match CTAs per SM the register budget allows
#define KVG_GM_MINB 4  // measured 3 (71 registers) / 4 / 5 / 6: C5 lookup 0.425 / 0.323 / 0.328 / 0.353 ms
#endif

#ifdef KVG_GRID_PROF  // dev-only phase timestamps of CTA 0 (tools/probe_grid.py)
__device__ unsigned long long g_gprof[32];
__device__ __forceinline__ void gprof(int k) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gprof[k] = t;
  }
}
#else
__device__ __forceinline__ void gprof(int) {}
#endif

// Shared prompt, probed ONCE per batch (every query's range starts with the
// same shared chunks): smask[c] = resident pages of shared chunk c.
__global__ void __launch_bounds__(1024) grid_match_prep_kernel(GridMatchArgs A) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const u64 chunks = (A.S + 31) / 32;
  for (u64 c = warp; c < chunks; c += nw) {
    const u64 tag = c * 32;  // owner 0
    u32 b = static_cast<u32>(hash64(tag)) & A.mask;
    bool found = false;
    Slot s{kEmptyKey, 0};
    for (;;) {
      s = ld_slot(&A.table[(size_t)b * kChunk + lane]);
      const u64 k0 = __shfl_sync(FULL, s.key, 0);
      if (k0 == tag) { found = true; break; }
      if (k0 == kEmptyKey) break;
      b = (b + 1) & A.mask;
    }
    const bool res = found && (s.meta & kResident) && tag + lane < A.S;
    const u32 m = __ballot_sync(FULL, res);
    if (lane == 0) A.smask[c] = m;
  }
}

// Probes chunk group g (kGridItemChunks chunks, all in flight) of query i's
// private range [S, len/ps), refreshes its resident pages to the query's
// clock (a private chunk has one writer per batch: the host splits batches so
// an agent appears once) and folds first miss / resident count into the
// query's accumulators. Returns true when the group had no miss.
__device__ __forceinline__ bool match_group(const GridMatchArgs& A, u32 i, u64 n, u64 g,
                                            int lane) {
  const u64 owner = (static_cast<u64>(A.agents[i]) + 1) << 32;
  const u64 c0 = (A.S >> 5) + g * kGridItemChunks;
  const u64 stamp = A.clock0 + i + 1;
  // every probe of the group in flight: one coalesced 512 B bucket load each
  u32 b[kGridItemChunks];
  Slot sl[kGridItemChunks];
  u32 pend = 0, fnd = 0;  // (warp-uniform) chunks still probing / found
#pragma unroll
  for (int j = 0; j < kGridItemChunks; ++j) {
    const u64 c = c0 + j;
    b[j] = 0;
    sl[j] = Slot{kEmptyKey, 0};
    if (c * 32 < n) {
      b[j] = static_cast<u32>(hash64(owner | (c * 32))) & A.mask;
      sl[j] = ld_slot(&A.table[(size_t)b[j] * kChunk + lane]);
      pend |= 1u << j;
    }
  }
  // linear-probe continuations of every colliding chunk in flight together:
  // one memory round trip per probe step of the group, not per collision
  for (;;) {
    u32 more = 0;
#pragma unroll
    for (int j = 0; j < kGridItemChunks; ++j) {
      if (!((pend >> j) & 1u)) continue;
      const u64 tag = owner | ((c0 + j) * 32);
      const u64 k0 = __shfl_sync(FULL, sl[j].key, 0);
      if (k0 == tag) {
        fnd |= 1u << j;
      } else if (k0 != kEmptyKey) {
        b[j] = (b[j] + 1) & A.mask;
        more |= 1u << j;
      }
    }
    if (!more) break;
#pragma unroll
    for (int j = 0; j < kGridItemChunks; ++j)
      if ((more >> j) & 1u) sl[j] = ld_slot(&A.table[(size_t)b[j] * kChunk + lane]);
    pend = more;
  }
  u32 miss = NIL32, res = 0;
#pragma unroll
  for (int j = 0; j < kGridItemChunks; ++j) {
    const u64 c = c0 + j;
    if (c * 32 >= n) break;  // warp-uniform
    const Slot cur = sl[j];
    const u32 cb = b[j];
    const bool found = (fnd >> j) & 1u;
    const u64 page = c * 32 + lane;
    const bool in = page >= A.S && page < n;
    const bool r = found && in && (cur.meta & kResident);
    if (in && !r && page < miss) miss = static_cast<u32>(page);
    res += r;
    if (__any_sync(FULL, r)) {  // refresh: every resident page in range takes the stamp
      const u64 nm = r ? m_make(stamp, m_pins(cur.meta)) : cur.meta;
      if (r) st_meta(&A.table[(size_t)cb * kChunk + lane], nm);
      summ_write(A.summ, cb, nm, lane);
    }
  }
  miss = __reduce_min_sync(FULL, miss);
  res = __reduce_add_sync(FULL, res);
  if (lane == 0) {
    if (miss != NIL32) atomicMin(&A.fm[i], miss);
    if (res) atomicAdd(&A.res[i], res);
  }
  return miss == NIL32;
}

#if KVG_GM_TMA
// ---- bulk-copy form of match_group (sm_90+/sm_100a async copy engine) ----
// Each warp owns kGridItemChunks 512 B bucket buffers in shared memory and
// one mbarrier. Lanes 0..7 each issue one cp.async.bulk of their chunk's
// bucket (global -> shared, completion counted in bytes on the mbarrier), the
// warp waits on the barrier phase once, and every later read of the group's
// slots is a shared-memory load: the 8 buckets in flight no longer occupy 32
// registers per lane, so more warps fit an SM. Collision steps re-issue the
// colliding chunks' copies as one more round.
__device__ __forceinline__ void mbar_init(u64* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(u64* bar, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, u64* bar) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(a), "r"(parity) : "memory");
}

struct GmWarp {
  Slot* buf;      // [kGridItemChunks][kChunk] this warp's bucket buffers
  u64* bar;
  unsigned phase; // parity of the barrier's current phase
};

__device__ __forceinline__ bool match_group(const GridMatchArgs& A, u32 i, u64 n, u64 g,
                                            int lane, GmWarp& W) {
  const u64 owner = (static_cast<u64>(A.agents[i]) + 1) << 32;
  const u64 c0 = (A.S >> 5) + g * kGridItemChunks;
  const u64 stamp = A.clock0 + i + 1;
  // lane j < kGridItemChunks tracks chunk j's bucket
  const u64 cj = c0 + (lane & (kGridItemChunks - 1));
  u32 bj = static_cast<u32>(hash64(owner | (cj * 32))) & A.mask;
  u32 pend = 0, fnd = 0;  // (warp-uniform)
  for (int j = 0; j < kGridItemChunks; ++j)
    if ((c0 + j) * 32 < n) pend |= 1u << j;
  u32 round = pend;
  for (;;) {
    // WAR across proxies: the previous reads of these buffers are done
    __syncwarp();
    if (lane == 0) mbar_expect(W.bar, __popc(round) * static_cast<unsigned>(kChunk * sizeof(Slot)));
    __syncwarp();
    if (lane < kGridItemChunks && ((round >> lane) & 1u)) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load(W.buf + lane * kChunk, A.table + static_cast<size_t>(bj) * kChunk,
                kChunk * sizeof(Slot), W.bar);
    }
    mbar_wait(W.bar, W.phase);
    W.phase ^= 1u;
    u32 more = 0;
    for (int j = 0; j < kGridItemChunks; ++j) {
      if (!((round >> j) & 1u)) continue;
      const u64 tag = owner | ((c0 + j) * 32);
      const u64 k0 = W.buf[j * kChunk].key;  // (broadcast read)
      if (k0 == tag) fnd |= 1u << j;
      else if (k0 != kEmptyKey) more |= 1u << j;
    }
    if (!more) break;
    if (lane < kGridItemChunks && ((more >> lane) & 1u)) bj = (bj + 1) & A.mask;
    round = more;
  }
  u32 miss = NIL32, res = 0;
  for (int j = 0; j < kGridItemChunks; ++j) {
    const u64 c = c0 + j;
    if (c * 32 >= n) break;  // warp-uniform
    const Slot cur = W.buf[j * kChunk + lane];
    const u32 cb = __shfl_sync(FULL, bj, j);
    const bool found = (fnd >> j) & 1u;
    const u64 page = c * 32 + lane;
    const bool in = page >= A.S && page < n;
    const bool r = found && in && (cur.meta & kResident);
    if (in && !r && page < miss) miss = static_cast<u32>(page);
    res += r;
    if (__any_sync(FULL, r)) {  // refresh: every resident page in range takes the stamp
      const u64 nm = r ? m_make(stamp, m_pins(cur.meta)) : cur.meta;
      if (r) st_meta(&A.table[(size_t)cb * kChunk + lane], nm);
      summ_write(A.summ, cb, nm, lane);
    }
  }
  miss = __reduce_min_sync(FULL, miss);
  res = __reduce_add_sync(FULL, res);
  if (lane == 0) {
    if (miss != NIL32) atomicMin(&A.fm[i], miss);
    if (res) atomicAdd(&A.res[i], res);
  }
  return miss == NIL32;
}

#define KVG_GM_WARP_SETUP                                                          \
  __shared__ __align__(128) Slot gm_buf[kGridMatchWarps][kGridItemChunks * kChunk]; \
  __shared__ __align__(8) u64 gm_bar[kGridMatchWarps];                              \
  GmWarp W{gm_buf[w], &gm_bar[w], 0u};                                              \
  if (lane == 0) mbar_init(W.bar);                                                  \
  __syncwarp();
#define KVG_GM_W , W
#else
#define KVG_GM_WARP_SETUP
#define KVG_GM_W
#endif

__device__ __forceinline__ u64 match_groups(const GridMatchArgs& A, u64 n) {
  if (n <= A.S) return 0;
  return (((n - 1) >> 5) - (A.S >> 5)) / kGridItemChunks + 1;
}

// Pass 1, one warp per query: files the shared range for the shared-stamp
// pass and probes the first private chunk group. Queries whose first group
// is fully resident (and that have more) go on the continuation list.
__global__ void __launch_bounds__(kGridMatchWarps * 32, KVG_GM_MINB) grid_match_kernel(GridMatchArgs A) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u32 gw = blockIdx.x * kGridMatchWarps + w, GW = gridDim.x * kGridMatchWarps;
  KVG_GM_WARP_SETUP
  for (u32 i = gw; i < A.n; i += GW) {
    const u64 n = A.lens[i] / A.ps;
    if (lane == 0) {
      const u64 sh = n < A.S ? n : A.S;
      if (sh > 0) atomicMax(&A.best[sh - 1], i + 1);
    }
    const u64 groups = match_groups(A, n);
    if (groups == 0) continue;
    if (match_group(A, i, n, 0, lane KVG_GM_W) && groups > 1) {  // (warp-uniform)
      // file groups [1, groups) as work items: one contiguous range per query
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(A.n_items, static_cast<unsigned>(groups - 1));
      base = __shfl_sync(FULL, base, 0);
      for (u64 t = lane; t + 1 < groups; t += 32)
        A.items[base + t] = make_ulonglong2((static_cast<u64>(i) << 32) | (t + 1), n);
    }
  }
}

// Pass 2: the remaining groups of the continued queries as a dense list of
// (query, group, pages) items filed by pass 1, so a long resident context
// spreads over many warps and no warp walks empty (query, group) slots
// (measured: the flattened query x max_groups enumeration spent a dependent
// load pair on every empty slot).
__global__ void __launch_bounds__(kGridMatchWarps * 32, KVG_GM_MINB) grid_match_rest_kernel(GridMatchArgs A) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u64 gw = blockIdx.x * kGridMatchWarps + w, GW = gridDim.x * kGridMatchWarps;
  KVG_GM_WARP_SETUP
  const u64 total = *A.n_items;
  for (u64 k = gw; k < total; k += GW) {
    const ulonglong2 it = A.items[k];  // {query << 32 | group, pages}
    match_group(A, static_cast<u32>(it.x >> 32), it.y, it.x & 0xffffffffu, lane KVG_GM_W);
  }
}

// One CTA: suffix max over best[] (page p's stamp is the last query whose
// shared range covers p), then every shared chunk's resident pages take it.
__global__ void __launch_bounds__(1024) grid_match_shared_kernel(GridMatchArgs A) {
  __shared__ u32 tile[1024];
  __shared__ u32 carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (A.S == 0) return;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (long long base = static_cast<long long>((A.S - 1) / 1024) * 1024; base >= 0; base -= 1024) {
    const u64 p = static_cast<u64>(base) + tid;
    tile[tid] = p < A.S ? A.best[p] : 0u;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const u32 x = tid + off < 1024 ? tile[tid + off] : 0u;
      __syncthreads();
      if (x > tile[tid]) tile[tid] = x;
      __syncthreads();
    }
    const u32 c = carry;
    const u32 v = tile[tid] > c ? tile[tid] : c;
    if (p < A.S) A.best[p] = v;
    __syncthreads();
    if (tid == 0) carry = v;
    __syncthreads();
  }
  __threadfence_block();
  const u64 chunks = (A.S + 31) / 32;
  for (u64 c = warp; c < chunks; c += nw) {
    const u64 tag = c * 32;  // owner 0
    u32 b = static_cast<u32>(hash64(tag)) & A.mask;
    Slot s;
    bool found = false;
    for (;;) {
      s = ld_slot(&A.table[(size_t)b * kChunk + lane]);
      const u64 k0 = __shfl_sync(FULL, s.key, 0);
      if (k0 == tag) { found = true; break; }
      if (k0 == kEmptyKey) break;
      b = (b + 1) & A.mask;
    }
    if (!found) continue;
    const u64 page = tag + lane;
    const u32 win = page < A.S ? A.best[page] : 0u;
    u64 nm = s.meta;
    if ((s.meta & kResident) && win) nm = m_make(A.clock0 + win, m_pins(s.meta));
    const bool wrote = nm != s.meta;
    if (wrote) st_meta(&A.table[(size_t)b * kChunk + lane], nm);
    if (__any_sync(FULL, wrote)) summ_write(A.summ, b, nm, lane);
  }
}

// ------------------------------------------------------------------ evict

// scan_summ for the grid: the same in-flight depth, but consecutive 32-bucket
// groups of the occupancy list go to consecutive warps of the whole grid
// (round robin), so a run of victims — the oldest chains sit together at the
// front of the list — is spread over every SM instead of a few warps.
template <int kDepth, typename F>
__device__ __forceinline__ void grid_scan_summ(const Op& op, u32 gw, int lane, u32 GW, F&& f) {
  const u32 n_occ = op.occ_n;
  const u32 groups = (n_occ + 31) / 32;
  for (u32 it = 0; it * kDepth * GW < groups; ++it) {
    u32 bk[kDepth];
    Summ e[kDepth];
#pragma unroll
    for (int g = 0; g < kDepth; ++g) {
      const u32 i = ((it * kDepth + g) * GW + gw) * 32u + lane;
      bk[g] = i < n_occ ? __ldcg(&op.occ[i]) : NIL32;
    }
#pragma unroll
    for (int g = 0; g < kDepth; ++g) {
      e[g] = Summ{0, 0, 0, 0, 0, 0};
      if (bk[g] != NIL32) e[g] = ld_summ(&op.summ[bk[g]]);
    }
#pragma unroll 1
    for (int g = 0; g < kDepth; ++g) {
      const u32 b0 = bk[0];
      const Summ e0 = e[0];
#pragma unroll
      for (int j = 0; j + 1 < kDepth; ++j) {
        bk[j] = bk[j + 1];
        e[j] = e[j + 1];
      }
      f(b0 != NIL32, b0, e0);
    }
  }
}

// select_bin over the staged histogram by the whole CTA (every thread calls
// it): each warp sums one contiguous segment (conflict-free: lane-strided
// reads), warp 0 scans the segment sums, then the 32-bin rounds of the one
// segment that crosses `need`: the smallest bin whose inclusive count
// reaches `need`, and the rank inside it. (The one-warp form it replaces
// read 64 consecutive bins per lane: a 32-way bank conflict on every read,
// 4-6 us per pass on the C5-size select.)
__device__ __forceinline__ u32 select_bin_cta(Op& op, const u32* cnt, u32 nbins, int d, int lane,
                                              int warp, int nw, u32* wsum, u64* sel,
                                              u64* rank_in_bin) {
  const u32 seg = (nbins + nw - 1) / nw;
  u32 s = 0;
  for (u32 i = lane; i < seg; i += 32) {
    const u32 b = warp * seg + i;
    if (b < nbins) s += cnt[b];
  }
  s = __reduce_add_sync(FULL, s);
  if (lane == 0) wsum[warp] = s;
  __syncthreads();
  if (warp == 0) {
    const u32 v = lane < nw ? wsum[lane] : 0u;
    u32 incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const u32 x = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += x;
    }
    const u64 need = op.need;
    const unsigned ballot = __ballot_sync(FULL, static_cast<u64>(incl) >= need);
    u32 bin = 0;
    u64 before = need - 1;  // (rank 1 on a mismatch)
    if (ballot == 0) {
      if (lane == 0) op.err = E_EVICT_MISMATCH;
    } else {
      const int W = __ffs(ballot) - 1;
      u64 cum = __shfl_sync(FULL, incl - v, W);
      for (u32 r = 0; r < seg; r += 32) {
        const u32 b = W * seg + r + lane;
        const u32 c = (r + lane < seg && b < nbins) ? cnt[b] : 0u;
        u32 in2 = c;
        for (int o = 1; o < 32; o <<= 1) {
          const u32 x = __shfl_up_sync(FULL, in2, o);
          if (lane >= o) in2 += x;
        }
        const unsigned hit = __ballot_sync(FULL, cum + in2 >= need);
        if (hit) {
          const int j = __ffs(hit) - 1;
          bin = W * seg + r + j;
          before = cum + __shfl_sync(FULL, in2 - c, j);
          break;
        }
        cum += __shfl_sync(FULL, in2, 31);
      }
      if (lane == 0) {
        op.need = need - before;
        op.prefix = (op.prefix << d) | bin;
      }
    }
    if (lane == 0) {
      sel[0] = bin;
      sel[1] = need - before;
    }
  }
  __syncthreads();
  *rank_in_bin = sel[1];
  return static_cast<u32>(sel[0]);
}

__global__ void __launch_bounds__(512) grid_evict_kernel(GridEvictArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ Op op;
  __shared__ u32 scnt[kGridBins], sdmax[kGridBins];
  __shared__ u32 swsum[32];
  __shared__ u64 ssel[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int nt = blockDim.x;
  const int gw = blockIdx.x * nw + warp, GW = gridDim.x * nw;
  if (tid == 0) {
    op.table = A.table;
    op.summ = A.summ;
    op.occ = A.occ;
    op.occ_n = A.occ_n;
    op.mask = A.mask;
    op.shared_pages = A.S;
    op.implicit_pins = 0;
    op.agents = nullptr;
    op.log = nullptr;
    op.log_victims = 1;
    op.vic = A.vic;
    op.vic_cap = A.vic_cap;
    op.vic_n = A.vic_n;
    op.agent = 0;
    op.k = A.k;
    op.evictable = A.evictable;
    op.clock = A.clock;
    op.all = A.k >= A.evictable;
    op.prefix = 0;
    op.need = A.k;
    op.err = E_NONE;
  }
  __syncthreads();
  gprof(0);
  const bool all = op.all;
  u64 T = 0, cut = 0;
  if (!all) {
    Hist hs{scnt, sdmax, true};
    int lo_bits = 64 - __clzll(A.clock | 1ull);
    int pass = 0;
    while (lo_bits > 0) {
      const int d = lo_bits < kGridDigit ? lo_bits : kGridDigit;
      const int shift = lo_bits - d;
      const bool last = shift == 0;
      const u32 nbins = 1u << d;
      for (u32 i = tid; i < nbins; i += nt) {
        scnt[i] = 0;
        sdmax[i] = 0;
      }
      __syncthreads();
      const u64 prefix = op.prefix;
      grid_scan_summ<kGridSumDepth>(op, gw, lane, GW, [&](bool valid, u32 b, const Summ& e) {
        const bool mixed = valid && (e.sf & kMixed);
        u32 c = 0;
        u64 st = 0;
        if (valid && !mixed) {
          c = e.dev;
          st = e.sf & kStampMask;
        }
        const bool act = c != 0 && (st >> lo_bits) == prefix;
        const u32 bin = act ? static_cast<u32>((st >> shift) & (nbins - 1)) : 0xffffffffu;
        const unsigned peers = __match_any_sync(FULL, bin);
        if (act) {
          const int leader = __ffs(peers) - 1;
          const u32 wsum = __reduce_add_sync(peers, static_cast<u32>(__popc(c)));
          if (lane == leader) atomicAdd(&scnt[bin], wsum);
          if (last) {
            const u32 dm = static_cast<u32>(e.tag & 0xffffffffu) + 31u - __clz(c);
            const u32 mx = __reduce_max_sync(peers, dm);
            if (lane == leader) atomicMax(&sdmax[bin], mx);
          }
        }
        if (mixed) hist_mixed(op, hs, b, prefix, lo_bits, shift, nbins, last);
      });
      gprof(1 + 4 * pass);
      __syncthreads();
      u32* gc = A.ghist + static_cast<size_t>(pass % 3) * 2 * kGridBins;
      u32* gd = gc + kGridBins;
      for (u32 i = tid; i < nbins; i += nt) {
        if (scnt[i]) atomicAdd(&gc[i], scnt[i]);
        if (last && sdmax[i]) atomicMax(&gd[i], sdmax[i]);
      }
      gprof(2 + 4 * pass);
      grid.sync();
      gprof(3 + 4 * pass);
      // every CTA stages the merged histogram in shared memory and selects
      // the same bin from it
      for (u32 i = tid; i < nbins; i += nt) {
        scnt[i] = __ldcg(&gc[i]);
        if (last) sdmax[i] = __ldcg(&gd[i]);
      }
      __syncthreads();
      {
        u64 rank = 0;
        const u32 bin = select_bin_cta(op, scnt, nbins, d, lane, warp, nw, swsum, ssel, &rank);
        if (last && tid == 0) op.cut_depth = static_cast<u64>(sdmax[bin]) + 1 - rank;
      }
      if (blockIdx.x == 0) {  // the buffer of pass + 2 (read last in pass - 1)
        u32* z = A.ghist + static_cast<size_t>((pass + 2) % 3) * 2 * kGridBins;
        for (u32 i = tid; i < 2 * kGridBins; i += nt) z[i] = 0;
      }
      __syncthreads();
      gprof(4 + 4 * pass);
      lo_bits = shift;
      ++pass;
    }
    T = op.prefix;
    cut = op.cut_depth;
  }
  unsigned int freed = 0;
  grid_scan_summ<kGridSumDepth>(op, gw, lane, GW, [&](bool valid, u32 b, const Summ& e) {
    u32 v = 0;
    u64 st = 0;
    if (valid) {
      if (e.sf & kMixed) {
        freed += scatter_mixed(op, b, all, T, cut);
      } else if (e.dev != 0) {
        st = e.sf & kStampMask;
        v = (all || st < T) ? e.dev : (st == T ? e.dev & ge_mask(e.tag & 0xffffffffull, cut) : 0u);
      }
    }
    if (v) {
      freed += __popc(v);
      if (op.vic)
        for (u32 m = v; m != 0; m &= m - 1) emit_victim(op, e.tag + (__ffs(m) - 1), st, 0);
      __stcg(&op.summ[b].dev, e.dev & ~v);
    }
    // the victims' slots, one coalesced bucket store per bucket with victims
    for (unsigned todo = __ballot_sync(FULL, v != 0); todo != 0; todo &= todo - 1) {
      const int j = __ffs(todo) - 1;
      const u32 bj = __shfl_sync(FULL, b, j), vj = __shfl_sync(FULL, v, j);
      if ((vj >> lane) & 1u) st_meta(&op.table[(size_t)bj * kChunk + lane], 0ull);
    }
  });
  gprof(30);
  freed = __reduce_add_sync(FULL, freed);
  if (lane == 0 && freed) atomicAdd(A.freed, freed);
  if (tid == 0 && op.err) atomicMax(A.err, op.err);
}

}  // namespace kvg
