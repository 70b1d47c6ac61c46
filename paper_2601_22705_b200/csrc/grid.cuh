// Grid-wide page-table kernels for the CacheTree seam (discard mode): the
// bandwidth form of kernels 1 and 2 on C2 / C5-size tables, where one CTA per
// operation (cache_kernel) cannot pull more than a single SM's share of HBM.
//
//  * grid_match_kernel / grid_match_shared_kernel — a BATCH of match_prefix
//    calls (cache_tree.cpp:114-142) that leaves the table exactly as the same
//    calls issued one by one: query i runs at clock0 + i + 1, every resident
//    page a query's range covers is refreshed, so a page's final stamp is the
//    clock of the LAST query covering it (residency never changes inside a
//    match batch). One warp per query (dynamic work queue over all SMs) probes
//    its shared-prompt chunks read-only and refreshes its private chunks in
//    place (the host splits batches so an agent appears at most once, making a
//    private chunk single-writer); shared-prompt pages get max{i : query i
//    covers p} through one atomicMax per query and a suffix max, and are
//    rewritten by one small CTA afterwards.
//  * grid_evict_kernel — evict(needed) (cache_tree.cpp:270-319, per-page form
//    SURVEY.md A.2) as ONE cooperative launch over every SM: the radix select
//    of coop_evict with 11-bit digits, per-CTA shared-memory histograms
//    (warp-aggregated atomics) merged into a small global histogram once per
//    pass, a grid barrier per pass, then the scatter-free pass. Same victims,
//    same order after the host's per-op sort.
#pragma once

#include <cooperative_groups.h>

namespace kvg {

constexpr int kGridMatchWarps = 8;

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

// One warp per work item: item k covers up to kGridItemChunks private chunks
// of query item_q[k] starting at chunk item_c[k] (the host splits every
// query's private range [S, len/ps) so long contexts spread over many warps).
// Each item probes its chunks (all in flight), refreshes their resident
// pages to the query's clock (a private chunk has one writer per batch: the
// host splits batches so an agent appears once) and folds first miss /
// resident count into the query's accumulators. A query's first item also
// files its shared range for the shared-stamp pass.
__global__ void __launch_bounds__(kGridMatchWarps * 32) grid_match_kernel(GridMatchArgs A) {
  __shared__ Op wops[kGridMatchWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Op& op = wops[w];
  if (lane == 0) {
    op.table = A.table;
    op.summ = A.summ;
    op.mask = A.mask;
    op.shared_pages = A.S;
    op.implicit_pins = 0;
    op.agents = nullptr;
    op.log = nullptr;
    op.vic = nullptr;
    op.log_victims = 0;
  }
  __syncwarp();
  const u32 gw = blockIdx.x * kGridMatchWarps + w, GW = gridDim.x * kGridMatchWarps;
  for (u32 k = gw; k < A.n_items; k += GW) {
    const u32 i = A.item_q[k];
    const u64 c0 = A.item_c[k];
    const u64 n = A.lens[i] / A.ps;
    if (c0 == ~0u) {  // head item of a query without private pages
      if (lane == 0) {
        const u64 sh = n < A.S ? n : A.S;
        if (sh > 0) atomicMax(&A.best[sh - 1], i + 1);
      }
      continue;
    }
    const u64 lo = c0 * 32 > A.S ? c0 * 32 : A.S;
    const u64 hi_c = (c0 + kGridItemChunks) * 32;
    const u64 hi = hi_c < n ? hi_c : n;
    if (lane == 0) {
      post_range(op, A.agents[i], lo, hi, RF_STAMP, 0, A.clock0 + i + 1);
      if (lo == A.S) {  // the query's first item
        const u64 sh = n < A.S ? n : A.S;
        if (sh > 0) atomicMax(&A.best[sh - 1], i + 1);
      }
    }
    __syncwarp();
    coop_range<kGridItemChunks>(op, 0, lane, 1);
    __syncwarp();
    if (lane == 0) {
      if (op.first_miss != ~0ull) atomicMin(&A.fm[i], static_cast<u32>(op.first_miss));
      if (op.resident) atomicAdd(&A.res[i], op.resident);
    }
    __syncwarp();
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

__global__ void __launch_bounds__(512) grid_evict_kernel(GridEvictArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ Op op;
  __shared__ u32 scnt[kGridBins], sdmax[kGridBins];
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
  const bool all = op.all;
  u64 T = 0, cut = 0;
  if (!all) {
    Hist hs{scnt, sdmax};
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
      scan_summ<kGridSumDepth>(op, gw, lane, GW, [&](bool valid, u32 b, const Summ& e) {
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
      __syncthreads();
      u32* gc = A.ghist + static_cast<size_t>(pass % 3) * 2 * kGridBins;
      u32* gd = gc + kGridBins;
      for (u32 i = tid; i < nbins; i += nt) {
        if (scnt[i]) atomicAdd(&gc[i], scnt[i]);
        if (last && sdmax[i]) atomicMax(&gd[i], sdmax[i]);
      }
      grid.sync();
      if (warp == 0) {  // every CTA selects the same bin from the merged histogram
        Hist hg{gc, gd};
        u64 rank = 0;
        const u32 bin = select_bin(op, hg, nbins, d, lane, &rank);
        if (last && lane == 0) op.cut_depth = static_cast<u64>(__ldcg(&gd[bin])) + 1 - rank;
      }
      if (blockIdx.x == 0) {  // the buffer of pass + 2 (read last in pass - 1)
        u32* z = A.ghist + static_cast<size_t>((pass + 2) % 3) * 2 * kGridBins;
        for (u32 i = tid; i < 2 * kGridBins; i += nt) z[i] = 0;
      }
      __syncthreads();
      lo_bits = shift;
      ++pass;
    }
    T = op.prefix;
    cut = op.cut_depth;
  }
  unsigned int freed = 0;
  scan_summ<kGridSumDepth>(op, gw, lane, GW, [&](bool valid, u32 b, const Summ& e) {
    if (!valid) return;
    if (e.sf & kMixed) {
      freed += scatter_mixed(op, b, all, T, cut);
      return;
    }
    const u32 c = e.dev;
    if (c == 0) return;
    const u64 st = e.sf & kStampMask;
    const u32 v = (all || st < T) ? c : (st == T ? c & ge_mask(e.tag & 0xffffffffull, cut) : 0u);
    if (v == 0) return;
    freed += __popc(v);
    Slot* bk = &op.table[(size_t)b * kChunk];
    for (u32 m = v; m != 0; m &= m - 1) {
      const int l = __ffs(m) - 1;
      st_meta(&bk[l], 0ull);
      emit_victim(op, e.tag + l, st, 0);
    }
    __stcg(&op.summ[b].dev, e.dev & ~v);
  });
  freed = __reduce_add_sync(FULL, freed);
  if (lane == 0 && freed) atomicAdd(A.freed, freed);
  if (tid == 0 && op.err) atomicMax(A.err, op.err);
}

}  // namespace kvg
