// B200 (sm_100a) engine for the kvadmit simulator hot path.
//
// Replaces kvadmit::run_simulation (/root/reference/proj/src/engine.cpp:446-456)
// and the CacheTree operations it drives per event (cache_tree.cpp:114-437).
//
// Execution model:
//  * one CTA per simulation (NW warps, NW = 1 for small sims so thousands of
//    sweep sims are resident at once; up to 32 for big sims);
//  * thread 0 is the LEADER: it runs the event loop, controller, cost model and
//    all scalar bookkeeping as an explicit state machine, in IEEE double with
//    FMA contraction disabled (-fmad=false) so every simulated time is
//    bit-identical to the reference;
//  * whenever the leader needs page-level work it posts a COOPERATIVE OP in
//    shared memory and the whole CTA executes it:
//      RANGE   warp-cooperative block-hash prefix lookup / stamp refresh /
//              pin / create / free over an agent's page range (kernel 1),
//      EVICT   shared-memory radix select over page last-use stamps plus a
//              scatter that frees the chosen pages (kernel 2),
//      REBUILD rehash of live buckets into the alternate table.
//    The event heap, ready set and pin bookkeeping are leader-only O(log n) /
//    O(1) structures (leader.cuh), so ticks and admissions never need the CTA.
//  * tick signals (kernel 3) and the agent state machine (kernel 4) are
//    leader-side O(1) steps fused into the same persistent kernel, because the
//    reference's strictly sequential event order (engine.cpp:98-136) leaves no
//    independent work to spread over a launch per tick.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kvg_device.h"

namespace kvg {

constexpr unsigned FULL = 0xffffffffu;

// ------------------------------------------------------------------------
// small device helpers

__device__ __forceinline__ u64 hash64(u64 x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// 128-bit slot load that bypasses L1: other warps of the CTA claim buckets
// with L2 atomics, so a stale L1 line must never satisfy a probe.
__device__ __forceinline__ Slot ld_slot(const Slot* p) {
  ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(p));
  return Slot{v.x, v.y};
}
__device__ __forceinline__ void st_meta(Slot* p, u64 meta) { __stcg(&p->meta, meta); }

__device__ __forceinline__ u64 m_stamp(u64 m) { return m & kStampMask; }
__device__ __forceinline__ u64 m_pins(u64 m) { return (m >> kPinShift) & kPinMask; }
__device__ __forceinline__ u64 m_make(u64 stamp, u64 pins) {
  return kResident | (pins << kPinShift) | (stamp & kStampMask);
}

// ------------------------------------------------------------------------
// cooperative ops

enum OpKind : int {
  OP_NONE = 0,
  OP_EXIT,
  OP_RANGE,      // per-page work over an agent's page range
  OP_EVICT,      // radix select + scatter free
  OP_REBUILD,    // rehash live buckets into the alternate table
  OP_SCANFREE,   // free pages by (owner, min index) over the whole table
};

enum RangeFlags : u32 {
  RF_STAMP = 1,   // set stamp of resident pages
  RF_PIN = 2,     // add pin_delta to resident pages (error if missing/underflow)
  RF_CREATE = 4,  // create missing pages (stamp, pins = max(pin_delta, 0))
  RF_FREE = 8,    // free resident pages (error if pinned)
  RF_STRICT = 16, // every page in range must be resident (pin/unpin paths)
};

enum ErrCode : int {
  E_NONE = 0,
  E_PIN_MISSING = 1,
  E_UNPIN_UNDERFLOW = 2,
  E_DISCARD_PINNED = 3,
  E_ILLEGAL_TRANSITION = 4,
  E_NOT_ACTIVE = 5,
  E_EVICT_MISMATCH = 6,
  E_TABLE_FULL = 7,
  E_DRAINED = 8,
  E_PREFIX_BROKEN = 9,
  E_OFFLOAD = 10,
  E_TWO_ADMISSIONS = 11,
  E_EVENT_BUSY = 12,
};

// Table context + op descriptor + results, all in shared memory.
struct Op {
  int kind;
  int err;
  u32 agent;
  u32 flags;
  int pin_delta;
  int log_victims;      // 1: append victims to the log / victim list
  int implicit_pins;    // engine mode: pins derived from per-agent pinned prefixes
  u64 pin_max;          // engine mode: shared-prompt pages [0, pin_max) are pinned
  const AgentDev* agents;
  u64 p0, p1;
  u64 stamp;
  u64 k;                // EVICT: pages needed
  u64 evictable;        // EVICT: resident unpinned pages
  u64 clock;            // EVICT: upper bound of candidate stamps
  u64 owner_filter;     // SCANFREE: owner or ~0 for all
  // results
  unsigned long long first_miss;
  unsigned int created, freed, pin_up, pin_down, resident;
  unsigned int pad;
  // radix select state
  u64 prefix, need, cut_depth, thresh;
  int all;
  // argmin result
  double amin_t;
  u64 amin_o;
  u32 amin_a, amin_any;
  // table context
  Slot* table;
  Slot* alt;
  u32* occ;
  u32* alt_occ;
  u32 mask;
  unsigned int occ_n;
  unsigned int alt_n;
  u32 pad2;
  u64 shared_pages;
  // victim sink (engine log or cache victim list)
  kvg_log_record* log;
  u64 log_cap;
  unsigned long long* log_n;
  u64 log_clock;
  kvg_victim* vic;
  u64 vic_cap;
  unsigned long long* vic_n;
};

constexpr int kBins = 512;

// Radix-select histogram. Lives in per-simulation global scratch (L2): it is
// touched only by eviction selects, and keeping it out of shared memory leaves
// the SM's unified L1 to the leader's hot agent records.
struct Hist {
  unsigned int* cnt;   // [kBins]
  unsigned int* dmax;  // [kBins]
};

// Continues a linear probe for chunk `tag` from bucket `b`. Returns true and
// this lane's slot when present; otherwise *bucket is the first empty bucket.
__device__ __forceinline__ bool probe_from(const Op& op, u64 tag, u32 b, int lane, u32* bucket,
                                           Slot* mine) {
  for (;;) {
    Slot s = ld_slot(&op.table[(size_t)b * kChunk + lane]);
    u64 k0 = __shfl_sync(FULL, s.key, 0);
    if (k0 == tag) {
      *bucket = b;
      *mine = s;
      return true;
    }
    if (k0 == kEmptyKey) {
      *bucket = b;
      return false;
    }
    b = (b + 1) & op.mask;
  }
}

// Claims an empty bucket for `tag`, starting at bucket `b`; returns it.
__device__ __noinline__ u32 claim(Op& op, Slot* table, u32* occ, unsigned int* occ_n, u32 mask,
                     u64 tag, u32 b, int lane) {
  for (;;) {
    int won = 0;
    if (lane == 0) {
      u64 k0 = __ldcg(&table[(size_t)b * kChunk].key);
      if (k0 == kEmptyKey)
        won = atomicCAS(reinterpret_cast<unsigned long long*>(&table[(size_t)b * kChunk].key),
                        kEmptyKey, tag) == kEmptyKey;
    }
    won = __shfl_sync(FULL, won, 0);
    if (won) {
      Slot* s = &table[(size_t)b * kChunk + lane];
      if (lane != 0) __stcg(&s->key, tag + lane);
      __stcg(&s->meta, 0ull);
      if (lane == 0) {
        unsigned int idx = atomicAdd(occ_n, 1u);
        __stcg(&occ[idx], b);
      }
      __syncwarp();
      return b;
    }
    b = (b + 1) & mask;
  }
}

struct RangeAcc {
  unsigned int created, freed, up, down, resident;
  u64 miss;
  int err;
};

// Per-lane work on one 32-page chunk whose bucket probe already completed.
__device__ __forceinline__ void range_chunk(Op& op, u64 tag, u64 lo, u64 hi, u32 b, Slot s,
                                            bool found, int lane, RangeAcc& acc) {
  const u32 flags = op.flags;
  const int delta = op.pin_delta;
  const u64 page = (tag & 0xffffffffull) + lane;
  const bool in = page >= lo && page < hi;
  if (!found && (flags & RF_CREATE) && __any_sync(FULL, in)) {
    b = claim(op, op.table, op.occ, &op.occ_n, op.mask, tag, b, lane);
    found = true;
    s = Slot{tag + lane, 0};
  }
  if (!in) return;
  const bool res = found && (s.meta & kResident);
  Slot* slot = found ? &op.table[(size_t)b * kChunk + lane] : nullptr;
  if (!res) {
    if (flags & RF_CREATE) {
      const u64 pins = delta > 0 ? static_cast<u64>(delta) : 0;
      st_meta(slot, m_make(op.stamp, pins));
      ++acc.created;
      if (pins) ++acc.up;
    } else {
      acc.miss = page < acc.miss ? page : acc.miss;
      if (flags & RF_STRICT) acc.err = E_PIN_MISSING;
    }
    return;
  }
  ++acc.resident;
  const u64 m = s.meta;
  if (flags & RF_FREE) {
    if (!op.implicit_pins && m_pins(m) != 0) {
      acc.err = E_DISCARD_PINNED;
      return;
    }
    st_meta(slot, 0ull);
    ++acc.freed;
    return;
  }
  const u64 stamp = (flags & RF_STAMP) ? op.stamp : m_stamp(m);
  long long pins = static_cast<long long>(m_pins(m));
  if (flags & RF_PIN) {
    long long np = pins + delta;
    if (np < 0) {
      acc.err = E_UNPIN_UNDERFLOW;
      np = 0;
    }
    if (pins == 0 && np > 0) ++acc.up;
    if (pins > 0 && np == 0) ++acc.down;
    pins = np;
  }
  const u64 nm = m_make(stamp, static_cast<u64>(pins));
  if (nm != m) st_meta(slot, nm);
}

// RANGE: agent `op.agent`, pages [p0, p1). Pages below shared_pages belong to
// the shared prompt (owner 0), the rest to owner agent+1 (workload.cpp:167-171).
// Each warp owns every nw-th 32-page chunk and keeps kProbeDepth bucket probes
// in flight (one 512 B coalesced load each) before consuming any of them, so a
// context of C chunks costs ~C/(nw*kProbeDepth) DRAM round trips, not C.
constexpr int kProbeDepth = 8;

__device__ __noinline__ void coop_range(Op& op, int warp, int lane, int nw) {
  const u64 p0 = op.p0, p1 = op.p1;
  if (p0 >= p1) return;
  const u64 S = op.shared_pages;
  const u64 s_lo = p0, s_hi = p1 < S ? p1 : S;
  const u64 q_lo = p0 > S ? p0 : S, q_hi = p1;
  const u64 n_sh = s_lo < s_hi ? ((s_hi - 1) >> 5) - (s_lo >> 5) + 1 : 0;
  const u64 n_pr = q_lo < q_hi ? ((q_hi - 1) >> 5) - (q_lo >> 5) + 1 : 0;
  const u64 total = n_sh + n_pr;
  const u64 owner_priv = static_cast<u64>(op.agent) + 1;
  RangeAcc acc{0, 0, 0, 0, 0, ~0ull, E_NONE};
  auto tag_of = [&](u64 it) -> u64 {
    return it < n_sh ? ((s_lo >> 5) + it) << 5
                     : (owner_priv << 32) | (((q_lo >> 5) + (it - n_sh)) << 5);
  };
  for (u64 base = warp; base < total; base += static_cast<u64>(nw) * kProbeDepth) {
    Slot s[kProbeDepth];
    u32 b[kProbeDepth];
#pragma unroll
    for (int g = 0; g < kProbeDepth; ++g) {
      const u64 it = base + static_cast<u64>(g) * nw;
      if (it < total) {
        b[g] = static_cast<u32>(hash64(tag_of(it))) & op.mask;
        s[g] = ld_slot(&op.table[(size_t)b[g] * kChunk + lane]);
      }
    }
#pragma unroll 1
    for (int g = 0; g < kProbeDepth; ++g) {
      const u64 it = base + static_cast<u64>(g) * nw;
      if (it >= total) break;
      const u64 tag = tag_of(it);
      const u64 k0 = __shfl_sync(FULL, s[g].key, 0);
      bool found;
      if (k0 == tag) {
        found = true;
      } else if (k0 == kEmptyKey) {
        found = false;
      } else {
        found = probe_from(op, tag, (b[g] + 1) & op.mask, lane, &b[g], &s[g]);
      }
      const bool shared = it < n_sh;
      range_chunk(op, tag, shared ? s_lo : q_lo, shared ? s_hi : q_hi, b[g], s[g], found, lane,
                  acc);
    }
  }
  // warp reductions, then one shared atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    acc.created += __shfl_down_sync(FULL, acc.created, o);
    acc.freed += __shfl_down_sync(FULL, acc.freed, o);
    acc.up += __shfl_down_sync(FULL, acc.up, o);
    acc.down += __shfl_down_sync(FULL, acc.down, o);
    acc.resident += __shfl_down_sync(FULL, acc.resident, o);
    const u64 om = __shfl_down_sync(FULL, acc.miss, o);
    acc.miss = om < acc.miss ? om : acc.miss;
    const int oe = __shfl_down_sync(FULL, acc.err, o);
    acc.err = oe > acc.err ? oe : acc.err;
  }
  if (lane == 0) {
    if (acc.created) atomicAdd(&op.created, acc.created);
    if (acc.freed) atomicAdd(&op.freed, acc.freed);
    if (acc.up) atomicAdd(&op.pin_up, acc.up);
    if (acc.down) atomicAdd(&op.pin_down, acc.down);
    if (acc.resident) atomicAdd(&op.resident, acc.resident);
    if (acc.miss != ~0ull) atomicMin(&op.first_miss, acc.miss);
    if (acc.err) atomicMax(&op.err, acc.err);
  }
}

// Visits every claimed bucket (the dense occupancy list), kScanDepth buckets in
// flight per warp; f(bucket, slot, pin_threshold) runs per lane. With implicit
// pins (engine mode) the bucket owner's pinned prefix length is fetched in the
// same wave: page (owner, idx) is pinned iff idx < threshold.
constexpr int kScanDepth = 4;

template <typename F>
__device__ __forceinline__ void scan_buckets(const Op& op, int warp, int lane, int nw, F&& f) {
  const unsigned int n_occ = op.occ_n;
  for (u32 base = warp; base < n_occ; base += static_cast<u32>(nw) * kScanDepth) {
    u32 bk[kScanDepth];
    Slot s[kScanDepth];
    u64 thr[kScanDepth];
#pragma unroll
    for (int g = 0; g < kScanDepth; ++g) {
      const u32 i = base + g * nw;
      bk[g] = i < n_occ ? __ldcg(&op.occ[i]) : 0u;
    }
#pragma unroll
    for (int g = 0; g < kScanDepth; ++g) {
      const u32 i = base + g * nw;
      if (i < n_occ) s[g] = ld_slot(&op.table[(size_t)bk[g] * kChunk + lane]);
    }
#pragma unroll
    for (int g = 0; g < kScanDepth; ++g) {
      const u32 i = base + g * nw;
      thr[g] = 0;
      if (i < n_occ && op.implicit_pins) {
        const u64 owner = __shfl_sync(FULL, s[g].key, 0) >> 32;
        // plain load: the records may live in shared memory (leader wrote them
        // before the barrier that started this op)
        thr[g] = owner == 0 ? op.pin_max : op.agents[owner - 1].pinned_pg;
      }
    }
#pragma unroll 1
    for (int g = 0; g < kScanDepth; ++g) {
      const u32 i = base + g * nw;
      if (i < n_occ) f(bk[g], s[g], thr[g]);
    }
  }
}

// Eviction candidate: resident and unpinned (cache_tree.cpp:230-234 per page).
__device__ __forceinline__ bool is_candidate(const Op& op, const Slot& s, u64 thr) {
  if (!(s.meta & kResident)) return false;
  if (op.implicit_pins) return (s.key & 0xffffffffull) >= thr;
  return m_pins(s.meta) == 0;
}

__device__ __forceinline__ void emit_victim(Op& op, u64 key, u64 stamp, u32 agent) {
  if (op.log) {
    unsigned long long i = atomicAdd(op.log_n, 1ull);
    if (i < op.log_cap)
      op.log[i] = kvg_log_record{KVG_LOG_VICTIM, agent, op.log_clock, key, stamp};
  }
  if (op.vic) {
    unsigned long long i = atomicAdd(op.vic_n, 1ull);
    if (i < op.vic_cap) op.vic[i] = kvg_victim{key, stamp};
  }
}

// Warp 0: find the histogram bin holding rank op.need (1-based) among
// nbins bins. Returns the bin; *rank_in_bin receives the rank inside it.
// Every lane gets both values through shuffles (no smem read-after-write).
__device__ __noinline__ u32 select_bin(Op& op, Hist& h, u32 nbins, int d, int lane, u64* rank_in_bin) {
  const u32 per = (nbins + 31) / 32;
  const u32 base = lane * per;
  u32 local = 0;
  for (u32 i = 0; i < per; ++i)
    if (base + i < nbins) local += __ldcg(&h.cnt[base + i]);
  u32 incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    u32 v = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += v;
  }
  const u64 need = op.need;
  const unsigned ballot = __ballot_sync(FULL, static_cast<u64>(incl) >= need);
  if (ballot == 0) {  // fewer candidates than the leader's count: inconsistent state
    if (lane == 0) op.err = E_EVICT_MISMATCH;
    *rank_in_bin = 1;
    return 0;
  }
  const int L = __ffs(ballot) - 1;  // first lane whose inclusive prefix reaches need
  u64 cum = __shfl_sync(FULL, incl - local, L);
  u32 bin = 0;
  if (lane == L) {
    u32 i = 0;
    for (; i + 1 < per; ++i) {
      const u32 c = __ldcg(&h.cnt[base + i]);
      if (cum + c >= need) break;
      cum += c;
    }
    bin = base + i;
  }
  bin = __shfl_sync(FULL, bin, L);
  cum = __shfl_sync(FULL, cum, L);
  *rank_in_bin = need - cum;
  if (lane == 0) {
    op.need = need - cum;
    op.prefix = (op.prefix << d) | bin;
  }
  return bin;
}

// EVICT (cache_tree.cpp:270-319, per-page form SURVEY.md A.2): free the
// op.k smallest (stamp asc, page index desc) resident unpinned pages.
// Radix select over stamps (9-bit digits, shared-memory histogram with
// warp-aggregated atomics), exact threshold stamp T and the deepest-j cut
// inside it (equal stamps lie on one root path), then one scatter pass.
__device__ __noinline__ void coop_evict(Op& op, Hist& h, int tid, int warp, int lane, int nw) {
  const int nt = nw * 32;
  if (tid == 0) {
    op.all = op.k >= op.evictable;
    op.prefix = 0;
    op.need = op.k;
    op.freed = 0;
  }
  __syncthreads();
  const bool all = op.all;
  u64 T = 0, cut = 0;
  if (!all) {
    int lo_bits = 64 - __clzll(op.clock | 1ull);
    while (lo_bits > 0) {
      const int d = lo_bits < 9 ? lo_bits : 9;
      const int shift = lo_bits - d;
      const bool last = shift == 0;
      const u32 nbins = 1u << d;
      for (u32 i = tid; i < nbins; i += nt) {
        __stcg(&h.cnt[i], 0u);
        __stcg(&h.dmax[i], 0u);
      }
      __syncthreads();
      const u64 prefix = op.prefix;
      scan_buckets(op, warp, lane, nw, [&](u32, const Slot& s, u64 thr) {
        const u64 st = m_stamp(s.meta);
        const bool act = is_candidate(op, s, thr) && (st >> lo_bits) == prefix;
        const u32 bin = act ? static_cast<u32>((st >> shift) & (nbins - 1)) : 0xffffffffu;
        const unsigned peers = __match_any_sync(FULL, bin);
        if (act) {
          const int leader = __ffs(peers) - 1;
          if (lane == leader) atomicAdd(&h.cnt[bin], static_cast<u32>(__popc(peers)));
          if (last) {
            const u32 depth = static_cast<u32>(s.key & 0xffffffffu);
            const u32 mx = __reduce_max_sync(peers, depth);
            if (lane == leader) atomicMax(&h.dmax[bin], mx);
          }
        }
      });
      __syncthreads();
      if (warp == 0) {
        u64 rank = 0;
        const u32 bin = select_bin(op, h, nbins, d, lane, &rank);
        if (last && lane == 0) op.cut_depth = static_cast<u64>(__ldcg(&h.dmax[bin])) + 1 - rank;
      }
      __syncthreads();
      lo_bits = shift;
    }
    T = op.prefix;
    cut = op.cut_depth;
  }
  // scatter-free pass
  unsigned int freed = 0;
  scan_buckets(op, warp, lane, nw, [&](u32 b, const Slot& s, u64 thr) {
    if (!is_candidate(op, s, thr)) return;
    const u64 st = m_stamp(s.meta);
    const u64 depth = s.key & 0xffffffffu;
    if (all || st < T || (st == T && depth >= cut)) {
      st_meta(&op.table[(size_t)b * kChunk + lane], 0ull);
      ++freed;
      if (op.log_victims) emit_victim(op, s.key, st, op.agent);
    }
  });
  for (int o = 16; o > 0; o >>= 1) freed += __shfl_down_sync(FULL, freed, o);
  if (lane == 0 && freed) atomicAdd(&op.freed, freed);
}

// SCANFREE: free resident pages with index >= p0 and (owner == owner_filter
// or owner_filter == ~0). Cache-API discard_suffix below a shared head.
__device__ __noinline__ void coop_scanfree(Op& op, int warp, int lane, int nw) {
  unsigned int freed = 0;
  int err = 0;
  scan_buckets(op, warp, lane, nw, [&](u32 b, const Slot& s, u64) {
    if (!(s.meta & kResident)) return;
    const u64 owner = s.key >> 32, idx = s.key & 0xffffffffu;
    if (idx < op.p0) return;
    if (op.owner_filter != ~0ull && owner != op.owner_filter) return;
    if (m_pins(s.meta)) {
      err = E_DISCARD_PINNED;
      return;
    }
    st_meta(&op.table[(size_t)b * kChunk + lane], 0ull);
    ++freed;
  });
  for (int o = 16; o > 0; o >>= 1) {
    freed += __shfl_down_sync(FULL, freed, o);
    int oe = __shfl_down_sync(FULL, err, o);
    err = oe > err ? oe : err;
  }
  if (lane == 0) {
    if (freed) atomicAdd(&op.freed, freed);
    if (err) atomicMax(&op.err, err);
  }
}

// REBUILD: copy buckets holding at least one resident page into the
// alternate table (pre-cleared here), then swap tables.
__device__ __noinline__ void coop_rebuild(Op& op, int tid, int warp, int lane, int nw) {
  const int nt = nw * 32;
  const size_t nslots = (static_cast<size_t>(op.mask) + 1) * kChunk;
  for (size_t i = tid; i < nslots; i += nt) {
    __stcg(&op.alt[i].key, kEmptyKey);
    __stcg(&op.alt[i].meta, kEmptyKey);
  }
  if (tid == 0) op.alt_n = 0;
  __syncthreads();
  const unsigned int n_occ = op.occ_n;
  for (u32 i = warp; i < n_occ; i += nw) {
    const u32 b = __ldcg(&op.occ[i]);
    const Slot s = ld_slot(&op.table[(size_t)b * kChunk + lane]);
    if (!__any_sync(FULL, (s.meta & kResident) != 0)) continue;
    const u64 tag = __shfl_sync(FULL, s.key, 0);
    u32 nb = static_cast<u32>(hash64(tag)) & op.mask;
    nb = claim(op, op.alt, op.alt_occ, &op.alt_n, op.mask, tag, nb, lane);
    __stcg(&op.alt[(size_t)nb * kChunk + lane].meta, s.meta);
  }
  __syncthreads();
  if (tid == 0) {
    Slot* t = op.table;
    op.table = op.alt;
    op.alt = t;
    u32* o = op.occ;
    op.occ = op.alt_occ;
    op.alt_occ = o;
    op.occ_n = op.alt_n;
  }
}

}  // namespace kvg

// ==========================================================================
// The engine leader: event loop, controller, dispatch, handlers.
// ==========================================================================

#include "leader.cuh"

namespace kvg {

// Compacts each simulation's trace rows (ragged, capacity-strided in HBM)
// into one dense array so the host receives them in a single DMA.
// Block b copies sim b's rows as 8-byte words (rows are 88 B, so a 16-byte
// vector would misalign at odd row offsets).
__global__ void __launch_bounds__(256) pack_traces(const SimDev* __restrict__ sims,
                                                   const u64* __restrict__ dst_off,
                                                   kvg_trace_row* __restrict__ packed) {
  const SimDev& D = sims[blockIdx.x];
  const u64 rows = D.counts[0] < D.trace_cap ? D.counts[0] : D.trace_cap;
  const u64* src = reinterpret_cast<const u64*>(D.trace);
  u64* dst = reinterpret_cast<u64*>(packed + dst_off[blockIdx.x]);
  const u64 words = rows * sizeof(kvg_trace_row) / sizeof(u64);
  for (u64 i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldcs(src + i);
}

}  // namespace kvg
