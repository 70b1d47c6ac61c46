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
//  * the discard-mode cache is held in CHAIN form on the benchmarked path
//    (verify off: per-agent chains, stamp-ordered eviction, no page table,
//    leader.cuh); with verify on, and in the CacheTree seam, it is the page
//    table below and the leader posts COOPERATIVE OPS the CTA executes:
//      RANGE   warp-cooperative block-hash prefix lookup / stamp refresh /
//              pin / create / free over an agent's page range (kernel 1),
//      EVICT   radix select over the bucket summaries' last-use stamps plus
//              a scatter that frees the chosen pages (kernel 2),
//      REBUILD rehash of live buckets into the alternate table;
//    grid-wide forms of kernels 1-2 for big tables are in grid.cuh;
//  * warp-cooperative leader steps: pipelined control ticks (kernel 3),
//    completion-group advance of the agent state machines and stall-storm
//    runs (kernel 4), phase labels, trace-row streaming (leader.cuh). The
//    reference's strictly sequential event order (engine.cpp:98-136) leaves no
//    independent work for a launch per tick, so all of it lives in one
//    persistent kernel per batch.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>

#include "kvg_device.h"

namespace kvg {

constexpr unsigned FULL = 0xffffffffu;
constexpr u32 NIL32 = 0xffffffffu;

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
  OP_FRONTIER,   // offload tree: compact eviction-frontier nodes (tree.cuh)
  OP_TICKS,      // warp 0: pipelined control ticks + no-op admission checks
  OP_PHASES,     // warp 0: phase labels over the trace rows
  OP_GROUP,      // warp 0: a dispatch batch's completions advanced together
  OP_STORM,      // warp 0: a run of dispatch attempts that all stall, together
  OP_FLUSH,      // warp 0: stream pending trace rows to the host block
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
  u64 lazy_sh;          // engine mode: stamp of every resident shared page
  unsigned int l0_min;  // engine mode: smallest shared page an eviction freed
  AgentDev* agents;
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
  Summ* summ;
  Summ* alt_summ;
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
  // offload tree frontier scan
  const TNodeDev* tnodes;
  FrEnt* fr;
  u32 t_n;
  unsigned int fr_n;
  u32 tw_off, tw_n;  // the shared-memory mirror (tree.cuh): ids [0, tw_n)
};

constexpr int kBins = 512;

// Radix-select histogram: in shared memory wherever the CTA has room (the
// one-CTA-per-SM kernels, the CacheTree seam, the grid select); in
// per-simulation global scratch (L2) in the 28-CTA/SM sweep kernel, whose
// shared memory holds the hot agent records. Global bins are read with
// L1-bypassing loads (other warps update them with L2 atomics).
struct Hist {
  unsigned int* cnt;   // [kBins]
  unsigned int* dmax;  // [kBins]
  bool smem;
};
__device__ __forceinline__ u32 hist_ld(const Hist& h, const unsigned int* p) {
  return h.smem ? *reinterpret_cast<const volatile unsigned int*>(p) : __ldcg(p);
}
__device__ __forceinline__ void hist_zero(const Hist& h, unsigned int* p) {
  if (h.smem) *p = 0u;
  else __stcg(p, 0u);
}

__device__ __forceinline__ Summ ld_summ(const Summ* p) {
  const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p);
  const ulonglong2 a = __ldcg(q), b = __ldcg(q + 1);
  Summ s;
  s.tag = a.x;
  s.sf = a.y;
  s.dev = static_cast<u32>(b.x);
  s.host = static_cast<u32>(b.x >> 32);
  s.bnd = static_cast<u32>(b.y);
  s.pad = 0;
  return s;
}

// Rewrites bucket b's summary from the per-lane metas the calling warp holds
// (every lane of the warp must call; lane l owns slot l).
__device__ __forceinline__ void summ_write(Summ* summ, u32 b, u64 m, int lane) {
  const bool res = (m & kResident) != 0;
  const u32 dev = __ballot_sync(FULL, res);
  const u64 st = m_stamp(m);
  const int l0 = dev ? __ffs(dev) - 1 : 0;
  const u64 s0 = __shfl_sync(FULL, st, l0);
  const bool mixed = __any_sync(FULL, res && (st != s0 || m_pins(m) != 0));
  if (lane == 0) {
    Summ* e = &summ[b];
    __stcg(&e->sf, (dev ? s0 : 0ull) | (mixed ? kMixed : 0ull));
    __stcg(&e->dev, dev);
  }
}

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

// Claims an empty bucket for `tag`, starting at bucket `b`; returns it. The
// bucket's summary starts empty.
__device__ __noinline__ u32 claim(Slot* table, Summ* summ, u32* occ, unsigned int* occ_n,
                                  u32 mask, u64 tag, u32 b, int lane, bool seen_empty = false) {
  for (;;) {
    int won = 0;
    if (lane == 0) {
      // the probe that led here already saw bucket b empty: go straight to
      // the CAS (one DRAM round trip less); a lost race falls back to the scan
      const u64 k0 = seen_empty ? kEmptyKey : __ldcg(&table[(size_t)b * kChunk].key);
      if (k0 == kEmptyKey)
        won = atomicCAS(reinterpret_cast<unsigned long long*>(&table[(size_t)b * kChunk].key),
                        kEmptyKey, tag) == kEmptyKey;
    }
    seen_empty = false;
    won = __shfl_sync(FULL, won, 0);
    if (won) {
      Slot* s = &table[(size_t)b * kChunk + lane];
      if (lane != 0) __stcg(&s->key, tag + lane);
      __stcg(&s->meta, 0ull);
      if (lane == 0) {
        ulonglong2* q = reinterpret_cast<ulonglong2*>(&summ[b]);
        __stcg(q, make_ulonglong2(tag, 0ull));
        __stcg(q + 1, make_ulonglong2(0ull, 0ull));
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
// `found` is warp-uniform. Every lane reports its slot's final meta so the
// warp can rewrite the bucket summary when anything changed.
__device__ __forceinline__ void range_chunk(Op& op, u64 tag, u64 lo, u64 hi, u32 b, Slot s,
                                            bool found, int lane, RangeAcc& acc) {
  const u32 flags = op.flags;
  const int delta = op.pin_delta;
  const u64 page = (tag & 0xffffffffull) + lane;
  const bool in = page >= lo && page < hi;
  if (!found && (flags & RF_CREATE) && __any_sync(FULL, in)) {
    b = claim(op.table, op.summ, op.occ, &op.occ_n, op.mask, tag, b, lane, true);
    found = true;
    s = Slot{tag + lane, 0};
  }
  if (!found) {
    if (in) {
      acc.miss = page < acc.miss ? page : acc.miss;
      if (flags & RF_STRICT) acc.err = E_PIN_MISSING;
    }
    return;
  }
  const u64 m = s.meta;
  u64 nm = m;
  if (in) {
    if (!(m & kResident)) {
      if (flags & RF_CREATE) {
        const u64 pins = delta > 0 ? static_cast<u64>(delta) : 0;
        nm = m_make(op.stamp, pins);
        ++acc.created;
        if (pins) ++acc.up;
      } else {
        acc.miss = page < acc.miss ? page : acc.miss;
        if (flags & RF_STRICT) acc.err = E_PIN_MISSING;
      }
    } else {
      ++acc.resident;
      if (flags & RF_FREE) {
        if (!op.implicit_pins && m_pins(m) != 0) {
          acc.err = E_DISCARD_PINNED;
        } else {
          nm = 0ull;
          ++acc.freed;
        }
      } else {
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
        nm = m_make(stamp, static_cast<u64>(pins));
      }
    }
  }
  const bool wrote = nm != m;
  if (wrote) st_meta(&op.table[(size_t)b * kChunk + lane], nm);
  if (__any_sync(FULL, wrote)) summ_write(op.summ, b, nm, lane);
}

// RANGE: agent `op.agent`, pages [p0, p1). Pages below shared_pages belong to
// the shared prompt (owner 0), the rest to owner agent+1 (workload.cpp:167-171).
// Each warp owns every nw-th 32-page chunk and keeps kProbeDepth bucket probes
// in flight (one 512 B coalesced load each) before consuming any of them, so a
// context of C chunks costs ~C/(nw*kProbeDepth) DRAM round trips, not C
// (depth 8 for the big-sim kernel, 4 for the register-lean 1-warp kernel). The
// in-flight probes rotate through registers (no dynamically indexed arrays,
// so nothing spills to local memory).
template <int kProbeDepth>
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
  const u64 step = static_cast<u64>(nw);
  for (u64 base = warp; base < total; base += step * kProbeDepth) {
    Slot s[kProbeDepth];
    u32 b[kProbeDepth];
#pragma unroll
    for (int g = 0; g < kProbeDepth; ++g) {
      const u64 it = base + static_cast<u64>(g) * step;
      b[g] = 0;
      s[g] = Slot{kEmptyKey, 0};
      if (it < total) {
        b[g] = static_cast<u32>(hash64(tag_of(it))) & op.mask;
        s[g] = ld_slot(&op.table[(size_t)b[g] * kChunk + lane]);
      }
    }
    const u64 left = (total - base + step - 1) / step;
    const int cnt = left < kProbeDepth ? static_cast<int>(left) : kProbeDepth;
#pragma unroll 1
    for (int g = 0; g < cnt; ++g) {
      const u64 it = base + static_cast<u64>(g) * step;
      Slot cur = s[0];
      u32 cb = b[0];
#pragma unroll
      for (int j = 0; j + 1 < kProbeDepth; ++j) {
        s[j] = s[j + 1];
        b[j] = b[j + 1];
      }
      const u64 tag = tag_of(it);
      const u64 k0 = __shfl_sync(FULL, cur.key, 0);
      bool found;
      if (k0 == tag) {
        found = true;
      } else if (k0 == kEmptyKey) {
        found = false;
      } else {
        found = probe_from(op, tag, (cb + 1) & op.mask, lane, &cb, &cur);
      }
      const bool shared = it < n_sh;
      range_chunk(op, tag, shared ? s_lo : q_lo, shared ? s_hi : q_hi, cb, cur, found, lane, acc);
    }
  }
  // warp reductions (one REDUX each), then one shared atomic per warp
  const u32 created = __reduce_add_sync(FULL, acc.created);
  const u32 freed = __reduce_add_sync(FULL, acc.freed);
  const u32 up = __reduce_add_sync(FULL, acc.up);
  const u32 down = __reduce_add_sync(FULL, acc.down);
  const u32 resident = __reduce_add_sync(FULL, acc.resident);
  const u32 miss = __reduce_min_sync(FULL, acc.miss == ~0ull ? NIL32 : static_cast<u32>(acc.miss));
  const u32 err = __reduce_max_sync(FULL, static_cast<u32>(acc.err));
  if (lane == 0) {
    if (created) atomicAdd(&op.created, created);
    if (freed) atomicAdd(&op.freed, freed);
    if (up) atomicAdd(&op.pin_up, up);
    if (down) atomicAdd(&op.pin_down, down);
    if (resident) atomicAdd(&op.resident, resident);
    if (miss != NIL32) atomicMin(&op.first_miss, static_cast<unsigned long long>(miss));
    if (err) atomicMax(&op.err, static_cast<int>(err));
  }
}

// Visits every claimed bucket, one WARP per bucket (lane l holds slot l):
// the whole-bucket passes (suffix discard, rehash). kScanDepth buckets in
// flight per warp, rotated through registers.
#ifndef KVG_SCAN_DEPTH
#define KVG_SCAN_DEPTH 2
#endif
constexpr int kScanDepth = KVG_SCAN_DEPTH;

template <typename F>
__device__ __forceinline__ void scan_buckets(const Op& op, int warp, int lane, int nw, F&& f) {
  const unsigned int n_occ = op.occ_n;
  for (u32 base = warp; base < n_occ; base += static_cast<u32>(nw) * kScanDepth) {
    u32 bk[kScanDepth];
    Slot s[kScanDepth];
#pragma unroll
    for (int g = 0; g < kScanDepth; ++g) {
      const u32 i = base + g * nw;
      bk[g] = i < n_occ ? __ldcg(&op.occ[i]) : 0u;
    }
#pragma unroll
    for (int g = 0; g < kScanDepth; ++g) {
      const u32 i = base + g * nw;
      s[g] = Slot{kEmptyKey, 0};
      if (i < n_occ) s[g] = ld_slot(&op.table[(size_t)bk[g] * kChunk + lane]);
    }
    const u32 left = (n_occ - base + nw - 1) / nw;
    const int cnt = left < kScanDepth ? static_cast<int>(left) : kScanDepth;
#pragma unroll 1
    for (int g = 0; g < cnt; ++g) {
      const u32 cb = bk[0];
      const Slot cur = s[0];
#pragma unroll
      for (int j = 0; j + 1 < kScanDepth; ++j) {
        bk[j] = bk[j + 1];
        s[j] = s[j + 1];
      }
      f(cb, cur);
    }
  }
}

// Visits every claimed bucket's SUMMARY, one LANE per bucket: the eviction
// select's input. kSumDepth summaries in flight per lane; f(valid, bucket,
// summary) is called by every lane of the warp together (warp-convergent, so
// f may use warp collectives).
#ifndef KVG_SUM_DEPTH
#define KVG_SUM_DEPTH 2
#endif
constexpr int kSumDepth = KVG_SUM_DEPTH;

template <int kDepth = kSumDepth, typename F>
__device__ __forceinline__ void scan_summ(const Op& op, int warp, int lane, int nw, F&& f) {
  const u32 n_occ = op.occ_n;
  const u32 stride = static_cast<u32>(nw) * 32u * kDepth;
  for (u32 base = static_cast<u32>(warp) * 32u * kDepth; base < n_occ; base += stride) {
    u32 bk[kDepth];
    Summ e[kDepth];
#pragma unroll
    for (int g = 0; g < kDepth; ++g) {
      const u32 i = base + g * 32u + lane;
      bk[g] = i < n_occ ? __ldcg(&op.occ[i]) : NIL32;
    }
#pragma unroll
    for (int g = 0; g < kDepth; ++g) {
      e[g] = Summ{0, 0, 0, 0, 0, 0};
      if (bk[g] != NIL32) e[g] = ld_summ(&op.summ[bk[g]]);
    }
    // one copy of f's body: the loads above stay in flight, the calls rotate
    // through registers (f is large: the radix-select histogram step)
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

__device__ __forceinline__ u32 ge_mask(u64 base, u64 thr) {  // slots with page index >= thr
  if (thr <= base) return FULL;
  const u64 d = thr - base;
  return d >= 32 ? 0u : (FULL << d);
}

__device__ __forceinline__ u32 lt_mask(u64 base, u64 lim) {  // slots with page index < lim
  if (lim <= base) return 0u;
  const u64 d = lim - base;
  return d >= 32 ? FULL : ((1u << d) - 1u);
}

// Engine mode: a finished agent's private pages at or beyond its held length
// (the discarded suffix) are absent even if still in the table. Only finished
// agents hold such pages (evictions free pages physically), and their held
// length is at most one page past the shared prompt, so the eviction
// scatter's concurrent atomicMin on live agents' lengths never feeds back
// into a candidate mask.
__device__ __forceinline__ u32 held_mask(const Op& op, u64 tag) {
  const u64 owner = tag >> 32;
  if (owner == 0) return FULL;
  const AgentDev& a = op.agents[owner - 1];
  if (a.state != S_DONE) return FULL;
  return lt_mask(tag & 0xffffffffull, op.shared_pages + a.priv);
}

__device__ __forceinline__ u64 pin_thr(const Op& op, u64 owner) {
  // plain load: the records may live in shared memory (the leader wrote them
  // before the barrier that started this op)
  return owner == 0 ? op.pin_max : static_cast<u64>(op.agents[owner - 1].pinned_pg);
}

// Eviction candidates of a summarised (non-mixed) bucket: resident and
// unpinned (cache_tree.cpp:230-234 per page). Engine mode: page (owner, idx)
// is pinned iff idx < its owner's pinned prefix.
__device__ __forceinline__ u32 cand_of(const Op& op, const Summ& e) {
  if (!op.implicit_pins) return e.dev;  // explicit pins make a bucket mixed
  return e.dev & ge_mask(e.tag & 0xffffffffull, pin_thr(op, e.tag >> 32)) & held_mask(op, e.tag);
}

// Stamp of a summarised bucket's resident pages. Engine mode: every
// resident page of a chain carries its chain's latest refresh stamp (the
// shared chain: op.lazy_sh; agent a's private chain: agents[a].lazy), so raw
// page stamps are never consulted.
__device__ __forceinline__ u64 stamp_of(const Op& op, const Summ& e) {
  if (!op.implicit_pins) return e.sf & kStampMask;
  const u64 owner = e.tag >> 32;
  return owner == 0 ? op.lazy_sh : op.agents[owner - 1].lazy;
}

// Per-page candidate test (mixed buckets).
__device__ __forceinline__ bool page_cand(const Op& op, u64 key, u64 meta) {
  if (!(meta & kResident)) return false;
  if (op.implicit_pins) return (key & 0xffffffffull) >= pin_thr(op, key >> 32);
  return m_pins(meta) == 0;
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
  for (u32 k = 0; k < per; ++k) {  // lane-rotated order: ~no bank conflicts in shared memory
    const u32 i = (k + lane) % per;
    if (base + i < nbins) local += hist_ld(h, &h.cnt[base + i]);
  }
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
      const u32 c = hist_ld(h, &h.cnt[base + i]);
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

// Histogram contribution of a mixed bucket, page by page (one lane).
__device__ __noinline__ void hist_mixed(const Op& op, Hist& h, u32 b, u64 prefix, int lo_bits,
                                        int shift, u32 nbins, bool last) {
  const Slot* bk = &op.table[(size_t)b * kChunk];
  for (int l = 0; l < kChunk; ++l) {
    const Slot s = ld_slot(&bk[l]);
    if (!page_cand(op, s.key, s.meta)) continue;
    const u64 st = m_stamp(s.meta);
    if ((st >> lo_bits) != prefix) continue;
    const u32 bin = static_cast<u32>((st >> shift) & (nbins - 1));
    atomicAdd(&h.cnt[bin], 1u);
    if (last) atomicMax(&h.dmax[bin], static_cast<u32>(s.key & 0xffffffffu));
  }
}

// Scatter-free of a mixed bucket, page by page (one lane). Returns pages freed.
__device__ __noinline__ u32 scatter_mixed(Op& op, u32 b, bool all, u64 T, u64 cut) {
  Slot* bk = &op.table[(size_t)b * kChunk];
  u32 freed = 0, dev = 0;
  for (int l = 0; l < kChunk; ++l) {
    const Slot s = ld_slot(&bk[l]);
    const bool res = (s.meta & kResident) != 0;
    if (res && page_cand(op, s.key, s.meta)) {
      const u64 st = m_stamp(s.meta);
      const u64 depth = s.key & 0xffffffffu;
      if (all || st < T || (st == T && depth >= cut)) {
        st_meta(&bk[l], 0ull);
        ++freed;
        if (op.log_victims) emit_victim(op, s.key, st, op.agent);
        continue;
      }
    }
    if (res) dev |= 1u << l;
  }
  __stcg(&op.summ[b].dev, dev);
  return freed;
}

// EVICT (cache_tree.cpp:270-319, per-page form SURVEY.md A.2): free the
// op.k smallest (stamp asc, page index desc) resident unpinned pages.
// Radix select over stamps (9-bit digits) on the bucket SUMMARIES, one lane
// per bucket with weight popc(candidates): the histogram holds page counts,
// warp-aggregated through __match_any_sync / __reduce_add_sync. It finds the
// exact threshold stamp T and the cut depth inside it (equal stamps lie on
// one root path, so "deepest j" is a depth cut); one scatter pass then frees
// the chosen pages and rewrites the summaries.
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
        hist_zero(h, &h.cnt[i]);
        hist_zero(h, &h.dmax[i]);
      }
      __syncthreads();
      const u64 prefix = op.prefix;
      scan_summ(op, warp, lane, nw, [&](bool valid, u32 b, const Summ& e) {
        const bool mixed = valid && !op.implicit_pins && (e.sf & kMixed);
        u32 c = 0;
        u64 st = 0;
        if (valid && !mixed) {
          c = cand_of(op, e);
          st = stamp_of(op, e);
        }
        const bool act = c != 0 && (st >> lo_bits) == prefix;
        const u32 bin = act ? static_cast<u32>((st >> shift) & (nbins - 1)) : 0xffffffffu;
        const unsigned peers = __match_any_sync(FULL, bin);
        if (act) {
          const int leader = __ffs(peers) - 1;
          const u32 w = __reduce_add_sync(peers, static_cast<u32>(__popc(c)));
          if (lane == leader) atomicAdd(&h.cnt[bin], w);
          if (last) {
            const u32 dm = static_cast<u32>(e.tag & 0xffffffffu) + 31u - __clz(c);
            const u32 mx = __reduce_max_sync(peers, dm);
            if (lane == leader) atomicMax(&h.dmax[bin], mx);
          }
        }
        if (mixed) hist_mixed(op, h, b, prefix, lo_bits, shift, nbins, last);
      });
      __syncthreads();
      if (warp == 0) {
        u64 rank = 0;
        const u32 bin = select_bin(op, h, nbins, d, lane, &rank);
        if (last && lane == 0) op.cut_depth = static_cast<u64>(hist_ld(h, &h.dmax[bin])) + 1 - rank;
      }
      __syncthreads();
      lo_bits = shift;
    }
    T = op.prefix;
    cut = op.cut_depth;
  }
  // scatter-free pass
  unsigned int freed = 0;
  scan_summ(op, warp, lane, nw, [&](bool valid, u32 b, const Summ& e) {
    if (!valid) return;
    if (!op.implicit_pins && (e.sf & kMixed)) {
      freed += scatter_mixed(op, b, all, T, cut);
      return;
    }
    const u32 c = cand_of(op, e);
    if (c == 0) return;
    const u64 st = stamp_of(op, e);
    const u32 v = (all || st < T) ? c : (st == T ? c & ge_mask(e.tag & 0xffffffffull, cut) : 0u);
    if (v == 0) return;
    freed += __popc(v);
    if (op.implicit_pins) {  // chains lose tails: the lowest victim is the new length
      const u64 owner = e.tag >> 32;
      const u32 low = static_cast<u32>(e.tag & 0xffffffffull) + static_cast<u32>(__ffs(v) - 1);
      if (owner == 0) atomicMin(&op.l0_min, low);
      else atomicMin(&op.agents[owner - 1].priv, low - static_cast<u32>(op.shared_pages));
    }
    Slot* bk = &op.table[(size_t)b * kChunk];
    for (u32 m = v; m != 0; m &= m - 1) {
      const int l = __ffs(m) - 1;
      st_meta(&bk[l], 0ull);
      if (op.log_victims) emit_victim(op, e.tag + l, st, op.agent);
    }
    __stcg(&op.summ[b].dev, e.dev & ~v);
  });
  freed = __reduce_add_sync(FULL, freed);
  if (lane == 0 && freed) atomicAdd(&op.freed, freed);
}

// SCANFREE: free resident pages with index >= p0 and (owner == owner_filter
// or owner_filter == ~0). Cache-API discard_suffix below a shared head.
__device__ __noinline__ void coop_scanfree(Op& op, int warp, int lane, int nw) {
  unsigned int freed = 0;
  int err = 0;
  scan_buckets(op, warp, lane, nw, [&](u32 b, const Slot& s) {
    u64 nm = s.meta;
    if (s.meta & kResident) {
      const u64 owner = s.key >> 32, idx = s.key & 0xffffffffu;
      if (idx >= op.p0 && (op.owner_filter == ~0ull || owner == op.owner_filter)) {
        if (m_pins(s.meta)) {
          err = E_DISCARD_PINNED;
        } else {
          nm = 0ull;
          st_meta(&op.table[(size_t)b * kChunk + lane], 0ull);
          ++freed;
        }
      }
    }
    if (__any_sync(FULL, nm != s.meta)) summ_write(op.summ, b, nm, lane);
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

// REBUILD: copy buckets holding at least one resident page (with their
// summaries) into the alternate table (pre-cleared here), then swap tables.
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
    const u64 tag = __shfl_sync(FULL, s.key, 0);
    // engine mode: pages beyond their chain's held length are not copied
    const bool live = (s.meta & kResident) != 0 &&
                      (!op.implicit_pins || ((held_mask(op, tag) >> lane) & 1u));
    if (!__any_sync(FULL, live)) continue;
    u32 nb = static_cast<u32>(hash64(tag)) & op.mask;
    nb = claim(op.alt, op.alt_summ, op.alt_occ, &op.alt_n, op.mask, tag, nb, lane);
    const u64 m = live ? s.meta : 0ull;
    __stcg(&op.alt[(size_t)nb * kChunk + lane].meta, m);
    summ_write(op.alt_summ, nb, m, lane);
  }
  __syncthreads();
  if (tid == 0) {
    Slot* t = op.table;
    op.table = op.alt;
    op.alt = t;
    u32* o = op.occ;
    op.occ = op.alt_occ;
    op.alt_occ = o;
    Summ* sm = op.summ;
    op.summ = op.alt_summ;
    op.alt_summ = sm;
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

#include "grid.cuh"

namespace kvg {
// Test hook (kvg_check_ready_next): both forms of the ready-set walk over a
// caller's two-level bitmap, one query per thread.
__global__ void ready_probe_kernel(const u32* rbits, const u32* rl1, u32 n, const u32* from,
                                   u32 nq, u32* out_narrow, u32* out_wide) {
  Lead L;
  L.n = n;
  L.nwords = (n + 31) / 32;
  L.rbits = const_cast<u32*>(rbits);
  L.rl1 = const_cast<u32*>(rl1);
  SimDev D;
  for (u32 q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    out_narrow[q] = ready_next(D, L, from[q]);
    out_wide[q] = ready_next_wide(D, L, from[q]);
  }
}
}  // namespace kvg

namespace kvg_engine_cfg {
cudaError_t check_ready_next(const unsigned* rbits, const unsigned* rl1, unsigned n,
                             const unsigned* from, unsigned nq, unsigned* out_narrow,
                             unsigned* out_wide) {
  const unsigned nblocks = (nq + 255) / 256 < 1024 ? (nq + 255) / 256 : 1024;
  kvg::ready_probe_kernel<<<nblocks ? nblocks : 1, 256>>>(rbits, rl1, n, from, nq, out_narrow,
                                                          out_wide);
  return cudaGetLastError();
}
}  // namespace kvg_engine_cfg

#ifdef KVG_GRID_PROF
extern "C" __attribute__((visibility("default"))) int kvg_debug_gprof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, kvg::g_gprof, sizeof(kvg::g_gprof));
  return 0;
}
#endif

#ifdef KVG_PROFILE
// dev-only: read and clear the phase profile (tools/probe_phases.py)
extern "C" __attribute__((visibility("default"))) int kvg_debug_profile(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, kvg::g_prof, sizeof(kvg::g_prof));
  static const unsigned long long zero[48] = {0};
  cudaMemcpyToSymbol(kvg::g_prof, zero, sizeof(zero));
  return 0;
}
#endif

// --------------------------------------------------------------------------
// Host glue of the offload-mode CacheTree seam (used by capi.cu, which does
// not see the Lead layout).
namespace kvg_tree_seam {

size_t state_bytes() { return sizeof(kvg::TreeCacheDev); }

cudaError_t init(void* d_state, const kvg::SimDev& sim, unsigned long long capacity,
                 unsigned long long page_size, unsigned long long shared_pages) {
  kvg::TreeCacheDev h;
  std::memset(&h, 0, sizeof h);
  h.sim = sim;
  h.lead.capacity = capacity;
  h.lead.capacity_d = static_cast<double>(capacity);
  h.lead.ps = page_size;
  h.lead.ps_shift = (page_size & (page_size - 1)) == 0 ? __builtin_ctzll(page_size) : -1;
  h.lead.S = shared_pages;
  h.lead.offload = 1;
  h.lead.log_on = sim.log != nullptr;  // victims are reported through the log
  cudaError_t e = cudaMemcpy(d_state, &h, sizeof h, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  kvg::cache_tree_init<<<1, 1>>>(static_cast<kvg::TreeCacheDev*>(d_state));
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e;
}

cudaError_t exec(void* d_state, const kvg_cache_op* d_ops, unsigned n, kvg_cache_op_result* d_res,
                 kvg_victim* d_vic, unsigned long long vic_cap, unsigned long long* d_nvic) {
  kvg::cache_tree_kernel<<<1, 32>>>(static_cast<kvg::TreeCacheDev*>(d_state), d_ops, n, d_res,
                                    d_vic, vic_cap, d_nvic);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e;
}

cudaError_t hit_window(const void* d_state, double* m, double* r) {
  kvg::TreeCacheDev h;
  cudaError_t e = cudaMemcpy(&h, d_state, sizeof h, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) {
    *m = h.lead.hit_m;
    *r = h.lead.hit_r;
  }
  return e;
}

}  // namespace kvg_tree_seam

// --------------------------------------------------------------------------
// Host glue of the grid-wide seam kernels (grid.cuh), used by capi.cu.
namespace kvg_grid_seam {

// Launch geometry (SM count and occupancy), computed once per device and
// cached, so no host-side query runs inside a timed launch window.
struct Geom {
  int sms = 0, match_per_sm = 0, evict_per_sm = 0;
};
static Geom geom_of(int dev) {
  static Geom g[64];
  static bool have[64] = {false};
  if (dev < 0 || dev >= 64) dev = 0;
  if (!have[dev]) {
    Geom x;
    cudaDeviceGetAttribute(&x.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x.match_per_sm, kvg::grid_match_kernel,
                                                  kvg::kGridMatchWarps * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x.evict_per_sm, kvg::grid_evict_kernel, 512, 0);
    x.sms = x.sms > 0 ? x.sms : 1;
    x.match_per_sm = x.match_per_sm > 0 ? x.match_per_sm : 1;
    x.evict_per_sm = x.evict_per_sm > 0 ? (x.evict_per_sm < 2 ? x.evict_per_sm : 2) : 1;
    g[dev] = x;
    have[dev] = true;
  }
  return g[dev];
}

unsigned match_blocks(int dev) {
  const Geom g = geom_of(dev);
  return static_cast<unsigned>(g.sms * g.match_per_sm);
}

// no more CTAs than 32-bucket lane groups to scan (a grid barrier costs the
// same either way): one CTA per KVG_EVICT_UNIT claimed buckets
#ifndef KVG_EVICT_UNIT
#define KVG_EVICT_UNIT 512  // measured 4,096 / 2,048 / 1,024 / 512 / 256: C2-size evict 38 / 33 / 29 / 27 / 28 us
#endif
unsigned evict_blocks(int dev, unsigned occ_n) {
  const Geom g = geom_of(dev);
  unsigned blocks = static_cast<unsigned>(g.sms * g.evict_per_sm);
  const unsigned need = (occ_n + KVG_EVICT_UNIT - 1) / KVG_EVICT_UNIT;
  if (blocks > need) blocks = need > 0 ? need : 1;
  return blocks;
}

cudaError_t match(const kvg::GridMatchArgs& a, unsigned blocks, cudaStream_t s) {
  const unsigned need = (a.n + kvg::kGridMatchWarps - 1) / kvg::kGridMatchWarps;
  if (a.S > 0) kvg::grid_match_prep_kernel<<<1, 1024, 0, s>>>(a);
  kvg::grid_match_kernel<<<need < blocks ? (need ? need : 1) : blocks, kvg::kGridMatchWarps * 32, 0,
                           s>>>(a);
  if (a.max_groups > 1)
    kvg::grid_match_rest_kernel<<<blocks, kvg::kGridMatchWarps * 32, 0, s>>>(a);
  if (a.S > 0) kvg::grid_match_shared_kernel<<<1, 1024, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t evict(const kvg::GridEvictArgs& a, unsigned blocks, cudaStream_t s) {
  void* args[] = {const_cast<kvg::GridEvictArgs*>(&a)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kvg::grid_evict_kernel),
                                     dim3(blocks), dim3(512), args, 0, s);
}

}  // namespace kvg_grid_seam
