// Leader state machine of the B200 engine (included by engine.cu).
//
// Thread 0 of each CTA executes the reference's sequential semantics; every
// function below cites the reference lines it follows. Whenever page-level
// work is needed it posts a cooperative op (engine.cu) and returns; the CTA
// executes the op and thread 0 resumes at the continuation phase.
//
// Leader-only structures (no CTA involvement, shared memory for small sims):
//   * agent events: binary min-heap of (time, ordinal, agent) — equivalent to
//     the reference's priority queue since an agent has at most one pending
//     event; a dispatch batch's completions are ONE entry (a
//     completion group, kernel 4); tick and admission are two scalar slots;
//   * ready set: two-level bitmap of (active && AwaitingAdmission) agents,
//     iterated in id order exactly like dispatch_batch's sorted vector;
//   * pins: each agent holds at most one pin, on its own root prefix
//     [0, pinned_len) (engine.cpp:340-342, 374-377). The pin count of private
//     page (a, k) is [k < pinned_pg(a)] and of shared page k is
//     #{a : pinned_pg(a) > k}; only the prefix max matters for eviction, kept
//     with a histogram. No page-table pass is ever spent on pin/unpin;
//   * chain form of the discard-mode cache: per-agent chains
//     with one stamp each, evicted in stamp order (chain heap / scan).
#pragma once

namespace kvg {

constexpr u32 NIL = 0xffffffffu;
constexpr uint8_t EV_GROUP_POP = 0xff;  // popped heap key of a completion group

// Leader helpers called from many phases. Inlined: measured on C4, calls
// (register save/restore through local memory) cost more than the smaller
// code saves in instruction fetch (59.9 ms out of line vs 47.0 ms inlined).
#ifndef KVG_TICK_AHEAD  // pipelined ticks when at least KVG_TICK_AHEAD + 1 are due
#define KVG_TICK_AHEAD 3.0
#endif
#ifndef KVG_MID_FN  // helpers with many call sites: one out-of-line copy
#define KVG_MID_FN __forceinline__
#endif
#ifndef KVG_LEADER_FN
#define KVG_LEADER_FN __forceinline__
#endif
#ifndef KVG_PIN_FN  // set_pinned (8 call sites)
#define KVG_PIN_FN KVG_LEADER_FN
#endif
#ifndef KVG_READY_FN  // ready_sync / ready_next
#define KVG_READY_FN KVG_LEADER_FN
#endif

enum Phase : int {
  PH_EVENT = 0,
  PH_MEMBER,
  PH_M_MATCHED,
  PH_M_INSERT,
  PH_M_EVICTED,
  PH_M_COMMIT,
  PH_M_CREATED,
  PH_M_FAIL,
  PH_M_RESTORED,
  PH_BATCH_END,
  PH_GEN_DISCARDED,
  PH_GROUP_DONE,
  // offload mode (node-level tree, tree.cuh)
  PH_O_MEMBER,
  PH_O_RELOAD_CHUNK,
  PH_O_RELOAD_EVICTED,
  PH_O_RELOAD_END,
  PH_O_INSERT_START,
  PH_O_INSERT_COUNT,
  PH_O_INSERT_EVICTED,
  PH_O_INSERT_FAIL,
  PH_O_EVICT_POP,
  PH_DONE,
  PH_FINAL,
  PH_EXITED,
};

struct Lead {
  int phase, status, err, rebuilt;
  // event queue (engine.cpp:46-68, 139-154)
  double clock, gpu_busy, makespan, device_busy, tick_t, adm_t;
  u64 ord, tick_o, adm_o;
  int tick_on, adm_on;
  u32 hsize, finished, n_ready, ev_agent;
  // cache scalars (cache_tree.hpp:187-197)
  u64 used, cclock, discarded, lookups, agent_steps, events, evict_calls, evicted;
  u64 pin_max, pin_priv;  // implicit pins: shared prefix max, private pinned pages
  u64 L0, lazy_sh;        // discard mode: resident shared pages, their stamp
  int verify, pad4;
  u64 hit_pages, created_pages, refreshed_pages, evict_scanned, agent_events;
  long long t_start;
#ifdef KVG_GTIMER
  u64 g_start;
#endif
  double hit_m, hit_r;
  // controller (controller.hpp:117-126)
  double window, su, sh;
  int have_s, gated;
  u64 ticks;
  u32 act_seq, act_size, pend_head, pend_size, paus_head, paus_size, nwords, pad2;
  // metrics
  u64 decoded_cum, rec_cum;
  kvg_ledger ledger;
  unsigned long long n_trace, n_log;
  // dispatch context
  u32 batch_n, m_id, m_next, pad1;
  u64 m_ctx0, m_f, m_nctx, m_nafter, m_now, m_k, m_e;
  // hot per-agent structures: shared memory for small sims, else HBM
  AgentDev* ag;
  HeapEnt* heap;
  u32* rbits;
  u32* rl1;
  // config snapshot
  double interval, decay, horizon, capacity_d;
  u64 capacity, ps, shared_len, S;
  u32 n, steps, kind, cap;
  kvg_controller_config cfg;
  // offload mode: tree pool, link queue, dispatch continuation (tree.cuh)
  int offload, o_full, o_then, pad3;
  u32 t_alloc, t_free_n, x_head, x_size, o_node, o_c;
  u64 t_next_ord, offloaded, reloaded;
  u64 n_flushed;     // trace rows already streamed to D.trace_out (flush_rows)
  int stream_on;     // D.trace_out != nullptr and rows are not written through
  u32 log_on;        // D.log != nullptr
  double b_wall, b_total;  // dispatch batch: max and sum of member times so far
  int ps_shift;      // log2(ps) when ps is a power of two, else -1 (pdiv / pmod)
  u32 tw_off, tw_n;  // walk mirror of node ids [0, tw_n) at this dynamic-smem offset (tree.cuh)
  double pcie_busy, link_busy;
  double abort_t;    // event time that passed the horizon (KVG_ERR_HORIZON)
  // chain mode (discard, verify off): the cache is held as chains, no page
  // table. lru = the chain heap (big-sim kernel; nullptr: scan the records):
  // lru[0, n) heap of agent ids, lru[n, 2n) each agent's heap position
  // pages, in chain-stamp order
  u32* lru;
  u32 ch_n;
  int chain;
  // completion groups (kernel 4): member ring gring[0, n) (FIFO: groups
  // complete in dispatch order); the group being advanced starts at grp_start
  u32* gring;
  u32 gr_head, gr_n, grp_start, grp_cnt;
  u32 group_min;
  u32 stall_streak;  // consecutive stalled members in the current dispatch batch
  u32 storm_on;
  u64 o_matched, o_hm, o_promoted, o_offl, o_pos, o_ka, o_now, o_ev_need, o_ev_rec;
#ifdef KVG_PROFILE
  // dev-only phase profile (tools/probe_phases.py): cycles per leader phase,
  // per cooperative op kind, in fast_housekeeping
  u64 prof[48];
  long long prof_t;
  int prof_ph;
#endif
};

#ifdef KVG_PROFILE
__device__ unsigned long long g_prof[48];
__device__ __forceinline__ void prof_mark(Lead& L, int next_slot) {
  const long long t = clock64();
  L.prof[L.prof_ph] += static_cast<u64>(t - L.prof_t);
  L.prof_t = t;
  L.prof_ph = next_slot;
}
#define PROF_MARK(L, slot) prof_mark(L, slot)
#else
#define PROF_MARK(L, slot) ((void)0)
#endif

// ------------------------------------------------------------------ helpers

// event log (tests / tracing): the on/off flag lives in the Lead (shared
// memory), the store path out of line, so the 13 call sites cost a branch
__device__ __noinline__ void log_store(const SimDev& D, Lead& L, u32 kind, u32 agent, u64 a,
                                       u64 b) {
  unsigned long long i = L.n_log++;
  if (i < D.log_cap) D.log[i] = kvg_log_record{kind, agent, L.cclock, a, b};
}
__device__ __forceinline__ void log_rec(const SimDev& D, Lead& L, u32 kind, u32 agent, u64 a,
                                        u64 b) {
  if (L.log_on) log_store(D, L, kind, agent, a, b);
}

// Trace rows go to HBM (the phase classifier reads them back); a batch
// delivering to the host streams them to its slice of the mapped pinned host
// block in warp-wide flushes (flush_rows: after pipelined tick rounds and,
// through OP_FLUSH, whenever kFlushRows are pending at an event), so the PCIe
// writes spread over the run instead of queueing behind its end.
// (KVG_ROW_WT=1: write every row through from the producing thread.)
#ifndef KVG_FLUSH_ROWS
#define KVG_FLUSH_ROWS 128
#endif
constexpr u64 kFlushRows = KVG_FLUSH_ROWS;
#ifndef KVG_ROW_WT  // measured: single-thread 8 B stores to host memory, 2x slower
#define KVG_ROW_WT 0
#endif
__device__ __forceinline__ void put_row(const SimDev& D, u64 i, const kvg_trace_row& row) {
  D.trace[i] = row;
  if (KVG_ROW_WT && D.trace_out && !D.pack_mode) D.trace_out[i] = row;
}

// lifecycle_edge (workload.cpp:110-128)
__device__ __forceinline__ bool legal_edge(uint8_t from, uint8_t to) {
  switch (from) {
    case S_PENDING: return to == S_AWAIT;
    case S_AWAIT: return to == S_GEN || to == S_PAUSED;
    case S_GEN: return to == S_TOOL || to == S_DONE || to == S_AWAIT;
    case S_TOOL: return to == S_AWAIT;
    case S_PAUSED: return to == S_AWAIT;
    default: return false;
  }
}

// Per-agent statistics accumulate in HBM. KVG_STATS_RED=1 issues the
// accumulations as fire-and-forget reductions (same order, same IEEE adds);
// measured on C4 it is 7% SLOWER than the plain read-modify-write, so off.
#ifndef KVG_STATS_RED
#define KVG_STATS_RED 0
#endif
__device__ __forceinline__ void st_add(uint64_t& f, u64 v) {
  if (KVG_STATS_RED)
    atomicAdd(reinterpret_cast<unsigned long long*>(&f), static_cast<unsigned long long>(v));
  else
    f += v;
}
__device__ __forceinline__ void st_add(double& f, double v) {
  if (KVG_STATS_RED) atomicAdd(&f, v);
  else f += v;
}

// token <-> page conversions: a shift for the power-of-two page sizes every
// config uses, one out-of-line 64-bit divide otherwise
__device__ __noinline__ u64 pdiv_slow(u64 x, u64 ps) { return x / ps; }
__device__ __forceinline__ u64 pdiv(const Lead& L, u64 x) {
  return L.ps_shift >= 0 ? x >> L.ps_shift : pdiv_slow(x, L.ps);
}
__device__ __forceinline__ u64 pmod(const Lead& L, u64 x) {
  return L.ps_shift >= 0 ? x & (L.ps - 1) : x - pdiv_slow(x, L.ps) * L.ps;
}

__device__ __forceinline__ void fail(Lead& L, int code) {
  if (L.err == E_NONE) L.err = code;
  L.status = KVG_ERR_STATE;
}

// ready bitmap: bit a <=> agent a is active and AwaitingAdmission
__device__ KVG_READY_FN void ready_sync(const SimDev& D, Lead& L, AgentDev& a, u32 id) {
  const uint8_t want = a.in_active && a.state == S_AWAIT;
  if (want == a.ready) return;
  a.ready = want;
  const u32 w = id >> 5, bit = 1u << (id & 31);
  u32 v = L.rbits[w];
  if (want) {
    if (v == 0) L.rl1[w >> 5] |= 1u << (w & 31);
    L.rbits[w] = v | bit;
    ++L.n_ready;
  } else {
    v &= ~bit;
    L.rbits[w] = v;
    if (v == 0) L.rl1[w >> 5] &= ~(1u << (w & 31));
    --L.n_ready;
  }
}

// smallest ready agent id >= from, or NIL
__device__ KVG_READY_FN u32 ready_next(const SimDev& D, const Lead& L, u32 from) {
  if (from >= L.n) return NIL;
  const u32 w = from >> 5;
  const u32 bits = L.rbits[w] & (~0u << (from & 31));
  if (bits) return (w << 5) + __ffs(bits) - 1;
  for (u32 w1 = w + 1; w1 < L.nwords;) {
    const u32 m = L.rl1[w1 >> 5] & (~0u << (w1 & 31));
    if (m) {
      const u32 ww = ((w1 >> 5) << 5) + __ffs(m) - 1;
      return (ww << 5) + __ffs(L.rbits[ww]) - 1;
    }
    w1 = ((w1 >> 5) + 1) << 5;
  }
  return NIL;
}

// ready_next for the one-CTA-per-SM kernels (dispatch's member walk): the
// same answer, the second-level words read four at a time (C5: 64 words,
// the walk between sparse ready agents was ~18 % of the leader's samples).
// Separate from ready_next so the sweep kernel's inlined copies stay as small.
__device__ __forceinline__ u32 ready_next_wide(const SimDev& D, const Lead& L, u32 from) {
  if (from >= L.n) return NIL;
  const u32 w = from >> 5;
  const u32 bits = L.rbits[w] & (~0u << (from & 31));
  if (bits) return (w << 5) + __ffs(bits) - 1;
  const u32 w1 = w + 1;
  if (w1 >= L.nwords) return NIL;
  const u32 n1 = (L.nwords + 31) >> 5;
  const bool al = (reinterpret_cast<uintptr_t>(L.rl1) & 15) == 0;
  u32 j = w1 >> 5;
  u32 m = L.rl1[j] & (~0u << (w1 & 31));
  while (!m && j + 1 < n1) {
    ++j;
    if (al && (j & 3) == 0 && j + 4 <= n1) {
      const uint4 q = *reinterpret_cast<const uint4*>(L.rl1 + j);
      if (q.x) m = q.x;
      else if (q.y) { m = q.y; j += 1; }
      else if (q.z) { m = q.z; j += 2; }
      else if (q.w) { m = q.w; j += 3; }
      else j += 3;
    } else {
      m = L.rl1[j];
    }
  }
  if (!m) return NIL;
  const u32 ww = (j << 5) + __ffs(m) - 1;
  return (ww << 5) + __ffs(L.rbits[ww]) - 1;
}
template <bool kWide>
__device__ __forceinline__ u32 ready_next_k(const SimDev& D, const Lead& L, u32 from) {
  return kWide ? ready_next_wide(D, L, from) : ready_next(D, L, from);
}

// AgentRecord::set_state (workload.cpp:130-137)
__device__ KVG_MID_FN void set_state(const SimDev& D, Lead& L, u32 id, uint8_t s) {
  AgentDev& a = L.ag[id];
  if (!legal_edge(a.state, s)) {
    fail(L, E_ILLEGAL_TRANSITION);
    return;
  }
  a.state = s;
  ready_sync(D, L, a, id);
}

// active_ is an insertion-ordered vector in the reference (controller.hpp:122).
// Only its size and "the newest member at a step boundary" (the pause victim,
// controller.cpp:130-136) are ever needed, so membership is a flag plus an
// admission sequence number; the victim is the ready agent (active and
// AwaitingAdmission = at_boundary) with the largest sequence number.
__device__ KVG_LEADER_FN void act_push(const SimDev& D, Lead& L, u32 id) {
  AgentDev& a = L.ag[id];
  a.in_active = 1;
  a.act_seq = ++L.act_seq;
  ++L.act_size;
  ready_sync(D, L, a, id);
}

__device__ KVG_LEADER_FN bool act_erase(const SimDev& D, Lead& L, u32 id) {
  AgentDev& a = L.ag[id];
  if (!a.in_active) {
    fail(L, E_NOT_ACTIVE);
    return false;
  }
  a.in_active = 0;
  --L.act_size;
  ready_sync(D, L, a, id);
  return true;
}

// newest active agent at a step boundary, or NIL
__device__ __noinline__ u32 pause_victim(const SimDev& D, const Lead& L) {
  if (L.n_ready == 0) return NIL;
  u32 best = NIL, best_seq = 0;
  for (u32 id = ready_next(D, L, 0); id != NIL; id = ready_next(D, L, id + 1)) {
    const u32 q = L.ag[id].act_seq;
    if (best == NIL || q > best_seq) {
      best = id;
      best_seq = q;
    }
  }
  return best;
}

// FIFO rings for pending_ and paused_ (controller.hpp:123-124); an agent is
// in at most one of active/pending/paused, so capacity n suffices.
__device__ __forceinline__ u32 ring_at(u32 head, u32 k, u32 n) {
  u32 i = head + k;
  return i >= n ? i - n : i;
}
__device__ __forceinline__ void pend_push(const SimDev& D, Lead& L, u32 id) {
  D.pend[ring_at(L.pend_head, L.pend_size, L.n)] = id;
  ++L.pend_size;
}
__device__ __forceinline__ u32 pend_pop(const SimDev& D, Lead& L) {
  u32 id = D.pend[L.pend_head];
  L.pend_head = ring_at(L.pend_head, 1, L.n);
  --L.pend_size;
  return id;
}
__device__ __forceinline__ void paus_push(const SimDev& D, Lead& L, u32 id) {
  D.paus[ring_at(L.paus_head, L.paus_size, L.n)] = id;
  ++L.paus_size;
}
__device__ __forceinline__ u32 paus_pop(const SimDev& D, Lead& L) {
  u32 id = D.paus[L.paus_head];
  L.paus_head = ring_at(L.paus_head, 1, L.n);
  --L.paus_size;
  return id;
}

// Implicit pins: agent `id` now pins its path prefix [0, tokens).
__device__ KVG_PIN_FN void set_pinned(const SimDev& D, Lead& L, u32 id, u64 tokens) {
  AgentDev& a = L.ag[id];
  const u64 old_pg = a.pinned_pg, new_pg = pdiv(L, tokens);
  a.pinned_pg = static_cast<u32>(new_pg);
  if (old_pg == new_pg) return;
  const u64 S = L.S;
  L.pin_priv += (new_pg > S ? new_pg - S : 0);
  L.pin_priv -= (old_pg > S ? old_pg - S : 0);
  if (S == 0) return;
  const u64 jo = old_pg < S ? old_pg : S, jn = new_pg < S ? new_pg : S;
  if (jo == jn) return;
  if (jo > 0 && --D.pin_hist[jo] == 0) D.pin_lvl[jo >> 5] &= ~(1u << (jo & 31));
  if (jn > 0 && D.pin_hist[jn]++ == 0) D.pin_lvl[jn >> 5] |= 1u << (jn & 31);
  if (jn > L.pin_max) {
    L.pin_max = jn;
  } else if (jo == L.pin_max && D.pin_hist[jo] == 0) {
    u64 w = jo >> 5;  // highest non-empty level below jo
    u32 bits = D.pin_lvl[w] & ((1u << (jo & 31)) - 1);
    while (bits == 0 && w > 0) bits = D.pin_lvl[--w];
    L.pin_max = bits ? (w << 5) + 31 - __clz(bits) : 0;
  }
}

// ---------------------------------------------------------------- chain LRU
// Discard mode holds every agent's resident private pages as ONE chain
// [S, S + priv) whose pages all carry the agent's latest refresh stamp
// (a.lazy), and the shared prompt as the chain [0, L0) stamped lazy_sh, the
// newest stamp of all. Every refresh stamps with the next
// clock value, so ordering chains by stamp is an LRU list: a refresh moves the
// agent to the tail. evict(needed) = "the needed smallest (stamp asc, page
// index desc) unpinned resident pages" (cache_tree.cpp:270-319)
// therefore takes chain tails from the LRU head on, then the shared chain's
// tail (its stamp ties only with the newest agent's chain, whose pages are
// deeper and go first). The list holds exactly the agents with priv > 0.
// The chain heap: a min-heap (by chain stamp) of the agents whose private
// chain is evictable right now — resident (priv > 0) and unpinned. An agent
// pins its whole path from its match until its generation completes (or its
// insert fails), so it leaves the heap at its match and returns at the unpin
// with the stamp of its last refresh; pinned agents (thousands in a big
// dispatch batch) are never walked over. O(log n) per move.
__device__ __forceinline__ bool ch_has(const Lead& L, u32 id) { return L.lru[L.n + id] != NIL; }

__device__ __forceinline__ void ch_place(Lead& L, u32 i, u32 id) {
  L.lru[i] = id;
  L.lru[L.n + id] = i;
}

__device__ __noinline__ void ch_sift(Lead& L, u32 i) {
  u32* h = L.lru;
  const u32 id = h[i];
  const u64 key = L.ag[id].lazy;
  while (i > 0) {  // up
    const u32 p = (i - 1) >> 1;
    if (L.ag[h[p]].lazy <= key) break;
    ch_place(L, i, h[p]);
    i = p;
  }
  for (;;) {  // down
    u32 c = 2 * i + 1;
    if (c >= L.ch_n) break;
    if (c + 1 < L.ch_n && L.ag[h[c + 1]].lazy < L.ag[h[c]].lazy) ++c;
    if (L.ag[h[c]].lazy >= key) break;
    ch_place(L, i, h[c]);
    i = c;
  }
  ch_place(L, i, id);
}

// agent `id` became evictable (unpinned with priv > 0)
__device__ __forceinline__ void ch_insert(Lead& L, u32 id) {
  if (!L.lru || ch_has(L, id)) return;
  const u32 i = L.ch_n++;
  ch_place(L, i, id);
  ch_sift(L, i);
}

// agent `id` pins its path or lost its last private page
__device__ __forceinline__ void ch_remove(Lead& L, u32 id) {
  if (!L.lru || !ch_has(L, id)) return;
  const u32 i = L.lru[L.n + id];
  L.lru[L.n + id] = NIL;
  const u32 last = L.lru[--L.ch_n];
  if (i < L.ch_n) {
    ch_place(L, i, last);
    ch_sift(L, i);
  }
}

// Without the heap (the one-warp kernel's small simulations, whose shared
// memory holds no extra links) the next chain is found by a scan for the
// smallest stamp among agents with candidates: stamps are distinct per agent.
__device__ __forceinline__ u32 chain_min(const Lead& L, u64 S) {
  u32 best = NIL;
  u64 best_st = 0;
  for (u32 i = 0; i < L.n; ++i) {
    const AgentDev& a = L.ag[i];
    const u64 lo = a.pinned_pg > S ? a.pinned_pg : S;
    if (S + a.priv > lo && (best == NIL || a.lazy < best_st)) {
      best = i;
      best_st = a.lazy;
    }
  }
  return best;
}

// Frees `need` (> 0, <= evictable) pages in reference eviction order: each
// chain from the LRU head loses its unpinned tail (pages [max(S, pinned),
// S + priv), deepest first), then the shared chain [pin_max, L0). Victims are
// logged in that order. Chains visited count as scanned (roofline).
__device__ __noinline__ void chain_evict(const SimDev& D, Lead& L, u64 need) {
  const u64 S = L.S;
  const bool scan = L.lru == nullptr;
  u32 id = scan ? chain_min(L, S) : (L.ch_n ? L.lru[0] : NIL);
  while (need > 0 && id != NIL) {
    AgentDev& a = L.ag[id];
    const u64 lo = a.pinned_pg > S ? a.pinned_pg : S;
    const u64 hi = S + a.priv;
    ++L.evict_scanned;
    if (hi > lo) {
      const u64 t = hi - lo < need ? hi - lo : need;
      if (L.log_on) {
        const u64 owner = (static_cast<u64>(id) + 1) << 32;
        for (u64 p = hi; p > hi - t;) {
          --p;
          log_store(D, L, KVG_LOG_VICTIM, L.m_id, owner | p, a.lazy);
        }
      }
      a.priv -= static_cast<u32>(t);
      need -= t;
    } else if (!scan) {
      fail(L, E_EVICT_MISMATCH);  // a heap member must be evictable
      return;
    }
    if (!scan && a.priv == 0) ch_remove(L, id);
    if (need == 0) break;
    id = scan ? chain_min(L, S) : (L.ch_n ? L.lru[0] : NIL);
  }
  if (need > 0 && L.L0 > L.pin_max) {
    const u64 t = L.L0 - L.pin_max < need ? L.L0 - L.pin_max : need;
    if (L.log_on)
      for (u64 p = L.L0; p > L.L0 - t;) {
        --p;
        log_store(D, L, KVG_LOG_VICTIM, L.m_id, p, L.lazy_sh);
      }
    L.L0 -= t;
    need -= t;
  }
  if (need > 0) fail(L, E_EVICT_MISMATCH);
}

__device__ __forceinline__ bool heap_less(const HeapEnt& x, const HeapEnt& y) {
  return x.t < y.t || (x.t == y.t && x.k < y.k);
}

__device__ KVG_MID_FN void heap_push(Lead& L, const HeapEnt e);

// Engine::schedule for agent events (engine.cpp:143-145)
__device__ KVG_MID_FN void sched_agent(const SimDev& D, Lead& L, u32 id, double t,
                                            uint8_t kind) {
  AgentDev& a = L.ag[id];
  if (a.ev_kind != EV_NONE) {
    fail(L, E_EVENT_BUSY);
    return;
  }
  a.ev_kind = kind;
  heap_push(L, HeapEnt{t, (L.ord++ << kKeyShift) | id});
}

__device__ KVG_MID_FN void heap_push(Lead& L, const HeapEnt e) {
  HeapEnt* h = L.heap;
  u32 i = L.hsize++;
  while (i > 0) {
    const u32 p = (i - 1) >> 1;
    const HeapEnt pe = h[p];
    if (!heap_less(e, pe)) break;
    h[i] = pe;
    i = p;
  }
  h[i] = e;
}

__device__ KVG_LEADER_FN void heap_pop(const SimDev& D, Lead& L) {
  HeapEnt* h = L.heap;
  const u32 n = --L.hsize;
  if (n == 0) return;
  const HeapEnt last = h[n];
  u32 i = 0;
  for (;;) {
    const u32 l = 2 * i + 1;
    if (l >= n) break;
    u32 c = l;
    HeapEnt ce = h[l];
    if (l + 1 < n) {
      const HeapEnt re = h[l + 1];
      if (heap_less(re, ce)) {
        c = l + 1;
        ce = re;
      }
    }
    if (!heap_less(ce, last)) break;
    h[i] = ce;
    i = c;
  }
  h[i] = last;
}

// Engine::schedule_admission (engine.cpp:149-154)
__device__ __forceinline__ void sched_admission(Lead& L) {
  if (L.adm_on && L.adm_t == L.clock) return;
  if (L.adm_on) {
    fail(L, E_TWO_ADMISSIONS);
    return;
  }
  L.adm_on = 1;
  L.adm_t = L.clock;
  L.adm_o = L.ord++;
}

}  // namespace kvg

#include "tree.cuh"

namespace kvg {

// cost_model.cpp:28-41 (compiled with -fmad=false: no contraction)
__device__ __forceinline__ double prefill_t(const kvg_cost_params& c, u64 n, u64 ctx) {
  double x = static_cast<double>(n), y = static_cast<double>(ctx);
  return c.prefill_linear * x + c.prefill_quadratic * x * y;
}
__device__ __forceinline__ double decode_t(const kvg_cost_params& c, u64 n, u64 ctx) {
  double x = static_cast<double>(n), y = static_cast<double>(ctx);
  return c.decode_base * x + c.decode_context * (x * y + x * (x - 1.0) / 2.0);
}

// Controller::admission_limit / display_window (controller.cpp:93-117)
__device__ __forceinline__ u64 adm_limit(const Lead& L) {
  switch (L.kind) {
    case KVG_POLICY_UNCONTROLLED: return ~0ull;
    case KVG_POLICY_AIMD: return static_cast<u64>(floor(L.window));
    default: return L.cap;
  }
}
__device__ __forceinline__ double display_window(const Lead& L) {
  switch (L.kind) {
    case KVG_POLICY_UNCONTROLLED: return static_cast<double>(L.n);
    case KVG_POLICY_AIMD: return L.window;
    default: return static_cast<double>(L.cap);
  }
}

// Controller::update_window (controller.cpp:67-91)
__device__ __forceinline__ void update_window(Lead& L, double usage, double hit) {
  ++L.ticks;
  if (L.kind != KVG_POLICY_AIMD) return;
  const kvg_controller_config& c = L.cfg;
  double u = usage, h = hit;
  if (c.signal_smoothing > 0) {
    if (L.have_s) {
      u = c.signal_smoothing * L.su + (1 - c.signal_smoothing) * usage;
      h = c.signal_smoothing * L.sh + (1 - c.signal_smoothing) * hit;
    }
    L.su = u;
    L.sh = h;
    L.have_s = 1;
  }
  double w = L.window;
  if (u < c.u_low)
    w = w + c.alpha;
  else if (u > c.u_high && h < c.h_thresh)
    w = w * c.beta;
  L.window = w < c.w_min ? c.w_min : (c.w_max < w ? c.w_max : w);
}

// -------------------------------------------------------------- op posting

__device__ __forceinline__ void post_range(Op& op, u32 agent, u64 p0, u64 p1, u32 flags,
                                           int delta, u64 stamp) {
  op.kind = OP_RANGE;
  op.agent = agent;
  op.p0 = p0;
  op.p1 = p1;
  op.flags = flags;
  op.pin_delta = delta;
  op.stamp = stamp;
  op.first_miss = ~0ull;
  op.created = op.freed = op.pin_up = op.pin_down = op.resident = 0;
  op.err = E_NONE;
}

__device__ __forceinline__ u64 range_chunks(u64 p0, u64 p1) {
  return p1 > p0 ? (p1 - p0) / kChunk + 2 : 0;
}

// ------------------------------------------------------------ the handlers

// Engine::on_control_tick (engine.cpp:245-266) — the kernel-3 signal step.
__device__ __noinline__ void on_tick(const SimDev& D, Lead& L) {
  const double usage = static_cast<double>(L.used) / L.capacity_d;
  const double m = L.hit_m, r = L.hit_r;
  const double hit = r > 0 ? m / r : 1.0;
  update_window(L, usage, hit);
  const unsigned long long i = L.n_trace++;
  if (i < D.trace_cap) {
    kvg_trace_row row;
    row.time = L.clock;
    row.usage = usage;
    row.hit_rate = hit;
    row.window = display_window(L);
    row.active = L.act_size;
    row.pending = static_cast<u64>(L.pend_size) + L.paus_size;
    row.decoded_cum = L.decoded_cum;
    row.recompute_cum = L.rec_cum;
    row.transfers = L.offload ? x_in_flight(D, L, L.clock) : 0;
    row.hit_matched = m;
    row.hit_requested = r;
    put_row(D, i, row);
  }
  L.hit_m *= L.decay;  // CacheTree::decay_hit_window (cache_tree.cpp:453-456)
  L.hit_r *= L.decay;
  L.tick_on = 1;
  L.tick_t = L.clock + L.interval;
  L.tick_o = L.ord++;
  sched_admission(L);
}

__device__ __forceinline__ void pause_one(const SimDev& D, Lead& L, u32 id) {
  act_erase(D, L, id);
  paus_push(D, L, id);
  set_state(D, L, id, S_PAUSED);
  st_add(D.stats[id].pause_events, 1);
}

// Pauses the K ready agents with the largest admission sequence numbers, in
// descending order (= K successive pause_victim calls). D.batch is free
// scratch here (dispatch_batch has not started).
__device__ __noinline__ void pause_top_k(const SimDev& D, Lead& L, u32 K) {
  u64* h = reinterpret_cast<u64*>(D.batch);  // key = act_seq << 32 | id (seqs are unique)
  u32 m = 0;
  for (u32 id = ready_next(D, L, 0); id != NIL; id = ready_next(D, L, id + 1)) {
    const u64 key = (static_cast<u64>(L.ag[id].act_seq) << 32) | id;
    if (m < K) {  // min-heap of the K largest keys
      u32 i = m++;
      while (i > 0) {
        const u32 p = (i - 1) >> 1;
        if (h[p] <= key) break;
        h[i] = h[p];
        i = p;
      }
      h[i] = key;
    } else if (key > h[0]) {
      u32 i = 0;
      for (;;) {
        u32 c = 2 * i + 1;
        if (c >= K) break;
        if (c + 1 < K && h[c + 1] < h[c]) ++c;
        if (h[c] >= key) break;
        h[i] = h[c];
        i = c;
      }
      h[i] = key;
    }
  }
  // in-place heapsort: each pop moves the current minimum to the end of the
  // shrinking heap, leaving h[0..m) in descending key order
  for (u32 n = m; n > 0; --n) {
    const u64 top = h[0], last = h[n - 1];
    u32 i = 0;
    for (;;) {
      u32 c = 2 * i + 1;
      if (c >= n - 1) break;
      if (c + 1 < n - 1 && h[c + 1] < h[c]) ++c;
      if (h[c] >= last) break;
      h[i] = h[c];
      i = c;
    }
    if (n > 1) h[i] = last;
    h[n - 1] = top;
  }
  for (u32 k = 0; k < m; ++k) pause_one(D, L, static_cast<u32>(h[k] & 0xffffffffu));
}

// Controller::admission_pass (controller.cpp:124-160) with the commands
// applied as Engine::on_admission_check does (engine.cpp:268-291). Commands
// can be applied immediately: pausing only removes agents from active_ and
// happens before any admit, which never reads agent state.
__device__ __noinline__ void admission_pass(const SimDev& D, Lead& L) {
  const u64 limit = adm_limit(L);
  if (L.gated && L.act_size > limit) {
    // The reference pauses the newest at-boundary active agent until the
    // limit holds or none is left: the victims are the ready agents in
    // descending admission order, at most K of them. Few: scan per victim.
    // Many (an AIMD cut in a big simulation): one gather + top-K selection
    // instead of K scans (O(n_ready log K), not O(K n_ready)).
    const u64 over = L.act_size - limit;
    const u64 K = over < L.n_ready ? over : L.n_ready;
#ifndef KVG_TOPK_MIN
#define KVG_TOPK_MIN 3
#endif
    if (K < KVG_TOPK_MIN) {
      while (L.act_size > limit) {
        const u32 id = pause_victim(D, L);
        if (id == NIL) break;
        pause_one(D, L, id);
      }
    } else {
      pause_top_k(D, L, static_cast<u32>(K));
    }
  }
  while (L.act_size < limit) {
    if (L.gated && L.paus_size > 0) {
      u32 id = paus_pop(D, L);
      act_push(D, L, id);
      set_state(D, L, id, S_AWAIT);  // resume
    } else if (L.pend_size > 0) {
      u32 id = pend_pop(D, L);
      act_push(D, L, id);
      if (L.ag[id].state == S_PENDING) set_state(D, L, id, S_AWAIT);  // admit
    } else {
      break;
    }
  }
}

__device__ __noinline__ void finalize(const SimDev& D, Lead& L) {
  kvg_sim_result* r = D.result;
  r->status = L.status;
  // r->n_phases / r->phases: written by coop_phases (classify_phases,
  // metrics.cpp:41-81), which every run passes through (PH_DONE) before this
  r->ledger = L.ledger;
  r->makespan = L.makespan < L.pcie_busy ? L.pcie_busy : L.makespan;  // engine.cpp:400
  r->device_busy = L.device_busy;
  r->link_busy = L.link_busy;
  r->decoded_tokens = L.decoded_cum;
  r->recompute_tokens = L.rec_cum;
  u64 rec_ev = 0, stalls = 0;
  double wait = 0.0;
  for (u32 i = 0; i < L.n; ++i) {  // engine.cpp:407-412, agent order
    // L2 reads (with KVG_STATS_RED the counters were accumulated at L2)
    const kvg_agent_stats& st = D.stats[i];
    rec_ev += __ldcg(reinterpret_cast<const unsigned long long*>(&st.recompute_events));
    stalls += __ldcg(reinterpret_cast<const unsigned long long*>(&st.stall_events));
    wait += __ldcg(&st.wait_time);
  }
  r->recompute_events = rec_ev;
  r->stall_events = stalls;
  r->offloaded_tokens = L.offloaded;
  r->reloaded_tokens = L.reloaded;
  r->discarded_tokens = L.discarded;
  r->total_wait_time = wait;
  r->ticks = L.n_trace;
  r->workload_hash = D.workload_hash;
  r->agent_steps = L.agent_steps;
  r->lookups = L.lookups;
  r->events = L.events;
  r->evict_calls = L.evict_calls;
  r->evicted_pages = L.evicted;
  r->cache_clock = L.cclock;
  r->pool_used = L.used;
  r->hit_matched = L.hit_m;
  r->hit_requested = L.hit_r;
  r->hit_pages = L.hit_pages;
  r->created_pages = L.created_pages;
  r->refreshed_pages = L.refreshed_pages;
  r->evict_scanned = L.evict_scanned;
  r->agent_events = L.agent_events;
  r->device_cycles = static_cast<u64>(clock64() - L.t_start);
  r->abort_time = L.status == KVG_ERR_HORIZON ? L.abort_t : 0.0;
#ifdef KVG_GTIMER  // dev probe only: start / end in globaltimer ns, SM id
  {
    u64 g_end;
    unsigned smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    r->evict_scanned = r->device_cycles;
    r->device_cycles = g_end;
    r->abort_time = static_cast<double>(L.g_start);
    r->evicted_pages = smid;
  }
#endif
  r->unfinished = L.n - L.finished;
  D.counts[0] = L.n_trace;
  D.counts[1] = L.n_log;
  D.counts[2] = static_cast<u64>(L.err);
}

__device__ __noinline__ void lead_init(const SimDev& D, Lead& L, Op& op) {
  L.status = KVG_OK;
  L.err = E_NONE;
  L.rebuilt = 0;
  L.t_start = clock64();
#ifdef KVG_GTIMER  // dev probe: wall-clock placement of each simulation in the launch
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(L.g_start));
#endif
  L.clock = L.gpu_busy = L.makespan = L.device_busy = 0.0;
  L.ord = 0;
  L.hsize = 0;
  L.finished = 0;
  L.n_ready = 0;
  L.used = L.cclock = L.discarded = L.lookups = 0;
  L.n_flushed = 0;
  L.stream_on = D.trace_out != nullptr && !D.pack_mode && !KVG_ROW_WT;
  L.log_on = D.log != nullptr;
  L.agent_steps = L.events = L.evict_calls = L.evicted = 0;
  L.pin_max = L.pin_priv = 0;
  L.L0 = L.lazy_sh = 0;
  L.verify = D.verify != 0;
  L.group_min = D.group_min;
  L.ch_n = 0;
  L.gr_head = L.gr_n = 0;
  L.stall_streak = 0;
  L.storm_on = D.storm_on;
  L.hit_pages = L.created_pages = L.refreshed_pages = L.evict_scanned = L.agent_events = 0;
  L.hit_m = L.hit_r = 0.0;
  L.n = D.n_agents;
  L.nwords = (D.n_agents + 31) / 32;
  L.steps = D.n_steps;
  L.kind = D.policy.kind;
  L.cap = D.policy.cap;
  L.cfg = D.policy.aimd;
  L.gated = L.kind == KVG_POLICY_AGENT_CAP || L.kind == KVG_POLICY_AIMD;
  L.window = 1.0;  // Controller::window_ default (controller.hpp:119)
  if (L.kind == KVG_POLICY_AIMD) {  // Controller ctor (controller.cpp:55-65)
    if (L.cfg.w_max == 0) L.cfg.w_max = fmax(L.cfg.w_min, static_cast<double>(L.n));
    if (L.cfg.initial_window == 0) L.cfg.initial_window = L.cfg.w_min;
    L.window = L.cfg.initial_window;
  }
  L.su = L.sh = 0.0;
  L.have_s = 0;
  L.ticks = 0;
  L.act_seq = 0;
  L.act_size = 0;
  L.pend_head = 0;
  L.pend_size = L.n;  // every agent starts pending (engine.cpp:89-93)
  L.paus_head = 0;
  L.paus_size = 0;
  L.decoded_cum = L.rec_cum = 0;
  L.ledger = kvg_ledger{0, 0, 0, 0, 0};
  L.n_trace = L.n_log = 0;
  L.interval = D.policy.aimd.control_interval;
  L.decay = D.engine.hit_window_decay;
  L.horizon = D.engine.horizon;
  L.capacity = D.engine.capacity;
  L.capacity_d = static_cast<double>(D.engine.capacity);
  L.ps = D.engine.page_size;
  L.ps_shift = (L.ps & (L.ps - 1)) == 0 ? 63 - __clzll(static_cast<long long>(L.ps)) : -1;
  L.shared_len = D.shared_len;
  L.S = D.shared_pages;
  // Engine::run: admission check at t=0 (ordinal 0), first tick (ordinal 1)
  L.adm_on = 1;
  L.adm_t = 0.0;
  L.adm_o = L.ord++;
  L.tick_on = 1;
  L.tick_t = L.interval;
  L.tick_o = L.ord++;
  // table context
  op.table = D.table;
  op.alt = D.alt;
  op.occ = D.occ;
  op.alt_occ = D.alt_occ;
  op.summ = D.summ;
  op.alt_summ = D.alt_summ;
  op.mask = D.bucket_mask;
  op.occ_n = 0;
  op.alt_n = 0;
  op.shared_pages = D.shared_pages;
  op.log = D.log;
  op.log_cap = D.log_cap;
  op.log_n = &L.n_log;
  op.vic = nullptr;
  op.vic_cap = 0;
  op.vic_n = nullptr;
  op.log_victims = D.log != nullptr;
  op.implicit_pins = 1;
  op.pin_max = 0;
  op.agents = L.ag;
  op.tnodes = D.tnodes;
  op.fr = D.fr;
  L.offload = D.engine.eviction == KVG_EVICT_OFFLOAD;
  L.pcie_busy = L.link_busy = 0.0;
  L.offloaded = L.reloaded = 0;
  if (L.offload) tree_init(D, L);
  L.chain = !L.offload && !L.verify;
  L.phase = PH_EVENT;
}

// Fast path for the dominant event stream of a controlled run: control ticks
// and admission checks that change nothing (C2 has
// 760K of them against 32K agent events). Processes them with the hot state in
// registers until the next event that needs the general path: an agent event,
// an admission check that would admit / resume / pause / dispatch, the horizon,
// or the end of the run. Same arithmetic, same order as on_tick /
// on_admission_check (engine.cpp:245-291, controller.cpp:67-160).
// kHoist: loop invariants of the trace row held in registers (the row stores
// go through a generic pointer, after which the compiler reloads Lead
// fields). Measured: C3 264 -> 254 ms in the one-CTA-per-SM kernels, C4 +8 %
// in the 72-register sweep kernel (spills), so only the former hoist.
template <bool kHoist>
__device__ __forceinline__ void fast_housekeeping(const SimDev& D, Lead& L) {
  if (L.finished == L.n || L.status != KVG_OK) return;
  const double t_agent = L.hsize > 0 ? L.heap[0].t : __longlong_as_double(0x7ff0000000000000ll);
  const double horizon = L.horizon;
  {  // nothing to do unless a housekeeping event precedes the next agent
     // event: leave before loading the whole state (most calls)
    const bool tk = L.tick_on && (!L.adm_on || L.tick_t <= L.adm_t);
    if (!tk && !L.adm_on) return;
    const double t0 = tk ? L.tick_t : L.adm_t;
    if (!(t0 < t_agent) || t0 > horizon) return;
  }
  // state that no housekeeping event can change
  const bool nready0 = L.n_ready == 0;
  const u64 act = L.act_size;
  const bool admit_src = L.pend_size > 0 || (L.gated && L.paus_size > 0);
  const u32 kind = L.kind;
  const double usage = static_cast<double>(L.used) / L.capacity_d;
  const double decay = L.decay, interval = L.interval;
  // (the row's pending / decoded / recompute counts are read from Lead at
  // each row: held in registers across the loop they spill at 72)
  const u64 trace_cap = D.trace_cap;
  const kvg_controller_config c = L.cfg;
  const bool offload_h = kHoist ? L.offload : false;
  const double win_fixed_h = !kHoist ? 0.0
                             : kind == KVG_POLICY_UNCONTROLLED ? static_cast<double>(L.n)
                                                               : static_cast<double>(L.cap);
  const u64 cap_h = kHoist ? static_cast<u64>(L.cap) : 0;
  // evolving state
  double clock = L.clock, tick_t = L.tick_t, adm_t = L.adm_t;
  double hit_m = L.hit_m, hit_r = L.hit_r, window = L.window;
  int tick_on = L.tick_on, adm_on = L.adm_on;  // (smoothing state: read / written in place)
  // the scheduled slots' ordinals are stored in place; event and tick counts
  // are kept as 32-bit deltas (registers are what the sweep kernel lacks)
  u64 ord = L.ord;
  u32 d_events = 0, d_ticks = 0;
  unsigned long long n_trace = L.n_trace;
  for (;;) {
    // next housekeeping event, if it precedes every agent event (rank 0)
    bool tick;
    if (tick_on && (!adm_on || tick_t <= adm_t)) {
      if (!(tick_t < t_agent)) break;
      tick = true;
    } else if (adm_on) {
      if (!(adm_t < t_agent)) break;
      tick = false;
    } else {
      break;
    }
    const double bt = tick ? tick_t : adm_t;
    if (bt > horizon) break;
    if (tick) {
      clock = bt;
      tick_on = 0;
      const double m = hit_m, r = hit_r;
      const double hit = r > 0 ? m / r : 1.0;
      ++d_ticks;  // Controller::update_window
      if (kind == KVG_POLICY_AIMD) {
        double u = usage, h = hit;
        if (c.signal_smoothing > 0) {
          if (L.have_s) {
            u = c.signal_smoothing * L.su + (1 - c.signal_smoothing) * usage;
            h = c.signal_smoothing * L.sh + (1 - c.signal_smoothing) * hit;
          }
          L.su = u;
          L.sh = h;
          L.have_s = 1;
        }
        double w = window;
        if (u < c.u_low)
          w = w + c.alpha;
        else if (u > c.u_high && h < c.h_thresh)
          w = w * c.beta;
        window = w < c.w_min ? c.w_min : (c.w_max < w ? c.w_max : w);
      }
      const unsigned long long i = n_trace++;
      if (i < trace_cap) {
        kvg_trace_row row;
        row.time = clock;
        row.usage = usage;
        row.hit_rate = hit;
        if (kHoist)
          row.window = kind == KVG_POLICY_AIMD ? window : win_fixed_h;
        else
          row.window = kind == KVG_POLICY_AIMD ? window
                       : kind == KVG_POLICY_UNCONTROLLED ? static_cast<double>(L.n)
                                                         : static_cast<double>(L.cap);
        row.active = act;
        row.pending = static_cast<u64>(L.pend_size) + L.paus_size;
        row.decoded_cum = L.decoded_cum;
        row.recompute_cum = L.rec_cum;
        row.transfers = (kHoist ? offload_h : L.offload) ? x_in_flight(D, L, clock) : 0;
        row.hit_matched = m;
        row.hit_requested = r;
        put_row(D, i, row);
      }
      hit_m = m * decay;
      hit_r = r * decay;
      tick_on = 1;
      tick_t = clock + interval;
      L.tick_o = ord++;
      if (!(adm_on && adm_t == clock)) {  // schedule_admission
        if (adm_on) break;                // cannot happen; general path reports it
        adm_on = 1;
        adm_t = clock;
        L.adm_o = ord++;
        ++d_events;
        // the admission check just scheduled is the very next event (agent
        // events are later than this tick and, unless clock + interval
        // rounds to clock, so is the next tick): a no-op check is taken here
        // without another loop turn
        const u64 limit = kind == KVG_POLICY_UNCONTROLLED ? ~0ull
                          : kind == KVG_POLICY_AIMD ? static_cast<u64>(floor(window))
                                                    : kHoist ? cap_h : static_cast<u64>(L.cap);
        if (tick_t > clock && nready0 && !(act < limit && admit_src)) {
          adm_on = 0;
          ++d_events;
        }
        continue;
      }
      ++d_events;
    } else {
      const u64 limit = kind == KVG_POLICY_UNCONTROLLED ? ~0ull
                        : kind == KVG_POLICY_AIMD ? static_cast<u64>(floor(window))
                                                  : kHoist ? cap_h : static_cast<u64>(L.cap);
      // nothing ready => no pause victim and nothing to dispatch
      const bool noop = nready0 && !(act < limit && admit_src);
      if (!noop) break;  // the general path runs the real admission pass
      clock = bt;
      adm_on = 0;
      ++d_events;
    }
  }
  L.clock = clock;
  L.tick_t = tick_t;
  L.adm_t = adm_t;
  L.hit_m = hit_m;
  L.hit_r = hit_r;
  L.window = window;
  L.tick_on = tick_on;
  L.adm_on = adm_on;
  L.ord = ord;
  L.events += d_events;
  L.ticks += d_ticks;
  L.n_trace = n_trace;
}

// Whether the warp-pipelined tick op applies: the next housekeeping event is
// a control tick well before the next agent event, with no admission check
// pending in front of it (the steady state between agent events). Smoothed
// signals (an EMA chain per tick) and offload mode (a link-queue purge per
// tick) stay on the scalar path.
template <bool kOff>
__device__ __forceinline__ bool ticks_apply(const Lead& L) {
  // (checked every event-loop turn: the usual exit, a pending admission
  // check, first; the offload flag only where the tier is compiled in)
  if (L.adm_on || !L.tick_on || L.status != KVG_OK || L.finished == L.n) return false;
  if (kOff && L.offload) return false;
  if (L.kind == KVG_POLICY_AIMD && L.cfg.signal_smoothing > 0) return false;
  const double t_agent = L.hsize > 0 ? L.heap[0].t : __longlong_as_double(0x7ff0000000000000ll);
  return L.tick_t < t_agent && !(L.tick_t > L.horizon) &&
         L.tick_t + KVG_TICK_AHEAD * L.interval < t_agent;  // >= 4 ticks: cheaper than the scalar loop
}

// OP_TICKS (warp 0): the same event sequence as fast_housekeeping — control
// tick k at t_k, then the admission check it schedules at t_k, repeated —
// 32 ticks per round. Lane k computes tick k's own chain values exactly as
// the scalar loop would (t_{k+1} = t_k + interval, hit_m / hit_r decayed by
// k repeated multiplications, hit = m / r): independent per lane, so the
// divisions and the trace-row stores run in parallel. The window recurrence
// (controller.cpp:67-91) stays sequential but is a few flops per tick with
// every hit rate already in a register. Stops exactly where the scalar loop
// stops: before a tick that is not earlier than the next agent event or is
// past the horizon, or after a tick whose admission check would act
// (engine.cpp:245-291, controller.cpp:124-160).
__device__ __noinline__ void coop_ticks(const SimDev& D, Lead& L, int lane) {
  const double t_agent = L.hsize > 0 ? L.heap[0].t : __longlong_as_double(0x7ff0000000000000ll);
  const double horizon = L.horizon, interval = L.interval, decay = L.decay;
  const double usage = static_cast<double>(L.used) / L.capacity_d;
  const bool nready0 = L.n_ready == 0;
  const u64 act = L.act_size;
  const bool admit_src = L.pend_size > 0 || (L.gated && L.paus_size > 0);
  const u32 kind = L.kind;
  const kvg_controller_config c = L.cfg;
  const u64 pending = static_cast<u64>(L.pend_size) + L.paus_size;
  const u64 dec = L.decoded_cum, rec = L.rec_cum;
  const double fixed_window = kind == KVG_POLICY_UNCONTROLLED ? static_cast<double>(L.n)
                                                              : static_cast<double>(L.cap);
  double t0 = L.tick_t, m0 = L.hit_m, r0 = L.hit_r, w = L.window;
  u64 ord = L.ord, events = L.events, ticks = L.ticks;
  unsigned long long n_trace = L.n_trace;
  bool done = false, adm_pending = false;
  double clock = L.clock;
  while (!done) {
    // ticks that can precede the next agent event this round (an upper
    // bound: validity is still checked per lane), so short runs do not pay
    // for 32 chain steps
    const double span = (t_agent - t0) / interval;
    const int kmax = span >= 30.0 ? 32 : static_cast<int>(span) + 2;
    // lane k: tick k's time and hit window (sequential chains, exact order)
    double t = t0, m = m0, r = r0;
    const int steps = lane < kmax ? lane : kmax;
    for (int i = 0; i < steps; ++i) {
      t = t + interval;
      m = m * decay;
      r = r * decay;
    }
    const double hit = r > 0 ? m / r : 1.0;
    const bool in_time = lane < kmax && t < t_agent && !(t > horizon);
    // window recurrence, every lane in lockstep; lane k keeps w_k
    double wk = w;
    for (int k = 0; k < kmax; ++k) {
      const double h = __shfl_sync(FULL, hit, k);
      if (kind == KVG_POLICY_AIMD) {
        double x = w;
        if (usage < c.u_low) x = x + c.alpha;
        else if (usage > c.u_high && h < c.h_thresh) x = x * c.beta;
        w = x < c.w_min ? c.w_min : (c.w_max < x ? c.w_max : x);
      }
      if (lane == k) wk = w;
    }
    const u64 limit = kind == KVG_POLICY_UNCONTROLLED ? ~0ull
                      : kind == KVG_POLICY_AIMD ? static_cast<u64>(floor(wk))
                                                : static_cast<u64>(L.cap);
    const bool noop = nready0 && !(act < limit && admit_src);
    // processed ticks: [0, K); tick K-1's admission stays pending if it acts
    const unsigned late = __ballot_sync(FULL, !in_time);
    const unsigned acts = __ballot_sync(FULL, !noop);
    const int k_time = late ? __ffs(late) - 1 : 32;  // first tick not taken
    const int k_act = acts ? __ffs(acts) - 1 : 32;   // first tick whose check acts
    int K = k_time;
    if (k_act < K) {
      K = k_act + 1;
      adm_pending = true;
      done = true;
    }
    if (k_time < 32) done = true;
    if (K == 0) break;
    if (lane < K && n_trace + lane < D.trace_cap) {
      kvg_trace_row row;
      row.time = t;
      row.usage = usage;
      row.hit_rate = hit;
      row.window = kind == KVG_POLICY_AIMD ? wk : fixed_window;
      row.active = act;
      row.pending = pending;
      row.decoded_cum = dec;
      row.recompute_cum = rec;
      row.transfers = 0;
      row.hit_matched = m;
      row.hit_requested = r;
      put_row(D, n_trace + lane, row);
    }
    // carry the state of the last processed tick
    const int last = K - 1;
    clock = __shfl_sync(FULL, t, last);
    const double m_last = __shfl_sync(FULL, m, last), r_last = __shfl_sync(FULL, r, last);
    m0 = m_last * decay;
    r0 = r_last * decay;
    t0 = clock + interval;
    w = __shfl_sync(FULL, wk, last);
    n_trace += K;
    ticks += K;
    ord += 2 * K;
    events += 2 * K - (adm_pending ? 1 : 0);
  }
  if (lane == 0) {
    L.clock = clock;
    L.tick_t = t0;
    L.hit_m = m0;
    L.hit_r = r0;
    L.window = w;
    L.tick_o = ord - 2;
    if (adm_pending) {
      L.adm_on = 1;
      L.adm_t = clock;
      L.adm_o = ord - 1;
    }
    L.ord = ord;
    L.events = events;
    L.ticks = ticks;
    L.n_trace = n_trace;
  }
}

// classify_phases (metrics.cpp:41-81, called by finish_result,
// engine.cpp:413) over this simulation's own trace rows, on warp 0: rows are
// read 32 at a time (one per lane) and reduced to a hot-tick ballot; lane 0
// walks the bits. Warmup until the first saturated cache-cold tick, middle
// until `hysteresis` consecutive ticks leave that state, then cooldown.
__device__ __noinline__ void coop_phases(const SimDev& D, Lead& L, int lane) {
  const kvg_phase_params& pp = D.engine.phases;
  const double mk = L.makespan < L.pcie_busy ? L.pcie_busy : L.makespan;
  const u64 n = L.n_trace < D.trace_cap ? L.n_trace : D.trace_cap;
  u32 np = 0;
  kvg_phase_label ph[3];
  if (mk > 0) {
    u64 enter = n, leave = n;  // first hot row; row that ends the middle
    long long bad = 0;         // non-hot rows since the last hot one (after enter)
    const long long H = pp.hysteresis;
    // each lane reads two fields of one row; the next 32 rows are loaded
    // while lane 0 walks the current ballot run by run (ffs), not bit by bit
    double u_nx = 0.0, h_nx = 0.0;
    if (static_cast<u64>(lane) < n) {
      u_nx = D.trace[lane].usage;
      h_nx = D.trace[lane].hit_rate;
    }
    for (u64 base = 0; base < n && leave == n; base += 32) {
      const u64 i = base + lane;
      const bool hot = i < n && u_nx >= pp.sat_threshold && h_nx < pp.hit_threshold;
      if (i + 32 < n) {
        u_nx = D.trace[i + 32].usage;
        h_nx = D.trace[i + 32].hit_rate;
      }
      const unsigned m = __ballot_sync(FULL, hot);
      if (lane == 0) {
        const u32 cnt = n - base < 32 ? static_cast<u32>(n - base) : 32u;
        u32 p = 0;
        if (enter == n) {  // warmup until the first hot row
          if (m) {
            const u32 k0 = __ffs(m) - 1;
            enter = base + k0;
            p = k0 + 1;
          } else {
            p = cnt;
          }
        }
        while (p < cnt) {
          const u32 rest = m >> p;
          if (rest & 1u) {  // a run of hot rows resets the count
            const u32 inv = ~rest;
            p += inv ? static_cast<u32>(__ffs(inv) - 1) : 32u - p;
            bad = 0;
            continue;
          }
          // a run of non-hot rows [p, p + z): the middle ends at the row that
          // brings the count to H (the row-by-row rule ++bad >= H)
          u32 z = rest ? static_cast<u32>(__ffs(rest) - 1) : 32u - p;
          if (z > cnt - p) z = cnt - p;
          const long long t = H - bad - 1 > 0 ? H - bad - 1 : 0;
          if (t < static_cast<long long>(z)) {
            leave = static_cast<u64>(static_cast<long long>(base + p) + t + 1 - H);
            break;
          }
          bad += z;
          p += z;
        }
      }
      leave = __shfl_sync(FULL, leave, 0);
    }
    if (lane == 0) {
      if (enter == n) {
        ph[np++] = kvg_phase_label{KVG_PHASE_WARMUP, 0, 0.0, mk};
      } else {
        const double ms = D.trace[enter].time;
        const double me = leave < n ? D.trace[leave].time : mk;
        if (ms > 0) ph[np++] = kvg_phase_label{KVG_PHASE_WARMUP, 0, 0.0, ms};
        ph[np++] = kvg_phase_label{KVG_PHASE_MIDDLE, 0, ms, me};
        if (me < mk) ph[np++] = kvg_phase_label{KVG_PHASE_COOLDOWN, 0, me, mk};
      }
    }
  }
  if (lane == 0) {  // straight into the result (not held in Lead: shared memory per CTA)
    kvg_sim_result* r = D.result;
    r->n_phases = np;
    for (u32 k = 0; k < 3; ++k) r->phases[k] = k < np ? ph[k] : kvg_phase_label{0, 0, 0.0, 0.0};
  }
}

// The successful tail of dispatch_member (engine.cpp:378-395): recompute
// attribution, the member's cost-model times, InFlight, wait time, state.
__device__ __forceinline__ void member_success(const SimDev& D, Lead& L, u32 id, u64 ctx0,
                                            u64 matched) {
  AgentDev& a = L.ag[id];
  const u64 stored = a.ctx - pmod(L, a.ctx);
  const u64 missing = ctx0 - matched;
  const u64 rec = a.high_water > matched ? a.high_water - matched : 0;
  const u64 fresh = missing - rec;
  a.high_water = stored;
  const kvg_step_plan& plan = D.plans[static_cast<size_t>(id) * L.steps + a.step];
  Member m;
  m.id = id;
  m.pad = 0;
  m.f = prefill_t(D.cost, fresh, ctx0);
  m.r = prefill_t(D.cost, rec, ctx0);
  m.d = decode_t(D.cost, plan.gen_tokens, ctx0);
  m.t = m.f + m.r + m.d;
  D.batch[L.batch_n++] = m;
  // the batch wall (max) and total (sum, member order) of engine.cpp:317-324,
  // accumulated as members commit: same operations in the same order
  L.b_wall = L.b_wall < m.t ? m.t : L.b_wall;
  L.b_total += m.t;
  a.f_gen = static_cast<u32>(plan.gen_tokens);
  a.f_rec = static_cast<u32>(rec);
  a.f_has_tool = plan.has_tool != 0;
  a.f_obs = static_cast<u32>(plan.obs_tokens);
  a.f_tool = plan.tool_latency;
  st_add(D.stats[id].wait_time, L.clock - a.ready_since);
  set_state(D, L, id, S_GEN);
  a.stalled = 0;  // (stall bookkeeping, informational)
  ++L.agent_steps;
}

// Offload-mode dispatch_member (engine.cpp:337-396) on the node-level tree.
// Returns true when it posted the cooperative frontier scan (the CTA runs
// it, then PH_O_EVICT_POP resumes); false when the phase just advanced.
__device__ __noinline__ bool offload_step(const SimDev& D, Lead& L, Op& op) {
  TNodeDev* N = D.tnodes;
  const u32 id = L.m_id;
  AgentDev& a = L.ag[id];
  auto post_frontier = [&](u64 need, int then) {
    L.o_ev_need = need;
    L.o_then = then;
    op.kind = OP_FRONTIER;
    op.fr_n = 0;
    op.t_n = L.t_alloc;
    op.tw_off = L.tw_off;
    op.tw_n = L.tw_n;
    L.phase = PH_O_EVICT_POP;
  };
  auto next_member = [&]() {
    L.m_next = ready_next(D, L, id + 1);
    L.phase = PH_O_MEMBER;
  };
  switch (L.phase) {
    case PH_O_RELOAD_CHUNK:
    case PH_O_RELOAD_EVICTED: {  // reload's chunk loop, cache_tree.cpp:337-366
      const u64 len = L.m_ctx0, n = pdiv(L, len);
      if (L.phase == PH_O_RELOAD_CHUNK) {
        if (!(L.o_pos < len && L.o_promoted < L.o_hm)) {
          L.phase = PH_O_RELOAD_END;
          return false;
        }
        const u32 c = t_find_child(D, L, L.o_node, id, pdiv(L, L.o_pos), n);
        const TWc W = tw_ctx(D, L);
        if (c == 0 || !tw_is_host(tw_get(W, c))) {
          L.phase = PH_O_RELOAD_END;
          return false;
        }
        u64 ka = t_common(D, L, c, id, pdiv(L, L.o_pos), n);
        const u32 np = tw_get(W, c).npages;
        bool full = ka == np;
        const u64 want = pdiv(L, L.o_hm - L.o_promoted);
        if (ka > want) {
          ka = want;
          full = false;
        }
        if (ka == 0) {
          L.phase = PH_O_RELOAD_END;
          return false;
        }
        if (ka < np) t_split(D, L, c, ka);
        L.o_c = c;
        L.o_ka = ka;
        L.o_full = full;
        if (L.capacity - L.used < ka) {
          post_frontier(ka - (L.capacity - L.used), PH_O_RELOAD_EVICTED);
          return true;
        }
      } else if (L.capacity - L.used < L.o_ka) {  // evicted, still no room
        L.phase = PH_O_RELOAD_END;
        return false;
      }
      const u32 c = L.o_c;
      N[c].host = 0;
      tw_host(tw_ctx(D, L), c, 0);
      tm_slots(tw_ctx(D, L), c, static_cast<u32>(L.o_ka));
      N[c].last_access = L.o_now;
      L.used += L.o_ka;
      t_gain(D, L, c);
      L.o_promoted += L.o_ka * L.ps;
      L.o_pos += L.o_ka * L.ps;
      L.o_node = c;
      L.phase = L.o_full ? PH_O_RELOAD_CHUNK : PH_O_RELOAD_END;
      return false;
    }
    case PH_O_RELOAD_END: {  // engine.cpp:347-360
      x_account(D, L, L.o_offl);
      log_rec(D, L, KVG_LOG_RELOAD, id, L.o_promoted, L.o_offl);
      if (L.o_promoted > 0) {
        const u64 m = L.o_matched;
        t_pin_move(D, L, id, m + L.o_promoted, m);
        a.pinned_pg = static_cast<u32>(pdiv(L, m + L.o_promoted));
        L.reloaded += L.o_promoted;
        const double end =
            x_enqueue(D, L, static_cast<double>(L.o_promoted) * D.cost.bytes_per_token);
        st_add(D.stats[id].wait_time, L.clock - a.ready_since);
        set_state(D, L, id, S_GEN);
        sched_agent(D, L, id, end, EV_XFER);
        next_member();
        return false;
      }
      L.phase = PH_O_INSERT_START;
      return false;
    }
    case PH_O_INSERT_START: {
      const kvg_step_plan& plan = D.plans[static_cast<size_t>(id) * L.steps + a.step];
      a.ctx += plan.gen_tokens;  // append_tokens
      L.m_nafter = pdiv(L, a.ctx);
      L.o_offl = 0;
      L.phase = PH_O_INSERT_COUNT;
      return false;
    }
    case PH_O_INSERT_COUNT:
    case PH_O_INSERT_EVICTED: {  // insert, cache_tree.cpp:170-228
      if (L.phase == PH_O_INSERT_EVICTED && L.o_ev_rec == 0) {
        L.phase = PH_O_INSERT_FAIL;
        return false;
      }
      u64 created = 0;
      const u64 stored = a.ctx - pmod(L, a.ctx);
      if (L.m_nafter > 0) {
        const u64 need = t_missing(D, L, id, L.m_nafter);
        const u64 free_slots = L.capacity - L.used;
        if (need > free_slots) {
          post_frontier(need - free_slots, PH_O_INSERT_EVICTED);
          return true;
        }
        // insert, pin(+1, stored), unpin(-1, matched): one walk (tree.cuh)
        created = t_insert_commit(D, L, id, L.m_nafter, static_cast<u32>(pdiv(L, L.o_matched)), true);
      }
      x_account(D, L, L.o_offl);
      log_rec(D, L, KVG_LOG_INSERT, id, 1, stored);
      if (L.m_nafter == 0) t_pin_move(D, L, id, stored, L.o_matched);
      a.pinned_pg = static_cast<u32>(pdiv(L, stored));
      L.created_pages += created;
      if (L.m_nafter > 0) L.refreshed_pages += pdiv(L, L.o_matched);
      member_success(D, L, id, L.m_ctx0, L.o_matched);
      next_member();
      return false;
    }
    case PH_O_INSERT_FAIL: {  // engine.cpp:366-373
      x_account(D, L, L.o_offl);
      log_rec(D, L, KVG_LOG_INSERT, id, 0, 0);
      a.ctx = L.m_ctx0;
      t_pin(D, L, id, L.o_matched, -1);
      a.pinned_pg = 0;
      st_add(D.stats[id].stall_events, 1);
      next_member();
      return false;
    }
    case PH_O_EVICT_POP: {
      L.evict_scanned += L.t_alloc;
      L.o_ev_rec = t_evict_pop(D, L, op.fr_n, L.o_ev_need, &L.o_offl);
      op.kind = OP_NONE;
      L.phase = L.o_then;
      return false;
    }
    default: {  // PH_O_MEMBER: match, pins, reload start (engine.cpp:337-346)
      const u32 nid = L.m_next;
      if (nid == NIL) {
        L.phase = PH_BATCH_END;
        return false;
      }
      AgentDev& b = L.ag[nid];
      L.m_id = nid;
      L.m_ctx0 = b.ctx;
      L.m_nctx = pdiv(L, b.ctx);
      u64 hm = 0;
      // match, pin(+1, matched), unpin(-1, pinned_len): one walk (tree.cuh)
      const u64 matched =
          t_match_pin(D, L, nid, b.ctx, static_cast<u64>(b.pinned_pg) * L.ps, &hm);
      const u64 r = pdiv(L, matched + hm);
      L.lookups += r + (r < L.m_nctx ? 1 : 0);
      L.hit_pages += pdiv(L, matched);
      log_rec(D, L, KVG_LOG_MATCH, nid, matched, hm);
      b.pinned_pg = static_cast<u32>(pdiv(L, matched));
      L.o_matched = matched;
      L.o_hm = hm;
      L.o_offl = 0;
      L.o_promoted = 0;
      if (hm == 0) {
        L.phase = PH_O_INSERT_START;
        return false;
      }
      // reload: walk to `from` = matched (cache_tree.cpp:323-335)
      if (matched >= b.ctx) {
        L.phase = PH_O_RELOAD_END;
        return false;
      }
      const TWc W = tw_ctx(D, L);
      const u64 mp = pdiv(L, matched);  // matched is whole pages
      u32 node = 0, fc = tw_get(W, 0).first_child;
      u64 pp = 0;
      while (pp < mp) {
        const u32 c = w_find_child(D, W, node, fc, nid, static_cast<u32>(pp),
                                   static_cast<u32>(L.m_nctx));
        const TWalk w = c == 0 ? TWalk{0, 0, 0, 0} : tw_get(W, c);
        if (c == 0 || pp + w.npages > mp) {
          fail(L, E_OFFLOAD);
          return false;
        }
        pp += w.npages;
        node = c;
        fc = w.first_child;
      }
      L.o_now = ++L.cclock;
      L.o_pos = matched;
      L.o_node = node;
      L.phase = PH_O_RELOAD_CHUNK;
      return false;
    }
  }
}

// Runs the state machine until a cooperative op is posted in `op`.
// kOff = false compiles the discard-only state machine: no offload phases,
// no tree code, a smaller hot loop for sweeps of discard-mode simulations.
// dispatch_member (engine.cpp:337-396) in chain mode after its match_prefix
// (PH_MEMBER): the insert loop with chain evictions, the commit / leaf and the
// success or stall bookkeeping — the same statements as the phases
// PH_M_MATCHED .. PH_M_RESTORED, straight through: no cooperative op is ever
// needed in chain mode, so the member does not return to the phase dispatch
// between them.
template <bool kBig>
__device__ __forceinline__ void chain_member(const SimDev& D, Lead& L) {
  const u64 f = L.m_f;
  const u64 matched = f * L.ps;
  L.lookups += f + (f < L.m_nctx ? 1 : 0);
  L.hit_pages += f;
  L.hit_m += static_cast<double>(matched);
  L.hit_r += static_cast<double>(L.m_ctx0);
  log_rec(D, L, KVG_LOG_MATCH, L.m_id, matched, 0);
  set_pinned(D, L, L.m_id, matched);  // pin(matched) (engine.cpp:340-342)
  AgentDev& a = L.ag[L.m_id];
  const kvg_step_plan& plan = D.plans[static_cast<size_t>(L.m_id) * L.steps + a.step];
  a.ctx += plan.gen_tokens;  // append_tokens
  L.m_nafter = pdiv(L, a.ctx);
  u64 created = 0;
  bool ok = true;
  if (L.m_nafter > 0) {  // (nothing to cache: ok, no clock bump)
    for (;;) {  // CacheTree::insert loop (cache_tree.cpp:170-187)
      const u64 need = L.m_nafter - f;  // path [0,f) is pinned: recount is constant
      const u64 free_slots = L.capacity - L.used;
      if (need <= free_slots) {
        ++L.cclock;  // insert clock bump (cache_tree.cpp:188)
        a.lazy = L.cclock;
        L.lazy_sh = L.cclock;
        created = f < L.m_nafter ? L.m_nafter - f : 0;  // the leaf extends the chain
        break;
      }
      const u64 k = need - free_slots;
      const u64 e = L.used - (L.pin_max + L.pin_priv);
      ++L.evict_calls;
      log_rec(D, L, KVG_LOG_EVICT, L.m_id, k, k < e ? k : e);
      if (e == 0) {  // O(1) nothing-evictable fast path
        ok = false;
        break;
      }
      const u64 r = k < e ? k : e;
      chain_evict(D, L, r);
      if (L.status == KVG_ERR_STATE) return;
      L.used -= r;
      L.discarded += r * L.ps;
      L.evicted += r;
    }
  }
  if (ok) {  // PH_M_CREATED
    L.used += created;
    L.created_pages += created;
    if (L.m_nafter > 0) {  // the whole path [0, n_after) is resident now
      L.refreshed_pages += f;
      const u64 sh = L.m_nafter < L.S ? L.m_nafter : L.S;
      if (sh > L.L0) L.L0 = sh;
      a.priv = static_cast<u32>(L.m_nafter > L.S ? L.m_nafter - L.S : 0);
    }
    const u64 stored = a.ctx - pmod(L, a.ctx);
    log_rec(D, L, KVG_LOG_INSERT, L.m_id, 1, stored);
    set_pinned(D, L, L.m_id, stored);  // pin(stored), unpin(matched)
    member_success(D, L, L.m_id, L.m_ctx0, matched);
    L.stall_streak = 0;
  } else {  // PH_M_FAIL + PH_M_RESTORED (engine.cpp:366-373)
    a.ctx = static_cast<u32>(L.m_ctx0);  // context.resize + token_counter rollback
    a.stalled = 1;
    set_pinned(D, L, L.m_id, 0);  // unpin(matched); pinned_len = 0
    if (a.priv > 0) ch_insert(L, L.m_id);
    st_add(D.stats[L.m_id].stall_events, 1);
    ++L.stall_streak;
    log_rec(D, L, KVG_LOG_INSERT, L.m_id, 0, 0);
  }
  L.m_next = ready_next_k<kBig>(D, L, L.m_id + 1);
}

// dispatch_batch's end (engine.cpp:317-332): the batch wall starts at
// max(clock, device busy), the ledger shares, and the completions (one group
// entry for a batch of >= group_min members, kernel 4).
template <bool kOff>
__device__ __forceinline__ void batch_end(const SimDev& D, Lead& L) {
  const u32 nb = L.batch_n;
  if (nb > 0) {
    const double wall = L.b_wall, total = L.b_total;
    const double start = L.clock < L.gpu_busy ? L.gpu_busy : L.clock;
    L.gpu_busy = start + wall;
    L.device_busy += wall;
    const double share = total > 0 ? wall / total : 0.0;
    const bool group = !(kOff && L.offload) && nb >= L.group_min;
    u32 tail = ring_at(L.gr_head, L.gr_n, L.n);
    // the ledger sums in registers across the members (same additions in
    // the same order; through Lead each would be a shared-memory round trip,
    // reloaded after every member read through the generic batch pointer)
    double lf = L.ledger.prefill_fresh, lr = L.ledger.prefill_recompute,
           ld = L.ledger.decode;
    for (u32 i = 0; i < nb; ++i) {
      const Member& m = D.batch[i];
      lf += share * m.f;
      lr += share * m.r;
      ld += share * m.d;
      if (!group) {
        sched_agent(D, L, m.id, start + wall, EV_GEN);
        continue;
      }
      // every member completes at start + wall with consecutive
      // ordinals: nothing can order between them, so the batch
      // completes as ONE group (kernel 4, coop_group)
      AgentDev& a = L.ag[m.id];
      if (a.ev_kind != EV_NONE) fail(L, E_EVENT_BUSY);
      a.ev_kind = EV_GEN;
      L.gring[tail] = m.id;
      tail = ring_at(tail, 1, L.n);
    }
    L.ledger.prefill_fresh = lf;
    L.ledger.prefill_recompute = lr;
    L.ledger.decode = ld;
    if (group) {
      L.gr_n += nb;
      heap_push(L, HeapEnt{start + wall, (L.ord << kKeyShift) | kGroupFlag | nb});
      L.ord += nb;  // the members' ordinals (engine.cpp:331)
    }
  }
  ++L.events;
}

// dispatch_batch's member loop (engine.cpp:305-333) from L.m_next on. Returns
// true when it posted a cooperative op (the caller returns to the CTA);
// otherwise L.phase says where to go on (PH_EVENT after an inline batch end in
// chain mode; a member phase in table / verify mode).
template <bool kOff, bool kChain, bool kBig = false>
__device__ __forceinline__ bool member_loop(const SimDev& D, Lead& L, Op& op) {
  for (;;) {  // chain mode: whole member attempts inline, one after another
  const u32 id = L.m_next;
  if (id == NIL) {
    if (kChain || L.chain) {  // the batch ends here, straight back to the event loop
      batch_end<kOff>(D, L);
      L.phase = PH_EVENT;
    } else {
      L.phase = PH_BATCH_END;
    }
    break;
  }
  AgentDev& a = L.ag[id];
  L.m_id = id;
  if (a.pinned_pg > 0) {  // only reachable with offload transfers
    fail(L, E_OFFLOAD);
    break;
  }
  if ((kChain || L.chain) && L.stall_streak > 0 && L.storm_on) {  // a stall storm: the warp takes the run
    op.kind = OP_STORM;
    op.err = E_NONE;
    return true;  // (coop_storm leaves L.phase at PH_MEMBER)
  }
  L.m_ctx0 = a.ctx;
  L.m_nctx = pdiv(L, a.ctx);
  L.m_now = ++L.cclock;  // match_prefix clock bump (cache_tree.cpp:115)
  // match_prefix (cache_tree.cpp:114-142). Residency is prefix-closed
  // along a path and chains only gain pages at their ends (insert) and
  // lose tails (eviction, discard), so the first miss is held
  // incrementally: L0 resident shared pages, a.priv resident private
  // ones. The refresh stamps the whole resident path; every resident
  // page of a chain carries its chain's latest stamp, so the refresh is
  // two scalar writes. verify=1 re-derives f with the
  // block-hash probe (kernel 1) and checks it.
  {
    const u64 fres = L.L0 < L.S ? L.L0 : L.S + a.priv;
    L.m_f = fres < L.m_nctx ? fres : L.m_nctx;
  }
  a.lazy = L.m_now;
  L.lazy_sh = L.m_now;
  ch_remove(L, id);  // its path is pinned from the match on
  if (kChain || L.chain) {
    chain_member<kBig>(D, L);
    if (L.status == KVG_ERR_STATE) break;
    continue;  // the next member
  }
  L.phase = PH_M_MATCHED;
  if (L.verify && L.m_nctx > 0) {
    post_range(op, id, 0, L.m_nctx, 0, 0, 0);
    return true;
  }
  op.err = E_NONE;
  break;
  }  // member loop
  return false;
}

template <bool kOff, bool kChain, bool kBig = false>  // kBig: a one-CTA-per-SM kernel
__device__ void leader_step(const SimDev& D, Lead& L, Op& op) {
  op.kind = OP_NONE;
  for (;;) {
    if (L.status == KVG_ERR_STATE && L.phase != PH_DONE && L.phase != PH_EXITED)
      L.phase = PH_DONE;
    PROF_MARK(L, L.phase);
    switch (L.phase) {
      // ------------------------------------------------ event loop (98-136)
      case PH_EVENT: {
        for (;;) {
        if (L.status == KVG_ERR_STATE) break;
        if (L.stream_on) {  // streamed host delivery: flush pending rows on the warp
          const u64 nt = L.n_trace < D.trace_cap ? L.n_trace : D.trace_cap;
          if (nt >= L.n_flushed + kFlushRows) {
            op.kind = OP_FLUSH;
            return;
          }
        }
        if (ticks_apply<kOff>(L)) {  // pipelined ticks on warp 0, then back here
          op.kind = OP_TICKS;
          return;
        }
        PROF_MARK(L, 24);
        fast_housekeeping<kBig>(D, L);
        PROF_MARK(L, PH_EVENT);
        int which = -1;  // 0 agent, 1 tick, 2 admission (the event ranks)
        double bt = 0;
        if (L.hsize > 0) {
          which = 0;
          bt = L.heap[0].t;
        }
        // ranks break time ties: completions, then the tick, then admission
        if (L.tick_on && (which < 0 || L.tick_t < bt)) {
          which = 1;
          bt = L.tick_t;
        }
        if (L.adm_on && (which < 0 || L.adm_t < bt)) {
          which = 2;
          bt = L.adm_t;
        }
        if (which < 0) {
          if (L.finished != L.n) fail(L, E_DRAINED);
          L.phase = PH_DONE;
          break;  // phase changed: through the dispatch
        }
        u32 agent = 0;
        uint8_t kind = EV_NONE;
        if (which == 0) {
          const u64 key = L.heap[0].k;
          agent = static_cast<u32>(key & ((1u << kAgentBits) - 1));
          heap_pop(D, L);
          if (key & kGroupFlag) {
            kind = EV_GROUP_POP;
          } else {
            kind = L.ag[agent].ev_kind;
            L.ag[agent].ev_kind = EV_NONE;
          }
        } else if (which == 1) {
          L.tick_on = 0;
        } else {
          L.adm_on = 0;
        }
        if (which != 0 && L.finished == L.n) continue;  // housekeeping after the end
        if (bt > L.horizon) {
          L.status = KVG_ERR_HORIZON;
          L.abort_t = bt;
          L.phase = PH_DONE;
          break;  // phase changed: through the dispatch
        }
        L.clock = bt;
        if (which == 1) {
          on_tick(D, L);
          ++L.events;
          continue;
        }
        if (which == 2) {  // on_admission_check (engine.cpp:268-291)
          PROF_MARK(L, 27);
          admission_pass(D, L);
          PROF_MARK(L, PH_EVENT);
          if (L.n_ready == 0) {  // dispatch_batch with an empty ready set
            ++L.events;
            continue;
          }
          L.batch_n = 0;
          L.stall_streak = 0;
          L.b_wall = L.b_total = 0.0;
          L.m_next = ready_next_k<kBig>(D, L, 0);  // dispatch_batch (engine.cpp:305-333)
          L.phase = PH_MEMBER;
          if (kChain || L.chain) {  // members and the batch end inline, then this loop
            PROF_MARK(L, 25);
            const bool posted = member_loop<kOff, kChain, kBig>(D, L, op);
            PROF_MARK(L, PH_EVENT);
            if (posted) return;
            if (L.phase == PH_EVENT) continue;
          }
          break;  // phase changed: through the dispatch
        }
        if (kind == EV_GROUP_POP) {  // a dispatch batch completes (kernel 4)
          L.grp_cnt = agent;  // the group's member count; members at the ring head
          L.grp_start = L.gr_head;
          L.gr_head = ring_at(L.gr_head, L.grp_cnt, L.n);
          L.gr_n -= L.grp_cnt;
          L.makespan = L.makespan < L.clock ? L.clock : L.makespan;
          op.kind = OP_GROUP;
          L.phase = PH_GROUP_DONE;
          return;
        }
        L.ev_agent = agent;
        PROF_MARK(L, 26);
        ++L.agent_events;
        AgentDev& a = L.ag[agent];
        if (kind == EV_GEN) {  // on_generation_complete (engine.cpp:184-222)
          L.makespan = L.makespan < L.clock ? L.clock : L.makespan;
          if (!(kOff && L.offload)) {
            set_pinned(D, L, agent, 0);  // unpin(pinned_len) — implicit pins
            if (a.priv > 0) ch_insert(L, agent);
          } else if (a.pinned_pg > 0) {  // engine.cpp:188-191 on the tree
            t_pin(D, L, agent, static_cast<u64>(a.pinned_pg) * L.ps, -1);
            a.pinned_pg = 0;
          }
          kvg_agent_stats& st = D.stats[agent];
          L.decoded_cum += a.f_gen;
          L.rec_cum += a.f_rec;
          st_add(st.generated_tokens, a.f_gen);
          st_add(st.recompute_tokens, a.f_rec);
          if (a.f_rec > 0) st_add(st.recompute_events, 1);
          ++a.step;
          if (a.step >= L.steps) {
            set_state(D, L, agent, S_DONE);
            if (kOff && L.offload) {  // discard_suffix on the tree (device and host pages)
              op.freed = static_cast<unsigned int>(t_discard(D, L, agent, a.ctx, L.shared_len));
              op.err = E_NONE;
              L.phase = PH_GEN_DISCARDED;
              break;  // phase changed: through the dispatch
            }
            // discard_suffix(context, shared_len) (cache_tree.cpp:404-437) on
            // the held state: the finished agent's private pages from
            // page_ceil(shared_len) on leave the cache (a straddling page
            // stays, quirk Q2). Its chain only shrinks to `keep`; the pages
            // left in the table beyond a chain's held length are absent to
            // every reader (eviction candidates, rehash).
            {
              const u64 fp = pdiv(L, L.shared_len + L.ps - 1);
              const u64 keep = fp > L.S ? fp - L.S : 0;
              op.freed = a.priv > keep ? static_cast<unsigned int>(a.priv - keep) : 0u;
            }
            op.err = E_NONE;
            L.phase = PH_GEN_DISCARDED;
            break;  // phase changed: through the dispatch
          }
          const bool req = L.kind == KVG_POLICY_REQUEST_CAP;
          if (a.f_has_tool) {
            set_state(D, L, agent, S_TOOL);
            L.ledger.tool_wait += a.f_tool;
            if (req) act_erase(D, L, agent);
            sched_agent(D, L, agent, L.clock + a.f_tool, EV_TOOL);
          } else {
            set_state(D, L, agent, S_AWAIT);
            a.ready_since = L.clock;
            if (req) {
              act_erase(D, L, agent);
              pend_push(D, L, agent);
            }
          }
          sched_admission(L);
          ++L.events;
          continue;
        }
        if (kind == EV_XFER) {  // on_transfer_complete (engine.cpp:237-243)
          L.makespan = L.makespan < L.clock ? L.clock : L.makespan;
          set_state(D, L, agent, S_AWAIT);
          a.ready_since = L.clock;
          sched_admission(L);
          ++L.events;
          continue;
        }
        if (kind == EV_TOOL) {  // on_tool_complete (engine.cpp:224-235)
          L.makespan = L.makespan < L.clock ? L.clock : L.makespan;
          a.ctx += a.f_obs;
          a.f_obs = 0;
          a.f_has_tool = 0;
          set_state(D, L, agent, S_AWAIT);
          a.ready_since = L.clock;
          if (L.kind == KVG_POLICY_REQUEST_CAP) pend_push(D, L, agent);
          else if (!a.in_active) fail(L, E_NOT_ACTIVE);
          sched_admission(L);
          ++L.events;
          continue;
        }
        fail(L, E_OFFLOAD);
        break;
        }  // an event that leaves the phase at PH_EVENT loops here, not through the switch
        continue;
      }
      // --------------------------------------------- dispatch_member (337-396)
      case PH_MEMBER: {
        if (kOff && L.offload) {
          L.phase = PH_O_MEMBER;
          continue;
        }
        if (member_loop<kOff, kChain, kBig>(D, L, op)) return;
        continue;
      }
      case PH_M_MATCHED: {
        if constexpr (kChain) __builtin_unreachable();
        const u64 f = L.m_f;
        if (L.verify && L.m_nctx > 0) {  // the probe must agree with the held state
          if (op.err) fail(L, op.err);
          const u64 fp = op.first_miss < L.m_nctx ? op.first_miss : L.m_nctx;
          if (fp != f || op.resident != f) fail(L, E_PREFIX_BROKEN);
        }
        const u64 matched = f * L.ps;
        L.lookups += f + (f < L.m_nctx ? 1 : 0);
        L.hit_pages += f;
        L.hit_m += static_cast<double>(matched);
        L.hit_r += static_cast<double>(L.m_ctx0);
        log_rec(D, L, KVG_LOG_MATCH, L.m_id, matched, 0);
        set_pinned(D, L, L.m_id, matched);  // pin(matched) (engine.cpp:340-342)
        AgentDev& a = L.ag[L.m_id];
        const kvg_step_plan& plan = D.plans[static_cast<size_t>(L.m_id) * L.steps + a.step];
        a.ctx += plan.gen_tokens;  // append_tokens
        L.m_nafter = pdiv(L, a.ctx);
        L.m_f = f;
        L.rebuilt = 0;
        L.phase = PH_M_INSERT;
        continue;
      }
      case PH_M_INSERT: {  // CacheTree::insert loop (cache_tree.cpp:170-187)
        if constexpr (kChain) __builtin_unreachable();
        if (L.m_nafter == 0) {  // nothing to cache: ok, no clock bump
          op.created = 0;
          L.phase = PH_M_CREATED;
          continue;
        }
        const u64 need = L.m_nafter - L.m_f;  // path [0,f) is pinned: recount is constant
        const u64 free_slots = L.capacity - L.used;
        if (need <= free_slots) {
          L.phase = PH_M_COMMIT;
          continue;
        }
        const u64 k = need - free_slots;
        const u64 e = L.used - (L.pin_max + L.pin_priv);
        ++L.evict_calls;
        log_rec(D, L, KVG_LOG_EVICT, L.m_id, k, k < e ? k : e);
        if (e == 0) {  // O(1) nothing-evictable fast path
          L.phase = PH_M_FAIL;
          continue;
        }
        if (L.chain) {  // chain LRU: no page table, no cooperative op
          const u64 r = k < e ? k : e;
          chain_evict(D, L, r);
          L.used -= r;
          L.discarded += r * L.ps;
          L.evicted += r;
          continue;  // PH_M_INSERT again (cache_tree.cpp:176-186)
        }
        L.m_k = k;
        L.m_e = e;
        L.evict_scanned += L.used;
        op.kind = OP_EVICT;
        op.k = k;
        op.evictable = e;
        op.clock = L.cclock;
        op.agent = L.m_id;
        op.log_clock = L.cclock;
        op.pin_max = L.pin_max;
        op.lazy_sh = L.lazy_sh;
        op.l0_min = NIL;
        op.err = E_NONE;
        L.phase = PH_M_EVICTED;
        return;
      }
      case PH_M_EVICTED: {
        if constexpr (kChain) __builtin_unreachable();
        const u64 r = op.freed;
        const u64 expect = L.m_k < L.m_e ? L.m_k : L.m_e;
        if (r != expect || op.err) fail(L, E_EVICT_MISMATCH);
        if (op.l0_min < L.L0) L.L0 = op.l0_min;  // (private tails: a.priv, in the scatter)
        L.used -= r;
        L.discarded += r * L.ps;
        L.evicted += r;
        L.phase = PH_M_INSERT;
        continue;
      }
      case PH_M_COMMIT: {
        if constexpr (kChain) __builtin_unreachable();
        if (!L.chain && static_cast<u64>(op.occ_n) + range_chunks(L.m_f, L.m_nafter) >
                            (static_cast<u64>(op.mask) + 1) / 2) {
          if (L.rebuilt) {
            fail(L, E_TABLE_FULL);
            continue;
          }
          L.rebuilt = 1;
          op.kind = OP_REBUILD;
          L.phase = PH_M_COMMIT;
          return;
        }
        ++L.cclock;  // insert clock bump (cache_tree.cpp:188) == m_now + 1
        // the walk refreshes the whole path (chain stamps) and a leaf holds
        // the missing pages [f, n_after): kernel 1 creates them
        L.ag[L.m_id].lazy = L.cclock;
        L.lazy_sh = L.cclock;
        L.phase = PH_M_CREATED;
        if (L.chain) {  // the leaf [f, n_after) extends the agent's chain
          op.created = L.m_f < L.m_nafter ? static_cast<unsigned int>(L.m_nafter - L.m_f) : 0u;
          op.err = E_NONE;
          continue;
        }
        if (L.m_f < L.m_nafter) {
          post_range(op, L.m_id, L.m_f, L.m_nafter, RF_CREATE, 0, L.cclock);
          return;
        }
        op.kind = OP_NONE;
        op.created = 0;
        op.err = E_NONE;
        continue;
      }
      case PH_M_CREATED: {
        if constexpr (kChain) __builtin_unreachable();
        if (op.err) fail(L, op.err);
        L.used += op.created;
        L.created_pages += op.created;
        if (L.m_nafter > 0) L.refreshed_pages += L.m_f;
        AgentDev& a = L.ag[L.m_id];
        if (L.m_nafter > 0) {  // the whole path [0, n_after) is resident now
          const u64 sh = L.m_nafter < L.S ? L.m_nafter : L.S;
          if (sh > L.L0) L.L0 = sh;
          a.priv = static_cast<u32>(L.m_nafter > L.S ? L.m_nafter - L.S : 0);

        }
        const u64 stored = a.ctx - pmod(L, a.ctx);
        const u64 matched = L.m_f * L.ps;
        log_rec(D, L, KVG_LOG_INSERT, L.m_id, 1, stored);
        set_pinned(D, L, L.m_id, stored);  // pin(stored), unpin(matched)
        member_success(D, L, L.m_id, L.m_ctx0, matched);
        L.stall_streak = 0;
        L.m_next = ready_next(D, L, L.m_id + 1);
        L.phase = PH_MEMBER;
        continue;
      }
      case PH_M_FAIL: {  // insert failed: engine.cpp:366-373
        if constexpr (kChain) __builtin_unreachable();
        AgentDev& a = L.ag[L.m_id];
        a.ctx = static_cast<u32>(L.m_ctx0);  // context.resize + token_counter rollback
        a.stalled = 1;
        op.err = E_NONE;  // the path keeps the match's stamp (a.lazy, lazy_sh)
        L.phase = PH_M_RESTORED;
        continue;
      }
      case PH_M_RESTORED: {
        if constexpr (kChain) __builtin_unreachable();
        if (op.err) fail(L, op.err);
        set_pinned(D, L, L.m_id, 0);  // unpin(matched); pinned_len = 0
        if (L.ag[L.m_id].priv > 0) ch_insert(L, L.m_id);
        st_add(D.stats[L.m_id].stall_events, 1);
        ++L.stall_streak;
        log_rec(D, L, KVG_LOG_INSERT, L.m_id, 0, 0);
        L.m_next = ready_next(D, L, L.m_id + 1);
        L.phase = PH_MEMBER;
        continue;
      }
      case PH_BATCH_END: {  // engine.cpp:317-332
        batch_end<kOff>(D, L);
        L.phase = PH_EVENT;
        continue;
      }
      case PH_GEN_DISCARDED: {
        if (op.err) fail(L, op.err);
        const u32 id = L.ev_agent;
        if (!(kOff && L.offload)) {  // (the tree discard accounted for itself)
          L.used -= op.freed;
          L.discarded += static_cast<u64>(op.freed) * L.ps;
          // pages from page_ceil(shared_len) on are gone (a straddling page stays, Q2)
          const u64 fp = pdiv(L, L.shared_len + L.ps - 1);
          const u64 keep = fp > L.S ? fp - L.S : 0;
          AgentDev& a = L.ag[id];
          if (a.priv > keep) a.priv = static_cast<u32>(keep);
          if (a.priv == 0) ch_remove(L, id);
        }
        log_rec(D, L, KVG_LOG_DISCARD, id, 0, op.freed);
        act_erase(D, L, id);  // on_request_complete / on_agent_finished
        ++L.finished;
        D.stats[id].finish_time = L.clock;
        D.stats[id].finish_ordinal = L.events;
        log_rec(D, L, KVG_LOG_FINISH, id, __double_as_longlong(L.clock), L.events);
        sched_admission(L);
        ++L.events;
        L.phase = PH_EVENT;
        continue;
      }
      case PH_GROUP_DONE:  // coop_group did every member's completion
        if (op.err) fail(L, op.err);
        L.phase = PH_EVENT;
        continue;
      case PH_O_MEMBER:
      case PH_O_RELOAD_CHUNK:
      case PH_O_RELOAD_EVICTED:
      case PH_O_RELOAD_END:
      case PH_O_INSERT_START:
      case PH_O_INSERT_COUNT:
      case PH_O_INSERT_EVICTED:
      case PH_O_INSERT_FAIL:
      case PH_O_EVICT_POP:
        if constexpr (kOff) {
          if (offload_step(D, L, op)) return;
        }
        continue;
      case PH_DONE:  // phase labels over the trace rows (warp 0), then the result
        op.kind = OP_PHASES;
        L.phase = PH_FINAL;
        return;
      case PH_FINAL:
        finalize(D, L);
        L.phase = PH_EXITED;
        op.kind = OP_EXIT;
        return;
      default:
        op.kind = OP_EXIT;
        return;
    }
  }
}

// ------------------------------------------------------ kernel 4: group advance
// OP_GROUP (warp 0): the completions of one dispatch batch. Every member of a
// batch completes at start + wall (engine.cpp:317-332) with consecutive event
// ordinals, so the reference processes them back to back — no other event can
// order between them (ticks and admission checks rank after completions at
// equal times, new events get later ordinals). The agent state machines
// (on_generation_complete, engine.cpp:184-222: unpin, statistics, step,
// Generating -> Finished | ToolExecuting | AwaitingAdmission, discard_suffix
// of finishers) therefore advance one member per LANE; the order-dependent
// side effects — event ordinals of tool completions and of the admission
// check, the ledger's tool-wait sum, pending-FIFO pushes, finish ordinals,
// the event log — are applied by lane 0 in member order afterwards, with the
// same operations in the same order as the per-event path.
__device__ __noinline__ void coop_group(const SimDev& D, Lead& L, Op& op, int lane) {
  const u32 cnt = L.grp_cnt, n = L.n;
  const double T = L.clock;
  const u64 S = L.S;
  const bool req = L.kind == KVG_POLICY_REQUEST_CAP;
  const u64 fp = pdiv(L, L.shared_len + L.ps - 1);
  const u64 keep = fp > S ? fp - S : 0;  // discard_suffix keeps page_ceil(shared) (Q2)
  const u64 ev0 = L.events;
  u64 gen = 0, rec = 0, ppriv = 0;
  u32 finished = 0, erased = 0, readied = 0;
  int bad = 0;
  for (u32 off = 0; off < cnt; off += 32) {
    const u32 k = off + lane;
    if (k < cnt) {
      const u32 id = L.gring[ring_at(L.grp_start, k, n)];
      AgentDev& a = L.ag[id];
      if (a.ev_kind != EV_GEN || a.state != S_GEN) bad = E_ILLEGAL_TRANSITION;
      a.ev_kind = EV_NONE;
      // unpin(pinned_len) (engine.cpp:188-191): implicit pins, histogram
      const u64 old_pg = a.pinned_pg;
      a.pinned_pg = 0;
      ppriv += old_pg > S ? old_pg - S : 0;
      const u64 jo = old_pg < S ? old_pg : S;
      if (jo > 0 && atomicSub(&D.pin_hist[jo], 1u) == 1u)
        atomicAnd(&D.pin_lvl[jo >> 5], ~(1u << (jo & 31)));
      kvg_agent_stats& st = D.stats[id];
      gen += a.f_gen;
      rec += a.f_rec;
      st_add(st.generated_tokens, a.f_gen);
      st_add(st.recompute_tokens, a.f_rec);
      if (a.f_rec > 0) st_add(st.recompute_events, 1);
      ++a.step;
      if (a.step >= L.steps) {  // Finished: discard_suffix (lane 0, below) + on_agent_finished
        a.state = S_DONE;
        if (!a.in_active) bad = E_NOT_ACTIVE;
        a.in_active = 0;
        ++erased;
        ++finished;
        st.finish_time = T;
        st.finish_ordinal = ev0 + k;
      } else if (a.f_has_tool) {
        a.state = S_TOOL;
        if (req) {
          if (!a.in_active) bad = E_NOT_ACTIVE;
          a.in_active = 0;
          ++erased;
        }
      } else {
        a.state = S_AWAIT;
        a.ready_since = T;
        if (req) {
          if (!a.in_active) bad = E_NOT_ACTIVE;
          a.in_active = 0;
          ++erased;
        } else if (a.in_active) {  // ready_sync: active and at a step boundary
          a.ready = 1;
          const u32 w = id >> 5;
          if (atomicOr(&L.rbits[w], 1u << (id & 31)) == 0u) atomicOr(&L.rl1[w >> 5], 1u << (w & 31));
          ++readied;
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    gen += __shfl_xor_sync(FULL, gen, o);
    rec += __shfl_xor_sync(FULL, rec, o);
    ppriv += __shfl_xor_sync(FULL, ppriv, o);
  }
  finished = __reduce_add_sync(FULL, finished);
  erased = __reduce_add_sync(FULL, erased);
  readied = __reduce_add_sync(FULL, readied);
  bad = static_cast<int>(__reduce_max_sync(FULL, static_cast<u32>(bad)));
  __syncwarp();
  if (lane != 0) return;
  op.err = bad;
  L.decoded_cum += gen;
  L.rec_cum += rec;
  L.pin_priv -= ppriv;
  if (S > 0 && L.pin_max > 0 && D.pin_hist[L.pin_max] == 0) {  // highest pinned level left
    u64 w = L.pin_max >> 5;
    u32 bits = D.pin_lvl[w] & ((1u << (L.pin_max & 31)) - 1);
    while (bits == 0 && w > 0) bits = D.pin_lvl[--w];
    L.pin_max = bits ? (w << 5) + 31 - __clz(bits) : 0;
  }
  L.finished += finished;
  L.act_size -= erased;
  L.n_ready += readied;
  L.agent_events += cnt;
  // member order: the sequential side effects of each completion handler
  for (u32 k = 0; k < cnt; ++k) {
    const u32 id = L.gring[ring_at(L.grp_start, k, n)];
    AgentDev& a = L.ag[id];
    if (a.state == S_DONE) {  // PH_GEN_DISCARDED's order
      const u64 fr = a.priv > keep ? a.priv - keep : 0;
      if (fr) {
        a.priv = static_cast<u32>(keep);
        L.used -= fr;
        L.discarded += fr * L.ps;
      }
      if (a.priv > 0) ch_insert(L, id);
      if (L.log_on) {
        log_store(D, L, KVG_LOG_DISCARD, id, 0, fr);
        log_store(D, L, KVG_LOG_FINISH, id, __double_as_longlong(T), ev0 + k);
      }
    } else if (a.state == S_TOOL) {
      if (a.priv > 0) ch_insert(L, id);
      L.ledger.tool_wait += a.f_tool;
      a.ev_kind = EV_TOOL;
      heap_push(L, HeapEnt{T + a.f_tool, (L.ord++ << kKeyShift) | id});
    } else {
      if (a.priv > 0) ch_insert(L, id);
      if (req) pend_push(D, L, id);
    }
    sched_admission(L);
  }
  L.events += cnt;
}

// ---------------------------------------------------- stall storms (dispatch)
// OP_STORM (warp 0): in an overcommitted run every dispatch attempt of an
// admission check can stall — insert finds need > free slots and nothing
// evictable (cache_tree.cpp:176-186), the member is restored and stays ready
// (engine.cpp:366-373). While attempts keep failing nothing they depend on
// changes (used pages, resident chains, the other agents' pins: each attempt
// pins its matched prefix and unpins it again), so every attempt's outcome
// follows from the state at the start of the run plus its own match: lane k
// evaluates the k-th next ready agent's match / insert / evictability exactly
// as the per-member path would. The leading lanes that stall form the run;
// lane 0 then applies the order-dependent effects member by member (clock
// bumps and stamps, the hit-window sums, chain-heap moves, the log). The
// first attempt that would not stall is left to the per-member path.
__device__ __noinline__ void coop_storm(const SimDev& D, Lead& L, Op& op, int lane) {
  const u64 S = L.S, ps = L.ps;
  const u64 free_slots = L.capacity - L.used;
  u32 cur = L.m_next;
  for (;;) {
    // lane k <- the k-th ready agent from `cur` on: the bitmap words from
    // cur's on, 32 per round (one coalesced load), set bits ranked by a warp
    // prefix sum of their popcounts
    u32 id = NIL;
    {
      const u32 w0 = cur >> 5;
      u32 found = 0;
      for (u32 base = 0; found < 32 && w0 + base < L.nwords; base += 32) {
        const u32 w = w0 + base + static_cast<u32>(lane);
        u32 word = w < L.nwords ? L.rbits[w] : 0u;
        if (base == 0 && lane == 0) word &= ~0u << (cur & 31);
        const u32 cnt = __popc(word);
        u32 incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
          const u32 v = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += v;
        }
        const u32 total = __shfl_sync(FULL, incl, 31);
        const u32 want = static_cast<u32>(lane) - found;  // rank within this round
        const bool mine = static_cast<u32>(lane) >= found && want < total;
        u32 src = 0;  // the first lane whose inclusive count exceeds `want`
        for (int bb = 16; bb > 0; bb >>= 1) {
          const u32 v = __shfl_sync(FULL, incl, src + bb - 1);
          if (mine && v <= want) src += bb;
        }
        const u32 wsrc = __shfl_sync(FULL, word, src);
        const u32 before = __shfl_sync(FULL, incl - cnt, src);
        if (mine) {
          u32 m = wsrc;
          for (u32 q = want - before; q > 0; --q) m &= m - 1;
          id = ((w0 + base + src) << 5) + static_cast<u32>(__ffs(m) - 1);
        }
        found += total;
      }
    }
    // this lane's attempt, evaluated on the state the run leaves unchanged
    bool stalls = false, heaped = false;
    u64 ctx0 = 0, nctx = 0, f = 0, k_evict = 0;
    if (id != NIL) {
      const AgentDev& a = L.ag[id];
      heaped = L.lru != nullptr && (a.priv > 0 || ch_has(L, id));
      ctx0 = a.ctx;
      nctx = pdiv(L, ctx0);
      const u64 fres = L.L0 < S ? L.L0 : S + a.priv;
      f = fres < nctx ? fres : nctx;
      const kvg_step_plan& plan = D.plans[static_cast<size_t>(id) * L.steps + a.step];
      const u64 nafter = pdiv(L, ctx0 + plan.gen_tokens);
      const u64 need = nafter - f;
      // evictable with this attempt's own pin of [0, f) in place
      const u64 jn = f < S ? f : S;
      const u64 pmax = L.pin_max > jn ? L.pin_max : jn;
      const u64 ppriv = L.pin_priv + (f > S ? f - S : 0);
      const u64 e = L.used - (pmax + ppriv);
      stalls = a.pinned_pg == 0 && nafter > 0 && need > free_slots && e == 0;
      k_evict = need - free_slots;
    }
    const unsigned ok = __ballot_sync(FULL, !stalls);
    const u32 run = ok ? static_cast<u32>(__ffs(ok) - 1) : 32u;
    const u64 c0 = L.cclock;
    const bool in_run = static_cast<u32>(lane) < run;
    if (in_run) {
      AgentDev& a = L.ag[id];
      a.stalled = 1;
      if (!heaped) a.lazy = c0 + lane + 1;  // match_prefix's refresh stamp
      st_add(D.stats[id].stall_events, 1);
    }
    u32 lk = in_run ? static_cast<u32>(f + (f < nctx ? 1 : 0)) : 0u;
    u32 hp = in_run ? static_cast<u32>(f) : 0u;
    lk = __reduce_add_sync(FULL, lk);
    hp = __reduce_add_sync(FULL, hp);
    const unsigned hmask = __ballot_sync(FULL, in_run && heaped);
    // member order on lane 0 (values of member k broadcast from lane k): the
    // hit-window sums, chain-heap moves, the log
    for (u32 k = 0; k < run; ++k) {
      const u64 fk = __shfl_sync(FULL, f, k);
      const u64 ck = __shfl_sync(FULL, ctx0, k);
      if (lane == 0) {
        L.hit_m += static_cast<double>(fk * ps);
        L.hit_r += static_cast<double>(ck);
      }
      if ((hmask >> k) & 1u || L.log_on) {
        const u32 idk = __shfl_sync(FULL, id, k);
        const u64 kk = __shfl_sync(FULL, k_evict, k);
        if (lane == 0) {
          if ((hmask >> k) & 1u) {  // out at the match, back with the new stamp
            ch_remove(L, idk);
            L.ag[idk].lazy = c0 + k + 1;
            if (L.ag[idk].priv > 0) ch_insert(L, idk);
          }
          if (L.log_on) {
            L.cclock = c0 + k + 1;
            log_store(D, L, KVG_LOG_MATCH, idk, fk * ps, 0);
            log_store(D, L, KVG_LOG_EVICT, idk, kk, 0);
            log_store(D, L, KVG_LOG_INSERT, idk, 0, 0);
          }
        }
      }
    }
    const u32 next = __shfl_sync(FULL, id, run < 32 ? run : 31);
    const u32 last = __shfl_sync(FULL, id, run > 0 ? run - 1 : 0);
    u32 after = NIL;
    if (run == 32) after = ready_next(D, L, last + 1);  // every lane: no broadcast
    if (lane == 0) {
      op.err = E_NONE;
      L.cclock = c0 + run;
      if (run > 0) {
        L.lazy_sh = L.cclock;
        L.lookups += lk;
        L.hit_pages += hp;
        L.evict_calls += run;
        L.stall_streak += run;
      }
      if (run < 32) {  // lane `run` holds the next attempt, which does not stall
        L.m_next = next;  // (NIL: the ready list ended; the gather covers it all)
        L.stall_streak = 0;
      } else {
        L.m_next = after;
      }
    }
    __syncwarp();
    if (run < 32 || after == NIL) break;
    cur = after;
  }
}

// ==========================================================================
// Kernels
// ==========================================================================

template <int kDepth>
__device__ __forceinline__ void run_op(Op& op, Hist& h, int tid, int warp, int lane, int nw) {
  switch (op.kind) {
    case OP_RANGE: coop_range<kDepth>(op, warp, lane, nw); break;
    case OP_EVICT: coop_evict(op, h, tid, warp, lane, nw); break;
    case OP_REBUILD: coop_rebuild(op, tid, warp, lane, nw); break;
    case OP_SCANFREE: coop_scanfree(op, warp, lane, nw); break;
    case OP_FRONTIER: coop_frontier(op, warp, lane, nw); break;
    default: break;
  }
}

// Hot agent records / event heap / ready bitmaps go to dynamic shared memory
// when the host sized it for them (capi.cu hot_smem).

__device__ __forceinline__ size_t smem_bytes_for(u32 n, bool lru) {
  const u32 nwords = (n + 31) / 32;
  return static_cast<size_t>(n) * (sizeof(AgentDev) + sizeof(HeapEnt) + 4 + (lru ? 8 : 0)) +
         (nwords + (nwords + 31) / 32) * sizeof(u32);
}

// Streamed host delivery: copies the trace rows produced since the last flush
// into this simulation's slice of the mapped pinned host array, 8 B words on
// consecutive lanes (full PCIe write bursts). Rows are append-only, so a
// flushed row never changes. Called by warp 0 after a control-tick round
// (when at least `min_rows` are pending) and by the whole CTA at the end.

__device__ __noinline__ void flush_rows(const SimDev& D, Lead& L, int t, int nt, u64 min_rows) {
  const u64 n = L.n_trace < D.trace_cap ? L.n_trace : D.trace_cap;
  const u64 f = L.n_flushed;
  if (n < f + min_rows || n == f) return;
  constexpr u64 kW = sizeof(kvg_trace_row) / sizeof(u64);
  // 16 B stores: the HBM and host slices share their 16 B alignment (both are
  // 256 B aligned per simulation), so only a leading / trailing word is single
  const u64* src = reinterpret_cast<const u64*>(D.trace);
  u64* dst = reinterpret_cast<u64*>(D.trace_out);
  u64 w0 = f * kW;
  const u64 w1 = n * kW;
  if (w0 & 1) {
    if (t == 0) dst[w0] = src[w0];
    ++w0;
  }
  const u64 pairs = (w1 - w0) >> 1;
  const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src + w0);
  ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dst + w0);
  for (u64 i = t; i < pairs; i += nt) d2[i] = s2[i];
  if (((w1 - w0) & 1) && t == nt - 1) dst[w1 - 1] = src[w1 - 1];
  if (nt == 32) __syncwarp();
  else __syncthreads();
  if (t == 0) L.n_flushed = n;
}

// Copy-mode host delivery (host_outputs == 2): at its end the simulation
// copies its rows into the batch's dense row region at a base taken from the
// batch-wide cursor (published in counts word 3), so the host receives
// exactly the rows produced in ONE copy-engine DMA after the kernel.
__device__ __noinline__ void pack_rows(const SimDev& D, Lead& L, int t, int nt) {
  const u64 n = L.n_trace < D.trace_cap ? L.n_trace : D.trace_cap;
  if (t == 0) {
    const u64 base = n ? atomicAdd(D.pack_cursor, static_cast<unsigned long long>(n)) : 0;
    D.counts[3] = base;
    L.n_flushed = base;  // (broadcast)
  }
  if (nt == 32) __syncwarp();
  else __syncthreads();
  constexpr u64 kW = sizeof(kvg_trace_row) / sizeof(u64);
  const u64* src = reinterpret_cast<const u64*>(D.trace);
  u64* dst = reinterpret_cast<u64*>(D.trace_out + L.n_flushed);
  for (u64 w = t; w < n * kW; w += nt) dst[w] = src[w];
}

template <int kDepth, bool kOff, bool kSmemDesc, bool kLru, bool kChain = false>
__device__ __forceinline__ void engine_body(const SimDev* __restrict__ sims) {
  __shared__ Lead L;
  __shared__ Op op;
  extern __shared__ __align__(16) unsigned char dyn[];
  // kSmemDesc: the descriptor (read on every event: buffer pointers, limits,
  // cost and policy parameters) is copied to shared memory once, so its
  // fields are LDS hits instead of L1 lookups that the 28 co-resident
  // simulations of the one-warp kernel keep evicting (C4: -6%)
  __shared__ __align__(16) SimDev Ds[kSmemDesc ? 1 : 1];
  if (kSmemDesc) {
    static_assert(sizeof(SimDev) % 8 == 0, "SimDev copy in 8 B words");
    const u64* src = reinterpret_cast<const u64*>(sims + blockIdx.x);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(SimDev) / 8); i += blockDim.x)
      reinterpret_cast<u64*>(Ds)[i] = src[i];
    __syncthreads();
  }
  const SimDev& D = kSmemDesc ? Ds[0] : sims[blockIdx.x];
  // radix-select bins: shared memory in the one-CTA-per-SM kernels
  __shared__ unsigned int shist[kLru ? 2 * kBins : 1];
  Hist h{kLru ? shist : D.hist, kLru ? shist + kBins : D.hist + kBins, kLru};
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const u32 n = D.n_agents;
  const u32 nwords = (n + 31) / 32;
  if (tid == 0) {
    unsigned int dyn_bytes;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn_bytes));
    size_t used = 0;
    if (n > 0 && smem_bytes_for(n, kLru) <= dyn_bytes) {  // the host sized it (capi.cu hot_smem)
      used = (smem_bytes_for(n, kLru) + 15) / 16 * 16;
      L.ag = reinterpret_cast<AgentDev*>(dyn);
      L.heap = reinterpret_cast<HeapEnt*>(dyn + static_cast<size_t>(n) * sizeof(AgentDev));
      u32* w = reinterpret_cast<u32*>(dyn + static_cast<size_t>(n) * (sizeof(AgentDev) + sizeof(HeapEnt)));
      L.gring = w;
      w += n;
      L.lru = kLru ? w : nullptr;
      if (kLru) w += 2 * static_cast<size_t>(n);
      L.rbits = w;
      L.rl1 = L.rbits + nwords;
    } else {
      L.ag = D.agents;
      L.heap = D.heap;
      L.lru = kLru ? D.lru : nullptr;
      L.gring = D.gring;
      L.rbits = D.rbits;
      L.rl1 = D.rl1;
      // a one-CTA-per-SM simulation too big for shared memory (C5: 65,536
      // agents) still keeps its ready bitmaps there (8.4 KB): dispatch walks
      // them for every member (capi.cu hot_smem sizes the same bytes)
      const size_t bm = static_cast<size_t>(nwords + (nwords + 31) / 32) * sizeof(u32);
      if (kLru && n > 0 && bm <= dyn_bytes) {
        L.rbits = reinterpret_cast<u32*>(dyn);
        L.rl1 = L.rbits + nwords;
        used = (bm + 15) / 16 * 16;
      }
    }
    // offload: the tree's walk mirror takes the rest (capi.cu big_smem)
    const size_t room = used < dyn_bytes ? (dyn_bytes - used) / kTWalkSmemBytes : 0;
    L.tw_off = static_cast<u32>(used);
    L.tw_n = kOff && D.engine.eviction == KVG_EVICT_OFFLOAD
                 ? static_cast<u32>(room < D.tcap ? room : D.tcap) : 0;
  }
  __syncthreads();
  AgentDev* const ag = L.ag;
  for (u32 i = tid; i < n; i += blockDim.x) {
    AgentDev a;
    a.ctx = static_cast<u32>(D.prompt_tokens);
    a.high_water = 0;
    a.lazy = 0;
    a.priv = 0;
    a.pinned_pg = 0;
    a.ready_since = 0;
    a.f_gen = a.f_rec = a.f_obs = 0;
    a.f_tool = 0;
    a.step = 0;
    a.stalled = 0;
    a.state = S_PENDING;
    a.ev_kind = EV_NONE;
    a.f_has_tool = 0;
    a.in_active = 0;
    a.act_seq = 0;
    a.ready = 0;
    ag[i] = a;
    if (kLru) L.lru[n + i] = NIL;  // not in the chain heap
    D.pend[i] = i;
    D.stats[i] = kvg_agent_stats{0, 0, 0, 0, 0, 0.0, -1.0, 0};
  }
  for (u32 i = tid; i < nwords; i += blockDim.x) L.rbits[i] = 0;
  for (u32 i = tid; i < (nwords + 31) / 32; i += blockDim.x) L.rl1[i] = 0;
  for (u64 i = tid; i <= D.shared_pages; i += blockDim.x) D.pin_hist[i] = 0;
  for (u64 i = tid; i <= D.shared_pages / 32; i += blockDim.x) D.pin_lvl[i] = 0;
  __syncthreads();
  if (tid == 0) lead_init(D, L, op);
  __syncthreads();
#ifdef KVG_PROFILE
  if (tid == 0) {
    for (int i = 0; i < 48; ++i) L.prof[i] = 0;
    L.prof_t = clock64();
    L.prof_ph = 47;
  }
#endif
  const bool stream = D.trace_out != nullptr && !D.pack_mode;  // streamed host delivery
  for (;;) {
    if (tid == 0) leader_step<kOff, kChain, kLru>(D, L, op);
    __syncthreads();
    if (op.kind == OP_EXIT) break;
    if (tid == 0) PROF_MARK(L, 32 + op.kind);
    if (op.kind == OP_TICKS) {
      if (warp == 0) {
        coop_ticks(D, L, lane);
        if (stream && !KVG_ROW_WT) {
          __syncwarp();
          flush_rows(D, L, lane, 32, kFlushRows);
        }
      }
    } else if (op.kind == OP_PHASES) {
      if (warp == 0) coop_phases(D, L, lane);
    } else if (op.kind == OP_GROUP) {
      if (warp == 0) coop_group(D, L, op, lane);
    } else if (op.kind == OP_STORM) {
      if (warp == 0) coop_storm(D, L, op, lane);
    } else if (op.kind == OP_FLUSH) {
      if (warp == 0) flush_rows(D, L, lane, 32, 0);
    } else if constexpr (!kChain) {  // (the chain kernel posts no page op)
      run_op<kDepth>(op, h, tid, warp, lane, nw);
    }
    __syncthreads();
    if (tid == 0) PROF_MARK(L, 46);
  }
  if (stream && !KVG_ROW_WT) flush_rows(D, L, tid, blockDim.x, 0);  // the rest
  if (D.pack_mode) pack_rows(D, L, tid, blockDim.x);
#ifdef KVG_PROFILE
  if (tid == 0) {
    PROF_MARK(L, 47);
    for (int i = 0; i < 48; ++i) atomicAdd(&g_prof[i], L.prof[i]);
  }
#endif
}

// Throughput variant: one warp per simulation, register budget (72) sized so 28
// simulations stay resident per SM: 148 x 28 = 4144 >= the 4096 C4 sweep sims,
// all in flight in one wave (measured: 24/SM leaves a 544-sim second wave).
// Shared memory is the other limit: per CTA, static (Lead + Op + descriptor
// copy) + dynamic (64 agents: 5,392 B) rounded up to 128 B, + 1 KB reserved:
// 28 x 8,320 B fits the SM's 228 KB with 512 B to spare, so Lead must not
// grow by a 128 B granule (measured: at 27 CTAs/SM the last 100 C4 sims ran
// as a second wave, 18.5 ms instead of 13.7 ms; tests/test_gpu_batch.py
// test_c4_sweep_runs_in_one_wave guards it via kvg_batch_geometry).

#ifndef KVG_SMALL_DEPTH
#define KVG_SMALL_DEPTH 2
#endif
#ifndef KVG_BIG_SMEM_DESC
#define KVG_BIG_SMEM_DESC false
#endif
#ifndef KVG_BIG_DEPTH
#define KVG_BIG_DEPTH 4
#endif
#ifndef KVG_SMALL_MINB
#define KVG_SMALL_MINB 28
#endif
__global__ void __launch_bounds__(32, KVG_SMALL_MINB) engine_kernel_small(const SimDev* __restrict__ sims) {
  engine_body<KVG_SMALL_DEPTH, false, true, false>(sims);
}

// The same for batches whose small simulations are all in chain form (discard
// mode, verify off): the table-mode phases and page ops compile out, so the
// hot state machine is smaller (the kernel is instruction-fetch bound).
__global__ void __launch_bounds__(32, KVG_SMALL_MINB) engine_kernel_small_chain(const SimDev* __restrict__ sims) {
  engine_body<KVG_SMALL_DEPTH, false, true, false, true>(sims);
}

// The same with the offload tier compiled in (batches holding offload sims).
__global__ void __launch_bounds__(32, KVG_SMALL_MINB) engine_kernel_small_off(const SimDev* __restrict__ sims) {
  engine_body<KVG_SMALL_DEPTH, true, true, false>(sims);
}

// Latency variant: up to 32 warps cooperate on one big simulation.
__global__ void __launch_bounds__(1024, 1) engine_kernel_big(const SimDev* __restrict__ sims) {
  engine_body<KVG_BIG_DEPTH, true, KVG_BIG_SMEM_DESC, true>(sims);
}

// Up to 16 warps (table / offload mode lone simulations): 128 registers.
__global__ void __launch_bounds__(512, 1) engine_kernel_mid(const SimDev* __restrict__ sims) {
  engine_body<KVG_BIG_DEPTH, true, KVG_BIG_SMEM_DESC, true>(sims);
}

// Lone chain-form simulations (discard mode, verify off; 1-2 warps: nothing to
// parallelise inside an event but the warp steps): the register budget of a
// 64-thread CTA, so the leader's state machine does not spill, and only the
// chain-form code (no table phases, page ops or offload tier).
__global__ void __launch_bounds__(64, 1) engine_kernel_lone(const SimDev* __restrict__ sims) {
  engine_body<KVG_BIG_DEPTH, false, KVG_BIG_SMEM_DESC, true, true>(sims);
}

}  // namespace kvg

#include "cache.cuh"
