// Leader state machine of the B200 engine (included by engine.cu).
//
// Thread 0 of each CTA executes the reference's sequential semantics; every
// function below cites the reference lines it follows. Whenever page-level
// work is needed it posts a cooperative op (engine.cu) and returns; the CTA
// executes the op and thread 0 resumes at the continuation phase.
#pragma once

namespace kvg {

constexpr u32 NIL = 0xffffffffu;

enum Phase : int {
  PH_INIT = 0,
  PH_EVENT,
  PH_ARGMIN_DONE,
  PH_ADM_READY,
  PH_MEMBER,
  PH_M_MATCHED,
  PH_M_INSERT,
  PH_M_EVICTED,
  PH_M_COMMIT,
  PH_M_REBUILT,
  PH_M_CREATED,
  PH_M_FAIL,
  PH_M_RESTORED,
  PH_BATCH_END,
  PH_GEN_UNPINNED,
  PH_GEN_DISCARDED,
  PH_DONE,
  PH_EXITED,
};

struct Lead {
  int phase, status, err, rebuilt;
  // event queue (engine.cpp:46-68, 139-154)
  double clock, gpu_busy, makespan, device_busy, tick_t, adm_t;
  u64 ord, tick_o, adm_o;
  int tick_on, adm_on, amin_valid, amin_any;
  double amin_t;
  u64 amin_o;
  u32 amin_a, finished, n_ready, ev_agent;
  // cache scalars (cache_tree.hpp:187-197)
  u64 used, cclock, pinned_pages, discarded, lookups, agent_steps, events, evict_calls,
      evicted;
  u64 hit_pages, created_pages, refreshed_pages, evict_scanned, agent_events;
  double hit_m, hit_r;
  // controller (controller.hpp:117-126)
  double window, su, sh;
  int have_s, gated;
  u64 ticks;
  u32 act_head, act_tail, act_size, pend_head, pend_size, paus_head, paus_size, pad0;
  // metrics
  u64 decoded_cum, rec_cum;
  kvg_ledger ledger;
  unsigned long long n_trace, n_log;
  // dispatch context
  u32 nready, ready_i, batch_n, m_id;
  u64 m_ctx0, m_f, m_nctx, m_nafter, m_now, m_k, m_e;
  // config snapshot
  double interval, decay, horizon, capacity_d;
  u64 capacity, ps, shared_len;
  u32 n, steps, kind, cap;
  kvg_controller_config cfg;
};

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ void log_rec(const SimDev& D, Lead& L, u32 kind, u32 agent, u64 a,
                                        u64 b) {
  if (D.log == nullptr) return;
  unsigned long long i = L.n_log++;
  if (i < D.log_cap) D.log[i] = kvg_log_record{kind, agent, L.cclock, a, b};
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

__device__ __forceinline__ void fail(Lead& L, int code) {
  if (L.err == E_NONE) L.err = code;
  L.status = KVG_ERR_STATE;
}

// AgentRecord::set_state (workload.cpp:130-137) + ready-count upkeep.
__device__ __forceinline__ void set_state(const SimDev& D, Lead& L, u32 id, uint8_t s) {
  AgentDev& a = D.agents[id];
  if (!legal_edge(a.state, s)) {
    fail(L, E_ILLEGAL_TRANSITION);
    return;
  }
  if (a.in_active) {
    if (a.state == S_AWAIT) --L.n_ready;
    if (s == S_AWAIT) ++L.n_ready;
  }
  a.state = s;
}

__device__ __forceinline__ void act_push(const SimDev& D, Lead& L, u32 id) {
  AgentDev& a = D.agents[id];
  a.in_active = 1;
  a.next = NIL;
  a.prev = L.act_tail;
  if (L.act_tail != NIL) D.agents[L.act_tail].next = id;
  else L.act_head = id;
  L.act_tail = id;
  ++L.act_size;
  if (a.state == S_AWAIT) ++L.n_ready;
}

__device__ __forceinline__ bool act_erase(const SimDev& D, Lead& L, u32 id) {
  AgentDev& a = D.agents[id];
  if (!a.in_active) {
    fail(L, E_NOT_ACTIVE);
    return false;
  }
  if (a.prev != NIL) D.agents[a.prev].next = a.next;
  else L.act_head = a.next;
  if (a.next != NIL) D.agents[a.next].prev = a.prev;
  else L.act_tail = a.prev;
  a.in_active = 0;
  --L.act_size;
  if (a.state == S_AWAIT) --L.n_ready;
  return true;
}

__device__ __forceinline__ void pend_push(const SimDev& D, Lead& L, u32 id) {
  D.pend[(L.pend_head + L.pend_size) % L.n] = id;
  ++L.pend_size;
}
__device__ __forceinline__ u32 pend_pop(const SimDev& D, Lead& L) {
  u32 id = D.pend[L.pend_head];
  L.pend_head = (L.pend_head + 1) % L.n;
  --L.pend_size;
  return id;
}
__device__ __forceinline__ void paus_push(const SimDev& D, Lead& L, u32 id) {
  D.paus[(L.paus_head + L.paus_size) % L.n] = id;
  ++L.paus_size;
}
__device__ __forceinline__ u32 paus_pop(const SimDev& D, Lead& L) {
  u32 id = D.paus[L.paus_head];
  L.paus_head = (L.paus_head + 1) % L.n;
  --L.paus_size;
  return id;
}

// Engine::schedule for agent events (engine.cpp:143-145); keeps the cached
// minimum current so ticks never need a rescan.
__device__ __forceinline__ void sched_agent(const SimDev& D, Lead& L, u32 id, double t,
                                            uint8_t kind) {
  AgentDev& a = D.agents[id];
  if (a.ev_kind != EV_NONE) {
    fail(L, E_EVENT_BUSY);
    return;
  }
  const u64 o = L.ord++;
  a.ev_time = t;
  a.ev_ord = o;
  a.ev_kind = kind;
  if (L.amin_valid && (!L.amin_any || t < L.amin_t || (t == L.amin_t && o < L.amin_o))) {
    L.amin_any = 1;
    L.amin_t = t;
    L.amin_o = o;
    L.amin_a = id;
  }
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

// Engine::on_control_tick (engine.cpp:245-266) — kernel-3 signals.
__device__ void on_tick(const SimDev& D, Lead& L) {
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
    row.transfers = 0;
    row.hit_matched = m;
    row.hit_requested = r;
    D.trace[i] = row;
  }
  L.hit_m *= L.decay;  // CacheTree::decay_hit_window (cache_tree.cpp:453-456)
  L.hit_r *= L.decay;
  L.tick_on = 1;
  L.tick_t = L.clock + L.interval;
  L.tick_o = L.ord++;
  sched_admission(L);
}

// Controller::admission_pass (controller.cpp:124-160) with the commands
// applied as Engine::on_admission_check does (engine.cpp:268-291).
__device__ void admission_pass(const SimDev& D, Lead& L) {
  const u64 limit = adm_limit(L);
  if (L.gated) {
    while (L.act_size > limit) {
      u32 id = L.act_tail;
      while (id != NIL && D.agents[id].state != S_AWAIT) id = D.agents[id].prev;
      if (id == NIL) break;
      act_erase(D, L, id);
      paus_push(D, L, id);
      set_state(D, L, id, S_PAUSED);
      ++D.stats[id].pause_events;
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
      if (D.agents[id].state == S_PENDING) set_state(D, L, id, S_AWAIT);  // admit
    } else {
      break;
    }
  }
}

__device__ void finalize(const SimDev& D, Lead& L) {
  kvg_sim_result* r = D.result;
  r->status = L.status;
  r->n_phases = 0;
  r->ledger = L.ledger;
  r->makespan = L.makespan;  // max(makespan, pcie_busy_until=0) (engine.cpp:401)
  r->device_busy = L.device_busy;
  r->link_busy = 0.0;
  r->decoded_tokens = L.decoded_cum;
  r->recompute_tokens = L.rec_cum;
  u64 rec_ev = 0, stalls = 0;
  double wait = 0.0;
  for (u32 i = 0; i < L.n; ++i) {  // engine.cpp:407-412, agent order
    rec_ev += D.stats[i].recompute_events;
    stalls += D.stats[i].stall_events;
    wait += D.stats[i].wait_time;
  }
  r->recompute_events = rec_ev;
  r->stall_events = stalls;
  r->offloaded_tokens = 0;
  r->reloaded_tokens = 0;
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
  D.counts[0] = L.n_trace;
  D.counts[1] = L.n_log;
  D.counts[2] = static_cast<u64>(L.err);
}

__device__ void lead_init(const SimDev& D, Lead& L, Op& op) {
  L.status = KVG_OK;
  L.err = E_NONE;
  L.rebuilt = 0;
  L.clock = L.gpu_busy = L.makespan = L.device_busy = 0.0;
  L.ord = 0;
  L.amin_valid = 1;
  L.amin_any = 0;
  L.finished = 0;
  L.n_ready = 0;
  L.used = L.cclock = L.pinned_pages = L.discarded = L.lookups = 0;
  L.agent_steps = L.events = L.evict_calls = L.evicted = 0;
  L.hit_pages = L.created_pages = L.refreshed_pages = L.evict_scanned = L.agent_events = 0;
  L.hit_m = L.hit_r = 0.0;
  L.n = D.n_agents;
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
  L.act_head = L.act_tail = NIL;
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
  L.shared_len = D.shared_len;
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
  L.phase = PH_EVENT;
}

// Runs the state machine until a cooperative op is posted in `op`.
__device__ void leader_step(const SimDev& D, Lead& L, Op& op) {
  op.kind = OP_NONE;
  for (;;) {
    if (L.status == KVG_ERR_STATE && L.phase != PH_DONE && L.phase != PH_EXITED)
      L.phase = PH_DONE;
    switch (L.phase) {
      // ------------------------------------------------ event loop (98-136)
      case PH_EVENT: {
        if (!L.amin_valid) {
          op.kind = OP_ARGMIN;
          L.phase = PH_ARGMIN_DONE;
          return;
        }
        int which = -1;  // 0 agent, 1 tick, 2 admission
        double bt = 0;
        u64 bo = 0;
        if (L.amin_any) {
          which = 0;
          bt = L.amin_t;
          bo = L.amin_o;
        }
        if (L.tick_on && (which < 0 || L.tick_t < bt || (L.tick_t == bt && (which > 1 ||
                                                                           (which == 1 && L.tick_o < bo))))) {
          which = 1; bt = L.tick_t; bo = L.tick_o;
        }
        if (L.adm_on && (which < 0 || L.adm_t < bt || (L.adm_t == bt && (which > 2 ||
                                                                         (which == 2 && L.adm_o < bo))))) {
          which = 2; bt = L.adm_t; bo = L.adm_o;
        }
        if (which < 0) {
          if (L.finished != L.n) fail(L, E_DRAINED);
          L.phase = PH_DONE;
          continue;
        }
        u32 agent = 0;
        uint8_t kind = EV_NONE;
        if (which == 0) {
          agent = L.amin_a;
          kind = D.agents[agent].ev_kind;
          D.agents[agent].ev_kind = EV_NONE;
          L.amin_valid = 0;
        } else if (which == 1) {
          L.tick_on = 0;
        } else {
          L.adm_on = 0;
        }
        if (which != 0 && L.finished == L.n) continue;  // housekeeping after the end
        if (bt > L.horizon) {
          L.status = KVG_ERR_HORIZON;
          L.phase = PH_DONE;
          continue;
        }
        L.clock = bt;
        if (which == 1) {
          on_tick(D, L);
          ++L.events;
          continue;
        }
        if (which == 2) {  // on_admission_check (engine.cpp:268-291)
          admission_pass(D, L);
          if (L.n_ready == 0) {  // dispatch_batch with an empty ready set
            ++L.events;
            continue;
          }
          op.kind = OP_READY;
          op.created = 0;
          L.phase = PH_ADM_READY;
          return;
        }
        L.ev_agent = agent;
        ++L.agent_events;
        AgentDev& a = D.agents[agent];
        if (kind == EV_GEN) {  // on_generation_complete (engine.cpp:184-222)
          L.makespan = L.makespan < L.clock ? L.clock : L.makespan;
          if (a.pinned > 0) {
            post_range(op, agent, 0, a.pinned / L.ps, RF_PIN | RF_STRICT, -1, 0);
            L.phase = PH_GEN_UNPINNED;
            return;
          }
          op.pin_down = 0;
          op.err = E_NONE;
          L.phase = PH_GEN_UNPINNED;
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
        continue;
      }
      case PH_ARGMIN_DONE:
        L.amin_valid = 1;
        L.amin_any = op.amin_any;
        L.amin_t = op.amin_t;
        L.amin_o = op.amin_o;
        L.amin_a = op.amin_a;
        L.phase = PH_EVENT;
        continue;
      // --------------------------------------------- dispatch_batch (305-333)
      case PH_ADM_READY:
        L.nready = op.created;
        L.ready_i = 0;
        L.batch_n = 0;
        L.phase = PH_MEMBER;
        continue;
      case PH_MEMBER: {  // dispatch_member (engine.cpp:337-396)
        if (L.ready_i >= L.nready) {
          L.phase = PH_BATCH_END;
          continue;
        }
        const u32 id = D.ready[L.ready_i];
        AgentDev& a = D.agents[id];
        L.m_id = id;
        if (a.pinned > 0) {  // only reachable with offload transfers
          fail(L, E_OFFLOAD);
          continue;
        }
        L.m_ctx0 = a.ctx;
        L.m_nctx = a.ctx / L.ps;
        L.m_now = ++L.cclock;  // match_prefix clock bump (cache_tree.cpp:115)
        // fused match_prefix + pin(matched): stamp the matched path with the
        // insert's stamp (now+1). If the insert fails it is restored to `now`;
        // while pinned its stamp is invisible to eviction.
        post_range(op, id, 0, L.m_nctx, RF_STAMP | RF_PIN, +1, L.m_now + 1);
        L.phase = PH_M_MATCHED;
        if (L.m_nctx == 0) {
          op.kind = OP_NONE;
          continue;
        }
        return;
      }
      case PH_M_MATCHED: {
        if (op.err) fail(L, op.err);
        const u64 f = op.first_miss < L.m_nctx ? op.first_miss : L.m_nctx;
        if (op.resident != f) fail(L, E_PREFIX_BROKEN);
        L.pinned_pages += op.pin_up;
        const u64 matched = f * L.ps;
        L.lookups += f + (f < L.m_nctx ? 1 : 0);
        L.hit_pages += f;
        L.hit_m += static_cast<double>(matched);
        L.hit_r += static_cast<double>(L.m_ctx0);
        log_rec(D, L, KVG_LOG_MATCH, L.m_id, matched, 0);
        AgentDev& a = D.agents[L.m_id];
        a.pinned = matched;
        const kvg_step_plan& plan = D.plans[static_cast<size_t>(L.m_id) * L.steps + a.step];
        a.ctx += plan.gen_tokens;  // append_tokens
        L.m_nafter = a.ctx / L.ps;
        L.m_f = f;
        L.rebuilt = 0;
        L.phase = PH_M_INSERT;
        continue;
      }
      case PH_M_INSERT: {  // CacheTree::insert loop (cache_tree.cpp:170-187)
        if (L.m_nafter == 0) {  // nothing to cache: ok, no clock bump
          op.created = 0;
          op.pin_up = 0;
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
        const u64 e = L.used - L.pinned_pages;
        ++L.evict_calls;
        log_rec(D, L, KVG_LOG_EVICT, L.m_id, k, k < e ? k : e);
        if (e == 0) {  // O(1) nothing-evictable fast path
          L.phase = PH_M_FAIL;
          continue;
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
        op.err = E_NONE;
        L.phase = PH_M_EVICTED;
        return;
      }
      case PH_M_EVICTED: {
        const u64 r = op.freed;
        const u64 expect = L.m_k < L.m_e ? L.m_k : L.m_e;
        if (r != expect || op.err) fail(L, E_EVICT_MISMATCH);
        L.used -= r;
        L.discarded += r * L.ps;
        L.evicted += r;
        L.phase = PH_M_INSERT;
        continue;
      }
      case PH_M_COMMIT: {
        if (static_cast<u64>(op.occ_n) + range_chunks(L.m_f, L.m_nafter) >
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
        post_range(op, L.m_id, L.m_f, L.m_nafter, RF_CREATE, +1, L.cclock);
        L.phase = PH_M_CREATED;
        if (L.m_f == L.m_nafter) {
          op.kind = OP_NONE;
          continue;
        }
        return;
      }
      case PH_M_CREATED: {
        if (op.err) fail(L, op.err);
        L.used += op.created;
        L.pinned_pages += op.pin_up;
        L.created_pages += op.created;
        if (L.m_nafter > 0) L.refreshed_pages += L.m_f;
        AgentDev& a = D.agents[L.m_id];
        const u64 stored = a.ctx - a.ctx % L.ps;
        const u64 matched = L.m_f * L.ps;
        log_rec(D, L, KVG_LOG_INSERT, L.m_id, 1, stored);
        a.pinned = stored;
        const u64 ctx0 = L.m_ctx0;
        const u64 missing = ctx0 - matched;
        const u64 rec = a.high_water > matched ? a.high_water - matched : 0;
        const u64 fresh = missing - rec;
        a.high_water = stored;
        const kvg_step_plan& plan = D.plans[static_cast<size_t>(L.m_id) * L.steps + a.step];
        Member m;
        m.id = L.m_id;
        m.pad = 0;
        m.f = prefill_t(D.cost, fresh, ctx0);
        m.r = prefill_t(D.cost, rec, ctx0);
        m.d = decode_t(D.cost, plan.gen_tokens, ctx0);
        m.t = m.f + m.r + m.d;
        D.batch[L.batch_n++] = m;
        a.f_gen = plan.gen_tokens;
        a.f_rec = rec;
        a.f_has_tool = plan.has_tool != 0;
        a.f_obs = plan.obs_tokens;
        a.f_tool = plan.tool_latency;
        D.stats[L.m_id].wait_time += L.clock - a.ready_since;
        set_state(D, L, L.m_id, S_GEN);
        ++L.agent_steps;
        ++L.ready_i;
        L.phase = PH_MEMBER;
        continue;
      }
      case PH_M_FAIL: {  // insert failed: engine.cpp:366-373
        AgentDev& a = D.agents[L.m_id];
        a.ctx = L.m_ctx0;  // context.resize + token_counter rollback
        post_range(op, L.m_id, 0, L.m_f, RF_STAMP | RF_PIN | RF_STRICT, -1, L.m_now);
        L.phase = PH_M_RESTORED;
        if (L.m_f == 0) {
          op.kind = OP_NONE;
          continue;
        }
        return;
      }
      case PH_M_RESTORED: {
        if (op.err) fail(L, op.err);
        L.pinned_pages -= op.pin_down;
        D.agents[L.m_id].pinned = 0;
        ++D.stats[L.m_id].stall_events;
        log_rec(D, L, KVG_LOG_INSERT, L.m_id, 0, 0);
        ++L.ready_i;
        L.phase = PH_MEMBER;
        continue;
      }
      case PH_BATCH_END: {  // engine.cpp:317-332
        const u32 nb = L.batch_n;
        if (nb > 0) {
          double wall = 0.0, total = 0.0;
          for (u32 i = 0; i < nb; ++i) {
            const double t = D.batch[i].t;
            wall = wall < t ? t : wall;
            total += t;
          }
          const double start = L.clock < L.gpu_busy ? L.gpu_busy : L.clock;
          L.gpu_busy = start + wall;
          L.device_busy += wall;
          const double share = total > 0 ? wall / total : 0.0;
          for (u32 i = 0; i < nb; ++i) {
            const Member& m = D.batch[i];
            L.ledger.prefill_fresh += share * m.f;
            L.ledger.prefill_recompute += share * m.r;
            L.ledger.decode += share * m.d;
            sched_agent(D, L, m.id, start + wall, EV_GEN);
          }
        }
        ++L.events;
        L.phase = PH_EVENT;
        continue;
      }
      // ------------------------------------ on_generation_complete (184-222)
      case PH_GEN_UNPINNED: {
        if (op.err) fail(L, op.err);
        const u32 id = L.ev_agent;
        AgentDev& a = D.agents[id];
        if (a.pinned > 0) {
          L.pinned_pages -= op.pin_down;
          a.pinned = 0;
        }
        kvg_agent_stats& st = D.stats[id];
        L.decoded_cum += a.f_gen;
        L.rec_cum += a.f_rec;
        st.generated_tokens += a.f_gen;
        st.recompute_tokens += a.f_rec;
        if (a.f_rec > 0) ++st.recompute_events;
        ++a.step;
        if (a.step >= L.steps) {
          set_state(D, L, id, S_DONE);
          // discard_suffix(context, shared_len) (cache_tree.cpp:404-437):
          // page_ceil(shared_len) keeps a straddling page (quirk Q2)
          const u64 fp = (L.shared_len + L.ps - 1) / L.ps;
          const u64 np = a.ctx / L.ps;
          if (fp * L.ps < a.ctx && fp < np) {
            post_range(op, id, fp, np, RF_FREE, 0, 0);
            L.phase = PH_GEN_DISCARDED;
            return;
          }
          op.freed = 0;
          op.err = E_NONE;
          L.phase = PH_GEN_DISCARDED;
          continue;
        }
        const bool req = L.kind == KVG_POLICY_REQUEST_CAP;
        if (a.f_has_tool) {
          set_state(D, L, id, S_TOOL);
          L.ledger.tool_wait += a.f_tool;
          if (req) act_erase(D, L, id);
          sched_agent(D, L, id, L.clock + a.f_tool, EV_TOOL);
        } else {
          set_state(D, L, id, S_AWAIT);
          a.ready_since = L.clock;
          if (req) {
            act_erase(D, L, id);
            pend_push(D, L, id);
          }
        }
        sched_admission(L);
        ++L.events;
        L.phase = PH_EVENT;
        continue;
      }
      case PH_GEN_DISCARDED: {
        if (op.err) fail(L, op.err);
        const u32 id = L.ev_agent;
        L.used -= op.freed;
        L.discarded += static_cast<u64>(op.freed) * L.ps;
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
      case PH_DONE:
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

// ==========================================================================
// Kernels
// ==========================================================================

__device__ __forceinline__ void run_op(Op& op, Hist& h, Red& red, const AgentDev* ag, u32 n,
                                       u32* ready, int tid, int warp, int lane, int nw) {
  switch (op.kind) {
    case OP_RANGE: coop_range(op, warp, lane, nw); break;
    case OP_EVICT: coop_evict(op, h, tid, warp, lane, nw); break;
    case OP_ARGMIN: coop_argmin(op, red, ag, n, tid, warp, lane, nw); break;
    case OP_REBUILD: coop_rebuild(op, tid, warp, lane, nw); break;
    case OP_SCANFREE: coop_scanfree(op, warp, lane, nw); break;
    case OP_READY: coop_ready(op, ag, n, ready, tid, warp, lane, nw); break;
    default: break;
  }
}

__device__ __forceinline__ void engine_body(const SimDev* __restrict__ sims) {
  __shared__ Lead L;
  __shared__ Op op;
  __shared__ Hist h;
  __shared__ Red red;
  const SimDev& D = sims[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const u32 n = D.n_agents;
  for (u32 i = tid; i < n; i += blockDim.x) {
    AgentDev a;
    a.ev_time = 0;
    a.ev_ord = 0;
    a.ctx = D.prompt_tokens;
    a.high_water = a.pinned = 0;
    a.ready_since = 0;
    a.f_gen = a.f_rec = a.f_obs = 0;
    a.f_tool = 0;
    a.step = 0;
    a.state = S_PENDING;
    a.ev_kind = EV_NONE;
    a.f_has_tool = 0;
    a.in_active = 0;
    a.next = a.prev = NIL;
    D.agents[i] = a;
    D.pend[i] = i;
    D.stats[i] = kvg_agent_stats{0, 0, 0, 0, 0, 0.0, -1.0, 0};
  }
  if (tid == 0) lead_init(D, L, op);
  __syncthreads();
  for (;;) {
    if (tid == 0) leader_step(D, L, op);
    __syncthreads();
    if (op.kind == OP_EXIT) break;
    run_op(op, h, red, D.agents, n, D.ready, tid, warp, lane, nw);
    __syncthreads();
  }
}

// Throughput variant: one warp per simulation, register budget sized so ~24
// simulations stay resident per SM (C4: 4096 sweep sims all in flight).
__global__ void __launch_bounds__(32, 24) engine_kernel_small(const SimDev* __restrict__ sims) {
  engine_body(sims);
}

// Latency variant: up to 32 warps cooperate on one big simulation.
__global__ void __launch_bounds__(1024, 1) engine_kernel_big(const SimDev* __restrict__ sims) {
  engine_body(sims);
}

// --------------------------------------------------------------------------
// Cache-op executor (CacheTree seam). One CTA executes ops in order.

enum CPhase : int {
  C_NEXT = 0, C_MATCH_DONE, C_INS_COUNT, C_INS_COUNTED, C_INS_EVICTED, C_INS_COMMIT,
  C_INS_DONE, C_EVICT_DONE, C_PIN_DONE, C_DISC_PROBED, C_DISC_DONE, C_END
};

struct CLead {
  int phase;
  u32 i;
  u64 used, clock, pinned, discarded, n0_victims;
  double hit_m, hit_r;
  u64 n, k, e, fp, head_owner;
  int rebuilt;
};

__device__ void cache_result(const CacheDev& C, CLead& L, Op& op, int status, u64 r0, u64 r1) {
  kvg_cache_op_result& r = C.results[L.i];
  r.status = status;
  r.r0 = r0;
  r.r1 = r1;
  r.clock = L.clock;
  r.used = L.used;
  r.victims_begin = L.n0_victims;
  r.victims_end = __ldcg(op.vic_n);
  ++L.i;
  L.phase = C_NEXT;
}

__device__ void cache_leader(const CacheDev& C, CLead& L, Op& op) {
  op.kind = OP_NONE;
  for (;;) {
    const kvg_cache_op* o = &C.ops[L.i < C.n_ops ? L.i : 0];
    switch (L.phase) {
      case C_NEXT: {
        if (L.i >= C.n_ops) {
          L.phase = C_END;
          continue;
        }
        L.n0_victims = __ldcg(op.vic_n);
        L.rebuilt = 0;
        const u64 ps = C.page_size;
        switch (o->kind) {
          case KVG_OP_MATCH:  // cache_tree.cpp:114-142
            L.n = o->len / ps;
            ++L.clock;
            post_range(op, o->agent, 0, L.n, RF_STAMP, 0, L.clock);
            L.phase = C_MATCH_DONE;
            if (L.n == 0) { op.kind = OP_NONE; continue; }
            return;
          case KVG_OP_INSERT:  // cache_tree.cpp:170-228
            L.n = o->len / ps;
            if (L.n == 0) { cache_result(C, L, op, KVG_OK, 1, 0); continue; }
            L.phase = C_INS_COUNT;
            continue;
          case KVG_OP_EVICT:
            L.k = o->arg;
            L.e = L.used - L.pinned;
            if (L.k == 0 || L.e == 0) { cache_result(C, L, op, KVG_OK, 0, 0); continue; }
            op.kind = OP_EVICT; op.k = L.k; op.evictable = L.e; op.clock = L.clock;
            op.agent = 0; op.err = E_NONE;
            L.phase = C_EVICT_DONE;
            return;
          case KVG_OP_PIN:
          case KVG_OP_UNPIN:
            if (o->arg % ps != 0 || o->arg > o->len) {
              cache_result(C, L, op, KVG_ERR_CONFIG, 0, 0);
              continue;
            }
            post_range(op, o->agent, 0, o->arg / ps, RF_PIN | RF_STRICT, o->kind == KVG_OP_PIN ? 1 : -1, 0);
            L.phase = C_PIN_DONE;
            if (o->arg == 0) { op.kind = OP_NONE; continue; }
            return;
          case KVG_OP_DISCARD: {  // cache_tree.cpp:404-437
            L.fp = (o->arg + ps - 1) / ps;
            if (L.fp * ps >= o->len || L.fp >= o->len / ps) {
              cache_result(C, L, op, KVG_OK, 0, 0);
              continue;
            }
            post_range(op, o->agent, 0, L.fp + 1, 0, 0, 0);  // path + branch head present?
            L.phase = C_DISC_PROBED;
            return;
          }
          default:
            cache_result(C, L, op, KVG_ERR_CONFIG, 0, 0);
            continue;
        }
      }
      case C_MATCH_DONE: {
        const u64 f = op.first_miss < L.n ? op.first_miss : L.n;
        const u64 matched = f * C.page_size;
        L.hit_m += static_cast<double>(matched);
        L.hit_r += static_cast<double>(o->len);
        cache_result(C, L, op, op.resident == f ? KVG_OK : KVG_ERR_STATE, matched, 0);
        continue;
      }
      case C_INS_COUNT:  // count_missing_slots (cache_tree.cpp:144-168)
        post_range(op, o->agent, 0, L.n, 0, 0, 0);
        L.phase = C_INS_COUNTED;
        return;
      case C_INS_COUNTED: {
        const u64 f = op.first_miss < L.n ? op.first_miss : L.n;
        L.fp = f;
        const u64 need = L.n - f;
        const u64 free_slots = C.capacity - L.used;
        if (need <= free_slots) { L.phase = C_INS_COMMIT; continue; }
        L.k = need - free_slots;
        L.e = L.used - L.pinned;
        if (L.e == 0) { cache_result(C, L, op, KVG_OK, 0, 0); continue; }
        op.kind = OP_EVICT; op.k = L.k; op.evictable = L.e; op.clock = L.clock;
        op.agent = o->agent; op.err = E_NONE;
        L.phase = C_INS_EVICTED;
        return;
      }
      case C_INS_EVICTED: {
        const u64 r = op.freed;
        L.used -= r;
        L.discarded += r * C.page_size;
        L.phase = C_INS_COUNT;  // eviction may strip the unpinned path: recount
        continue;
      }
      case C_INS_COMMIT: {
        if (static_cast<u64>(op.occ_n) + range_chunks(0, L.n) > (static_cast<u64>(op.mask) + 1) / 2) {
          if (L.rebuilt) { cache_result(C, L, op, KVG_ERR_STATE, 0, 0); continue; }
          L.rebuilt = 1;
          op.kind = OP_REBUILD;
          return;
        }
        ++L.clock;
        post_range(op, o->agent, 0, L.n, RF_STAMP | RF_CREATE, 0, L.clock);
        L.phase = C_INS_DONE;
        return;
      }
      case C_INS_DONE:
        L.used += op.created;
        cache_result(C, L, op, KVG_OK, 1, op.created);
        continue;
      case C_EVICT_DONE: {
        const u64 r = op.freed;
        L.used -= r;
        L.discarded += r * C.page_size;
        cache_result(C, L, op, KVG_OK, r, 0);
        continue;
      }
      case C_PIN_DONE:
        L.pinned += op.pin_up;
        L.pinned -= op.pin_down;
        cache_result(C, L, op, op.err ? KVG_ERR_STATE : KVG_OK, 0, 0);
        continue;
      case C_DISC_PROBED: {
        if (op.first_miss <= L.fp) { cache_result(C, L, op, KVG_OK, 0, 0); continue; }
        const u64 head_owner = L.fp < C.shared_pages ? 0 : static_cast<u64>(o->agent) + 1;
        op.kind = OP_SCANFREE;
        op.p0 = L.fp;
        op.owner_filter = head_owner == 0 ? ~0ull : head_owner;
        op.freed = 0;
        op.err = E_NONE;
        L.phase = C_DISC_DONE;
        return;
      }
      case C_DISC_DONE:
        L.used -= op.freed;
        L.discarded += static_cast<u64>(op.freed) * C.page_size;
        cache_result(C, L, op, op.err ? KVG_ERR_STATE : KVG_OK, op.freed, 0);
        continue;
      default:
        op.kind = OP_EXIT;
        return;
    }
  }
}

__global__ void __launch_bounds__(1024) cache_kernel(const CacheDev* __restrict__ cd) {
  __shared__ CLead L;
  __shared__ Op op;
  __shared__ Hist h;
  __shared__ Red red;
  const CacheDev& C = *cd;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  CacheState* st = reinterpret_cast<CacheState*>(C.state);
  if (tid == 0) {
    L.phase = C_NEXT;
    L.i = 0;
    L.used = st->used;
    L.clock = st->clock;
    L.pinned = st->pinned_pages;
    L.discarded = st->discarded;
    L.hit_m = st->hit_m;
    L.hit_r = st->hit_r;
    const bool sw = st->swapped & 1;
    op.table = sw ? C.alt : C.table;
    op.alt = sw ? C.table : C.alt;
    op.occ = sw ? C.alt_occ : C.occ;
    op.alt_occ = sw ? C.occ : C.alt_occ;
    op.mask = C.bucket_mask;
    op.occ_n = static_cast<unsigned int>(st->occ_n);
    op.shared_pages = C.shared_pages;
    op.log = nullptr;
    op.log_cap = 0;
    op.log_n = nullptr;
    op.vic = C.victims;
    op.vic_cap = C.victim_cap;
    op.vic_n = reinterpret_cast<unsigned long long*>(&st->n_victims);
    op.log_victims = 1;
    op.log_clock = 0;
  }
  __syncthreads();
  for (;;) {
    if (tid == 0) {
      Slot* before = op.table;
      cache_leader(C, L, op);
      (void)before;
    }
    __syncthreads();
    if (op.kind == OP_EXIT) break;
    run_op(op, h, red, nullptr, 0, nullptr, tid, warp, lane, nw);
    __syncthreads();
    if (tid == 0 && op.kind == OP_REBUILD) st->swapped ^= 1;
  }
  if (tid == 0) {
    st->used = L.used;
    st->clock = L.clock;
    st->pinned_pages = L.pinned;
    st->discarded = L.discarded;
    st->hit_m = L.hit_m;
    st->hit_r = L.hit_r;
    st->occ_n = op.occ_n;
  }
}

}  // namespace kvg
