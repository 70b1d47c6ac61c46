/* kvoracle — CPU restatement of the reference hot path. TEST INFRASTRUCTURE.
 *
 * Parity status: PINNED. Checked against the unmodified reference
 * (oracle/_ref/libkvref.so) per event (state digests through the paranoid
 * hooks), per result field (bit-exact doubles) and per eviction victim list;
 * see tests/test_oracle_vs_reference.py and tests/golden/.
 *
 * What it restates (every function cites the reference lines it follows):
 *  - the radix prefix cache as a FLAT PER-PAGE table. Every page of an
 *    agent's context is named by (owner, page index): owner 0 for a page
 *    wholly inside a shared prompt, agent+1 otherwise. This is exact for the
 *    population token scheme (workload.cpp:139-142, 167-171) and is the
 *    per-page reduction of CacheTree that SURVEY.md fact 0.3-2 / probe P4
 *    established: discard-mode eviction = the `needed` smallest
 *    (stamp asc, page index desc) unpinned resident pages.
 *  - the event loop with one outstanding event per agent plus one tick and at
 *    most one admission check, popped by (time, rank, ordinal) — equivalent
 *    to the reference heap.
 *  - controller (controller.cpp), cost model (cost_model.cpp), dispatch
 *    (engine.cpp:305-396) and completion handlers (engine.cpp:184-291).
 * Eviction-mode offload is not restated here.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py may load this library,
 * and only as the checker. The product never links it.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <limits>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../include/kvgpu.h"
#include "digest.h"

#define KVO_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string t_err = "no error";

struct Horizon : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::logic_error {
  using std::logic_error::logic_error;
};

/* ======================= flat page cache (cache_tree.cpp) =================== */

struct Page {
  std::uint64_t stamp = 0;
  std::int64_t pins = 0;
};

struct FlatCache {
  std::uint64_t capacity = 0, ps = 1, prompt = 0, shared_pages = 0;
  bool shared = false;
  std::unordered_map<std::uint64_t, Page> pages;  // resident (device) pages
  std::uint64_t used = 0, clock = 0, discarded = 0, offloaded = 0;
  double hit_m = 0, hit_r = 0;
  std::uint64_t evict_calls = 0, evicted = 0;
  std::uint64_t pinned = 0;  // resident pages with pins > 0 (evictable = used - pinned)
  std::uint64_t dsum = 0;    // running sum of kvdigest::page_term over resident pages
  std::vector<std::pair<std::uint64_t, std::uint64_t>>* victims = nullptr;
  std::vector<kvg_log_record>* log = nullptr;  // EVICT + VICTIM records
  std::uint32_t log_agent = 0;

  void init(std::uint64_t cap, std::uint64_t page, std::uint64_t p, bool sh) {
    if (cap == 0 || page == 0) throw std::invalid_argument("capacity and page size must be > 0");
    capacity = cap;
    ps = page;
    prompt = p;
    shared = sh;
    shared_pages = sh ? p / page : 0;  // pages wholly inside the shared prompt
  }
  std::uint64_t key(std::uint32_t a, std::uint64_t k) const {
    std::uint64_t owner = k < shared_pages ? 0 : std::uint64_t(a) + 1;
    return (owner << 32) | k;
  }
  static std::uint64_t term(std::uint64_t key, const Page& p) {
    return kvdigest::page_term(key >> 32, key & 0xffffffffULL, p.stamp,
                               static_cast<std::uint64_t>(p.pins), 0);
  }
  void restamp(std::uint64_t key, Page* p, std::uint64_t stamp) {
    dsum -= term(key, *p);
    p->stamp = stamp;
    dsum += term(key, *p);
  }
  void add_page(std::uint64_t key, std::uint64_t stamp) {
    Page pg{stamp, 0};
    pages.emplace(key, pg);
    dsum += term(key, pg);
    ++used;
  }
  void drop_page(std::unordered_map<std::uint64_t, Page>::iterator it) {
    dsum -= term(it->first, it->second);
    if (it->second.pins > 0) --pinned;
    pages.erase(it);
    --used;
  }
  Page* find(std::uint32_t a, std::uint64_t k) {
    auto it = pages.find(key(a, k));
    return it == pages.end() ? nullptr : &it->second;
  }
  std::uint64_t first_miss(std::uint32_t a, std::uint64_t n) {
    std::uint64_t k = 0;
    while (k < n && find(a, k) != nullptr) ++k;
    return k;
  }

  /* match_prefix, cache_tree.cpp:114-142 (discard mode: no host phase). */
  std::uint64_t match(std::uint32_t a, std::uint64_t len) {
    const std::uint64_t now = ++clock;
    const std::uint64_t f = first_miss(a, len / ps);
    for (std::uint64_t k = 0; k < f; ++k) restamp(key(a, k), find(a, k), now);
    hit_m += static_cast<double>(f * ps);
    hit_r += static_cast<double>(len);
    return f * ps;
  }

  /* descendants-first order: (stamp asc, page index desc). */
  static bool lru_before(const std::pair<std::uint64_t, Page*>& x,
                         const std::pair<std::uint64_t, Page*>& y) {
    if (x.second->stamp != y.second->stamp) return x.second->stamp < y.second->stamp;
    return (x.first & 0xffffffffULL) > (y.first & 0xffffffffULL);
  }

  /* evict, cache_tree.cpp:270-319 in its per-page form. */
  std::uint64_t evict(std::uint64_t needed) {
    if (needed == 0) return 0;
    ++evict_calls;
    if (used == pinned) {  // nothing evictable: the common stall-storm case
      if (log) log->push_back(kvg_log_record{KVG_LOG_EVICT, log_agent, clock, needed, 0});
      return 0;
    }
    std::vector<std::pair<std::uint64_t, Page*>> cand;
    for (auto& kv : pages)
      if (kv.second.pins == 0) cand.emplace_back(kv.first, &kv.second);
    std::uint64_t take = std::min<std::uint64_t>(needed, cand.size());
    if (log) log->push_back(kvg_log_record{KVG_LOG_EVICT, log_agent, clock, needed, take});
    if (take == 0) return 0;
    std::partial_sort(cand.begin(), cand.begin() + take, cand.end(), lru_before);
    for (std::uint64_t i = 0; i < take; ++i) {
      if (victims) victims->emplace_back(cand[i].first, cand[i].second->stamp);
      if (log)
        log->push_back(kvg_log_record{KVG_LOG_VICTIM, log_agent, clock, cand[i].first,
                                      cand[i].second->stamp});
      drop_page(pages.find(cand[i].first));
    }
    evicted += take;
    discarded += take * ps;
    return take;
  }

  /* insert, cache_tree.cpp:170-228. Returns ok; *inserted = new slots. */
  bool insert(std::uint32_t a, std::uint64_t len, std::uint64_t* inserted,
              std::uint64_t* evicted) {
    const std::uint64_t n = len / ps;
    if (inserted) *inserted = 0;
    if (n == 0) return true;
    for (;;) {
      std::uint64_t need = n - first_miss(a, n);  // count_missing_slots:144-168
      std::uint64_t free_slots = capacity - used;
      if (need <= free_slots) break;
      std::uint64_t ev = evict(need - free_slots);
      if (evicted) *evicted += ev;
      if (ev == 0) return false;  // evictions so far persist (Q3)
    }
    const std::uint64_t now = ++clock;
    for (std::uint64_t k = 0; k < n; ++k) {
      Page* p = find(a, k);
      if (p == nullptr) {
        add_page(key(a, k), now);
        if (inserted) ++*inserted;
      } else {
        restamp(key(a, k), p, now);
      }
    }
    return true;
  }

  /* pin / unpin, cache_tree.cpp:370-402 (page-aligned lengths). */
  void pin(std::uint32_t a, std::uint64_t len, int delta) {
    if (len % ps != 0) throw std::invalid_argument("pin length not on a node boundary");
    for (std::uint64_t k = 0; k < len / ps; ++k) {
      Page* p = find(a, k);
      if (p == nullptr) throw StateError("pin path missing from tree");
      if (delta < 0 && p->pins == 0) throw StateError("unpin on a node with zero pin count");
      const std::uint64_t kk = key(a, k);
      dsum -= term(kk, *p);
      if (p->pins == 0 && delta > 0) ++pinned;
      p->pins += delta;
      if (p->pins == 0) --pinned;
      dsum += term(kk, *p);
    }
  }

  /* discard_suffix, cache_tree.cpp:404-437. */
  void discard_suffix(std::uint32_t a, std::uint64_t len, std::uint64_t from) {
    from = (from + ps - 1) / ps * ps;  // page_ceil (Q2: straddling page survives)
    if (from >= len) return;
    const std::uint64_t fp = from / ps;
    if (fp >= len / ps) return;            // no full page at `from`
    for (std::uint64_t k = 0; k <= fp; ++k)  // path to `from` and the branch head
      if (find(a, k) == nullptr) return;
    // the branch subtree: pages on any path through page fp
    std::vector<std::uint64_t> doomed;
    const std::uint64_t head_owner = key(a, fp) >> 32;
    if (head_owner != 0) {
      // private head: the subtree is this agent's chain from fp (resident
      // pages of a chain are a contiguous prefix: walk until the first miss)
      for (std::uint64_t k = fp;; ++k) {
        auto it = pages.find((head_owner << 32) | k);
        if (it == pages.end()) break;
        if (it->second.pins > 0) throw StateError("discard_suffix would drop pinned nodes");
        doomed.push_back(it->first);
      }
    } else {
      // shared head: every page deeper than it, shared or private
      for (auto& kv : pages) {
        if ((kv.first & 0xffffffffULL) < fp) continue;
        if (kv.second.pins > 0) throw StateError("discard_suffix would drop pinned nodes");
        doomed.push_back(kv.first);
      }
    }
    for (std::uint64_t k : doomed) drop_page(pages.find(k));
    discarded += doomed.size() * ps;
  }

  std::uint64_t digest() const {  // O(1): dsum is maintained incrementally
    std::uint64_t h = kvdigest::fold(0x1234, dsum);
    h = kvdigest::fold(h, used);
    h = kvdigest::fold(h, clock);
    h = kvdigest::fold(h, kvdigest::dbits(hit_m));
    h = kvdigest::fold(h, kvdigest::dbits(hit_r));
    h = kvdigest::fold(h, discarded);
    h = kvdigest::fold(h, offloaded);
    return h;
  }
};

/* ======================= controller (controller.cpp) ======================== */

struct Ctl {
  std::uint32_t kind = KVG_POLICY_UNCONTROLLED, cap = 1, total = 0;
  kvg_controller_config cfg{};
  double window = 1.0, su = 0, sh = 0;
  bool have_smoothed = false;
  std::vector<std::uint32_t> active;
  std::deque<std::uint32_t> pending, paused;
  std::uint64_t ticks = 0;

  void init(const kvg_policy& p, std::uint32_t n) {  // controller.cpp:55-65
    kind = p.kind;
    cap = p.cap;
    cfg = p.aimd;
    total = n;
    if (kind == KVG_POLICY_AIMD) {
      if (cfg.w_max == 0) cfg.w_max = std::max(cfg.w_min, static_cast<double>(n));
      if (cfg.initial_window == 0) cfg.initial_window = cfg.w_min;
      window = cfg.initial_window;
    }
  }
  bool agent_gated() const { return kind == KVG_POLICY_AGENT_CAP || kind == KVG_POLICY_AIMD; }
  /* update_window, controller.cpp:67-91 */
  void update(double usage, double hit) {
    ++ticks;
    if (kind != KVG_POLICY_AIMD) return;
    double u = usage, h = hit;
    if (cfg.signal_smoothing > 0) {
      if (have_smoothed) {
        u = cfg.signal_smoothing * su + (1 - cfg.signal_smoothing) * usage;
        h = cfg.signal_smoothing * sh + (1 - cfg.signal_smoothing) * hit;
      }
      su = u;
      sh = h;
      have_smoothed = true;
    }
    double w = window;
    if (u < cfg.u_low)
      w = w + cfg.alpha;
    else if (u > cfg.u_high && h < cfg.h_thresh)
      w = w * cfg.beta;
    window = w < cfg.w_min ? cfg.w_min : (cfg.w_max < w ? cfg.w_max : w);
  }
  std::uint64_t limit() const {  // controller.cpp:93-104
    switch (kind) {
      case KVG_POLICY_UNCONTROLLED: return std::numeric_limits<std::uint64_t>::max();
      case KVG_POLICY_AIMD: return static_cast<std::uint64_t>(std::floor(window));
      default: return cap;
    }
  }
  double display() const {  // controller.cpp:106-117
    switch (kind) {
      case KVG_POLICY_UNCONTROLLED: return static_cast<double>(total);
      case KVG_POLICY_AIMD: return window;
      default: return static_cast<double>(cap);
    }
  }
  void remove_active(std::uint32_t id, const char* what) {
    auto it = std::find(active.begin(), active.end(), id);
    if (it == active.end()) throw StateError(what);
    active.erase(it);
  }
  std::uint64_t digest() const {
    std::uint64_t h = 0x5678;
    for (auto id : active) h = kvdigest::fold(h, id);
    h = kvdigest::fold(h, 0xAAAA);
    for (auto id : pending) h = kvdigest::fold(h, id);
    h = kvdigest::fold(h, 0xBBBB);
    for (auto id : paused) h = kvdigest::fold(h, id);
    h = kvdigest::fold(h, kvdigest::dbits(window));
    h = kvdigest::fold(h, ticks);
    return h;
  }
};

/* ======================= engine (engine.cpp) ================================ */

enum : std::uint8_t { S_PENDING, S_AWAIT, S_GEN, S_TOOL, S_PAUSED, S_DONE };
enum : std::uint8_t { EV_GEN = 0, EV_TOOL = 1, EV_XFER = 2 };

/* lifecycle_edge, workload.cpp:110-128 */
bool legal(std::uint8_t from, std::uint8_t to) {
  switch (from) {
    case S_PENDING: return to == S_AWAIT;
    case S_AWAIT: return to == S_GEN || to == S_PAUSED;
    case S_GEN: return to == S_TOOL || to == S_DONE || to == S_AWAIT;
    case S_TOOL: return to == S_AWAIT;
    case S_PAUSED: return to == S_AWAIT;
    default: return false;
  }
}

struct AgentRec {
  std::uint8_t state = S_PENDING;
  std::uint32_t step = 0;
  std::uint64_t ctx = 0, high_water = 0, pinned = 0;
  double ready_since = 0;
  std::uint64_t f_gen = 0, f_rec = 0, f_obs = 0;
  double f_tool = 0;
  bool f_has_tool = false;
  kvg_agent_stats st{};
};

struct Sim {
  const kvg_sim_desc* d;
  const kvg_step_plan* plans;
  std::uint32_t n = 0, steps = 0;
  FlatCache cache;
  Ctl ctl;
  std::vector<AgentRec> ag;
  std::set<std::tuple<double, std::uint64_t, std::uint32_t>> agent_q;  // rank 0
  std::vector<std::uint8_t> ev_kind;
  std::uint64_t ord = 0;
  bool tick_on = false, adm_on = false;
  double tick_t = 0, adm_t = 0;
  std::uint64_t tick_o = 0, adm_o = 0;
  double clock = 0, gpu_busy = 0, makespan = 0;
  std::uint32_t finished = 0;
  std::uint64_t decoded_cum = 0, rec_cum = 0, lookups = 0, agent_steps = 0;
  std::uint64_t events = 0;
  kvg_ledger ledger{};
  double device_busy = 0;
  std::vector<kvg_trace_row> trace;
  std::vector<std::uint64_t>* digests = nullptr;
  std::vector<kvg_log_record>* log = nullptr;

  void logrec(std::uint32_t kind, std::uint32_t agent, std::uint64_t a, std::uint64_t b) {
    if (log) log->push_back(kvg_log_record{kind, agent, cache.clock, a, b});
  }
  void set_state(std::uint32_t id, std::uint8_t s) {  // workload.cpp:130-137
    if (!legal(ag[id].state, s)) throw StateError("illegal lifecycle transition");
    ag[id].state = s;
  }
  double interval() const { return d->policy.aimd.control_interval; }
  /* cost_model.cpp:28-41 */
  double prefill(std::uint64_t nt, std::uint64_t c) const {
    double x = static_cast<double>(nt), y = static_cast<double>(c);
    return d->cost.prefill_linear * x + d->cost.prefill_quadratic * x * y;
  }
  double decode(std::uint64_t nt, std::uint64_t c) const {
    double x = static_cast<double>(nt), y = static_cast<double>(c);
    return d->cost.decode_base * x + d->cost.decode_context * (x * y + x * (x - 1.0) / 2.0);
  }
  void schedule_agent(double t, std::uint8_t kind, std::uint32_t id) {  // engine.cpp:143-145
    agent_q.emplace(t, ord++, id);
    ev_kind[id] = kind;
  }
  void schedule_admission() {  // engine.cpp:149-154
    if (adm_on && adm_t == clock) return;
    if (adm_on) throw StateError("two admission checks outstanding");
    adm_on = true;
    adm_t = clock;
    adm_o = ord++;
  }

  void init(const kvg_sim_desc* desc) {
    d = desc;
    const kvg_population* pop = d->population;
    n = pop->agents;
    steps = pop->steps;
    plans = pop->plans;
    cache.init(d->engine.capacity, d->engine.page_size, pop->prompt_tokens,
               pop->shared_prompt != 0);
    ctl.init(d->policy, n);
    ag.assign(n, AgentRec{});
    ev_kind.assign(n, 0);
    for (std::uint32_t i = 0; i < n; ++i) {
      ag[i].ctx = pop->prompt_tokens;
      ctl.pending.push_back(i);  // engine.cpp:89-93
      ag[i].st.finish_time = -1.0;
    }
  }

  /* engine.cpp:337-396 */
  bool dispatch_member(std::uint32_t id, double* t_out, double* ft, double* rt, double* dt) {
    AgentRec& a = ag[id];
    const std::uint64_t ctx = a.ctx;
    const std::uint64_t matched = cache.match(id, ctx);
    {
      std::uint64_t r = matched / cache.ps;
      lookups += r + (r < ctx / cache.ps ? 1 : 0);
    }
    logrec(KVG_LOG_MATCH, id, matched, 0);
    cache.pin(id, matched, +1);
    if (a.pinned > 0) cache.pin(id, a.pinned, -1);
    a.pinned = matched;
    const kvg_step_plan& plan = plans[std::size_t(id) * steps + a.step];
    a.ctx += plan.gen_tokens;  // append_tokens
    std::uint64_t inserted = 0;
    cache.log = log;
    cache.log_agent = id;
    bool ok = cache.insert(id, a.ctx, &inserted, nullptr);
    cache.log = nullptr;
    logrec(KVG_LOG_INSERT, id, ok ? 1 : 0, ok ? a.ctx / cache.ps * cache.ps : 0);
    if (!ok) {
      a.ctx = ctx;
      cache.pin(id, matched, -1);
      a.pinned = 0;
      ++a.st.stall_events;
      return false;
    }
    const std::uint64_t stored = a.ctx - a.ctx % cache.ps;
    cache.pin(id, stored, +1);
    cache.pin(id, matched, -1);
    a.pinned = stored;
    const std::uint64_t missing = ctx - matched;
    const std::uint64_t rec = a.high_water > matched ? a.high_water - matched : 0;
    const std::uint64_t fresh = missing - rec;
    a.high_water = stored;
    *ft = prefill(fresh, ctx);
    *rt = prefill(rec, ctx);
    *dt = decode(plan.gen_tokens, ctx);
    *t_out = *ft + *rt + *dt;
    a.f_gen = plan.gen_tokens;
    a.f_rec = rec;
    a.f_has_tool = plan.has_tool != 0;
    a.f_obs = plan.obs_tokens;
    a.f_tool = plan.tool_latency;
    a.st.wait_time += clock - a.ready_since;
    set_state(id, S_GEN);
    ++agent_steps;
    return true;
  }

  /* engine.cpp:305-333 */
  void dispatch_batch() {
    std::vector<std::uint32_t> ready;
    for (std::uint32_t id : ctl.active)
      if (ag[id].state == S_AWAIT) ready.push_back(id);
    std::sort(ready.begin(), ready.end());
    struct M { std::uint32_t id; double t, f, r, dd; };
    std::vector<M> batch;
    for (std::uint32_t id : ready) {
      M m{id, 0, 0, 0, 0};
      if (dispatch_member(id, &m.t, &m.f, &m.r, &m.dd)) batch.push_back(m);
    }
    if (batch.empty()) return;
    double wall = 0.0, total = 0.0;
    for (const M& m : batch) {
      wall = wall < m.t ? m.t : wall;
      total += m.t;
    }
    double start = clock < gpu_busy ? gpu_busy : clock;
    gpu_busy = start + wall;
    device_busy += wall;
    double share = total > 0 ? wall / total : 0.0;
    for (const M& m : batch) {
      ledger.prefill_fresh += share * m.f;
      ledger.prefill_recompute += share * m.r;
      ledger.decode += share * m.dd;
      schedule_agent(start + wall, EV_GEN, m.id);
    }
  }

  /* controller.cpp:124-160 + engine.cpp:268-291 */
  void on_admission() {
    adm_on = false;
    std::uint64_t lim = ctl.limit();
    struct Cmd { int kind; std::uint32_t id; };  // 0 admit 1 pause 2 resume
    std::vector<Cmd> cmds;
    if (ctl.agent_gated()) {
      while (ctl.active.size() > lim) {
        long victim = -1;
        for (long i = long(ctl.active.size()) - 1; i >= 0; --i)
          if (ag[ctl.active[i]].state == S_AWAIT) { victim = i; break; }
        if (victim < 0) break;
        std::uint32_t id = ctl.active[victim];
        ctl.active.erase(ctl.active.begin() + victim);
        ctl.paused.push_back(id);
        cmds.push_back({1, id});
      }
    }
    while (ctl.active.size() < lim) {
      if (ctl.agent_gated() && !ctl.paused.empty()) {
        std::uint32_t id = ctl.paused.front();
        ctl.paused.pop_front();
        ctl.active.push_back(id);
        cmds.push_back({2, id});
      } else if (!ctl.pending.empty()) {
        std::uint32_t id = ctl.pending.front();
        ctl.pending.pop_front();
        ctl.active.push_back(id);
        cmds.push_back({0, id});
      } else {
        break;
      }
    }
    for (const Cmd& c : cmds) {
      if (c.kind == 1) {
        set_state(c.id, S_PAUSED);
        ++ag[c.id].st.pause_events;
      } else if (c.kind == 0) {
        if (ag[c.id].state == S_PENDING) set_state(c.id, S_AWAIT);
      } else {
        set_state(c.id, S_AWAIT);
      }
    }
    dispatch_batch();
  }

  /* engine.cpp:184-222 */
  void on_generation_complete(std::uint32_t id) {
    AgentRec& a = ag[id];
    makespan = makespan < clock ? clock : makespan;
    if (a.pinned > 0) {
      cache.pin(id, a.pinned, -1);
      a.pinned = 0;
    }
    decoded_cum += a.f_gen;
    rec_cum += a.f_rec;
    a.st.generated_tokens += a.f_gen;
    a.st.recompute_tokens += a.f_rec;
    if (a.f_rec > 0) ++a.st.recompute_events;
    ++a.step;
    const bool req = ctl.kind == KVG_POLICY_REQUEST_CAP;
    if (a.step >= steps) {
      set_state(id, S_DONE);
      const std::uint64_t before = cache.used;
      cache.discard_suffix(id, a.ctx, d->population->shared_prompt_tokens);
      logrec(KVG_LOG_DISCARD, id, 0, before - cache.used);
      if (req)
        ctl.remove_active(id, "request completion for inactive agent");
      else
        ctl.remove_active(id, "finished agent is not active");
      ++finished;
      a.st.finish_time = clock;
      a.st.finish_ordinal = events;
      std::uint64_t tb;
      std::memcpy(&tb, &clock, 8);
      logrec(KVG_LOG_FINISH, id, tb, events);
    } else if (a.f_has_tool) {
      set_state(id, S_TOOL);
      ledger.tool_wait += a.f_tool;
      if (req) ctl.remove_active(id, "request completion for inactive agent");
      schedule_agent(clock + a.f_tool, EV_TOOL, id);
    } else {
      set_state(id, S_AWAIT);
      a.ready_since = clock;
      if (req) {
        ctl.remove_active(id, "request completion for inactive agent");
        ctl.pending.push_back(id);
      }
    }
    schedule_admission();
  }

  /* engine.cpp:224-235 */
  void on_tool_complete(std::uint32_t id) {
    AgentRec& a = ag[id];
    makespan = makespan < clock ? clock : makespan;
    a.ctx += a.f_obs;
    a.f_obs = 0;
    a.f_has_tool = false;
    set_state(id, S_AWAIT);
    a.ready_since = clock;
    if (ctl.kind == KVG_POLICY_REQUEST_CAP) {
      ctl.pending.push_back(id);
    } else if (std::find(ctl.active.begin(), ctl.active.end(), id) == ctl.active.end()) {
      throw StateError("tool return for inactive agent");
    }
    schedule_admission();
  }

  /* engine.cpp:245-266 */
  void on_tick() {
    const double usage = static_cast<double>(cache.used) / static_cast<double>(cache.capacity);
    const double m = cache.hit_m, r = cache.hit_r;
    const double hit = r > 0 ? m / r : 1.0;
    ctl.update(usage, hit);
    kvg_trace_row row{clock, usage, hit, ctl.display(),
                      ctl.active.size(), ctl.pending.size() + ctl.paused.size(),
                      decoded_cum, rec_cum, 0, m, r};
    trace.push_back(row);
    cache.hit_m *= d->engine.hit_window_decay;
    cache.hit_r *= d->engine.hit_window_decay;
    tick_on = true;
    tick_t = clock + interval();
    tick_o = ord++;
    schedule_admission();
  }

  /* engine.cpp:98-136 */
  int run() {
    adm_on = true;  // schedule(0.0, admission): ordinal 0
    adm_t = 0.0;
    adm_o = ord++;
    tick_on = true;  // schedule(interval, tick): ordinal 1
    tick_t = interval();
    tick_o = ord++;
    for (;;) {
      // pop the minimum (time, rank, ordinal)
      int which = -1;  // 0 agent, 1 tick, 2 admission
      double bt = 0;
      std::uint64_t bo = 0;
      if (!agent_q.empty()) {
        which = 0;
        bt = std::get<0>(*agent_q.begin());
        bo = std::get<1>(*agent_q.begin());
      }
      auto better = [&](double t, int rank, std::uint64_t o) {
        if (which < 0) return true;
        if (t != bt) return t < bt;
        if (rank != which) return rank < which;
        return o < bo;
      };
      if (tick_on && better(tick_t, 1, tick_o)) { which = 1; bt = tick_t; bo = tick_o; }
      if (adm_on && better(adm_t, 2, adm_o)) { which = 2; bt = adm_t; bo = adm_o; }
      if (which < 0) break;
      std::uint32_t agent = 0;
      if (which == 0) {
        agent = std::get<2>(*agent_q.begin());
        agent_q.erase(agent_q.begin());
      } else if (which == 1) {
        tick_on = false;
      } else {
        adm_on = false;
      }
      if (which != 0 && finished == n) continue;  // housekeeping after the end
      if (bt > d->engine.horizon) return KVG_ERR_HORIZON;
      clock = bt;
      if (which == 0) {
        switch (ev_kind[agent]) {
          case EV_GEN: on_generation_complete(agent); break;
          case EV_TOOL: on_tool_complete(agent); break;
          default: throw StateError("transfer event in discard mode");
        }
      } else if (which == 1) {
        on_tick();
      } else {
        on_admission();
      }
      ++events;
      if (digests) digests->push_back(kvdigest::fold(cache.digest(), ctl.digest()));
    }
    if (finished != n) throw StateError("event queue drained with unfinished agents");
    return KVG_OK;
  }

  void fill(kvg_sim_result* res, int status) const {  // engine.cpp:398-415
    std::memset(res, 0, sizeof *res);
    res->status = status;
    res->ledger = ledger;
    res->makespan = makespan;  // no link in discard mode: max(makespan, 0)
    res->device_busy = device_busy;
    res->link_busy = 0;
    res->decoded_tokens = decoded_cum;
    res->recompute_tokens = rec_cum;
    double wait = 0;
    for (const AgentRec& a : ag) {
      res->recompute_events += a.st.recompute_events;
      res->stall_events += a.st.stall_events;
      wait += a.st.wait_time;
    }
    res->total_wait_time = wait;
    res->discarded_tokens = cache.discarded;
    res->offloaded_tokens = cache.offloaded;
    res->ticks = trace.size();
    res->workload_hash = d->population->stream_hash;
    res->agent_steps = agent_steps;
    res->lookups = lookups;
    res->events = events;
    res->evict_calls = cache.evict_calls;
    res->evicted_pages = cache.evicted;
    res->cache_clock = cache.clock;
    res->pool_used = cache.used;
    res->hit_matched = cache.hit_m;
    res->hit_requested = cache.hit_r;
    classify(res);
  }

  /* classify_phases, metrics.cpp:41-81 (called from finish_result, engine.cpp:413) */
  void classify(kvg_sim_result* res) const {
    const kvg_phase_params& pp = d->engine.phases;
    const double mk = res->makespan;
    res->n_phases = 0;
    if (mk <= 0) return;
    auto hot = [&](const kvg_trace_row& r) {
      return r.usage >= pp.sat_threshold && r.hit_rate < pp.hit_threshold;
    };
    auto push = [&](std::uint32_t ph, double a, double b) {
      res->phases[res->n_phases++] = kvg_phase_label{ph, 0, a, b};
    };
    std::size_t enter = trace.size();
    for (std::size_t i = 0; i < trace.size(); ++i)
      if (hot(trace[i])) { enter = i; break; }
    if (enter == trace.size()) {
      push(KVG_PHASE_WARMUP, 0.0, mk);
      return;
    }
    const double ms = trace[enter].time;
    double me = mk;
    int bad = 0;
    for (std::size_t i = enter + 1; i < trace.size(); ++i) {
      if (hot(trace[i])) { bad = 0; continue; }
      if (++bad >= pp.hysteresis) {
        me = trace[i + 1 - static_cast<std::size_t>(pp.hysteresis)].time;
        break;
      }
    }
    if (ms > 0) push(KVG_PHASE_WARMUP, 0.0, ms);
    push(KVG_PHASE_MIDDLE, ms, me);
    if (me < mk) push(KVG_PHASE_COOLDOWN, me, mk);
  }
};

}  // namespace

KVO_API const char* kvo_last_error(void) { return t_err.c_str(); }

/* Runs one simulation on the CPU. Buffers may be NULL; counts are always
 * reported so a caller can size and retry. */
KVO_API int kvo_run(const kvg_sim_desc* d, kvg_sim_result* res, kvg_trace_row* trace,
                    size_t trace_cap, size_t* n_trace, kvg_agent_stats* agents,
                    size_t agents_cap, uint64_t* digests, size_t digest_cap,
                    size_t* n_digests, kvg_log_record* log, size_t log_cap,
                    size_t* n_log) {
  if (d->engine.eviction == KVG_EVICT_OFFLOAD) {
    t_err = "oracle restatement covers discard-mode eviction only";
    return KVG_ERR_CONFIG;
  }
  Sim sim;
  std::vector<std::uint64_t> dig;
  std::vector<kvg_log_record> lg;
  if (digests) sim.digests = &dig;
  if (log) sim.log = &lg;
  int status;
  try {
    sim.init(d);
    status = sim.run();
  } catch (const std::exception& e) {
    t_err = e.what();
    return KVG_ERR_STATE;
  }
  sim.fill(res, status);
  if (n_trace) *n_trace = sim.trace.size();
  if (trace)
    std::memcpy(trace, sim.trace.data(),
                std::min(trace_cap, sim.trace.size()) * sizeof(kvg_trace_row));
  if (agents)
    for (std::size_t i = 0; i < sim.n && i < agents_cap; ++i) agents[i] = sim.ag[i].st;
  if (n_digests) *n_digests = dig.size();
  if (digests)
    std::memcpy(digests, dig.data(), std::min(digest_cap, dig.size()) * sizeof(std::uint64_t));
  if (n_log) *n_log = lg.size();
  if (log)
    std::memcpy(log, lg.data(), std::min(log_cap, lg.size()) * sizeof(kvg_log_record));
  return status;
}

/* ----------------------- cache-level differential surface ------------------- */

KVO_API void* kvo_cache_new(uint64_t capacity, uint64_t page_size, uint32_t eviction,
                            uint64_t prompt_tokens, uint32_t shared) {
  if (eviction != KVG_EVICT_DISCARD) return nullptr;
  try {
    auto* c = new FlatCache();
    c->init(capacity, page_size, prompt_tokens, shared != 0);
    return c;
  } catch (const std::exception& e) {
    t_err = e.what();
    return nullptr;
  }
}

KVO_API void kvo_cache_free(void* h) { delete static_cast<FlatCache*>(h); }

KVO_API int kvo_cache_op(void* h, const kvg_cache_op* op, kvg_cache_op_result* r,
                         kvg_victim* victims, size_t cap, size_t* n_victims) {
  FlatCache* c = static_cast<FlatCache*>(h);
  std::vector<std::pair<std::uint64_t, std::uint64_t>> v;
  c->victims = &v;
  std::memset(r, 0, sizeof *r);
  int rc = KVG_OK;
  try {
    switch (op->kind) {
      case KVG_OP_MATCH: r->r0 = c->match(op->agent, op->len); break;
      case KVG_OP_INSERT: {
        std::uint64_t ins = 0;
        r->r0 = c->insert(op->agent, op->len, &ins, nullptr) ? 1 : 0;
        r->r1 = ins;
        break;
      }
      case KVG_OP_EVICT: r->r0 = c->evict(op->arg); break;
      case KVG_OP_PIN: c->pin(op->agent, op->arg, +1); break;
      case KVG_OP_UNPIN: c->pin(op->agent, op->arg, -1); break;
      case KVG_OP_DISCARD: c->discard_suffix(op->agent, op->len, op->arg); break;
      default: throw std::invalid_argument("unknown op");
    }
  } catch (const std::exception& e) {
    t_err = e.what();
    rc = KVG_ERR_STATE;
  }
  c->victims = nullptr;
  r->status = rc;
  r->clock = c->clock;
  r->used = c->used;
  if (n_victims) *n_victims = v.size();
  for (std::size_t i = 0; i < v.size() && i < cap && victims; ++i)
    victims[i] = kvg_victim{v[i].first, v[i].second};
  return rc;
}

KVO_API void kvo_cache_stats(void* h, double* m, double* r, uint64_t* discarded) {
  FlatCache* c = static_cast<FlatCache*>(h);
  if (m) *m = c->hit_m;
  if (r) *r = c->hit_r;
  if (discarded) *discarded = c->discarded;
}

KVO_API uint64_t kvo_cache_digest(void* h) { return static_cast<FlatCache*>(h)->digest(); }
