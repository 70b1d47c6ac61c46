/* Reference harness — TEST INFRASTRUCTURE ONLY (also the bench's CPU arm).
 *
 * Links the UNMODIFIED reference sources from /root/reference/proj/src
 * (compiled by oracle/Makefile into oracle/_ref/libkvref.so) and exposes a
 * small C surface over the reference's own hot-path entry points:
 *   - kvadmit::build_population   (workload.cpp:153-204)
 *   - kvadmit::run_simulation     (engine.cpp:446-456)
 *   - kvadmit::CacheTree methods  (cache_tree.cpp:114-437)
 * plus a per-event state digest taken through the paranoid-mode invariant
 * hooks (engine.cpp:128-131), intercepted with ld --wrap (see Makefile).
 * Only tests/, __graft_entry__.smoke() and bench.py's reference arm load it.
 */
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "cache_tree.hpp"
#include "controller.hpp"
#include "cost_model.hpp"
#include "engine.hpp"
#include "workload.hpp"

#include "../include/kvgpu.h"
#include "digest.h"

#define KVR_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string t_err = "no error";

int fail_with(int code, const std::string& what) {
  t_err = what;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return KVG_OK;
  } catch (const kvadmit::HorizonError& e) {
    return fail_with(KVG_ERR_HORIZON, e.what());
  } catch (const kvadmit::ConfigError& e) {
    return fail_with(KVG_ERR_CONFIG, e.what());
  } catch (const std::exception& e) {
    return fail_with(KVG_ERR_STATE, e.what());
  }
}

kvadmit::Distribution to_dist(const kvg_distribution& d) {
  kvadmit::Distribution o;
  o.kind = d.kind == KVG_DIST_UNIFORM     ? kvadmit::Distribution::Kind::kUniform
           : d.kind == KVG_DIST_LOGNORMAL ? kvadmit::Distribution::Kind::kLogNormal
                                          : kvadmit::Distribution::Kind::kConstant;
  o.a = d.a;
  o.b = d.b;
  return o;
}

kvadmit::WorkloadConfig to_workload(const kvg_workload_config& w) {
  kvadmit::WorkloadConfig c;
  c.agents = w.agents;
  c.shared_prompt = w.shared_prompt != 0;
  c.prompt_tokens = w.prompt_tokens;
  c.steps = w.steps;
  c.gen_tokens = to_dist(w.gen_tokens);
  c.obs_tokens = to_dist(w.obs_tokens);
  c.tool_latency = to_dist(w.tool_latency);
  c.tool_probability = w.tool_probability;
  return c;
}

kvadmit::Policy to_policy(const kvg_policy& p) {
  kvadmit::Policy o;
  switch (p.kind) {
    case KVG_POLICY_REQUEST_CAP: o.kind = kvadmit::PolicyKind::kFixedRequestCap; break;
    case KVG_POLICY_AGENT_CAP: o.kind = kvadmit::PolicyKind::kFixedAgentCap; break;
    case KVG_POLICY_AIMD: o.kind = kvadmit::PolicyKind::kCacheAwareAimd; break;
    default: o.kind = kvadmit::PolicyKind::kUncontrolled; break;
  }
  o.cap = p.cap;
  o.aimd.alpha = p.aimd.alpha;
  o.aimd.beta = p.aimd.beta;
  o.aimd.u_low = p.aimd.u_low;
  o.aimd.u_high = p.aimd.u_high;
  o.aimd.h_thresh = p.aimd.h_thresh;
  o.aimd.w_min = p.aimd.w_min;
  o.aimd.w_max = p.aimd.w_max;
  o.aimd.initial_window = p.aimd.initial_window;
  o.aimd.control_interval = p.aimd.control_interval;
  o.aimd.signal_smoothing = p.aimd.signal_smoothing;
  return o;
}

kvadmit::CostParams to_cost(const kvg_cost_params& c) {
  kvadmit::CostParams o;
  o.prefill_linear = c.prefill_linear;
  o.prefill_quadratic = c.prefill_quadratic;
  o.decode_base = c.decode_base;
  o.decode_context = c.decode_context;
  o.bytes_per_token = c.bytes_per_token;
  o.pcie_bandwidth = c.pcie_bandwidth;
  o.transfer_sync_overhead = c.transfer_sync_overhead;
  return o;
}

kvadmit::EngineParams to_engine(const kvg_engine_params& e) {
  kvadmit::EngineParams o;
  o.capacity = e.capacity;
  o.page_size = e.page_size;
  o.eviction = e.eviction == KVG_EVICT_OFFLOAD ? kvadmit::EvictionMode::kOffload
                                               : kvadmit::EvictionMode::kDiscard;
  o.hit_window_decay = e.hit_window_decay;
  o.horizon = e.horizon;
  o.phase_params.sat_threshold = e.phases.sat_threshold;
  o.phase_params.hit_threshold = e.phases.hit_threshold;
  o.phase_params.hysteresis = e.phases.hysteresis;
  o.paranoid = e.paranoid != 0;
  return o;
}

/* ---------------- per-event digest through the paranoid hooks ------------- */

struct DigestSink {
  std::vector<std::uint64_t>* out = nullptr;
  std::uint64_t pending_cache = 0;
  std::uint64_t page_size = 1;
  std::uint64_t q1_states = 0;   // events that ended in a Q1 state
  std::uint64_t cwd_states = 0;  // events that ended with a corrupted counter
};
thread_local DigestSink t_sink;

/* Owner of a page from its last token: ids below 2^32 are shared-prompt ids
 * (workload.cpp:167-171), others carry (agent+1) in the high half. */
std::uint64_t owner_of(kvadmit::TokenId t) { return t >> 32; }

std::uint64_t cache_digest(const kvadmit::CacheTree& tree) {
  const std::uint64_t ps = tree.page_size();
  std::uint64_t sum = 0;
  std::vector<kvadmit::TokenId> path;
  std::function<void(const kvadmit::CacheNode*)> walk =
      [&](const kvadmit::CacheNode* n) {
        for (const auto& [key, child] : n->children) {
          const kvadmit::CacheNode* c = child.get();
          std::size_t base = path.size();
          path.insert(path.end(), c->segment.begin(), c->segment.end());
          // pages fully covered by this node (device nodes are page aligned)
          std::size_t first = (base + ps - 1) / ps;
          std::size_t last = path.size() / ps;  // exclusive
          for (std::size_t pg = first; pg < last; ++pg) {
            kvadmit::TokenId tail = path[(pg + 1) * ps - 1];
            sum += kvdigest::page_term(owner_of(tail), pg, c->last_access,
                                       static_cast<std::uint64_t>(c->pin_count),
                                       c->tier == kvadmit::Tier::kHost ? 1 : 0);
          }
          walk(c);
          path.resize(base);
        }
      };
  walk(tree.root());
  std::uint64_t h = kvdigest::fold(0x1234, sum);
  h = kvdigest::fold(h, tree.pool().used);
  h = kvdigest::fold(h, tree.clock());
  h = kvdigest::fold(h, kvdigest::dbits(tree.hit_window_matched()));
  h = kvdigest::fold(h, kvdigest::dbits(tree.hit_window_requested()));
  h = kvdigest::fold(h, tree.total_discarded_tokens());
  h = kvdigest::fold(h, tree.total_offloaded_tokens());
  return h;
}

std::uint64_t controller_digest(const kvadmit::Controller& c) {
  std::uint64_t h = 0x5678;
  for (kvadmit::AgentId id : c.active()) h = kvdigest::fold(h, id);
  h = kvdigest::fold(h, 0xAAAA);
  for (kvadmit::AgentId id : c.pending()) h = kvdigest::fold(h, id);
  h = kvdigest::fold(h, 0xBBBB);
  for (kvadmit::AgentId id : c.paused()) h = kvdigest::fold(h, id);
  h = kvdigest::fold(h, kvdigest::dbits(c.window()));
  h = kvdigest::fold(h, c.tick_count());
  return h;
}

}  // namespace

extern "C" {
void __real__ZNK7kvadmit9CacheTree16check_invariantsEv(const kvadmit::CacheTree*);
void __real__ZNK7kvadmit10Controller16check_invariantsEv(const kvadmit::Controller*);

__attribute__((visibility("hidden"))) void
__wrap__ZNK7kvadmit9CacheTree16check_invariantsEv(const kvadmit::CacheTree* t) {
  // Quirk Q1: an offload-mode reload can leave a device node
  // below a host node, which check_invariants rejects. A production
  // (non-paranoid) run carries on with that state, so the digest harness
  // does too: that one violation is counted, never thrown.
  try {
    __real__ZNK7kvadmit9CacheTree16check_invariantsEv(t);
  } catch (const kvadmit::InvariantViolation& e) {
    // ... and the children_with_device over-count Q1 leads to: re-promoting a
    // host node whose subtree already holds device slots calls
    // propagate_gain a second time (cache_tree.cpp:94-102, 357-361)
    const std::string w = e.what();
    if (w.find("device node below a host node") != std::string::npos) ++t_sink.q1_states;
    else if (w.find("children_with_device mismatch") != std::string::npos) ++t_sink.cwd_states;
    else throw;
  }
  if (t_sink.out != nullptr) t_sink.pending_cache = cache_digest(*t);
}

__attribute__((visibility("hidden"))) void
__wrap__ZNK7kvadmit10Controller16check_invariantsEv(const kvadmit::Controller* c) {
  __real__ZNK7kvadmit10Controller16check_invariantsEv(c);
  if (t_sink.out != nullptr)
    t_sink.out->push_back(kvdigest::fold(t_sink.pending_cache, controller_digest(*c)));
}
}

/* ------------------------------------------------------------------------ */

KVR_API const char* kvr_last_error(void) { return t_err.c_str(); }

/* Events of this thread's last kvr_run (with digests) that ended in a Q1
 * state: device node below a host node. */
KVR_API uint64_t kvr_last_q1_states(void) { return t_sink.q1_states; }
KVR_API uint64_t kvr_last_cwd_states(void) { return t_sink.cwd_states; }

KVR_API int kvr_build_population(const kvg_workload_config* cfg, uint64_t seed,
                                 kvg_step_plan* plans, size_t cap,
                                 uint64_t* stream_hash,
                                 uint64_t* shared_prompt_tokens,
                                 uint64_t* peak_aggregate_tokens) {
  return guarded([&] {
    kvadmit::Population pop = kvadmit::build_population(to_workload(*cfg), seed);
    size_t k = 0;
    for (const auto& a : pop.agents) {
      for (const auto& s : a.spec.steps) {
        if (k < cap && plans != nullptr) {
          plans[k].gen_tokens = s.gen_tokens;
          plans[k].obs_tokens = s.obs_tokens;
          plans[k].tool_latency = s.tool_latency;
          plans[k].has_tool = s.has_tool ? 1u : 0u;
          plans[k]._pad = 0;
        }
        ++k;
      }
    }
    if (stream_hash) *stream_hash = pop.stream_hash;
    if (shared_prompt_tokens) *shared_prompt_tokens = pop.shared_prompt_tokens;
    if (peak_aggregate_tokens) *peak_aggregate_tokens = pop.peak_aggregate_tokens;
  });
}

namespace {

void fill_result(const kvadmit::SimulationResult& r, int status,
                 kvg_sim_result* res, kvg_trace_row* trace, size_t trace_cap,
                 size_t* n_trace, kvg_agent_stats* agents, size_t agents_cap) {
  std::memset(res, 0, sizeof *res);
  res->status = status;
  res->ledger.prefill_fresh = r.ledger.prefill_fresh;
  res->ledger.prefill_recompute = r.ledger.prefill_recompute;
  res->ledger.decode = r.ledger.decode;
  res->ledger.transfer = r.ledger.transfer;
  res->ledger.tool_wait = r.ledger.tool_wait;
  res->makespan = r.makespan;
  res->device_busy = r.device_busy;
  res->link_busy = r.link_busy;
  res->decoded_tokens = r.decoded_tokens;
  res->recompute_tokens = r.recompute_tokens;
  res->recompute_events = r.recompute_events;
  res->stall_events = r.stall_events;
  res->offloaded_tokens = r.offloaded_tokens;
  res->reloaded_tokens = r.reloaded_tokens;
  res->discarded_tokens = r.discarded_tokens;
  res->total_wait_time = r.total_wait_time;
  res->ticks = r.ticks;
  res->workload_hash = r.workload_hash;
  res->n_phases = static_cast<uint32_t>(std::min<size_t>(r.phases.size(), 3));
  for (uint32_t i = 0; i < res->n_phases; ++i) {
    res->phases[i].phase = static_cast<uint32_t>(r.phases[i].phase);
    res->phases[i].start = r.phases[i].start;
    res->phases[i].end = r.phases[i].end;
  }
  if (n_trace) *n_trace = r.trace.size();
  for (size_t i = 0; i < r.trace.size() && i < trace_cap && trace; ++i) {
    const auto& t = r.trace[i];
    trace[i] = kvg_trace_row{t.time, t.usage, t.hit_rate, t.window, t.active,
                             t.pending, t.decoded_cum, t.recompute_cum,
                             t.transfers, r.tick_hits[i].matched,
                             r.tick_hits[i].requested};
  }
  for (size_t i = 0; i < r.agent_stats.size() && i < agents_cap && agents; ++i) {
    const auto& s = r.agent_stats[i];
    agents[i] = kvg_agent_stats{s.generated_tokens, s.recompute_tokens,
                                s.recompute_events, s.stall_events,
                                s.pause_events, s.wait_time, 0.0, 0};
  }
}

}  // namespace

/* One reference run_simulation. digests != NULL turns on paranoid mode and
 * records one state digest per processed event. wall_s receives the
 * steady_clock time spent inside run_simulation only. */
KVR_API int kvr_run(const kvg_workload_config* wl, uint64_t seed,
                    const kvg_policy* policy, const kvg_cost_params* cost,
                    const kvg_engine_params* engine, kvg_sim_result* res,
                    kvg_trace_row* trace, size_t trace_cap, size_t* n_trace,
                    kvg_agent_stats* agents, size_t agents_cap,
                    uint64_t* digests, size_t digest_cap, size_t* n_digests,
                    double* wall_s) {
  std::vector<std::uint64_t> dig;
  kvadmit::SimulationResult partial;
  int status = KVG_OK;
  kvadmit::SimulationResult result;
  int rc = guarded([&] {
    kvadmit::EngineParams ep = to_engine(*engine);
    t_sink.q1_states = 0;
    t_sink.cwd_states = 0;
    if (digests != nullptr) {
      ep.paranoid = true;
      t_sink.out = &dig;
      t_sink.page_size = ep.page_size;
    }
    kvadmit::Population pop = kvadmit::build_population(to_workload(*wl), seed);
    auto t0 = std::chrono::steady_clock::now();
    try {
      result = kvadmit::run_simulation(std::move(pop), to_policy(*policy),
                                       to_cost(*cost), ep, &partial);
    } catch (const kvadmit::HorizonError&) {
      auto t1 = std::chrono::steady_clock::now();
      if (wall_s) *wall_s = std::chrono::duration<double>(t1 - t0).count();
      t_sink.out = nullptr;
      result = std::move(partial);
      throw;
    }
    auto t1 = std::chrono::steady_clock::now();
    if (wall_s) *wall_s = std::chrono::duration<double>(t1 - t0).count();
    t_sink.out = nullptr;
  });
  t_sink.out = nullptr;
  status = rc;
  if (rc != KVG_OK && rc != KVG_ERR_HORIZON) return rc;
  fill_result(result, status, res, trace, trace_cap, n_trace, agents, agents_cap);
  if (n_digests) *n_digests = dig.size();
  if (digests)
    std::memcpy(digests, dig.data(),
                std::min(dig.size(), digest_cap) * sizeof(std::uint64_t));
  return rc;
}

/* Many independent runs on `threads` host threads, like the reference's own
 * run_rows pool (experiment.cpp:75-108). Populations are built before the
 * clock starts; wall_s covers the run_simulation calls only. */
KVR_API int kvr_run_many(size_t n, const kvg_workload_config* wls,
                         const uint64_t* seeds, const kvg_policy* policies,
                         const kvg_cost_params* costs,
                         const kvg_engine_params* engines, unsigned threads,
                         double* makespans, uint64_t* decoded, double* wall_s) {
  return guarded([&] {
    std::vector<kvadmit::Population> pops;
    pops.reserve(n);
    for (size_t i = 0; i < n; ++i)
      pops.push_back(kvadmit::build_population(to_workload(wls[i]), seeds[i]));
    std::vector<std::exception_ptr> errs(n);
    std::atomic<size_t> next{0};
    auto worker = [&] {
      for (;;) {
        size_t i = next.fetch_add(1);
        if (i >= n) return;
        try {
          kvadmit::SimulationResult r = kvadmit::run_simulation(
              std::move(pops[i]), to_policy(policies[i]), to_cost(costs[i]),
              to_engine(engines[i]));
          if (makespans) makespans[i] = r.makespan;
          if (decoded) decoded[i] = r.decoded_tokens;
        } catch (...) {
          errs[i] = std::current_exception();
        }
      }
    };
    unsigned t = threads < 1 ? 1 : threads;
    auto t0 = std::chrono::steady_clock::now();
    if (t == 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (unsigned k = 0; k < t; ++k) pool.emplace_back(worker);
      for (auto& th : pool) th.join();
    }
    auto t1 = std::chrono::steady_clock::now();
    if (wall_s) *wall_s = std::chrono::duration<double>(t1 - t0).count();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

/* Many independent runs with their full outputs, for full-size golden
 * fixtures (e.g. all 4,096 C4 sweep simulations): res[i] receives run i's
 * SimulationResult scalars, trace[i * trace_stride ...] its trace rows
 * (n_trace[i] = the row count, which may exceed trace_stride: then only the
 * first trace_stride rows are written and the caller retries with a larger
 * stride), agents[agent_off[i] ...] its agent stats. Runs on `threads`
 * threads like kvr_run_many. Horizon aborts keep their partial results
 * (status KVG_ERR_HORIZON in res[i].status). */
KVR_API int kvr_run_many_out(size_t n, const kvg_workload_config* wls,
                             const uint64_t* seeds, const kvg_policy* policies,
                             const kvg_cost_params* costs,
                             const kvg_engine_params* engines, unsigned threads,
                             kvg_sim_result* res, kvg_trace_row* trace,
                             size_t trace_stride, size_t* n_trace,
                             kvg_agent_stats* agents, const size_t* agent_off) {
  return guarded([&] {
    std::vector<std::exception_ptr> errs(n);
    std::atomic<size_t> next{0};
    auto worker = [&] {
      for (;;) {
        size_t i = next.fetch_add(1);
        if (i >= n) return;
        try {
          kvadmit::Population pop = kvadmit::build_population(to_workload(wls[i]), seeds[i]);
          kvadmit::SimulationResult partial, r;
          int status = KVG_OK;
          try {
            r = kvadmit::run_simulation(std::move(pop), to_policy(policies[i]),
                                        to_cost(costs[i]), to_engine(engines[i]), &partial);
          } catch (const kvadmit::HorizonError&) {
            r = std::move(partial);
            status = KVG_ERR_HORIZON;
          }
          fill_result(r, status, &res[i], trace + i * trace_stride, trace_stride,
                      &n_trace[i], agents + agent_off[i], wls[i].agents);
        } catch (...) {
          errs[i] = std::current_exception();
        }
      }
    };
    unsigned t = threads < 1 ? 1 : threads;
    std::vector<std::thread> pool;
    for (unsigned k = 1; k < t; ++k) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

/* ---------------- run artifacts through the reference's own writers ------- */

/* execute_run's finalize (experiment.cpp:161-170) on a reference run:
 * summarize + export_trace / export_summary / export_phases into `dir`. */
KVR_API int kvr_run_artifacts(const kvg_workload_config* wl, uint64_t seed,
                              const kvg_policy* policy, const kvg_cost_params* cost,
                              const kvg_engine_params* engine, const char* name,
                              const char* policy_label, const char* dir) {
  return guarded([&] {
    kvadmit::Population pop = kvadmit::build_population(to_workload(*wl), seed);
    kvadmit::SimulationResult partial, result;
    const kvadmit::Policy pol = to_policy(*policy);
    try {
      result = kvadmit::run_simulation(std::move(pop), pol, to_cost(*cost), to_engine(*engine),
                                       &partial);
    } catch (const kvadmit::HorizonError&) {
      result = std::move(partial);
    }
    kvadmit::Summary s = kvadmit::summarize(result, name, pol, seed, wl->agents);
    s.policy = policy_label;
    const std::string d(dir);
    kvadmit::export_trace(result.trace, d + "/trace.csv");
    kvadmit::export_summary(s, d + "/summary.txt");
    kvadmit::export_phases(result.phases, d + "/phases.csv");
  });
}

/* ---------------- CacheTree differential surface ------------------------- */

namespace {

struct RefCache {
  kvadmit::CacheTree tree;
  std::uint64_t prompt_tokens;
  bool shared;
  std::vector<std::vector<kvadmit::TokenId>> sink;
  RefCache(std::uint64_t cap, std::uint64_t ps, kvadmit::EvictionMode m,
           std::uint64_t p, bool s)
      : tree(cap, ps, m), prompt_tokens(p), shared(s) {
    tree.set_victim_sink(&sink);
  }
  /* Token sequence agent `a` holds at length `len` (workload.cpp:139-142,
   * 167-171, 191): prompt then private counter ids. */
  std::vector<kvadmit::TokenId> seq(std::uint32_t a, std::uint64_t len) const {
    std::vector<kvadmit::TokenId> s(len);
    const kvadmit::TokenId base = (static_cast<kvadmit::TokenId>(a) + 1) << 32;
    for (std::uint64_t p = 0; p < len; ++p) {
      if (shared)
        s[p] = p < prompt_tokens ? p : (base | (p - prompt_tokens));
      else
        s[p] = base | p;
    }
    return s;
  }
};

}  // namespace

KVR_API void* kvr_cache_new(uint64_t capacity, uint64_t page_size,
                            uint32_t eviction, uint64_t prompt_tokens,
                            uint32_t shared) {
  try {
    return new RefCache(capacity, page_size,
                        eviction == KVG_EVICT_OFFLOAD
                            ? kvadmit::EvictionMode::kOffload
                            : kvadmit::EvictionMode::kDiscard,
                        prompt_tokens, shared != 0);
  } catch (const std::exception& e) {
    t_err = e.what();
    return nullptr;
  }
}

KVR_API void kvr_cache_free(void* h) { delete static_cast<RefCache*>(h); }

/* Executes one op. Victim pages (owner << 32 | page) are written in the
 * order the reference evicted them (one entry per page). */
KVR_API int kvr_cache_op(void* h, const kvg_cache_op* op, kvg_cache_op_result* r,
                         uint64_t* victims, size_t cap, size_t* n_victims) {
  RefCache* c = static_cast<RefCache*>(h);
  c->sink.clear();
  std::memset(r, 0, sizeof *r);
  int rc = guarded([&] {
    auto s = c->seq(op->agent, op->len);
    switch (op->kind) {
      case KVG_OP_MATCH: {
        auto m = c->tree.match_prefix(s);
        r->r0 = m.matched;
        r->r1 = m.host_matched;
        break;
      }
      case KVG_OP_INSERT: {
        auto o = c->tree.insert(s);
        r->r0 = o.ok ? 1 : 0;
        r->r1 = o.inserted_slots;
        break;
      }
      case KVG_OP_EVICT: r->r0 = c->tree.evict(op->arg).reclaimed_slots; break;
      case KVG_OP_PIN: c->tree.pin(s, op->arg); break;
      case KVG_OP_UNPIN: c->tree.unpin(s, op->arg); break;
      case KVG_OP_DISCARD: c->tree.discard_suffix(s, op->arg); break;
      case KVG_OP_RELOAD: {
        kvadmit::EvictStats ev;
        r->r0 = c->tree.reload(s, op->arg, op->arg2, &ev);
        r->r1 = ev.offloaded_tokens;
        break;
      }
      default: throw kvadmit::ConfigError("unknown op");
    }
  });
  r->status = rc;
  r->clock = c->tree.clock();
  r->used = c->tree.pool().used;
  const std::uint64_t ps = c->tree.page_size();
  size_t k = 0;
  for (const auto& path : c->sink) {
    if (path.size() % ps != 0) continue;  // one entry per page: its last token
    std::uint64_t page = path.size() / ps - 1;
    std::uint64_t key = (owner_of(path.back()) << 32) | page;
    if (victims && k < cap) victims[k] = key;
    ++k;
  }
  if (n_victims) *n_victims = k;
  return rc;
}

KVR_API void kvr_cache_stats(void* h, double* hit_matched, double* hit_requested,
                             uint64_t* discarded, uint64_t* offloaded) {
  RefCache* c = static_cast<RefCache*>(h);
  if (hit_matched) *hit_matched = c->tree.hit_window_matched();
  if (hit_requested) *hit_requested = c->tree.hit_window_requested();
  if (discarded) *discarded = c->tree.total_discarded_tokens();
  if (offloaded) *offloaded = c->tree.total_offloaded_tokens();
}

KVR_API uint64_t kvr_cache_digest(void* h) {
  return cache_digest(static_cast<RefCache*>(h)->tree);
}

KVR_API int kvr_cache_check(void* h) {
  return guarded([&] { static_cast<RefCache*>(h)->tree.check_invariants(); });
}
