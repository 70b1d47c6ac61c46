// kvadmit_gpu.hpp — the reference's C++ hot-path seam on a B200.
//
// Drop-in for
//   kvadmit::SimulationResult kvadmit::run_simulation(Population, const Policy&,
//       const CostParams&, const EngineParams&, SimulationResult* partial_on_abort)
//   (/root/reference/proj/src/engine.hpp:75-78, engine.cpp:446-456)
// with the same argument meaning, result and error behaviour:
//   * validates params, policy and cost first with the reference's own
//     validate() calls (engine.cpp:450-452: same ConfigError messages);
//   * a horizon abort fills *partial_on_abort (when non-null) and throws
//     HorizonError with the reference's message (engine.cpp:112-119);
//   * an invariant failure on the device throws InvariantViolation;
//   * a CUDA failure (or no device: there is no CPU fallback) throws
//     std::runtime_error.
// The simulation runs on the GPU through the C ABI in kvgpu.h (libkvgpu.so).
//
// Header-only. Compile it inside the reference's build (its src/ on the
// include path) and link libkvgpu.so. Two ways to use it, INTEGRATION.md §2:
//   (a) call kvgpu::run_simulation where kvadmit::run_simulation was called;
//   (b) define KVGPU_DEFINE_RUN_SIMULATION_WRAP in ONE translation unit and
//       link with -Wl,--wrap=<mangled kvadmit::run_simulation>: every
//       existing caller (execute_run, run_rows, the acceptance gate) then runs
//       on the GPU unchanged.
// kvgpu::run_simulations runs many independent simulations as ONE device
// batch (one CTA per simulation): the replacement for run_rows' thread pool
// (experiment.cpp:75-108).
//
// Populations must follow build_population's token scheme (workload.cpp:
// 153-204): the device never materialises contexts, it derives token p of
// agent a from (a, p). Anything else is rejected with ConfigError.
#ifndef KVGPU_KVADMIT_GPU_HPP_
#define KVGPU_KVADMIT_GPU_HPP_

#include <cstdint>
#include <cstdio>
#include <exception>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "engine.hpp"  // the reference's seam types (proj/src)
#include "kvgpu.h"

namespace kvgpu {

struct Options {
  int device = 0;       // CUDA device ordinal
  bool verify = false;  // re-derive every prefix match by the block-hash probe
};

// One run_simulation call's inputs (run_simulations).
struct Job {
  kvadmit::Population population;
  kvadmit::Policy policy;
  kvadmit::CostParams cost;
  kvadmit::EngineParams engine;
};

namespace detail {

inline std::string g6(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.6g", v);
  return buf;
}

// Owns the C-side population of one job.
struct CPop {
  kvg_population pop{};
  std::vector<kvg_step_plan> plans;
};

// Population -> kvg_population. The per-agent contexts are checked against
// the token scheme the device derives them from (workload.cpp:139-142,
// 167-171, 191): agent `id` at index `id`, Pending, context == prompt,
// prompt token t = t (shared) or ((id+1) << 32) | t (private), private
// counter starting past the prompt.
inline void convert_population(const kvadmit::Population& p, CPop& out) {
  using kvadmit::ConfigError;
  const std::size_t n = p.agents.size();
  if (n == 0) throw ConfigError("kvgpu: population has no agents");
  const std::uint64_t P = p.agents[0].spec.prompt.size();
  const std::size_t steps = p.agents[0].spec.steps.size();
  const bool shared = p.shared_prompt_tokens > 0;
  if (shared && p.shared_prompt_tokens != P)
    throw ConfigError("kvgpu: shared_prompt_tokens differs from the prompt length");
  out.plans.resize(n * steps);
  for (std::size_t i = 0; i < n; ++i) {
    const kvadmit::AgentRecord& a = p.agents[i];
    if (a.spec.id != i) throw ConfigError("kvgpu: agent ids must be 0..n-1 in order");
    if (a.spec.prompt.size() != P || a.spec.steps.size() != steps)
      throw ConfigError("kvgpu: agents must share prompt length and step count");
    if (a.state != kvadmit::AgentState::kPending || a.step_index != 0 || a.high_water != 0 ||
        a.pinned_len != 0)
      throw ConfigError("kvgpu: agents must start Pending at step 0");
    if (a.context != a.spec.prompt)
      throw ConfigError("kvgpu: agent context must equal its prompt at start");
    const std::uint64_t owner = (static_cast<std::uint64_t>(i) + 1) << 32;
    for (std::uint64_t t = 0; t < P; ++t) {
      const kvadmit::TokenId want = shared ? t : (owner | t);
      if (a.spec.prompt[t] != want)
        throw ConfigError("kvgpu: prompt tokens do not follow build_population's scheme");
    }
    if (a.token_counter != (shared ? 0 : P))
      throw ConfigError("kvgpu: private token counter does not follow build_population");
    for (std::size_t s = 0; s < steps; ++s) {
      const kvadmit::StepPlan& sp = a.spec.steps[s];
      kvg_step_plan& d = out.plans[i * steps + s];
      d.gen_tokens = sp.gen_tokens;
      d.obs_tokens = sp.obs_tokens;
      d.tool_latency = sp.tool_latency;
      d.has_tool = sp.has_tool ? 1u : 0u;
      d._pad = 0;
    }
  }
  kvg_population& c = out.pop;
  c.agents = static_cast<std::uint32_t>(n);
  c.steps = static_cast<std::uint32_t>(steps);
  c.prompt_tokens = P;
  c.shared_prompt = shared ? 1u : 0u;
  c.shared_prompt_tokens = p.shared_prompt_tokens;
  c.stream_hash = p.stream_hash;
  c.peak_aggregate_tokens = p.peak_aggregate_tokens;
  c.plans = out.plans.data();
}

inline kvg_sim_desc make_desc(const CPop& cp, const kvadmit::Policy& p,
                              const kvadmit::CostParams& c, const kvadmit::EngineParams& e) {
  kvg_sim_desc d{};
  d.population = &cp.pop;
  switch (p.kind) {  // controller.hpp:49-54
    case kvadmit::PolicyKind::kUncontrolled: d.policy.kind = KVG_POLICY_UNCONTROLLED; break;
    case kvadmit::PolicyKind::kFixedRequestCap: d.policy.kind = KVG_POLICY_REQUEST_CAP; break;
    case kvadmit::PolicyKind::kFixedAgentCap: d.policy.kind = KVG_POLICY_AGENT_CAP; break;
    case kvadmit::PolicyKind::kCacheAwareAimd: d.policy.kind = KVG_POLICY_AIMD; break;
  }
  d.policy.cap = p.cap;
  const kvadmit::ControllerConfig& a = p.aimd;
  d.policy.aimd = {a.alpha, a.beta, a.u_low, a.u_high, a.h_thresh, a.w_min, a.w_max,
                   a.initial_window, a.control_interval, a.signal_smoothing};
  d.cost = {c.prefill_linear, c.prefill_quadratic, c.decode_base, c.decode_context,
            c.bytes_per_token, c.pcie_bandwidth, c.transfer_sync_overhead};
  d.engine.capacity = e.capacity;
  d.engine.page_size = e.page_size;
  d.engine.eviction =
      e.eviction == kvadmit::EvictionMode::kOffload ? KVG_EVICT_OFFLOAD : KVG_EVICT_DISCARD;
  d.engine.paranoid = e.paranoid ? 1u : 0u;
  d.engine.hit_window_decay = e.hit_window_decay;
  d.engine.horizon = e.horizon;
  d.engine.phases.sat_threshold = e.phase_params.sat_threshold;
  d.engine.phases.hit_threshold = e.phase_params.hit_threshold;
  d.engine.phases.hysteresis = e.phase_params.hysteresis;
  return d;
}

// finish_result's fields (engine.cpp:398-415) from the device outputs.
inline kvadmit::SimulationResult to_result(kvg_batch* b, std::size_t i, const kvg_sim_result& s,
                                           std::size_t agents) {
  kvadmit::SimulationResult r;
  const kvg_trace_row* rows = nullptr;
  std::size_t n_rows = 0;
  if (kvg_batch_trace_view(b, i, &rows, &n_rows) != KVG_OK)
    throw std::runtime_error(std::string("kvgpu: ") + kvg_last_error());
  r.trace.reserve(n_rows);
  r.tick_hits.reserve(n_rows);
  for (std::size_t k = 0; k < n_rows; ++k) {
    const kvg_trace_row& t = rows[k];
    kvadmit::TraceRecord tr;
    tr.time = t.time;
    tr.usage = t.usage;
    tr.hit_rate = t.hit_rate;
    tr.window = t.window;
    tr.active = t.active;
    tr.pending = t.pending;
    tr.decoded_cum = t.decoded_cum;
    tr.recompute_cum = t.recompute_cum;
    tr.transfers = t.transfers;
    r.trace.push_back(tr);
    r.tick_hits.push_back({t.hit_matched, t.hit_requested});
  }
  for (std::uint32_t k = 0; k < s.n_phases && k < 3; ++k) {
    kvadmit::PhaseLabel pl;
    pl.phase = static_cast<kvadmit::Phase>(s.phases[k].phase);  // same enum order
    pl.start = s.phases[k].start;
    pl.end = s.phases[k].end;
    r.phases.push_back(pl);
  }
  r.ledger.prefill_fresh = s.ledger.prefill_fresh;
  r.ledger.prefill_recompute = s.ledger.prefill_recompute;
  r.ledger.decode = s.ledger.decode;
  r.ledger.transfer = s.ledger.transfer;
  r.ledger.tool_wait = s.ledger.tool_wait;
  r.makespan = s.makespan;
  r.device_busy = s.device_busy;
  r.link_busy = s.link_busy;
  r.decoded_tokens = s.decoded_tokens;
  r.recompute_tokens = s.recompute_tokens;
  r.recompute_events = s.recompute_events;
  r.stall_events = s.stall_events;
  r.offloaded_tokens = s.offloaded_tokens;
  r.reloaded_tokens = s.reloaded_tokens;
  r.discarded_tokens = s.discarded_tokens;
  r.total_wait_time = s.total_wait_time;
  r.ticks = s.ticks;
  r.workload_hash = s.workload_hash;
  std::vector<kvg_agent_stats> st(agents);
  std::size_t got = 0;
  if (kvg_batch_agent_stats(b, i, st.data(), st.size(), &got) != KVG_OK)
    throw std::runtime_error(std::string("kvgpu: ") + kvg_last_error());
  r.agent_stats.reserve(got);
  for (std::size_t k = 0; k < got; ++k) {
    kvadmit::AgentStats a;
    a.generated_tokens = st[k].generated_tokens;
    a.recompute_tokens = st[k].recompute_tokens;
    a.recompute_events = st[k].recompute_events;
    a.stall_events = st[k].stall_events;
    a.pause_events = st[k].pause_events;
    a.wait_time = st[k].wait_time;
    r.agent_stats.push_back(a);
  }
  return r;
}

[[noreturn]] inline void throw_status(kvg_status st) {
  const std::string msg = kvg_last_error();
  switch (st) {
    case KVG_ERR_CONFIG: throw kvadmit::ConfigError(msg);
    case KVG_ERR_IO: throw kvadmit::IoError(msg);
    case KVG_ERR_STATE: throw kvadmit::InvariantViolation(msg);
    default: throw std::runtime_error("kvgpu: " + msg);
  }
}

// Frees the batch on every exit path.
struct BatchGuard {
  kvg_batch* b = nullptr;
  ~BatchGuard() { kvg_batch_free(b); }
};

}  // namespace detail

// Runs jobs as one device batch. results[i] / errors[i] hold job i's outcome:
// errors[i] is null on success, else the exception run_simulation would have
// thrown for it (a horizon abort still leaves the partial result in
// results[i], as partial_on_abort does). Inputs are validated per job first.
inline void run_simulations(const std::vector<Job>& jobs,
                            std::vector<kvadmit::SimulationResult>& results,
                            std::vector<std::exception_ptr>& errors, const Options& opt = {}) {
  const std::size_t n = jobs.size();
  results.assign(n, kvadmit::SimulationResult{});
  errors.assign(n, nullptr);
  std::vector<detail::CPop> cpops(n);
  std::vector<kvg_sim_desc> descs;
  std::vector<std::size_t> idx;  // batch slot -> job
  for (std::size_t i = 0; i < n; ++i) {
    try {
      jobs[i].engine.validate();  // engine.cpp:450-452, same order
      jobs[i].policy.validate();
      jobs[i].cost.validate();
      detail::convert_population(jobs[i].population, cpops[i]);
      descs.push_back(detail::make_desc(cpops[i], jobs[i].policy, jobs[i].cost, jobs[i].engine));
      idx.push_back(i);
    } catch (...) {
      errors[i] = std::current_exception();
    }
  }
  if (descs.empty()) return;
  kvg_batch_options o;
  kvg_batch_options_init(&o);
  o.host_outputs = 1;
  o.verify = opt.verify ? 1u : 0u;
  detail::BatchGuard g;
  kvg_status st = kvg_batch_create(opt.device, descs.data(), descs.size(), &o, &g.b);
  if (st != KVG_OK) detail::throw_status(st);
  st = kvg_batch_run(g.b);
  if (st != KVG_OK && st != KVG_ERR_HORIZON) detail::throw_status(st);
  for (std::size_t k = 0; k < descs.size(); ++k) {
    const std::size_t i = idx[k];
    kvg_sim_result s;
    if (kvg_batch_result(g.b, k, &s) != KVG_OK) detail::throw_status(KVG_ERR_CUDA);
    try {
      if (s.status == KVG_ERR_STATE)
        throw kvadmit::InvariantViolation("kvgpu: device simulation failed its invariant check");
      if (s.status != KVG_OK && s.status != KVG_ERR_HORIZON)
        throw std::runtime_error("kvgpu: simulation failed with status " +
                                 std::to_string(s.status));
      results[i] = detail::to_result(g.b, k, s, cpops[i].pop.agents);
      if (s.status == KVG_ERR_HORIZON)
        throw kvadmit::HorizonError("simulated time " + detail::g6(s.abort_time) +
                                    " exceeded horizon " + detail::g6(jobs[i].engine.horizon) +
                                    " with " + std::to_string(s.unfinished) +
                                    " agents unfinished");
    } catch (...) {
      errors[i] = std::current_exception();
    }
  }
}

// kvadmit::run_simulation on the GPU (engine.hpp:75-78).
inline kvadmit::SimulationResult run_simulation(kvadmit::Population population,
                                                const kvadmit::Policy& policy,
                                                const kvadmit::CostParams& cost,
                                                const kvadmit::EngineParams& params,
                                                kvadmit::SimulationResult* partial_on_abort = nullptr,
                                                const Options& opt = {}) {
  params.validate();  // engine.cpp:450-452
  policy.validate();
  cost.validate();
  std::vector<Job> jobs(1);
  jobs[0].population = std::move(population);
  jobs[0].policy = policy;
  jobs[0].cost = cost;
  jobs[0].engine = params;
  std::vector<kvadmit::SimulationResult> res;
  std::vector<std::exception_ptr> err;
  run_simulations(jobs, res, err, opt);
  if (err[0]) {
    try {
      std::rethrow_exception(err[0]);
    } catch (const kvadmit::HorizonError&) {
      if (partial_on_abort != nullptr) *partial_on_abort = std::move(res[0]);
      throw;
    }
  }
  return std::move(res[0]);
}

}  // namespace kvgpu

#ifdef KVGPU_DEFINE_RUN_SIMULATION_WRAP
// Link-time drop-in: with
//   -Wl,--wrap=_ZN7kvadmit14run_simulationENS_10PopulationERKNS_6PolicyERKNS_10CostParamsERKNS_12EngineParamsEPNS_16SimulationResultE
// every reference call of kvadmit::run_simulation lands here. KVGPU_DEVICE
// (environment) picks the device; KVGPU_VERIFY=1 turns on the probe check.
#include <cstdlib>
extern "C" kvadmit::SimulationResult
__wrap__ZN7kvadmit14run_simulationENS_10PopulationERKNS_6PolicyERKNS_10CostParamsERKNS_12EngineParamsEPNS_16SimulationResultE(
    kvadmit::Population population, const kvadmit::Policy& policy,
    const kvadmit::CostParams& cost, const kvadmit::EngineParams& params,
    kvadmit::SimulationResult* partial_on_abort) {
  kvgpu::Options o;
  if (const char* d = std::getenv("KVGPU_DEVICE")) o.device = std::atoi(d);
  if (const char* v = std::getenv("KVGPU_VERIFY")) o.verify = std::atoi(v) != 0;
  return kvgpu::run_simulation(std::move(population), policy, cost, params, partial_on_abort, o);
}
#endif

#endif  // KVGPU_KVADMIT_GPU_HPP_
