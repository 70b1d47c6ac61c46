// Host prologue/epilogue of the B200 engine (plain C++, compiled with the
// reference's -O2 and no -march so libm and double rounding match it).
//
//  * kvg_build_population — the workload sampling stream (workload.cpp:22-41,
//    76-96, 153-204): splitmix64 seeds, Box-Muller lognormal, FNV-1a hash.
//  * descriptor validation — EngineParams/Policy/ControllerConfig/CostParams/
//    PhaseParams::validate (engine.cpp:21-29, controller.cpp:24-52,
//    cost_model.cpp:20-27, metrics.cpp:34-39).
//  * kvg_classify_phases — metrics.cpp:41-81.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/kvgpu.h"
#include "host_internal.h"

namespace kvg_host {

thread_local std::string g_last_error = "no error";

int set_error(int code, const std::string& what) {
  g_last_error = what;
  return code;
}

namespace {

std::uint64_t next_sm64(std::uint64_t& s) {
  std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double unit(std::uint64_t& s) {  // 53 random bits in [0,1)
  return static_cast<double>(next_sm64(s) >> 11) * 0x1.0p-53;
}

double gauss(std::uint64_t& s) {  // cosine branch of Box-Muller, one draw
  const double u1 = 1.0 - unit(s);
  const double u2 = unit(s);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}

double draw(const kvg_distribution& d, std::uint64_t& s) {
  if (d.kind == KVG_DIST_UNIFORM) return d.a + (d.b - d.a) * unit(s);
  if (d.kind == KVG_DIST_LOGNORMAL) {
    const double sigma = d.b;
    const double mu = std::log(d.a) - sigma * sigma / 2.0;  // mean of the lognormal = a
    return std::exp(mu + sigma * gauss(s));
  }
  return d.a;
}

std::uint64_t draw_count(const kvg_distribution& d, std::uint64_t& s) {
  double v = draw(d, s);
  if (v < 0) v = 0;
  return static_cast<std::uint64_t>(std::llround(v));
}

std::uint64_t fnv_double(std::uint64_t h, double v) {
  unsigned char b[8];
  std::memcpy(b, &v, 8);
  for (unsigned char c : b) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

bool dist_ok(const kvg_distribution& d, const char* what, std::string* why) {
  switch (d.kind) {
    case KVG_DIST_CONSTANT:
      if (d.a < 0) { *why = std::string(what) + ": constant value must be >= 0"; return false; }
      return true;
    case KVG_DIST_UNIFORM:
      if (d.a < 0 || d.b < d.a) { *why = std::string(what) + ": uniform needs 0 <= min <= max"; return false; }
      return true;
    case KVG_DIST_LOGNORMAL:
      if (d.a <= 0) { *why = std::string(what) + ": lognormal mean must be > 0"; return false; }
      if (d.b < 0) { *why = std::string(what) + ": lognormal sigma must be >= 0"; return false; }
      return true;
    default:
      *why = std::string(what) + ": unknown distribution";
      return false;
  }
}

}  // namespace

/* Policy::validate + ControllerConfig::validate (controller.cpp:24-52). */
bool validate_policy(const kvg_policy& p, std::string* why) {
  if (p.kind > KVG_POLICY_AIMD) { *why = "unknown policy"; return false; }
  if ((p.kind == KVG_POLICY_REQUEST_CAP || p.kind == KVG_POLICY_AGENT_CAP) && p.cap < 1) { *why = "fixed cap policies need cap >= 1"; return false; }
  if (p.kind == KVG_POLICY_AIMD) {
    const kvg_controller_config& c = p.aimd;
    if (!(c.u_low >= 0 && c.u_low <= c.u_high && c.u_high <= 1)) { *why = "controller thresholds need 0 <= u_low <= u_high <= 1"; return false; }
    if (!(c.beta > 0 && c.beta < 1)) { *why = "controller.beta must be in (0,1)"; return false; }
    if (!(c.alpha > 0)) { *why = "controller.alpha must be > 0"; return false; }
    if (!(c.h_thresh >= 0 && c.h_thresh <= 1)) { *why = "controller.h_thresh must be in [0,1]"; return false; }
    if (!(c.w_min >= 1)) { *why = "controller.w_min must be >= 1"; return false; }
    if (c.w_max != 0 && c.w_max < c.w_min) { *why = "controller.w_max must be >= w_min"; return false; }
    if (c.initial_window != 0 && (c.initial_window < c.w_min || (c.w_max != 0 && c.initial_window > c.w_max))) { *why = "controller.initial_window outside [w_min, w_max]"; return false; }
    if (!(c.control_interval > 0)) { *why = "controller.control_interval must be > 0"; return false; }
    if (!(c.signal_smoothing >= 0 && c.signal_smoothing < 1)) { *why = "controller.signal_smoothing must be in [0,1)"; return false; }
  }
  return true;
}

bool validate_sim(const kvg_sim_desc& d, std::string* why) {
  const kvg_engine_params& e = d.engine;
  if (d.population == nullptr) { *why = "null population"; return false; }
  if (d.population->agents > 0 && d.population->plans == nullptr) { *why = "population has no plans"; return false; }
  if (d.population->steps < 1) { *why = "workload.steps must be >= 1"; return false; }
  if (e.capacity == 0) { *why = "cache.capacity must be positive"; return false; }
  if (e.page_size == 0) { *why = "cache.page_size must be positive"; return false; }
  if (!(e.hit_window_decay >= 0 && e.hit_window_decay < 1)) { *why = "cache.hit_window_decay must be in [0,1)"; return false; }
  if (!(e.horizon > 0)) { *why = "horizon must be positive"; return false; }
  if (!(e.phases.sat_threshold > 0 && e.phases.sat_threshold <= 1)) { *why = "phases.sat_threshold must be in (0,1]"; return false; }
  if (!(e.phases.hit_threshold >= 0 && e.phases.hit_threshold <= 1)) { *why = "phases.hit_threshold must be in [0,1]"; return false; }
  if (e.phases.hysteresis < 1) { *why = "phases.hysteresis must be >= 1"; return false; }
  if (e.eviction != KVG_EVICT_DISCARD && e.eviction != KVG_EVICT_OFFLOAD) { *why = "unknown eviction mode"; return false; }
  const kvg_policy& p = d.policy;
  if (!validate_policy(p, why)) return false;
  const kvg_cost_params& c = d.cost;
  if (c.prefill_linear < 0 || c.prefill_quadratic < 0 || c.decode_base < 0 || c.decode_context < 0 ||
      c.bytes_per_token < 0 || c.transfer_sync_overhead < 0) { *why = "cost parameters must be non-negative"; return false; }
  if (c.pcie_bandwidth <= 0) { *why = "pcie_bandwidth must be > 0"; return false; }
  if (!(p.aimd.control_interval > 0)) { *why = "controller.control_interval must be > 0"; return false; }
  return true;
}

}  // namespace kvg_host

using kvg_host::set_error;

extern "C" {

KVG_API const char* kvg_version(void) { return "0.1.0-b200"; }

KVG_API const char* kvg_last_error(void) { return kvg_host::g_last_error.c_str(); }

KVG_API kvg_status kvg_build_population(const kvg_workload_config* cfg, uint64_t seed,
                                        kvg_population* out) {
  if (cfg == nullptr || out == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  std::string why;
  if (cfg->steps < 1) return (kvg_status)set_error(KVG_ERR_CONFIG, "workload.steps must be >= 1");
  if (!kvg_host::dist_ok(cfg->gen_tokens, "workload.gen_tokens", &why) ||
      !kvg_host::dist_ok(cfg->obs_tokens, "workload.obs_tokens", &why) ||
      !kvg_host::dist_ok(cfg->tool_latency, "workload.tool_latency", &why))
    return (kvg_status)set_error(KVG_ERR_CONFIG, why);
  if (cfg->tool_probability < 0 || cfg->tool_probability > 1)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "workload.tool_probability must be in [0,1]");
  const std::size_t n = static_cast<std::size_t>(cfg->agents) * cfg->steps;
  kvg_step_plan* plans = static_cast<kvg_step_plan*>(std::calloc(n > 0 ? n : 1, sizeof(kvg_step_plan)));
  if (plans == nullptr) return (kvg_status)set_error(KVG_ERR_STATE, "out of memory");
  std::uint64_t hash = 0xcbf29ce484222325ULL;
  std::uint64_t shared_total = 0, private_total = 0;
  for (std::uint32_t id = 0; id < cfg->agents; ++id) {
    std::uint64_t s0 = seed;
    std::uint64_t rng = kvg_host::next_sm64(s0) ^ (0x9e3779b97f4a7c15ULL * (static_cast<std::uint64_t>(id) + 1));
    std::uint64_t final_ctx = cfg->prompt_tokens;
    for (std::uint32_t k = 0; k < cfg->steps; ++k) {
      kvg_step_plan& sp = plans[static_cast<std::size_t>(id) * cfg->steps + k];
      sp.gen_tokens = kvg_host::draw_count(cfg->gen_tokens, rng);
      sp.obs_tokens = kvg_host::draw_count(cfg->obs_tokens, rng);
      sp.tool_latency = kvg_host::draw(cfg->tool_latency, rng);
      const double roll = kvg_host::unit(rng);
      const bool last = k + 1 == cfg->steps;
      sp.has_tool = (!last && roll < cfg->tool_probability) ? 1u : 0u;
      if (!sp.has_tool) sp.obs_tokens = 0;
      hash = kvg_host::fnv_double(hash, static_cast<double>(sp.gen_tokens));
      hash = kvg_host::fnv_double(hash, static_cast<double>(sp.obs_tokens));
      hash = kvg_host::fnv_double(hash, sp.tool_latency);
      hash = kvg_host::fnv_double(hash, sp.has_tool ? 1.0 : 0.0);
      final_ctx += sp.gen_tokens + sp.obs_tokens;
    }
    if (cfg->shared_prompt) {
      if (shared_total == 0) shared_total = cfg->prompt_tokens;
      private_total += final_ctx - cfg->prompt_tokens;
    } else {
      private_total += final_ctx;
    }
  }
  out->agents = cfg->agents;
  out->steps = cfg->steps;
  out->prompt_tokens = cfg->prompt_tokens;
  out->shared_prompt = cfg->shared_prompt ? 1u : 0u;
  out->_pad = 0;
  out->shared_prompt_tokens = cfg->shared_prompt ? cfg->prompt_tokens : 0;
  out->stream_hash = hash;
  out->peak_aggregate_tokens = shared_total + private_total;
  out->plans = plans;
  return KVG_OK;
}

KVG_API void kvg_population_free(kvg_population* pop) {
  if (pop == nullptr) return;
  std::free(pop->plans);
  pop->plans = nullptr;
}

KVG_API void kvg_cost_params_init(kvg_cost_params* p) {
  if (p == nullptr) return;
  p->prefill_linear = 5e-5;
  p->prefill_quadratic = 5e-8;
  p->decode_base = 2e-3;
  p->decode_context = 2e-8;
  p->bytes_per_token = 6.67e9 / 4096.0;
  p->pcie_bandwidth = 25e9;
  p->transfer_sync_overhead = 0.05;
}

KVG_API void kvg_controller_config_init(kvg_controller_config* c) {
  if (c == nullptr) return;
  c->alpha = 2.0;
  c->beta = 0.5;
  c->u_low = 0.2;
  c->u_high = 0.5;
  c->h_thresh = 0.2;
  c->w_min = 1.0;
  c->w_max = 0.0;
  c->initial_window = 0.0;
  c->control_interval = 0.25;
  c->signal_smoothing = 0.0;
}

KVG_API void kvg_engine_params_init(kvg_engine_params* e) {
  if (e == nullptr) return;
  std::memset(e, 0, sizeof *e);
  e->page_size = 1;
  e->eviction = KVG_EVICT_DISCARD;
  e->hit_window_decay = 0.0;
  e->horizon = 1e6;
  e->phases.sat_threshold = 0.8;
  e->phases.hit_threshold = 0.5;
  e->phases.hysteresis = 3;
}

/* metrics.cpp:41-81: warmup until the first saturated, cache-cold tick;
 * middle until `hysteresis` consecutive ticks leave that state; cooldown. */
KVG_API kvg_status kvg_classify_phases(const kvg_trace_row* rows, size_t n, double makespan,
                                       const kvg_phase_params* params, kvg_phase_label* out,
                                       size_t cap, size_t* n_out) {
  if (params == nullptr || (n > 0 && rows == nullptr))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (!(params->sat_threshold > 0 && params->sat_threshold <= 1) ||
      !(params->hit_threshold >= 0 && params->hit_threshold <= 1) || params->hysteresis < 1)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "invalid phase parameters");
  kvg_phase_label tmp[3];
  size_t k = 0;
  auto push = [&](uint32_t ph, double a, double b) { tmp[k++] = kvg_phase_label{ph, 0, a, b}; };
  if (makespan > 0) {
    auto hot = [&](const kvg_trace_row& r) {
      return r.usage >= params->sat_threshold && r.hit_rate < params->hit_threshold;
    };
    size_t enter = n;
    for (size_t i = 0; i < n; ++i)
      if (hot(rows[i])) { enter = i; break; }
    if (enter == n) {
      push(KVG_PHASE_WARMUP, 0.0, makespan);
    } else {
      const double m_start = rows[enter].time;
      double m_end = makespan;
      int bad = 0;
      for (size_t i = enter + 1; i < n; ++i) {
        if (hot(rows[i])) { bad = 0; continue; }
        if (++bad >= params->hysteresis) {
          m_end = rows[i + 1 - static_cast<size_t>(params->hysteresis)].time;
          break;
        }
      }
      if (m_start > 0) push(KVG_PHASE_WARMUP, 0.0, m_start);
      push(KVG_PHASE_MIDDLE, m_start, m_end);
      if (m_end < makespan) push(KVG_PHASE_COOLDOWN, m_end, makespan);
    }
  }
  if (n_out) *n_out = k;
  for (size_t i = 0; i < k && i < cap && out; ++i) out[i] = tmp[i];
  return KVG_OK;
}

}  // extern "C"
