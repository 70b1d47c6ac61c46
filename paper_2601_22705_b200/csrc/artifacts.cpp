// Run artifacts from engine results, byte-identical to the reference's
// (SURVEY.md §8(f) item 2): trace.csv (metrics.cpp:89-101), summary.txt
// (metrics.cpp:141-183) from summarize() (engine.cpp:458-532) and phases.csv
// (metrics.cpp:266-276), written the way execute_run's finalize does
// (experiment.cpp:161-170). Host-side C++; inputs are the kvg_* result, trace
// and phase records the device produced.
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/kvgpu.h"
#include "host_internal.h"

using kvg_host::set_error;

namespace {

std::string g6(double v) {  // format_g6, metrics.cpp:83-87
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.6g", v);
  return buf;
}

const char* phase_name(uint32_t p) {  // metrics.cpp:24-31
  switch (p) {
    case KVG_PHASE_WARMUP: return "warmup";
    case KVG_PHASE_MIDDLE: return "middle";
    case KVG_PHASE_COOLDOWN: return "cooldown";
  }
  return "?";
}

struct File {
  FILE* f = nullptr;
  explicit File(const std::string& path) : f(std::fopen(path.c_str(), "wb")) {}
  ~File() {
    if (f) std::fclose(f);
  }
  void put(const std::string& s) { std::fwrite(s.data(), 1, s.size(), f); }
};

void copy_str(char* dst, size_t cap, const char* src) {
  std::snprintf(dst, cap, "%s", src ? src : "");
}

}  // namespace

extern "C" {

/* policy_name, controller.cpp:253-265 */
KVG_API kvg_status kvg_policy_name(const kvg_policy* p, char* out, size_t cap) {
  if (p == nullptr || out == nullptr || cap == 0)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  std::string s;
  switch (p->kind) {
    case KVG_POLICY_UNCONTROLLED: s = "uncontrolled"; break;
    case KVG_POLICY_REQUEST_CAP: s = "request_cap:" + std::to_string(p->cap); break;
    case KVG_POLICY_AGENT_CAP: s = "agent_cap:" + std::to_string(p->cap); break;
    case KVG_POLICY_AIMD: s = "aimd"; break;
    default: s = "?";
  }
  copy_str(out, cap, s.c_str());
  return KVG_OK;
}

/* summarize, engine.cpp:458-532 (same operation order, so every double is
 * bit-identical to the reference's Summary). */
KVG_API kvg_status kvg_summarize(const kvg_sim_result* r, const kvg_trace_row* rows, size_t n,
                                 const char* name, const char* policy_label, uint64_t seed,
                                 uint32_t agents, kvg_summary* s) {
  if (r == nullptr || s == nullptr || (n > 0 && rows == nullptr))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  std::memset(s, 0, sizeof *s);
  copy_str(s->name, sizeof s->name, name);
  copy_str(s->policy, sizeof s->policy, policy_label);
  s->seed = seed;
  s->agents = agents;
  s->makespan = r->makespan;
  s->throughput = r->makespan > 0 ? static_cast<double>(r->decoded_tokens) / r->makespan : 0.0;
  s->decoded_tokens = r->decoded_tokens;
  s->recompute_tokens = r->recompute_tokens;
  s->recompute_events = r->recompute_events;
  s->stall_events = r->stall_events;
  const double work = r->ledger.prefill_fresh + r->ledger.prefill_recompute + r->ledger.decode +
                      r->ledger.transfer;
  s->recompute_fraction = work > 0 ? r->ledger.prefill_recompute / work : 0.0;
  double matched = 0.0, requested = 0.0, usage_sum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    matched += rows[i].hit_matched;
    requested += rows[i].hit_requested;
    usage_sum += rows[i].usage;
  }
  s->mean_hit_rate = requested > 0 ? matched / requested : 1.0;
  s->mean_usage = n == 0 ? 0.0 : usage_sum / n;
  s->ledger = r->ledger;
  s->device_busy = r->device_busy;
  s->device_idle = r->makespan - r->device_busy;
  s->link_busy = r->link_busy;
  s->link_idle = r->makespan - r->link_busy;
  s->offloaded_tokens = r->offloaded_tokens;
  s->reloaded_tokens = r->reloaded_tokens;
  s->discarded_tokens = r->discarded_tokens;
  s->total_wait_time = r->total_wait_time;
  s->warmup_hit_rate = s->middle_hit_rate = s->cooldown_hit_rate = 1.0;
  for (uint32_t k = 0; k < r->n_phases && k < 3; ++k) {
    const kvg_phase_label& p = r->phases[k];
    const double span = p.end - p.start;
    double ph_m = 0.0, ph_r = 0.0, ph_u = 0.0;
    size_t ticks = 0;
    for (size_t i = 0; i < n; ++i) {
      const double t = rows[i].time;
      const bool inside = t >= p.start && (t < p.end || p.end == r->makespan);
      if (!inside) continue;
      ph_m += rows[i].hit_matched;
      ph_r += rows[i].hit_requested;
      ph_u += rows[i].usage;
      ++ticks;
    }
    const double rate = ph_r > 0 ? ph_m / ph_r : 1.0;
    switch (p.phase) {
      case KVG_PHASE_WARMUP:
        s->warmup_duration += span;
        s->warmup_hit_rate = rate;
        break;
      case KVG_PHASE_MIDDLE:
        s->middle_duration += span;
        s->middle_hit_rate = rate;
        s->middle_usage_mean = ticks > 0 ? ph_u / ticks : 0.0;
        break;
      default:
        s->cooldown_duration += span;
        s->cooldown_hit_rate = rate;
        break;
    }
  }
  s->middle_fraction = r->makespan > 0 ? s->middle_duration / r->makespan : 0.0;
  s->ticks = r->ticks;
  s->workload_hash = r->workload_hash;
  return KVG_OK;
}

/* export_trace, metrics.cpp:89-101 */
KVG_API kvg_status kvg_write_trace_csv(const char* path, const kvg_trace_row* rows, size_t n) {
  if (path == nullptr || (n > 0 && rows == nullptr))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  File f(path);
  if (!f.f) return (kvg_status)set_error(KVG_ERR_IO, std::string("cannot open trace file for writing: ") + path);
  f.put("time,usage,hit_rate,window,active,pending,decoded_cum,recompute_cum,transfers\n");
  std::string line;
  for (size_t i = 0; i < n; ++i) {
    const kvg_trace_row& r = rows[i];
    line = g6(r.time) + ',' + g6(r.usage) + ',' + g6(r.hit_rate) + ',' + g6(r.window) + ',' +
           std::to_string(r.active) + ',' + std::to_string(r.pending) + ',' +
           std::to_string(r.decoded_cum) + ',' + std::to_string(r.recompute_cum) + ',' +
           std::to_string(r.transfers) + '\n';
    f.put(line);
  }
  return KVG_OK;
}

/* export_summary, metrics.cpp:141-183 */
KVG_API kvg_status kvg_write_summary(const char* path, const kvg_summary* s) {
  if (path == nullptr || s == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  File f(path);
  if (!f.f) return (kvg_status)set_error(KVG_ERR_IO, std::string("cannot open summary file for writing: ") + path);
  auto put = [&](const char* k, const std::string& v) { f.put(std::string(k) + " = " + v + '\n'); };
  auto pu = [&](const char* k, uint64_t v) { put(k, std::to_string(v)); };
  auto pd = [&](const char* k, double v) { put(k, g6(v)); };
  put("name", s->name);
  put("policy", s->policy);
  pu("seed", s->seed);
  pu("agents", s->agents);
  pd("makespan", s->makespan);
  pd("throughput", s->throughput);
  pu("decoded_tokens", s->decoded_tokens);
  pu("recompute_tokens", s->recompute_tokens);
  pu("recompute_events", s->recompute_events);
  pu("stall_events", s->stall_events);
  pd("recompute_fraction", s->recompute_fraction);
  pd("mean_hit_rate", s->mean_hit_rate);
  pd("mean_usage", s->mean_usage);
  pd("prefill_fresh_time", s->ledger.prefill_fresh);
  pd("prefill_recompute_time", s->ledger.prefill_recompute);
  pd("decode_time", s->ledger.decode);
  pd("transfer_time", s->ledger.transfer);
  pd("tool_wait_time", s->ledger.tool_wait);
  pd("device_busy", s->device_busy);
  pd("device_idle", s->device_idle);
  pd("link_busy", s->link_busy);
  pd("link_idle", s->link_idle);
  pu("offloaded_tokens", s->offloaded_tokens);
  pu("reloaded_tokens", s->reloaded_tokens);
  pu("discarded_tokens", s->discarded_tokens);
  pd("total_wait_time", s->total_wait_time);
  pd("warmup_duration", s->warmup_duration);
  pd("middle_duration", s->middle_duration);
  pd("cooldown_duration", s->cooldown_duration);
  pd("middle_fraction", s->middle_fraction);
  pd("warmup_hit_rate", s->warmup_hit_rate);
  pd("middle_hit_rate", s->middle_hit_rate);
  pd("cooldown_hit_rate", s->cooldown_hit_rate);
  pd("middle_usage_mean", s->middle_usage_mean);
  pu("ticks", s->ticks);
  char hex[32];
  std::snprintf(hex, sizeof(hex), "0x%016" PRIx64, s->workload_hash);
  put("workload_hash", hex);
  return KVG_OK;
}

/* export_phases, metrics.cpp:266-276 */
KVG_API kvg_status kvg_write_phases_csv(const char* path, const kvg_phase_label* p, size_t n) {
  if (path == nullptr || (n > 0 && p == nullptr))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  File f(path);
  if (!f.f) return (kvg_status)set_error(KVG_ERR_IO, std::string("cannot open phases file for writing: ") + path);
  f.put("phase,start,end\n");
  for (size_t i = 0; i < n; ++i)
    f.put(std::string(phase_name(p[i].phase)) + ',' + g6(p[i].start) + ',' + g6(p[i].end) + '\n');
  return KVG_OK;
}

/* execute_run's finalize (experiment.cpp:161-170): summary + the three
 * artifacts of one run into `dir` (which must exist). */
KVG_API kvg_status kvg_write_run_artifacts(const char* dir, const char* name,
                                           const char* policy_label, uint64_t seed,
                                           uint32_t agents, const kvg_sim_result* r,
                                           const kvg_trace_row* rows, size_t n,
                                           kvg_summary* out) {
  if (dir == nullptr || r == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  kvg_summary s;
  kvg_status st = kvg_summarize(r, rows, n, name, policy_label, seed, agents, &s);
  if (st != KVG_OK) return st;
  const std::string d(dir);
  if ((st = kvg_write_trace_csv((d + "/trace.csv").c_str(), rows, n)) != KVG_OK) return st;
  if ((st = kvg_write_summary((d + "/summary.txt").c_str(), &s)) != KVG_OK) return st;
  if ((st = kvg_write_phases_csv((d + "/phases.csv").c_str(), r->phases, r->n_phases)) != KVG_OK)
    return st;
  if (out) *out = s;
  return KVG_OK;
}

}  // extern "C"
