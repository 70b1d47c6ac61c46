// TEST INFRASTRUCTURE: kvgpu::run_simulations (include/kvadmit_gpu.hpp), the
// batched form of the run_simulation seam, against the UNMODIFIED reference
// run_simulation (engine.cpp:446-456) in the same process: every shipped
// preset under several policies as ONE device batch, each job's
// SimulationResult compared field by field (doubles bit for bit, the trace,
// tick hits, phases, agent stats), plus the per-job errors a bad job raises
// without failing the others. Prints one line per job and "ALL OK".
// Built by oracle/Makefile (target gpuseam) into oracle/_ref/adapter_check.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "experiment.hpp"
#include "kvadmit_gpu.hpp"

using namespace kvadmit;

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

static std::string diff(const SimulationResult& x, const SimulationResult& y) {
#define CK(f) if (!same(static_cast<double>(x.f), static_cast<double>(y.f))) return #f;
  CK(makespan) CK(device_busy) CK(link_busy) CK(decoded_tokens) CK(recompute_tokens)
  CK(recompute_events) CK(stall_events) CK(offloaded_tokens) CK(reloaded_tokens)
  CK(discarded_tokens) CK(total_wait_time) CK(ticks) CK(workload_hash)
  CK(ledger.prefill_fresh) CK(ledger.prefill_recompute) CK(ledger.decode) CK(ledger.transfer)
  CK(ledger.tool_wait)
#undef CK
  if (!(x.trace == y.trace)) return "trace";
  if (x.tick_hits.size() != y.tick_hits.size()) return "tick_hits";
  for (size_t i = 0; i < x.tick_hits.size(); ++i)
    if (!same(x.tick_hits[i].matched, y.tick_hits[i].matched) ||
        !same(x.tick_hits[i].requested, y.tick_hits[i].requested))
      return "tick_hits";
  if (x.phases.size() != y.phases.size()) return "phases";
  for (size_t i = 0; i < x.phases.size(); ++i)
    if (x.phases[i].phase != y.phases[i].phase || !same(x.phases[i].start, y.phases[i].start) ||
        !same(x.phases[i].end, y.phases[i].end))
      return "phases";
  if (x.agent_stats.size() != y.agent_stats.size()) return "agent_stats";
  for (size_t i = 0; i < x.agent_stats.size(); ++i) {
    const AgentStats &a = x.agent_stats[i], &b = y.agent_stats[i];
    if (a.generated_tokens != b.generated_tokens || a.recompute_tokens != b.recompute_tokens ||
        a.recompute_events != b.recompute_events || a.stall_events != b.stall_events ||
        a.pause_events != b.pause_events || !same(a.wait_time, b.wait_time))
      return "agent_stats";
  }
  return "";
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "oracle/_ref/configs";
  std::vector<kvgpu::Job> jobs;
  std::vector<std::string> names;
  for (const char* preset : {"smoke", "thrash", "ample"}) {
    const ScenarioConfig cfg = load_scenario(dir + "/" + preset + ".toml");
    for (const char* pol : {"uncontrolled", "aimd", "agent_cap:4", "request_cap:8", "offload"}) {
      const ResolvedRun rr = resolve_run(cfg, pol);
      jobs.push_back({build_population(cfg.workload, cfg.seed), rr.policy, cfg.cost, rr.engine});
      names.push_back(std::string(preset) + "/" + pol);
    }
  }
  // a job the reference rejects: capacity 0 (EngineParams::validate)
  jobs.push_back(jobs[0]);
  jobs.back().engine.capacity = 0;
  names.push_back("smoke/bad-capacity");
  std::vector<SimulationResult> got;
  std::vector<std::exception_ptr> err;
  kvgpu::run_simulations(jobs, got, err);
  int bad = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    std::string want_err, got_err;
    SimulationResult ref;
    try {
      ref = run_simulation(jobs[i].population, jobs[i].policy, jobs[i].cost, jobs[i].engine);
    } catch (const std::exception& e) {
      want_err = e.what();
    }
    if (err[i]) {
      try {
        std::rethrow_exception(err[i]);
      } catch (const std::exception& e) {
        got_err = e.what();
      }
    }
    const std::string d = want_err.empty() && got_err.empty() ? diff(ref, got[i]) : "";
    const bool ok = want_err == got_err && d.empty();
    bad += !ok;
    std::printf("%s %-28s %s%s\n", ok ? "OK  " : "FAIL", names[i].c_str(),
                want_err.empty() ? "" : ("error: " + want_err).c_str(),
                d.empty() ? "" : (" differs: " + d).c_str());
  }
  std::printf(bad ? "%d FAILED\n" : "ALL OK\n", bad);
  return bad ? 1 : 0;
}
