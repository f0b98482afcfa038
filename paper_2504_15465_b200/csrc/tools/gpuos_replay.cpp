// gpuos-replay: run a scenario on the deterministic replay backend of the
// B200 library and print its dispatch/completion log (the parity artefact
// compared against the reference in tests/), or its run report.
//
//   gpuos_replay (--preset NAME | --config FILE) [--horizon-ms X]
//                [--policy P] [--seed N] [--set key=value]... [--report]
//                [--time-scale F]
//
// Log format (identical to oracle/harness/ref_golden.cpp):
//   D <now> <atom> <tag> <kid> <lo> <hi> <prio> <atomized> <tpc runs>
//   C <now> <atom> <tag> <dispatch_time>
//   A <app> <offered> <completed> <p99 | -1>
//   E <end time> <energy J> <TPC busy integral> <allocated TPC time>
// Exit codes follow the reference CLI: 2 config error, 3 invariant error.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "gpuos/replay.hpp"
#include "gpuos/scenario.hpp"

using namespace gpuos;

namespace {

std::string runs_of(const std::vector<int>& t) {
  std::string s;
  for (std::size_t i = 0; i < t.size();) {
    std::size_t j = i;
    while (j + 1 < t.size() && t[j + 1] == t[j] + 1) ++j;
    if (!s.empty()) s += ',';
    s += std::to_string(t[i]);
    if (j > i) s += '-' + std::to_string(t[j]);
    i = j + 1;
  }
  return s;
}

bool truthy(const std::string& v) {
  return v == "1" || v == "true" || v == "on" || v == "yes";
}

void set_knob(ScenarioConfig& c, const std::string& kv) {
  const auto eq = kv.find('=');
  if (eq == std::string::npos) throw ConfigError("--set needs key=value");
  const std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
  SchedulerConfig& s = c.sched;
  const double x = std::atof(v.c_str());
  if (k == "stealing") s.stealing_enabled = truthy(v);
  else if (k == "atomizer") s.atomizer_enabled = truthy(v);
  else if (k == "rightsizer") s.rightsizer_enabled = truthy(v);
  else if (k == "dvfs") s.dvfs_enabled = truthy(v);
  else if (k == "occupancy_filter") s.occupancy_filter = truthy(v);
  else if (k == "block_revocation") s.block_revocation = truthy(v);
  else if (k == "chain_launches") s.chain_launches = truthy(v);
  else if (k == "chain_depth") s.chain_depth = std::atoi(v.c_str());
  else if (k == "chain_best_effort") s.chain_best_effort = truthy(v);
  else if (k == "atom_duration_us") s.atom_duration = duration_from_us(x);
  else if (k == "steal_horizon_us") s.steal_horizon = duration_from_us(x);
  else if (k == "max_outstanding_atoms") s.max_outstanding_atoms = std::atoi(v.c_str());
  else if (k == "slip_k") s.rightsizer.slip_k = x;
  else if (k == "probe_depth_limit") s.rightsizer.probe_depth_limit = std::atoi(v.c_str());
  else if (k == "dvfs_slip_k") s.dvfs.slip_k = x;
  else if (k == "ewma_beta") s.predictor.ewma_beta = x;
  else if (k == "default_unknown_us") s.predictor.default_unknown = duration_from_us(x);
  else if (k == "disable_factor") s.disable_factor = x;
  else throw ConfigError("unknown knob: " + k);
}

}  // namespace

int main(int argc, char** argv) {
  try {
    std::string preset, config, policy;
    double horizon_ms = -1, scale = 0;
    long long seed = -1;
    bool report = false;
    std::vector<std::string> knobs;
    for (int i = 1; i < argc; ++i) {
      const std::string a = argv[i];
      auto val = [&]() -> std::string {
        if (i + 1 >= argc) throw ConfigError("missing value for " + a);
        return argv[++i];
      };
      if (a == "--preset") preset = val();
      else if (a == "--config") config = val();
      else if (a == "--horizon-ms") horizon_ms = std::atof(val().c_str());
      else if (a == "--policy") policy = val();
      else if (a == "--seed") seed = std::atoll(val().c_str());
      else if (a == "--set") knobs.push_back(val());
      else if (a == "--time-scale") scale = std::atof(val().c_str());
      else if (a == "--report") report = true;
      else throw ConfigError("unknown argument: " + a);
    }
    if (preset.empty() == config.empty())
      throw ConfigError("exactly one of --preset / --config is required");
    ScenarioConfig cfg = preset.empty() ? load_scenario_file(config) : preset_scenario(preset);
    if (horizon_ms > 0) cfg.horizon = duration_from_ms(horizon_ms);
    if (!policy.empty()) cfg.sched.policy = policy_from_string(policy);
    if (seed >= 0) cfg.seed = static_cast<std::uint64_t>(seed);
    for (const auto& k : knobs) set_knob(cfg, k);
    if (scale > 0) cfg = time_scaled(cfg, scale);

    if (report) {
      const RunResult res = run_scenario(cfg);
      std::printf("%s\n%s", res.report.to_json().c_str(), res.request_log.c_str());
      return 0;
    }
    cfg.validate();
    DeviceEngine engine(cfg.topo, cfg.freq, cfg.power);
    RunHooks hooks;
    hooks.on_dispatch = [](const DispatchRecord& d) {
      std::printf("D %lld %u %d %u %ld %ld %d %d %s\n", static_cast<long long>(d.now),
                  d.atom, d.app, d.kernel, d.lo, d.hi, d.priority, d.atomized ? 1 : 0,
                  runs_of(*d.tpcs).c_str());
    };
    hooks.on_complete = [](const AtomCompletion& c) {
      std::printf("C %lld %u %llu %lld\n", static_cast<long long>(c.complete_time), c.atom,
                  static_cast<unsigned long long>(c.tag),
                  static_cast<long long>(c.dispatch_time));
    };
    hooks.on_finish = [&](const Scheduler& s) {
      for (int i = 0; i < s.app_count(); ++i) {
        const auto lat = s.completed_latencies(i);
        const long long p99 = lat.empty() ? -1 : percentile(lat, 99);
        std::printf("A %d %ld %ld %lld\n", i, s.offered(i), s.completed(i), p99);
      }
      std::printf("E %lld %.17g %.17g %.17g\n", static_cast<long long>(engine.now()),
                  engine.energy_joules(), engine.tpc_busy_integral(), s.allocated_tpc_time());
    };
    run_scenario_on(engine, cfg, hooks);
    return 0;
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const InvariantError& e) {
    std::fprintf(stderr, "invariant error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
