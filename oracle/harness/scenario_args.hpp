// Shared command-line handling for the oracle harness programs. Test
// infrastructure only: these programs link the UNMODIFIED reference library
// (oracle/_ref/libgpuos_ref.a, built from /root/reference/proj/src by
// oracle/Makefile) and are never part of the product path.
//
//   --preset NAME | --config FILE.json      scenario (sim.hpp:36-41)
//   --horizon-ms X  --policy P  --seed N
//   --set key=value                         scheduler knob override
//
// Knob names follow the scenario JSON keys of sim.cpp:206-234.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpuos/sim.hpp"

namespace harness {

inline bool parse_bool(const std::string& v) {
  return v == "1" || v == "true" || v == "on" || v == "yes";
}

inline void apply_knob(gpuos::ScenarioConfig& c, const std::string& kv) {
  auto eq = kv.find('=');
  if (eq == std::string::npos) throw std::runtime_error("--set needs key=value");
  std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
  auto& s = c.sched;
  if (k == "stealing") s.stealing_enabled = parse_bool(v);
  else if (k == "atomizer") s.atomizer_enabled = parse_bool(v);
  else if (k == "rightsizer") s.rightsizer_enabled = parse_bool(v);
  else if (k == "dvfs") s.dvfs_enabled = parse_bool(v);
  else if (k == "occupancy_filter") s.occupancy_filter = parse_bool(v);
  else if (k == "atom_duration_us") s.atom_duration = gpuos::duration_from_us(std::atof(v.c_str()));
  else if (k == "steal_horizon_us") s.steal_horizon = gpuos::duration_from_us(std::atof(v.c_str()));
  else if (k == "max_outstanding_atoms") s.max_outstanding_atoms = std::atoi(v.c_str());
  else if (k == "slip_k") s.rightsizer.slip_k = std::atof(v.c_str());
  else if (k == "probe_depth_limit") s.rightsizer.probe_depth_limit = std::atoi(v.c_str());
  else if (k == "dvfs_slip_k") s.dvfs.slip_k = std::atof(v.c_str());
  else if (k == "ewma_beta") s.predictor.ewma_beta = std::atof(v.c_str());
  else if (k == "default_unknown_us") s.predictor.default_unknown = gpuos::duration_from_us(std::atof(v.c_str()));
  else if (k == "disable_factor") s.disable_factor = std::atof(v.c_str());
  else throw std::runtime_error("unknown knob: " + k);
}

struct Args {
  gpuos::ScenarioConfig cfg;
  std::vector<std::string> rest;  // unconsumed arguments
};

inline Args parse_args(int argc, char** argv) {
  Args a;
  std::string preset, config;
  double horizon_ms = -1;
  std::string policy;
  long long seed = -1;
  std::vector<std::string> knobs;
  for (int i = 1; i < argc; ++i) {
    std::string s = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::runtime_error("missing value for " + s);
      return argv[++i];
    };
    if (s == "--preset") preset = next();
    else if (s == "--config") config = next();
    else if (s == "--horizon-ms") horizon_ms = std::atof(next().c_str());
    else if (s == "--policy") policy = next();
    else if (s == "--seed") seed = std::atoll(next().c_str());
    else if (s == "--set") knobs.push_back(next());
    else a.rest.push_back(s);
  }
  if (preset.empty() == config.empty())
    throw std::runtime_error("exactly one of --preset / --config is required");
  a.cfg = preset.empty() ? gpuos::load_scenario_file(config)
                         : gpuos::preset_scenario(preset);
  if (horizon_ms > 0) a.cfg.horizon = gpuos::duration_from_ms(horizon_ms);
  if (!policy.empty()) a.cfg.sched.policy = gpuos::policy_from_string(policy);
  if (seed >= 0) a.cfg.seed = static_cast<std::uint64_t>(seed);
  for (const auto& k : knobs) apply_knob(a.cfg, k);
  return a;
}

}  // namespace harness
