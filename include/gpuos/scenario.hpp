// Scenarios, presets, the end-to-end runner and run reports.
//
// Drop-in for the reference's metrics.hpp (metrics.hpp:13-48) and sim.hpp
// (sim.hpp:15-46). Additions for the B200 build: run_scenario_on() runs a
// scenario on any Device (replay, live B200, GPU mirror), and
// time_scaled() rescales every time constant of a scenario for live runs.
#pragma once

#include <functional>
#include <map>
#include <string>
#include <vector>

#include "gpuos/core.hpp"
#include "gpuos/tenants.hpp"
#include "gpuos/tpc_scheduler.hpp"

namespace gpuos {

// ----------------------------------------------------------------- metrics
double capacity_savings(double rightsized_tpc_time, double baseline_tpc_time);
double energy_savings(double dvfs_joules, double maxfreq_joules);

struct AppReport {
  std::string app_id;
  bool high_priority = false;
  long offered = 0;
  long completed = 0;
  Duration p50 = 0, p95 = 0, p99 = 0;
  double throughput_vs_offered = 0.0;
  double goodput_vs_offered = 0.0;
  double slo_attainment = 1.0;
};

struct RunReport {
  std::vector<AppReport> apps;
  double tpc_utilization = 0.0;
  double allocated_tpc_time = 0.0;
  double energy_joules = 0.0;
  std::map<FreqMhz, Duration> freq_residency;
  double predictor_misprediction_rate_hp = 0.0;
  Duration predictor_p99_abs_error_hp = 0;
  long predictions_hp = 0;
  double weighted_r_squared = 0.0;
  long fitted_operators = 0;
  Duration horizon = 0;
  std::uint64_t seed = 0;
  std::string policy;

  std::string to_json() const;  // canonical: sorted keys, %.9g doubles
};

// --------------------------------------------------------------- scenarios
struct ScenarioConfig {
  std::string name = "scenario";
  DeviceTopology topo = DeviceTopology::a100_like();
  FrequencyDomain freq;
  PowerModel power;
  SchedulerConfig sched;
  std::vector<AppWorkload> apps;
  Duration horizon = kSecond;
  std::uint64_t seed = 1;

  void validate() const;
};

struct RunResult {
  RunReport report;
  std::string request_log;
};

std::vector<FreqMhz> default_freq_table();

ScenarioConfig parse_scenario(const std::string& json_text);
ScenarioConfig load_scenario_file(const std::string& path);
ScenarioConfig preset_scenario(const std::string& name);  // fig7, inf-inf, inf-train
std::vector<AppWorkload> resolve_workloads(const ScenarioConfig& cfg);
RunResult run_scenario(const ScenarioConfig& cfg);

// -------------------------------------------------------- B200 additions
// Observers attached to the scheduler for one run.
struct RunHooks {
  std::function<void(const DispatchRecord&)> on_dispatch;
  std::function<void(const AtomCompletion&)> on_complete;
  // Called with the finished scheduler before the report is assembled.
  std::function<void(const Scheduler&)> on_finish;
  // Called with the new scheduler before it runs (warm start).
  std::function<void(Scheduler&)> on_start;
};

// Runs `cfg` on an existing device (its topology must match cfg.topo's TPC
// count). run_scenario(cfg) == run_scenario_on(replay engine, cfg).
RunResult run_scenario_on(Device& dev, const ScenarioConfig& cfg,
                          const RunHooks& hooks = {});

// Divides every duration of the scenario (arrivals, block durations, SLOs,
// horizon, atom duration, steal horizon, default prediction, time-slice
// window, DVFS switch latency) by `factor`, so the reference's millisecond
// scale presets can run live at a chosen time scale.
ScenarioConfig time_scaled(const ScenarioConfig& cfg, double factor);

}  // namespace gpuos
