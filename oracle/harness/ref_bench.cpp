// CPU baseline timer for the UNMODIFIED reference (bench.py's cpu_baseline
// and --impl reference legs). Test/bench infrastructure only.
//
// Runs the scenario's full dispatch path exactly as run_scenario does
// (sim.cpp:375-380: DeviceEngine + Scheduler + run) `--reps` times on each of
// `--threads` independent replicas (the reference is single-owner per
// simulation; separate simulations may run in parallel,
// SPEC.md:112) and prints one JSON object:
//   {"threads", "reps", "wall_s", "atoms", "be_atoms", "hp_atoms",
//    "blocks", "hp_p99_ns", "be_completed_requests", "sim_horizon_ns"}
// Atom counts come from Scheduler::prediction_log (one entry per completed
// atom, scheduler.cpp:428-431).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

#include "gpuos/sim.hpp"
#include "scenario_args.hpp"

using namespace gpuos;

namespace {
struct Tally {
  long atoms = 0, be_atoms = 0, hp_atoms = 0, be_requests = 0;
  long long hp_p99 = -1;
};

Tally run_once(const ScenarioConfig& cfg) {
  DeviceEngine engine(cfg.topo, cfg.freq, cfg.power);
  Scheduler sched(engine, cfg.sched, resolve_workloads(cfg));
  sched.run(cfg.horizon);
  Tally t;
  for (const auto& e : sched.prediction_log()) {
    ++t.atoms;
    if (e.high_priority) ++t.hp_atoms;
    else ++t.be_atoms;
  }
  for (int i = 0; i < sched.app_count(); ++i) {
    bool hp = sched.app_spec(i).priority == PriorityClass::HP;
    auto lat = sched.completed_latencies(i);
    if (hp && !lat.empty())
      t.hp_p99 = std::max<long long>(t.hp_p99, percentile(lat, 99));
    if (!hp) t.be_requests += sched.completed(i);
  }
  return t;
}
}  // namespace

int main(int argc, char** argv) {
  try {
    harness::Args args = harness::parse_args(argc, argv);
    int threads = 1, reps = 1;
    for (std::size_t i = 0; i < args.rest.size(); ++i) {
      if (args.rest[i] == "--threads" && i + 1 < args.rest.size())
        threads = std::atoi(args.rest[++i].c_str());
      else if (args.rest[i] == "--reps" && i + 1 < args.rest.size())
        reps = std::atoi(args.rest[++i].c_str());
    }
    args.cfg.validate();
    std::vector<Tally> out(threads);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int th = 0; th < threads; ++th) {
      pool.emplace_back([&, th] {
        Tally acc;
        for (int r = 0; r < reps; ++r) {
          Tally t = run_once(args.cfg);
          acc.atoms += t.atoms;
          acc.be_atoms += t.be_atoms;
          acc.hp_atoms += t.hp_atoms;
          acc.be_requests += t.be_requests;
          acc.hp_p99 = t.hp_p99;
        }
        out[th] = acc;
      });
    }
    for (auto& p : pool) p.join();
    double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
            .count();
    Tally sum;
    for (const auto& t : out) {
      sum.atoms += t.atoms;
      sum.be_atoms += t.be_atoms;
      sum.hp_atoms += t.hp_atoms;
      sum.be_requests += t.be_requests;
      sum.hp_p99 = t.hp_p99;
    }
    std::printf(
        "{\"threads\": %d, \"reps\": %d, \"wall_s\": %.6f, \"atoms\": %ld, "
        "\"be_atoms\": %ld, \"hp_atoms\": %ld, \"hp_p99_ns\": %lld, "
        "\"be_completed_requests\": %ld, \"sim_horizon_ns\": %lld}\n",
        threads, reps, wall, sum.atoms, sum.be_atoms, sum.hp_atoms, sum.hp_p99,
        sum.be_requests, static_cast<long long>(args.cfg.horizon));
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
