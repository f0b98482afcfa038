// Golden dispatch/completion log extractor for the UNMODIFIED reference.
// Test infrastructure only (see oracle/README.md): never on the product path.
//
// The reference exports no atom->TPC log. This harness
// recovers it without touching the reference sources:
//   * dispatches: the call from Scheduler::dispatch_atom (scheduler.cpp:393)
//     into DeviceEngine::submit_atom (device.cpp:121) crosses object files,
//     so the link step wraps it with -Wl,--wrap=<mangled submit_atom>;
//   * completions: the engine's completion handler (device.hpp:102-104),
//     installed by the Scheduler ctor (scheduler.cpp:107), is chained.
//
// Output format (one event per line; the B200 replay engine emits the same):
//   D <now> <atom> <tag> <kid> <lo> <hi> <prio> <atomized> <tpcs as passed>
//   C <now> <atom> <tag> <dispatch_time>
// TPC lists keep the caller's order, compressed into ascending runs "a-b".
// Modes: default = D/C log; --report = run_scenario report + request log.
#include <cstdint>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

// Only this TU reaches the engine's private handler slot.
#define private public
#include "gpuos/sim.hpp"
#undef private

#include "scenario_args.hpp"

using namespace gpuos;

namespace {

FILE* g_out = stdout;
bool g_log = true;  // off in --report mode
DeviceEngine* g_engine = nullptr;

std::string tpc_runs(const std::vector<int>& t) {
  std::string s;
  std::size_t i = 0;
  while (i < t.size()) {
    std::size_t j = i;
    while (j + 1 < t.size() && t[j + 1] == t[j] + 1) ++j;
    if (!s.empty()) s += ',';
    s += std::to_string(t[i]);
    if (j > i) s += '-' + std::to_string(t[j]);
    i = j + 1;
  }
  return s;
}

}  // namespace

extern "C" {
AtomId __real__ZN5gpuos12DeviceEngine11submit_atomEjllRKSt6vectorIiSaIiEEibm(
    DeviceEngine* self, KernelId kernel, long lo, long hi,
    const std::vector<int>& tpcs, int priority, bool atomized,
    std::uint64_t tag);

AtomId __wrap__ZN5gpuos12DeviceEngine11submit_atomEjllRKSt6vectorIiSaIiEEibm(
    DeviceEngine* self, KernelId kernel, long lo, long hi,
    const std::vector<int>& tpcs, int priority, bool atomized,
    std::uint64_t tag) {
  AtomId id = __real__ZN5gpuos12DeviceEngine11submit_atomEjllRKSt6vectorIiSaIiEEibm(
      self, kernel, lo, hi, tpcs, priority, atomized, tag);
  if (!g_log) return id;
  std::fprintf(g_out, "D %lld %u %llu %u %ld %ld %d %d %s\n",
               static_cast<long long>(self->now()), id,
               static_cast<unsigned long long>(tag), kernel, lo, hi, priority,
               atomized ? 1 : 0, tpc_runs(tpcs).c_str());
  return id;
}
}

int main(int argc, char** argv) {
  try {
    harness::Args args = harness::parse_args(argc, argv);
    bool report = false;
    for (const auto& r : args.rest)
      if (r == "--report") report = true;
    ScenarioConfig& cfg = args.cfg;
    if (report) {
      g_log = false;
      RunResult res = run_scenario(cfg);
      std::printf("%s\n", res.report.to_json().c_str());
      std::printf("%s", res.request_log.c_str());
      return 0;
    }
    cfg.validate();
    DeviceEngine engine(cfg.topo, cfg.freq, cfg.power);
    g_engine = &engine;
    Scheduler sched(engine, cfg.sched, resolve_workloads(cfg));
    auto inner = engine.on_atom_complete_;
    engine.set_atom_complete_handler([inner](const AtomCompletion& c) {
      std::fprintf(g_out, "C %lld %u %llu %lld\n",
                   static_cast<long long>(c.complete_time), c.atom,
                   static_cast<unsigned long long>(c.tag),
                   static_cast<long long>(c.dispatch_time));
      inner(c);
    });
    sched.run(cfg.horizon);
    // Trailer: per-app completed requests and p99, plus engine accounting.
    for (int i = 0; i < sched.app_count(); ++i) {
      auto lat = sched.completed_latencies(i);
      long long p99 = lat.empty() ? -1 : percentile(lat, 99);
      std::fprintf(g_out, "A %d %ld %ld %lld\n", i, sched.offered(i),
                   sched.completed(i), p99);
    }
    std::fprintf(g_out, "E %lld %.17g %.17g %.17g\n",
                 static_cast<long long>(engine.now()), engine.energy_joules(),
                 engine.tpc_busy_integral(), sched.allocated_tpc_time());
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
