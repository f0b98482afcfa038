// Deterministic replay backend of the device seam.
//
// Reproduces the reference's discrete-event GPU (device.cpp:74-311) bit for
// bit: integer-ns clock, (time, seq) event order with one sequence counter
// shared by atoms and events, exact-rational per-TPC slot capacity, greedy
// block-index placement over the sorted TPC set, highest-priority refill
// with no bypass, 500 ns prelude per block of an atomized kernel, piecewise
// energy / busy / frequency-residency accounting clamped at the metrics
// horizon. Same name and public signatures as the reference's DeviceEngine
// so the reference's own tests compile against this library unchanged.
#pragma once

#include <optional>
#include <vector>

#include "gpuos/core.hpp"

namespace gpuos {

class DeviceEngine final : public Device {
 public:
  DeviceEngine(DeviceTopology topo, FrequencyDomain freq, PowerModel power);

  SimTime now() const override { return clock_; }
  const DeviceTopology& topology() const override { return topo_; }
  const FrequencyDomain& freq_domain() const override { return freq_; }
  FreqMhz current_mhz() const override { return mhz_; }

  KernelId register_kernel(const SimKernelSpec& spec) override;
  AtomId submit_atom(KernelId kernel, long lo, long hi,
                     const std::vector<int>& tpcs, int priority, bool atomized,
                     std::uint64_t tag) override;
  void set_atom_paused(AtomId atom, bool paused) override;
  // Chaining (off the reference's path: only SchedulerConfig::chain_launches
  // uses it): the atom is resident at once but starts no block until its
  // predecessor retires, at that same instant.
  bool supports_chaining() const override { return true; }
  AtomId submit_chained(AtomId after, KernelId kernel, long lo, long hi,
                        const std::vector<int>& tpcs, int priority, bool atomized,
                        std::uint64_t tag, bool chain_head, bool no_early = false) override;
  SimTime request_frequency(FreqMhz f) override;
  void schedule_call(SimTime t, std::function<void()> fn) override;
  void set_atom_complete_handler(
      std::function<void(const AtomCompletion&)> h) override {
    on_complete_ = std::move(h);
  }

  bool step() override;
  void run_all() override;

  void set_metrics_horizon(SimTime t) override { horizon_ = t; }
  double energy_joules() const override { return joules_; }
  double tpc_busy_integral() const override { return busy_tpc_ns_; }
  const std::map<FreqMhz, Duration>& freq_residency() const override {
    return residency_;
  }
  long blocks_executed(KernelId k) const override;

  // Replay-only introspection used by parity tests and the GPU mirror.
  const SimKernelSpec& kernel_spec(KernelId k) const { return kernels_.at(k); }
  std::size_t atom_count() const { return atoms_.size(); }

 private:
  // Exact rational occupancy of one TPC: a resident block of a kernel with
  // occupancy o holds 1/o of the TPC.
  struct Load {
    long num = 0, den = 1;
    bool admits(int o) const { return num * o + den <= den * o; }
    void add_share(int o);
    void drop_share(int o);
  };
  struct TpcState {
    std::vector<AtomId> queue;  // resident atoms, (priority desc, seq asc)
    Load load;
    int running = 0;  // blocks in flight
  };
  struct Atom {
    KernelId kernel;
    long cursor, end;  // next block to start, one past the last
    int running = 0;
    std::vector<int> tpcs;  // sorted, duplicates kept
    int priority;
    std::uint64_t seq;
    std::uint64_t tag;
    SimTime dispatched;
    bool atomized;
    bool paused = false;
    bool finished = false;
    bool held = false;         // chained: waiting for its predecessor
    AtomId succ = kNoAtom;     // chained successor
  };
  enum class Kind : std::uint8_t { BlockDone, Clock, Call };
  struct Event {
    SimTime t;
    std::uint64_t seq;
    Kind kind;
    int tpc;
    std::uint32_t ref;  // atom id, switch generation or call slot
  };

  void push(SimTime t, Kind kind, int tpc, std::uint32_t ref);
  void account_to(SimTime t);
  void refill(int tpc);
  void launch_block(int tpc, AtomId a);
  void retire(AtomId a);

  DeviceTopology topo_;
  FrequencyDomain freq_;
  PowerModel power_;
  FreqMhz mhz_;
  std::optional<std::pair<FreqMhz, SimTime>> pending_;  // target, effective
  std::uint32_t switch_gen_ = 0;

  SimTime clock_ = 0;
  std::uint64_t seq_ = 0;
  std::vector<Event> heap_;  // binary min-heap on (t, seq)
  std::vector<std::function<void()>> calls_;
  std::vector<std::uint32_t> free_calls_;

  std::vector<TpcState> tpc_;
  int busy_tpcs_ = 0;
  std::vector<SimKernelSpec> kernels_;
  std::vector<long> executed_;
  std::vector<Atom> atoms_;
  bool held_next_ = false;  // submit_chained: the next atom starts held
  std::function<void(const AtomCompletion&)> on_complete_;

  SimTime accounted_ = 0;
  SimTime horizon_ = -1;
  double joules_ = 0.0;
  double busy_tpc_ns_ = 0.0;
  std::map<FreqMhz, Duration> residency_;
};

}  // namespace gpuos
