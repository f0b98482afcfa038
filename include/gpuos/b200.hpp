// Live B200 backend of the device seam (and the GPU mirror used for replay
// verification), built on the C ABI in include/gpuos_dev.h.
//
//   B200Device  — the Scheduler's Device on a real B200: submit_atom posts
//                 the atom to the persistent sm_100a dispatcher; completions
//                 come back through the device->host ring; time is the host
//                 steady clock (ns since the run started). One run_all() is
//                 one dispatcher lifetime (start .. drain), timed with CUDA
//                 events.
//   MirrorDevice— deterministic replay timing (bit-exact with the reference)
//                 while every atom is also executed on the B200 on exactly
//                 the TPC set the replay chose; verify() checks per-block
//                 exactly-once execution, placement inside the atom's TPC
//                 set, and the body outputs.
//
// Bodies. A KernelRecord names its body (core.hpp BodyRef):
//   Stream: p0 = u32 words per block, p1 = salt (0: derived from kernel id),
//           p2 = distinct chunks (0: min(blocks, stream_chunk_cap));
//           workspace = buffer-pair slot shared by kernels of a tenant.
//   Spin:   p0 = ns per block.
//   GemmBf16: p = [M, N, K]; GemvBf16: p = [N, K, k_splits];
//   ConvBf16: p = [n, h, w, c, k, r, s, pad, stride]. Operands are random
//           bf16 per (workspace, shape), bf16 outputs; the kernel's grid
//           must equal the descriptor's (256 x 256 tiles / 256-row tiles).
//   None:   the reference's cost-only kernels; synthesised per
//           B200Options::synth (Stream sized from block_us, or Spin).
#pragma once

#include <array>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <queue>
#include <unordered_map>
#include <vector>

#include "gpuos/core.hpp"
#include "gpuos/replay.hpp"

struct gpuos_dev;

namespace gpuos {

struct B200Options {
  int device = 0;
  int workers_per_sm = 2;
  int idle_sleep_ns = 128;
  bool trace_blocks = false;        // per-block execution trace (verification)
  enum class Synth { Stream, Spin } synth = Synth::Stream;
  double stream_words_per_us = 2750.0;  // None -> Stream sizing (per worker)
  long stream_min_words = 256;
  long stream_chunk_cap = 4096;     // bound on distinct chunks per workspace
  // Preemption quantum: blocks longer than this run as independently
  // claimed slices, bounding how long a higher-priority atom waits for a
  // worker slot (0: whole blocks).
  std::int64_t quantum_ns = 0;
  // DVFS actuation: request_frequency() locks the SM clock (NVML) to the
  // power manager's choice. Off by default -- never on a pool whose
  // operator manages clocks.
  bool dvfs_actuate = false;
  // Live-run watchdog: no atom completion for this long while atoms are in
  // flight raises InvariantError with the device state (0: off).
  std::int64_t stall_timeout_ns = 20'000'000'000;
};

struct AtomTimeline {
  AtomId atom;
  std::uint64_t tag;
  KernelId kernel;
  long lo, hi;
  int priority;
  std::int64_t host_submit_ns, host_complete_ns;
  std::int64_t dev_first_start_ns, dev_last_end_ns;
  std::int64_t dev_ingest_ns, dev_armed_ns;  // ingest warp saw / armed the atom
  std::uint64_t touched[2];
  std::uint64_t mask[2];
};

struct VerifyReport {
  long kernels = 0;
  long blocks = 0;
  long missing = 0;      // blocks never executed
  long duplicated = 0;   // blocks executed more than once
  long misplaced = 0;    // blocks run on an SM outside the atom's TPC set
  long bad_words = 0;    // body output words differing from the oracle
  long checked_words = 0;
  // Tensor-core bodies (GEMM / GEMV / conv): sampled output elements of every
  // fully executed kernel against a float64 restatement of the same bf16
  // operands (tolerance: one bf16 rounding of the result plus fp32
  // accumulation, 2^-8 |ref| + 1e-5 sum |a b|).
  long tensor_kernels = 0;
  long tensor_checked = 0;
  long tensor_bad = 0;
  bool ok() const {
    return missing == 0 && duplicated == 0 && misplaced == 0 && bad_words == 0 && tensor_bad == 0;
  }
};

// Owns one dispatcher handle plus the tenant workspaces.
class B200Runtime {
 public:
  B200Runtime(int logical_tpcs, const B200Options& opt);
  ~B200Runtime();
  B200Runtime(const B200Runtime&) = delete;
  B200Runtime& operator=(const B200Runtime&) = delete;

  gpuos_dev* handle() const { return dev_; }
  const B200Options& options() const { return opt_; }
  int logical_tpcs() const { return tpcs_; }
  int workers_per_tpc() const;

  // Resolves a kernel's body into dispatcher arguments (allocating its
  // workspace on first use).
  struct Resolved {
    std::uint32_t body;
    std::uint64_t args[5];
    std::uint32_t* trace;   // indexed block * parts + part
    long words;  // Stream: words per block
    long chunks;
    std::uint32_t parts;    // preemption slices per block
  };
  Resolved resolve(KernelId kid, const SimKernelSpec& spec);
  // Allocates (and initialises) whatever the body needs without binding it
  // to a kernel id: called for every kernel of a scenario before the
  // dispatcher starts, so no allocation or fill kernel runs beside it.
  void prepare(const SimKernelSpec& spec) { (void)resolve_body(spec); }
  // Records a kernel's workspace need without allocating: called for every
  // kernel before prepare(), so a workspace shared by kernels of different
  // sizes is allocated once at the largest.
  void reserve(const SimKernelSpec& spec);

  void start();
  float stop(bool drain);  // returns the worker kernel's CUDA-event ms
  // Forget per-run kernel bindings (workspaces stay allocated and resident).
  void reset_kernels();
  // Body-resolution options (quantum, tracing, synthesis) may change between
  // runs; device, workers_per_sm and idle_sleep_ns are fixed at open.
  bool set_run_options(const B200Options& o);
  bool running() const { return running_; }

  // Verification against a CPU restatement of the bodies.
  struct KernelPlacement {  // blocks of one kernel -> allowed TPC masks
    std::vector<std::pair<long, long>> ranges;
    std::vector<std::array<std::uint64_t, 2>> masks;
  };
  VerifyReport verify_kernels(const std::vector<SimKernelSpec>& specs,
                              const std::vector<KernelPlacement>& placement);

  // Host copies of workspace inputs for the end-to-end path.
  std::uint64_t upload_inputs();   // H2D of every workspace source; bytes
  std::uint64_t download_digest(); // D2H of a per-workspace digest; bytes
  std::uint64_t workspace_bytes() const;

 private:
  struct Workspace {
    std::uint32_t* src = nullptr;
    std::uint32_t* dst = nullptr;
    std::uint64_t words = 0;  // capacity of each buffer
    std::uint32_t* host_src = nullptr;  // pinned tenant input
  };
  Workspace& workspace(std::uint32_t id, std::uint64_t words);
  Resolved resolve_body(const SimKernelSpec& spec);
  struct TensorBody {  // operands + descriptor of a tensor-core kernel shape
    std::vector<void*> bufs;  // gemm: A, B, C; gemv: W, x, y; conv: x, w, y
    void* desc = nullptr;
    std::int64_t blocks = 0;
    std::uint32_t body = 0;          // device body id (tenant bodies)
    std::uint64_t args[5] = {0, 0, 0, 0, 0};  // tenant bodies' atom args
    BodyRef ref;              // kind + shape (verify_kernels)
  };
  // Sampled float64 check of a tensor body's output (verify_kernels).
  void verify_tensor(const TensorBody& t, VerifyReport& rep);
  std::unordered_map<std::uint64_t, const TensorBody*> tensor_of_desc_;
  const TensorBody& tensor_body(const BodyRef& b);
  std::map<std::string, TensorBody> tensors_;
  void ensure_trace(KernelId kid, long blocks);

  gpuos_dev* dev_ = nullptr;
  B200Options opt_;
  int tpcs_ = 0;
  bool running_ = false;
  std::unordered_map<std::uint32_t, Workspace> ws_;
  std::unordered_map<std::uint32_t, std::uint64_t> ws_reserve_;  // words, from reserve()
  std::vector<std::uint32_t*> trace_of_;  // per kernel id
  // Trace pool: fixed-size chunks kept across runs (allocating during a
  // live run would stall it), zeroed between runs.
  static constexpr std::uint64_t kTraceChunkWords = 16ull << 20;
  std::vector<std::uint32_t*> trace_chunks_;
  std::vector<std::uint64_t> trace_chunk_words_;
  std::size_t trace_chunk_ = 0;           // chunk being filled
  std::uint64_t trace_pool_used_ = 0;     // words used in it
  std::vector<Resolved> resolved_;        // per kernel id
  std::vector<char> has_resolved_;
};

class B200Device final : public Device {
 public:
  B200Device(DeviceTopology topo, FrequencyDomain freq, B200Options opt = {});
  ~B200Device() override;

  SimTime now() const override { return now_; }
  const DeviceTopology& topology() const override { return topo_; }
  const FrequencyDomain& freq_domain() const override { return freq_; }
  FreqMhz current_mhz() const override { return freq_.f_max(); }

  KernelId register_kernel(const SimKernelSpec& spec) override;
  AtomId submit_atom(KernelId kernel, long lo, long hi,
                     const std::vector<int>& tpcs, int priority, bool atomized,
                     std::uint64_t tag) override;
  void set_atom_paused(AtomId atom, bool paused) override;
  SimTime request_frequency(FreqMhz f) override;  // no clock actuation: SPEC.md out of scope
  void schedule_call(SimTime t, std::function<void()> fn) override;
  void set_atom_complete_handler(std::function<void(const AtomCompletion&)> h) override {
    on_complete_ = std::move(h);
  }
  bool step() override;
  void run_all() override;

  void set_metrics_horizon(SimTime t) override { horizon_ = t; }
  // GPU energy counter (NVML) over the last run_all(); 0 without NVML.
  double energy_joules() const override { return energy_j_; }
  // NVML samples at the end of the last run_all() (0 without NVML).
  unsigned last_sm_mhz() const { return sm_mhz_; }
  unsigned last_power_mw() const { return power_mw_; }
  double tpc_busy_integral() const override { return busy_tpc_ns_; }
  const std::map<FreqMhz, Duration>& freq_residency() const override { return residency_; }
  long blocks_executed(KernelId k) const override { return executed_.at(k); }

  void set_tpc_fence(const std::vector<int>& tpcs, int min_priority, std::uint64_t owner_tag) override;
  void set_pair_fence(const std::vector<int>& tpcs, unsigned pair_slots, int min_priority) override;
  bool preempts_stolen() const override { return true; }
  bool supports_chaining() const override { return true; }
  AtomId submit_chained(AtomId after, KernelId kernel, long lo, long hi,
                        const std::vector<int>& tpcs, int priority, bool atomized,
                        std::uint64_t tag, bool chain_head, bool no_early = false) override;

  B200Runtime& runtime() { return *rt_; }
  // Clears per-run state so one device (and its workspaces) serves many runs.
  void reset_run();
  const std::vector<AtomTimeline>& timeline() const { return timeline_; }
  float last_kernel_ms() const { return last_ms_; }
  std::int64_t run_wall_ns() const { return run_wall_ns_; }
  const std::vector<SimKernelSpec>& kernels() const { return kernels_; }
  // submit_atom calls that found a TPC's resident list (32) or the atom
  // table full and waited for completions (last run).
  std::int64_t backpressure_waits() const { return backpressure_waits_; }

 private:
  SimTime host_now() const;
  void pump();

  SimTime last_progress_ns_ = 0;  // host time of the last completion (watchdog)
  double energy_j_ = 0.0;
  unsigned sm_mhz_ = 0, power_mw_ = 0;
  FreqMhz locked_mhz_ = 0;  // dvfs_actuate: clock currently locked (0: none)
  B200Options opt_;
  DeviceTopology topo_;
  FrequencyDomain freq_;
  std::unique_ptr<B200Runtime> rt_;
  SimTime now_ = 0;
  std::int64_t origin_ = 0;  // gpuos_dev_now_ns at run start
  struct Timer {
    SimTime t;
    std::uint64_t seq;
    bool operator>(const Timer& o) const { return t != o.t ? t > o.t : seq > o.seq; }
  };
  std::priority_queue<Timer, std::vector<Timer>, std::greater<Timer>> timers_;
  std::unordered_map<std::uint64_t, std::function<void()>> timer_fns_;
  std::uint64_t timer_seq_ = 0;
  std::vector<SimKernelSpec> kernels_;
  std::vector<long> executed_;
  std::unordered_map<AtomId, std::size_t> atom_index_;  // -> timeline_
  std::vector<AtomTimeline> timeline_;
  std::deque<AtomCompletion> ready_;
  std::function<void(const AtomCompletion&)> on_complete_;
  SimTime horizon_ = -1;
  double busy_tpc_ns_ = 0.0;
  std::int64_t backpressure_waits_ = 0;
  std::map<FreqMhz, Duration> residency_;
  float last_ms_ = 0.f;
  std::int64_t run_wall_ns_ = 0;
};

// Replay timing + execution of every atom on the B200 (verification mode).
class MirrorDevice final : public Device {
 public:
  MirrorDevice(DeviceTopology topo, FrequencyDomain freq, PowerModel power,
               B200Options opt = {});
  ~MirrorDevice() override;

  SimTime now() const override { return replay_.now(); }
  const DeviceTopology& topology() const override { return replay_.topology(); }
  const FrequencyDomain& freq_domain() const override { return replay_.freq_domain(); }
  FreqMhz current_mhz() const override { return replay_.current_mhz(); }
  KernelId register_kernel(const SimKernelSpec& spec) override;
  AtomId submit_atom(KernelId kernel, long lo, long hi, const std::vector<int>& tpcs,
                     int priority, bool atomized, std::uint64_t tag) override;
  void set_atom_paused(AtomId atom, bool paused) override { replay_.set_atom_paused(atom, paused); }
  SimTime request_frequency(FreqMhz f) override { return replay_.request_frequency(f); }
  void schedule_call(SimTime t, std::function<void()> fn) override {
    replay_.schedule_call(t, std::move(fn));
  }
  void set_atom_complete_handler(std::function<void(const AtomCompletion&)> h) override {
    replay_.set_atom_complete_handler(std::move(h));
  }
  bool step() override { return replay_.step(); }
  void run_all() override;
  void set_metrics_horizon(SimTime t) override { replay_.set_metrics_horizon(t); }
  double energy_joules() const override { return replay_.energy_joules(); }
  double tpc_busy_integral() const override { return replay_.tpc_busy_integral(); }
  const std::map<FreqMhz, Duration>& freq_residency() const override {
    return replay_.freq_residency();
  }
  long blocks_executed(KernelId k) const override { return replay_.blocks_executed(k); }

  // Drains the GPU and checks every mirrored block.
  VerifyReport verify();
  long gpu_atoms() const { return gpu_atoms_; }
  float gpu_kernel_ms() const { return gpu_ms_; }
  B200Runtime& runtime() { return *rt_; }

 private:
  void drain_some(bool all);

  DeviceEngine replay_;
  std::unique_ptr<B200Runtime> rt_;
  std::vector<SimKernelSpec> specs_;
  std::vector<B200Runtime::KernelPlacement> placement_;
  long gpu_atoms_ = 0;
  float gpu_ms_ = 0.f;
  bool verified_ = false;
};

}  // namespace gpuos
