// gpuos core: time base, errors, device description and the device seam.
//
// Drop-in for the reference's types.hpp (types.hpp:12-38) and the public
// surface of device.hpp (device.hpp:14-121). The reference has one concrete
// DeviceEngine; here the seam the Scheduler drives is the abstract `Device`
// so that two backends can sit behind it:
//   * DeviceEngine  (gpuos/replay.hpp) — deterministic replay with the
//     reference's wave/slot timing, bit-exact dispatch/completion logs;
//   * B200Device    (gpuos/b200.hpp)   — live execution on the sm_100a
//     persistent TPC dispatcher through the C ABI in include/gpuos_dev.h.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace gpuos {

// ---------------------------------------------------------------- time base
// Integer nanoseconds everywhere (types.hpp:12-13).
using SimTime = std::int64_t;
using Duration = std::int64_t;
using FreqMhz = int;

constexpr Duration kNanosecond = 1;
constexpr Duration kMicrosecond = 1000;
constexpr Duration kMillisecond = 1000 * kMicrosecond;
constexpr Duration kSecond = 1000 * kMillisecond;

// Rounded with llround, as device.cpp:9-14.
Duration duration_from_us(double us);
Duration duration_from_ms(double ms);
double duration_to_us(Duration d);
double duration_to_ms(Duration d);

// ------------------------------------------------------------------- errors
// ConfigError -> exit 2, InvariantError -> exit 3 (types.hpp:26-38).
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};
class InvariantError : public std::runtime_error {
 public:
  explicit InvariantError(const std::string& what) : std::runtime_error(what) {}
};

// Nearest-rank percentile, sorted[ceil(p/100*n)-1] (metrics.cpp:10-18).
Duration percentile(std::vector<Duration> samples, double p);

// ------------------------------------------------------- device description
struct DeviceTopology {
  int gpc_count = 1;
  int tpcs_per_gpc = 1;
  int sms_per_tpc = 2;

  int total_tpcs() const { return gpc_count * tpcs_per_gpc; }
  void validate() const;

  static DeviceTopology a100_like();  // 6 x 9 TPCs (device.cpp:23)
  static DeviceTopology h100_like();  // 8 x 9 TPCs (device.cpp:24)
  static DeviceTopology b200();       // 74 TPCs, 148 SMs (probed: profiles/)
};

struct FrequencyDomain {
  std::vector<FreqMhz> supported_mhz;  // ascending
  Duration switch_latency = 50 * kMillisecond;

  FreqMhz f_max() const { return supported_mhz.back(); }
  FreqMhz f_min() const { return supported_mhz.front(); }
  bool supports(FreqMhz f) const;
  void validate() const;
};

// What one block of a kernel does on the B200 (ignored by the replay
// engine). The reference's kernels are pure cost descriptors; live tenants
// also name a body and the workspace it runs over.
enum class BodyKind : std::uint32_t {
  None = 0,      // no device work (replay-only descriptors)
  Stream = 1,    // HBM-bound streaming transform, bytes_per_block per block
  GemmBf16 = 2,  // bf16 GEMM on tcgen05, one 256 x 256 output tile per block
  Spin = 3,      // fixed-duration compute spin (calibration / control)
  GemvBf16 = 4,  // decode GEMV (HBM-bound), 256 rows of W per block
  ConvBf16 = 5,  // NHWC implicit-GEMM convolution on tcgen05
  // Tenant-supplied bodies (include/gpuos_body.cuh, csrc/bodies): the device
  // id comes from gpuos_dev_body_id by name.
  RmsNormBf16 = 6,  // p = [rows, d]: one row per block
  SiluMulBf16 = 7,  // p = [n, chunk]: ceil(n / chunk) blocks
  AttnDecodeBf16 = 8,  // p = [ctx, chunk]: GQA decode attention, 8 x ceil(ctx / chunk) blocks
};

struct BodyRef {
  BodyKind kind = BodyKind::None;
  std::uint32_t workspace = 0;  // tenant workspace slot (buffers reused)
  std::int64_t p0 = 0, p1 = 0, p2 = 0;  // body parameters (see b200.hpp)
  std::int64_t px[7] = {0, 0, 0, 0, 0, 0, 0};  // parameters 3..9 (conv shapes)
  std::int64_t param(int i) const { return i == 0 ? p0 : i == 1 ? p1 : i == 2 ? p2 : px[i - 3]; }
  void set_param(int i, std::int64_t v) {
    if (i == 0) p0 = v;
    else if (i == 1) p1 = v;
    else if (i == 2) p2 = v;
    else px[i - 3] = v;
  }
  static constexpr int kParams = 10;
};

// Ground truth for one kernel launch (device.hpp:39-47).
struct SimKernelSpec {
  long total_blocks = 1;
  Duration block_duration_at_fmax = kMillisecond;
  double sensitivity_s = 1.0;
  int occupancy_per_tpc = 1;
  Duration prelude_overhead = 500;  // charged per block when atomized
  BodyRef body;                     // live backend only

  void validate() const;
};

struct PowerModel {
  double p_static_w = 50.0;
  double p_tpc_w = 5.0;
  double alpha = 2.0;

  double watts(int active_tpcs, FreqMhz f, FreqMhz f_max) const;
};

// d0 * (1 + s * (f_max/f - 1)) rounded to ns (device.cpp:56-64).
Duration block_latency(const SimKernelSpec& spec, FreqMhz f,
                       const FrequencyDomain& fd);
// ceil(N / (t * occ)) waves x block latency (device.cpp:66-72).
Duration reference_kernel_latency(const SimKernelSpec& spec, int t, FreqMhz f,
                                  const FrequencyDomain& fd);

using KernelId = std::uint32_t;
using AtomId = std::uint32_t;
constexpr AtomId kNoAtom = 0xffffffffu;

struct AtomCompletion {
  AtomId atom;
  std::uint64_t tag;
  SimTime dispatch_time;
  SimTime complete_time;
};

// --------------------------------------------------------------- the seam
// Every member the Scheduler uses (SURVEY.md §1 "Where the hot path sits")
// plus the metrics accessors run_scenario reads. One logical owner thread
// drives a Device; completions are delivered synchronously from step().
class Device {
 public:
  virtual ~Device() = default;

  virtual SimTime now() const = 0;
  virtual const DeviceTopology& topology() const = 0;
  virtual const FrequencyDomain& freq_domain() const = 0;
  virtual FreqMhz current_mhz() const = 0;

  virtual KernelId register_kernel(const SimKernelSpec& spec) = 0;
  virtual AtomId submit_atom(KernelId kernel, long lo, long hi,
                             const std::vector<int>& tpcs, int priority,
                             bool atomized, std::uint64_t tag) = 0;
  virtual void set_atom_paused(AtomId atom, bool paused) = 0;
  virtual SimTime request_frequency(FreqMhz f) = 0;
  virtual void schedule_call(SimTime t, std::function<void()> fn) = 0;
  virtual void set_atom_complete_handler(
      std::function<void(const AtomCompletion&)> h) = 0;

  virtual bool step() = 0;
  virtual void run_all() = 0;

  virtual void set_metrics_horizon(SimTime t) = 0;
  virtual double energy_joules() const = 0;
  virtual double tpc_busy_integral() const = 0;
  virtual const std::map<FreqMhz, Duration>& freq_residency() const = 0;
  virtual long blocks_executed(KernelId k) const = 0;

  // Live-backend hook: the owner of `tpc` has (or no longer has) pending
  // work, so blocks of atoms below `min_priority` must stop starting there
  // (block-granular revocation). The replay backend models the reference,
  // which revokes only at atom boundaries, and ignores it.
  // Block-granular revocation (live extension): on these TPCs only atoms
  // of `owner_tag` (the owning tenant's submit tag) or of priority >=
  // min_priority start new blocks (min_priority 0 lifts the fence).
  virtual void set_tpc_fence(const std::vector<int>& /*tpcs*/, int /*min_priority*/,
                             std::uint64_t /*owner_tag*/) {}
  // Pair fence (live extension): on these TPCs only the worker pairs in
  // `pair_slots` (bit i: the TPC's i-th pair) refuse blocks below
  // min_priority; the others accept every atom (0 lifts).
  virtual void set_pair_fence(const std::vector<int>& /*tpcs*/, unsigned /*pair_slots*/,
                              int /*min_priority*/) {}
  // Live-backend hook: true when TPCs holding only foreign stolen atoms may
  // be handed back to their owner immediately (device priority arbitration
  // preempts at the next block boundary).
  virtual bool preempts_stolen() const { return false; }
  // Live-backend hook: kernel chaining. submit_chained() posts an atom that
  // the device arms itself when atom `after` completes (kNoAtom: at once);
  // `chain_head` lets a later atom be chained behind this one. Completions
  // still arrive in chain order. Backends without it never see the call.
  virtual bool supports_chaining() const { return false; }
  // `no_early`: a tensor-core successor must not start its weight loads
  // before `after` completes (the predecessor may run for seconds).
  virtual AtomId submit_chained(AtomId after, KernelId kernel, long lo, long hi,
                                const std::vector<int>& tpcs, int priority,
                                bool atomized, std::uint64_t tag, bool chain_head,
                                bool no_early = false);
};

}  // namespace gpuos
