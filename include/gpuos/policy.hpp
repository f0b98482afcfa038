// Scheduling policy helpers of the hot path: atom planning, the online
// latency predictor, the right-sizer and the DVFS power manager.
//
// Drop-in for the reference's atomizer.hpp, predictor.hpp, rightsizer.hpp
// and power_manager.hpp (same names, signatures and semantics; file:line
// citations on each declaration point at the behaviour reproduced).
#pragma once

#include <algorithm>
#include <compare>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "gpuos/core.hpp"

namespace gpuos {

// ================================================================ atomizer
// Contiguous block range [lo, hi) of a kernel (atomizer.hpp:11-15).
struct AtomRange {
  long lo = 0;
  long hi = 0;
  long size() const { return hi - lo; }
};

// ceil(predicted/atom_duration) even contiguous ranges, count clamped to
// [1, N/min_blocks_per_atom] (atomizer.cpp:7-31).
std::vector<AtomRange> plan_atoms(long total_blocks, Duration predicted,
                                  Duration atom_duration,
                                  long min_blocks_per_atom);
// false for single-block kernels and predicted < factor * atom_duration
// (atomizer.cpp:33-40).
bool should_atomize(Duration predicted, long total_blocks,
                    Duration atom_duration, double disable_factor = 2.0);

// =============================================================== predictor
// (launch queue, ordinal within the batch) (predictor.hpp:16-20).
struct OperatorKey {
  int queue_id = 0;
  int ordinal = 0;
  auto operator<=>(const OperatorKey&) const = default;
};

struct PredictorConfig {
  double ewma_beta = 0.25;
  Duration default_unknown = 10 * kMillisecond;
};

enum class Confidence { Exact, Scaled, Unknown };

struct Prediction {
  Duration latency = 0;
  Confidence confidence = Confidence::Unknown;
};

// Lexicographic (tpc_count, freq, blocks): the nearest-config tie order.
struct ObsConfig {
  int tpc_count = 1;
  FreqMhz freq = 0;
  long blocks = 1;
  auto operator<=>(const ObsConfig&) const = default;
};

struct PredictionLogEntry {
  OperatorKey key;
  ObsConfig config;
  Duration predicted = 0;
  Duration actual = 0;
  bool high_priority = false;
  Confidence confidence = Confidence::Unknown;
};

struct MispredictionReport {
  double rate = 0.0;
  Duration p99_abs_error = 0;
  std::size_t count = 0;
};

// EWMA per (key, tpc_count, freq, blocks) with linear-scaling fallback
// (predictor.cpp:11-68). Stores are per queue.
class LatencyPredictor {
 public:
  explicit LatencyPredictor(PredictorConfig cfg = {}) : cfg_(cfg) {}

  Prediction predict(const OperatorKey& key, int tpc_count, FreqMhz f,
                     long blocks) const;
  void record(const OperatorKey& key, const ObsConfig& config,
              Duration observed);
  void batch_boundary(int queue_id);
  int next_ordinal(int queue_id);
  bool has_any(const OperatorKey& key) const;
  std::string dump_store(int queue_id) const;
  // Warm start (B200 sessions): take `other`'s learned tables, queue ids
  // mapped through `queue_map` (other's id -> this predictor's id).
  void absorb(const LatencyPredictor& other, const std::map<int, int>& queue_map);

 private:
  struct Ewma {
    double value_ns = 0.0;
    long samples = 0;
  };
  using Table = std::map<ObsConfig, Ewma>;
  PredictorConfig cfg_;
  std::map<OperatorKey, Table> tables_;
  std::map<int, int> next_ordinal_;
};

MispredictionReport misprediction_rate(
    const std::vector<PredictionLogEntry>& log,
    Duration threshold = 50 * kMicrosecond);

// ============================================================== right-sizer
// l(t) = m/t + b (rightsizer.hpp:12-16).
struct ScalingFit {
  double m_ns = 0.0;
  double b_ns = 0.0;
  bool valid = false;
  // B200 extension (0 in the reference): latency floor of the measured
  // curve, l(t) = max(m/t + b, floor_ns). HBM-bound bodies plateau once
  // enough TPCs saturate the memory system (STREAM from 48 of 74 TPCs);
  // the two-point l = m/t + b cannot see that and keeps them at full width.
  double floor_ns = 0.0;
  double at(int t) const {
    const double l = m_ns / t + b_ns;
    return floor_ns > 0.0 ? std::max(l, floor_ns) : l;
  }
};
// Three-point fit of a measured curve (B200 extension): m, b through
// (1, l1) and (t_mid, l_mid), floor = the full-width latency lT, so the
// model follows the compute-bound slope and stops at the measured plateau.
ScalingFit fit_scaling_plateau(Duration l1, int t_mid, Duration l_mid, Duration lT, int T);

ScalingFit fit_scaling(Duration l1, Duration lT, int T);      // rightsizer.cpp:8-19
int filter_cap(long total_blocks, int occupancy_per_tpc,
               int total_tpcs);                                 // :21-26
int choose_tpcs(const ScalingFit& fit, int t_alloc, double slip_k,
                int cap);                                       // :28-38
int choose_tpcs_wave(const ScalingFit& fit, int t_alloc, double slip_k,
                     long blocks, int occ);                     // :40-60

enum class ProbeDecision { UseFull, ProbeOneTpc, UseFit, ProbeWidth };

struct RightsizerConfig {
  double slip_k = 1.1;
  int probe_depth_limit = 1;
  // B200 extension (off = the reference's two probes and l = m/t + b): the
  // right-sizer works on the MEASURED curve -- after the full-width and
  // one-TPC probes it bisects the width (ProbeWidth, on quiet dispatches
  // like the one-TPC probe) between the widest measured width that misses
  // the slip budget and the narrowest one that meets it, and picks the
  // narrowest measured width within slip_k of the widest width's latency.
  // HBM-bound bodies, whose latency plateaus once enough TPCs saturate the
  // memory system, get the plateau's start; compute-bound ones keep the
  // width their measured speed-up needs.
  bool plateau = false;
};

// The measured-curve search (RightsizerConfig::plateau) over samples
// (width, mean latency): `ok` = narrowest width within slip_k of the widest
// sampled width's latency, `probe` = next width to measure (0: converged --
// the bracket [widest miss, ok] is within max(1, ok / 16) TPCs).
struct MeasuredChoice {
  int ok = 0;
  int probe = 0;
  int widest = 0;
};
MeasuredChoice choose_measured(const std::map<int, double>& mean_ns, double slip_k);

// full width -> one-TPC probe -> fitted width (rightsizer.cpp:62-103).
class Rightsizer {
 public:
  explicit Rightsizer(RightsizerConfig cfg = {}) : cfg_(cfg) {}

  ProbeDecision decide(const OperatorKey& key, int queue_depth,
                       bool slo_slack_ok) const;
  void observe(const OperatorKey& key, int tpc_count, Duration latency);
  const ScalingFit* fit_for(const OperatorKey& key) const;
  int choose(const OperatorKey& key, int t_alloc, long blocks, int occ) const;
  // Plateau mode: the next width to measure for `key` (0: none due).
  int probe_width(const OperatorKey& key) const;
  // Plateau mode: the measured-curve state of `key` (ok = 0: no samples).
  MeasuredChoice measured(const OperatorKey& key) const;
  // Warm start (B200 sessions): take `other`'s curves, queue ids mapped
  // through `queue_map` (other's id -> this scheduler's id).
  void absorb(const Rightsizer& other, const std::map<int, int>& queue_map);
  double weighted_r_squared(long* included = nullptr) const;
  const RightsizerConfig& config() const { return cfg_; }

 private:
  struct Curve {
    std::map<int, std::pair<double, long>> samples;  // t -> (sum ns, count)
    int wide_t = 0;
    Duration wide_ns = 0;
    Duration one_ns = 0;
    bool has_wide = false;
    bool has_one = false;
    ScalingFit fit;
  };
  RightsizerConfig cfg_;
  std::map<OperatorKey, Curve> curves_;
};

double r_squared(const ScalingFit& fit,
                 const std::vector<std::pair<int, double>>& points);

// ============================================================ power manager
double sensitivity(Duration lat_fth, Duration lat_fmax, FreqMhz f_th,
                   FreqMhz f_max);                              // power_manager.cpp:8-17
double aggregate_sensitivity(
    const std::vector<std::pair<double, double>>& ws);          // :19-25
FreqMhz select_frequency(double S, double slip_k, FreqMhz f_max,
                         const std::vector<FreqMhz>& supported,
                         double s_floor = 1e-6);                // :27-37

enum class DvfsPhase { Unseen, Probing, Confirmed };

struct SensitivityRecord {
  DvfsPhase phase = DvfsPhase::Unseen;
  double s = 1.0;
  double last_probe_s = -1.0;
  Duration baseline_fmax = 0;
  Duration runtime_last_batch = 0;
};

struct DvfsConfig {
  double slip_k = 0.1;
  double confirm_tolerance = 0.05;
};

// Per-app frequency planning (power_manager.cpp:39-122).
class PowerManager {
 public:
  PowerManager(DvfsConfig cfg, std::vector<FreqMhz> supported);

  void observe(const OperatorKey& key, Duration latency, FreqMhz f);
  FreqMhz plan_batch(int queue_id);
  DvfsPhase phase(const OperatorKey& key) const;
  double estimate(const OperatorKey& key) const;
  long frequency_requests() const { return requests_; }
  static FreqMhz arbitrate(const std::vector<FreqMhz>& app_targets);

 private:
  FreqMhz top() const { return table_.back(); }
  DvfsConfig cfg_;
  std::vector<FreqMhz> table_;
  std::map<OperatorKey, SensitivityRecord> records_;
  std::map<int, FreqMhz> last_target_;
  long requests_ = 0;
};

}  // namespace gpuos
