// Time base, device description and closed-form latency model.
// Semantics follow device.cpp:9-72 and metrics.cpp:10-18 of the reference.
#include <algorithm>
#include <cmath>

#include "gpuos/core.hpp"

namespace gpuos {

Duration duration_from_us(double us) { return std::llround(us * 1000.0); }
Duration duration_from_ms(double ms) { return std::llround(ms * 1e6); }
double duration_to_us(Duration d) { return static_cast<double>(d) / 1000.0; }
double duration_to_ms(Duration d) { return static_cast<double>(d) / 1e6; }

Duration percentile(std::vector<Duration> samples, double p) {
  if (samples.empty()) throw ConfigError("percentile of an empty sample set");
  if (!(p > 0.0 && p < 100.0))
    throw ConfigError("percentile p must be in (0,100)");
  const double n = static_cast<double>(samples.size());
  std::size_t rank = static_cast<std::size_t>(std::ceil(p / 100.0 * n));
  rank = std::max<std::size_t>(rank, 1);
  std::nth_element(samples.begin(), samples.begin() + (rank - 1),
                   samples.end());
  return samples[rank - 1];
}

void DeviceTopology::validate() const {
  if (std::min({gpc_count, tpcs_per_gpc, sms_per_tpc}) < 1)
    throw ConfigError("device topology counts must be >= 1");
}

DeviceTopology DeviceTopology::a100_like() { return DeviceTopology{6, 9, 2}; }
DeviceTopology DeviceTopology::h100_like() { return DeviceTopology{8, 9, 2}; }
// 148 SMs paired into 74 TPCs (2-CTA clusters always land on SMs {2k,2k+1}:
// profiles/topology_probe_r01.json). Physical GPCs hold 8-10 TPCs each, so a
// uniform gpc x tpcs grid cannot describe them; the two dies (37 TPCs each)
// are the GPC-like partition unit exposed for mig_like.
DeviceTopology DeviceTopology::b200() { return DeviceTopology{2, 37, 2}; }

bool FrequencyDomain::supports(FreqMhz f) const {
  return std::find(supported_mhz.begin(), supported_mhz.end(), f) !=
         supported_mhz.end();
}

void FrequencyDomain::validate() const {
  if (supported_mhz.empty()) throw ConfigError("frequency table must be non-empty");
  if (!std::is_sorted(supported_mhz.begin(), supported_mhz.end()))
    throw ConfigError("frequency table must be ascending");
  if (supported_mhz.front() <= 0) throw ConfigError("frequencies must be positive");
  if (switch_latency < 0) throw ConfigError("switch latency must be >= 0");
}

void SimKernelSpec::validate() const {
  if (total_blocks < 1) throw ConfigError("kernel needs >= 1 block");
  if (occupancy_per_tpc < 1) throw ConfigError("occupancy must be >= 1");
  if (block_duration_at_fmax <= 0) throw ConfigError("block duration must be > 0");
  if (sensitivity_s < 0.0 || sensitivity_s > 1.0)
    throw ConfigError("sensitivity must be in [0,1]");
  if (prelude_overhead < 0) throw ConfigError("prelude overhead must be >= 0");
}

double PowerModel::watts(int active_tpcs, FreqMhz f, FreqMhz f_max) const {
  const double rel = static_cast<double>(f) / static_cast<double>(f_max);
  const double dynamic = p_tpc_w * active_tpcs * std::pow(rel, alpha);
  return p_static_w + dynamic;
}

Duration block_latency(const SimKernelSpec& spec, FreqMhz f,
                       const FrequencyDomain& fd) {
  if (!fd.supports(f)) throw ConfigError("unsupported frequency");
  const double stretch =
      static_cast<double>(fd.f_max()) / static_cast<double>(f) - 1.0;
  const double factor = 1.0 + spec.sensitivity_s * stretch;
  return std::llround(static_cast<double>(spec.block_duration_at_fmax) * factor);
}

Duration reference_kernel_latency(const SimKernelSpec& spec, int t, FreqMhz f,
                                  const FrequencyDomain& fd) {
  if (t < 1) throw ConfigError("tpc count must be >= 1");
  const long per_wave = static_cast<long>(t) * spec.occupancy_per_tpc;
  const long waves = (spec.total_blocks + per_wave - 1) / per_wave;
  return waves * block_latency(spec, f, fd);
}

AtomId Device::submit_chained(AtomId, KernelId, long, long, const std::vector<int>&, int, bool,
                              std::uint64_t, bool, bool) {
  throw InvariantError("this backend does not chain kernels");
}

}  // namespace gpuos
