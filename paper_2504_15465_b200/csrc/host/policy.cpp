// Hot-path policy helpers: atomizer, latency predictor, right-sizer and
// power manager. Every function reproduces the reference arithmetic
// exactly (same operand order, same rounding) because its outputs feed the
// bit-exact dispatch/completion log; see the file:line tags per function.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <sstream>

#include "gpuos/policy.hpp"

namespace gpuos {

// ------------------------------------------------------------ atomizer.cpp
std::vector<AtomRange> plan_atoms(long total_blocks, Duration predicted,
                                  Duration atom_duration,
                                  long min_blocks_per_atom) {  // :7-31
  if (total_blocks < 1) throw ConfigError("total_blocks must be >= 1");
  long pieces = 1;
  if (predicted > 0 && atom_duration > 0)
    pieces = (predicted + atom_duration - 1) / atom_duration;
  const long most =
      min_blocks_per_atom > 1
          ? std::max(1L, total_blocks / min_blocks_per_atom)
          : total_blocks;
  pieces = std::clamp(pieces, 1L, most);

  const long base = total_blocks / pieces;
  const long extra = total_blocks % pieces;  // leading atoms get one more
  std::vector<AtomRange> out(static_cast<std::size_t>(pieces));
  long at = 0;
  for (long i = 0; i < pieces; ++i) {
    const long len = base + (i < extra ? 1 : 0);
    out[static_cast<std::size_t>(i)] = AtomRange{at, at + len};
    at += len;
  }
  return out;
}

bool should_atomize(Duration predicted, long total_blocks,
                    Duration atom_duration, double disable_factor) {  // :33-40
  if (total_blocks <= 1) return false;
  return !(static_cast<double>(predicted) <
           disable_factor * static_cast<double>(atom_duration));
}

// ----------------------------------------------------------- predictor.cpp
Prediction LatencyPredictor::predict(const OperatorKey& key, int tpc_count,
                                     FreqMhz f, long blocks) const {  // :11-45
  if (tpc_count < 1) throw ConfigError("tpc_count must be >= 1");
  auto it = tables_.find(key);
  if (it == tables_.end() || it->second.empty())
    return Prediction{cfg_.default_unknown, Confidence::Unknown};
  const Table& table = it->second;
  if (auto hit = table.find(ObsConfig{tpc_count, f, blocks}); hit != table.end())
    return Prediction{std::llround(hit->second.value_ns), Confidence::Exact};

  // Nearest recorded configuration: a frequency mismatch costs 4, a TPC
  // mismatch 2, a block-count mismatch 1; the first minimum in map order wins.
  const ObsConfig* near = nullptr;
  const Ewma* near_cell = nullptr;
  int best = 8;
  for (const auto& [c, cell] : table) {
    const int cost = (c.freq != f ? 4 : 0) + (c.tpc_count != tpc_count ? 2 : 0) +
                     (c.blocks != blocks ? 1 : 0);
    if (cost < best) {
      best = cost;
      near = &c;
      near_cell = &cell;
    }
  }
  double est = near_cell->value_ns;
  est *= static_cast<double>(near->tpc_count) / tpc_count;
  est *= static_cast<double>(blocks) / static_cast<double>(near->blocks);
  est *= static_cast<double>(near->freq) / static_cast<double>(f);
  return Prediction{std::llround(est), Confidence::Scaled};
}

void LatencyPredictor::record(const OperatorKey& key, const ObsConfig& config,
                              Duration observed) {  // :47-57
  if (observed <= 0) throw ConfigError("observed latency must be > 0");
  Ewma& e = tables_[key][config];
  const double x = static_cast<double>(observed);
  e.value_ns = e.samples == 0
                   ? x
                   : (1.0 - cfg_.ewma_beta) * e.value_ns + cfg_.ewma_beta * x;
  ++e.samples;
}

void LatencyPredictor::batch_boundary(int queue_id) {  // :59
  next_ordinal_[queue_id] = 0;
}

int LatencyPredictor::next_ordinal(int queue_id) {  // :61-63
  return next_ordinal_[queue_id]++;
}

bool LatencyPredictor::has_any(const OperatorKey& key) const {  // :65-68
  auto it = tables_.find(key);
  return it != tables_.end() && !it->second.empty();
}

std::string LatencyPredictor::dump_store(int queue_id) const {  // :70-81
  std::ostringstream os;
  for (const auto& [key, table] : tables_) {
    if (key.queue_id != queue_id) continue;
    for (const auto& [c, e] : table)
      os << key.queue_id << ' ' << key.ordinal << ' ' << c.tpc_count << ' '
         << c.freq << ' ' << c.blocks << ' ' << std::llround(e.value_ns) << ' '
         << e.samples << '\n';
  }
  return os.str();
}

MispredictionReport misprediction_rate(
    const std::vector<PredictionLogEntry>& log, Duration threshold) {  // :83-99
  if (log.empty()) throw ConfigError("misprediction rate of an empty log");
  std::vector<Duration> err;
  err.reserve(log.size());
  std::size_t over = 0;
  for (const PredictionLogEntry& e : log) {
    const Duration d = std::llabs(e.predicted - e.actual);
    err.push_back(d);
    over += d > threshold ? 1 : 0;
  }
  MispredictionReport r;
  r.count = log.size();
  r.rate = static_cast<double>(over) / static_cast<double>(log.size());
  r.p99_abs_error = percentile(std::move(err), 99.0);
  return r;
}

// ---------------------------------------------------------- rightsizer.cpp
ScalingFit fit_scaling(Duration l1, Duration lT, int T) {  // :8-19
  if (T < 2) throw ConfigError("fit needs T >= 2");
  if (l1 <= 0 || lT <= 0) throw ConfigError("fit latencies must be > 0");
  const double one = static_cast<double>(l1);
  const double wide = static_cast<double>(lT);
  ScalingFit f;
  f.m_ns = (one - wide) / (1.0 - 1.0 / static_cast<double>(T));
  f.b_ns = one - f.m_ns;
  f.valid = l1 >= lT && f.b_ns >= 0.0;
  return f;
}

ScalingFit fit_scaling_plateau(Duration l1, int t_mid, Duration l_mid, Duration lT, int T) {
  if (t_mid < 2) throw ConfigError("plateau fit needs t_mid >= 2");
  if (l1 <= 0 || l_mid <= 0 || lT <= 0) throw ConfigError("fit latencies must be > 0");
  if (l1 < l_mid) return fit_scaling(l1, lT, T);  // no speed-up to 1..t_mid: two-point
  ScalingFit f = fit_scaling(l1, l_mid, t_mid);
  if (f.b_ns < 0.0) {  // (super-linear to t_mid: pure m/t through the mid point)
    f.b_ns = 0.0;
    f.m_ns = static_cast<double>(l_mid) * t_mid;
  }
  f.valid = true;
  f.floor_ns = static_cast<double>(std::min(l_mid, lT));
  return f;
}

int filter_cap(long total_blocks, int occupancy_per_tpc, int total_tpcs) {  // :21-26
  if (total_blocks < 1 || occupancy_per_tpc < 1)
    throw ConfigError("filter_cap inputs must be >= 1");
  const long waves1 = (total_blocks + occupancy_per_tpc - 1) / occupancy_per_tpc;
  return static_cast<int>(std::clamp<long>(waves1, 1, total_tpcs));
}

int choose_tpcs(const ScalingFit& fit, int t_alloc, double slip_k, int cap) {  // :28-38
  if (t_alloc < 1) throw ConfigError("t_alloc must be >= 1");
  if (slip_k < 1.0) throw ConfigError("slip_k must be >= 1");
  const int t_full = std::min(t_alloc, cap);
  if (!fit.valid) return t_full;
  if (fit.m_ns <= 0.0) return 1;
  const double budget = slip_k * (fit.m_ns / t_full + fit.b_ns);
  if (budget <= fit.b_ns) return t_full;
  const int t = static_cast<int>(std::ceil(fit.m_ns / (budget - fit.b_ns)));
  return std::clamp(t, 1, t_full);
}

int choose_tpcs_wave(const ScalingFit& fit, int t_alloc, double slip_k,
                     long blocks, int occ) {  // :40-60
  if (blocks < 1 || occ < 1) throw ConfigError("blocks and occ must be >= 1");
  const int t_full = std::min(t_alloc, filter_cap(blocks, occ, t_alloc));
  if (!fit.valid) return t_full;
  const long max_waves = (blocks + occ - 1) / occ;
  if (fit.m_ns <= 0.0) return static_cast<int>(std::min<long>(t_full, max_waves));
  // (floor_ns is 0 for the reference's fit: at(t) = m/t + b exactly.)
  const double budget = slip_k * fit.at(t_full);
  // Measured plateau well above the compute curve at full width: the body
  // is bound by a shared resource (HBM), not by its TPCs' throughput, so
  // block waves do not set its latency -- the smallest width whose compute
  // part fits the budget is where the plateau starts.
  if (fit.floor_ns > 0.0 && fit.floor_ns > 1.02 * (fit.m_ns / t_full + fit.b_ns) && budget > fit.b_ns) {
    const int t = static_cast<int>(std::ceil(fit.m_ns / (budget - fit.b_ns)));
    return std::clamp(t, 1, t_full);
  }
  // Walk wave counts upward; only breakpoint widths change latency.
  int chosen = t_full;
  for (long waves = 1; waves <= max_waves; ++waves) {
    const long per_wave = (blocks + waves - 1) / waves;
    const int width = static_cast<int>((per_wave + occ - 1) / occ);
    if (width > t_full) continue;
    if (fit.at(width) > budget) break;
    chosen = width;
    if (width == 1) break;
  }
  return chosen;
}

ProbeDecision Rightsizer::decide(const OperatorKey& key, int queue_depth,
                                 bool slo_slack_ok) const {  // :62-72
  auto it = curves_.find(key);
  if (it == curves_.end() || !it->second.has_wide) return ProbeDecision::UseFull;
  const bool quiet = queue_depth < cfg_.probe_depth_limit && slo_slack_ok;
  if (cfg_.plateau) {  // measured-curve search (B200 extension)
    const MeasuredChoice mc = measured(key);
    if (mc.probe == 0 || !quiet) return ProbeDecision::UseFit;
    return mc.probe == 1 ? ProbeDecision::ProbeOneTpc : ProbeDecision::ProbeWidth;
  }
  if (it->second.has_one) return ProbeDecision::UseFit;
  return quiet ? ProbeDecision::ProbeOneTpc : ProbeDecision::UseFull;
}

MeasuredChoice choose_measured(const std::map<int, double>& mean_ns, double slip_k) {
  MeasuredChoice mc;
  if (mean_ns.empty()) return mc;
  mc.widest = mean_ns.rbegin()->first;
  const double budget = slip_k * mean_ns.rbegin()->second;
  mc.ok = mc.widest;
  for (const auto& [t, l] : mean_ns)
    if (l <= budget) {
      mc.ok = t;
      break;
    }
  int miss = 0;  // widest measured width below `ok` that misses the budget
  for (const auto& [t, l] : mean_ns)
    if (t < mc.ok && l > budget) miss = t;
  if (mc.ok == 1) return mc;
  if (miss == 0) {
    mc.probe = 1;  // the one-TPC probe first (as the reference)
    return mc;
  }
  if (mc.ok - miss > std::max(1, mc.ok / 16)) mc.probe = (miss + mc.ok) / 2;
  return mc;
}

MeasuredChoice Rightsizer::measured(const OperatorKey& key) const {
  auto it = curves_.find(key);
  if (it == curves_.end()) return {};
  std::map<int, double> mean;
  for (const auto& [t, s] : it->second.samples) mean[t] = s.first / static_cast<double>(s.second);
  return choose_measured(mean, cfg_.slip_k);
}

int Rightsizer::probe_width(const OperatorKey& key) const { return measured(key).probe; }

void Rightsizer::absorb(const Rightsizer& other, const std::map<int, int>& queue_map) {
  for (const auto& [key, c] : other.curves_) {
    const auto q = queue_map.find(key.queue_id);
    if (q != queue_map.end()) curves_[OperatorKey{q->second, key.ordinal}] = c;
  }
}

void LatencyPredictor::absorb(const LatencyPredictor& other, const std::map<int, int>& queue_map) {
  for (const auto& [key, table] : other.tables_) {
    const auto q = queue_map.find(key.queue_id);
    if (q != queue_map.end()) tables_[OperatorKey{q->second, key.ordinal}] = table;
  }
}

void Rightsizer::observe(const OperatorKey& key, int tpc_count,
                         Duration latency) {  // :74-90
  Curve& c = curves_[key];
  auto& s = c.samples[tpc_count];
  s.first += static_cast<double>(latency);
  s.second += 1;
  if (tpc_count == 1 && !c.has_one) {
    c.one_ns = latency;
    c.has_one = true;
  } else if (tpc_count > 1 && !c.has_wide) {
    c.wide_t = tpc_count;
    c.wide_ns = latency;
    c.has_wide = true;
  }
  if (c.has_wide && c.has_one && !c.fit.valid && c.wide_t >= 2)
    c.fit = fit_scaling(c.one_ns, c.wide_ns, c.wide_t);
}

const ScalingFit* Rightsizer::fit_for(const OperatorKey& key) const {  // :92-96
  auto it = curves_.find(key);
  return (it != curves_.end() && it->second.fit.valid) ? &it->second.fit
                                                      : nullptr;
}

int Rightsizer::choose(const OperatorKey& key, int t_alloc, long blocks,
                       int occ) const {  // :98-103
  if (cfg_.plateau) {  // measured-curve mode: the narrowest width within the slip
    const MeasuredChoice mc = measured(key);
    if (mc.ok > 0) return std::clamp(mc.ok, 1, std::min(t_alloc, filter_cap(blocks, occ, t_alloc)));
  }
  const ScalingFit* f = fit_for(key);
  if (f == nullptr) return std::min(t_alloc, filter_cap(blocks, occ, t_alloc));
  return choose_tpcs_wave(*f, t_alloc, cfg_.slip_k, blocks, occ);
}

double r_squared(const ScalingFit& fit,
                 const std::vector<std::pair<int, double>>& points) {  // :105-119
  if (points.size() < 2) throw ConfigError("r_squared needs >= 2 points");
  double mean = 0.0;
  for (const auto& p : points) mean += p.second;
  mean /= static_cast<double>(points.size());
  double res = 0.0, tot = 0.0;
  for (const auto& [t, l] : points) {
    const double model = fit.at(t);
    res += (l - model) * (l - model);
    tot += (l - mean) * (l - mean);
  }
  if (tot == 0.0) return res == 0.0 ? 1.0 : -res;
  return 1.0 - res / tot;
}

double Rightsizer::weighted_r_squared(long* included) const {  // :121-139
  double acc = 0.0, weight = 0.0;
  long n = 0;
  for (const auto& [key, c] : curves_) {
    if (!c.fit.valid) continue;
    std::vector<std::pair<int, double>> pts;
    double busy = 0.0;
    for (const auto& [t, s] : c.samples) {
      pts.emplace_back(t, s.first / static_cast<double>(s.second));
      busy += s.first;
    }
    if (pts.size() < 2) continue;
    acc += busy * r_squared(c.fit, pts);
    weight += busy;
    ++n;
  }
  if (included != nullptr) *included = n;
  return weight > 0.0 ? acc / weight : 0.0;
}

// ------------------------------------------------------- power_manager.cpp
double sensitivity(Duration lat_fth, Duration lat_fmax, FreqMhz f_th,
                   FreqMhz f_max) {  // :8-17
  if (lat_fth <= 0 || lat_fmax <= 0) throw ConfigError("latencies must be > 0");
  if (f_th >= f_max) throw ConfigError("f_th must be below f_max");
  const double slowdown =
      static_cast<double>(lat_fth) / static_cast<double>(lat_fmax) - 1.0;
  const double stretch = static_cast<double>(f_max) / static_cast<double>(f_th) - 1.0;
  return std::clamp(slowdown / stretch, 0.0, 1.0);
}

double aggregate_sensitivity(const std::vector<std::pair<double, double>>& ws) {  // :19-25
  if (ws.empty()) throw ConfigError("aggregate over empty record set");
  double S = 0.0;
  for (const auto& [w, s] : ws) S += w * s;
  return std::clamp(S, 0.0, 1.0);
}

FreqMhz select_frequency(double S, double slip_k, FreqMhz f_max,
                         const std::vector<FreqMhz>& supported,
                         double s_floor) {  // :27-37
  if (supported.empty()) throw ConfigError("empty frequency table");
  if (slip_k <= 0.0) throw ConfigError("slip_k must be > 0");
  if (S <= s_floor) return supported.front();
  const double raw = static_cast<double>(f_max) / (1.0 + slip_k / S);
  auto up = std::find_if(supported.begin(), supported.end(),
                         [&](FreqMhz f) { return static_cast<double>(f) >= raw; });
  return up != supported.end() ? *up : supported.back();
}

PowerManager::PowerManager(DvfsConfig cfg, std::vector<FreqMhz> supported)
    : cfg_(cfg), table_(std::move(supported)) {
  if (table_.empty()) throw ConfigError("empty frequency table");
}

void PowerManager::observe(const OperatorKey& key, Duration latency,
                           FreqMhz f) {  // :39-67
  SensitivityRecord& r = records_[key];
  r.runtime_last_batch += latency;
  if (r.phase == DvfsPhase::Unseen) {
    if (f == top()) {
      r.baseline_fmax = latency;
      r.phase = DvfsPhase::Probing;
      r.s = 1.0;
    }
    return;
  }
  if (r.phase != DvfsPhase::Probing) return;
  if (f == top()) {
    r.baseline_fmax = latency;
    return;
  }
  if (r.baseline_fmax <= 0) return;
  const double s_now = sensitivity(latency, r.baseline_fmax, f, top());
  const bool had = r.last_probe_s >= 0.0;
  if (had && std::abs(s_now - r.last_probe_s) <=
                 cfg_.confirm_tolerance * std::max(r.last_probe_s, 1e-9)) {
    r.phase = DvfsPhase::Confirmed;
  } else if (had && r.last_probe_s < 1e-9 && s_now < 1e-9) {
    r.phase = DvfsPhase::Confirmed;
  }
  r.last_probe_s = s_now;
  r.s = s_now;
}

FreqMhz PowerManager::plan_batch(int queue_id) {  // :69-103
  Duration total = 0;
  bool unseen = false;
  for (const auto& [key, r] : records_) {
    if (key.queue_id != queue_id) continue;
    total += r.runtime_last_batch;
    unseen = unseen || r.phase == DvfsPhase::Unseen;
  }
  FreqMhz target = top();
  if (!unseen && total > 0) {
    std::vector<std::pair<double, double>> ws;
    for (const auto& [key, r] : records_)
      if (key.queue_id == queue_id)
        ws.emplace_back(static_cast<double>(r.runtime_last_batch) /
                            static_cast<double>(total),
                        r.s);
    if (!ws.empty())
      target = select_frequency(aggregate_sensitivity(ws), cfg_.slip_k, top(),
                                table_);
  }
  for (auto& [key, r] : records_)
    if (key.queue_id == queue_id) r.runtime_last_batch = 0;
  auto it = last_target_.find(queue_id);
  if (it == last_target_.end() || it->second != target) {
    last_target_[queue_id] = target;
    ++requests_;
  }
  return target;
}

DvfsPhase PowerManager::phase(const OperatorKey& key) const {
  auto it = records_.find(key);
  return it == records_.end() ? DvfsPhase::Unseen : it->second.phase;
}

double PowerManager::estimate(const OperatorKey& key) const {
  auto it = records_.find(key);
  return it == records_.end() ? 1.0 : it->second.s;
}

FreqMhz PowerManager::arbitrate(const std::vector<FreqMhz>& app_targets) {
  if (app_targets.empty()) throw ConfigError("arbitrate over no apps");
  return *std::max_element(app_targets.begin(), app_targets.end());
}

}  // namespace gpuos
