// C ABI of the host scheduler path (include/gpuos_sim.h): scenario sessions
// on the replay / live B200 / mirror backends, and the pure policy functions.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "gpuos/b200.hpp"
#include "gpuos/replay.hpp"
#include "gpuos/scenario.hpp"
#include "gpuos_dev.h"
#include "gpuos_dev.h"
#include "gpuos_sim.h"
#include "json.hpp"

using nlohmann::json;
using namespace gpuos;

namespace {

// Allocate every tenant kernel's operands before the dispatcher starts (no
// allocation or initialisation kernel may run beside the resident workers).
void prepare_bodies(B200Runtime& rt, const ScenarioConfig& cfg) {
  const std::vector<AppWorkload> apps = resolve_workloads(cfg);
  for (const bool allocate : {false, true}) {  // sizes first, then allocation
    auto prep = [&](const RequestTemplate& tmpl) {
      for (const KernelRecord& k : tmpl.kernels) {
        SimKernelSpec spec;
        spec.total_blocks = k.total_blocks();
        spec.block_duration_at_fmax = k.block_duration_at_fmax;
        spec.sensitivity_s = k.sensitivity_s;
        spec.occupancy_per_tpc = k.occupancy_per_tpc;
        spec.body = k.body;
        if (allocate)
          rt.prepare(spec);
        else
          rt.reserve(spec);
      }
    };
    for (const AppWorkload& w : apps) {
      prep(w.request);
      for (const RequestTemplate& t : w.per_request) prep(t);
    }
  }
}


thread_local std::string g_error;

char* dup_text(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::string runs_of(const std::vector<int>& t) {
  std::string s;
  for (std::size_t i = 0; i < t.size();) {
    std::size_t j = i;
    while (j + 1 < t.size() && t[j + 1] == t[j] + 1) ++j;
    if (!s.empty()) s += ',';
    s += std::to_string(t[i]);
    if (j > i) s += '-' + std::to_string(t[j]);
    i = j + 1;
  }
  return s;
}

// Scheduler knobs by their scenario-JSON names (sim.cpp:206-234).
void apply_knob(ScenarioConfig& c, const std::string& k, const json& v) {
  SchedulerConfig& s = c.sched;
  auto flag = [&] { return v.is_boolean() ? v.get<bool>() : v.get<double>() != 0.0; };
  if (k == "stealing") s.stealing_enabled = flag();
  else if (k == "atomizer") s.atomizer_enabled = flag();
  else if (k == "rightsizer") s.rightsizer_enabled = flag();
  else if (k == "dvfs") s.dvfs_enabled = flag();
  else if (k == "occupancy_filter") s.occupancy_filter = flag();
  else if (k == "block_revocation") s.block_revocation = flag();
  else if (k == "chain_launches") s.chain_launches = flag();
  else if (k == "chain_depth") s.chain_depth = v.get<int>();
  else if (k == "chain_best_effort") s.chain_best_effort = flag();
  else if (k == "atom_lookahead") s.atom_lookahead = flag();
  else if (k == "be_coexist") s.be_coexist = flag();
  else if (k == "hp_pair_reserve") s.hp_pair_reserve = flag();
  else if (k == "hp_quota_full") s.hp_quota_full = flag();
  else if (k == "hp_steal_busy_be") s.hp_steal_busy_be = flag();
  else if (k == "atom_duration_us") s.atom_duration = duration_from_us(v.get<double>());
  else if (k == "steal_horizon_us") s.steal_horizon = duration_from_us(v.get<double>());
  else if (k == "max_outstanding_atoms") s.max_outstanding_atoms = v.get<int>();
  else if (k == "slip_k") s.rightsizer.slip_k = v.get<double>();
  else if (k == "probe_depth_limit") s.rightsizer.probe_depth_limit = v.get<int>();
  else if (k == "rightsizer_plateau") s.rightsizer.plateau = flag();
  else if (k == "rightsize_hp") s.rightsize_hp = flag();
  else if (k == "dvfs_slip_k") s.dvfs.slip_k = v.get<double>();
  else if (k == "ewma_beta") s.predictor.ewma_beta = v.get<double>();
  else if (k == "default_unknown_us") s.predictor.default_unknown = duration_from_us(v.get<double>());
  else if (k == "disable_factor") s.disable_factor = v.get<double>();
  else if (k == "time_slice_window_us") s.time_slice_window = duration_from_us(v.get<double>());
  else throw ConfigError("unknown scheduler knob: " + k);
}

ScenarioConfig scenario_from(const json& req) {
  const json& sc = req.contains("scenario") ? req.at("scenario") : req;
  ScenarioConfig cfg;
  if (sc.contains("preset")) cfg = preset_scenario(sc.at("preset").get<std::string>());
  else if (sc.contains("config")) cfg = parse_scenario(sc.at("config").dump());
  else if (sc.contains("config_path")) cfg = load_scenario_file(sc.at("config_path").get<std::string>());
  else throw ConfigError("request needs scenario.preset, scenario.config or scenario.config_path");
  return cfg;
}

void apply_overrides(ScenarioConfig& cfg, const json& o) {
  if (o.contains("device")) {
    const std::string d = o.at("device").get<std::string>();
    if (d == "b200") cfg.topo = DeviceTopology::b200();
    else if (d == "a100-like") cfg.topo = DeviceTopology::a100_like();
    else if (d == "h100-like") cfg.topo = DeviceTopology::h100_like();
    else throw ConfigError("unknown device profile: " + d);
  }
  if (o.contains("horizon_ms")) cfg.horizon = duration_from_ms(o.at("horizon_ms").get<double>());
  if (o.contains("policy")) cfg.sched.policy = policy_from_string(o.at("policy").get<std::string>());
  if (o.contains("seed")) cfg.seed = o.at("seed").get<std::uint64_t>();
  if (o.contains("set"))
    for (const auto& [k, v] : o.at("set").items()) apply_knob(cfg, k, v);
  if (o.contains("quota_scale")) {
    // Rescale quotas/caps to a larger device (e.g. a100-like 54 -> B200 74).
    const double f = o.at("quota_scale").get<double>();
    for (AppWorkload& wl : cfg.apps) {
      wl.spec.tpc_quota = static_cast<int>(std::floor(wl.spec.tpc_quota * f));
      if (wl.spec.tpc_cap > 0) wl.spec.tpc_cap = static_cast<int>(std::floor(wl.spec.tpc_cap * f));
    }
  }
  if (o.contains("drop_apps"))  // run a subset of tenants (e.g. "LC alone")
    for (const auto& id : o.at("drop_apps")) {
      const std::string name = id.get<std::string>();
      cfg.apps.erase(std::remove_if(cfg.apps.begin(), cfg.apps.end(),
                                    [&](const AppWorkload& a) { return a.spec.app_id == name; }),
                     cfg.apps.end());
    }
  if (o.contains("time_scale")) cfg = time_scaled(cfg, o.at("time_scale").get<double>());
}

B200Options b200_options(const json& o) {
  B200Options b;
  if (!o.is_object()) return b;
  b.device = o.value("device", b.device);
  b.workers_per_sm = o.value("workers_per_sm", b.workers_per_sm);
  b.idle_sleep_ns = o.value("idle_sleep_ns", b.idle_sleep_ns);
  b.trace_blocks = o.value("trace", b.trace_blocks);
  b.synth = o.value("synth", std::string("stream")) == "spin" ? B200Options::Synth::Spin
                                                              : B200Options::Synth::Stream;
  b.stream_words_per_us = o.value("words_per_us", b.stream_words_per_us);
  b.stream_min_words = o.value("min_words", b.stream_min_words);
  b.stream_chunk_cap = o.value("chunk_cap", b.stream_chunk_cap);
  b.quantum_ns = static_cast<std::int64_t>(o.value("quantum_us", 0.0) * 1000.0);
  b.dvfs_actuate = o.value("dvfs_actuate", b.dvfs_actuate);
  b.stall_timeout_ns = static_cast<std::int64_t>(o.value("stall_timeout_s", b.stall_timeout_ns * 1e-9) * 1e9);
  return b;
}

json verify_json(const VerifyReport& v) {
  return json{{"kernels", v.kernels},   {"blocks", v.blocks},
              {"missing", v.missing},   {"duplicated", v.duplicated},
              {"misplaced", v.misplaced}, {"bad_words", v.bad_words},
              {"checked_words", v.checked_words}, {"tensor_kernels", v.tensor_kernels},
              {"tensor_checked", v.tensor_checked}, {"tensor_bad", v.tensor_bad}, {"ok", v.ok()}};
}

}  // namespace

struct gpuos_session {
  json request;
  std::string backend;  // replay | b200 | mirror
  std::unique_ptr<B200Device> b200;
  // Warm start ("warm_start": true): what the last run's scheduler learned
  // (predictor tables, right-sizer curves), keyed back to app ids.
  struct Learned {
    LatencyPredictor pred;
    Rightsizer rs;
    std::vector<std::string> apps;
  };
  std::unique_ptr<Learned> learned;
};

namespace {

std::string run_session(gpuos_session* s, const json& overrides) {
  json merged = s->request;
  if (overrides.is_object())
    for (const auto& [k, v] : overrides.items()) merged[k] = v;
  ScenarioConfig cfg = scenario_from(merged);
  apply_overrides(cfg, merged);
  cfg.validate();
  const bool want_log = merged.value("log", false);
  const bool want_requests = merged.value("requests", false);
  const bool want_timeline = merged.value("timeline", false);
  const bool e2e = merged.value("e2e", false);

  std::ostringstream log;
  long hp_atoms = 0, be_atoms = 0;
  std::vector<long> app_atoms;
  std::vector<long long> app_blocks(cfg.apps.size(), 0);
  RunHooks hooks;
  hooks.on_dispatch = [&](const DispatchRecord& d) {
    app_blocks[static_cast<std::size_t>(d.app)] += d.hi - d.lo;
    if (want_log)
      log << "D " << d.now << ' ' << d.atom << ' ' << d.app << ' ' << d.kernel << ' ' << d.lo
          << ' ' << d.hi << ' ' << d.priority << ' ' << (d.atomized ? 1 : 0) << ' '
          << runs_of(*d.tpcs) << '\n';
  };
  if (want_log) {
    hooks.on_complete = [&](const AtomCompletion& c) {
      log << "C " << c.complete_time << ' ' << c.atom << ' ' << c.tag << ' ' << c.dispatch_time
          << '\n';
    };
  }
  double rs_used = 0.0, rs_unsized = 0.0;
  const bool warm = merged.value("warm_start", false);
  std::vector<std::string> app_ids;
  for (const AppWorkload& a : cfg.apps) app_ids.push_back(a.spec.app_id);
  if (warm && s->learned) {
    hooks.on_start = [&](Scheduler& sc) {
      std::map<int, int> qmap;  // learned app index -> this run's index, by app id
      for (std::size_t i = 0; i < s->learned->apps.size(); ++i)
        for (std::size_t j = 0; j < app_ids.size(); ++j)
          if (s->learned->apps[i] == app_ids[j]) qmap[static_cast<int>(i)] = static_cast<int>(j);
      sc.warm_start(s->learned->pred, s->learned->rs, qmap);
    };
  }
  hooks.on_finish = [&](const Scheduler& sc) {
    if (warm) {
      // Merge: keep what earlier runs learned for apps absent from this one.
      auto next = std::make_unique<gpuos_session::Learned>(
          gpuos_session::Learned{LatencyPredictor(cfg.sched.predictor), Rightsizer(cfg.sched.rightsizer), {}});
      std::vector<std::string> ids = s->learned ? s->learned->apps : std::vector<std::string>{};
      for (const std::string& id : app_ids)
        if (std::find(ids.begin(), ids.end(), id) == ids.end()) ids.push_back(id);
      auto map_to = [&](const std::vector<std::string>& from) {
        std::map<int, int> m;
        for (std::size_t i = 0; i < from.size(); ++i)
          m[static_cast<int>(i)] = static_cast<int>(std::find(ids.begin(), ids.end(), from[i]) - ids.begin());
        return m;
      };
      if (s->learned) {
        next->pred.absorb(s->learned->pred, map_to(s->learned->apps));
        next->rs.absorb(s->learned->rs, map_to(s->learned->apps));
      }
      next->pred.absorb(sc.predictor(), map_to(app_ids));
      next->rs.absorb(sc.rightsizer(), map_to(app_ids));
      next->apps = ids;
      s->learned = std::move(next);
    }
    rs_used = sc.rightsized_tpc_ns();
    rs_unsized = sc.unsized_tpc_ns();
    app_atoms.assign(sc.app_count(), 0);
    for (const PredictionLogEntry& e : sc.prediction_log()) {
      (e.high_priority ? hp_atoms : be_atoms) += 1;
      app_atoms[e.key.queue_id] += 1;
    }
  };

  json out;
  RunResult res;
  if (s->backend == "replay") {
    DeviceEngine engine(cfg.topo, cfg.freq, cfg.power);
    const auto t0 = std::chrono::steady_clock::now();
    res = run_scenario_on(engine, cfg, hooks);
    out["wall_ns"] = std::chrono::duration_cast<std::chrono::nanoseconds>(
                         std::chrono::steady_clock::now() - t0)
                         .count();
  } else if (s->backend == "mirror") {
    MirrorDevice dev(cfg.topo, cfg.freq, cfg.power, b200_options(merged.value("b200", json::object())));
    prepare_bodies(dev.runtime(), cfg);
    res = run_scenario_on(dev, cfg, hooks);
    out["verify"] = verify_json(dev.verify());
    out["gpu_atoms"] = dev.gpu_atoms();
    out["gpu_kernel_ms"] = dev.gpu_kernel_ms();
  } else if (s->backend == "b200") {
    const B200Options opt = b200_options(merged.value("b200", json::object()));
    if (!s->b200 || s->b200->topology().total_tpcs() != cfg.topo.total_tpcs() ||
        !s->b200->runtime().set_run_options(opt))
      s->b200 = std::make_unique<B200Device>(cfg.topo, cfg.freq, opt);
    B200Device& dev = *s->b200;
    dev.reset_run();
    prepare_bodies(dev.runtime(), cfg);
    std::uint64_t h2d = 0, d2h = 0;
    const auto t0 = std::chrono::steady_clock::now();
    // End-to-end leg: every tenant input is copied from host memory before
    // the run and a digest of every output is read back after it.
    if (e2e) h2d = dev.runtime().upload_inputs();
    res = run_scenario_on(dev, cfg, hooks);
    if (e2e) d2h = dev.runtime().download_digest();
    const std::int64_t e2e_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                 std::chrono::steady_clock::now() - t0)
                 .count();
    json b;
    b["kernel_ms"] = dev.last_kernel_ms();
    b["run_wall_ns"] = dev.run_wall_ns();
    b["e2e_wall_ns"] = e2e_ns;
    b["h2d_bytes"] = h2d;
    b["d2h_bytes"] = d2h;
    b["workspace_bytes"] = dev.runtime().workspace_bytes();
    b["workers_per_tpc"] = dev.runtime().workers_per_tpc();
    b["logical_tpcs"] = cfg.topo.total_tpcs();
    b["tpc_busy_integral"] = dev.tpc_busy_integral();
    b["backpressure_waits"] = dev.backpressure_waits();
    {
      gpuos_dev_stats st{};
      gpuos_dev_get_stats(dev.runtime().handle(), &st);
      b["worker_busy_ns_total"] = st.worker_busy_ns;  // (cumulative over the handle's runs)
      b["tpc_busy_ns_total"] = st.tpc_busy_ns;
    }
    long blocks = 0;
    for (std::size_t k = 0; k < dev.kernels().size(); ++k) blocks += dev.blocks_executed(static_cast<KernelId>(k));
    b["blocks"] = blocks;
    b["atoms"] = dev.timeline().size();
    // Algorithmic HBM bytes of the STREAM bodies executed: 8 per word.
    double stream_bytes = 0.0;
    for (const AtomTimeline& a : dev.timeline()) {
      const auto r = dev.runtime().resolve(a.kernel, dev.kernels()[a.kernel]);
      if (r.body == 1u) stream_bytes += 8.0 * static_cast<double>(r.words) * static_cast<double>(a.hi - a.lo);
    }
    b["stream_bytes"] = stream_bytes;
    b["energy_j"] = dev.energy_joules();  // GPU energy counter over the run (NVML)
    b["sm_mhz_end"] = dev.last_sm_mhz();
    b["power_w_end"] = dev.last_power_mw() * 1e-3;
    // Executed work per tenant in calibrated block time (blocks x the
    // kernel's block duration): a throughput measure that counts partial
    // requests (a closed-loop training iteration is ~40 ms of a 1 s run).
    std::vector<double> work_us(cfg.apps.size(), 0.0);
    for (const AtomTimeline& a : dev.timeline())
      if (a.tag < work_us.size())
        work_us[a.tag] += static_cast<double>(a.hi - a.lo) *
                          static_cast<double>(dev.kernels()[a.kernel].block_duration_at_fmax) * 1e-3;
    b["work_us_per_app"] = work_us;
    if (want_timeline) {
      json tl = json::object();
      std::vector<long long> submit, complete, first, last, lo, hi, tag, prio, kern, ingest, armed;
      std::vector<unsigned long long> m0, m1, t0v, t1v;
      for (const AtomTimeline& a : dev.timeline()) {
        submit.push_back(a.host_submit_ns);
        complete.push_back(a.host_complete_ns);
        first.push_back(a.dev_first_start_ns);
        last.push_back(a.dev_last_end_ns);
        ingest.push_back(a.dev_ingest_ns);
        armed.push_back(a.dev_armed_ns);
        lo.push_back(a.lo);
        hi.push_back(a.hi);
        tag.push_back(static_cast<long long>(a.tag));
        prio.push_back(a.priority);
        kern.push_back(a.kernel);
        m0.push_back(a.mask[0]);
        m1.push_back(a.mask[1]);
        t0v.push_back(a.touched[0]);
        t1v.push_back(a.touched[1]);
      }
      tl["submit"] = submit;
      tl["complete"] = complete;
      tl["dev_first"] = first;
      tl["dev_last"] = last;
      tl["dev_ingest"] = ingest;
      tl["dev_armed"] = armed;
      tl["lo"] = lo;
      tl["hi"] = hi;
      tl["tag"] = tag;
      tl["prio"] = prio;
      tl["kernel"] = kern;
      tl["mask0"] = m0;
      tl["mask1"] = m1;
      tl["touched0"] = t0v;
      tl["touched1"] = t1v;
      std::vector<long long> words;
      for (std::size_t k = 0; k < dev.kernels().size(); ++k)
        words.push_back(dev.runtime().resolve(static_cast<KernelId>(k), dev.kernels()[k]).words);
      tl["kernel_words"] = words;
      b["timeline"] = std::move(tl);
    }
    if (merged.value("verify", false)) {
      std::vector<B200Runtime::KernelPlacement> pl(dev.kernels().size());
      for (const AtomTimeline& a : dev.timeline()) {
        pl[a.kernel].ranges.emplace_back(a.lo, a.hi);
        pl[a.kernel].masks.push_back({a.mask[0], a.mask[1]});
      }
      out["verify"] = verify_json(dev.runtime().verify_kernels(dev.kernels(), pl));
    }
    out["b200"] = std::move(b);
  } else {
    throw ConfigError("backend must be replay, b200 or mirror");
  }
  out["report"] = json::parse(res.report.to_json());
  if (cfg.sched.rightsizer_enabled)
    out["rightsizer"] = json{{"tpc_ns_used", rs_used}, {"tpc_ns_unsized", rs_unsized},
                             {"capacity_savings", rs_unsized > 0.0 ? 1.0 - rs_used / rs_unsized : 0.0},
                             {"plateau", cfg.sched.rightsizer.plateau}};
  if (want_requests) out["request_log"] = res.request_log;
  if (want_log) out["log"] = log.str();
  out["atoms"] = json{{"hp", hp_atoms}, {"be", be_atoms}, {"per_app", app_atoms}};
  out["blocks_per_app"] = app_blocks;
  out["horizon_ns"] = cfg.horizon;
  out["total_tpcs"] = cfg.topo.total_tpcs();
  return out.dump();
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_error = e.what();
    return 2;
  } catch (const InvariantError& e) {
    g_error = e.what();
    return 3;
  } catch (const json::exception& e) {
    g_error = std::string("json: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 3;
  }
}

}  // namespace

extern "C" {

const char* gpuos_sim_last_error(void) { return g_error.c_str(); }

void gpuos_free_text(char* text) { std::free(text); }

int gpuos_session_open(const char* request_json, gpuos_session** out) {
  return guarded([&] {
    if (!out) throw ConfigError("null out pointer");
    auto s = std::make_unique<gpuos_session>();
    s->request = json::parse(request_json ? request_json : "{}");
    s->backend = s->request.value("backend", std::string("replay"));
    if (s->backend != "replay" && s->backend != "b200" && s->backend != "mirror")
      throw ConfigError("backend must be replay, b200 or mirror");
    *out = s.release();
  });
}

int gpuos_session_run(gpuos_session* s, const char* overrides_json, char** result_json) {
  return guarded([&] {
    if (!s || !result_json) throw ConfigError("null argument");
    const json o = overrides_json ? json::parse(overrides_json) : json::object();
    *result_json = dup_text(run_session(s, o));
  });
}

int gpuos_session_close(gpuos_session* s) {
  return guarded([&] { delete s; });
}

int gpuos_run_json(const char* request_json, char** result_json) {
  gpuos_session* s = nullptr;
  int rc = gpuos_session_open(request_json, &s);
  if (rc != 0) return rc;
  rc = gpuos_session_run(s, nullptr, result_json);
  gpuos_session_close(s);
  return rc;
}

// ------------------------------------------------------------ dispatch probe
// Dispatcher overhead on the live path, measured in C against the C ABI:
//  * serial: n one-block SPIN(0) atoms, each submitted after the previous
//    completion was polled -> host round trip (submit .. completion seen)
//    and publish -> first block start (device clock, calibrated);
//  * pipelined: empty atoms kept `depth` deep in flight on one TPC set ->
//    sustained atoms/s; per-atom overhead = 1 / rate.
int gpuos_probe_dispatch(const char* opts_json, char** result_json) {
  return guarded([&] {
    const json o = json::parse(opts_json ? opts_json : "{}");
    const int n = o.value("serial", 2000);
    const int m = o.value("pipelined", 20000);
    const int depth = o.value("depth", 16);
    const int tpc = o.value("tpc", 0);
    gpuos_dev_config cfg{};
    cfg.device_ordinal = o.value("device", 0);
    cfg.workers_per_sm = o.value("workers_per_sm", 2);
    cfg.idle_sleep_ns = o.value("idle_sleep_ns", 0);  // 0: the default
    gpuos_dev* d = nullptr;
    if (gpuos_dev_open(&cfg, &d) != GPUOS_OK) throw InvariantError(gpuos_dev_last_error());
    std::unique_ptr<gpuos_dev, int (*)(gpuos_dev*)> guard(d, gpuos_dev_close);
    auto must = [&](int rc) {
      if (rc < 0) throw InvariantError(gpuos_dev_last_error());
      return rc;
    };
    gpuos_atom_desc a{};
    a.lo = 0;
    a.hi = 1;
    a.tpc_mask[tpc >> 6] = 1ull << (tpc & 63);
    a.priority = 20;
    a.body = GPUOS_BODY_SPIN;
    must(gpuos_dev_start(d));
    std::vector<double> rtt, to_start, to_end, ingest_to_armed, armed_to_start, start_to_host;
    gpuos_completion c{};
    for (int i = 0; i < n + 50; ++i) {
      std::uint32_t id = 0;
      must(gpuos_dev_submit_atom(d, &a, &id));
      while (must(gpuos_dev_poll(d, &c, 1)) == 0) {
      }
      if (i < 50) continue;  // warm-up
      rtt.push_back(static_cast<double>(c.host_complete_ns - c.host_submit_ns));
      to_start.push_back(static_cast<double>(c.dev_first_start_ns - c.host_submit_ns));
      to_end.push_back(static_cast<double>(c.host_complete_ns - c.dev_last_end_ns));
      ingest_to_armed.push_back(static_cast<double>(c.dev_armed_ns - c.dev_ingest_ns));
      armed_to_start.push_back(static_cast<double>(c.dev_first_start_ns - c.dev_armed_ns));
      start_to_host.push_back(static_cast<double>(c.host_complete_ns - c.dev_first_start_ns));
    }
    // Pipelined: keep `depth` empty atoms in flight.
    gpuos_completion buf[64];
    int sent = 0, got = 0;
    const std::int64_t t0 = gpuos_dev_now_ns(d);
    while (got < m) {
      while (sent < m && sent - got < depth) {
        std::uint32_t id = 0;
        must(gpuos_dev_submit_atom(d, &a, &id));
        ++sent;
      }
      got += must(gpuos_dev_poll(d, buf, 64));
    }
    const double secs = static_cast<double>(gpuos_dev_now_ns(d) - t0) * 1e-9;
    float ms = 0.f;
    must(gpuos_dev_stop(d, 1, &ms));
    auto pct = [](std::vector<double> v, double p) {
      std::sort(v.begin(), v.end());
      return v[static_cast<std::size_t>(p / 100.0 * (v.size() - 1))];
    };
    json out;
    out["serial_roundtrip_ns"] = {{"p50", pct(rtt, 50)}, {"p90", pct(rtt, 90)}, {"p99", pct(rtt, 99)}};
    out["publish_to_first_block_ns"] = {{"p50", pct(to_start, 50)}, {"p90", pct(to_start, 90)},
                                        {"p99", pct(to_start, 99)}};
    out["last_block_to_host_ns"] = {{"p50", pct(to_end, 50)}, {"p90", pct(to_end, 90)}};
    // Device-clock-only breakdown (no host/device offset error).
    out["device_ingest_to_armed_ns_p50"] = pct(ingest_to_armed, 50);
    out["device_armed_to_first_block_ns_p50"] = pct(armed_to_start, 50);
    out["host_submit_to_device_ingest_ns_p50_offset_sensitive"] =
        pct(to_start, 50) - pct(ingest_to_armed, 50) - pct(armed_to_start, 50);
    out["pipelined_atoms_per_s"] = m / secs;
    out["pipelined_ns_per_atom"] = secs * 1e9 / m;
    out["depth"] = depth;
    *result_json = dup_text(out.dump());
  });
}

// ------------------------------------------------------------ policy ABI
int64_t gpuos_plan_atoms(int64_t n, int64_t pred, int64_t atom, int64_t minb,
                         int64_t* out, int64_t cap) {
  int64_t count = -2;
  guarded([&] {
    const auto a = plan_atoms(n, pred, atom, minb);
    for (std::size_t i = 0; i < a.size() && static_cast<int64_t>(i) < cap; ++i) {
      out[2 * i] = a[i].lo;
      out[2 * i + 1] = a[i].hi;
    }
    count = static_cast<int64_t>(a.size());
  });
  return count;
}

int gpuos_should_atomize(int64_t pred, int64_t n, int64_t atom, double factor) {
  return should_atomize(pred, n, atom, factor) ? 1 : 0;
}

int gpuos_filter_cap(int64_t n, int32_t occ, int32_t total) {
  int r = -2;
  guarded([&] { r = filter_cap(n, occ, total); });
  return r;
}

int gpuos_fit_scaling(int64_t l1, int64_t lT, int32_t T, double* m, double* b, int32_t* valid) {
  return guarded([&] {
    const ScalingFit f = fit_scaling(l1, lT, T);
    *m = f.m_ns;
    *b = f.b_ns;
    *valid = f.valid ? 1 : 0;
  });
}

int gpuos_choose_tpcs(double m, double b, int32_t valid, int32_t t_alloc, double slip, int32_t cap) {
  int r = -2;
  guarded([&] { r = choose_tpcs(ScalingFit{m, b, valid != 0}, t_alloc, slip, cap); });
  return r;
}

int gpuos_choose_tpcs_wave(double m, double b, int32_t valid, int32_t t_alloc, double slip,
                           int64_t blocks, int32_t occ) {
  int r = -2;
  guarded([&] { r = choose_tpcs_wave(ScalingFit{m, b, valid != 0}, t_alloc, slip, blocks, occ); });
  return r;
}

int gpuos_fit_scaling_plateau(int64_t l1, int32_t t_mid, int64_t l_mid, int64_t lT, int32_t T, double* m,
                              double* b, double* floor_ns, int32_t* valid) {
  return guarded([&] {
    const ScalingFit f = fit_scaling_plateau(l1, t_mid, l_mid, lT, T);
    *m = f.m_ns;
    *b = f.b_ns;
    *floor_ns = f.floor_ns;
    *valid = f.valid ? 1 : 0;
  });
}

int gpuos_choose_tpcs_wave_floor(double m, double b, double floor_ns, int32_t valid, int32_t t_alloc,
                                 double slip, int64_t blocks, int32_t occ) {
  int r = -2;
  guarded([&] {
    ScalingFit f{m, b, valid != 0};
    f.floor_ns = floor_ns;
    r = choose_tpcs_wave(f, t_alloc, slip, blocks, occ);
  });
  return r;
}

int gpuos_choose_measured(const int32_t* t, const double* l_ns, int32_t n, double slip_k, int32_t* ok,
                          int32_t* probe) {
  return guarded([&] {
    if ((n > 0 && (!t || !l_ns)) || !ok || !probe) throw ConfigError("null argument");
    std::map<int, double> mean;
    for (int32_t i = 0; i < n; ++i) mean[t[i]] = l_ns[i];
    const MeasuredChoice mc = choose_measured(mean, slip_k);
    *ok = mc.ok;
    *probe = mc.probe;
  });
}

int64_t gpuos_block_latency(int64_t d0, double s, int32_t f) {
  int64_t r = -2;
  guarded([&] {
    FrequencyDomain fd;
    fd.supported_mhz = default_freq_table();
    SimKernelSpec k;
    k.block_duration_at_fmax = d0;
    k.sensitivity_s = s;
    r = block_latency(k, f, fd);
  });
  return r;
}

int64_t gpuos_reference_kernel_latency(int64_t blocks, int64_t d0, double s, int32_t occ, int32_t t,
                                       int32_t f) {
  int64_t r = -2;
  guarded([&] {
    FrequencyDomain fd;
    fd.supported_mhz = default_freq_table();
    SimKernelSpec k;
    k.total_blocks = blocks;
    k.block_duration_at_fmax = d0;
    k.sensitivity_s = s;
    k.occupancy_per_tpc = occ;
    r = reference_kernel_latency(k, t, f, fd);
  });
  return r;
}

int32_t gpuos_select_frequency(double S, double slip) {
  int32_t r = -2;
  guarded([&] { r = select_frequency(S, slip, 1410, default_freq_table()); });
  return r;
}

int gpuos_predictor_replay(const int64_t* records, int32_t n, const int64_t* queries, int32_t q,
                           int64_t* out_latency, int32_t* out_conf) {
  return guarded([&] {
    LatencyPredictor p;
    const OperatorKey key{0, 0};
    for (int i = 0; i < n; ++i) {
      const int64_t* r = records + 4 * i;
      p.record(key, ObsConfig{static_cast<int>(r[0]), static_cast<FreqMhz>(r[1]), r[2]}, r[3]);
    }
    for (int i = 0; i < q; ++i) {
      const int64_t* x = queries + 3 * i;
      const Prediction pr = p.predict(key, static_cast<int>(x[0]), static_cast<FreqMhz>(x[1]), x[2]);
      out_latency[i] = pr.latency;
      out_conf[i] = static_cast<int32_t>(pr.confidence);
    }
  });
}

}  // extern "C"
