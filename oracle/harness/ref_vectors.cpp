// Known-answer vector generator for the pure policy functions of the hot
// path, computed by the UNMODIFIED reference. Test infrastructure only.
//
// Emits JSON lines, one case each, from fixed seeds:
//   plan_atoms        atomizer.cpp:7-31
//   should_atomize    atomizer.cpp:33-40
//   filter_cap        rightsizer.cpp:21-26
//   fit_scaling       rightsizer.cpp:8-19
//   choose_tpcs       rightsizer.cpp:28-38
//   choose_tpcs_wave  rightsizer.cpp:40-60
//   block_latency / reference_kernel_latency   device.cpp:56-72
//   predict (after a seeded record sequence)    predictor.cpp:11-57
//   select_frequency  power_manager.cpp:27-37
// These vectors pin both oracle/policy.py and the B200 library.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "gpuos/sim.hpp"

using namespace gpuos;

int main() {
  std::mt19937_64 rng(20250417);
  auto U = [&](long lo, long hi) {  // inclusive
    return lo + static_cast<long>(rng() % static_cast<unsigned long>(hi - lo + 1));
  };

  for (int i = 0; i < 600; ++i) {
    long n = U(1, 10000);
    long pred = U(1, 60'000'000);
    long atom = U(1, 5'000'000);
    long minb = i % 3 == 0 ? 1 : U(1, 200);
    auto atoms = plan_atoms(n, pred, atom, minb);
    std::printf("{\"fn\":\"plan_atoms\",\"n\":%ld,\"pred\":%ld,\"atom\":%ld,\"min\":%ld,\"out\":[",
                n, pred, atom, minb);
    for (std::size_t k = 0; k < atoms.size(); ++k)
      std::printf("%s[%ld,%ld]", k ? "," : "", atoms[k].lo, atoms[k].hi);
    std::printf("]}\n");
  }
  for (int i = 0; i < 300; ++i) {
    long pred = U(1, 5'000'000);
    long n = U(1, 5);
    if (i % 2) n = U(1, 4000);
    long atom = U(1, 2'000'000);
    double df = (i % 4 == 0) ? 2.0 : 0.5 + 0.25 * U(0, 10);
    std::printf("{\"fn\":\"should_atomize\",\"pred\":%ld,\"n\":%ld,\"atom\":%ld,\"df\":%.17g,\"out\":%d}\n",
                pred, n, atom, df, should_atomize(pred, n, atom, df) ? 1 : 0);
  }
  for (int i = 0; i < 300; ++i) {
    long n = U(1, 20000);
    int occ = static_cast<int>(U(1, 32));
    int total = static_cast<int>(U(1, 148));
    std::printf("{\"fn\":\"filter_cap\",\"n\":%ld,\"occ\":%d,\"total\":%d,\"out\":%d}\n",
                n, occ, total, filter_cap(n, occ, total));
  }
  for (int i = 0; i < 400; ++i) {
    long l1 = U(1, 200'000'000);
    long lT = i % 5 == 0 ? U(1, 300'000'000) : U(1, l1);
    int T = static_cast<int>(U(2, 148));
    ScalingFit f = fit_scaling(l1, lT, T);
    std::printf("{\"fn\":\"fit_scaling\",\"l1\":%ld,\"lT\":%ld,\"T\":%d,\"m\":%.17g,\"b\":%.17g,\"valid\":%d}\n",
                l1, lT, T, f.m_ns, f.b_ns, f.valid ? 1 : 0);
    int t_alloc = static_cast<int>(U(1, 148));
    int cap = static_cast<int>(U(1, 148));
    double slip = 1.0 + 0.01 * U(0, 50);
    long blocks = U(1, 6000);
    int occ = static_cast<int>(U(1, 8));
    std::printf("{\"fn\":\"choose_tpcs\",\"m\":%.17g,\"b\":%.17g,\"valid\":%d,\"t_alloc\":%d,\"slip\":%.17g,\"cap\":%d,\"out\":%d}\n",
                f.m_ns, f.b_ns, f.valid ? 1 : 0, t_alloc, slip, cap,
                choose_tpcs(f, t_alloc, slip, cap));
    std::printf("{\"fn\":\"choose_tpcs_wave\",\"m\":%.17g,\"b\":%.17g,\"valid\":%d,\"t_alloc\":%d,\"slip\":%.17g,\"blocks\":%ld,\"occ\":%d,\"out\":%d}\n",
                f.m_ns, f.b_ns, f.valid ? 1 : 0, t_alloc, slip, blocks, occ,
                choose_tpcs_wave(f, t_alloc, slip, blocks, occ));
  }
  FrequencyDomain fd;
  fd.supported_mhz = default_freq_table();
  for (int i = 0; i < 300; ++i) {
    SimKernelSpec k;
    k.total_blocks = U(1, 5000);
    k.block_duration_at_fmax = U(1, 3'000'000);
    k.sensitivity_s = static_cast<double>(U(0, 100)) / 100.0;
    k.occupancy_per_tpc = static_cast<int>(U(1, 8));
    FreqMhz f = fd.supported_mhz[U(0, fd.supported_mhz.size() - 1)];
    int t = static_cast<int>(U(1, 74));
    std::printf("{\"fn\":\"block_latency\",\"blocks\":%ld,\"d0\":%lld,\"s\":%.17g,\"occ\":%d,\"f\":%d,\"t\":%d,\"lat\":%lld,\"ref\":%lld}\n",
                k.total_blocks, static_cast<long long>(k.block_duration_at_fmax),
                k.sensitivity_s, k.occupancy_per_tpc, f, t,
                static_cast<long long>(block_latency(k, f, fd)),
                static_cast<long long>(reference_kernel_latency(k, t, f, fd)));
  }
  // Predictor: seeded record streams, then queries.
  for (int i = 0; i < 100; ++i) {
    LatencyPredictor p;
    OperatorKey key{static_cast<int>(U(0, 3)), static_cast<int>(U(0, 5))};
    int nrec = static_cast<int>(U(0, 6));
    std::printf("{\"fn\":\"predictor\",\"key\":[%d,%d],\"records\":[", key.queue_id, key.ordinal);
    for (int r = 0; r < nrec; ++r) {
      ObsConfig c{static_cast<int>(U(1, 8)),
                  fd.supported_mhz[U(0, fd.supported_mhz.size() - 1)],
                  U(1, 4)};
      long obs = U(1, 20'000'000);
      p.record(key, c, obs);
      std::printf("%s[%d,%d,%ld,%ld]", r ? "," : "", c.tpc_count, c.freq, c.blocks, obs);
    }
    std::printf("],\"queries\":[");
    for (int q = 0; q < 6; ++q) {
      int t = static_cast<int>(U(1, 8));
      FreqMhz f = fd.supported_mhz[U(0, fd.supported_mhz.size() - 1)];
      long b = U(1, 4);
      Prediction pr = p.predict(key, t, f, b);
      std::printf("%s[%d,%d,%ld,%lld,%d]", q ? "," : "", t, f, b,
                  static_cast<long long>(pr.latency),
                  static_cast<int>(pr.confidence));
    }
    std::printf("]}\n");
  }
  for (int i = 0; i < 200; ++i) {
    double S = static_cast<double>(U(0, 1000)) / 1000.0;
    double slip = 0.01 * U(1, 60);
    std::printf("{\"fn\":\"select_frequency\",\"S\":%.17g,\"slip\":%.17g,\"out\":%d}\n",
                S, slip, select_frequency(S, slip, 1410, fd.supported_mhz));
  }
  return 0;
}
