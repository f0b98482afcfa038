// Live B200 backend and GPU mirror of the device seam (include/gpuos/b200.hpp),
// written purely against the C ABI of the sm_100a dispatcher (gpuos_dev.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <set>
#include <thread>

#include "gpuos/b200.hpp"
#include "gpuos/tenants.hpp"
#include "gpuos_dev.h"

namespace gpuos {

namespace {

[[noreturn]] void raise(int rc, const char* what) {
  std::string msg = std::string(what) + ": " + gpuos_dev_last_error();
  if (rc == GPUOS_E_CONFIG) throw ConfigError(msg);
  throw InvariantError(msg);
}

void check(int rc, const char* what) {
  if (rc < 0) raise(rc, what);
}

// splitmix64: deterministic workspace contents.
std::uint64_t mix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

std::uint32_t salt_of(std::uint32_t workspace) {
  return static_cast<std::uint32_t>(mix64(0xB200u + workspace)) | 1u;
}

// CPU restatement of the STREAM body (bodies.cuh), the verification oracle.
inline std::uint32_t stream_expect(std::uint32_t x, std::uint32_t salt, std::uint64_t e) {
  return (x ^ salt) * 0x9E3779B1u + static_cast<std::uint32_t>(e);
}

std::array<std::uint64_t, 2> mask_of(const std::vector<int>& tpcs) {
  std::array<std::uint64_t, 2> m{0, 0};
  for (int t : tpcs) m[t >> 6] |= 1ull << (t & 63);
  return m;
}

}  // namespace

// ================================================================ runtime
B200Runtime::B200Runtime(int logical_tpcs, const B200Options& opt)
    : opt_(opt), tpcs_(logical_tpcs) {
  if (logical_tpcs < 1 || logical_tpcs > GPUOS_MAX_TPCS)
    throw ConfigError("B200 backend supports 1..128 logical TPCs");
  gpuos_dev_config cfg{};
  cfg.device_ordinal = opt.device;
  cfg.workers_per_sm = opt.workers_per_sm;
  cfg.logical_tpcs = logical_tpcs;
  cfg.idle_sleep_ns = opt.idle_sleep_ns;
  check(gpuos_dev_open(&cfg, &dev_), "gpuos_dev_open");
}

B200Runtime::~B200Runtime() {
  if (running_) {
    float ms;
    gpuos_dev_stop(dev_, 0, &ms);
  }
  for (auto& [id, w] : ws_) {
    gpuos_dev_free(dev_, w.src);
    gpuos_dev_free(dev_, w.dst);
    gpuos_dev_host_free(dev_, w.host_src);
  }
  for (auto* p : trace_chunks_) gpuos_dev_free(dev_, p);
  for (auto& [key, t] : tensors_) {
    gpuos_dev_free(dev_, t.desc);
    for (void* p : t.bufs) gpuos_dev_free(dev_, p);
  }
  gpuos_dev_close(dev_);
}

int B200Runtime::workers_per_tpc() const {
  gpuos_dev_topology t{};
  gpuos_dev_get_topology(dev_, &t);
  return t.workers_per_tpc;
}

void B200Runtime::reserve(const SimKernelSpec& spec) {
  const BodyRef& b = spec.body;
  if (b.kind != BodyKind::Stream || b.p0 <= 0) return;
  const std::uint64_t cap = b.p2 > 0 ? static_cast<std::uint64_t>(b.p2)
                                     : static_cast<std::uint64_t>(opt_.stream_chunk_cap);
  std::uint64_t& r = ws_reserve_[b.workspace];
  r = std::max<std::uint64_t>(r, static_cast<std::uint64_t>(b.p0) * cap);
}

B200Runtime::Workspace& B200Runtime::workspace(std::uint32_t id, std::uint64_t words) {
  Workspace& w = ws_[id];
  if (w.words >= words) return w;
  if (!w.src) {
    const auto it = ws_reserve_.find(id);
    if (it != ws_reserve_.end()) words = std::max(words, it->second);
  }
  // Buffers may be referenced by atoms in flight: never reallocate.
  if (w.src) throw ConfigError("workspace " + std::to_string(id) + " is smaller than a later kernel needs");
  words = (words + 3) & ~3ull;
  void* p = nullptr;
  check(gpuos_dev_alloc(dev_, words * 4, &p), "workspace alloc");
  w.src = static_cast<std::uint32_t*>(p);
  check(gpuos_dev_alloc(dev_, words * 4, &p), "workspace alloc");
  w.dst = static_cast<std::uint32_t*>(p);
  w.words = words;
  check(gpuos_dev_host_alloc(dev_, words * 4, &p), "pinned input alloc");
  w.host_src = static_cast<std::uint32_t*>(p);
  std::uint64_t s = mix64(id);
  for (std::uint64_t i = 0; i < words; i += 2) {
    s = mix64(s);
    w.host_src[i] = static_cast<std::uint32_t>(s);
    if (i + 1 < words) w.host_src[i + 1] = static_cast<std::uint32_t>(s >> 32);
  }
  check(gpuos_dev_copy(dev_, w.src, w.host_src, words * 4, 1), "workspace upload");
  check(gpuos_dev_memset(dev_, w.dst, 0, words * 4), "workspace clear");
  return w;
}

// Tensor-core tenant kernels: operands random-initialised on the device
// (uniform in [-1, 1), bf16) and a descriptor, per (workspace, shape). Each
// workspace id is a distinct set of weights, so model traces that give
// every layer its own id stream their real weight bytes from HBM.
const B200Runtime::TensorBody& B200Runtime::tensor_body(const BodyRef& b) {
  std::string key = std::to_string(static_cast<int>(b.kind)) + "/" + std::to_string(b.workspace);
  for (int i = 0; i < BodyRef::kParams; ++i) key += "/" + std::to_string(b.param(i));
  auto it = tensors_.find(key);
  if (it != tensors_.end()) return it->second;
  TensorBody t;
  const std::uint64_t seed = mix64(std::hash<std::string>{}(key));
  auto tensor = [&](std::uint64_t elems, bool fill) {
    void* p = nullptr;
    check(gpuos_dev_alloc(dev_, std::max<std::uint64_t>(elems, 8) * 2, &p), "tensor alloc");
    if (fill) check(gpuos_dev_fill_bf16(dev_, p, elems, seed + t.bufs.size()), "tensor init");
    t.bufs.push_back(p);
    return p;
  };
  if (b.kind == BodyKind::GemmBf16) {
    const std::int64_t M = b.p0, N = b.p1, K = b.p2;
    if (M <= 0 || N <= 0 || K <= 0) throw ConfigError("gemm_bf16 needs p = [M, N, K(, k_splits)]");
    void* A = tensor(static_cast<std::uint64_t>(M) * K, true);
    void* B = tensor(static_cast<std::uint64_t>(N) * K, true);
    void* C = tensor(static_cast<std::uint64_t>(M) * N, false);
    int32_t tm = 0, tn = 0;
    const std::int64_t splits = std::max<std::int64_t>(1, b.param(3));  // p[3]: split-K
    check(gpuos_dev_gemm_desc_splitk(dev_, A, B, C, M, N, K, N, GPUOS_GEMM_OUT_BF16, static_cast<int32_t>(splits),
                                     &t.desc, &t.blocks, &tm, &tn),
          "gemm descriptor");
  } else if (b.kind == BodyKind::GemvBf16) {
    const std::int64_t N = b.p0, K = b.p1, splits = std::max<std::int64_t>(1, b.p2);
    if (N <= 0 || K <= 0) throw ConfigError("gemv_bf16 needs p = [N, K, k_splits]");
    void* W = tensor(static_cast<std::uint64_t>(N) * K, true);
    void* X = tensor(static_cast<std::uint64_t>(K), true);
    void* Y = tensor(static_cast<std::uint64_t>(N), false);
    check(gpuos_dev_gemv_desc(dev_, W, X, Y, N, K, GPUOS_GEMV_OUT_BF16, static_cast<int32_t>(splits),
                              &t.desc, &t.blocks),
          "gemv descriptor");
  } else if (b.kind == BodyKind::AttnDecodeBf16) {
    // Decode attention (csrc/bodies/llama_attention.cu): q [32][128], K and V
    // caches [ctx][8][128], workspace (result, counters, chunk partials).
    check(gpuos_dev_body_id(body_kind_name(b.kind), &t.body), "tenant body lookup");
    const std::int64_t ctx = b.p0, chunk = b.p1 > 0 ? b.p1 : 32;
    if (ctx <= 0 || chunk > 32 || chunk <= 0) throw ConfigError("attn_decode_bf16 needs p = [ctx, chunk <= 32]");
    const std::int64_t chunks = (ctx + chunk - 1) / chunk;
    if (chunks > 256) throw ConfigError("attn_decode_bf16 merges at most 256 context chunks");
    void* Q = tensor(32 * 128, true);
    void* KV = tensor(static_cast<std::uint64_t>(2 * ctx * 8 * 128), true);
    const std::uint64_t ws_elems = (8448 + 32ull * chunks * 130 * 4) / 2;
    void* WS = tensor(ws_elems, false);
    check(gpuos_dev_memset(dev_, WS, 0, ws_elems * 2), "attention workspace");
    t.blocks = chunks * 8;
    t.args[0] = reinterpret_cast<std::uint64_t>(Q);
    t.args[1] = reinterpret_cast<std::uint64_t>(KV);
    t.args[2] = reinterpret_cast<std::uint64_t>(WS);
    t.args[3] = static_cast<std::uint64_t>(ctx) | (static_cast<std::uint64_t>(chunk) << 32);
    t.args[4] = static_cast<std::uint64_t>(chunks) | (8ull << 21);  // GPUOS_GRID(chunks, 8)
    t.desc = reinterpret_cast<void*>(t.args[2]);  // (verify key: the result buffer)
  } else if (b.kind == BodyKind::RmsNormBf16 || b.kind == BodyKind::SiluMulBf16) {
    // Tenant bodies (csrc/bodies/llama_elementwise.cu), by name.
    const bool rms = b.kind == BodyKind::RmsNormBf16;
    check(gpuos_dev_body_id(body_kind_name(b.kind), &t.body), "tenant body lookup");
    if (rms) {
      const std::int64_t rows = b.p0, d = b.p1;
      if (rows <= 0 || d <= 0 || d % 8 != 0) throw ConfigError("rmsnorm_bf16 needs p = [rows, d], d % 8 == 0");
      void* X = tensor(static_cast<std::uint64_t>(rows) * d, true);
      void* Wn = tensor(static_cast<std::uint64_t>(d), true);
      void* Y = tensor(static_cast<std::uint64_t>(rows) * d, false);
      const float eps = 1e-5f;
      std::uint32_t eb;
      std::memcpy(&eb, &eps, 4);
      t.args[0] = reinterpret_cast<std::uint64_t>(X);
      t.args[1] = reinterpret_cast<std::uint64_t>(Wn);
      t.args[2] = reinterpret_cast<std::uint64_t>(Y);
      t.args[3] = static_cast<std::uint64_t>(d) | (static_cast<std::uint64_t>(eb) << 32);
      t.args[4] = static_cast<std::uint64_t>(rows);  // GPUOS_GRID(rows)
      t.blocks = rows;
    } else {
      const std::int64_t n = b.p0, chunk = b.p1;
      if (n <= 0 || n > 0xffffffffll || chunk <= 0 || chunk % 8 != 0)
        throw ConfigError("silu_mul_bf16 needs p = [n, chunk], chunk % 8 == 0");
      void* G = tensor(static_cast<std::uint64_t>(n) + 8, true);
      void* U = tensor(static_cast<std::uint64_t>(n) + 8, true);
      void* O = tensor(static_cast<std::uint64_t>(n) + 8, false);
      t.blocks = (n + chunk - 1) / chunk;
      t.args[0] = reinterpret_cast<std::uint64_t>(G);
      t.args[1] = reinterpret_cast<std::uint64_t>(U);
      t.args[2] = reinterpret_cast<std::uint64_t>(O);
      t.args[3] = static_cast<std::uint64_t>(n) | (static_cast<std::uint64_t>(chunk) << 32);
      t.args[4] = static_cast<std::uint64_t>(t.blocks);
    }
    t.desc = reinterpret_cast<void*>(t.args[2]);  // (verify key: the output buffer)
  } else {
    const std::int64_t n = b.p0, h = b.p1, w = b.p2, c = b.param(3), k = b.param(4), r = b.param(5),
                       sd = b.param(6), pad = b.param(7), st = std::max<std::int64_t>(1, b.param(8));
    if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || k <= 0 || r <= 0 || sd <= 0)
      throw ConfigError("conv_bf16 needs p = [n, h, w, c, k, r, s, pad, stride]");
    const std::int64_t cb = (c + 63) / 64 * 64;
    const std::int64_t P = (h + 2 * pad - r) / st + 1, Q = (w + 2 * pad - sd) / st + 1;
    void* X = tensor(static_cast<std::uint64_t>(n) * h * w * c, true);
    void* Wt = tensor(static_cast<std::uint64_t>(k) * r * sd * cb, true);
    void* Y = tensor(static_cast<std::uint64_t>(std::max<std::int64_t>(0, n * P * Q * k)), false);
    int32_t po = 0, qo = 0;
    check(gpuos_dev_conv_desc(dev_, X, Wt, Y, static_cast<int32_t>(n), static_cast<int32_t>(h),
                              static_cast<int32_t>(w), static_cast<int32_t>(c), static_cast<int32_t>(k),
                              static_cast<int32_t>(r), static_cast<int32_t>(sd), static_cast<int32_t>(pad),
                              static_cast<int32_t>(st), GPUOS_CONV_OUT_BF16, &t.desc, &t.blocks, &po, &qo),
          "conv descriptor");
  }
  t.ref = b;
  const TensorBody& out = tensors_.emplace(key, t).first->second;
  tensor_of_desc_[reinterpret_cast<std::uint64_t>(out.desc)] = &out;
  return out;
}

namespace {
float bf16_to_float(std::uint16_t v) {
  const std::uint32_t u = static_cast<std::uint32_t>(v) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
}  // namespace

void B200Runtime::verify_tensor(const TensorBody& t, VerifyReport& rep) {
  // Up to 48 sampled outputs per kernel, each recomputed in float64 from
  // the operands read back from HBM (only the rows / windows it needs).
  const BodyRef& b = t.ref;
  std::uint64_t rng = mix64(reinterpret_cast<std::uint64_t>(t.desc));
  auto next = [&](std::uint64_t n) { rng = mix64(rng); return n ? rng % n : 0ull; };
  auto fetch = [&](const void* base, std::uint64_t elem, std::uint64_t n, std::vector<std::uint16_t>& out) {
    out.resize(n);
    check(gpuos_dev_copy(dev_, out.data(), static_cast<const std::uint16_t*>(base) + elem, n * 2, 2),
          "verify download");
  };
  auto judge = [&](double got, double ref, double mag) {
    ++rep.tensor_checked;
    if (!(std::fabs(got - ref) <= std::ldexp(std::fabs(ref), -8) + 1e-5 * mag + 1e-6)) ++rep.tensor_bad;
  };
  std::vector<std::uint16_t> ra, rb, out1;
  constexpr int kSamples = 48;
  ++rep.tensor_kernels;
  if (b.kind == BodyKind::RmsNormBf16) {
    const std::uint64_t rows = static_cast<std::uint64_t>(b.p0), d = static_cast<std::uint64_t>(b.p1);
    fetch(t.bufs[1], 0, d, rb);  // w
    for (int i = 0; i < kSamples / 8; ++i) {
      const std::uint64_t row = next(rows);
      fetch(t.bufs[0], row * d, d, ra);
      fetch(t.bufs[2], row * d, d, out1);
      double ss = 0;
      for (std::uint64_t k = 0; k < d; ++k) ss += static_cast<double>(bf16_to_float(ra[k])) * bf16_to_float(ra[k]);
      const double scale = 1.0 / std::sqrt(ss / static_cast<double>(d) + 1e-5);
      for (int j = 0; j < 8; ++j) {
        const std::uint64_t k = next(d);
        const double ref = bf16_to_float(ra[k]) * scale * bf16_to_float(rb[k]);
        judge(bf16_to_float(out1[k]), ref, std::fabs(ref) * 8.0);
      }
    }
    return;
  }
  if (b.kind == BodyKind::AttnDecodeBf16) {
    // Sampled query heads recomputed in float64: RoPE (base 500000,
    // interleaved pairs) at position ctx, softmax over the whole cache.
    const std::int64_t ctx = b.p0;
    std::vector<std::uint16_t> q, kv, out;
    fetch(t.bufs[0], 0, 32 * 128, q);
    fetch(t.bufs[1], 0, static_cast<std::uint64_t>(2 * ctx * 8 * 128), kv);
    fetch(t.bufs[2], 0, 32 * 128, out);
    for (int i = 0; i < 6; ++i) {
      const int h = static_cast<int>(next(32)), g = h / 4;
      double qr[128];
      for (int j = 0; j < 64; ++j) {
        const double inv = std::pow(500000.0, -2.0 * j / 128.0), a = static_cast<double>(ctx) * inv;
        const double x0 = bf16_to_float(q[h * 128 + 2 * j]), x1 = bf16_to_float(q[h * 128 + 2 * j + 1]);
        qr[2 * j] = x0 * std::cos(a) - x1 * std::sin(a);
        qr[2 * j + 1] = x0 * std::sin(a) + x1 * std::cos(a);
      }
      std::vector<double> s(static_cast<std::size_t>(ctx));
      double m = -1e300;
      for (std::int64_t p = 0; p < ctx; ++p) {
        double d = 0;
        for (int j = 0; j < 128; ++j) d += qr[j] * bf16_to_float(kv[static_cast<std::size_t>((p * 8 + g) * 128 + j)]);
        s[static_cast<std::size_t>(p)] = d / std::sqrt(128.0);
        m = std::max(m, s[static_cast<std::size_t>(p)]);
      }
      double l = 0;
      for (auto& v : s) l += (v = std::exp(v - m));
      for (int k = 0; k < 4; ++k) {
        const int j = static_cast<int>(next(128));
        double o = 0, mag = 0;
        for (std::int64_t p = 0; p < ctx; ++p) {
          const double v = bf16_to_float(kv[static_cast<std::size_t>(((ctx + p) * 8 + g) * 128 + j)]);
          o += s[static_cast<std::size_t>(p)] * v;
          mag += s[static_cast<std::size_t>(p)] * std::fabs(v);
        }
        judge(bf16_to_float(out[static_cast<std::size_t>(h * 128 + j)]), o / l, mag / l * 64.0);
      }
    }
    return;
  }
  if (b.kind == BodyKind::SiluMulBf16) {
    const std::uint64_t n = static_cast<std::uint64_t>(b.p0);
    for (int i = 0; i < kSamples; ++i) {
      const std::uint64_t e = next(n);
      fetch(t.bufs[0], e, 1, ra);
      fetch(t.bufs[1], e, 1, rb);
      fetch(t.bufs[2], e, 1, out1);
      const double g = bf16_to_float(ra[0]);
      const double ref = g / (1.0 + std::exp(-g)) * bf16_to_float(rb[0]);
      judge(bf16_to_float(out1[0]), ref, std::fabs(ref) * 8.0);
    }
    return;
  }
  if (b.kind == BodyKind::GemmBf16 || b.kind == BodyKind::GemvBf16) {
    const bool gemm = b.kind == BodyKind::GemmBf16;
    const std::uint64_t M = gemm ? static_cast<std::uint64_t>(b.p0) : 1;
    const std::uint64_t N = static_cast<std::uint64_t>(gemm ? b.p1 : b.p0);
    const std::uint64_t K = static_cast<std::uint64_t>(gemm ? b.p2 : b.p1);
    for (int i = 0; i < kSamples; ++i) {
      const std::uint64_t m = next(M), n = next(N);
      fetch(t.bufs[0], gemm ? m * K : n * K, K, ra);   // A row m / W row n
      fetch(t.bufs[1], gemm ? n * K : 0, K, rb);       // B row n / x
      fetch(t.bufs[2], gemm ? m * N + n : n, 1, out1);
      double ref = 0, mag = 0;
      for (std::uint64_t k = 0; k < K; ++k) {
        const double p = static_cast<double>(bf16_to_float(ra[k])) * bf16_to_float(rb[k]);
        ref += p;
        mag += std::fabs(p);
      }
      judge(bf16_to_float(out1[0]), ref, mag);
    }
    return;
  }
  // conv: x [n, h, w, c], w [k, r, s, cb], y [n, P, Q, k] (NHWC, bf16)
  const std::int64_t n = b.p0, h = b.p1, w = b.p2, c = b.param(3), k = b.param(4), r = b.param(5),
                     sd = b.param(6), pad = b.param(7), st = std::max<std::int64_t>(1, b.param(8));
  const std::int64_t cb = (c + 63) / 64 * 64;
  const std::int64_t P = (h + 2 * pad - r) / st + 1, Q = (w + 2 * pad - sd) / st + 1;
  for (int i = 0; i < kSamples / 4; ++i) {
    const std::int64_t in = static_cast<std::int64_t>(next(n)), p = static_cast<std::int64_t>(next(P)),
                       q = static_cast<std::int64_t>(next(Q)), kk = static_cast<std::int64_t>(next(k));
    fetch(t.bufs[1], static_cast<std::uint64_t>(kk * r * sd * cb), static_cast<std::uint64_t>(r * sd * cb), rb);
    double ref = 0, mag = 0;
    for (std::int64_t rr = 0; rr < r; ++rr)
      for (std::int64_t ss = 0; ss < sd; ++ss) {
        const std::int64_t y = p * st - pad + rr, x = q * st - pad + ss;
        if (y < 0 || y >= h || x < 0 || x >= w) continue;
        fetch(t.bufs[0], static_cast<std::uint64_t>(((in * h + y) * w + x) * c), static_cast<std::uint64_t>(c), ra);
        for (std::int64_t ci = 0; ci < c; ++ci) {
          const double v = static_cast<double>(bf16_to_float(ra[ci])) *
                           bf16_to_float(rb[static_cast<std::size_t>((rr * sd + ss) * cb + ci)]);
          ref += v;
          mag += std::fabs(v);
        }
      }
    fetch(t.bufs[2], static_cast<std::uint64_t>(((in * P + p) * Q + q) * k + kk), 1, out1);
    judge(bf16_to_float(out1[0]), ref, mag);
  }
}

void B200Runtime::ensure_trace(KernelId kid, long blocks) {
  if (trace_of_.size() <= kid) trace_of_.resize(kid + 1, nullptr);
  if (trace_of_[kid]) return;
  const std::uint64_t need = static_cast<std::uint64_t>(blocks);
  while (trace_chunk_ < trace_chunks_.size() &&
         trace_pool_used_ + need > trace_chunk_words_[trace_chunk_]) {
    ++trace_chunk_;
    trace_pool_used_ = 0;
  }
  if (trace_chunk_ == trace_chunks_.size()) {
    const std::uint64_t cap = std::max<std::uint64_t>(need, kTraceChunkWords);
    void* p = nullptr;
    check(gpuos_dev_alloc(dev_, cap * 4, &p), "trace alloc");
    check(gpuos_dev_memset(dev_, p, 0, cap * 4), "trace clear");
    trace_chunks_.push_back(static_cast<std::uint32_t*>(p));
    trace_chunk_words_.push_back(cap);
    trace_pool_used_ = 0;
  }
  trace_of_[kid] = trace_chunks_[trace_chunk_] + trace_pool_used_;
  trace_pool_used_ += need;
}

B200Runtime::Resolved B200Runtime::resolve(KernelId kid, const SimKernelSpec& spec) {
  if (has_resolved_.size() > kid && has_resolved_[kid]) return resolved_[kid];
  Resolved r = resolve_body(spec);
  if (opt_.trace_blocks) {
    ensure_trace(kid, spec.total_blocks * static_cast<long>(r.parts));
    r.trace = trace_of_[kid];
  }
  if (resolved_.size() <= kid) {
    resolved_.resize(kid + 1);
    has_resolved_.resize(kid + 1, 0);
  }
  resolved_[kid] = r;
  has_resolved_[kid] = 1;
  return r;
}

B200Runtime::Resolved B200Runtime::resolve_body(const SimKernelSpec& spec) {
  Resolved r{};
  BodyRef b = spec.body;
  if (b.kind == BodyKind::None) {
    // The reference's cost-only kernel: synthesise a body of the same length.
    const double us = static_cast<double>(spec.block_duration_at_fmax) / 1000.0;
    if (opt_.synth == B200Options::Synth::Spin) {
      b.kind = BodyKind::Spin;
      b.p0 = spec.block_duration_at_fmax;
    } else {
      long words = static_cast<long>(std::llround(us * opt_.stream_words_per_us));
      words = std::max(opt_.stream_min_words, (words + 3) & ~3L);
      b.kind = BodyKind::Stream;
      b.p0 = words;
      b.workspace = 0x100000u + static_cast<std::uint32_t>(words / 4);
    }
  }
  switch (b.kind) {
    case BodyKind::Stream: {
      const long words = static_cast<long>(b.p0);
      if (words <= 0 || words % 4 != 0) throw ConfigError("stream body needs words % 4 == 0");
      const long cap = b.p2 > 0 ? static_cast<long>(b.p2) : opt_.stream_chunk_cap;
      const long chunks = std::min<long>(spec.total_blocks, cap);
      Workspace& w = workspace(b.workspace, static_cast<std::uint64_t>(words) * cap);
      r.body = GPUOS_BODY_STREAM;
      r.args[0] = reinterpret_cast<std::uint64_t>(w.src);
      r.args[1] = reinterpret_cast<std::uint64_t>(w.dst);
      r.args[2] = static_cast<std::uint64_t>(words);
      r.args[3] = b.p1 != 0 ? static_cast<std::uint32_t>(b.p1) : salt_of(b.workspace);
      r.args[4] = static_cast<std::uint64_t>(chunks);
      r.words = words;
      r.chunks = chunks;
      break;
    }
    case BodyKind::Spin:
      r.body = GPUOS_BODY_SPIN;
      r.args[0] = static_cast<std::uint64_t>(b.p0);
      break;
    case BodyKind::GemmBf16:
    case BodyKind::GemvBf16:
    case BodyKind::ConvBf16: {
      const TensorBody& t = tensor_body(b);
      if (spec.total_blocks != t.blocks)
        throw ConfigError(std::string(body_kind_name(b.kind)) + " kernel of this shape has " +
                          std::to_string(t.blocks) + " blocks, the descriptor says " +
                          std::to_string(spec.total_blocks));
      r.body = static_cast<std::uint32_t>(b.kind);
      r.args[0] = reinterpret_cast<std::uint64_t>(t.desc);
      break;
    }
    case BodyKind::RmsNormBf16:
    case BodyKind::SiluMulBf16:
    case BodyKind::AttnDecodeBf16: {
      const TensorBody& t = tensor_body(b);
      if (spec.total_blocks != t.blocks)
        throw ConfigError(std::string(body_kind_name(b.kind)) + " kernel of this shape has " +
                          std::to_string(t.blocks) + " blocks, the trace says " +
                          std::to_string(spec.total_blocks));
      r.body = t.body;
      for (int i = 0; i < 5; ++i) r.args[i] = t.args[i];
      break;
    }
    case BodyKind::None:
      break;
  }
  r.parts = 1;
  // Preemption slices apply to CUDA-core bodies; a tensor-core tile runs whole.
  if (opt_.quantum_ns > 0 && (r.body == GPUOS_BODY_STREAM || r.body == GPUOS_BODY_SPIN)) {
    const std::int64_t block_ns = b.kind == BodyKind::Spin ? b.p0 : spec.block_duration_at_fmax;
    std::int64_t parts = (block_ns + opt_.quantum_ns - 1) / opt_.quantum_ns;
    if (r.body == GPUOS_BODY_STREAM) parts = std::min<std::int64_t>(parts, r.words / 4);
    r.parts = static_cast<std::uint32_t>(std::clamp<std::int64_t>(parts, 1, 4096));
  }
  return r;
}

bool B200Runtime::set_run_options(const B200Options& o) {
  if (o.device != opt_.device || o.workers_per_sm != opt_.workers_per_sm ||
      o.idle_sleep_ns != opt_.idle_sleep_ns)
    return false;
  opt_ = o;
  return true;
}

void B200Runtime::reset_kernels() {
  resolved_.clear();
  has_resolved_.clear();
  trace_of_.clear();
  // Keep the chunks; zero what the last run used.
  for (std::size_t c = 0; c < trace_chunks_.size() && c <= trace_chunk_; ++c) {
    const std::uint64_t used = c < trace_chunk_ ? trace_chunk_words_[c] : trace_pool_used_;
    if (used) check(gpuos_dev_memset(dev_, trace_chunks_[c], 0, used * 4), "trace clear");
  }
  trace_chunk_ = 0;
  trace_pool_used_ = 0;
  if (opt_.trace_blocks && trace_chunks_.empty()) {
    void* p = nullptr;  // first chunk up front, outside any run
    check(gpuos_dev_alloc(dev_, kTraceChunkWords * 4, &p), "trace alloc");
    check(gpuos_dev_memset(dev_, p, 0, kTraceChunkWords * 4), "trace clear");
    trace_chunks_.push_back(static_cast<std::uint32_t*>(p));
    trace_chunk_words_.push_back(kTraceChunkWords);
  }
}

void B200Runtime::start() {
  check(gpuos_dev_start(dev_), "gpuos_dev_start");
  running_ = true;
}

float B200Runtime::stop(bool drain) {
  float ms = 0.f;
  running_ = false;
  check(gpuos_dev_stop(dev_, drain ? 1 : 0, &ms), "gpuos_dev_stop");
  return ms;
}

std::uint64_t B200Runtime::workspace_bytes() const {
  std::uint64_t b = 0;
  for (const auto& [id, w] : ws_) b += w.words * 4;
  return b;
}

std::uint64_t B200Runtime::upload_inputs() {
  std::uint64_t bytes = 0;
  for (auto& [id, w] : ws_) {
    check(gpuos_dev_copy(dev_, w.src, w.host_src, w.words * 4, 1), "upload");
    bytes += w.words * 4;
  }
  return bytes;
}

std::uint64_t B200Runtime::download_digest() {
  // The step's result as seen by a tenant: the first 64 KiB of every output.
  std::uint64_t bytes = 0;
  std::vector<std::uint32_t> sink;
  for (auto& [id, w] : ws_) {
    const std::uint64_t n = std::min<std::uint64_t>(w.words, 16384);
    sink.resize(n);
    check(gpuos_dev_copy(dev_, sink.data(), w.dst, n * 4, 2), "download");
    bytes += n * 4;
  }
  return bytes;
}

VerifyReport B200Runtime::verify_kernels(const std::vector<SimKernelSpec>& specs,
                                         const std::vector<KernelPlacement>& placement) {
  VerifyReport rep;
  // Chunks of each workspace that some executed block wrote.
  std::unordered_map<std::uint64_t, std::vector<char>> touched;  // args[1] -> chunks
  std::set<std::uint64_t> verified;  // tensor descriptors already value-checked
  std::vector<std::uint32_t> trace;
  for (std::size_t k = 0; k < specs.size(); ++k) {
    if (k >= has_resolved_.size() || !has_resolved_[k]) continue;
    const Resolved& r = resolved_[k];
    const long blocks = specs[k].total_blocks;
    const KernelPlacement& pl = placement[k];
    if (pl.ranges.empty()) continue;  // never dispatched
    ++rep.kernels;
    rep.blocks += blocks;
    if (!r.trace) continue;
    const long parts = static_cast<long>(r.parts);
    trace.assign(static_cast<std::size_t>(blocks * parts), 0u);
    check(gpuos_dev_copy(dev_, trace.data(), r.trace, blocks * parts * 4ull, 2), "trace download");
    std::vector<char>* tc = nullptr;
    bool complete = true;  // every block of the kernel placed and run once
    long covered = 0;
    for (const auto& rg : pl.ranges) covered += rg.second - rg.first;
    if (covered != blocks) complete = false;
    if (r.body == GPUOS_BODY_STREAM) {
      auto& v = touched[r.args[1]];
      v.resize(static_cast<std::size_t>(r.chunks), 0);
      tc = &v;
    }
    for (std::size_t a = 0; a < pl.ranges.size(); ++a) {
      for (long b = pl.ranges[a].first; b < pl.ranges[a].second; ++b) {
        bool whole = true;
        for (long part = 0; part < parts; ++part) {
          const std::uint32_t v = trace[static_cast<std::size_t>(b * parts + part)];
          const std::uint32_t count = v >> 16;
          if (count != 1) {
            whole = false;
            (count == 0 ? rep.missing : rep.duplicated) += 1;
            continue;
          }
          const int sm = static_cast<int>(v & 0xffffu) - 1;
          const int tpc = sm >> 1;  // identity logical map (gpuos_dev_open)
          if (tpc < 0 || tpc >= GPUOS_MAX_TPCS || !((pl.masks[a][tpc >> 6] >> (tpc & 63)) & 1ull))
            ++rep.misplaced;
        }
        if (tc && whole) (*tc)[static_cast<std::size_t>(b % r.chunks)] = 1;
        complete = complete && whole;
      }
    }
    // A tensor-core kernel every block of which ran: its output values.
    // (Tenant bodies: keyed by their output buffer, args[2].)
    const bool tenant = r.body >= GPUOS_BODY_USER0;
    if (complete && (r.body == GPUOS_BODY_GEMM_BF16 || r.body == GPUOS_BODY_GEMV_BF16 ||
                     r.body == GPUOS_BODY_CONV_BF16 || tenant)) {
      const std::uint64_t key = tenant ? r.args[2] : r.args[0];
      const auto it = tensor_of_desc_.find(key);
      if (it != tensor_of_desc_.end() && verified.insert(key).second) verify_tensor(*it->second, rep);
    }
  }
  // Body outputs against the CPU restatement.
  for (auto& [id, w] : ws_) {
    auto it = touched.find(reinterpret_cast<std::uint64_t>(w.dst));
    if (it == touched.end()) continue;
    // words per chunk: any kernel on this workspace shares the chunk geometry.
    long words = 0;
    std::uint32_t salt = 0;
    for (std::size_t k = 0; k < resolved_.size(); ++k)
      if (has_resolved_[k] && resolved_[k].args[1] == reinterpret_cast<std::uint64_t>(w.dst)) {
        words = resolved_[k].words;
        salt = static_cast<std::uint32_t>(resolved_[k].args[3]);
        break;
      }
    std::vector<std::uint32_t> out(w.words);
    check(gpuos_dev_copy(dev_, out.data(), w.dst, w.words * 4, 2), "output download");
    const auto& chunks = it->second;
    for (std::size_t c = 0; c < chunks.size(); ++c) {
      if (!chunks[c]) continue;
      const std::uint64_t base = c * static_cast<std::uint64_t>(words);
      for (long i = 0; i < words; ++i) {
        const std::uint64_t e = base + static_cast<std::uint64_t>(i);
        ++rep.checked_words;
        if (out[e] != stream_expect(w.host_src[e], salt, e)) ++rep.bad_words;
      }
    }
  }
  return rep;
}

// ============================================================ B200Device
B200Device::B200Device(DeviceTopology topo, FrequencyDomain freq, B200Options opt)
    : opt_(opt), topo_(topo), freq_(std::move(freq)) {
  topo_.validate();
  freq_.validate();
  rt_ = std::make_unique<B200Runtime>(topo_.total_tpcs(), opt);
}

B200Device::~B200Device() {
  if (locked_mhz_ != 0) gpuos_power_lock_sm_clock(opt_.device, 0);  // (best effort)
}

void B200Device::reset_run() {
  if (rt_->running()) throw InvariantError("reset_run while the dispatcher runs");
  rt_->reset_kernels();
  kernels_.clear();
  executed_.clear();
  atom_index_.clear();
  timeline_.clear();
  ready_.clear();
  while (!timers_.empty()) timers_.pop();
  timer_fns_.clear();
  now_ = 0;
  busy_tpc_ns_ = 0.0;
  backpressure_waits_ = 0;
  residency_.clear();
}

SimTime B200Device::host_now() const { return gpuos_dev_now_ns(rt_->handle()) - origin_; }

KernelId B200Device::register_kernel(const SimKernelSpec& spec) {
  spec.validate();
  const KernelId kid = static_cast<KernelId>(kernels_.size());
  kernels_.push_back(spec);
  executed_.push_back(0);
  rt_->resolve(kid, spec);
  return kid;
}

AtomId B200Device::submit_atom(KernelId kernel, long lo, long hi, const std::vector<int>& tpcs,
                               int priority, bool atomized, std::uint64_t tag) {
  return submit_chained(kNoAtom, kernel, lo, hi, tpcs, priority, atomized, tag, false);
}

AtomId B200Device::submit_chained(AtomId after, KernelId kernel, long lo, long hi,
                                  const std::vector<int>& tpcs, int priority, bool atomized,
                                  std::uint64_t tag, bool chain_head, bool no_early) {
  const SimKernelSpec& spec = kernels_.at(kernel);
  if (tpcs.empty()) throw ConfigError("atom needs a non-empty TPC set");
  if (lo < 0 || hi <= lo || hi > spec.total_blocks)
    throw ConfigError("atom block range out of bounds");
  for (int t : tpcs)
    if (t < 0 || t >= topo_.total_tpcs()) throw ConfigError("TPC id out of range");
  if (!rt_->running()) throw InvariantError("submit_atom outside run_all()");
  const B200Runtime::Resolved r = rt_->resolve(kernel, spec);
  const auto m = mask_of(tpcs);
  gpuos_atom_desc d{};
  d.lo = lo;
  d.hi = hi;
  d.tpc_mask[0] = m[0];
  d.tpc_mask[1] = m[1];
  d.priority = priority;
  d.body = r.body;
  std::memcpy(d.args, r.args, sizeof d.args);
  d.tag = tag;
  d.trace = r.trace;
  d.atomized = atomized ? 1 : 0;
  d.parts = r.parts;
  d.after = after == kNoAtom ? 0u : after + 1u;
  d.flags = (chain_head ? GPUOS_ATOM_CHAIN_HEAD : 0u) | (no_early ? GPUOS_ATOM_NO_EARLY : 0u);
  d.tenant = tag < 0xffffu ? static_cast<std::uint32_t>(tag) + 1u : 0u;  // the scheduler tags atoms with their app
  std::uint32_t id = 0;
  // Back-pressure: a TPC holds at most 32 resident atoms and the atom table
  // is finite (the reference has no cap). When either is full, collect
  // completions (queued for step(), not delivered here: no re-entry into
  // the scheduler) until the device frees room; every atom ahead of this
  // one is already submitted, so room always comes.
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(60);
  for (;;) {
    const int rc = gpuos_dev_submit_atom(rt_->handle(), &d, &id);
    if (rc == GPUOS_OK) break;
    if (rc != GPUOS_E_FULL) raise(rc, "gpuos_dev_submit_atom");
    ++backpressure_waits_;
    pump();
    if (std::chrono::steady_clock::now() > deadline)
      throw InvariantError("submit_atom: no room on the device for 60 s");
    std::this_thread::yield();
  }
  AtomTimeline tl{};
  tl.atom = id;
  tl.tag = tag;
  tl.kernel = kernel;
  tl.lo = lo;
  tl.hi = hi;
  tl.priority = priority;
  tl.mask[0] = m[0];
  tl.mask[1] = m[1];
  atom_index_[id] = timeline_.size();
  timeline_.push_back(tl);
  return id;
}

void B200Device::set_atom_paused(AtomId atom, bool paused) {
  check(gpuos_dev_set_atom_paused(rt_->handle(), atom, paused ? 1 : 0), "pause");
}

void B200Device::set_tpc_fence(const std::vector<int>& tpcs, int min_priority, std::uint64_t owner_tag) {
  if (!rt_->running() || tpcs.empty()) return;
  const auto m = mask_of(tpcs);
  const std::uint64_t mask[2] = {m[0], m[1]};
  const std::uint32_t owner = owner_tag < 0xffffu ? static_cast<std::uint32_t>(owner_tag) + 1u : 0u;
  check(gpuos_dev_set_tpc_owner(rt_->handle(), mask, owner, min_priority), "fence");
}

void B200Device::set_pair_fence(const std::vector<int>& tpcs, unsigned pair_slots, int min_priority) {
  if (!rt_->running() || tpcs.empty()) return;
  const auto m = mask_of(tpcs);
  const std::uint64_t mask[2] = {m[0], m[1]};
  check(gpuos_dev_set_pair_fence(rt_->handle(), mask, pair_slots, min_priority), "pair fence");
}

SimTime B200Device::request_frequency(FreqMhz f) {
  if (!freq_.supports(f)) throw ConfigError("unsupported frequency");
  // Actuation (opt-in): the power manager's frequency as a locked SM clock
  // (power_manager.cpp:27-105 decides; device.cpp:221-242 models the
  // switch). Off: clocks stay where the operator set them.
  if (opt_.dvfs_actuate && f != locked_mhz_) {
    if (gpuos_power_lock_sm_clock(opt_.device, static_cast<std::uint32_t>(f)) != GPUOS_OK)
      throw InvariantError("NVML could not lock the SM clock");
    locked_mhz_ = f;
  }
  return now_;
}

void B200Device::schedule_call(SimTime t, std::function<void()> fn) {
  if (t < now_) throw InvariantError("scheduling a call in the past");
  const std::uint64_t seq = timer_seq_++;
  timers_.push(Timer{t, seq});
  timer_fns_.emplace(seq, std::move(fn));
}

void B200Device::pump() {
  gpuos_completion buf[64];
  const int n = gpuos_dev_poll(rt_->handle(), buf, 64);
  if (n < 0) raise(n, "gpuos_dev_poll");
  for (int i = 0; i < n; ++i) {
    const gpuos_completion& c = buf[i];
    auto it = atom_index_.find(c.atom_id);
    if (it == atom_index_.end()) throw InvariantError("completion for unknown atom");
    AtomTimeline& tl = timeline_[it->second];
    tl.host_submit_ns = c.host_submit_ns - origin_;
    tl.host_complete_ns = c.host_complete_ns - origin_;
    tl.dev_first_start_ns = c.dev_first_start_ns - origin_;
    tl.dev_last_end_ns = c.dev_last_end_ns - origin_;
    tl.dev_ingest_ns = c.dev_ingest_ns - origin_;
    tl.dev_armed_ns = c.dev_armed_ns - origin_;
    tl.touched[0] = c.tpc_touched[0];
    tl.touched[1] = c.tpc_touched[1];
    executed_[tl.kernel] += c.blocks;
    ready_.push_back(AtomCompletion{c.atom_id, c.tag, tl.host_submit_ns, tl.host_complete_ns});
  }
}

bool B200Device::step() {
  if (ready_.empty()) pump();
  if (!ready_.empty()) {
    const AtomCompletion c = ready_.front();
    ready_.pop_front();
    now_ = std::max(now_, c.complete_time);
    last_progress_ns_ = host_now();
    if (on_complete_) on_complete_(c);
    return true;
  }
  const SimTime t = host_now();
  if (!timers_.empty() && timers_.top().t <= t) {
    const Timer top = timers_.top();
    timers_.pop();
    auto node = timer_fns_.extract(top.seq);
    now_ = std::max(now_, t);
    node.mapped()();
    return true;
  }
  const int in_flight = gpuos_dev_in_flight(rt_->handle());
  if (timers_.empty() && in_flight == 0) return false;
  now_ = std::max(now_, t);
  // Watchdog: atoms in flight and no completion for stall_timeout_ns -- a
  // live run that stopped making progress fails loudly (with the device's
  // view of the in-flight atoms) instead of spinning until the kernel's
  // 30-minute hang guard.
  if (in_flight == 0) last_progress_ns_ = t;  // (idle: nothing can be stuck)
  if (in_flight > 0 && opt_.stall_timeout_ns > 0 && t - last_progress_ns_ > opt_.stall_timeout_ns) {
    std::string dump(8192, '\0');
    const int n = gpuos_dev_debug_dump(rt_->handle(), dump.data(), static_cast<int32_t>(dump.size()));
    dump.resize(n > 0 ? std::min<std::size_t>(static_cast<std::size_t>(n), dump.size() - 1) : 0);
    throw InvariantError("live run made no progress for " + std::to_string(opt_.stall_timeout_ns / 1000000) +
                         " ms with " + std::to_string(in_flight) + " atoms in flight:\n" + dump);
  }
  if (in_flight == 0 && !timers_.empty()) {
    // Nothing on the GPU: sleep towards the next arrival, waking a full
    // millisecond early (OS sleeps overshoot) and spinning the rest.
    const SimTime gap = timers_.top().t - t;
    if (gap > 2'000'000) std::this_thread::sleep_for(std::chrono::nanoseconds(gap - 1'000'000));
  }
  return true;
}

void B200Device::run_all() {
  gpuos_dev_stats before{};
  gpuos_dev_get_stats(rt_->handle(), &before);
  gpuos_power_sample_t p0{}, p1{};
  const bool nvml = gpuos_power_sample(opt_.device, &p0) == GPUOS_OK;
  rt_->start();
  origin_ = gpuos_dev_now_ns(rt_->handle());
  now_ = 0;
  last_progress_ns_ = 0;
  const auto w0 = std::chrono::steady_clock::now();
  try {
    while (step()) {
    }
  } catch (...) {
    rt_->stop(false);
    throw;
  }
  last_ms_ = rt_->stop(true);
  run_wall_ns_ = std::chrono::duration_cast<std::chrono::nanoseconds>(
                     std::chrono::steady_clock::now() - w0)
                     .count();
  pump();  // nothing should remain; keep the ring consistent regardless
  gpuos_dev_stats st{};
  gpuos_dev_get_stats(rt_->handle(), &st);
  // TPC-ns with >= 1 running block (the reference's definition,
  // device.cpp:264-275), sampled on the device, counted up to the metrics
  // horizon (time after it is scaled out pro rata).
  double busy = static_cast<double>(st.tpc_busy_ns - before.tpc_busy_ns);
  if (horizon_ > 0 && now_ > horizon_) busy *= static_cast<double>(horizon_) / static_cast<double>(now_);
  busy_tpc_ns_ = busy;
  residency_[locked_mhz_ != 0 ? locked_mhz_ : freq_.f_max()] = now_;
  if (nvml && gpuos_power_sample(opt_.device, &p1) == GPUOS_OK) {
    energy_j_ = static_cast<double>(p1.energy_mj - p0.energy_mj) * 1e-3;
    sm_mhz_ = p1.sm_mhz;
    power_mw_ = p1.power_mw;
  }
}

// ============================================================ MirrorDevice
MirrorDevice::MirrorDevice(DeviceTopology topo, FrequencyDomain freq, PowerModel power,
                           B200Options opt)
    : replay_(topo, std::move(freq), power) {
  opt.trace_blocks = true;
  rt_ = std::make_unique<B200Runtime>(topo.total_tpcs(), opt);
  rt_->reset_kernels();  // first trace chunk now: no allocation inside the live run
}

MirrorDevice::~MirrorDevice() = default;

KernelId MirrorDevice::register_kernel(const SimKernelSpec& spec) {
  const KernelId kid = replay_.register_kernel(spec);
  specs_.push_back(spec);
  placement_.emplace_back();
  rt_->resolve(kid, spec);
  return kid;
}

void MirrorDevice::drain_some(bool all) {
  gpuos_completion buf[256];
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(120);
  for (;;) {
    const int n = gpuos_dev_poll(rt_->handle(), buf, 256);
    if (n < 0) raise(n, "gpuos_dev_poll");
    if (!all || gpuos_dev_in_flight(rt_->handle()) == 0) return;
    if (n == 0) std::this_thread::yield();
    if (std::chrono::steady_clock::now() > deadline)
      throw InvariantError("mirror: GPU made no progress for 120 s");
  }
}

AtomId MirrorDevice::submit_atom(KernelId kernel, long lo, long hi, const std::vector<int>& tpcs,
                                 int priority, bool atomized, std::uint64_t tag) {
  const AtomId id = replay_.submit_atom(kernel, lo, hi, tpcs, priority, atomized, tag);
  if (!rt_->running()) rt_->start();
  const B200Runtime::Resolved r = rt_->resolve(kernel, specs_.at(kernel));
  const auto m = mask_of(tpcs);
  gpuos_atom_desc d{};
  d.lo = lo;
  d.hi = hi;
  d.tpc_mask[0] = m[0];
  d.tpc_mask[1] = m[1];
  d.priority = priority;
  d.body = r.body;
  std::memcpy(d.args, r.args, sizeof d.args);
  d.tag = tag;
  d.trace = r.trace;
  d.parts = r.parts;
  std::uint32_t gid = 0;
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(120);
  for (;;) {
    const int rc = gpuos_dev_submit_atom(rt_->handle(), &d, &gid);
    if (rc == GPUOS_OK) break;
    if (rc != GPUOS_E_FULL) raise(rc, "mirror submit");
    drain_some(false);  // the GPU lags the replay clock: wait for room
    std::this_thread::yield();
    if (std::chrono::steady_clock::now() > deadline)
      throw InvariantError("mirror: no room on the GPU for 120 s");
  }
  ++gpu_atoms_;
  placement_[kernel].ranges.emplace_back(lo, hi);
  placement_[kernel].masks.push_back(m);
  drain_some(false);
  return id;
}

void MirrorDevice::run_all() {
  replay_.run_all();
  if (rt_->running()) {
    drain_some(true);
    gpu_ms_ = rt_->stop(true);
  }
}

VerifyReport MirrorDevice::verify() {
  if (rt_->running()) {
    drain_some(true);
    gpu_ms_ = rt_->stop(true);
  }
  return rt_->verify_kernels(specs_, placement_);
}

}  // namespace gpuos
