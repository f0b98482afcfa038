// Decode attention as a tenant body (include/gpuos_body.cuh): one token of
// Llama-3-8B grouped-query attention over a KV cache -- 32 query heads of
// 128, 8 KV heads (4 query heads each), RoPE on the query -- split over the
// context (flash-decoding): block (x, y) = context chunk x of KV head y.
//
// attn_decode_bf16:
//   args[0] q   bf16 [32][128] (this token's query, before RoPE)
//   args[1] kv  bf16 K cache [ctx][8][128] followed by V cache [ctx][8][128]
//               (keys stored already rotated)
//   args[2] ws  workspace: o bf16 [32][128] at 0 (the result), arrival
//               counters u32 [8] at 8192 (zero; self-resetting), partials
//               fp32 [32][chunks][2 + 128] at 8448
//   args[3] ctx | chunk << 32 (chunk: positions per block, <= 32)
//   args[4] GPUOS_GRID(chunks, 8)
// Query position = ctx (the cache holds positions 0 .. ctx-1); RoPE base
// 500000 on interleaved pairs (2i, 2i+1). Each block writes, per query
// head, its chunk's running max m, sum l = sum exp(s - m) and o = sum
// exp(s - m) v; the KV head's last block (arrival counter) merges the
// chunks in chunk order (deterministic) and writes o / l as bf16.
// fp32 arithmetic throughout; HBM-bound on the cache (4 KiB of K and V per
// position across the 8 heads).
#include <cuda_bf16.h>

#include "gpuos_body.cuh"

namespace gpuos_bodies_attn {
constexpr unsigned kHeadDim = 128, kKvHeads = 8, kQPerKv = 4, kQHeads = 32, kMaxChunk = 32;
constexpr unsigned kPerWarp = kMaxChunk / 8;  // positions per warp
constexpr unsigned kMaxChunks = 256;          // context chunks merged per head
constexpr unsigned kWsCounters = 8192, kWsPartials = 8448;
}  // namespace gpuos_bodies_attn

GPUOS_USER_BODY(attn_decode_bf16) {
  using namespace gpuos_bodies_attn;
  const unsigned ctx = static_cast<unsigned>(args[3]);
  const unsigned chunk = static_cast<unsigned>((args[3] >> 32) & 0x7fffffffu);
  // Profiling (args[3] bit 63): 4 globaltimer stamps per block after the
  // partials (start, K/V loaded, partials written, end).
  unsigned long long* stamps = nullptr;
  const unsigned chunks = b.gx, kvh = b.y, cx = b.x;
  const unsigned p0 = cx * chunk, p1 = p0 + chunk < ctx ? p0 + chunk : ctx;
  const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(args[0]);
  const __nv_bfloat16* kc = reinterpret_cast<const __nv_bfloat16*>(args[1]);
  const __nv_bfloat16* vc = kc + static_cast<size_t>(ctx) * kKvHeads * kHeadDim;
  unsigned char* ws = reinterpret_cast<unsigned char*>(args[2]);
  unsigned* counters = reinterpret_cast<unsigned*>(ws + kWsCounters);
  float* part = reinterpret_cast<float*>(ws + kWsPartials);
  if (args[3] >> 63)
    stamps = reinterpret_cast<unsigned long long*>(ws + kWsPartials + 4ull * kQHeads * chunks * (2 + kHeadDim)) +
             4ull * static_cast<unsigned long long>(b.block);
  auto stamp = [&](int i) {
    if (stamps && b.tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      stamps[i] = t;
    }
  };
  stamp(0);
  const int warp = b.tid >> 5, lane = b.tid & 31;
  // Shared: per-warp o partials [8 warps][4][128], the per-warp max / sum of
  // each head, the merge flag; the merge reuses the o area.
  float* ow = reinterpret_cast<float*>(b.smem);
  float* wm = ow + 8 * kQPerKv * kHeadDim;  // [8 warps][4 heads][2]
  unsigned* last = reinterpret_cast<unsigned*>(wm + 8 * kQPerKv * 2);

  // Warp w owns positions p0 + w + 8 i (i < kPerWarp): every K and V row it
  // needs is loaded up front (one memory latency, not one per position); a
  // lane holds 4 of the 128 dims (coalesced 256-byte rows).
  uint2 kr[kPerWarp], vr[kPerWarp];
#pragma unroll
  for (unsigned i = 0; i < kPerWarp; ++i) {
    const unsigned p = p0 + warp + 8 * i;
    const size_t off = (static_cast<size_t>(p < p1 ? p : p0) * kKvHeads + kvh) * kHeadDim + 4 * lane;
    kr[i] = *reinterpret_cast<const uint2*>(kc + off);
    vr[i] = *reinterpret_cast<const uint2*>(vc + off);
  }
  stamp(1);  // (loads issued; their latency lands on the first use below)
  // This lane's 4 dims of the 4 query heads, rotated (RoPE at position ctx).
  float qr[kQPerKv][4];
  const float pos = static_cast<float>(ctx);
#pragma unroll
  for (unsigned pr = 0; pr < 2; ++pr) {
    const unsigned i = 2 * lane + pr;  // pair index 0..63
    const float inv = exp2f(-2.f * static_cast<float>(i) / static_cast<float>(kHeadDim) * 18.931568569324174f);  // 500000^-2i/128
    float sn, cs;
    sincosf(pos * inv, &sn, &cs);
#pragma unroll
    for (unsigned h = 0; h < kQPerKv; ++h) {
      const __nv_bfloat16* qh = q + (kvh * kQPerKv + h) * kHeadDim + 4 * lane;
      const float x0 = __bfloat162float(qh[2 * pr]), x1 = __bfloat162float(qh[2 * pr + 1]);
      qr[h][2 * pr] = x0 * cs - x1 * sn;
      qr[h][2 * pr + 1] = x0 * sn + x1 * cs;
    }
  }
  const float scale = rsqrtf(static_cast<float>(kHeadDim));
  // Scores (4 heads x kPerWarp positions, warp reductions interleaved).
  float s[kPerWarp][kQPerKv];
#pragma unroll
  for (unsigned i = 0; i < kPerWarp; ++i) {
    const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kr[i]);
    const float2 ka = __bfloat1622float2(k2[0]), kb = __bfloat1622float2(k2[1]);
#pragma unroll
    for (unsigned h = 0; h < kQPerKv; ++h) s[i][h] = qr[h][0] * ka.x + qr[h][1] * ka.y + qr[h][2] * kb.x + qr[h][3] * kb.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (unsigned i = 0; i < kPerWarp; ++i)
#pragma unroll
      for (unsigned h = 0; h < kQPerKv; ++h) s[i][h] += __shfl_xor_sync(0xffffffffu, s[i][h], o);
  float m[kQPerKv], l[kQPerKv];
#pragma unroll
  for (unsigned h = 0; h < kQPerKv; ++h) {
    m[h] = -INFINITY;
#pragma unroll
    for (unsigned i = 0; i < kPerWarp; ++i)
      if (p0 + warp + 8 * i < p1) m[h] = fmaxf(m[h], s[i][h] * scale);
  }
  if (lane == 0)
#pragma unroll
    for (unsigned h = 0; h < kQPerKv; ++h) wm[(warp * kQPerKv + h) * 2] = m[h];
  __syncthreads();
  // Chunk max per head, then weights e = exp(s - M) and this warp's o.
  float M[kQPerKv];
#pragma unroll
  for (unsigned h = 0; h < kQPerKv; ++h) {
    M[h] = -INFINITY;
#pragma unroll
    for (unsigned w = 0; w < 8; ++w) M[h] = fmaxf(M[h], wm[(w * kQPerKv + h) * 2]);
    l[h] = 0.f;
  }
  float acc[kQPerKv][4] = {};
#pragma unroll
  for (unsigned i = 0; i < kPerWarp; ++i) {
    if (p0 + warp + 8 * i >= p1) continue;
    const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vr[i]);
    const float2 va = __bfloat1622float2(v2[0]), vb = __bfloat1622float2(v2[1]);
#pragma unroll
    for (unsigned h = 0; h < kQPerKv; ++h) {
      const float e = __expf(s[i][h] * scale - M[h]);
      l[h] += e;
      acc[h][0] += e * va.x;
      acc[h][1] += e * va.y;
      acc[h][2] += e * vb.x;
      acc[h][3] += e * vb.y;
    }
  }
  __syncthreads();  // (every warp has read the maxima before wm is reused)
#pragma unroll
  for (unsigned h = 0; h < kQPerKv; ++h) {
#pragma unroll
    for (unsigned d = 0; d < 4; ++d) ow[(warp * kQPerKv + h) * kHeadDim + 4 * lane + d] = acc[h][d];
    if (lane == 0) wm[(warp * kQPerKv + h) * 2 + 1] = l[h];
  }
  __syncthreads();
  // This chunk's partials: thread t < 4 x 128 sums its (head, dim) over warps
  // (all relative to the chunk max M).
  for (unsigned t = b.tid; t < kQPerKv * kHeadDim; t += GPUOS_BLOCK_THREADS) {
    const unsigned h = t / kHeadDim, d = t % kHeadDim;
    float o = 0.f;
#pragma unroll
    for (unsigned w = 0; w < 8; ++w) o += ow[(w * kQPerKv + h) * kHeadDim + d];
    float* ph = part + (static_cast<size_t>(kvh * kQPerKv + h) * chunks + cx) * (2 + kHeadDim);
    ph[2 + d] = o;
    if (d == 0) {
      float mm = -INFINITY, ll = 0.f;
#pragma unroll
      for (unsigned w = 0; w < 8; ++w) {
        mm = fmaxf(mm, wm[(w * kQPerKv + h) * 2]);
        ll += wm[(w * kQPerKv + h) * 2 + 1];
      }
      ph[0] = mm;
      ph[1] = ll;
    }
  }
  stamp(2);
  // The KV head's last chunk merges (self-resetting counter, as split-K):
  // the block's partials precede its count (CTA barrier, then a release
  // add), and the last block's acquire sees every other block's.
  __syncthreads();
  if (b.tid == 0) {
    unsigned before;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(before) : "l"(counters + kvh) : "memory");
    *last = before == chunks - 1;
    if (*last) counters[kvh] = 0u;  // (ready for the kernel's next run)
  }
  __syncthreads();
  if (*last) {
    // Merge. The KV head's partials -- [4 heads][chunks][m, l, o[128]],
    // contiguous -- are copied into shared memory with cp.async (every
    // 16-byte piece in flight at once: one L2 round trip on the critical
    // path, no registers held); warp h turns head h's (m, l) into weights
    // w = exp(m_c - M) / L (M the head's max, L = sum l_c exp(m_c - M)),
    // then each thread sums its two (head, dim) outputs over the chunks.
    const unsigned row = 2 + kHeadDim;
    const unsigned long long bytes = 4ull * kQPerKv * chunks * row;
    float* P = reinterpret_cast<float*>(b.smem);  // [4][chunks][row]
    float* W = P + kQPerKv * chunks * row;        // [4][chunks] weights
    if (bytes + 4ull * kQPerKv * chunks <= b.smem_bytes) {
      const unsigned char* src = reinterpret_cast<const unsigned char*>(part + static_cast<size_t>(kvh) * kQPerKv * chunks * row);
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(P));
      for (unsigned q16 = b.tid; q16 < bytes / 16; q16 += GPUOS_BLOCK_THREADS)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * q16), "l"(src + 16ull * q16) : "memory");
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
      __syncthreads();
      if (warp < static_cast<int>(kQPerKv)) {  // warp h: head h's weights
        const unsigned h = static_cast<unsigned>(warp);
        float Mx = -INFINITY;
        for (unsigned c = lane; c < chunks; c += 32) Mx = fmaxf(Mx, P[(h * chunks + c) * row]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
        float L = 0.f;
        for (unsigned c = lane; c < chunks; c += 32) {
          const float w = __expf(P[(h * chunks + c) * row] - Mx);
          W[h * chunks + c] = w;
          L += P[(h * chunks + c) * row + 1] * w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        const float inv = 1.f / L;
        for (unsigned c = lane; c < chunks; c += 32) W[h * chunks + c] *= inv;
      }
      __syncthreads();
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ws) + kvh * kQPerKv * kHeadDim;
      for (unsigned t = b.tid; t < kQPerKv * kHeadDim; t += GPUOS_BLOCK_THREADS) {
        const unsigned h = t / kHeadDim, d = t % kHeadDim;
        float O = 0.f;
        for (unsigned c = 0; c < chunks; ++c) O += W[h * chunks + c] * P[(h * chunks + c) * row + 2 + d];
        out[t] = __float2bfloat16_rn(O);
      }
    } else {
      // (more chunks than shared memory holds: the same merge from L2)
      float* mw = ow;  // [4][kMaxChunks]
      float* lw = mw + kQPerKv * kMaxChunks;
      for (unsigned t = b.tid; t < kQPerKv * chunks; t += GPUOS_BLOCK_THREADS) {
        const unsigned h = t / chunks, c = t % chunks;
        const float* pc = part + (static_cast<size_t>(kvh * kQPerKv + h) * chunks + c) * row;
        mw[h * kMaxChunks + c] = __ldcg(pc);
        lw[h * kMaxChunks + c] = __ldcg(pc + 1);
      }
      __syncthreads();
      if (warp < static_cast<int>(kQPerKv)) {
        const unsigned h = static_cast<unsigned>(warp);
        float Mx = -INFINITY;
        for (unsigned c = lane; c < chunks; c += 32) Mx = fmaxf(Mx, mw[h * kMaxChunks + c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
        float L = 0.f;
        for (unsigned c = lane; c < chunks; c += 32) {
          const float w = __expf(mw[h * kMaxChunks + c] - Mx);
          mw[h * kMaxChunks + c] = w;
          L += lw[h * kMaxChunks + c] * w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        const float inv = 1.f / L;
        for (unsigned c = lane; c < chunks; c += 32) mw[h * kMaxChunks + c] *= inv;
      }
      __syncthreads();
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ws);
      for (unsigned t = b.tid; t < kQPerKv * kHeadDim; t += GPUOS_BLOCK_THREADS) {
        const unsigned h = t / kHeadDim, d = t % kHeadDim;
        const float* ph = part + static_cast<size_t>(kvh * kQPerKv + h) * chunks * row + 2 + d;
        float O = 0.f;
#pragma unroll 16
        for (unsigned c = 0; c < chunks; ++c) O += mw[h * kMaxChunks + c] * __ldcg(ph + c * row);
        out[(kvh * kQPerKv + h) * kHeadDim + d] = __float2bfloat16_rn(O);
      }
    }
  }
  stamp(3);
  __syncthreads();  // (shared memory reused by the worker's next block)
}
