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
//   args[3] ctx | chunk << 32 (chunk: positions per block, <= 256)
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
constexpr unsigned kHeadDim = 128, kKvHeads = 8, kQPerKv = 4, kQHeads = 32, kMaxChunk = 256;
constexpr unsigned kWsCounters = 8192, kWsPartials = 8448;
}  // namespace gpuos_bodies_attn

GPUOS_USER_BODY(attn_decode_bf16) {
  using namespace gpuos_bodies_attn;
  const unsigned ctx = static_cast<unsigned>(args[3]);
  const unsigned chunk = static_cast<unsigned>(args[3] >> 32);
  const unsigned chunks = b.gx, kvh = b.y, cx = b.x;
  const unsigned p0 = cx * chunk, p1 = p0 + chunk < ctx ? p0 + chunk : ctx;
  const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(args[0]);
  const __nv_bfloat16* kc = reinterpret_cast<const __nv_bfloat16*>(args[1]);
  const __nv_bfloat16* vc = kc + static_cast<size_t>(ctx) * kKvHeads * kHeadDim;
  unsigned char* ws = reinterpret_cast<unsigned char*>(args[2]);
  unsigned* counters = reinterpret_cast<unsigned*>(ws + kWsCounters);
  float* part = reinterpret_cast<float*>(ws + kWsPartials);
  const int warp = b.tid >> 5, lane = b.tid & 31;
  // Shared: scores [4][chunk], per-warp o partials [8 warps][4][128].
  float* sc = reinterpret_cast<float*>(b.smem);
  float* ow = sc + kQPerKv * kMaxChunk;
  __shared__ float red[kQPerKv][8];
  __shared__ unsigned last;

  // This lane's 4 dims (4 lane .. 4 lane + 3) of the 4 query heads, rotated.
  float qr[kQPerKv][4];
  const float pos = static_cast<float>(ctx);
#pragma unroll
  for (unsigned h = 0; h < kQPerKv; ++h) {
    const __nv_bfloat16* qh = q + (kvh * kQPerKv + h) * kHeadDim + 4 * lane;
#pragma unroll
    for (unsigned pr = 0; pr < 2; ++pr) {
      const unsigned i = 2 * lane + pr;  // pair index 0..63
      const float inv = __powf(500000.f, -2.f * static_cast<float>(i) / static_cast<float>(kHeadDim));
      float sn, cs;
      sincosf(pos * inv, &sn, &cs);
      const float x0 = __bfloat162float(qh[2 * pr]), x1 = __bfloat162float(qh[2 * pr + 1]);
      qr[h][2 * pr] = x0 * cs - x1 * sn;
      qr[h][2 * pr + 1] = x0 * sn + x1 * cs;
    }
  }
  const float scale = rsqrtf(static_cast<float>(kHeadDim));
  // Scores: warp w takes positions p0 + w, p0 + w + 8, ...; a lane holds 4
  // dims of the key row (coalesced 256-byte row per position).
  for (unsigned p = p0 + warp; p < p1; p += 8) {
    const uint2 kv2 = *reinterpret_cast<const uint2*>(kc + (static_cast<size_t>(p) * kKvHeads + kvh) * kHeadDim + 4 * lane);
    const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv2);
    const float2 ka = __bfloat1622float2(k2[0]), kb = __bfloat1622float2(k2[1]);
#pragma unroll
    for (unsigned h = 0; h < kQPerKv; ++h) {
      float d = qr[h][0] * ka.x + qr[h][1] * ka.y + qr[h][2] * kb.x + qr[h][3] * kb.y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (lane == 0) sc[h * kMaxChunk + (p - p0)] = d * scale;
    }
  }
  __syncthreads();
  // Chunk max and sum per head (warp h < 4 reduces head h).
  const unsigned n = p1 - p0;
  if (warp < static_cast<int>(kQPerKv)) {
    float m = -INFINITY;
    for (unsigned i = lane; i < n; i += 32) m = fmaxf(m, sc[warp * kMaxChunk + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.f;
    for (unsigned i = lane; i < n; i += 32) {
      const float e = __expf(sc[warp * kMaxChunk + i] - m);
      sc[warp * kMaxChunk + i] = e;
      l += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      red[warp][0] = m;
      red[warp][1] = l;
    }
  }
  __syncthreads();
  // o = sum_p e_p v_p: warp w over positions w, w + 8, ...; lane: 4 dims.
  float acc[kQPerKv][4] = {};
  for (unsigned p = p0 + warp; p < p1; p += 8) {
    const uint2 vv = *reinterpret_cast<const uint2*>(vc + (static_cast<size_t>(p) * kKvHeads + kvh) * kHeadDim + 4 * lane);
    const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vv);
    const float2 va = __bfloat1622float2(v2[0]), vb = __bfloat1622float2(v2[1]);
#pragma unroll
    for (unsigned h = 0; h < kQPerKv; ++h) {
      const float e = sc[h * kMaxChunk + (p - p0)];
      acc[h][0] += e * va.x;
      acc[h][1] += e * va.y;
      acc[h][2] += e * vb.x;
      acc[h][3] += e * vb.y;
    }
  }
#pragma unroll
  for (unsigned h = 0; h < kQPerKv; ++h)
#pragma unroll
    for (unsigned d = 0; d < 4; ++d) ow[(warp * kQPerKv + h) * kHeadDim + 4 * lane + d] = acc[h][d];
  __syncthreads();
  // Partials of this chunk: thread t < 4 x 128 sums its (head, dim) over warps.
  for (unsigned t = b.tid; t < kQPerKv * kHeadDim; t += GPUOS_BLOCK_THREADS) {
    const unsigned h = t / kHeadDim, d = t % kHeadDim;
    float s = 0.f;
#pragma unroll
    for (unsigned w = 0; w < 8; ++w) s += ow[(w * kQPerKv + h) * kHeadDim + d];
    float* ph = part + (static_cast<size_t>(kvh * kQPerKv + h) * chunks + cx) * (2 + kHeadDim);
    ph[2 + d] = s;
    if (d == 0) {
      ph[0] = red[h][0];
      ph[1] = red[h][1];
    }
  }
  // The KV head's last chunk merges (self-resetting counter, as split-K).
  __threadfence();
  __syncthreads();
  if (b.tid == 0) {
    last = atomicAdd(counters + kvh, 1u) == chunks - 1;
    if (last) {
      __threadfence();
      counters[kvh] = 0u;
    }
  }
  __syncthreads();
  if (last) {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ws);
    for (unsigned t = b.tid; t < kQPerKv * kHeadDim; t += GPUOS_BLOCK_THREADS) {
      const unsigned h = t / kHeadDim, d = t % kHeadDim;
      const float* ph = part + static_cast<size_t>(kvh * kQPerKv + h) * chunks * (2 + kHeadDim);
      float M = -INFINITY;
      for (unsigned c = 0; c < chunks; ++c) M = fmaxf(M, __ldcg(ph + c * (2 + kHeadDim)));
      float L = 0.f, O = 0.f;
      for (unsigned c = 0; c < chunks; ++c) {
        const float* pc = ph + c * (2 + kHeadDim);
        const float w = __expf(__ldcg(pc) - M);
        L += __ldcg(pc + 1) * w;
        O += __ldcg(pc + 2 + d) * w;
      }
      out[(kvh * kQPerKv + h) * kHeadDim + d] = __float2bfloat16_rn(O / L);
    }
  }
  __syncthreads();  // (shared scores reused by the worker's next block)
}
