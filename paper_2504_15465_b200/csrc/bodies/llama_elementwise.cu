// Tenant bodies written against include/gpuos_body.cuh, compiled into the
// dispatcher by the body plug-in build (build.py): the elementwise kernels
// of a Llama decode step, which the model traces otherwise model as
// byte-equivalent STREAM kernels (models.py).
//
// rmsnorm_bf16: y[r] = x[r] * rsqrt(mean(x[r]^2) + eps) * w, block b = row b.
//   args: [0] x bf16 [rows, d], [1] w bf16 [d], [2] y bf16 [rows, d],
//         [3] d | float_bits(eps) << 32. 16-byte aligned rows, d % 8 == 0.
// silu_mul_bf16: out[i] = silu(gate[i]) * up[i] over the block's chunk.
//   args: [0] gate bf16, [1] up bf16, [2] out bf16, [3] n | chunk << 32
//         (chunk % 8 == 0, 16-byte aligned arrays); block b covers
//         [b chunk, min(n, (b + 1) chunk)).
// Both: fp32 arithmetic, one bf16 rounding of the result. HBM-bound: 128-bit
// loads and stores, every byte read and written once.
#include <cuda_bf16.h>

#include "gpuos_body.cuh"

namespace gpuos_bodies_llama {

__device__ __forceinline__ void unpack8(const uint4& v, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 p = __bfloat1622float2(h[i]);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

}  // namespace gpuos_bodies_llama

GPUOS_USER_BODY(rmsnorm_bf16) {
  using namespace gpuos_bodies_llama;
  const unsigned d = static_cast<unsigned>(args[3]);
  const float eps = __uint_as_float(static_cast<unsigned>(args[3] >> 32));
  const uint4* x = reinterpret_cast<const uint4*>(args[0]) + static_cast<size_t>(b.block) * (d / 8);
  const uint4* w = reinterpret_cast<const uint4*>(args[1]);
  uint4* y = reinterpret_cast<uint4*>(args[2]) + static_cast<size_t>(b.block) * (d / 8);
  const unsigned vecs = d / 8;
  float ss = 0.f;
  for (unsigned i = b.tid; i < vecs; i += GPUOS_BLOCK_THREADS) {
    float f[8];
    unpack8(x[i], f);
#pragma unroll
    for (int k = 0; k < 8; ++k) ss += f[k] * f[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  float* red = reinterpret_cast<float*>(b.smem);
  if ((b.tid & 31) == 0) red[b.tid >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int k = 0; k < GPUOS_BLOCK_THREADS / 32; ++k) tot += red[k];
  const float scale = rsqrtf(tot / static_cast<float>(d) + eps);
  for (unsigned i = b.tid; i < vecs; i += GPUOS_BLOCK_THREADS) {
    float f[8], g[8];
    unpack8(x[i], f);
    unpack8(w[i], g);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = f[k] * scale * g[k];
    y[i] = pack8(f);
  }
  __syncthreads();  // (red is reused by the next block)
}

GPUOS_USER_BODY(silu_mul_bf16) {
  using namespace gpuos_bodies_llama;
  const unsigned long long n = static_cast<unsigned>(args[3]);
  const unsigned long long chunk = args[3] >> 32;
  const unsigned long long lo = static_cast<unsigned long long>(b.block) * chunk;
  const unsigned long long hi = lo + chunk < n ? lo + chunk : n;
  const uint4* g = reinterpret_cast<const uint4*>(args[0]);
  const uint4* u = reinterpret_cast<const uint4*>(args[1]);
  uint4* o = reinterpret_cast<uint4*>(args[2]);
  for (unsigned long long e = lo + 8ull * b.tid; e < hi; e += 8ull * GPUOS_BLOCK_THREADS) {
    float gf[8], uf[8];
    if (e + 8 <= hi) {
      unpack8(g[e / 8], gf);
      unpack8(u[e / 8], uf);
#pragma unroll
      for (int k = 0; k < 8; ++k) gf[k] = gf[k] / (1.f + __expf(-gf[k])) * uf[k];
      o[e / 8] = pack8(gf);
    } else {  // ragged tail (n % 8)
      const __nv_bfloat16* gs = reinterpret_cast<const __nv_bfloat16*>(args[0]);
      const __nv_bfloat16* us = reinterpret_cast<const __nv_bfloat16*>(args[1]);
      __nv_bfloat16* os = reinterpret_cast<__nv_bfloat16*>(args[2]);
      for (unsigned long long i = e; i < hi; ++i) {
        const float gv = __bfloat162float(gs[i]);
        os[i] = __float2bfloat16_rn(gv / (1.f + __expf(-gv)) * __bfloat162float(us[i]));
      }
    }
  }
}

// The prelude's index recovery, observable: out[linear block] =
// x | y << 10 | z << 20 (args[0]: u32 out).
GPUOS_USER_BODY(grid_probe) {
  if (b.tid == 0)
    reinterpret_cast<unsigned*>(args[0])[b.block] = b.x | (b.y << 10) | (b.z << 20);
}
