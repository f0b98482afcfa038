// Convolution atom body: implicit GEMM on the TPC pair's tensor cores
// (tcgen05.mma.cta_group::2), NHWC bf16 activations, [K][R][S][Cb] bf16
// weights (Cb = C rounded up to 64, zero-padded), fp32 accumulation, NHWC
// bf16 or fp32 output. The reference models a conv block only as a duration
// (device.hpp:39-47); ResNet traces need the real thing.
//
// GEMM view: M = output pixels, N = K output channels, reduction = (r, s, c).
// A CTA's 128 rows of a pair tile are one output patch of Wb x Hb x Nb
// pixels (Wb Hb Nb = 128; Wb, Hb powers of two covering Q, P). For tap
// (r, s) and a 64-channel slice the patch's input pixels are ONE 4-D TMA
// box of the NHWC tensor: start (c, q0 st - pad + s, p0 st - pad + r, n0),
// traversal strides (1, st, st, 1), box (64, Wb st, Hb st, Nb). Rows land
// in (w, h, n) order with 128-byte swizzle -- exactly the K-major A tile the
// GEMM body uses; padding and patch overhang are the TMA's zero fill (no
// im2col buffer). Weights are a 2-D [K, R S Cb] tensor read like GEMM B.
// Pair tile t covers patches 2t (leader) and 2t + 1 (peer) by 256 output
// channels; block b = (pair tile b % pair_tiles, channel tile b / pair_tiles).
// Algorithmic flops per block: 2 x 256 x 256 x R S C (less the overhang).
//
// args: [0] descriptor from gpuos_dev_conv_desc().
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "bodies.cuh"
#include "gemm_body.cuh"

namespace gpuos_dev_impl {

constexpr unsigned kConvOutBf16 = 1u;

struct alignas(128) ConvDesc {
  CUtensorMap act;               // x [N, H, W, C]: dims {C, W, H, N}, box {64, Wb st, Hb st, Nb}
  CUtensorMap wgt;               // w [K, R S Cb]: box {64, 128}
  unsigned long long y;          // [N, P, Q, K]
  unsigned n, h, w, c, k, r, s, pad, stride, p, q;
  unsigned wb, hb, nb;           // patch (wb hb nb = 128)
  unsigned tiles_q, tiles_p, patches, pair_tiles, k_tiles, c_blocks, flags;
};

__device__ __forceinline__ void tma_load_4d_pair(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 int c2, int c3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)) & 0xFEFFFFFFu)
      : "memory");
}

// Both CTAs of the pair, all threads; rank 0 is the leader. Shares the GEMM
// pipe (stage = 16 KiB A + 16 KiB B, same barriers and TMEM columns).
__device__ __forceinline__ void body_conv2(const BlockCmd& c, int tid, unsigned rank, GemmPipe& G) {
  const ConvDesc* D = reinterpret_cast<const ConvDesc*>(c.args[0]);
  const unsigned pt = static_cast<unsigned>(c.block) % D->pair_tiles;
  const unsigned kt = static_cast<unsigned>(c.block) / D->pair_tiles;
  const unsigned patch = 2 * pt + rank;
  const unsigned pq = patch % D->tiles_q, pp = (patch / D->tiles_q) % D->tiles_p;
  const unsigned pn = patch / (D->tiles_q * D->tiles_p);
  const int q0 = static_cast<int>(pq * D->wb), p0 = static_cast<int>(pp * D->hb);
  const int n0 = static_cast<int>(pn * D->nb);
  const unsigned taps = D->r * D->s;
  const unsigned nk = taps * D->c_blocks;
  const unsigned S = G.stages;
  const unsigned long long g0 = G.kb_used;
  if (S == 0) {
    cluster_sync_all();
    return;
  }
  if (tid == 0) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&D->act) : "memory");
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&D->wgt) : "memory");
    const int st = static_cast<int>(D->stride), pad = static_cast<int>(D->pad);
    const int k_row = static_cast<int>(kt * kGemmTile + rank * kGemmHalf);
    const unsigned cb_count = D->c_blocks;
    for (unsigned j = 0; j < nk; ++j) {
      const unsigned tap = j / cb_count, cb = j - tap * cb_count;
      const int rr = static_cast<int>(tap / D->s), ss = static_cast<int>(tap % D->s);
      const unsigned long long k = g0 + j;
      const unsigned s = static_cast<unsigned>(k % S);
      const unsigned long long r = k / S;
      if (r >= 1) mbar_wait_bounded(G.empty + s, static_cast<unsigned>((r - 1) & 1));
      unsigned char* stg = G.tiles + s * kGemmStageBytes;
      if (rank == 0) mbar_expect_tx(G.full + s, 2 * kGemmStageBytes);
      tma_load_4d_pair(stg, &D->act, static_cast<int>(cb * kGemmBK), q0 * st - pad + ss,
                       p0 * st - pad + rr, n0, G.full + s);
      tma_load_2d_pair(stg + kGemmABytes, &D->wgt, static_cast<int>(j * kGemmBK), k_row, G.full + s);
    }
  } else if (tid == 32 && rank == 0) {
    tc_fence_after();
    const unsigned idesc = umma_idesc_bf16(kGemmTile, kGemmTile);
    for (unsigned j = 0; j < nk; ++j) {
      const unsigned long long k = g0 + j;
      const unsigned s = static_cast<unsigned>(k % S);
      mbar_wait_bounded(G.full + s, static_cast<unsigned>((k / S) & 1));
      tc_fence_after();
      const unsigned a0 = smem_u32(G.tiles + s * kGemmStageBytes);
      const unsigned b0 = a0 + kGemmABytes;
#pragma unroll
      for (unsigned kk = 0; kk < kGemmBK / 16; ++kk)
        umma2_bf16(G.tmem, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                   (j | kk) != 0u);
      umma2_commit_both(G.empty + s);
    }
    umma2_commit_both(G.accum);
  }
  // Epilogue: TMEM lane i of this CTA = patch pixel i in (w, h, n) order.
  mbar_wait_bounded(G.accum, G.accum_used & 1u);
  tc_fence_after();
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned qd = static_cast<unsigned>(warp & 3), h = static_cast<unsigned>(warp >> 2);
  constexpr unsigned half = kGemmTile / 2;
  const unsigned i = qd * 32 + static_cast<unsigned>(lane);
  const unsigned oq = static_cast<unsigned>(q0) + i % D->wb;
  const unsigned op = static_cast<unsigned>(p0) + (i / D->wb) % D->hb;
  const unsigned on = static_cast<unsigned>(n0) + i / (D->wb * D->hb);
  const bool valid = oq < D->q && op < D->p && on < D->n;
  const size_t orow = (static_cast<size_t>(on) * D->p + op) * D->q + oq;
  const unsigned K = D->k;
  const bool bf16_out = (D->flags & kConvOutBf16) != 0;
#pragma unroll 1
  for (unsigned ch = 0; ch < half / 32; ++ch) {
    const unsigned col0 = kt * kGemmTile + h * half + ch * 32u;
    if (col0 >= K) break;  // warp-uniform: narrow layers skip the empty columns
    unsigned v[32];
    tmem_ld32(G.tmem + ((qd * 32u) << 16) + h * half + ch * 32u, v);
    if (!valid) continue;
    const bool full_row = col0 + 32 <= K;
    if (!bf16_out) {
      float* out = reinterpret_cast<float*>(D->y) + orow * K + col0;
      if (full_row && (K % 4) == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          st_stream(reinterpret_cast<uint4*>(out) + e,
                    make_uint4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]));
      } else {
#pragma unroll
        for (unsigned e = 0; e < 32; ++e)
          if (col0 + e < K) out[e] = __uint_as_float(v[e]);
      }
    } else {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(D->y) + orow * K + col0;
      if (full_row && (K % 8) == 0) {
        unsigned pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const __nv_bfloat162 t2 = __floats2bfloat162_rn(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
          pk[e] = *reinterpret_cast<const unsigned*>(&t2);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          st_stream(reinterpret_cast<uint4*>(out) + e, make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]));
      } else {
#pragma unroll
        for (unsigned e = 0; e < 32; ++e)
          if (col0 + e < K) out[e] = __float2bfloat16_rn(__uint_as_float(v[e]));
      }
    }
  }
  tc_fence_before();
  G.kb_used = g0 + nk;
  G.accum_used += 1;
  cluster_sync_all();  // both patches written, both TMEMs read
}

}  // namespace gpuos_dev_impl
