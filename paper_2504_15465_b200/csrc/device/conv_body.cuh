// Convolution atom body: implicit GEMM on the TPC pair's tensor cores
// (tcgen05.mma.cta_group::2), NHWC bf16 activations, [K][R][S][Cb] bf16
// weights (Cb = C rounded up to 64, zero-padded), fp32 accumulation, NHWC
// bf16 or fp32 output. The reference models a conv block only as a duration
// (device.hpp:39-47); ResNet traces need the real thing.
//
// GEMM view: M = output pixels (n, p, q) in NPQ order, N = K output
// channels, reduction = (r, s, c). A CTA's 128 rows of a pair tile are 128
// consecutive output pixels -- across row and image boundaries -- loaded by
// the TMA's im2col mode: the activation map is encoded with the filter's
// bounding box (lower corner -pad, upper corner pad - (R - 1) per spatial
// dim, traversal stride = conv stride), so one cp.async.bulk.tensor ...
// .im2col per (tap, 64-channel slice) gathers the 128 pixels' input
// channels at offset (s, r) from each pixel's window origin, padding and
// the tail past the last image as zero fill (no im2col buffer, no padded
// patches: every MMA row is a real output pixel except the final tile's
// tail). Semantics pinned on the hardware by scratch/im2col_probe.cu:
// pixel i of a load is the i-th window origin after (w0, h0, n0) in
// (w, h, n) order over the bounding box. Rows land with 128-byte swizzle
// -- the K-major A tile the GEMM body uses. Weights are a 2-D [K, R S Cb]
// tensor read like GEMM B. Pair tile t covers pixels [256 t, 256 t + 256)
// (leader the first 128) by 256 output channels; block b = (pair tile
// b % pair_tiles, channel tile b / pair_tiles).
// Algorithmic flops per block: 2 x 256 x 256 x R S C (less the tail).
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
  CUtensorMap act;               // x [N, H, W, C]: im2col map, 64 channels x 128 pixels per load
  CUtensorMap wgt;               // w [K, R S Cb]: box {64, 128}
  unsigned long long y;          // [N, P, Q, K]
  unsigned n, h, w, c, k, r, s, pad, stride, p, q;
  unsigned pixels;               // N P Q
  unsigned pair_tiles, k_tiles, c_blocks, flags;
  unsigned n_tile;               // output channels per block: 64, 128 or 256
  unsigned pad0;
  unsigned long long* timing;    // optional: 4 globaltimer stamps per tile (profiling, tools/conv_batch.py)
};
static_assert(offsetof(ConvDesc, timing) == 336, "ConvDesc layout (tools/conv_batch.py)");

__device__ __forceinline__ void tma_load_im2col_pair(void* dst, const CUtensorMap* map, int c0, int w0,
                                                     int h0, int n0, unsigned short off_w,
                                                     unsigned short off_h, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
      "l"(map), "r"(c0), "r"(w0), "r"(h0), "r"(n0),
      "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)) & 0xFEFFFFFFu), "h"(off_w), "h"(off_h)
      : "memory");
}

// Both CTAs of the pair, all threads; rank 0 is the leader. Shares the GEMM
// pipe (stage = 16 KiB A + 16 KiB B, same barriers and TMEM columns).
// `gate`: early-start gate, as in body_gemm2 (weights first, activations
// once the predecessor has written them).
template <class NextTile>
__device__ __forceinline__ void conv2_tile(const ConvDesc* D, unsigned blk, int tid, unsigned rank,
                                           GemmPipe& G, const unsigned* gate, NextTile& next_tile) {
  const unsigned pt = blk % D->pair_tiles;
  const unsigned kt = blk / D->pair_tiles;
  const unsigned m0 = pt * kGemmTile + rank * kGemmHalf;  // this CTA's first output pixel
  const unsigned pq = D->p * D->q;
  const unsigned n0 = m0 / pq, rem = m0 - n0 * pq;
  const unsigned p0 = rem / D->q, q0 = rem - p0 * D->q;
  const unsigned taps = D->r * D->s;
  const unsigned nk = taps * D->c_blocks;
  const unsigned S = G.stages;
  const unsigned long long g0 = G.kb_used;
  if (S == 0) {
    if (tid == 0 && rank == 0) next_tile(true);  // (ends the run)
    cluster_sync_all();
    return;
  }
  unsigned long long* tm = D->timing != nullptr && rank == 0 ? D->timing + 4ull * blk : nullptr;
  if (tm && tid == 0) tm[0] = gtimer();
  if (tid == 0) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&D->act) : "memory");
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&D->wgt) : "memory");
    const int st = static_cast<int>(D->stride), pad = static_cast<int>(D->pad);
    const int w0 = static_cast<int>(q0) * st - pad, h0 = static_cast<int>(p0) * st - pad;
    const unsigned n_tile = D->n_tile;
    const int k_row = static_cast<int>(kt * n_tile + rank * (n_tile / 2));
    const unsigned tx = 2 * (kGemmABytes + n_tile / 2 * kGemmBK * 2);  // both CTAs' A and B halves
    const unsigned cb_count = D->c_blocks;
    // Weights for the first stages first, then activations once the atom's
    // gate is open (early start; otherwise the gate read overlaps).
    const unsigned pre = gate ? (nk < S ? nk : S) : 0u;  // (no gate: loads in stage order)
    for (unsigned j = 0; j < pre; ++j) {
      const unsigned s = static_cast<unsigned>((g0 + j) % S);
      if ((g0 + j) / S >= 1) mbar_wait_bounded(G.empty + s, static_cast<unsigned>(((g0 + j) / S - 1) & 1), *G.guard);
      if (rank == 0) mbar_expect_tx(G.full + s, tx);
      tma_load_2d_pair(G.tiles + s * kGemmStageBytes + kGemmABytes, &D->wgt, static_cast<int>(j * kGemmBK),
                       k_row, G.full + s);
    }
    if (gate) {
      gate_spin(gate, *G.guard);  // DevAtom::paused, kGatedBit
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    for (unsigned j = 0; j < pre; ++j) {
      const unsigned tap = j / cb_count, cb = j - tap * cb_count;
      const unsigned rr = tap / D->s, ss = tap - rr * D->s;
      const unsigned s = static_cast<unsigned>((g0 + j) % S);
      tma_load_im2col_pair(G.tiles + s * kGemmStageBytes, &D->act, static_cast<int>(cb * kGemmBK), w0, h0,
                           static_cast<int>(n0), static_cast<unsigned short>(ss),
                           static_cast<unsigned short>(rr), G.full + s);
    }
    for (unsigned j = pre; j < nk; ++j) {
      const unsigned tap = j / cb_count, cb = j - tap * cb_count;
      const unsigned rr = tap / D->s, ss = tap - rr * D->s;
      const unsigned long long k = g0 + j;
      const unsigned s = static_cast<unsigned>(k % S);
      const unsigned long long r = k / S;
      if (r >= 1) mbar_wait_bounded(G.empty + s, static_cast<unsigned>((r - 1) & 1), *G.guard);
      unsigned char* stg = G.tiles + s * kGemmStageBytes;
      if (rank == 0) mbar_expect_tx(G.full + s, tx);
      tma_load_im2col_pair(stg, &D->act, static_cast<int>(cb * kGemmBK), w0, h0, static_cast<int>(n0),
                           static_cast<unsigned short>(ss), static_cast<unsigned short>(rr), G.full + s);
      tma_load_2d_pair(stg + kGemmABytes, &D->wgt, static_cast<int>(j * kGemmBK), k_row, G.full + s);
    }
    if (rank == 0) next_tile();  // claim + post the run's next tile (body_gemm2)
  } else if (tid == 32 && rank == 0) {
    if (gate) gate_spin(gate, *G.guard);  // the bounded waits measure the pipeline only
    tc_fence_after();
    const unsigned idesc = umma_idesc_bf16(kGemmTile, D->n_tile);
    for (unsigned j = 0; j < nk; ++j) {
      const unsigned long long k = g0 + j;
      const unsigned s = static_cast<unsigned>(k % S);
      mbar_wait_bounded(G.full + s, static_cast<unsigned>((k / S) & 1), *G.guard);
      tc_fence_after();
      if (tm && j == 0) tm[1] = gtimer();
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
  // Epilogue: TMEM lane i of this CTA = output pixel m0 + i (NPQ order).
  gate_wait(gate, *G.guard);  // (unbounded: the predecessor may run long)
  mbar_wait_bounded(G.accum, G.accum_used & 1u, *G.guard);
  tc_fence_after();
  if (tm && tid == 0) tm[2] = gtimer();
  // The tile's rows are consecutive rows of the [N P Q, K] output: the
  // GEMM body's staged, coalesced epilogue applies as is.
  const unsigned col0 = kt * D->n_tile;
  epilogue_staged(G, tid, m0, col0, D->pixels, D->k - col0 < D->n_tile ? D->k : col0 + D->n_tile, D->k,
                  (D->flags & kConvOutBf16) != 0, reinterpret_cast<void*>(D->y));
  tc_fence_before();
  if (tm) {
    __syncthreads();
    if (tid == 0) tm[3] = gtimer();
  }
  G.kb_used = g0 + nk;
  G.accum_used += 1;
  cluster_sync_tile_end();  // both halves written, both TMEMs read; the next tile posted
}

// A pair run of conv tiles (see PairTiles, gemm_body.cuh).
template <class NextTile>
__device__ __forceinline__ void body_conv2(const BlockCmd& c, int tid, unsigned rank, GemmPipe& G,
                                           const unsigned* gate, const PairTiles& run,
                                           NextTile& next_tile) {
  const ConvDesc* D = reinterpret_cast<const ConvDesc*>(c.args[0]);
  long long blk = c.block;
  for (;;) {
    conv2_tile(D, static_cast<unsigned>(blk), tid, rank, G, gate, next_tile);
    blk = next_block(run);
    if (blk < 0) break;
    gate = nullptr;
  }
  cluster_sync_all();  // both CTAs' outputs released before the run is counted (body_gemm2)
}

}  // namespace gpuos_dev_impl
