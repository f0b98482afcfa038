// GEMV atom body: the HBM-bound matrix-vector product of batch-1 decode
// (y = W . x, W bf16 [N, K] row-major, x bf16 [K], fp32 accumulation, fp32
// or bf16 y), run by a TPC's worker pair. Block b owns rows [256 b, 256 b +
// 256) of W; the reference models such a block only as a duration with
// sensitivity s ~ 0 (device.hpp:39-47).
//
// The multiply-adds go to the tensor cores so the CUDA cores only issue
// copies: per 64-wide K slice each CTA TMA-loads its 128 rows of W (16 KiB,
// 128-byte swizzle) and a 16-row x tile whose first row is x and whose other
// rows are the tensor map's zero fill (x is a [1, K] tensor read with a
// 16-row box), and the leader issues tcgen05.mma.cta_group::2 with M = 256,
// N = 32: column 0 of the TMEM accumulator is y. A CUDA-core version of
// this body (fp32 FMAs on bf16 pairs unpacked from shared memory) issued
// ~50 instructions per 512 bytes of W and stopped at 3.5 TB/s, 53 % of HBM
// (tools/gemv_batch.py, round 1); here the math costs the SMs nothing.
// Algorithmic bytes per block: 256 K 2 (W) + K 2 (x) + 256 x 4 or 2 (y).
//
// Decode shapes have few 256-row tiles (N = 4096: 16), so the descriptor may
// split K: block b = (row tile b % row_tiles, K split b / row_tiles); each
// block stores its partial sums, and the row tile's last block (a counter
// that resets itself) adds them in split order and writes y.
//
// args: [0] descriptor from gpuos_dev_gemv_desc().
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "bodies.cuh"
#include "gemm_body.cuh"

namespace gpuos_dev_impl {

constexpr unsigned kGemvTile = 256;       // rows of W per block (pair tile M)
constexpr unsigned kGemvN = 32;           // UMMA N (x plus zero rows)
constexpr unsigned kGemvXRows = kGemvN / 2;  // x-tile rows each CTA loads
constexpr unsigned kGemvWBytes = kGemmHalf * kGemmBK * 2;    // 16 KiB
constexpr unsigned kGemvXBytes = kGemvXRows * kGemmBK * 2;   // 2 KiB
constexpr unsigned kGemvStageBytes = kGemvWBytes + kGemvXBytes;
constexpr unsigned kGemvMaxStages = 8;
constexpr unsigned kGemvOutBf16 = 1u;
// W pre-packed (gpuos_dev_gemv_pack): [ceil(N/128)][ceil(K/64)][128][64],
// every ring stage's 16 KiB one contiguous HBM range.
constexpr unsigned kGemvPacked = 2u;

struct alignas(128) GemvDesc {
  CUtensorMap w;                 // W [N, K] bf16: box {64, 128}, SWIZZLE_128B (packed: [rows, 64])
  CUtensorMap x;                 // x [1, K] bf16: box {64, 16}, SWIZZLE_128B (rows >= 1 zero)
  unsigned long long y;
  unsigned n, k, blocks, flags;  // flags: kGemvOutBf16
  unsigned row_tiles;            // ceil(N / 256)
  unsigned k_slices_per_block;   // 64-wide K slices per block (split-K)
  unsigned splits;               // K splits (1: no split)
  unsigned pad0;
  float* partial;                // [splits][N] fp32 partial sums (split-K)
  unsigned* arrivals;            // [row_tiles] self-resetting split counters
  unsigned long long* timing;    // optional: 4 globaltimer stamps per block (profiling)
};

// (tools/corun_probe.py writes `timing` at this offset for profiling)
static_assert(offsetof(GemvDesc, timing) == 312, "GemvDesc layout");

struct GemvPipe {
  unsigned char* tiles;          // stages x 18 KiB, 1024-aligned
  unsigned long long* full;      // [kGemvMaxStages]
  unsigned long long* empty;     // [kGemvMaxStages]
  unsigned long long* accum;
  unsigned stages;
  unsigned accum_used;
  unsigned long long kb_used;
  unsigned tmem;
  const WaitGuard* guard;        // in shared memory (slow path only)
};

// Once per CTA, all threads (barriers at smem + 256 .. 392; tiles share the
// region from smem + 1024 with the other bodies).
__device__ __forceinline__ void gemv_pipe_init(GemvPipe& G, unsigned char* smem,
                                               unsigned smem_bytes, unsigned tmem_cols, int tid) {
  G.full = reinterpret_cast<unsigned long long*>(smem + 256);
  G.empty = G.full + kGemvMaxStages;
  G.accum = G.empty + kGemvMaxStages;
  G.tiles = smem + 1024;
  G.stages = tmem_cols >= kGemvN && smem_bytes > 1024 ? (smem_bytes - 1024) / kGemvStageBytes : 0;
  if (G.stages > kGemvMaxStages) G.stages = kGemvMaxStages;
  G.accum_used = 0;
  G.kb_used = 0;
  if (tid == 0) {
    for (unsigned s = 0; s < kGemvMaxStages; ++s) {
      mbar_init(G.full + s, 1);
      mbar_init(G.empty + s, 1);
    }
    mbar_init(G.accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// One TMEM column (fp32) of 32 lanes into one register per thread.
__device__ __forceinline__ unsigned tmem_ld1(unsigned taddr) {
  unsigned v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return v;
}

// Both CTAs of the pair, all threads; rank 0 is the leader.
// `gate`: the atom's early-start gate (dispatcher.cu): while it is 1 the
// block streams its first stages of W but loads no x (the predecessor is
// still producing it).
template <class NextTile>
__device__ __forceinline__ void gemv2_tile(const GemvDesc* D, unsigned block, int tid, unsigned rank, GemvPipe& G,
                                           const unsigned* gate, NextTile& next_tile) {
  // Block b: row tile b % row_tiles, K split b / row_tiles (decode shapes
  // have few row tiles; splitting K keeps every TPC streaming W).
  const unsigned blk = block % D->row_tiles;
  const unsigned split = block / D->row_tiles;
  const unsigned nk_all = (D->k + kGemmBK - 1) / kGemmBK;
  const unsigned kb0 = split * D->k_slices_per_block;
  const unsigned kb1 = kb0 + D->k_slices_per_block < nk_all ? kb0 + D->k_slices_per_block : nk_all;
  const unsigned nk = kb1 > kb0 ? kb1 - kb0 : 0u;
  const unsigned S = G.stages;
  const unsigned long long g0 = G.kb_used;
  if (S == 0 || nk == 0) {  // host validated; never on the path
    if (tid == 0 && rank == 0) next_tile(true);  // (ends the run)
    cluster_sync_all();
    return;
  }
  unsigned long long* tm = D->timing != nullptr && rank == 0 ? D->timing + 4ull * block : nullptr;
  if (tm && tid == 0) tm[0] = gtimer();
  if (tid == 0) {
    // TMA producer (both CTAs); descriptor written by a host copy while
    // this persistent kernel runs: acquire it into the tensor-map proxy.
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&D->w) : "memory");
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&D->x) : "memory");
    // Packed W: the 128-row half-tile's K slice j starts at packed row
    // ((2 blk + rank) nk_all + j) 128, column 0.
    const bool packed = (D->flags & kGemvPacked) != 0;
    const int w_row = static_cast<int>(blk * kGemvTile + rank * kGemmHalf);
    const int p_row = static_cast<int>(((2u * blk + rank) * nk_all + kb0) * kGemmHalf);
    auto w_c0 = [&](unsigned j) { return packed ? 0 : static_cast<int>((kb0 + j) * kGemmBK); };
    auto w_c1 = [&](unsigned j) { return packed ? p_row + static_cast<int>(j * kGemmHalf) : w_row; };
    const int x_row = static_cast<int>(rank * kGemvXRows);  // rank 1: all zero fill
    // W for the first stages first, then x once the atom's gate is open:
    // an early-started block streams W while its predecessor still writes
    // x; for any other block the gate read overlaps the W loads.
    const unsigned pre = gate ? (nk < S ? nk : S) : 0u;  // (no gate: loads in stage order)
    for (unsigned j = 0; j < pre; ++j) {
      const unsigned long long k = g0 + j;
      const unsigned s = static_cast<unsigned>(k % S);
      const unsigned long long r = k / S;
      if (r >= 1) mbar_wait_bounded(G.empty + s, static_cast<unsigned>((r - 1) & 1), *G.guard);
      if (rank == 0) mbar_expect_tx(G.full + s, 2 * kGemvStageBytes);
      tma_load_2d_pair(G.tiles + s * kGemvStageBytes, &D->w, w_c0(j), w_c1(j), G.full + s);
    }
    if (gate) {
      gate_spin(gate, *G.guard);  // DevAtom::paused, kGatedBit
      asm volatile("fence.proxy.async.global;" ::: "memory");  // x: generic-proxy writes, TMA reads
    }
    for (unsigned j = 0; j < pre; ++j) {
      const unsigned s = static_cast<unsigned>((g0 + j) % S);
      tma_load_2d_pair(G.tiles + s * kGemvStageBytes + kGemvWBytes, &D->x,
                       static_cast<int>((kb0 + j) * kGemmBK), x_row, G.full + s);
    }
    for (unsigned j = pre; j < nk; ++j) {
      const unsigned long long k = g0 + j;
      const unsigned s = static_cast<unsigned>(k % S);
      const unsigned long long r = k / S;
      if (r >= 1) mbar_wait_bounded(G.empty + s, static_cast<unsigned>((r - 1) & 1), *G.guard);
      unsigned char* st = G.tiles + s * kGemvStageBytes;
      if (rank == 0) mbar_expect_tx(G.full + s, 2 * kGemvStageBytes);
      const int kc = static_cast<int>((kb0 + j) * kGemmBK);
      tma_load_2d_pair(st, &D->w, w_c0(j), w_c1(j), G.full + s);
      tma_load_2d_pair(st + kGemvWBytes, &D->x, kc, x_row, G.full + s);
    }
    if (rank == 0) next_tile();  // claim + post the run's next block (both CTAs)
  } else if (tid == 32 && rank == 0) {
    if (gate) gate_spin(gate, *G.guard);  // the bounded waits measure the pipeline only
    tc_fence_after();
    const unsigned idesc = umma_idesc_bf16(kGemvTile, kGemvN);
    for (unsigned j = 0; j < nk; ++j) {
      const unsigned long long k = g0 + j;
      const unsigned s = static_cast<unsigned>(k % S);
      mbar_wait_bounded(G.full + s, static_cast<unsigned>((k / S) & 1), *G.guard);
      tc_fence_after();
      if (tm && j == 0) tm[1] = gtimer();
      const unsigned a0 = smem_u32(G.tiles + s * kGemvStageBytes);
      const unsigned b0 = a0 + kGemvWBytes;
#pragma unroll
      for (unsigned kk = 0; kk < kGemmBK / 16; ++kk)
        umma2_bf16(G.tmem, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                   (j | kk) != 0u);
      umma2_commit_both(G.empty + s);
    }
    umma2_commit_both(G.accum);
  }
  // Epilogue: warps 0-3 of both CTAs read TMEM column 0 (y) of their lanes.
  gate_wait(gate, *G.guard);  // (unbounded: the predecessor may run long)
  mbar_wait_bounded(G.accum, G.accum_used & 1u, *G.guard);
  tc_fence_after();
  if (tm && tid == 0) tm[2] = gtimer();
  const int warp = tid >> 5, lane = tid & 31;
  const bool bf16_y = (D->flags & kGemvOutBf16) != 0;
  if (warp < 4) {
    const float v = __uint_as_float(tmem_ld1(G.tmem + ((static_cast<unsigned>(warp) * 32u) << 16)));
    const unsigned row = blk * kGemvTile + rank * kGemmHalf + static_cast<unsigned>(warp) * 32u +
                         static_cast<unsigned>(lane);
    if (row < D->n) {
      if (D->splits > 1)
        D->partial[static_cast<size_t>(split) * D->n + row] = v;
      else if (bf16_y)
        reinterpret_cast<__nv_bfloat16*>(D->y)[row] = __float2bfloat16_rn(v);
      else
        reinterpret_cast<float*>(D->y)[row] = v;
    }
  }
  tc_fence_before();
  G.kb_used = g0 + nk;
  G.accum_used += 1;
  cluster_sync_all();  // both halves written, both TMEMs read
  if (D->splits > 1) {
    // Split-K: the last block of the row tile (self-resetting arrival
    // counter) sums the partials in split order -- deterministic, no
    // zeroed output or float atomics -- and writes y.
    __shared__ int last_split;
    if (rank == 0) {
      if (tid == 0) {
        // acq_rel: this tile's partials (both CTAs, observed through the
        // cluster barrier: the release is cumulative) precede the count, and
        // the last split acquires every other split's.
        unsigned before;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(before) : "l"(D->arrivals + blk) : "memory");
        last_split = before == D->splits - 1;
        if (last_split) D->arrivals[blk] = 0u;  // ready for the kernel's next run
      }
      __syncthreads();
      if (last_split) {
        const unsigned row = blk * kGemvTile + static_cast<unsigned>(tid);
        if (row < D->n) {
          // Up to 16 splits: every partial load in flight at once (one L2
          // round trip, not one per split), summed in split order.
          float acc = 0.f;
          const unsigned splits = D->splits;
          if (splits <= 16) {
            float v[16];
#pragma unroll
            for (unsigned sp = 0; sp < 16; ++sp)
              v[sp] = sp < splits ? __ldcg(D->partial + static_cast<size_t>(sp) * D->n + row) : 0.f;
#pragma unroll
            for (unsigned sp = 0; sp < 16; ++sp)
              if (sp < splits) acc += v[sp];
          } else {
            for (unsigned sp = 0; sp < splits; ++sp)
              acc += __ldcg(D->partial + static_cast<size_t>(sp) * D->n + row);
          }
          if (bf16_y)
            reinterpret_cast<__nv_bfloat16*>(D->y)[row] = __float2bfloat16_rn(acc);
          else
            reinterpret_cast<float*>(D->y)[row] = acc;
        }
      }
    }
  }
  if (tm && tid == 0) tm[3] = gtimer();
}

// A pair run of GEMV blocks (PairTiles, gemm_body.cuh): the leader claims
// the next block after the current one's last load; no arbitration, peer
// join or per-block accounting between two blocks of a run.
template <class NextTile>
__device__ __forceinline__ void body_gemv2(const BlockCmd& c, int tid, unsigned rank, GemvPipe& G,
                                           const unsigned* gate, const PairTiles& run, NextTile& next_tile) {
  const GemvDesc* D = reinterpret_cast<const GemvDesc*>(c.args[0]);
  long long blk = c.block;
  for (;;) {
    gemv2_tile(D, static_cast<unsigned>(blk), tid, rank, G, gate, next_tile);
    blk = next_block(run);
    if (blk < 0) break;
    gate = nullptr;  // (open: the run's first block waited for it)
  }
}

}  // namespace gpuos_dev_impl
