// GEMM atom body on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// run by a TPC's worker pair (the 2-CTA cluster on SMs 2k, 2k+1).
//
// A tenant GEMM C[M,N] = A[M,K] . B[N,K]^T (bf16 in, fp32 accumulate, fp32
// or bf16 out; both operands K-major, i.e. a row-major activation times a
// row-major nn.Linear weight) is a grid of ceil(M/256) x ceil(N/256) blocks;
// block b computes one 256 x 256 output tile (grouped raster, body_gemm2).
// The reference models such a block only as a duration with sensitivity
// s ~ 1 (device.hpp:39-47); here the pair executes it:
//
//   thread 0 of each CTA   TMA producer: per 64-wide K slice, a 2-SM
//              tensor-map load of its 128 rows of A and its 128 rows of B
//              (128-byte swizzle) into its own stage, completing on the
//              LEADER's `full` mbarrier (the leader expects both halves).
//   thread 32 of the leader  MMA issuer: 4 x tcgen05.mma.cta_group::2
//              (M=256, N=256, K=16) per stage, reading A and B from both
//              CTAs' shared memory, accumulating into both CTAs' TMEM
//              (rows 0-127 in the leader, 128-255 in the peer);
//              tcgen05.commit multicasts `empty` (stage free) to both CTAs
//              and, after the last slice, `accum`.
//   all warps of both CTAs  epilogue: tcgen05.ld 32x32b.x32 (warp w reads
//              TMEM lanes 32(w%4).., column half w/4) -> registers -> global.
//
// Per SM and K step the pair moves 128 + 128 operand rows for 128 x 256
// MACs, two thirds of a 1-SM 128 x 256 tile's 128 + 256: the L2 -> SM
// traffic that bounds a 1-SM tile (profiles/ncu_gemm_1sm_r01.txt).
// Each worker CTA owns 512/W TMEM columns for its lifetime (allocated once
// at dispatcher start, W = workers per SM). Pipeline phases persist in
// GemmPipe across blocks, like the STREAM ring.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "bodies.cuh"
#include "ptx.cuh"

namespace gpuos_dev_impl {

constexpr unsigned kGemmTile = 256;   // pair tile: 256 x 256 (UMMA M = N = 256)
constexpr unsigned kGemmHalf = 128;   // rows of A and of B each CTA loads
constexpr unsigned kGemmBK = 64;      // K per stage: 64 bf16 = one 128-byte swizzle row
constexpr unsigned kGemmMaxStages = 4;
constexpr unsigned kGemmABytes = kGemmHalf * kGemmBK * 2;  // 16 KiB
constexpr unsigned kGemmStageBytes = 2 * kGemmABytes;      // A half + B half
constexpr unsigned kEpiRowBytes = 272;  // epilogue staging row: 256 B + 16 B pad (bank spread)

struct alignas(128) GemmDesc {
  CUtensorMap a;                 // A [M, K] bf16: box {64, 128}, SWIZZLE_128B
  CUtensorMap b;                 // B [N, K] bf16: box {64, 128}, SWIZZLE_128B
  unsigned long long c;          // C [M, N] row-major (ldc elements)
  unsigned m, n, k, ldc;
  unsigned m_tiles, n_tiles, n_tile, flags;  // n_tile: 64, 128 or 256 columns; flags bit 0: bf16 output
  unsigned long long* timing;    // optional: 4 globaltimer stamps per tile (profiling)
  // Split-K (splits > 1): block b = (tile b % tiles, K split b / tiles); a
  // split adds its fp32 tile into the tile's accumulator with vector float
  // reductions in L2 (red.global.add.v4.f32: every split's adds run in
  // parallel; the order of the fp32 sums is the arrival order), and the
  // tile's last split (self-resetting arrival counter) converts the
  // accumulator to C and zeroes it for the next run. (A first cut stored
  // per-split partials and let the last split sum them: that reduction
  // read splits x 64-256 KB in one CTA, 0.8 ms for 98 splits.)
  unsigned splits, k_slices_per_split, tiles, pad0;
  float* partial;                // [tiles][256][n_tile] fp32 accumulators (zero between runs)
  unsigned* arrivals;            // [tiles]
};
constexpr unsigned kGemmOutBf16 = 1u;

struct WaitGuard {
  unsigned* fault;              // DevCtl::fault (0: none)
  unsigned* quit;               // DevCtl::quit
  unsigned long long bound_ns;  // per wait
  unsigned long long* info;     // DevCtl::fault_info: where the first fault was raised
  const unsigned long long* ctx;  // the CTA's current block command (RoundCmd words)
};
constexpr unsigned kFaultPipeline = 1u;     // an mbarrier wait expired
constexpr unsigned kFaultAdoptedPair = 2u;  // a peer CTA claimed a 2-SM block (dispatcher.cu)
// The first fault also records where it was raised (host error text):
// SM, cluster rank, thread, the barrier's shared-memory offset and parity,
// and the block being run (descriptor args[0], block index, body | slice).
__device__ __noinline__ void raise_fault(const WaitGuard& g, unsigned code, unsigned bar = 0u,
                                            unsigned parity = 0u) {
  if (atomicCAS(g.fault, 0u, code) == 0u && g.info != nullptr) {
    unsigned sm, crank;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    g.info[0] = sm | (static_cast<unsigned long long>(crank) << 16) |
                (static_cast<unsigned long long>(threadIdx.x) << 32);
    g.info[1] = bar | (static_cast<unsigned long long>(parity) << 32);
    g.info[2] = g.ctx ? g.ctx[0] : 0ull;
    g.info[3] = g.ctx ? g.ctx[5] : 0ull;
    g.info[4] = g.ctx ? g.ctx[6] : 0ull;
    __threadfence();
  }
  atomicExch(g.quit, 1u);
}
struct GemmPipe {
  unsigned char* tiles;          // stages x 32 KiB (A half, B half), 1024-aligned
  unsigned long long* full;      // [kGemmMaxStages]
  unsigned long long* empty;     // [kGemmMaxStages]
  unsigned long long* accum;     // accumulator ready
  unsigned stages;
  unsigned n_tile;
  unsigned tmem;                 // TMEM base address of this worker's columns
  unsigned accum_used;           // tiles completed by this CTA (accum parity)
  unsigned long long kb_used;    // K slices streamed by this CTA so far
  const WaitGuard* guard;        // in shared memory (slow path only)
};

// Pipeline waits are bounded so a stuck tile cannot hang the persistent
// kernel. On expiry the wait raises the dispatcher's fault word (first
// fault wins) and its quit flag, then returns: the worker unwinds, the
// kernel drains out, and the host reports GPUOS_E_TIMEOUT with the fault
// code -- no `trap`, which would abort the CUDA context for every tenant.
// After a fault every bounded wait returns at once.
__device__ __forceinline__ void mbar_wait_bounded(unsigned long long* b, unsigned parity,
                                                  const WaitGuard& g) {
  const unsigned a = smem_u32(b);
  unsigned ok = 0;
  unsigned long long t0 = 0;
  for (unsigned spins = 0;; ++spins) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if ((spins & 1023u) == 0) {
      if (ld_relaxed_gpu(g.fault) != 0u) return;
      const unsigned long long t = gtimer();
      if (t0 == 0) {
        t0 = t;
      } else if (t - t0 > g.bound_ns) {
        raise_fault(g, kFaultPipeline, a, parity);
        return;
      }
    }
  }
}

// One thread: spin until the gate opens (the TMA producer before its
// activation loads, the MMA issuer before its first wait).
__device__ __forceinline__ void gate_spin(const unsigned* gate, const WaitGuard& g) {
  for (unsigned spins = 0; ld_acquire_gpu(gate) & 2u; ++spins) {
    if ((spins & 63u) == 63u && ld_relaxed_gpu(g.quit) != 0u) break;
    __nanosleep(64);
  }
}

// An early-started tile's gate (DevAtom::paused bit 1): every thread that
// is about to enter a bounded pipeline wait first waits here, unbounded
// (the predecessor may legitimately run for a long time), so the bound
// only ever measures the pipeline itself. Lane 0 of each warp polls; a
// quit (hang guard, fault) releases the wait.
__device__ __forceinline__ void gate_wait(const unsigned* gate, const WaitGuard& g) {
  if (gate == nullptr) return;
  if ((threadIdx.x & 31u) == 0u) {
    for (unsigned spins = 0; ld_acquire_gpu(gate) & 2u; ++spins) {
      if ((spins & 63u) == 63u && ld_relaxed_gpu(g.quit) != 0u) break;
      __nanosleep(128);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// K-major operand tile with 128-byte swizzle: rows of 128 B, 8-row core
// groups 1024 B apart (SBO), version 1 (sm_100), layout type 2.
__device__ __forceinline__ unsigned long long umma_desc_sw128(unsigned saddr) {
  return static_cast<unsigned long long>((saddr >> 4) & 0x3FFFu) |
         (1ull << 16) |                 // LBO (unused for swizzled K-major)
         (64ull << 32) |                // SBO = 1024 B >> 4
         (1ull << 46) |                 // descriptor version (Blackwell)
         (2ull << 61);                  // SWIZZLE_128B
}

// kind::f16 instruction descriptor: bf16 A/B, f32 D, both K-major.
__device__ __forceinline__ unsigned umma_idesc_bf16(unsigned m, unsigned n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

// 32 lanes x 32 columns of fp32 from TMEM into 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(unsigned taddr, unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// The pair's variants: cta_group::2 allocation (same columns in both CTAs,
// issued by the same warp of each), MMA, multicast commit, 2-SM TMA load.
__device__ __forceinline__ void tmem_alloc2(unsigned* holder, unsigned cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(holder))),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free2(unsigned base, unsigned cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols)
               : "memory");
}
__device__ __forceinline__ void umma2_bf16(unsigned tmem_d, unsigned long long a,
                                           unsigned long long b, unsigned idesc,
                                           unsigned accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on the mbarrier at the same offset in both CTAs of the pair once
// every prior tcgen05 operation of this thread has completed.
__device__ __forceinline__ void umma2_commit_both(unsigned long long* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
      "h"(static_cast<unsigned short>(3))
      : "memory");
}
// 2-SM tensor-map load into this CTA's shared memory, completing on the
// leader's mbarrier (the peer bit of the shared::cluster address cleared).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
      "l"(map), "r"(c0), "r"(c1),
      "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// End of a pair tile inside a run. A relaxed arrive (GPUOS_RELAXED_TILE_END)
// measured ~3 % faster on GEMM / conv -- the epilogue's global stores are not
// drained before the next tile -- but model-config runs then faulted about
// once per few hundred live runs (a pair desynchronised: an "unspecified
// launch failure" or an expired pipeline wait; 0 in 8 x ~60 runs with the
// release barrier), so tiles end with the release barrier; the next tile
// still reaches both CTAs through the posted count (next_block).
__device__ __forceinline__ void cluster_sync_tile_end() {
#ifdef GPUOS_RELAXED_TILE_END
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
#else
  cluster_sync_all();
#endif
}

// Called once per CTA by all threads (barrier memory at smem + 128 .. 256;
// the STREAM ring's barriers occupy smem + 0 .. 128, tiles start at 1024).
__device__ __forceinline__ void gemm_pipe_init(GemmPipe& G, unsigned char* smem,
                                               unsigned smem_bytes, unsigned tmem_cols, int tid) {
  G.full = reinterpret_cast<unsigned long long*>(smem + 128);
  G.empty = G.full + kGemmMaxStages;
  G.accum = G.empty + kGemmMaxStages;
  G.tiles = smem + 1024;
  G.n_tile = kGemmTile;
  G.stages = tmem_cols >= kGemmTile && smem_bytes > 1024 ? (smem_bytes - 1024) / kGemmStageBytes : 0;
  if (G.stages > kGemmMaxStages) G.stages = kGemmMaxStages;
  G.accum_used = 0;
  G.kb_used = 0;
  if (tid == 0) {
    for (unsigned s = 0; s < kGemmMaxStages; ++s) {
      mbar_init(G.full + s, 1);
      mbar_init(G.empty + s, 1);
    }
    mbar_init(G.accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// Accumulator -> global for one CTA's 128 rows of a pair tile (all 8
// warps; the operand stages must be free). Warp w reads TMEM lanes
// 32(w%4)..+31 and column half w/4. Rows cta_row0.. of a row-major [M, N]
// matrix (ldc elements), columns col_base..col_base+255, ragged edges
// masked.
__device__ __forceinline__ void epilogue_staged(const GemmPipe& G, int tid, unsigned cta_row0,
                                                unsigned col_base, unsigned M, unsigned N,
                                                unsigned ldc, bool bf16_out, void* C) {
  // (N here is the tile's column limit: min(matrix N, col_base + tile width).)
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned q = static_cast<unsigned>(warp & 3), h = static_cast<unsigned>(warp >> 2);
  constexpr unsigned half = kGemmTile / 2;
  const unsigned row0 = cta_row0 + q * 32;  // warp's first row
  // Staged through shared memory (the operand stages are free now): each
  // thread writes its row's values, then the warp stores two 256-byte rows
  // per instruction -- coalesced, where storing straight from the TMEM
  // registers wrote 32 scattered 16-byte pieces per instruction (9 us per
  // tile, tools/gemm_batch.py timing hook).
  const unsigned esz = bf16_out ? 2u : 4u;
  const unsigned pass_cols = 256u / esz;                 // 256 bytes of a row per pass
  unsigned char* stg = G.tiles + static_cast<unsigned>(warp) * (32u * kEpiRowBytes);
  const bool vec_ok = (static_cast<size_t>(ldc) * esz) % 16 == 0;
#pragma unroll 1
  for (unsigned pc = 0; pc < half; pc += pass_cols) {
    if (col_base + h * half + pc >= N) break;  // warp-uniform: ragged last tile
#pragma unroll 1
    for (unsigned ch = 0; ch < pass_cols / 32; ++ch) {
      unsigned v[32];
      tmem_ld32(G.tmem + ((q * 32u) << 16) + h * half + pc + ch * 32u, v);
      uint4* dst = reinterpret_cast<uint4*>(stg + static_cast<unsigned>(lane) * kEpiRowBytes + ch * 32u * esz);
      if (bf16_out) {
        unsigned pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const __nv_bfloat162 t = __floats2bfloat162_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
          pk[i] = *reinterpret_cast<const unsigned*>(&t);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) dst[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
    }
    __syncwarp();
    // 16 lanes per row, 16 bytes each: rows 2i and 2i + 1 per instruction.
    const unsigned seg = static_cast<unsigned>(lane) & 15u;
    const unsigned col = col_base + h * half + pc + seg * (16u / esz);
#pragma unroll 4
    for (unsigned i = 0; i < 16; ++i) {
      const unsigned r = 2 * i + (static_cast<unsigned>(lane) >> 4);
      const unsigned grow = row0 + r;
      if (grow >= M || col >= N) continue;
      const uint4 val = *reinterpret_cast<const uint4*>(stg + r * kEpiRowBytes + seg * 16u);
      unsigned char* out = reinterpret_cast<unsigned char*>(C) + (static_cast<size_t>(grow) * ldc + col) * esz;
      if (vec_ok && col + 16u / esz <= N) {
        st_stream(reinterpret_cast<uint4*>(out), val);
      } else {
        const unsigned char* src = reinterpret_cast<const unsigned char*>(&val);
        for (unsigned e = 0; e < 16u / esz && col + e < N; ++e)
          for (unsigned byte = 0; byte < esz; ++byte) out[e * esz + byte] = src[e * esz + byte];
      }
    }
    __syncwarp();  // staging reused by the next pass
  }
}

// A pair run: after the first tile (claimed by the dispatcher's arbitration)
// the pair keeps claiming tiles of the same atom inside the body. The
// leader's producer thread claims the next tile right after issuing the
// current tile's last load (the claim's L2 round trip overlaps the last
// stages and the epilogue) and posts it to both CTAs' `next` word; the
// tile's closing cluster barrier publishes it (barrier.cluster arrive.release
// / wait.acquire), so no extra handshake, arbitration, peer join or per-tile
// accounting sits between two tiles of a run. `next_tile` (dispatcher.cu,
// PairRun) returns the next absolute block or -1 (atom drained, or the TPC's
// candidate set changed: the pair goes back to full arbitration).
// `run_next`: this CTA's copy of the posted block.
struct PairTiles {
  volatile long long* run_next;
  const unsigned* run_posts;  // posts received (NextTile writes it with release)
  unsigned* seen;             // this thread's count of posts consumed (per worker)
};

// Every thread of both CTAs, after a pair tile: the run's next block as the
// leader posted it for this tile. The post (run.next, then the count with a
// release store, NextTile) is awaited with an acquire load of the count, so
// the value read is this tile's whatever barrier ends the tile (a relaxed
// arrive orders nothing); it was posted before the epilogue, so the wait is
// normally free.
__device__ __forceinline__ long long next_block(const PairTiles& run) {
  const unsigned want = ++*run.seen;
  unsigned v;
  for (;;) {
    asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v)
                 : "r"(static_cast<unsigned>(__cvta_generic_to_shared(run.run_posts))) : "memory");
    if (static_cast<int>(v - want) >= 0) break;
  }
  return *run.run_next;
}

// Both CTAs of the pair, all threads; rank 0 is the leader.
// `gate`: the atom's early-start gate (dispatcher.cu): while it is 1 the
// tile loads its first stages of B (weights) but no A (the predecessor is
// still producing the activations).
// Split-K: this CTA's 128 accumulator rows added into the tile's fp32
// accumulator in L2 (all 8 warps; warp w: TMEM lanes 32 (w % 4).., column
// half w / 4), 16 bytes per reduction.
__device__ __forceinline__ void epilogue_red_f32(const GemmPipe& G, int tid, float* acc, unsigned cta_row0,
                                                 unsigned n_tile) {
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned q = static_cast<unsigned>(warp & 3), h = static_cast<unsigned>(warp >> 2);
  constexpr unsigned half = kGemmTile / 2;
  float* row = acc + static_cast<size_t>(cta_row0 + q * 32u + static_cast<unsigned>(lane)) * n_tile;
#pragma unroll 1
  for (unsigned pc = 0; pc < half; pc += 32) {
    const unsigned col0 = h * half + pc;
    if (col0 >= n_tile) break;  // warp-uniform: narrow tiles
    unsigned v[32];
    tmem_ld32(G.tmem + ((q * 32u) << 16) + col0, v);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + col0 + 4 * i),
                   "f"(__uint_as_float(v[4 * i])), "f"(__uint_as_float(v[4 * i + 1])),
                   "f"(__uint_as_float(v[4 * i + 2])), "f"(__uint_as_float(v[4 * i + 3]))
                   : "memory");
  }
}

// Split-K, the tile's last split (leader CTA, 256 threads): the fp32
// accumulator -> C (ragged edges masked), and back to zero for the next run.
// 16 threads per row of 64 columns, 16 bytes each.
__device__ __forceinline__ void gemm_reduce_tile(const GemmDesc* D, unsigned tile, unsigned mt, unsigned nt,
                                                 int tid) {
  const unsigned n_tile = D->n_tile;
  float* base = D->partial + static_cast<size_t>(tile) * kGemmTile * n_tile;
  const bool bf16_out = (D->flags & kGemmOutBf16) != 0;
  const unsigned vecs = n_tile / 4;               // float4 per row
  const unsigned per_pass = 256u / vecs;          // rows per pass
#pragma unroll 4
  for (unsigned r0 = 0; r0 < kGemmTile; r0 += per_pass) {
    const unsigned r = r0 + static_cast<unsigned>(tid) / vecs;
    const unsigned c4 = static_cast<unsigned>(tid) % vecs;
    float4* src = reinterpret_cast<float4*>(base + static_cast<size_t>(r) * n_tile + 4 * c4);
    const float4 v = __ldcg(src);
    __stcg(src, make_float4(0.f, 0.f, 0.f, 0.f));
    const unsigned grow = mt * kGemmTile + r, gcol = nt * n_tile + 4 * c4;
    if (grow >= D->m || gcol >= D->n) continue;
    const float a4[4] = {v.x, v.y, v.z, v.w};
    const size_t o = static_cast<size_t>(grow) * D->ldc + gcol;
    for (unsigned e = 0; e < 4 && gcol + e < D->n; ++e) {
      if (bf16_out) reinterpret_cast<__nv_bfloat16*>(D->c)[o + e] = __float2bfloat16_rn(a4[e]);
      else reinterpret_cast<float*>(D->c)[o + e] = a4[e];
    }
  }
}

template <class NextTile>
__device__ __forceinline__ void gemm2_tile(const GemmDesc* D, unsigned blk_in, int tid, unsigned rank,
                                           GemmPipe& G, const unsigned* gate, NextTile& next_tile) {
  const unsigned m_tiles = D->m_tiles, n_tiles = D->n_tiles, n_tile = D->n_tile;
  // Split-K: this block's output tile and K range.
  const unsigned blk = D->splits > 1 ? blk_in % D->tiles : blk_in;
  const unsigned split = D->splits > 1 ? blk_in / D->tiles : 0u;
  // Grouped raster: blocks walk 8 M-tiles down an N column before moving
  // right, so ~150 concurrent tiles touch 8 A panels and ~18 B panels (fits
  // L2) instead of every A panel (8192^3: DRAM reads 3x the operands).
  constexpr unsigned kGroup = 8;
  const unsigned group = blk / (kGroup * n_tiles);
  const unsigned first_m = group * kGroup;
  const unsigned gm = m_tiles - first_m < kGroup ? m_tiles - first_m : kGroup;
  const unsigned in_group = blk - group * kGroup * n_tiles;
  const unsigned mt = first_m + in_group % gm, nt = in_group / gm;
  const unsigned nk_all = (D->k + kGemmBK - 1) / kGemmBK;
  const unsigned kb0 = split * D->k_slices_per_split;
  const unsigned nk = D->splits > 1 ? (kb0 + D->k_slices_per_split < nk_all ? D->k_slices_per_split : nk_all - kb0)
                                    : nk_all;
  const unsigned S = G.stages;
  const unsigned long long g0 = G.kb_used;
  if (S == 0) {  // host validated; never on the path
    if (tid == 0 && rank == 0) next_tile(true);  // (ends the run)
    cluster_sync_all();
    return;
  }

  unsigned long long* tm = D->timing != nullptr && rank == 0 ? D->timing + 4ull * blk_in : nullptr;
  if (tm && tid == 0) tm[0] = gtimer();
  if (tid == 0) {
    // TMA producer (both CTAs). The descriptor was written by a host copy
    // while this persistent kernel runs: acquire it into the tensor-map proxy.
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&D->a) : "memory");
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(&D->b) : "memory");
    const int a_row = static_cast<int>(mt * kGemmTile + rank * kGemmHalf);
    const int b_row = static_cast<int>(nt * n_tile + rank * (n_tile / 2));
    const unsigned tx = 2 * (kGemmABytes + n_tile / 2 * kGemmBK * 2);  // both CTAs' A and B halves
    // B (weights) for the first stages first, then A once the atom's gate
    // is open (early start; otherwise the gate read overlaps the B loads).
    const unsigned pre = gate ? (nk < S ? nk : S) : 0u;  // (no gate: loads in stage order)
    for (unsigned j = 0; j < pre; ++j) {
      const unsigned s = static_cast<unsigned>((g0 + j) % S);
      if ((g0 + j) / S >= 1) mbar_wait_bounded(G.empty + s, static_cast<unsigned>(((g0 + j) / S - 1) & 1), *G.guard);
      if (rank == 0) mbar_expect_tx(G.full + s, tx);
      tma_load_2d_pair(G.tiles + s * kGemmStageBytes + kGemmABytes, &D->b, static_cast<int>((kb0 + j) * kGemmBK),
                       b_row, G.full + s);
    }
    if (gate) {
      gate_spin(gate, *G.guard);  // DevAtom::paused, kGatedBit
      asm volatile("fence.proxy.async.global;" ::: "memory");  // A: generic-proxy writes, TMA reads
    }
    for (unsigned j = 0; j < pre; ++j)
      tma_load_2d_pair(G.tiles + static_cast<unsigned>((g0 + j) % S) * kGemmStageBytes, &D->a,
                       static_cast<int>((kb0 + j) * kGemmBK), a_row, G.full + static_cast<unsigned>((g0 + j) % S));
    for (unsigned j = pre; j < nk; ++j) {
      const unsigned long long k = g0 + j;
      const unsigned s = static_cast<unsigned>(k % S);
      const unsigned long long r = k / S;
      if (r >= 1) mbar_wait_bounded(G.empty + s, static_cast<unsigned>((r - 1) & 1), *G.guard);
      unsigned char* st = G.tiles + s * kGemmStageBytes;
      if (rank == 0) mbar_expect_tx(G.full + s, tx);
      const int kc = static_cast<int>((kb0 + j) * kGemmBK);
      tma_load_2d_pair(st, &D->a, kc, a_row, G.full + s);
      tma_load_2d_pair(st + kGemmABytes, &D->b, kc, b_row, G.full + s);
    }
    if (rank == 0) next_tile();  // claim + post the run's next tile (both CTAs)
  } else if (tid == 32 && rank == 0) {
    if (gate) gate_spin(gate, *G.guard);  // the bounded waits measure the pipeline only
    // MMA issuer: one thread of the leader drives both SMs' tensor cores.
    tc_fence_after();
    const unsigned idesc = umma_idesc_bf16(kGemmTile, n_tile);
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
      umma2_commit_both(G.empty + s);  // stage free in both CTAs once read
    }
    umma2_commit_both(G.accum);        // every MMA of the tile has completed
  }

  // Epilogue: all 8 warps of both CTAs. Warp w reads TMEM lanes 32(w%4)..+31
  // (this CTA's 128 tile rows) and column half w/4.
  gate_wait(gate, *G.guard);  // (unbounded: the predecessor may run long)
  mbar_wait_bounded(G.accum, G.accum_used & 1u, *G.guard);
  tc_fence_after();
  if (tm && tid == 0) tm[2] = gtimer();
  const unsigned col0 = nt * n_tile;
  if (D->splits > 1) {
    // This split's contribution, added into the tile's fp32 accumulator.
    epilogue_red_f32(G, tid, D->partial + static_cast<size_t>(blk) * kGemmTile * n_tile, rank * kGemmHalf,
                     n_tile);
  } else {
    epilogue_staged(G, tid, mt * kGemmTile + rank * kGemmHalf, col0, D->m,
                    D->n - col0 < n_tile ? D->n : col0 + n_tile, D->ldc,
                    (D->flags & kGemmOutBf16) != 0, reinterpret_cast<void*>(D->c));
  }
  tc_fence_before();  // the next tile's MMAs overwrite this accumulator
  if (tm) {
    __syncthreads();
    if (tid == 0) tm[3] = gtimer();
  }
  G.kb_used = g0 + nk;
  G.accum_used += 1;
  // Both halves of the tile are written (and both TMEMs read) before the
  // leader records the tile or issues the next tile's MMAs; the posted next
  // tile is visible in both CTAs after it. Split-K keeps the release: the
  // peer's reductions into the fp32 accumulator must precede the leader's
  // count below.
  if (D->splits > 1) cluster_sync_all();
  else cluster_sync_tile_end();
  if (D->splits > 1 && rank == 0) {
    // Split-K: the tile's last split converts the accumulator.
    __shared__ int last_split;
    if (tid == 0) {
      // acq_rel: this split's reductions (both CTAs, observed through the
      // cluster barrier: the release is cumulative) precede the count, and
      // the last split acquires every other split's.
      unsigned before;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(before) : "l"(D->arrivals + blk) : "memory");
      last_split = before == D->splits - 1;
      if (last_split) D->arrivals[blk] = 0u;  // ready for the kernel's next run
    }
    __syncthreads();
    if (last_split) gemm_reduce_tile(D, blk, mt, nt, tid);
    __syncthreads();  // (last_split is read before thread 0 rewrites it)
  }
}

template <class NextTile>
__device__ __forceinline__ void body_gemm2(const BlockCmd& c, int tid, unsigned rank, GemmPipe& G,
                                           const unsigned* gate, const PairTiles& run,
                                           NextTile& next_tile) {
  const GemmDesc* D = reinterpret_cast<const GemmDesc*>(c.args[0]);
  long long blk = c.block;
  for (;;) {
    gemm2_tile(D, static_cast<unsigned>(blk), tid, rank, G, gate, next_tile);
    blk = next_block(run);
    if (blk < 0) break;
    gate = nullptr;  // (open: the run's first tile waited for it)
  }
  // Tiles end with a relaxed arrive; before the leader counts the run done
  // (which releases C to a chained successor) both CTAs' C stores must be
  // released: one release barrier per run.
  cluster_sync_all();
}

}  // namespace gpuos_dev_impl
