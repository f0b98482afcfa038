// Atom bodies: what one block of a tenant kernel executes inside a resident
// dispatcher worker CTA (256 threads). The reference models a block only
// as a duration (device.hpp:39-47); on the B200 each block does real work.
//
//   STREAM  HBM-bound transform, dst[i] = (src[i] ^ salt) * 0x9E3779B1 + i
//           over a contiguous chunk of `words` u32 per block (block b works
//           on chunk b % chunks when args[4] = chunks > 0, so a large grid
//           can stream through a bounded workspace); TMA bulk loads into a
//           shared-memory ring, 128-bit coalesced non-allocating stores.
//           Algorithmic bytes: 8 per word.
//   SPIN    holds the worker for a fixed time (dispatcher-overhead probes).
#pragma once

#include "ptx.cuh"

namespace gpuos_dev_impl {

constexpr int kWorkerThreads = 256;
constexpr unsigned kStreamMul = 0x9E3779B1u;

struct BlockCmd {
  unsigned long long args[5];
  long long block;  // absolute block index within the tenant kernel
  unsigned body;
  unsigned part;    // preemption slice of the block, 0 .. parts-1
  unsigned parts;
};

__device__ __forceinline__ unsigned stream_word(unsigned x, unsigned salt,
                                                unsigned long long index) {
  return (x ^ salt) * kStreamMul + static_cast<unsigned>(index);
}

// ---------------------------------------------------------------- STREAM
// TMA-staged (cp.async.bulk) pipeline: one elected thread streams the
// block's input through a ring of `stages` shared-memory tiles guarded by
// full/empty mbarriers; all 8 warps transform each landed tile and write it
// out with 128-bit non-allocating stores. Bytes in flight per worker are
// stages x 16 KiB of shared memory, not registers, which is what the
// register-staged version lacked (profiles/ncu_k_worker_r01_ldg.txt: 75 %
// of HBM peak, loads stalled on long-scoreboard with 16 warps per SM).
constexpr unsigned kTile = 16384;
constexpr unsigned kMaxStages = 8;

struct StreamPipe {
  unsigned char* tiles;        // stages x kTile, 1024-byte aligned
  unsigned long long* full;    // [stages] tile landed (1 arrive + tx bytes)
  unsigned long long* empty;   // [stages] tile consumed (8 warp arrivals)
  unsigned stages;
  unsigned long long used;     // tiles streamed by this CTA so far (all threads agree)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  const unsigned a = smem_u32(b);
  unsigned ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Called once per CTA by all threads before the first block.
__device__ __forceinline__ void stream_pipe_init(StreamPipe& P, unsigned char* smem,
                                                 unsigned smem_bytes, int tid) {
  P.full = reinterpret_cast<unsigned long long*>(smem);
  P.empty = P.full + kMaxStages;
  P.tiles = smem + 1024;
  P.stages = smem_bytes > 1024 ? (smem_bytes - 1024) / kTile : 0;
  if (P.stages > kMaxStages) P.stages = kMaxStages;
  P.used = 0;
  if (tid == 0) {
    for (unsigned s = 0; s < P.stages; ++s) {
      mbar_init(P.full + s, 1);
      mbar_init(P.empty + s, kWorkerThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

__device__ __forceinline__ void body_stream(const BlockCmd& c, int tid, StreamPipe& P) {
  const unsigned* src = reinterpret_cast<const unsigned*>(c.args[0]);
  unsigned* dst = reinterpret_cast<unsigned*>(c.args[1]);
  const unsigned long long words = c.args[2];
  const unsigned salt = static_cast<unsigned>(c.args[3]);
  const unsigned long long chunks = c.args[4];
  const unsigned long long chunk =
      chunks ? static_cast<unsigned long long>(c.block) % chunks
             : static_cast<unsigned long long>(c.block);
  // Slice `part` of the block covers a 16-byte-aligned share of its words.
  const unsigned long long quads = words / 4;
  const unsigned long long q0 = quads * c.part / c.parts;
  const unsigned long long q1 = quads * (c.part + 1) / c.parts;
  const unsigned long long first = chunk * words + 4 * q0;
  const unsigned long long bytes = 16 * (q1 - q0);
  if (bytes == 0) return;
  const unsigned n = static_cast<unsigned>((bytes + kTile - 1) / kTile);
  const unsigned S = P.stages;
  const unsigned long long g0 = P.used;
  const unsigned char* gin = reinterpret_cast<const unsigned char*>(src + first);
  uint4* gout = reinterpret_cast<uint4*>(dst + first);

  auto issue = [&](unsigned j) {  // thread 0 only
    const unsigned long long k = g0 + j;
    const unsigned s = static_cast<unsigned>(k % S);
    const unsigned long long r = k / S;
    if (r >= 1) mbar_wait(P.empty + s, static_cast<unsigned>((r - 1) & 1));
    const unsigned long long off = static_cast<unsigned long long>(j) * kTile;
    const unsigned tb = static_cast<unsigned>(bytes - off < kTile ? bytes - off : kTile);
    mbar_expect_tx(P.full + s, tb);
    bulk_load(P.tiles + s * kTile, gin + off, tb, P.full + s);
  };
  if (tid == 0)
    for (unsigned j = 0; j < n && j < S; ++j) issue(j);

  for (unsigned j = 0; j < n; ++j) {
    const unsigned long long k = g0 + j;
    const unsigned s = static_cast<unsigned>(k % S);
    mbar_wait(P.full + s, static_cast<unsigned>((k / S) & 1));
    const unsigned long long off = static_cast<unsigned long long>(j) * kTile;
    const unsigned tb = static_cast<unsigned>(bytes - off < kTile ? bytes - off : kTile);
    const uint4* t = reinterpret_cast<const uint4*>(P.tiles + s * kTile);
    uint4* out = gout + off / 16;
    const unsigned long long e0 = first + off / 4;
    for (unsigned v = tid; v < tb / 16; v += kWorkerThreads) {
      const uint4 x = t[v];
      const unsigned long long e = e0 + 4ull * v;
      uint4 y;
      y.x = stream_word(x.x, salt, e);
      y.y = stream_word(x.y, salt, e + 1);
      y.z = stream_word(x.z, salt, e + 2);
      y.w = stream_word(x.w, salt, e + 3);
      st_stream(out + v, y);
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(P.empty + s);
    if (tid == 0 && j + S < n) issue(j + S);
  }
  P.used = g0 + n;
}

__device__ __forceinline__ void body_spin(const BlockCmd& c, int tid) {
  if (tid != 0) return;
  const unsigned long long ns = c.args[0] * (c.part + 1) / c.parts - c.args[0] * c.part / c.parts;
  const unsigned long long t0 = gtimer();
  while (gtimer() - t0 < ns) {
  }
}

}  // namespace gpuos_dev_impl
