// Atom bodies: what one block of a tenant kernel executes inside a resident
// dispatcher worker CTA (256 threads). The reference models a block only
// as a duration (device.hpp:39-47); on the B200 each block does real work.
//
//   STREAM  HBM-bound transform, dst[i] = (src[i] ^ salt) * 0x9E3779B1 + i
//           over a contiguous chunk of `words` u32 per block (block b works
//           on chunk b % chunks when args[4] = chunks > 0, so a large grid
//           can stream through a bounded workspace); 128-bit
//           coalesced non-allocating loads/stores, 8 x 16 B in flight per
//           thread (32 KiB per worker). Algorithmic bytes: 8 per word.
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
};

__device__ __forceinline__ unsigned stream_word(unsigned x, unsigned salt,
                                                unsigned long long index) {
  return (x ^ salt) * kStreamMul + static_cast<unsigned>(index);
}

__device__ __forceinline__ void body_stream(const BlockCmd& c, int tid) {
  const uint4* src = reinterpret_cast<const uint4*>(c.args[0]);
  uint4* dst = reinterpret_cast<uint4*>(c.args[1]);
  const unsigned long long words = c.args[2];
  const unsigned salt = static_cast<unsigned>(c.args[3]);
  const unsigned long long chunks = c.args[4];
  const unsigned long long chunk =
      chunks ? static_cast<unsigned long long>(c.block) % chunks
             : static_cast<unsigned long long>(c.block);
  const unsigned long long first = chunk * words;
  const uint4* s = src + first / 4;
  uint4* d = dst + first / 4;
  const unsigned n4 = static_cast<unsigned>(words / 4);
  constexpr int U = 8;
  for (unsigned i0 = tid; i0 < n4; i0 += kWorkerThreads * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned i = i0 + u * kWorkerThreads;
      if (i < n4) v[u] = ld_stream(s + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned i = i0 + u * kWorkerThreads;
      if (i < n4) {
        const unsigned long long e = first + 4ull * i;
        uint4 o;
        o.x = stream_word(v[u].x, salt, e);
        o.y = stream_word(v[u].y, salt, e + 1);
        o.z = stream_word(v[u].z, salt, e + 2);
        o.w = stream_word(v[u].w, salt, e + 3);
        st_stream(d + i, o);
      }
    }
  }
}

__device__ __forceinline__ void body_spin(const BlockCmd& c, int tid) {
  if (tid != 0) return;
  const unsigned long long t0 = gtimer();
  while (gtimer() - t0 < c.args[0]) {
  }
}

}  // namespace gpuos_dev_impl
