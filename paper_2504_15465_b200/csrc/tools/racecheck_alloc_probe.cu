// Minimal reproducer for the only racecheck report on the dispatcher
// (profiles/sanitizer_racecheck_r02.txt): a hazard between a write and the
// shared-memory access of `tcgen05.alloc` itself. This kernel does nothing
// but the dispatcher's allocation sequence -- warp 1 allocates TMEM columns
// into a __shared__ word, tcgen05 fence, __syncthreads, every thread reads
// the word, dealloc -- so a report here is the tool's model of tcgen05.alloc
// (an asynchronous tensor-memory-allocator write to shared memory), not a
// race in the dispatcher.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o racecheck_alloc_probe racecheck_alloc_probe.cu
//   compute-sanitizer --tool racecheck ./racecheck_alloc_probe
#include <cstdio>

__global__ void k_alloc(unsigned* out, int variant) {
  __shared__ unsigned holder;
  __shared__ unsigned other;
  if (threadIdx.x == 0) other = 1u;  // an ordinary shared write beside it (variant 1)
  if (threadIdx.x / 32 == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(&holder))),
                 "r"(64u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned base = holder;
  if (variant == 1) out[blockIdx.x * blockDim.x + threadIdx.x] = base + other;
  else out[blockIdx.x * blockDim.x + threadIdx.x] = base;
  __syncthreads();
  if (threadIdx.x / 32 == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(64u) : "memory");
}

int main() {
  unsigned* out = nullptr;
  cudaMalloc(&out, 148 * 128 * sizeof(unsigned));
  for (int v = 0; v < 2; ++v) k_alloc<<<148, 128>>>(out, v);
  const cudaError_t e = cudaDeviceSynchronize();
  std::printf("racecheck_alloc_probe: %s\n", cudaGetErrorString(e));
  cudaFree(out);
  return e == cudaSuccess ? 0 : 1;
}
