// Residency probe: launches W CTAs per SM of a persistent-style kernel (one
// small CTA first on another stream, like the dispatcher's ingest warp) and
// records %smid at start and after a spin, to check that every SM hosts
// exactly W CTAs and whether %smid changes while CTAs stay resident.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));               \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

__device__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ unsigned long long gt() {
  unsigned long long r;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(r));
  return r;
}

__global__ void k_small(volatile int* stop) {
  while (!*stop) __nanosleep(1000);
}

__global__ void __launch_bounds__(256, 1) k_big(unsigned* s0, unsigned* s1, unsigned long long ns,
                                                volatile int* arrived, int total) {
  extern __shared__ unsigned char smem[];
  if (threadIdx.x == 0) {
    s0[blockIdx.x] = smid();
    smem[0] = 1;
    atomicAdd((int*)arrived, 1);
    unsigned long long t0 = gt();
    while (gt() - t0 < ns) {
    }
    s1[blockIdx.x] = smid();
  }
  __syncthreads();
}

int main(int argc, char** argv) {
  int W = argc > 1 ? std::atoi(argv[1]) : 2;
  int with_small = argc > 2 ? std::atoi(argv[2]) : 1;
  int carve = argc > 3 ? std::atoi(argv[3]) : 0;      // 1: max-shared carveout on both
  int big_first = argc > 4 ? std::atoi(argv[4]) : 0;  // 1: launch the big kernel first
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  int smem = (int)p.sharedMemPerMultiprocessor / W - 2048;
  smem -= smem % 1024;
  CK(cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (carve) {
    CK(cudaFuncSetAttribute(k_big, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaFuncSetAttribute(k_small, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  }
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_big, 256, smem));
  int grid = nsm * W;
  unsigned *s0, *s1;
  int *stop, *arrived;
  CK(cudaMallocManaged(&s0, grid * 4));
  CK(cudaMallocManaged(&s1, grid * 4));
  CK(cudaHostAlloc(&stop, 4, cudaHostAllocMapped));
  CK(cudaMallocManaged(&arrived, 4));
  *stop = 0;
  *arrived = 0;
  cudaStream_t a, b;
  CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
  int* stop_d;
  CK(cudaHostGetDevicePointer(&stop_d, stop, 0));
  if (with_small && !big_first) k_small<<<1, 32, 0, a>>>(stop_d);
  k_big<<<grid, 256, smem, b>>>(s0, s1, 2000000000ull, arrived, grid);
  if (with_small && big_first) k_small<<<1, 32, 0, a>>>(stop_d);
  CK(cudaStreamSynchronize(b));
  *stop = 1;
  CK(cudaDeviceSynchronize());
  std::map<unsigned, int> c0, c1;
  int changed = 0;
  for (int i = 0; i < grid; ++i) {
    c0[s0[i]]++;
    c1[s1[i]]++;
    changed += s0[i] != s1[i];
  }
  int bad0 = 0, bad1 = 0;
  for (auto& [k, v] : c0) bad0 += v != W;
  for (auto& [k, v] : c1) bad1 += v != W;
  std::printf("{\"carve\": %d, \"big_first\": %d, \"W\": %d, \"small\": %d, \"smem\": %d, \"occ_api\": %d, \"grid\": %d, "
              "\"distinct_start\": %zu, \"sms_not_W_start\": %d, \"distinct_end\": %zu, "
              "\"sms_not_W_end\": %d, \"smid_changed\": %d}\n",
              carve, big_first, W, with_small, smem, per, grid, c0.size(), bad0, c1.size(), bad1, changed);
  return 0;
}
