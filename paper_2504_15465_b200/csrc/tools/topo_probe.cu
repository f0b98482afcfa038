// Topology probe for the B200 TPC dispatcher.
//
// Measures, on the live device, the facts the persistent dispatcher depends
// on and that the reference only models (DeviceTopology, device.hpp:14-24):
//   * SM count and %nsmid;
//   * which SM ids a 2-CTA cluster lands on (TPC pairing: expect {2k, 2k+1});
//   * GPC membership, from the SM sets of maximal clusters;
//   * %globaltimer resolution and its offset to the host's CLOCK_REALTIME;
//   * the host <-> device round trip through pinned mapped memory, which
//     bounds the dispatcher's publish -> first-block latency.
// Output: one JSON document on stdout.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <thread>
#include <vector>
#include <time.h>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x,       \
                   cudaGetErrorString(e_));                                \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned nsmid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long r;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}

__global__ void k_where(unsigned* out_smid, unsigned* out_nsmid, int spin_ns) {
  unsigned long long t0 = gtimer();
  // Hold the SM briefly so every CTA of the wave is co-resident.
  while (gtimer() - t0 < (unsigned long long)spin_ns) {
  }
  if (threadIdx.x == 0) {
    out_smid[blockIdx.x] = smid();
    out_nsmid[blockIdx.x] = nsmid();
  }
}

__global__ void k_cluster(unsigned* out_smid, unsigned* out_rank,
                          unsigned* out_cid, int spin_ns) {
  unsigned long long t0 = gtimer();
  while (gtimer() - t0 < (unsigned long long)spin_ns) {
  }
  if (threadIdx.x == 0) {
    out_smid[blockIdx.x] = smid();
    out_rank[blockIdx.x] = cluster_rank();
    out_cid[blockIdx.x] = cluster_id_x();
  }
}

__global__ void k_timer(unsigned long long* deltas, int n) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long prev = gtimer();
  int k = 0;
  while (k < n) {
    unsigned long long t = gtimer();
    if (t != prev) {
      deltas[k++] = t - prev;
      prev = t;
    }
  }
}

__global__ void k_gt_now(unsigned long long* out) { *out = gtimer(); }

// Ping-pong through pinned mapped host memory: host writes ping=i, device
// answers pong=i. Device polls with system-scope acquire loads.
__global__ void k_pingpong(volatile unsigned* ping, volatile unsigned* pong,
                           int iters) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = 1; i <= iters; ++i) {
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];"
                   : "=r"(v)
                   : "l"(ping)
                   : "memory");
    } while (v != (unsigned)i);
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pong), "r"(i)
                 : "memory");
  }
}

static long long host_realtime_ns() {
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return (long long)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int nsm = prop.multiProcessorCount;
  std::printf("{\n  \"name\": \"%s\", \"cc\": \"%d.%d\", \"sm_count\": %d,\n",
              prop.name, prop.major, prop.minor, nsm);
  std::printf("  \"smem_per_block_optin\": %zu, \"smem_per_sm\": %zu, "
              "\"regs_per_sm\": %d, \"l2_bytes\": %d, \"clock_khz\": %d,\n",
              prop.sharedMemPerBlockOptin, prop.sharedMemPerMultiprocessor,
              prop.regsPerMultiprocessor, prop.l2CacheSize, prop.clockRate);

  // 1. Plain launch: which SM ids exist.
  {
    int grid = nsm;
    unsigned *d_s, *d_n;
    CK(cudaMalloc(&d_s, grid * 4));
    CK(cudaMalloc(&d_n, grid * 4));
    k_where<<<grid, 32>>>(d_s, d_n, 200000);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned> s(grid), n(grid);
    CK(cudaMemcpy(s.data(), d_s, grid * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(n.data(), d_n, grid * 4, cudaMemcpyDeviceToHost));
    std::set<unsigned> uniq(s.begin(), s.end());
    std::printf("  \"nsmid\": %u, \"distinct_smid_one_wave\": %zu, "
                "\"max_smid\": %u,\n  \"bid_to_smid\": [",
                n[0], uniq.size(), *uniq.rbegin());
    for (int i = 0; i < grid; ++i) std::printf("%s%u", i ? "," : "", s[i]);
    std::printf("],\n");
    CK(cudaFree(d_s));
    CK(cudaFree(d_n));
  }

  // 2. Cluster launches of size 2 (TPC pairing) and the largest size that
  //    launches (GPC membership).
  for (int csz : {2, 16, 8}) {
    if (csz == 16) {
      cudaError_t e = cudaFuncSetAttribute(
          k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csz;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(32);
    int max_clusters = 0;
    cfg.gridDim = dim3(csz * 4);
    if (cudaOccupancyMaxActiveClusters(&max_clusters, k_cluster, &cfg) !=
        cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (max_clusters < 1) continue;
    int grid = max_clusters * csz;
    cfg.gridDim = dim3(grid);
    unsigned *d_s, *d_r, *d_c;
    CK(cudaMalloc(&d_s, grid * 4));
    CK(cudaMalloc(&d_r, grid * 4));
    CK(cudaMalloc(&d_c, grid * 4));
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, d_s, d_r, d_c, 200000);
    if (e != cudaSuccess) {
      std::printf("  \"cluster%d_error\": \"%s\",\n", csz, cudaGetErrorString(e));
      cudaGetLastError();
      continue;
    }
    CK(cudaDeviceSynchronize());
    std::vector<unsigned> s(grid), r(grid), c(grid);
    CK(cudaMemcpy(s.data(), d_s, grid * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r.data(), d_r, grid * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(c.data(), d_c, grid * 4, cudaMemcpyDeviceToHost));
    std::map<unsigned, std::vector<std::pair<unsigned, unsigned>>> by_cluster;
    for (int i = 0; i < grid; ++i) by_cluster[c[i]].push_back({r[i], s[i]});
    std::printf("  \"cluster%d_max_active\": %d,\n  \"cluster%d_sm_sets\": [",
                csz, max_clusters, csz);
    bool first = true;
    int pairs_tpc_aligned = 0, pairs = 0;
    for (auto& [cid, v] : by_cluster) {
      std::sort(v.begin(), v.end());
      std::printf("%s[", first ? "" : ",");
      first = false;
      for (size_t k = 0; k < v.size(); ++k)
        std::printf("%s%u", k ? "," : "", v[k].second);
      std::printf("]");
      if (csz == 2 && v.size() == 2) {
        ++pairs;
        unsigned a = v[0].second, b = v[1].second;
        if ((a >> 1) == (b >> 1)) ++pairs_tpc_aligned;
      }
    }
    std::printf("],\n");
    if (csz == 2)
      std::printf("  \"cluster2_pairs\": %d, \"cluster2_pairs_same_smid_div2\": %d,\n",
                  pairs, pairs_tpc_aligned);
    CK(cudaFree(d_s));
    CK(cudaFree(d_r));
    CK(cudaFree(d_c));
  }

  // 3. %globaltimer resolution.
  {
    const int n = 256;
    unsigned long long* d;
    CK(cudaMalloc(&d, n * 8));
    k_timer<<<1, 32>>>(d, n);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> v(n);
    CK(cudaMemcpy(v.data(), d, n * 8, cudaMemcpyDeviceToHost));
    std::sort(v.begin(), v.end());
    std::printf("  \"globaltimer_delta_ns\": {\"min\": %llu, \"median\": %llu, "
                "\"max\": %llu},\n",
                v[0], v[n / 2], v[n - 1]);
    // Offset to host CLOCK_REALTIME.
    unsigned long long* g;
    CK(cudaHostAlloc(&g, 8, cudaHostAllocMapped));
    unsigned long long* gd;
    CK(cudaHostGetDevicePointer(&gd, g, 0));
    long long best = 1LL << 62, off = 0;
    for (int i = 0; i < 20; ++i) {
      long long h0 = host_realtime_ns();
      k_gt_now<<<1, 1>>>(gd);
      CK(cudaDeviceSynchronize());
      long long h1 = host_realtime_ns();
      if (h1 - h0 < best) {
        best = h1 - h0;
        off = (long long)*g - (h0 + h1) / 2;
      }
    }
    std::printf("  \"globaltimer_minus_realtime_ns\": %lld, "
                "\"launch_sync_roundtrip_ns\": %lld,\n",
                off, best);
    CK(cudaFree(d));
    CK(cudaFreeHost(g));
  }

  // 4. Host <-> device ping-pong through mapped pinned memory.
  {
    unsigned* h;
    CK(cudaHostAlloc(&h, 256, cudaHostAllocMapped));
    volatile unsigned* ping = h;
    volatile unsigned* pong = h + 32;
    *ping = 0;
    *pong = 0;
    unsigned* d;
    CK(cudaHostGetDevicePointer(&d, h, 0));
    const int iters = 2000;
    k_pingpong<<<1, 32>>>(d, d + 32, iters);
    std::vector<double> rt;
    for (int i = 1; i <= iters; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      __atomic_store_n((unsigned*)ping, (unsigned)i, __ATOMIC_RELEASE);
      while (__atomic_load_n((unsigned*)pong, __ATOMIC_ACQUIRE) != (unsigned)i) {
      }
      auto t1 = std::chrono::steady_clock::now();
      rt.push_back(std::chrono::duration<double, std::nano>(t1 - t0).count());
    }
    CK(cudaDeviceSynchronize());
    std::sort(rt.begin(), rt.end());
    std::printf("  \"mapped_pingpong_rtt_ns\": {\"p10\": %.0f, \"p50\": %.0f, "
                "\"p90\": %.0f, \"p99\": %.0f},\n",
                rt[iters / 10], rt[iters / 2], rt[iters * 9 / 10],
                rt[iters * 99 / 100]);
    CK(cudaFreeHost(h));
  }
  std::printf("  \"ok\": true\n}\n");
  return 0;
}
