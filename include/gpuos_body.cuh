/* gpuos_body.cuh -- tenant-supplied atom bodies (device side).
 *
 * The reference atomizes a tenant's own kernel: a prelude makes every block
 * outside the atom's [lo, hi) exit at once, and the kept blocks recover
 * their blockIdx from the linearised index z (gy gx) + y gx + x
 * (PAPER.md:290-306). On the B200 the persistent dispatcher
 * hands a worker exactly the blocks of [lo, hi), so a tenant kernel runs as
 * atoms once its per-block code is written against this header instead of
 * the CUDA built-ins:
 *
 *   #include "gpuos_body.cuh"
 *   GPUOS_USER_BODY(my_kernel) {          // (const gpuos_block& b,
 *     ... b.x, b.y, b.z, b.tid ...        //  const unsigned long long* args)
 *   }
 *
 * blockIdx -> b.x / b.y / b.z (the prelude's decomposition of the linear
 * block index), gridDim -> b.gx / b.gy / b.gz (packed into args[4] with
 * GPUOS_GRID), threadIdx.x / blockDim.x -> b.tid / 256 (one worker CTA,
 * 256 threads), dynamic shared memory -> b.smem (b.smem_bytes bytes; no
 * asynchronous copy may be left in flight when the body returns).
 * __syncthreads() is allowed (every thread of the CTA runs the body).
 * args[0..3] are the tenant's.
 *
 * Bodies are compiled into the dispatcher: the build scans the body
 * sources (paper_2504_15465_b200/csrc/bodies/*.cu and build(user_bodies=))
 * for GPUOS_USER_BODY(name), assigns ids GPUOS_BODY_USER0 + i in sorted
 * name order, and generates the dispatch switch. The host looks a body up
 * by name (gpuos_dev_body_id) and submits atoms with that id.             */
#ifndef GPUOS_BODY_CUH_
#define GPUOS_BODY_CUH_

struct gpuos_block {
  long long block;        /* linear block index within the tenant's grid  */
  unsigned x, y, z;       /* blockIdx recovered from it      */
  unsigned gx, gy, gz;    /* gridDim (args[4], GPUOS_GRID)                 */
  int tid;                /* threadIdx.x: 0 .. 255                         */
  unsigned part, parts;   /* preemption slice of the block (parts >= 1)    */
  unsigned char* smem;    /* worker shared memory, 1024-byte aligned       */
  unsigned smem_bytes;
};

#define GPUOS_BLOCK_THREADS 256
#define GPUOS_GRID(gx, gy, gz)                                                  \
  ((unsigned long long)(gx) | ((unsigned long long)(gy) << 21) |               \
   ((unsigned long long)(gz) << 42))
#define GPUOS_USER_BODY(name) \
  __device__ void name(const gpuos_block& b, const unsigned long long* args)

#endif /* GPUOS_BODY_CUH_ */
