/*
 * gpuos_dev.h — C ABI of the B200 TPC dispatcher (the device seam).
 *
 * The reference's scheduler drives a concrete C++ DeviceEngine
 * (reference: proj/include/gpuos/device.hpp:79-121). On the B200 that seam
 * becomes a persistent sm_100a dispatcher kernel; this header is the thin,
 * language-neutral boundary a host scheduler (the gpuos:: C++ library in
 * this repo, or any FFI) binds to. Plain pointers and sizes only; every
 * function returns 0 on success or a negative GPUOS_E_* code and never
 * throws. The mapping to the reference seam (file:line in
 * proj/include/gpuos/device.hpp / proj/src/device.cpp):
 *
 *   gpuos_dev_open / _close        DeviceEngine ctor/dtor      device.hpp:81, device.cpp:74-81
 *   gpuos_dev_get_topology         topology()                  device.hpp:84
 *   gpuos_dev_submit_atom          submit_atom()               device.hpp:92-94, device.cpp:121-163
 *   gpuos_dev_set_atom_paused      set_atom_paused()           device.hpp:97, device.cpp:165-171
 *   gpuos_dev_poll                 completion handler / step() device.hpp:102-107, device.cpp:208-219,277-306
 *   gpuos_dev_now_ns               now()                       device.hpp:83
 *   gpuos_dev_set_tpc_fence        (new) TPC-ownership table: block-granular revocation
 *   gpuos_dev_start / _stop        (new) persistent-kernel lifetime, CUDA-event timing
 *   gpuos_dev_get_stats            tpc_busy_integral() etc.    device.hpp:112-118
 *
 * Threading: one host thread owns a handle (reference: device.hpp:76-78,
 * SPEC.md:111-112). The persistent kernel is the only concurrent actor.
 */
#ifndef GPUOS_DEV_H_
#define GPUOS_DEV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define GPUOS_OK 0
#define GPUOS_E_CONFIG (-2)    /* bad argument; maps to gpuos::ConfigError   */
#define GPUOS_E_INVARIANT (-3) /* internal state violated; InvariantError    */
#define GPUOS_E_CUDA (-4)      /* CUDA runtime failure; InvariantError       */
#define GPUOS_E_FULL (-5)      /* ring / atom table / TPC residency full      */
#define GPUOS_E_STATE (-6)     /* call not valid in the current state         */
#define GPUOS_E_TIMEOUT (-7)

/* ------------------------------------------------------------------ limits */
#define GPUOS_MAX_TPCS 128     /* logical TPC ids are < 128 (two 64-bit words) */
#define GPUOS_RESIDENT_PER_TPC 32

/* ------------------------------------------------------------ config flags */
/* start() prepares the run but does not launch the dispatcher; atoms
 * submitted before gpuos_dev_launch_workers() wait in the submit ring (at
 * most ring_entries of them), so the kernel starts with a backlog.        */
#define GPUOS_DEV_DEFER_WORKERS 1u

/* ------------------------------------------------------------ body kinds */
/* What one block of an atom executes (args per kind).                     */
#define GPUOS_BODY_STREAM 1u  /* args: src u32*, dst u32*, words/block (mult.
                                 of 4, 16 B aligned), salt, chunks (0 = none)
                                 block b covers chunk c = chunks ? b % chunks : b:
                                 dst[i] = (src[i] ^ salt) * 0x9E3779B1 + i
                                 for i in [c * words, (c + 1) * words)       */
#define GPUOS_BODY_GEMM_BF16 2u /* args: [0] = descriptor from
                                   gpuos_dev_gemm_desc(); block b = one
                                   256 x 256 output tile (grouped raster) of
                                   C = A . B^T on the tensor cores       */
#define GPUOS_BODY_SPIN 3u    /* args: ns to spin per block (globaltimer)    */
#define GPUOS_BODY_GEMV_BF16 4u /* args: [0] = descriptor from
                                   gpuos_dev_gemv_desc(); block b = rows
                                   [256 b, 256 b + 256) of y = W . x (decode
                                   GEMV, HBM-bound, tensor-core MACs)      */

/* Tenant-supplied bodies (include/gpuos_body.cuh), compiled into the
 * dispatcher by the body plug-in build: ids GPUOS_BODY_USER0 + i; look one
 * up by name with gpuos_dev_body_id. args[4] = GPUOS_GRID(gx, gy, gz).   */
#define GPUOS_BODY_USER0 64u
#define GPUOS_BODY_CONV_BF16 5u /* args: [0] = descriptor from
                                   gpuos_dev_conv_desc(); block b = 256
                                   output pixels x 256 output channels of an
                                   implicit-GEMM convolution on tcgen05    */

/* Launch-time configuration. Zero fields take the defaults in brackets.   */
typedef struct gpuos_dev_config {
  int32_t device_ordinal;   /* [0] */
  int32_t workers_per_sm;   /* resident worker CTAs per SM, 1 or 2 [2]
                               (each owns 512/W TMEM columns)             */
  int32_t logical_tpcs;     /* TPCs exposed, mapped onto physical TPCs
                               0..n-1 (smid>>1) [all = 74 on B200]        */
  int32_t atom_slots;       /* in-flight atom table size [4096]           */
  int32_t ring_entries;     /* host->device submit ring [4096]            */
  int32_t idle_sleep_ns;    /* worker back-off while idle [256]           */
  uint32_t flags;           /* GPUOS_DEV_* flags                          */
  int32_t pipeline_timeout_ms; /* bound on one tensor-core pipeline wait
                               (TMA / MMA / accumulator mbarriers) [2000];
                               on expiry the device raises a fault, the
                               dispatcher drains out and the host gets
                               GPUOS_E_TIMEOUT -- no context-killing trap.
                               Early-start gate waits are not bounded.   */
} gpuos_dev_config;

typedef struct gpuos_dev_topology {
  int32_t sm_count;          /* physical SMs (148 on B200)                */
  int32_t physical_tpcs;     /* sm_count / 2                              */
  int32_t logical_tpcs;      /* TPC ids accepted by submit_atom           */
  int32_t workers_per_sm;
  int32_t workers_per_tpc;   /* resident worker CTAs per logical TPC      */
  int32_t threads_per_worker;
  int32_t smem_per_worker;   /* bytes of dynamic shared memory            */
  int32_t reserved;
} gpuos_dev_topology;

/* One atom: a contiguous block range [lo, hi) of a tenant kernel, bound to
 * a TPC set at a priority (reference: submit_atom, device.cpp:121-163).    */
typedef struct gpuos_atom_desc {
  int64_t lo, hi;            /* block range, 0 <= lo < hi                   */
  uint64_t tpc_mask[2];      /* logical TPC set, bit t of word t/64         */
  int32_t priority;          /* higher wins freed slots (30 HP, 20 BE, 10
                                stolen); clamped to [0, 254]                */
  uint32_t body;             /* GPUOS_BODY_*                                */
  uint64_t args[5];          /* body arguments                              */
  uint64_t tag;              /* caller cookie, echoed in the completion     */
  uint32_t* trace;           /* optional per-block execution trace, indexed
                                by block id: += 0x10000 | (smid + 1)        */
  int32_t atomized;          /* informational (the prelude is free on B200) */
  uint32_t parts;            /* preemption quanta per block (0/1: whole
                                blocks). Each block runs as `parts` slices
                                claimed independently, so a higher-priority
                                atom waits at most one slice for a slot.
                                trace is then indexed block * parts + part. */
  uint32_t after;            /* kernel chaining: 1 + atom id of the
                                predecessor this atom runs behind (0: none).
                                The atom becomes claimable on the device the
                                moment the predecessor's last block ends --
                                no host round trip between the two. The
                                predecessor must carry GPUOS_ATOM_CHAIN_HEAD;
                                if it already completed (was polled) the atom
                                runs at once. poll() never reports an atom
                                before its predecessor.                     */
  uint32_t flags;            /* GPUOS_ATOM_*                                */
  uint32_t tenant;           /* 1 + the submitting tenant's id (< 65535), or
                                0: none. A TPC's owner (gpuos_dev_set_tpc_owner)
                                starts its own atoms there whatever its
                                fence floor.                               */
  uint32_t reserved;
} gpuos_atom_desc;

#define GPUOS_ATOM_CHAIN_HEAD 1u /* a successor may be chained behind this
                                    atom (its completion then arms it: one
                                    extra L2 atomic on the last block)    */
#define GPUOS_ATOM_NO_EARLY 2u   /* a chained tensor-core atom that must not
                                    start early (weights before its
                                    predecessor ends): set when the
                                    predecessor may run longer than the
                                    bodies' 2 s pipeline hang guard     */

typedef struct gpuos_completion {
  uint32_t atom_id;          /* id returned by gpuos_dev_submit_atom        */
  uint32_t blocks;           /* blocks executed                             */
  uint64_t tag;
  int64_t host_submit_ns;    /* gpuos_dev_now_ns() at submit                */
  int64_t host_complete_ns;  /* gpuos_dev_now_ns() when polled              */
  int64_t dev_first_start_ns;/* first block start, device clock, relative to open */
  int64_t dev_last_end_ns;   /* last block end, same clock                  */
  uint64_t tpc_touched[2];   /* logical TPCs that ran at least one block    */
  int64_t dev_ingest_ns;     /* ingest warp read the ring entry (device clock) */
  int64_t dev_armed_ns;      /* atom claimable on every TPC of its set      */
} gpuos_completion;

typedef struct gpuos_dev_stats {
  uint64_t blocks_executed;
  uint64_t atoms_completed;
  uint64_t worker_busy_ns;   /* summed block time over all workers          */
  uint64_t claim_retries;    /* lost CAS races on block claims              */
  int64_t kernel_elapsed_ns; /* CUDA-event time of the last start..stop     */
  int64_t ingest_entries;    /* ring entries consumed by the device         */
  int64_t worker_span_ns;    /* last run: first worker CTA entry .. last
                                exit on the device clock (the CUDA-event
                                time minus this is launch + teardown)      */
  int64_t first_block_ns;    /* last run: first worker entry .. first block
                                start (per-CTA setup: TMEM, barriers)      */
  uint64_t tpc_busy_ns;      /* summed over logical TPCs: time with >= 1
                                running block (the reference's
                                tpc_busy_integral, device.cpp:264-275),
                                sampled on the device by the ingest warp  */
  uint32_t fault;            /* last run's device fault code (0: none;
                                1: a pipeline wait expired; 2: a 2-SM
                                block claimed by a pair's second CTA)     */
  uint32_t reserved;
} gpuos_dev_stats;

int gpuos_dev_open(const gpuos_dev_config* cfg, struct gpuos_dev** out);
int gpuos_dev_close(struct gpuos_dev* dev);
int gpuos_dev_get_topology(struct gpuos_dev* dev, gpuos_dev_topology* out);

/* Launch the persistent dispatcher: ONE kernel (k_worker; its cluster 0
 * hosts the ingest warp), launched from a helper thread so a profiler that
 * serialises the launch (ncu) still lets this thread feed the ring.       */
int gpuos_dev_start(struct gpuos_dev* dev);
/* With GPUOS_DEV_DEFER_WORKERS: launch the dispatcher kernel now. */
int gpuos_dev_launch_workers(struct gpuos_dev* dev);
/* Batch mode (dispatcher stopped): stage n atoms directly into the device
 * tables and run the worker kernel alone until all complete. Returns its
 * CUDA-event time; completions are then read with gpuos_dev_poll. A single
 * self-contained launch: the path ncu profiles and rooflines are taken on. */
int gpuos_dev_run_batch(struct gpuos_dev* dev, const gpuos_atom_desc* descs, int32_t n,
                        float* elapsed_ms);
/* Ring entries consumed by the device / published by the host so far. */
int gpuos_dev_consumed(struct gpuos_dev* dev, uint64_t* consumed, uint64_t* published);
/* drain != 0: wait until every submitted atom completed, then stop.
 * Returns the worker kernel's CUDA-event elapsed time in *elapsed_ms.       */
int gpuos_dev_stop(struct gpuos_dev* dev, int drain, float* elapsed_ms);

int gpuos_dev_submit_atom(struct gpuos_dev* dev, const gpuos_atom_desc* desc,
                          uint32_t* atom_id);
int gpuos_dev_set_atom_paused(struct gpuos_dev* dev, uint32_t atom_id,
                              int paused);
/* Blocks of atoms below min_priority stop starting on `tpc` (0 lifts). */
int gpuos_dev_set_tpc_fence(struct gpuos_dev* dev, int32_t tpc,
                            int32_t min_priority);
/* Same for every TPC in the mask, as one ring entry. */
int gpuos_dev_set_fence_mask(struct gpuos_dev* dev, const uint64_t mask[2],
                             int32_t min_priority);
/* The device-resident TPC-ownership table: every TPC in the mask gets
 * `owner` (1 + tenant id, 0: none) and a fence floor. Atoms of the owner
 * (gpuos_atom_desc::tenant == owner) start blocks there at any priority;
 * other atoms only at priority >= min_priority (0 lifts the fence). This
 * is block-granular revocation: a busy owner's quota stops accepting
 * other tenants' stolen blocks without fencing the owner's own atoms that
 * span its quota and stolen TPCs (reference: the ledger's owner field and
 * revocation, scheduler.hpp:61-66, scheduler.cpp:239-270).              */
int gpuos_dev_set_tpc_owner(struct gpuos_dev* dev, const uint64_t mask[2], uint32_t owner,
                            int32_t min_priority);
/* Pair fence: on every TPC in the mask, only the worker pairs whose slot
 * bit is set in pair_slots (bit i: the TPC's i-th pair, W pairs per TPC)
 * stop starting blocks of atoms below min_priority (0 lifts); the TPC's
 * other pairs accept every atom. Replaces the TPC's owner entry. Lets a
 * latency-critical tenant keep one pair per TPC free of best-effort tiles
 * while best-effort work keeps the other (no reference counterpart: the
 * reference's TPC is the unit of revocation, scheduler.cpp:239-270).     */
int gpuos_dev_set_pair_fence(struct gpuos_dev* dev, const uint64_t mask[2], uint32_t pair_slots,
                             int32_t min_priority);
/* Non-blocking; returns the number of completions written to out[0..max). */
int gpuos_dev_poll(struct gpuos_dev* dev, gpuos_completion* out, int32_t max);
int64_t gpuos_dev_now_ns(struct gpuos_dev* dev);
int32_t gpuos_dev_in_flight(struct gpuos_dev* dev);
int gpuos_dev_get_stats(struct gpuos_dev* dev, gpuos_dev_stats* out);

/* GEMM body descriptor (GPUOS_BODY_GEMM_BF16): C[M,N] = A[M,K] . B[N,K]^T
 * with bf16 operands (both K-major, rows 16-byte aligned: K % 8 == 0), fp32
 * accumulation on tcgen05 tensor cores, fp32 output (flags 0) or bf16
 * (GPUOS_GEMM_OUT_BF16), row-major C with leading dimension ldc elements.
 * Builds the TMA tensor maps, writes the descriptor to device memory and
 * returns it in *desc (pass as args[0]; release with gpuos_dev_free), the
 * tenant kernel's grid in *blocks and the tile shape in *tile_m / *tile_n
 * (256 x 256: one tile per block, computed by a TPC's two SMs together with
 * tcgen05.mma.cta_group::2). No reference counterpart: the reference's
 * "block" is a duration (device.hpp:39-47).                              */
#define GPUOS_GEMM_OUT_BF16 1u
int gpuos_dev_gemm_desc(struct gpuos_dev* dev, const void* a, const void* b, void* c,
                        int64_t m, int64_t n, int64_t k, int64_t ldc, uint32_t flags,
                        void** desc, int64_t* blocks, int32_t* tile_m, int32_t* tile_n);
/* Split-K variant: k_splits > 1 also splits K (shapes with few output tiles
 * and a long K, e.g. weight gradients): block b = (tile b % tiles, K split
 * b / tiles), *blocks = tiles x splits; each split adds its fp32 tile into
 * the tile's accumulator (vector float reductions in L2, so the fp32 sum
 * order is the splits' arrival order) and the tile's last split writes C.
 * One run of a descriptor at a time. k_splits <= 1 is gpuos_dev_gemm_desc.*/
int gpuos_dev_gemm_desc_splitk(struct gpuos_dev* dev, const void* a, const void* b, void* c,
                               int64_t m, int64_t n, int64_t k, int64_t ldc, uint32_t flags,
                               int32_t k_splits, void** desc, int64_t* blocks, int32_t* tile_m,
                               int32_t* tile_n);

/* GEMV body descriptor (GPUOS_BODY_GEMV_BF16): y[N] = W[N,K] . x[K] with
 * bf16 W and x (16-byte aligned, K % 8 == 0), fp32 accumulation, fp32 y
 * (flags 0) or bf16 (GPUOS_GEMV_OUT_BF16). Blocks are 256-row tiles of W
 * computed by a TPC's two SMs (tcgen05.mma.cta_group::2, M = 256, N = 32
 * with x as the only non-zero column). k_splits > 1 also splits K (decode
 * shapes have few row tiles): block b = (row tile b % row_tiles, K split
 * b / row_tiles); the row tile's last block sums the partials in split
 * order (deterministic) and writes y. One run of a descriptor at a time.
 * The content of x (and W) may change between runs; the descriptor holds
 * addresses. Release with gpuos_dev_free. No reference counterpart
 * (device.hpp:39-47).                                                    */
#define GPUOS_GEMV_OUT_BF16 1u
/* W pre-packed by gpuos_dev_gemv_pack (each ring stage one contiguous
 * 16 KiB range): pass the packed buffer as w.                            */
#define GPUOS_GEMV_W_PACKED 2u
int gpuos_dev_gemv_desc(struct gpuos_dev* dev, const void* w, const void* x, void* y,
                        int64_t n, int64_t k, uint32_t flags, int32_t k_splits, void** desc,
                        int64_t* blocks);

/* Repacks row-major bf16 W [n, k] into the GEMV's packed layout
 * [ceil(n/128)][ceil(k/64)][128][64] (zero beyond n, k) on the side
 * stream; dst holds GPUOS_GEMV_PACKED_BYTES(n, k) bytes. Weights are packed
 * once, when a tenant loads them.                                        */
int gpuos_dev_gemv_pack(struct gpuos_dev* dev, void* dst, const void* src, int64_t n, int64_t k);
#define GPUOS_GEMV_PACKED_BYTES(n, k) \
  ((uint64_t)(((n) + 127) / 128) * (uint64_t)(((k) + 63) / 64) * 128u * 64u * 2u)

/* Convolution body descriptor (GPUOS_BODY_CONV_BF16): y = conv2d(x, w),
 * x NHWC bf16 [n, h, wd, c] (c % 8 == 0), w bf16 [k][r][s][cb] with cb = c
 * rounded up to 64 (zero-padded channels), padding `pad`, stride 1 or 2,
 * y NHWC [n, p, q, k] fp32 (flags 0) or bf16 (GPUOS_CONV_OUT_BF16) with
 * p = (h + 2 pad - r) / stride + 1 (q likewise). Implicit GEMM on a TPC's
 * two SMs: each K-step is one 4-D TMA box of x (an output patch's input
 * pixels for one filter tap and 64 channels; padding is the TMA's zero
 * fill) and one 2-D box of w. Returns the descriptor (args[0]; release with
 * gpuos_dev_free), the grid and the output size.                        */
#define GPUOS_CONV_OUT_BF16 1u
int gpuos_dev_conv_desc(struct gpuos_dev* dev, const void* x, const void* w, void* y, int32_t n,
                        int32_t h, int32_t wd, int32_t c, int32_t k, int32_t r, int32_t s,
                        int32_t pad, int32_t stride, uint32_t flags, void** desc, int64_t* blocks,
                        int32_t* p, int32_t* q);

/* Uniform [-1, 1) bf16 contents from a counter hash (tenant operand init),
 * on the side stream.                                                     */
int gpuos_dev_fill_bf16(struct gpuos_dev* dev, void* ptr, uint64_t count, uint64_t seed);

/* Device memory helpers (stream-ordered on a side stream: safe while the
 * persistent dispatcher runs; never synchronise the whole device).        */
int gpuos_dev_alloc(struct gpuos_dev* dev, uint64_t bytes, void** ptr);
int gpuos_dev_free(struct gpuos_dev* dev, void* ptr);
int gpuos_dev_copy(struct gpuos_dev* dev, void* dst, const void* src,
                   uint64_t bytes, int kind /* 1 H2D, 2 D2H, 3 D2D */);
int gpuos_dev_memset(struct gpuos_dev* dev, void* dst, int value, uint64_t bytes);
/* Pinned host memory for tenant inputs/outputs (fast, truly async H2D/D2H). */
int gpuos_dev_host_alloc(struct gpuos_dev* dev, uint64_t bytes, void** ptr);
int gpuos_dev_host_free(struct gpuos_dev* dev, void* ptr);

const char* gpuos_dev_last_error(void);

/* Diagnostics: the in-flight atoms' device state (claim offset, done
 * count, pause / gate bits, chaining) as text into buf (truncated to len);
 * safe while the dispatcher runs. Returns the full length.               */
int gpuos_dev_debug_dump(struct gpuos_dev* dev, char* buf, int32_t len);

/* Id of the tenant body GPUOS_USER_BODY(name) compiled into this library
 * (GPUOS_BODY_USER0 + i); GPUOS_E_CONFIG if there is none. Host only.    */
int gpuos_dev_body_id(const char* name, uint32_t* id);

/* ---- power and clocks (NVML, loaded at run time) --------------------
 * The reference models power and integrates it into energy
 * (device.cpp:221-242) and its power manager picks frequencies
 * (power_manager.cpp:27-105). On the B200 the energy is the GPU's own
 * counter; a chosen frequency can be applied as a locked SM clock
 * (B200Options::dvfs_actuate -- off wherever the operator manages clocks).
 * By CUDA device ordinal; GPUOS_E_CUDA when NVML is unavailable.          */
typedef struct gpuos_power_sample_t {
  uint64_t energy_mj;            /* total energy since driver load, mJ     */
  uint64_t clock_event_reasons;  /* NVML clocks-event (throttle) reasons   */
  uint32_t sm_mhz, mem_mhz;      /* current clocks                         */
  uint32_t power_mw;             /* current board power                    */
  uint32_t reserved;
} gpuos_power_sample_t;
int gpuos_power_sample(int32_t cuda_device, gpuos_power_sample_t* out);
/* Locks the SM clock to mhz (min = max); 0 restores default boosting.    */
int gpuos_power_lock_sm_clock(int32_t cuda_device, uint32_t mhz);

#ifdef __cplusplus
}
#endif

#endif /* GPUOS_DEV_H_ */
