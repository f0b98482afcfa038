// Persistent sm_100a TPC dispatcher and its C ABI (include/gpuos_dev.h).
//
// The reference's DeviceEngine (device.cpp:74-311) models a GPU as a pool of
// TPCs whose block slots refill from the highest-priority resident atom.
// Here that model is executed for real:
//
//   host scheduler --submit ring (pinned, mapped)--> INGEST warp (1 CTA)
//        ^                                              | writes atom slot,
//        |                                              v inserts resident keys
//   completion ring <--last block-- WORKER CTAs (W per SM, 148 SMs)
//
// * Every worker CTA reads %smid; TPC = smid >> 1 (2-CTA clusters always land
//   on SMs {2k, 2k+1}: profiles/topology_probe_r01.json) and maps it to a
//   logical TPC id through a device table.
// * Each logical TPC owns a 32-entry resident list of 64-bit keys
//   (priority << 56 | ~seq << 24 | slot). Warp 0 of a free worker reads the
//   list (one entry per lane), keeps the atoms that still have waiting
//   blocks, are not paused and clear the TPC's fence, and takes the maximum
//   key: highest priority, then oldest atom -- the reference's refill rule
//   (device.cpp:188-206). There is no lower-priority bypass: a lane-parallel
//   max over eligible atoms picks exactly one.
// * Lane 0 claims a block with a fetch-add on the atom's claim word
//   (seq << 32 | next offset); the sequence tag tells a stale key for a
//   recycled slot apart (its offset is run for the slot's new occupant).
// * All 8 warps run the body; warp 0 then accounts the block and, for the
//   atom's last block, arms a chained successor (or opens its early-start
//   gate), writes the completion record (device timestamps, TPCs touched)
//   into host-mapped memory and removes its resident keys.
// * Block-granular revocation: fence[tpc] is a minimum priority; raising it
//   stops stolen atoms from starting new blocks there without a relaunch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <atomic>
#include <chrono>
#include <memory>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "bodies.cuh"
#include "gemm_body.cuh"
#include "gemv_body.cuh"
#include "conv_body.cuh"
#include "gpuos_dev.h"
#include "gpuos_user_bodies.cuh"  // generated (build.py): tenant bodies
#include "ptx.cuh"

namespace gpuos_dev_impl {

constexpr int kResident = GPUOS_RESIDENT_PER_TPC;  // keys per TPC (one per lane)
static_assert(kResident == 32, "one resident key per lane");

// Handoff probe (GPUOS_PROBE_HANDOFF builds only, tools/chain_gap_probe.py):
// SM clock stamps along a finisher's path into the block it handed itself.
#ifdef GPUOS_PROBE_HANDOFF
constexpr int kProbeStamps = 12;
__device__ unsigned long long g_probe_cur[1184][kProbeStamps];
__device__ unsigned long long g_probe_ring[4096][kProbeStamps];
__device__ unsigned g_probe_n;
#define PROBE_AT(i) (g_probe_cur[blockIdx.x][i] = clock64())
#else
#define PROBE_AT(i) ((void)0)
#endif

enum Op : unsigned { kOpSubmit = 1, kOpPause = 2, kOpResume = 3, kOpFence = 4,
                     kOpDrain = 5, kOpShutdown = 6, kOpFenceMask = 7 };

// Device-resident atom slot. The first 128-byte line holds everything a
// claiming worker reads (claim word, count, pause flag, block range, body and
// its arguments); the ingest warp writes the rest once.
struct alignas(128) DevAtom {
  unsigned long long claim;  // +0  seq << 32 | next slice offset (fetch-add)
  unsigned count;            // +8  slices = blocks x parts
  unsigned paused;           // +12 (claim, count, paused): one 16-byte load.
                             //     bit 0: paused; bit 1 (kGatedBit): early-started, gate
                             //     closed (its tiles wait for it to clear before reading x / A)
  long long lo;              // +16 first block
  unsigned body;             // +24
  unsigned parts;            // +28 slices per block
  unsigned long long args[5];  // +32 .. +72
  unsigned seq;              // +72
  int prio;                  // +76 1..255
  unsigned done;             // +80 finished slices
  unsigned pad0;             // +84
  unsigned long long tag;    // +88
  unsigned* trace;           // +96
  unsigned long long mask[2];  // +104
  unsigned chain;            // +120 kChainHead: completion arms a successor
  unsigned succ;             // +124 chained successor: slot + 1, kSuccDone once finished
  unsigned long long t_first, t_last;   // second line: first slice's start (t_last unused)
  unsigned long long touched[2];
  unsigned long long t_seen, t_armed;   // ingest instrumentation (globaltimer)
  unsigned pad1;
  unsigned armed;                       // claim armed (blocks claimable or claimed)
  unsigned char entry[GPUOS_MAX_TPCS];  // resident-list index per TPC
};
static_assert(offsetof(DevAtom, succ) + 4 <= 128, "hot fields must share one line");
static_assert(offsetof(DevAtom, chain) % 8 == 0 && offsetof(DevAtom, succ) == offsetof(DevAtom, chain) + 4,
              "chain | succ: one 64-bit load");

// Kernel chaining (gpuos_atom_desc::after). A successor is ingested
// unarmed (claim exhausted, keys resident); the ingest warp then registers
// it on the predecessor with a CAS on `succ`, and the predecessor's
// finishing worker swaps in kSuccDone. Whichever comes second arms the
// successor: exactly one does, and a successor registered after the
// predecessor finished is armed by the ingest warp itself.
constexpr unsigned kSuccDone = 0xffffffffu;
// DevAtom::succ: a look-ahead (the finisher that armed this atom) claimed
// the right to arm the registered successor early, behind a closed gate;
// this atom's finisher then opens that gate once the successor is armed
// (account_block). Set by CAS, so it never races the finisher's swap.
constexpr unsigned kSuccLook = 0x80000000u;
constexpr unsigned kGatedBit = 2u;  // DevAtom::paused: early start, gate closed

// Opens an early-started atom's gate (release: the predecessor's outputs,
// which the caller has acquired, become visible to the gate's waiters).
__device__ __forceinline__ void open_gate(unsigned* paused) {
  asm volatile("red.release.gpu.global.and.b32 [%0], %1;" ::"l"(paused), "r"(~kGatedBit) : "memory");
}
constexpr unsigned kChainHead = 1u;

// The TPC-ownership table (gpuos_dev_set_tpc_owner): fence[t] = owner << 16
// | floor, owner = 1 + tenant id (0: none). An atom starts blocks on t when
// its priority reaches the floor or it belongs to the owner -- the owner's
// atoms that span its quota and stolen TPCs run at the stolen priority
// and would otherwise be fenced off their own quota. An atom's tenant
// travels in DevAtom::paused bits 16..31 (read with the claim word).
// Bits 8..15: the worker-pair slots of the TPC the floor applies to (0: all;
// gpuos_dev_set_pair_fence). A TPC runs W worker pairs; each knows its slot
// (WorkerShared::pair_slot, numbered in arrival order at launch).
__device__ __forceinline__ bool fence_admits(int fence, int prio, unsigned tenant, unsigned pair_slot) {
  const unsigned slots = (static_cast<unsigned>(fence) >> 8) & 0xffu;
  if (slots != 0u && !((slots >> pair_slot) & 1u)) return true;
  const unsigned owner = static_cast<unsigned>(fence) >> 16;
  return prio >= (fence & 0xff) || (owner != 0u && owner == tenant);
}
__device__ __forceinline__ unsigned tenant_of(unsigned long long count_paused) {
  return static_cast<unsigned>(count_paused >> 48);
}
constexpr unsigned kAuxChainHead = 0x80000000u;  // ring kFAux: parts | chain head | no early
constexpr unsigned kAuxNoEarly = 0x40000000u;
constexpr unsigned kNoEarly = 2u;                 // DevAtom::chain: GPUOS_ATOM_NO_EARLY

struct DevCtl {
  unsigned quit;
  unsigned drain;
  int outstanding;      // ingested, not yet completed
  unsigned pad0;
  unsigned long long deadline;  // globaltimer: hard stop (hang guard)
  unsigned long long blocks, busy_ns, retries, atoms_done;
  unsigned long long stale_claims;  // claims that landed on a recycled slot
  unsigned arrived;                 // worker CTAs that have started
  unsigned pad1;
  unsigned long long t_enter, t_exit;  // first worker entry / last exit (globaltimer)
  unsigned long long t_first_block;    // earliest block start
  unsigned tc_active;                  // TPCs whose tensor cores run a pair tile
  unsigned idle_leaders;               // leaders waiting with nothing eligible
  unsigned fault;                      // first device fault (kFault*; 0: none)
  unsigned pad2;
  unsigned long long fault_info[5];    // raise_fault (gemm_body.cuh): where it was raised
};

// 128-byte submit-ring entry: four 32-byte sectors, each = 7 data words +
// a ticket word. The host stores every sector's data before its ticket, so
// a sector whose ticket matches is internally consistent no matter how the
// device read is split into PCIe requests.
struct RingEntry {
  unsigned w[32];
};
__host__ __device__ constexpr int ring_word(int d) { return (d / 7) * 8 + d % 7; }
enum RingField : int {
  kFOp = 0, kFSlot = 1, kFSeq = 2, kFPrio = 3, kFLo = 4 /*2*/, kFCount = 6,
  kFBody = 7, kFMask0 = 8 /*2*/, kFMask1 = 10 /*2*/, kFPred = 12, kFAux = 13,
  kFArgs = 14 /*10*/, kFTag = 24 /*2*/, kFTrace = 26 /*2*/
};

// 64-byte completion record written by the device into mapped host memory:
// four 16-byte chunks, word 3 of each is the ticket (the atom's sequence).
struct CompRec {
  unsigned w[16];
};

struct Params {
  DevAtom* atoms;
  unsigned long long* resident;  // [tpcs][32]
  unsigned* version;             // [tpcs] bumped when a TPC's candidates change
  int* fence;                    // [tpcs] minimum priority allowed to start
  unsigned* tc_busy;             // [tpcs] pair tiles running on the TPC's tensor cores
  unsigned* pair_seq;            // [tpcs] worker pairs started on the TPC (pair slots)
  DevCtl* ctl;
  const int* phys2log;           // [physical tpcs]
  RingEntry* ring;               // mapped host memory
  CompRec* comp;                 // mapped host memory
  unsigned long long* consumed;  // mapped host memory
  unsigned* alive;               // mapped host memory, one word per worker CTA
  unsigned ring_cap;
  unsigned comp_cap;
  int logical_tpcs;
  int idle_sleep_ns;
  unsigned smem_bytes;  // dynamic shared memory per worker (STREAM / GEMM rings)
  unsigned tmem_cols;   // TMEM columns each worker owns (GEMM accumulator)
  unsigned ingest;      // live mode: cluster 0 runs the ingest warp (0: batch mode)
  unsigned pad0;
  unsigned long long wait_bound_ns;  // bodies' pipeline-wait bound (fault after it)
  unsigned* tpc_occ;                 // [tpcs] blocks running on the TPC (workers +-1)
  unsigned long long* tpc_busy;      // [tpcs] ns with >= 1 running block (ingest's sampler)
};

__device__ __forceinline__ void st_release_gpu64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned long long field64(unsigned lo, unsigned hi) {
  return static_cast<unsigned long long>(lo) | (static_cast<unsigned long long>(hi) << 32);
}

__device__ __forceinline__ bool body_is_pair(unsigned body) {
  return body == GPUOS_BODY_GEMM_BF16 || body == GPUOS_BODY_GEMV_BF16 ||
         body == GPUOS_BODY_CONV_BF16;
}

// ------------------------------------------------------------ ingest warp
// Ring entries are read kIngestBatch at a time: two 512-byte PCIe reads per
// poll (lane l loads 16 B: entry head + l/8, words 4(l%8)..4(l%8)+3), so a
// backlog of submissions costs one host round trip per batch, not per atom.
// Publication uses two GPU-scope fences per batch, not per atom:
//   A  slot fields (claim exhausted), resident-list entry choice, outstanding
//      += 1, pause / fence words                              -- MEMBAR --
//   B  arm claims, insert resident keys                       -- MEMBAR --
//   C  bump the version of every TPC whose candidates changed (release
//      pattern: workers read versions with acquire), drain / quit flags.
// A worker that acquires a key therefore sees the slot fields (A precedes
// the fence before B), and a worker whose acquire of a TPC version observes
// phase C sees every key and armed claim of the batch (no lost wake-up).
constexpr int kIngestBatch = 8;  // two 512-byte reads per poll

struct IngestSubmit {
  unsigned slot, seq;
  unsigned pred;  // chained: predecessor slot + 1 (0: none)
  unsigned early; // chained and armed at once behind a closed gate
  unsigned long long mask[2];
  unsigned long long key;
};

__device__ __forceinline__ uint4 ld_relaxed_sys_v4(const unsigned* p) {
  uint4 r;
  asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ void st_relaxed_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Shared memory of the ingest warp (carved from the dynamic region of the
// ingest cluster's CTA 0, which runs no bodies).
struct IngestShared {
  // Shadow occupancy of every TPC's resident list. Only this warp inserts
  // keys, so an entry whose shadow bit is clear is certainly empty; workers
  // clear entries behind its back, which the shadow learns on refresh.
  unsigned shadow[GPUOS_MAX_TPCS];
  // Entries chosen in the current batch whose keys are not stored yet (a
  // refresh from the list must not hand them out twice). TPC t is only ever
  // touched by lane t % 32, so neither array needs synchronisation.
  unsigned pend[GPUOS_MAX_TPCS];
  IngestSubmit subs[kIngestBatch];
};

// TPC utilisation with the reference's definition (device.cpp:264-275,
// sim.cpp:423-426): the time integral of "TPCs with >= 1 running block".
// Workers add +-1 to tpc_occ[t] around every block (fire-and-forget
// reductions, nothing on their path); the ingest warp samples the counters
// between ring polls (every ~1-2 us, against blocks of 10s of us) and
// integrates per TPC, lane t % 32 owning TPC t.
struct OccSampler {
  unsigned long long busy[(GPUOS_MAX_TPCS + 31) / 32] = {};
  unsigned prev = 0;  // bit i: TPC lane + 32 i was occupied at the last sample
  unsigned long long t_prev = 0;
  __device__ __forceinline__ void sample(const Params& p, unsigned lane) {
    const unsigned long long now = gtimer();
    unsigned cur = 0;
#pragma unroll
    for (int i = 0; i < (GPUOS_MAX_TPCS + 31) / 32; ++i) {
      const int t = static_cast<int>(lane) + 32 * i;
      if (t < p.logical_tpcs) {
        if (((prev >> i) & 1u) && t_prev != 0) busy[i] += now - t_prev;
        if (ld_relaxed_gpu(p.tpc_occ + t) != 0u) cur |= 1u << i;
      }
    }
    prev = cur;
    t_prev = now;
  }
  __device__ __forceinline__ void flush(const Params& p, unsigned lane) {
    sample(p, lane);
#pragma unroll
    for (int i = 0; i < (GPUOS_MAX_TPCS + 31) / 32; ++i) {
      const int t = static_cast<int>(lane) + 32 * i;
      if (t < p.logical_tpcs) p.tpc_busy[t] = busy[i];
    }
  }
};

// The ingest warp: warp 0 of the ingest cluster's CTA 0 (live mode). It is
// part of the worker grid, so the dispatcher is ONE self-contained launch
// (ncu and compute-sanitizer can replay it; nothing depends on two kernels
// being co-resident).
__device__ __forceinline__ void ingest_loop(const Params& p, IngestShared& ish) {
  unsigned* shadow = ish.shadow;
  unsigned* pend = ish.pend;
  IngestSubmit* subs = ish.subs;
  const unsigned lane = threadIdx.x & 31u;
  for (int t = lane; t < GPUOS_MAX_TPCS; t += 32) shadow[t] = pend[t] = 0u;  // lists start empty
  __syncwarp();
  OccSampler occ;
  unsigned long long head = 0;
  unsigned polls = 0;
  for (;;) {
    if ((++polls & 15u) == 1u) {
      if (ld_relaxed_gpu(&p.ctl->quit)) break;
      if (gtimer() > p.ctl->deadline) {
        atomicExch(&p.ctl->quit, 1u);
        break;
      }
    }
    const unsigned el = lane >> 3;  // entry of this lane's 16 bytes (and el + 4)
    const uint4 va = ld_relaxed_sys_v4(p.ring[(head + el) % p.ring_cap].w + 4 * (lane & 7));
    const uint4 vb = ld_relaxed_sys_v4(p.ring[(head + 4 + el) % p.ring_cap].w + 4 * (lane & 7));
    occ.sample(p, lane);  // (its L2 loads overlap the ring's PCIe reads)
    // Sector s of entry e ends with its ticket: word 8s+7 = lane 8e+2s+1, .w
    const bool tka = (lane & 1u) == 0u || va.w == static_cast<unsigned>(head + el + 1);
    const bool tkb = (lane & 1u) == 0u || vb.w == static_cast<unsigned>(head + 4 + el + 1);
    const unsigned long long okm = static_cast<unsigned long long>(__ballot_sync(0xffffffffu, tka)) |
                                   (static_cast<unsigned long long>(__ballot_sync(0xffffffffu, tkb)) << 32);
    int n = 0;
    while (n < kIngestBatch && ((okm >> (8 * n)) & 0xffull) == 0xffull) ++n;
    if (n == 0) {
      __nanosleep(32);
      continue;
    }
    const unsigned long long t_seen = gtimer();
    int n_sub = 0;
    unsigned long long bump0 = 0, bump1 = 0;  // TPCs whose candidate set changed
    bool stop = false, set_drain = false, set_quit = false;
    for (int j = 0; j < n && !stop; ++j) {
      // Transpose: lane l gets word l of entry j.
      const int src = 8 * (j & 3) + static_cast<int>(lane >> 2);
      const uint4 v = j < 4 ? va : vb;
      const unsigned x0 = __shfl_sync(0xffffffffu, v.x, src);
      const unsigned x1 = __shfl_sync(0xffffffffu, v.y, src);
      const unsigned x2 = __shfl_sync(0xffffffffu, v.z, src);
      const unsigned x3 = __shfl_sync(0xffffffffu, v.w, src);
      const unsigned c = lane & 3u;
      const unsigned w = c == 0 ? x0 : c == 1 ? x1 : c == 2 ? x2 : x3;
      auto get = [&](int d) { return __shfl_sync(0xffffffffu, w, ring_word(d)); };
      const unsigned op = get(kFOp);
      if (op == kOpSubmit) {
        const unsigned slot = get(kFSlot);
        const unsigned seq = get(kFSeq);
        const unsigned prio_word = get(kFPrio);  // prio | tenant << 16
        const int prio = static_cast<int>(prio_word & 0xffu);
        const unsigned tenant_bits = prio_word & 0xffff0000u;
        const unsigned long long mask0 = field64(get(kFMask0), get(kFMask0 + 1));
        const unsigned long long mask1 = field64(get(kFMask1), get(kFMask1 + 1));
        unsigned long long args[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) args[k] = field64(get(kFArgs + 2 * k), get(kFArgs + 2 * k + 1));
        const unsigned long long tag = field64(get(kFTag), get(kFTag + 1));
        const unsigned long long trace = field64(get(kFTrace), get(kFTrace + 1));
        const long long lo = static_cast<long long>(field64(get(kFLo), get(kFLo + 1)));
        const unsigned count = get(kFCount);  // slices = blocks x parts
        const unsigned body = get(kFBody);
        const unsigned pred = get(kFPred);
        const unsigned aux = get(kFAux);
        const unsigned parts = aux & ~(kAuxChainHead | kAuxNoEarly);
        DevAtom* a = p.atoms + slot;
        if (lane == 0) {
          // Exhausted (offset == count) until armed in phase B: a stale
          // fetch-add from a worker still holding the previous occupant's
          // key cannot carry into the sequence bits, and arming overwrites it.
          a->claim = (static_cast<unsigned long long>(seq) << 32) | count;
          a->count = count;
          a->paused = 0;  // (the early-start bit is set below)
          a->lo = lo;
          a->body = body;
          a->parts = parts;
#pragma unroll
          for (int k = 0; k < 5; ++k) a->args[k] = args[k];
          a->seq = seq;
          a->prio = prio;
          a->done = 0;
          a->succ = 0;
          a->chain = ((aux & kAuxChainHead) ? kChainHead : 0u) | ((aux & kAuxNoEarly) ? kNoEarly : 0u);
          // Early start: a chained GEMV is armed at once behind a closed gate
          // -- its blocks stream W while the predecessor runs and read x
          // when the predecessor's finisher opens the gate. Only at a
          // priority no higher than the predecessor's, so the
          // predecessor's unclaimed blocks always win a free slot first.
          // The predecessor must be armed already: its unclaimed blocks then
          // win every slot before ours, so our waiting blocks cannot starve
          // it (an unarmed predecessor could find every worker parked at
          // our gate).
          const bool early = pred != 0u && body_is_pair(body) && !(aux & kAuxNoEarly) &&
                             prio <= p.atoms[pred - 1u].prio &&
                             ld_relaxed_gpu(&p.atoms[pred - 1u].armed) != 0u;
          a->paused = tenant_bits | (early ? kGatedBit : 0u);
          a->armed = 0u;
          a->tag = tag;
          a->trace = reinterpret_cast<unsigned*>(trace);
          a->mask[0] = mask0;
          a->mask[1] = mask1;
          a->t_first = ~0ull;
          a->t_last = 0;
          a->touched[0] = 0;
          a->touched[1] = 0;
          a->t_seen = t_seen;
          a->t_armed = 0;
          atomicAdd(&p.ctl->outstanding, 1);  // before any worker can claim
          IngestSubmit& s = subs[n_sub];
          s.slot = slot;
          s.seq = seq;
          s.pred = pred;
          s.early = early ? 1u : 0u;
          s.mask[0] = mask0;
          s.mask[1] = mask1;
          s.key = (static_cast<unsigned long long>(prio & 0xff) << 56) |
                  (static_cast<unsigned long long>(~seq) << 24) | (slot & 0xffffffu);
        }
        // Choose each TPC's resident-list entry now (the finishing worker
        // needs a->entry[] for every TPC), insert the key in phase B.
        for (int t = lane; t < p.logical_tpcs; t += 32) {
          const unsigned long long m = t < 64 ? mask0 : mask1;
          if (!((m >> (t & 63)) & 1ull)) continue;
          const unsigned long long* list = p.resident + static_cast<size_t>(t) * kResident;
          unsigned occ = shadow[t];
          while (occ == ~0u) {  // refresh from the list (host admission keeps room)
            occ = pend[t];
            for (int k = 0; k < kResident; ++k)
              if (ld_relaxed_gpu64(list + k) != 0ull) occ |= 1u << k;
            if (occ == ~0u) __nanosleep(128);
          }
          const int k = __ffs(~occ) - 1;
          shadow[t] = occ | (1u << k);
          pend[t] |= 1u << k;
          a->entry[t] = static_cast<unsigned char>(k);
        }
        bump0 |= mask0;
        bump1 |= mask1;
        ++n_sub;
      } else if (op == kOpPause || op == kOpResume) {
        // Shuffles are warp-collective: read every field before lane-0 work.
        const unsigned slot = get(kFSlot);
        DevAtom* a = p.atoms + slot;
        if (lane == 0) {
          if (op == kOpPause) atomicOr(&a->paused, 1u);
          else atomicAnd(&a->paused, ~1u);
        }
        // Workers drain one atom on a fast path while their TPC's version is
        // unchanged, so pause and resume both bump it.
        // Lane 0 wrote the mask if the atom arrived in this batch: read it
        // there (program order) and broadcast.
        unsigned long long m0 = 0, m1 = 0;
        if (lane == 0) {
          m0 = ld_relaxed_gpu64(&a->mask[0]);
          m1 = ld_relaxed_gpu64(&a->mask[1]);
        }
        bump0 |= __shfl_sync(0xffffffffu, m0, 0);
        bump1 |= __shfl_sync(0xffffffffu, m1, 0);
      } else if (op == kOpFence) {
        const int t = static_cast<int>(get(kFAux));
        const int floor_prio = static_cast<int>(get(kFPrio) & 0xffu);  // (no owner)
        if (t >= 0 && t < p.logical_tpcs) {
          if (lane == 0) atomicExch(p.fence + t, floor_prio);
          if (t < 64) bump0 |= 1ull << t; else bump1 |= 1ull << (t - 64);
        }
      } else if (op == kOpFenceMask) {
        const unsigned long long m0 = field64(get(kFMask0), get(kFMask0 + 1));
        const unsigned long long m1 = field64(get(kFMask1), get(kFMask1 + 1));
        // floor | pair-slot mask << 8 | owner << 16
        const int floor_prio = static_cast<int>((get(kFPrio) & 0xffffu) | (get(kFAux) << 16));
        for (int t = lane; t < p.logical_tpcs; t += 32) {
          const unsigned long long m = t < 64 ? m0 : m1;
          if ((m >> (t & 63)) & 1ull) atomicExch(p.fence + t, floor_prio);
        }
        bump0 |= m0;
        bump1 |= m1;
      } else if (op == kOpDrain) {
        set_drain = true;
        stop = true;
      } else if (op == kOpShutdown) {
        set_quit = true;
        stop = true;
      }
      ++head;
    }
    __syncwarp();
    if (n_sub > 0) {
      fence_acq_rel_gpu();  // every lane: phase A before its phase-B stores
      __syncwarp();
      const unsigned long long t_armed = gtimer();
      bool chained = false;
      for (int i = 0; i < n_sub; ++i) {
        const IngestSubmit s = subs[i];
        DevAtom* a = p.atoms + s.slot;
        if (lane == 0 && (s.pred == 0u || s.early)) {
          st_relaxed_gpu64(&a->claim, static_cast<unsigned long long>(s.seq) << 32);
          a->t_armed = t_armed;
          a->armed = 1u;
        }
        chained = chained || s.pred != 0u;
        for (int t = lane; t < p.logical_tpcs; t += 32) {
          const unsigned long long m = s.mask[t >> 6];
          if ((m >> (t & 63)) & 1ull)
            st_relaxed_gpu64(p.resident + static_cast<size_t>(t) * kResident + a->entry[t], s.key);
        }
      }
      for (int t = lane; t < p.logical_tpcs; t += 32) pend[t] = 0u;
      if (chained) {
        // Keys (and slot fields) before the registration: the finisher that
        // reads it arms the successor and wakes its TPCs.
        __syncwarp();
        fence_acq_rel_gpu();
        if (lane == 0) {
          for (int i = 0; i < n_sub; ++i) {
            const IngestSubmit s = subs[i];
            if (s.pred == 0u) continue;
            DevAtom* a = p.atoms + s.slot;
            if (atomicCAS(&p.atoms[s.pred - 1u].succ, 0u, s.slot + 1u) == kSuccDone) {
              // Predecessor already finished: arm here (woken below), or
              // open an early successor's gate.
              if (s.early) {
                open_gate(&a->paused);
              } else {
                st_relaxed_gpu64(&a->claim, static_cast<unsigned long long>(s.seq) << 32);
                a->t_armed = gtimer();
                a->armed = 1u;
              }
            }
          }
        }
      }
    }
    __syncwarp();
    fence_acq_rel_gpu();  // phase B (and pause / fence words) before the bumps
    for (int t = lane; t < p.logical_tpcs; t += 32) {
      const unsigned long long m = t < 64 ? bump0 : bump1;
      if ((m >> (t & 63)) & 1ull) red_relaxed_gpu_add(p.version + t, 1u);
    }
    if (lane == 0) {
      if (set_drain) atomicExch(&p.ctl->drain, 1u);
      if (set_quit) atomicExch(&p.ctl->quit, 1u);
      // The entries' words are in registers: the host may overwrite them.
      st_relaxed_sys64(p.consumed, head);
    }
    __syncwarp();
    if (stop) break;
  }
  // Drain: keep integrating utilisation until the workers leave.
  for (unsigned k = 0;; ++k) {
    occ.sample(p, lane);
    if ((k & 7u) == 7u &&
        (ld_relaxed_gpu(&p.ctl->quit) ||
         (ld_relaxed_gpu(&p.ctl->drain) && ld_relaxed_gpu_s32(&p.ctl->outstanding) == 0) ||
         gtimer() > p.ctl->deadline))
      break;
    __nanosleep(1000);
  }
  occ.flush(p, lane);
}

// ------------------------------------------------------------ worker CTAs
// Workers run as 2-CTA clusters, one CTA on each SM of a TPC (a 2-CTA
// cluster always lands on SMs {2k, 2k+1}: profiles/topology_probe_r01.json).
// Each CTA arbitrates its TPC's resident atoms and claims blocks on its own,
// so 1-SM bodies (STREAM, SPIN) see 2W independent workers per TPC. A 2-SM
// body (GEMM: one 256 x 256 tile per block on tcgen05.mma.cta_group::2) is
// claimed only by the pair's leader (rank 0), which hands the tile to its
// peer through distributed shared memory (join_rc + join_full mbarrier);
// the peer takes the request at its next decision point (after its current
// block, or at once while idle) and confirms on the leader's `joined`
// mbarrier. A peer whose arbitration winner is a 2-SM atom does not bypass
// it with a lower-priority block: it waits for the leader's request.
struct RoundCmd {
  BlockCmd cmd;                 // block to run: args, block id, body, slice
  long long lo;                 // first block of the atom
  unsigned long long key;       // resident key of the atom
  unsigned slot;
  unsigned count;               // slices of the atom (1: single-block fast path)
  unsigned gated;               // the atom was early-started: its body checks the gate
  unsigned pad;
};
constexpr int kRoundCmdWords64 = sizeof(RoundCmd) / 8;
static_assert(sizeof(RoundCmd) % 8 == 0, "RoundCmd copied as 64-bit words");

// Pair bodies' descriptors start with their two TMA tensor maps (128 B each):
// fetch them into this SM's tensor-map cache ahead of the body's first load.
__device__ __forceinline__ void prefetch_tile_maps(unsigned long long desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
  asm volatile("prefetch.tensormap [%0];" ::"l"(desc + 128) : "memory");
}

enum WorkerGo : int { kGoExit = 0, kGoOwn = 1, kGoPair = 2, kGoJoin = 3 };

// Spreading pair tiles: a leader whose TPC's tensor cores already run a
// pair tile (the other pair of the TPC) waits up to this long before
// claiming another, so a wave with fewer tiles than TPCs lands one tile per
// TPC instead of two sharing one TPC while others idle (measured: a 16-tile
// GEMM on 16 TPCs ran 26 % slower than on 32 without it). In a full wave the
// second pair just starts a little later and overlaps its partner's epilogue.
constexpr unsigned long long kSpreadNs = 4000;

// A pair run (PairTiles, gemm_body.cuh): the leader's claim context for
// GEMM / conv / GEMV tiles claimed inside the body after the run's first tile.
struct PairRun {
  DevAtom* atom;                // atom the run may claim from (null: a single tile)
  unsigned long long key;       // its resident key (sequence for claim_block)
  long long lo;                 // its first block
  unsigned count;               // its slices
  unsigned ver;                 // the TPC's candidate-set version at the first claim
  unsigned extra;               // tiles claimed inside the body (beyond the first)
  unsigned spread;              // GEMM / conv: the spreading rule applies (not GEMV)
  long long next;               // posted next block, -1: end of run (leader writes both CTAs')
  unsigned posts;               // posts so far (leader writes both CTAs', with release: next_block)
};

// A finished atom's bookkeeping held back while its handed-off successor
// runs (account_block / write_done).
struct PendingDone {
  unsigned long long t0, t1, m0, m1, tag, ts, ta;  // t0, m0, m1: single-slice atoms (else read here)
  unsigned slot, tk, n, flags;                     // flags: kPendValid | kPendSingle
};
constexpr unsigned kPendValid = 1u, kPendSingle = 2u;

struct WorkerShared {
  RoundCmd rc;                  // this CTA's block for the round
  PairRun run;                  // pair run state (leader) / posted next tile (both)
  RoundCmd join_rc;             // peer: pair tile posted by the leader
  unsigned long long t_start;
  unsigned long long join_full; // mbarrier (peer): leader posted join_rc
  unsigned long long joined;    // mbarrier (leader): peer took the request
  int go;                       // WorkerGo
  unsigned long long touched_key;  // warp 0: atom whose `touched` word has this TPC
  unsigned tmem_base;           // this worker's TMEM columns (tcgen05.alloc)
  WaitGuard guard;              // the bodies' bounded pipeline waits
  PendingDone pend;             // warp 0: a handed-off predecessor's bookkeeping
  unsigned pair_slot;           // this pair's slot on its TPC (pair fences)
};

// Lane 0 broadcasts a field of sh.rc it wrote itself; the other lanes do
// not touch the shared copy (a volatile load cannot be speculated).
__device__ __forceinline__ unsigned lane0_field(const unsigned& f, unsigned lane) {
  unsigned v = 0u;
  if (lane == 0) v = *static_cast<const volatile unsigned*>(&f);
  return __shfl_sync(0xffffffffu, v, 0);
}

__device__ __forceinline__ unsigned atom_add_acq_rel32(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void ld_relaxed_gpu_v2(const void* p, unsigned long long& a,
                                                  unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Address of this CTA's shared variable `p` in cluster CTA `rank`.
__device__ __forceinline__ unsigned map_rank(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u64(unsigned addr, unsigned long long v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* b, unsigned parity) {
  const unsigned a = smem_u32(b);
  unsigned ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ bool mbar_test_cluster(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
      "selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Lane 0: claim `n` consecutive slices of the atom behind `key` with one
// relaxed fetch-add on its claim word; the slot fields were read by the lane
// that acquired the key and are handed over by shuffle. Fetch-add never
// retries, so 300 workers draining one atom cost one L2 atomic each; the
// CAS loop it replaced spent ~140 failed attempts per claim under that
// contention (profiles/ncu_k_worker_r01_cas.txt). Returns the first slice
// offset (or -1) and in *got how many of the n are valid.
// A worker holding a stale key for a recycled slot (the host recycles slots
// FIFO over the whole table, so this needs a worker stalled for thousands of
// atom lifetimes) sees a foreign sequence in the returned word; valid
// offsets then belong to the slot's new occupant and are run for it
// (stale = true: the caller re-reads the slot), never lost.
__device__ __forceinline__ long long claim_block(DevAtom* a, unsigned long long key,
                                                 unsigned count, unsigned n, DevCtl* ctl,
                                                 bool& stale, unsigned& got) {
  const unsigned seq = ~static_cast<unsigned>(key >> 24);
  const unsigned long long old = atomicAdd(&a->claim, static_cast<unsigned long long>(n));
  const unsigned off = static_cast<unsigned>(old);
  stale = static_cast<unsigned>(old >> 32) != seq;
  if (stale) {
    fence_acq_rel_gpu();
    count = ld_relaxed_gpu(&a->count);
    if (off < count) atomicAdd(&ctl->stale_claims, 1ull);
  }
  // `count` was read with the key's hot line; it never changes while the
  // sequence matches.
  got = off < count ? (count - off < n ? count - off : n) : 0u;
  return got ? static_cast<long long>(off) : -1;
}

// The leader's producer thread, after the last load of a pair tile: claim
// the run's next tile and post it to both CTAs (PairTiles, gemm_body.cuh).
// The run continues only while the TPC's candidate set is unchanged (no new
// atom, fence or pause here since the first claim: otherwise the pair goes
// back to full arbitration, which may pick a higher-priority atom) and, as
// in the arbitration's spreading rule, only if no idle leader elsewhere
// would start the tile sooner (some leader idle and the atom has fewer
// tiles in flight than TPCs). Our own unfinished tile keeps the atom from
// completing, so its slot cannot be recycled under the claim (no stale
// case). A claimed tile is traced here; the run's tiles are counted done
// with the first one (account_block, `extra`).
struct NextTile {
  const Params& p;
  PairRun& run;
  unsigned peer_next;  // shared::cluster address of the peer's run.next
  unsigned peer_posts;  // ... and of its run.posts
  int tpc;
  unsigned sm;
  __device__ __forceinline__ void operator()(bool stop = false) const {
#ifdef GPUOS_NO_PAIR_RUNS
    stop = true;  // diagnostic builds: every pair tile is a run of one
#endif
    long long nb = -1;
    DevAtom* a = run.atom;
    if (!stop && a != nullptr && ld_acquire_gpu(p.version + tpc) == run.ver) {
      bool ok = true;
      if (run.spread && ld_relaxed_gpu(&p.ctl->idle_leaders) != 0u) {
        const unsigned in_flight = static_cast<unsigned>(ld_relaxed_gpu64(&a->claim)) - ld_relaxed_gpu(&a->done);
        const unsigned width = __popcll(ld_relaxed_gpu64(&a->mask[0])) + __popcll(ld_relaxed_gpu64(&a->mask[1]));
        ok = in_flight >= width;
      }
      if (ok) {
        bool stale = false;
        unsigned got = 0;
        const long long off = claim_block(a, run.key, run.count, 1u, p.ctl, stale, got);
        if (off >= 0) {
          nb = run.lo + off;
          ++run.extra;
          if (a->trace != nullptr) atomicAdd(a->trace + nb, 0x10000u + sm + 1u);
        }
      }
    }
    // The post: the block, then the count with release (next_block waits
    // for it with acquire in every thread of both CTAs).
    run.next = nb;
    st_cluster_u64(peer_next, static_cast<unsigned long long>(nb));
    const unsigned posts = run.posts + 1u;
    asm volatile("st.release.cluster.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(&run.posts)), "r"(posts) : "memory");
    asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(peer_posts), "r"(posts) : "memory");
  }
};

// Warp 0 of the CTA that ran `rc`: record the block on its atom and, for the
// atom's last block, publish the completion and retire its resident keys.
// Returns 0 (more blocks to go), 1 (atom done) or 2 (atom done, and `rc`
// now holds block 0 of its chained successor, claimed for this worker).
// A chained successor's hot-line fields (account_block).
struct SuccFields {
  unsigned long long count_paused, lo, body_parts, args[5], seq_prio, mask[2];
  __device__ __forceinline__ void load(const DevAtom* b) {
    unsigned long long claim;
    ld_relaxed_gpu_v2(b, claim, count_paused);
    ld_relaxed_gpu_v2(&b->lo, lo, body_parts);
    ld_relaxed_gpu_v2(&b->args[0], args[0], args[1]);
    ld_relaxed_gpu_v2(&b->args[2], args[2], args[3]);
    ld_relaxed_gpu_v2(&b->args[4], args[4], seq_prio);
    mask[0] = ld_relaxed_gpu64(&b->mask[0]);  // (+104: 8-byte aligned)
    mask[1] = ld_relaxed_gpu64(&b->mask[1]);
  }
};

__device__ __forceinline__ unsigned atom_exch_acq_rel32(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// A finished atom's bookkeeping: completion record, resident-list clears,
// counters. After a handoff it is held back until the successor's block has
// run (the next account_block writes it, after that block's own chain work),
// so the successor starts without waiting for it.

// All lanes of warp 0; `d` (shared memory) was filled by lane 0 before a
// __syncwarp.
__device__ __forceinline__ void write_done(const Params& p, PendingDone& d, unsigned lane) {
  const DevAtom* a = p.atoms + d.slot;
  __syncwarp();  // every lane has read d.slot before lane 0 retires the record (d.flags)
  if (lane == 0) {
    // Completion record (the host is waiting on it), in the slot's own
    // record: four 16-byte chunks, each three data words and the ticket
    // (= seq). Each chunk is one PCIe write, so a chunk whose ticket matches
    // is complete; no system-scope fence (~1 us) sits on the completion path.
    const bool single = (d.flags & kPendSingle) != 0u;
    CompRec* rec = p.comp + d.slot;
    const unsigned long long t0 = single ? d.t0 : ld_relaxed_gpu64(&a->t_first);
    const unsigned long long m0 = single ? d.m0 : ld_relaxed_gpu64(&a->touched[0]);
    const unsigned long long m1 = single ? d.m1 : ld_relaxed_gpu64(&a->touched[1]);
    const unsigned tk = d.tk;
    const unsigned long long span = d.t1 - t0;
    st_relaxed_sys_v4(rec->w + 0, d.n, static_cast<unsigned>(d.tag), static_cast<unsigned>(d.tag >> 32), tk);
    st_relaxed_sys_v4(rec->w + 4, static_cast<unsigned>(t0), static_cast<unsigned>(t0 >> 32),
                      span > 0xffffffffull ? 0xffffffffu : static_cast<unsigned>(span), tk);
    st_relaxed_sys_v4(rec->w + 8, static_cast<unsigned>(m0), static_cast<unsigned>(m0 >> 32),
                      static_cast<unsigned>(m1), tk);
    // t_seen / t_armed as ns before t_first (0 in batch mode).
    st_relaxed_sys_v4(rec->w + 12, static_cast<unsigned>(m1 >> 32),
                      d.ts ? static_cast<unsigned>(t0 - d.ts) : 0u,
                      d.ta ? static_cast<unsigned>(t0 - d.ta) : 0u, tk);
  }
  // Device-side bookkeeping after the record; the host recycles this slot
  // only after thousands of others, long after these land. Our key still
  // occupies its list entries (only this finisher clears them, and the
  // ingest warp fills only cleared entries): plain stores, no round trip.
  for (int t = lane; t < p.logical_tpcs; t += 32) {
    const unsigned long long m = a->mask[t >> 6];
    if ((m >> (t & 63)) & 1ull)
      st_relaxed_gpu64(p.resident + static_cast<size_t>(t) * kResident + a->entry[t], 0ull);
  }
  if (lane == 0) {
    // Plain reductions: atoms_done is read after the kernel ends, and the
    // drain check only needs outstanding to reach zero eventually.
    atomicAdd(&p.ctl->atoms_done, 1ull);
    atomicSub(&p.ctl->outstanding, 1);
    d.flags = 0u;
  }
  __syncwarp();
}

__device__ __forceinline__ void flush_pending(const Params& p, PendingDone& d, unsigned lane) {
  const unsigned f = __shfl_sync(0xffffffffu, lane == 0 ? d.flags : 0u, 0);
  if (f & kPendValid) write_done(p, d, lane);
}

__device__ __forceinline__ int account_block(const Params& p, RoundCmd& rc,
                                             unsigned long long t_start, int tpc, unsigned sm,
                                             unsigned rank, unsigned lane, unsigned extra,
                                             unsigned long long& n_blocks,
                                             unsigned long long& busy,
                                             unsigned long long& touched_key,
                                             PendingDone& pend, unsigned pair_slot) {
  DevAtom* a = p.atoms + rc.slot;
  int last = 0;
  // A single-slice atom is complete with its only block: its first / last
  // times and TPC are this block's, so no atomics on the slot (three L2
  // round trips less on every small kernel).
  const bool single = rc.count == 1u;
  unsigned long long s_t0 = t_start, s_t1 = 0;
  // Fields fixed for the atom's lifetime, read by its finisher (for a
  // single-slice atom up front, overlapping the accounting). A chain head's
  // registered successor is always taken by the swap below (a look-ahead
  // may mark the registration until then).
  unsigned long long tag = 0, ts = 0, ta = 0;
  unsigned chain = 0;
  SuccFields bf;
  auto finisher_fields = [&] {
    tag = a->tag;
    ts = ld_relaxed_gpu64(&a->t_seen);
    ta = ld_relaxed_gpu64(&a->t_armed);
    chain = ld_acquire_gpu(&a->chain);
  };
  if (lane == 0) {
    const unsigned long long t_end = gtimer();
    PROBE_AT(0);
    s_t1 = t_end;
    if (single) finisher_fields();
    if (a->trace != nullptr)
      atomicAdd(a->trace + rc.cmd.block * rc.cmd.parts + rc.cmd.part, 0x10000u + sm + 1u);
    busy += t_end - t_start;
    n_blocks += 1u + extra;
    if (single) {
      // The body's output (and trace) precede the completion record; a
      // chain head fences after arming its successor (off its path).
      if (!(chain & kChainHead)) __threadfence();
      PROBE_AT(1);
      last = 1;
    } else {
      // Per-block records kept off the atom's hot line (every worker of
      // a wide atom claims and counts there, and same-address atomics
      // serialise in their L2 slice: 4.3 us per pair-tile claim with five
      // atomics per block, scratch/gemm_gaps.py): the first slice stamps
      // the start, each worker ORs its TPC into `touched` once per atom,
      // and the last finisher's own clock (after every other block's count)
      // is the end.
      if (rc.cmd.block == rc.lo && rc.cmd.part == 0u) st_relaxed_gpu64(&a->t_first, t_start);
      if (touched_key != rc.key) {
        atomicOr(&a->touched[tpc >> 6], 1ull << (tpc & 63));
        touched_key = rc.key;
      }
      // acq_rel: this block's records (and the body's output stores, ordered
      // by the CTA barrier before this) precede the count; the last finisher
      // observes every other block's records.
      // (A pair run counts its in-body tiles here too: `extra`.)
      last = atom_add_acq_rel32(&a->done, 1u + extra) + 1u + extra == rc.count;
      if (last) {
        s_t1 = gtimer();  // every block has ended (each counted after its end)
        finisher_fields();
      }
    }
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) {
    flush_pending(p, pend, lane);
    return 0;
  }
  // Chain head: arm the registered successor (or mark this atom finished so
  // the ingest warp arms it) before anything else -- the successor's start
  // is the chain's critical path. The swap is acq_rel: our outputs (ordered
  // by the fence / acq_rel count above) precede it, and it acquires the
  // successor's fields and keys (the ingest warp fenced them before
  // registering). When this worker may run the successor here (its TPC is
  // in the set, the fence admits it, and a 2-SM body has this CTA as the
  // pair's leader) the arming store claims block 0 for it: no version
  // wake-up, list scan or claim atomic before the successor's first block
  // (the other workers are woken for the rest).
  RoundCmd ho;
  int handoff = 0;
  unsigned look = 0;  // lane 0: successor's successor armed early (slot + 1)
  unsigned long long look_m0 = 0, look_m1 = 0;  // lane 0: its TPC set
  chain = __shfl_sync(0xffffffffu, chain, 0);
  if (chain & kChainHead) {
    unsigned next = 0;
    if (lane == 0) {
      // Always swapped (never taken from an earlier read): a look-ahead may
      // mark the registration (kSuccLook) until this swap.
      next = atom_exch_acq_rel32(&a->succ, kSuccDone);
      if (next != 0u) PROBE_AT(2);
      const bool look_armed = (next & kSuccLook) != 0u;
      next &= ~kSuccLook;
      // The successor's hot line, this TPC's fence and b's own registered
      // successor are loaded together (one L2 round trip, not four in a
      // row): this chain is the gap between two dependent kernels.
      int floor_prio = 0;
      unsigned cn = 0;
      if (next != 0u) {
        bf.load(p.atoms + (next - 1u));
        floor_prio = ld_relaxed_gpu_s32(p.fence + tpc);
        cn = ld_acquire_gpu(&p.atoms[next - 1u].succ);
      }
      if (next != 0u && (look_armed || ((bf.count_paused >> 32) & kGatedBit))) {
        // Early-started successor (at ingest, or by a look-ahead -- wait for
        // its gated arming to land): our outputs, acquired through the count
        // above, are released to its gate waiters.
        if (look_armed)
          while (ld_acquire_gpu(&p.atoms[next - 1u].armed) == 0u) {
          }
        open_gate(&p.atoms[next - 1u].paused);
        next = 0;
      }
      if (next != 0u) {
        DevAtom* b = p.atoms + (next - 1u);
        const unsigned bseq = static_cast<unsigned>(bf.seq_prio);
        const int bprio = static_cast<int>(bf.seq_prio >> 32);
        const unsigned bcount = static_cast<unsigned>(bf.count_paused);
        const unsigned bbody = static_cast<unsigned>(bf.body_parts);
        const bool here = (((tpc < 64 ? bf.mask[0] : bf.mask[1]) >> (tpc & 63)) & 1ull) && ((bf.count_paused >> 32) & 1ull) == 0u &&
                          fence_admits(floor_prio, bprio, tenant_of(bf.count_paused), pair_slot) &&
                          (!body_is_pair(bbody) || rank == 0u);
        PROBE_AT(3);
        st_relaxed_gpu64(&b->claim, (static_cast<unsigned long long>(bseq) << 32) | (here ? 1u : 0u));
        b->t_armed = gtimer();
        b->armed = 1u;
        // Lookahead: b's own registered successor, if a GEMV that may start
        // early, is armed now behind a closed gate (b opens it). Every field
        // of c this needs is loaded in one round trip (fixed since c's
        // registration, which the acquire of cn ordered before these loads).
        if (cn != 0u && cn != kSuccDone && !(cn & kSuccLook)) {
          DevAtom* c = p.atoms + (cn - 1u);
          unsigned long long c_claim, c_cp, c_lo, c_bp;
          ld_relaxed_gpu_v2(c, c_claim, c_cp);      // claim, count | paused
          ld_relaxed_gpu_v2(&c->lo, c_lo, c_bp);    // lo, body | parts
          const unsigned long long c_sp = ld_relaxed_gpu64(reinterpret_cast<const unsigned long long*>(&c->seq));  // seq | prio
          const unsigned long long c_m0 = ld_relaxed_gpu64(&c->mask[0]);
          const unsigned long long c_m1 = ld_relaxed_gpu64(&c->mask[1]);
          const unsigned long long c_cs = ld_relaxed_gpu64(reinterpret_cast<const unsigned long long*>(&c->chain));  // chain | succ
          const unsigned c_armed = ld_relaxed_gpu(&c->armed);
          // The mark on b's registration decides against b's own finisher:
          // if b already finished (swapped in DONE), it armed c itself.
          if (body_is_pair(static_cast<unsigned>(c_bp)) && !(static_cast<unsigned>(c_cs) & kNoEarly) &&
              static_cast<int>(c_sp >> 32) <= bprio && c_armed == 0u &&
              atomicCAS(&b->succ, cn, cn | kSuccLook) == cn) {
            // Armed claim and closed gate in one 16-byte store: a claimer
            // never sees one without the other.
            const unsigned cpz = (static_cast<unsigned>(c_cp >> 32) & 0xffff0000u) | kGatedBit;  // (tenant kept)
            const unsigned long long cc = (c_cp & 0xffffffffull) | (static_cast<unsigned long long>(cpz) << 32);
            asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(&c->claim),
                         "l"(static_cast<unsigned long long>(static_cast<unsigned>(c_sp)) << 32), "l"(cc)
                         : "memory");
            c->t_armed = gtimer();
            // (release: b's finisher opens the gate only after this arming)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&c->armed), "r"(1u) : "memory");
            look = cn;
            look_m0 = c_m0;
            look_m1 = c_m1;
          }
        }
        PROBE_AT(4);
        if (here) {
          handoff = 1;
#pragma unroll
          for (int k = 0; k < 5; ++k) ho.cmd.args[k] = bf.args[k];
          ho.cmd.body = bbody;
          ho.cmd.parts = static_cast<unsigned>(bf.body_parts >> 32);
          ho.cmd.part = 0;
          ho.lo = static_cast<long long>(bf.lo);
          ho.cmd.block = ho.lo;
          ho.key = (static_cast<unsigned long long>(bprio & 0xff) << 56) |
                   (static_cast<unsigned long long>(~bseq) << 24) | (next - 1u);
          ho.slot = next - 1u;
          ho.count = bcount;
          ho.gated = 0u;  // armed by this finisher: not early
          if (bcount == 1u) next = 0;  // nothing left for other workers: no wake-up
        }
      }
    }
    next = __shfl_sync(0xffffffffu, next, 0);
    handoff = __shfl_sync(0xffffffffu, handoff, 0);
    look = __shfl_sync(0xffffffffu, look, 0);
    if (next != 0u || look != 0u) {
      // The TPC sets to wake (lane 0 loaded them with the fields).
      const unsigned long long m0 = __shfl_sync(0xffffffffu, (next ? bf.mask[0] : 0ull) | look_m0, 0);
      const unsigned long long m1 = __shfl_sync(0xffffffffu, (next ? bf.mask[1] : 0ull) | look_m1, 0);
      fence_acq_rel_gpu();  // every lane: the armed claims before the version bumps
      for (int t = lane; t < p.logical_tpcs; t += 32)
        if ((((t < 64) ? m0 : m1) >> (t & 63)) & 1ull) red_relaxed_gpu_add(p.version + t, 1u);
    }
  }
  // The previous handoff's bookkeeping (its successor -- this block -- is
  // past its own chain work now), then this atom's: written at once, or
  // held back while the successor handed off here runs.
  if (lane == 0) PROBE_AT(5);
  flush_pending(p, pend, lane);
  if (lane == 0) {
    PROBE_AT(6);
    if (single && (chain & kChainHead)) __threadfence();  // outputs before the record
    pend.slot = rc.slot;
    pend.tag = tag;
    pend.ts = ts;
    pend.ta = ta;
    pend.tk = ~static_cast<unsigned>(rc.key >> 24);
    pend.n = rc.count / rc.cmd.parts;
    pend.t0 = s_t0;
    pend.t1 = s_t1;
    pend.m0 = tpc < 64 ? 1ull << tpc : 0ull;
    pend.m1 = tpc >= 64 ? 1ull << (tpc - 64) : 0ull;
    pend.flags = kPendValid | (single ? kPendSingle : 0u);
  }
  __syncwarp();
  if (!handoff) write_done(p, pend, lane);
  if (lane == 0 && handoff) rc = ho;  // (rc's old contents are no longer needed)
  __syncwarp();
  if (lane == 0) PROBE_AT(7);
  return 1 + handoff;
}

__device__ __forceinline__ void run_body(const RoundCmd& rc, int tid, unsigned rank,
                                         StreamPipe& pipe, GemmPipe& gemm, GemvPipe& gemv,
                                         const DevAtom* atoms, PairRun& run, const NextTile& nt,
                                         unsigned& posts_seen) {
  // Only an early-started atom's blocks check its gate (weights first).
  const unsigned* gate = rc.gated ? &atoms[rc.slot].paused : nullptr;
  const PairTiles tiles{&run.next, &run.posts, &posts_seen};
  switch (rc.cmd.body) {
    case GPUOS_BODY_STREAM: body_stream(rc.cmd, tid, pipe); break;
    case GPUOS_BODY_GEMV_BF16: body_gemv2(rc.cmd, tid, rank, gemv, gate, tiles, nt); break;
    case GPUOS_BODY_CONV_BF16: body_conv2(rc.cmd, tid, rank, gemm, gate, tiles, nt); break;
    case GPUOS_BODY_SPIN: body_spin(rc.cmd, tid); break;
    case GPUOS_BODY_GEMM_BF16: body_gemm2(rc.cmd, tid, rank, gemm, gate, tiles, nt); break;
    default:
      if (rc.cmd.body >= GPUOS_BODY_USER0) {
        // A tenant-supplied body (include/gpuos_body.cuh): the prelude's
        // blockIdx recovery from the linear index, then the
        // tenant's code on this CTA's 256 threads and shared tile region.
        const unsigned long long g = rc.cmd.args[4];
        gpuos_block b;
        b.block = rc.cmd.block;
        b.gx = static_cast<unsigned>(g & 0x1fffffull);
        b.gy = static_cast<unsigned>((g >> 21) & 0x1fffffull);
        b.gz = static_cast<unsigned>((g >> 42) & 0x1fffffull);
        if (b.gx == 0u) b.gx = 1u;
        if (b.gy == 0u) b.gy = 1u;
        if (b.gz == 0u) b.gz = 1u;
        const unsigned long long lin = static_cast<unsigned long long>(rc.cmd.block);
        b.x = static_cast<unsigned>(lin % b.gx);
        b.y = static_cast<unsigned>((lin / b.gx) % b.gy);
        b.z = static_cast<unsigned>(lin / (static_cast<unsigned long long>(b.gx) * b.gy));
        b.tid = tid;
        b.part = rc.cmd.part;
        b.parts = rc.cmd.parts;
        b.smem = pipe.tiles;
        b.smem_bytes = pipe.stages * kTile;
        gpuos_user_bodies::run(rc.cmd.body - GPUOS_BODY_USER0, b, rc.cmd.args);
      }
      break;
  }
}

// Workers own TMEM (GEMM accumulators); the hardware co-schedules at most
// two TMEM-using CTAs of this kernel per SM (measured: a W=4 launch leaves
// half the CTAs unlaunched), so W is 1 or 2.
// Register budget: an SM sub-partition holds 16 K registers; with W = 2 it
// hosts two warps of each worker (4 x 32 x R) plus, on one SM, the ingest
// warp (32 x 64). R = 104 keeps that SM able to host both workers: a pair
// that cannot be co-placed there is never launched (measured at R = 103
// with a 122-register ingest warp).
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(104) k_worker(const __grid_constant__ Params p) {
  __shared__ WorkerShared sh;
  extern __shared__ __align__(1024) unsigned char dsmem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const unsigned lane = tid & 31;
  const unsigned rank = cluster_rank();
  unsigned sm = smid();
  int tpc = p.phys2log[sm >> 1];
  // Live mode: cluster 0 is the ingest cluster. Its CTA 0's warp 0 runs the
  // ingest warp for the kernel's lifetime; the TPC it lands on keeps one
  // worker pair (of W) for bodies.
  const bool ingest_cluster = p.ingest != 0u && blockIdx.x < 2u;
  if (tid == 0) {
    atomicMin(&p.ctl->t_enter, gtimer());
    st_release_sys(p.alive + blockIdx.x, (sm + 1) | (tpc < 0 || ingest_cluster ? 0x80000000u : 0u));
    atomicAdd(&p.ctl->arrived, 1u);
  }
  if (tpc < 0 || ingest_cluster) {
    // No bodies here (a TPC not exposed to the scheduler, or the ingest
    // cluster). Give up the TMEM allocation permit at once (an SM does not
    // start a second CTA of a TMEM-using kernel while the first still holds
    // it: measured, every unexposed SM then hosted one worker), then stay
    // until every worker CTA has started: leaving at once would free this SM
    // for a cluster meant for an exposed TPC, leaving that TPC short. Only
    // one thread needs to stay for the CTA to stay resident.
    if (warp == 1) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    if (ingest_cluster && rank == 0 && warp == 0) {
      ingest_loop(p, *reinterpret_cast<IngestShared*>(dsmem));
      return;
    }
    if (tid == 0)
      while (ld_relaxed_gpu(&p.ctl->arrived) < gridDim.x && !ld_relaxed_gpu(&p.ctl->quit) &&
             gtimer() < p.ctl->deadline)
        __nanosleep(1000);
    return;
  }

  StreamPipe pipe;
  stream_pipe_init(pipe, dsmem, p.smem_bytes, tid);
  GemmPipe gemm;
  gemm_pipe_init(gemm, dsmem, p.smem_bytes, p.tmem_cols, tid);
  GemvPipe gemv;
  gemv_pipe_init(gemv, dsmem, p.smem_bytes, p.tmem_cols, tid);
  if (tid == 0) {
    sh.guard = WaitGuard{&p.ctl->fault, &p.ctl->quit, p.wait_bound_ns, p.ctl->fault_info,
                         reinterpret_cast<const unsigned long long*>(&sh.rc)};
    sh.pend.flags = 0u;
    sh.run.posts = 0u;
  }
  gemm.guard = gemv.guard = &sh.guard;
  if (tid == 0) {
    mbar_init(&sh.join_full, 1);
    mbar_init(&sh.joined, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // This pair's slot on its TPC (pair fences): drawn by the leader; the peer
  // reads it from the leader's shared memory after the cluster barrier below
  // (no distributed-shared-memory access before both CTAs have started).
  if (tid == 0 && rank == 0) sh.pair_slot = atomicAdd(p.pair_seq + tpc, 1u);
  // TMEM for the pair's GEMM accumulators: allocated once for the CTA's
  // lifetime by warp 1 of both CTAs (cta_group::2: same columns in both),
  // 512 / W columns so the W workers of an SM never contend.
  if (warp == 1) tmem_alloc2(&sh.tmem_base, p.tmem_cols);
  tc_fence_before();
  __syncthreads();     // (the CTA-level order of the allocation's shared write)
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  gemm.tmem = gemv.tmem = sh.tmem_base;
  unsigned pslot = sh.pair_slot;
  if (rank != 0) {
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(pslot) : "r"(map_rank(&sh.pair_slot, 0)) : "memory");
  }
  unsigned long long n_blocks = 0, busy = 0, retries = 0;
  unsigned long long first_start = ~0ull;
  // Remote addresses inside the pair.
  const unsigned peer_join_rc = map_rank(&sh.join_rc, 1);
  const unsigned peer_join_full = map_rank(&sh.join_full, 1);
  const unsigned leader_joined = map_rank(&sh.joined, 0);
  const unsigned peer_run_next = map_rank(&sh.run.next, 1);
  const unsigned peer_run_posts = map_rank(&sh.run.posts, 1);
  unsigned posts_seen = 0;  // pair-tile posts this thread has consumed (next_block)
  unsigned joins = 0;  // pair tiles this CTA has run (join_full / joined parity)
  // Warp 0's draining state: the atom it last claimed from and the TPC's
  // candidate-set version at that time. While the version is unchanged no
  // higher-priority atom arrived, nothing was paused or fenced, so the next
  // block comes from the same atom without rescanning the resident list.
  unsigned long long cur_key = 0ull;
  unsigned cur_ver = 0u;
  unsigned cur_slot = 0u;
  unsigned cur_count = 0u;
  unsigned cur_body = 0u;
  int cur_tpc = -1;
  unsigned long long spread_since = 0;  // leader: deferring a pair tile since
  bool tc_hold = false;                 // leader thread 0: holds the TPC's tensor reservation
  bool handoff = false;                 // warp 0: sh.rc holds a chained successor's block 0

  for (;;) {
    // %smid can change if the CTA is ever preempted and restored elsewhere;
    // re-derive the TPC whenever it does so placement stays exact (the
    // table load stays off the common path: one L2 round trip per block).
    if (const unsigned now_sm = smid(); now_sm != sm) {
      sm = now_sm;
      tpc = p.phys2log[sm >> 1];
    }
    if (tpc != cur_tpc) {
      cur_key = 0ull;
      if (tid == 0) sh.touched_key = 0ull;
      cur_tpc = tpc;
    }
    if (warp == 0) {
      int go = kGoExit;
      if (handoff) {
        // Block 0 of a chained successor, claimed when its predecessor ended
        // here (account_block); a pair tile takes the tensor reservation.
        handoff = false;
        if (lane == 0) PROBE_AT(8);
        cur_key = 0ull;
        cur_body = lane0_field(sh.rc.cmd.body, lane);
        go = body_is_pair(cur_body) ? kGoPair : kGoOwn;
        if (lane == 0) {
          sh.run.atom = nullptr;  // a single tile: no pair run
          sh.run.extra = 0u;
        }
        if (go == kGoPair && cur_body != GPUOS_BODY_GEMV_BF16 && lane == 0) {
          if (atomicAdd(p.tc_busy + tpc, 1u) == 0u) atomicAdd(&p.ctl->tc_active, 1u);
          tc_hold = true;
        }
      } else if (tpc >= 0) {
        unsigned long long* list = p.resident + static_cast<size_t>(tpc) * kResident;
        unsigned ver = ld_acquire_gpu(p.version + tpc);  // latest observed
        for (;;) {
          // The peer serves a posted pair tile before anything else.
          if (rank != 0 && mbar_test_cluster(&sh.join_full, joins & 1u)) {
            go = kGoJoin;
            break;
          }
          long long off = -1;
          unsigned got = 0;
          unsigned long long key = 0ull;
          bool stale = false;
          // Fast path: next slice of the atom being drained (a GEMV tile
          // only on the leader; GEMM / conv tiles go through the full
          // arbitration, which takes the TPC's tensor-core reservation --
          // keeping it across tiles measured 3 % slower on conv). The
          // version is re-read alongside the claim; a change noticed only
          // after it costs at most one slice of priority inversion.
          const bool fast = cur_key != 0ull && ver == cur_ver &&
                            (!body_is_pair(cur_body) || (rank == 0 && cur_body == GPUOS_BODY_GEMV_BF16));
          if (fast) {
            if (lane == 0)
              off = claim_block(p.atoms + cur_slot, cur_key, cur_count, 1u, p.ctl, stale, got);
            ver = ld_acquire_gpu(p.version + tpc);
            off = __shfl_sync(0xffffffffu, off, 0);
            if (off >= 0) key = cur_key;
            if (stale && lane == 0) sh.rc.key = 0ull;  // slot recycled: reload its fields
          }
          bool defer = false;  // peer: the winner is a 2-SM atom for the leader
          bool nothing = false;  // nothing eligible on this TPC
          if (off < 0) {
            cur_key = 0ull;
            // Full arbitration: eligible = waiting slices, not paused, not
            // fenced off this TPC; highest priority then oldest wins. Each
            // lane reads one key (acquire) and then that atom's hot line, so
            // the winner's fields arrive with the arbitration itself.
            const int floor_prio = ld_relaxed_gpu_s32(p.fence + tpc);
            const unsigned long long k = ld_acquire_gpu64(list + lane);
            bool eligible = false;
            unsigned long long f_lo = 0, f_bp = 0, f_cp = 0, f_cw = 0, f_a[5] = {0, 0, 0, 0, 0};
            if (k != 0ull) {
              const DevAtom* a = p.atoms + (k & 0xffffffull);
              unsigned long long cw, cp;
              ld_relaxed_gpu_v2(a, cw, cp);  // claim | count, paused
              f_cp = cp;
              f_cw = cw;
              ld_relaxed_gpu_v2(&a->lo, f_lo, f_bp);  // lo | body, parts
              ld_relaxed_gpu_v2(&a->args[0], f_a[0], f_a[1]);
              ld_relaxed_gpu_v2(&a->args[2], f_a[2], f_a[3]);
              f_a[4] = ld_relaxed_gpu64(&a->args[4]);
              eligible = static_cast<unsigned>(cw >> 32) == ~static_cast<unsigned>(k >> 24) &&
                         static_cast<unsigned>(cw) < static_cast<unsigned>(cp) &&
                         ((cp >> 32) & 1ull) == 0u &&
                         fence_admits(floor_prio, static_cast<int>(k >> 56), tenant_of(cp), pslot);
            }
            // Candidates of this snapshot, best first: a claim lost to other
            // workers (the atom ran out) moves on to the next candidate
            // without reloading the list (32 small atoms drained by 148
            // pairs otherwise cost ~12 rescans per block: 1397 vs 36 retries
            // measured, tools/gemv_batch.py).
            for (;;) {
              key = warp_max_u64(eligible ? k : 0ull);
              if (key == 0ull) {
                spread_since = 0;  // nothing to defer any more
                nothing = true;
                break;
              }
              // The winner's count and body travel with the arbitration.
              const int win = __ffs(__ballot_sync(0xffffffffu, eligible && k == key)) - 1;
              const unsigned wcount = __shfl_sync(0xffffffffu, static_cast<unsigned>(f_cp), win);
              const unsigned wgated = __shfl_sync(0xffffffffu, static_cast<unsigned>(f_cp >> 32), win) & kGatedBit;
              const unsigned long long wbp = __shfl_sync(0xffffffffu, f_bp, win);
              const bool pair = body_is_pair(static_cast<unsigned>(wbp));
              // GEMV tiles are HBM-bound (their MMAs are a few percent of
              // the tensor cores): both pairs of a TPC stream at once, no
              // reservation or spreading.
              const bool tensor = pair && static_cast<unsigned>(wbp) != GPUOS_BODY_GEMV_BF16;
              // Leader and a pair tile: reserve the TPC's tensor cores. If
              // the other pair holds them, defer up to kSpreadNs so an idle
              // TPC takes the tile first; after that, claim anyway.
              // Deferring only helps while the atom runs fewer tiles than it
              // has TPCs and some leader is idle; in a full wave the second
              // pair claims at once.
              int reserved = 0;
              const unsigned long long wcw = __shfl_sync(0xffffffffu, f_cw, win);
              if (rank == 0 && tensor && lane == 0) {
                const bool expired = spread_since != 0 && gtimer() - spread_since >= kSpreadNs;
                const unsigned before = atomicAdd(p.tc_busy + tpc, 1u);
                reserved = before == 0u || expired ? 1 : 0;
                if (!reserved) {
                  const DevAtom* wa = p.atoms + (key & 0xffffffull);
                  const unsigned in_flight = static_cast<unsigned>(wcw) - ld_relaxed_gpu(&wa->done);
                  const unsigned width = __popcll(ld_relaxed_gpu64(&wa->mask[0])) +
                                         __popcll(ld_relaxed_gpu64(&wa->mask[1]));
                  if (in_flight >= width || ld_relaxed_gpu(&p.ctl->idle_leaders) == 0u)
                    reserved = 1;  // no idle leader would take it sooner
                }
                if (!reserved) atomicSub(p.tc_busy + tpc, 1u);
                else if (before == 0u) atomicAdd(&p.ctl->tc_active, 1u);
              }
              reserved = __shfl_sync(0xffffffffu, reserved, 0);
              if (rank != 0 && pair) {
                defer = true;  // no lower-priority bypass: wait for the leader
                break;
              }
              if (rank == 0 && tensor && !reserved) {
                defer = true;  // let an idle TPC take it first (kSpreadNs)
                if (spread_since == 0) spread_since = gtimer();
                break;
              }
              spread_since = 0;
              if (lane == 0)
                off = claim_block(p.atoms + (key & 0xffffffull), key, wcount, 1u, p.ctl, stale, got);
              off = __shfl_sync(0xffffffffu, off, 0);
              if (off < 0) {
                if (reserved && lane == 0 && atomicSub(p.tc_busy + tpc, 1u) == 1u)
                  atomicSub(&p.ctl->tc_active, 1u);
                ++retries;  // lost that atom's last slices to other workers
                if (eligible && k == key) eligible = false;
                continue;
              }
              // Hand the winner's fields to lane 0 (no second round trip).
              if (lane == 0 && reserved) tc_hold = true;
              cur_count = wcount;
              const unsigned long long wlo = __shfl_sync(0xffffffffu, f_lo, win);
              unsigned long long wa5[5];
#pragma unroll
              for (int k2 = 0; k2 < 5; ++k2) wa5[k2] = __shfl_sync(0xffffffffu, f_a[k2], win);
              if (lane == 0) {
                if (stale) {
                  sh.rc.key = 0ull;  // recycled slot: fields reloaded below
                } else {
#pragma unroll
                  for (int k2 = 0; k2 < 5; ++k2) sh.rc.cmd.args[k2] = wa5[k2];
                  sh.rc.cmd.body = static_cast<unsigned>(wbp);
                  sh.rc.cmd.parts = static_cast<unsigned>(wbp >> 32);
                  sh.rc.lo = static_cast<long long>(wlo);
                  sh.rc.key = key;
                  sh.rc.slot = static_cast<unsigned>(key & 0xffffffull);
                  sh.rc.count = wcount;
                  sh.rc.gated = wgated;
                }
              }
              break;
            }
          }
          if (off >= 0) {
            const unsigned slot = static_cast<unsigned>(key & 0xffffffull);
            if (lane == 0) {
              if (sh.rc.key == 0ull || sh.rc.slot != slot) {
                // Recycled slot adopted by claim_block (which fenced): read the
                // new occupant's fields.
                const DevAtom* a = p.atoms + slot;
#pragma unroll
                for (int k2 = 0; k2 < 5; ++k2) sh.rc.cmd.args[k2] = a->args[k2];
                sh.rc.cmd.body = a->body;
                sh.rc.cmd.parts = a->parts;
                sh.rc.lo = a->lo;
                sh.rc.slot = slot;
                sh.rc.key = key;
                sh.rc.count = ld_relaxed_gpu(&a->count);
                sh.rc.gated = ld_relaxed_gpu(&a->paused) & kGatedBit;
              }
              const unsigned parts = sh.rc.cmd.parts;
              sh.rc.cmd.block = sh.rc.lo + off / parts;
              sh.rc.cmd.part = static_cast<unsigned>(off % parts);
              // Pair tiles (GEMM / conv / GEMV) claimed by a leader start a
              // pair run; GEMV runs skip the spreading rule (HBM-bound: both
              // pairs of a TPC stream at once).
              const unsigned b = sh.rc.cmd.body;
              sh.run.atom = rank == 0 && !stale && body_is_pair(b) ? p.atoms + slot : nullptr;
              sh.run.spread = b != GPUOS_BODY_GEMV_BF16;
              sh.run.key = key;
              sh.run.lo = sh.rc.lo;
              sh.run.count = sh.rc.count;
              sh.run.ver = ver;
              sh.run.extra = 0u;
            }
            cur_key = stale ? 0ull : key;
            cur_slot = slot;
            cur_ver = ver;
            cur_body = lane0_field(sh.rc.cmd.body, lane);  // (lane 0 wrote it)
            spread_since = 0;
            go = body_is_pair(cur_body) ? kGoPair : kGoOwn;
            // A peer reaches a 2-SM block only by adopting a recycled slot
            // (stale claim, see claim_block): it cannot run it alone. A device
            // fault the host's stop reports, not a context-killing trap.
            if (go == kGoPair && rank != 0) {
              if (lane == 0) raise_fault(sh.guard, kFaultAdoptedPair);
              go = kGoExit;
            }
            break;
          }
          // Idle: wait for this TPC's candidate set to change (acquire: a
          // bump observed here makes the batch's keys and claims visible) or,
          // on the peer, for a pair tile. The control block is only consulted
          // when nothing changed, so a wake-up costs one version load.
          // Exit conditions are checked every 8 polls (a drained batch ends
          // within a few microseconds of its last atom). A leader with
          // nothing eligible counts itself idle (pair-tile spreading).
          const bool count_idle = rank == 0 && nothing && lane == 0;
          if (count_idle) atomicAdd(&p.ctl->idle_leaders, 1u);
          bool changed = false, leave = false;
          for (int k2 = 0; k2 < 64; ++k2) {
            // (A suspend-time hint on this wait stretched the peers' exit at
            // drain by ~250 us: the hardware sleeps far past the hint.)
            if (rank != 0 && mbar_test_cluster(&sh.join_full, joins & 1u)) {
              changed = true;
              break;
            }
            const unsigned v = ld_acquire_gpu(p.version + tpc);
            if (v != ver) {
              ver = v;
              changed = true;
              break;
            }
            if ((k2 & 7) == 7) {
              if (spread_since != 0 && gtimer() - spread_since >= kSpreadNs) {
                changed = true;  // spreading wait over: claim now
                break;
              }
              leave = ld_relaxed_gpu(&p.ctl->quit) ||
                      (!defer && ld_relaxed_gpu(&p.ctl->drain) &&
                       ld_relaxed_gpu_s32(&p.ctl->outstanding) == 0) ||
                      gtimer() > p.ctl->deadline;
              if (leave) break;
            }
            __nanosleep(p.idle_sleep_ns);
          }
          if (count_idle) atomicSub(&p.ctl->idle_leaders, 1u);
          if (changed) continue;
          if (leave) break;
        }
      }
      if (lane == 0) {
        if (go == kGoPair) {
          // (the TPC's tensor-core reservation was taken at the claim)
          // Post the tile to the peer (release: the command precedes the
          // arrival), then wait until it has taken it.
          const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&sh.rc);
#pragma unroll
          for (int w = 0; w < kRoundCmdWords64; ++w) st_cluster_u64(peer_join_rc + 8 * w, src[w]);
          mbar_arrive_remote(peer_join_full);
          prefetch_tile_maps(sh.rc.cmd.args[0]);  // while the peer joins
          // The peer takes it at its next decision point; only an abort
          // (quit, hang guard) can leave it untaken.
          for (unsigned polls = 0; !mbar_test_cluster(&sh.joined, joins & 1u); ++polls) {
            if ((polls & 255u) == 255u &&
                (ld_relaxed_gpu(&p.ctl->quit) || gtimer() > p.ctl->deadline)) {
              go = kGoExit;
              break;
            }
          }
        } else if (go == kGoJoin) {
          sh.rc = sh.join_rc;
          mbar_arrive_remote(leader_joined);
          prefetch_tile_maps(sh.rc.cmd.args[0]);
        }
        sh.go = go;
        sh.t_start = gtimer();
#ifdef GPUOS_PROBE_HANDOFF
        if (g_probe_cur[blockIdx.x][8] != 0ull) {
          PROBE_AT(9);
          const unsigned r = atomicAdd(&g_probe_n, 1u) & 4095u;
          for (int i = 0; i < kProbeStamps; ++i) {
            g_probe_ring[r][i] = g_probe_cur[blockIdx.x][i];
            g_probe_cur[blockIdx.x][i] = 0ull;
          }
        }
#endif
        if (go != kGoExit) {
          if (first_start == ~0ull) first_start = sh.t_start;
          red_relaxed_gpu_add(p.tpc_occ + tpc, 1u);  // utilisation sampler (OccSampler)
        }
      }
    }
    __syncthreads();
    const int go = sh.go;
    if (go == kGoExit) break;
    {
      const NextTile nt{p, sh.run, peer_run_next, peer_run_posts, tpc, sm};
      run_body(sh.rc, tid, rank, pipe, gemm, gemv, p.atoms, sh.run, nt, posts_seen);  // pair tiles end with a cluster barrier
    }
    if (go == kGoPair || go == kGoJoin) ++joins;
    if (tc_hold && tid == 0) {
      if (atomicSub(p.tc_busy + tpc, 1u) == 1u) atomicSub(&p.ctl->tc_active, 1u);
      tc_hold = false;
    }
    __syncthreads();
    if (tid == 0) PROBE_AT(10);
    if (tid == 0) red_relaxed_gpu_add(p.tpc_occ + tpc, ~0u);  // -1: the block has ended
    // The leader records pair tiles (the peer's half is complete: cluster
    // barrier at the end of the body).
    if (warp == 0 && go != kGoJoin) {
      const unsigned extra = go == kGoPair ? lane0_field(sh.run.extra, lane) : 0u;
      const int done = account_block(p, sh.rc, sh.t_start, tpc, sm, rank, lane, extra, n_blocks, busy,
                                     sh.touched_key, sh.pend, pslot);
      if (done) cur_key = 0ull;  // the atom is done: rescan rather than claim from it
      handoff = done == 2;
      __syncwarp();  // every lane has read sh.t_start / sh.rc before lane 0 rewrites them
    }
  }
  if (warp == 0) flush_pending(p, sh.pend, lane);  // (a handoff always runs its block first: none left)
  if (tid == 0) {
    atomicAdd(&p.ctl->blocks, n_blocks);
    atomicAdd(&p.ctl->busy_ns, busy);
    atomicAdd(&p.ctl->retries, retries);
    if (first_start != ~0ull) atomicMin(&p.ctl->t_first_block, first_start);
  }
  tc_fence_before();
  cluster_sync_all();  // neither CTA frees TMEM or leaves while the other may still use it
  if (warp == 1) tmem_free2(gemm.tmem, p.tmem_cols);
  if (tid == 0) atomicMax(&p.ctl->t_exit, gtimer());
}

__global__ void k_gtimer(unsigned long long* out) { *out = gtimer(); }

#ifdef GPUOS_PROBE_HANDOFF
extern "C" int gpuos_dev_probe_read(unsigned long long* out, unsigned* n) {
  if (cudaMemcpyFromSymbol(n, g_probe_n, sizeof(unsigned)) != cudaSuccess) return -1;
  return cudaMemcpyFromSymbol(out, g_probe_ring, sizeof(g_probe_ring)) == cudaSuccess ? 0 : -1;
}
#endif

// Packed GEMV weights (kGemvPacked): rows of 64 bf16; packed row
// ((h nk + j) 128 + i) = W row 128 h + i, columns 64 j .. 64 j + 63, zero
// beyond N or K.
__host__ __device__ inline long long gemv_packed_rows(long long n, long long k) {
  return (n + kGemmHalf - 1) / kGemmHalf * ((k + kGemmBK - 1) / kGemmBK) * kGemmHalf;
}
__global__ void k_gemv_pack(unsigned short* dst, const unsigned short* src, long long n, long long k,
                            long long total) {
  const long long nk = (k + kGemmBK - 1) / kGemmBK;
  for (long long e = blockIdx.x * 256ll + threadIdx.x; e < total; e += gridDim.x * 256ll) {
    const long long prow = e / kGemmBK, c = e % kGemmBK;
    const long long i = prow % kGemmHalf, hj = prow / kGemmHalf;
    const long long h = hj / nk, j = hj % nk;
    const long long row = h * kGemmHalf + i, col = j * kGemmBK + c;
    dst[e] = row < n && col < k ? src[row * k + col] : static_cast<unsigned short>(0);
  }
}

// Uniform [-1, 1) bf16 fill from a counter hash (tenant operand init).
__global__ void k_fill_bf16(unsigned short* p, unsigned long long n, unsigned long long seed) {
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
    unsigned long long x = seed + i * 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    const float u = static_cast<float>(x >> 40) * (2.0f / 16777216.0f) - 1.0f;
    const __nv_bfloat16 b = __float2bfloat16_rn(u);
    p[i] = *reinterpret_cast<const unsigned short*>(&b);
  }
}

}  // namespace gpuos_dev_impl

// ====================================================================== host
using namespace gpuos_dev_impl;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                        \
  do {                                                                        \
    cudaError_t e_ = (expr);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return fail(GPUOS_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int64_t steady_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct HostAtom {
  uint32_t atom_id = 0;
  uint32_t blocks = 0;
  uint32_t seq = 0;
  int64_t submit_ns = 0;
  uint64_t mask[2] = {0, 0};
  bool live = false;
  bool chain_head = false;   // submitted with GPUOS_ATOM_CHAIN_HEAD
  bool has_succ = false;     // a successor is chained behind it
  uint32_t pred_slot = 0;    // chained: predecessor's slot and sequence
  uint32_t pred_seq = 0;     // (0: not chained)
  uint64_t succ_ring = 0;    // ring entries the device must have consumed before
                             // this slot may be reused (its successor's entry
                             // registers on it by slot number)
};

}  // namespace

struct gpuos_dev {
  gpuos_dev_config cfg{};
  gpuos_dev_topology topo{};
  int device = 0;
  cudaStream_t s_work = nullptr, s_side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  // device tables
  DevAtom* atoms = nullptr;
  unsigned long long* resident = nullptr;
  unsigned* version = nullptr;
  int* fence = nullptr;
  unsigned* tc_busy = nullptr;
  unsigned* pair_seq = nullptr;
  DevCtl* ctl = nullptr;
  int* phys2log = nullptr;
  unsigned long long* gt_scratch = nullptr;
  unsigned* tpc_occ = nullptr;              // [T] running blocks (utilisation sampler)
  unsigned long long* tpc_busy = nullptr;   // [T] sampled busy ns
  // The dispatcher kernel is launched from this thread: under a profiler
  // that serialises launches (ncu) the launch call blocks until the kernel
  // ends, and the kernel only ends once this handle's owner has fed the
  // ring and drained it.
  std::thread launcher;
  std::atomic<int> launch_rc{0};            // 0 pending, 1 launched, < 0 failed
  std::string launch_error;
  // mapped host memory
  RingEntry* ring_h = nullptr;
  RingEntry* ring_d = nullptr;
  CompRec* comp_h = nullptr;
  CompRec* comp_d = nullptr;
  unsigned long long* consumed_h = nullptr;
  unsigned long long* consumed_d = nullptr;
  unsigned* alive_h = nullptr;
  unsigned* alive_d = nullptr;
  int grid = 0;
  // host bookkeeping
  uint64_t ring_head = 0;  // next ring index to publish
  std::vector<uint32_t> live;  // slots of atoms in flight (completion scan)
  uint32_t next_seq = 1;
  uint32_t next_atom_id = 0;
  std::deque<uint32_t> free_slots;  // FIFO: a freed slot is reused last
  // Completed chain heads whose successor's ring entry the device has not
  // consumed yet: (ring entries that must be consumed, slot).
  std::deque<std::pair<uint64_t, uint32_t>> deferred_free;
  int64_t exit_check_ns = 0;        // poll(): last check that the kernel still runs
  std::vector<HostAtom> slots;
  std::unordered_map<uint32_t, uint32_t> slot_of;  // live atom id -> slot
  std::vector<int> tpc_resident;  // keys currently resident per logical TPC
  int32_t in_flight = 0;
  bool running = false;
  bool workers_launched = false;
  bool calibrated = false;
  Params params{};
  int64_t t0_ns = 0;        // host origin
  int64_t gt_offset = 0;    // device globaltimer - host origin-relative ns
  float last_elapsed_ms = 0.f;
  gpuos_dev_stats stats{};
};

namespace {

int publish(gpuos_dev* d, const uint32_t* data /*28 words*/) {
  // Back-pressure: never overwrite an entry the device has not consumed.
  const int64_t deadline = steady_ns() + 10'000'000'000LL;
  while (d->ring_head - __atomic_load_n(d->consumed_h, __ATOMIC_ACQUIRE) >=
         static_cast<uint64_t>(d->cfg.ring_entries)) {
    if (!d->running || !d->workers_launched)
      return fail(GPUOS_E_FULL, "submit ring full and dispatcher not running");
    if (steady_ns() > deadline) return fail(GPUOS_E_TIMEOUT, "submit ring stalled");
  }
  RingEntry* e = d->ring_h + (d->ring_head % d->cfg.ring_entries);
  const uint32_t ticket = static_cast<uint32_t>(d->ring_head + 1);
  volatile uint32_t* w = e->w;
  for (int sector = 0; sector < 4; ++sector) {
    for (int k = 0; k < 7; ++k) w[sector * 8 + k] = data[sector * 7 + k];
    __atomic_store_n(const_cast<uint32_t*>(&w[sector * 8 + 7]), ticket, __ATOMIC_RELEASE);
  }
  ++d->ring_head;
  return GPUOS_OK;
}

void put64(uint32_t* data, int field, uint64_t v) {
  data[field] = static_cast<uint32_t>(v);
  data[field + 1] = static_cast<uint32_t>(v >> 32);
}

int map_priority(int32_t p) { return std::clamp(p, 0, 254) + 1; }

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The driver's tensor-map encoder, through the runtime (no libcuda link).
EncodeTiledFn tensor_map_encoder() {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  return encode;
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

EncodeIm2colFn im2col_map_encoder() {
  static EncodeIm2colFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<EncodeIm2colFn>(fn);
  }
  return encode;
}

void record_spans(gpuos_dev* d, const DevCtl& c) {
  const bool ok = c.t_enter != ~0ull && c.t_exit >= c.t_enter;
  d->stats.worker_span_ns = ok ? static_cast<int64_t>(c.t_exit - c.t_enter) : 0;
  d->stats.first_block_ns =
      ok && c.t_first_block != ~0ull ? static_cast<int64_t>(c.t_first_block - c.t_enter) : 0;
}

unsigned tmem_cols_for(int workers_per_sm);

Params make_params(gpuos_dev* d, bool ingest) {
  Params p{};
  p.atoms = d->atoms;
  p.resident = d->resident;
  p.version = d->version;
  p.fence = d->fence;
  p.tc_busy = d->tc_busy;
  p.pair_seq = d->pair_seq;
  p.ctl = d->ctl;
  p.phys2log = d->phys2log;
  p.ring = d->ring_d;
  p.comp = d->comp_d;
  p.consumed = d->consumed_d;
  p.alive = d->alive_d;
  p.ring_cap = static_cast<unsigned>(d->cfg.ring_entries);
  p.comp_cap = static_cast<unsigned>(d->cfg.atom_slots);
  p.logical_tpcs = d->cfg.logical_tpcs;
  p.idle_sleep_ns = d->cfg.idle_sleep_ns;
  p.smem_bytes = static_cast<unsigned>(d->topo.smem_per_worker);
  p.tmem_cols = tmem_cols_for(d->cfg.workers_per_sm);
  p.ingest = ingest ? 1u : 0u;
  p.wait_bound_ns = static_cast<unsigned long long>(d->cfg.pipeline_timeout_ms) * 1000000ull;
  p.tpc_occ = d->tpc_occ;
  p.tpc_busy = d->tpc_busy;
  return p;
}

// Kernel-exit bookkeeping shared by stop() and run_batch(): counters,
// spans, the sampled TPC-busy integral and the device fault word.
int collect_run(gpuos_dev* d, float ms, DevCtl& ctl) {
  CUDA_TRY(cudaMemcpy(&ctl, d->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost));
  std::vector<unsigned long long> busy(static_cast<size_t>(d->cfg.logical_tpcs), 0ull);
  CUDA_TRY(cudaMemcpy(busy.data(), d->tpc_busy, sizeof(unsigned long long) * busy.size(),
                      cudaMemcpyDeviceToHost));
  d->stats.blocks_executed += ctl.blocks;
  d->stats.worker_busy_ns += ctl.busy_ns;
  d->stats.claim_retries += ctl.retries;
  d->stats.kernel_elapsed_ns = static_cast<int64_t>(ms * 1e6);
  for (unsigned long long b : busy) d->stats.tpc_busy_ns += b;
  d->stats.fault = ctl.fault;
  record_spans(d, ctl);
  return GPUOS_OK;
}

const char* fault_name(unsigned f) {
  return f == kFaultPipeline      ? "a tensor-core pipeline wait expired (pipeline_timeout_ms)"
         : f == kFaultAdoptedPair ? "a 2-SM block was claimed by a pair's second CTA (recycled atom slot)"
                                  : "unknown fault";
}

// The fault and where the device raised it (DevCtl::fault_info).
std::string fault_text(const DevCtl& c) {
  char where[256];
  std::snprintf(where, sizeof where,
                " [sm %u rank %u thread %u, barrier smem+0x%x parity %u, block %lld of desc 0x%llx, body %u slice %u]",
                static_cast<unsigned>(c.fault_info[0] & 0xffffu), static_cast<unsigned>((c.fault_info[0] >> 16) & 0xffffu),
                static_cast<unsigned>(c.fault_info[0] >> 32), static_cast<unsigned>(c.fault_info[1] & 0xffffffffu),
                static_cast<unsigned>(c.fault_info[1] >> 32), static_cast<long long>(c.fault_info[3]),
                static_cast<unsigned long long>(c.fault_info[2]), static_cast<unsigned>(c.fault_info[4] & 0xffffffffu),
                static_cast<unsigned>(c.fault_info[4] >> 32));
  return std::string(fault_name(c.fault)) + where;
}

// UMMA N for a pair tile over `cols` output columns: 64, 128 or 256.
unsigned narrow_tile(int64_t cols) { return cols <= 64 ? 64u : cols <= 128 ? 128u : kGemmTile; }

// TMEM columns per worker: the largest power of two <= 512 / W (>= 32).
unsigned tmem_cols_for(int workers_per_sm) {
  unsigned c = 512;
  while (c > 32 && c * static_cast<unsigned>(workers_per_sm) > 512) c >>= 1;
  return c;
}

bool known_body(uint32_t b) {
  return b == GPUOS_BODY_STREAM || b == GPUOS_BODY_SPIN || b == GPUOS_BODY_GEMM_BF16 ||
         b == GPUOS_BODY_GEMV_BF16 || b == GPUOS_BODY_CONV_BF16 ||
         (b >= GPUOS_BODY_USER0 && b - GPUOS_BODY_USER0 < gpuos_user_bodies::kCount);
}

// Argument checks the device bodies rely on (empty string: valid).
std::string body_args_error(const gpuos_atom_desc& a) {
  if (a.body == GPUOS_BODY_GEMV_BF16 || a.body == GPUOS_BODY_GEMM_BF16 ||
      a.body == GPUOS_BODY_CONV_BF16) {
    if (a.args[0] == 0 || a.args[0] % 128 != 0) return "tensor-core bodies take a descriptor in args[0]";
    if ((a.parts == 0 ? 1u : a.parts) != 1u) return "tensor-core tiles cannot be sliced";
  }
  return {};
}

}  // namespace

extern "C" {

const char* gpuos_dev_last_error(void) { return g_last_error.c_str(); }

int gpuos_dev_body_id(const char* name, uint32_t* id) {
  if (!name || !id) return fail(GPUOS_E_CONFIG, "null argument");
  for (unsigned i = 0; i < gpuos_user_bodies::kCount; ++i)
    if (std::strcmp(gpuos_user_bodies::kNames[i], name) == 0) {
      *id = GPUOS_BODY_USER0 + i;
      return GPUOS_OK;
    }
  return fail(GPUOS_E_CONFIG, std::string("no tenant body named ") + name + " in this library");
}

int gpuos_dev_open(const gpuos_dev_config* cfg_in, gpuos_dev** out) {
  if (out == nullptr) return fail(GPUOS_E_CONFIG, "null out pointer");
  *out = nullptr;
  gpuos_dev_config cfg{};
  if (cfg_in) cfg = *cfg_in;
  if (cfg.workers_per_sm <= 0) cfg.workers_per_sm = 2;
  if (cfg.atom_slots <= 0) cfg.atom_slots = 4096;
  if (cfg.ring_entries <= 0) cfg.ring_entries = 4096;
  if (cfg.idle_sleep_ns <= 0) cfg.idle_sleep_ns = 128;
  if (cfg.pipeline_timeout_ms <= 0) {
    // (GPUOS_PIPELINE_TIMEOUT_MS: longer bounds for runs under sanitizers)
    const char* env = std::getenv("GPUOS_PIPELINE_TIMEOUT_MS");
    cfg.pipeline_timeout_ms = env != nullptr && std::atoi(env) > 0 ? std::atoi(env) : 2000;
  }
  if (cfg.workers_per_sm > 2)
    return fail(GPUOS_E_CONFIG, "workers_per_sm must be 1 or 2 (TMEM-owning workers per SM)");
  if (cfg.atom_slots > (1 << 24)) return fail(GPUOS_E_CONFIG, "atom_slots must be < 2^24");

  auto d = std::make_unique<gpuos_dev>();
  d->cfg = cfg;
  d->device = cfg.device_ordinal;
  CUDA_TRY(cudaSetDevice(d->device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, d->device));
  if (prop.major != 10)
    return fail(GPUOS_E_CONFIG, std::string("sm_100a dispatcher needs a Blackwell B200, found ") + prop.name);
  const int phys_tpcs = prop.multiProcessorCount / 2;
  if (cfg.logical_tpcs <= 0) cfg.logical_tpcs = std::min(phys_tpcs, GPUOS_MAX_TPCS);
  if (cfg.logical_tpcs > phys_tpcs || cfg.logical_tpcs > GPUOS_MAX_TPCS)
    return fail(GPUOS_E_CONFIG, "logical_tpcs exceeds the physical TPC count");
  d->cfg = cfg;

  // Size each worker's shared memory so that exactly W workers fit per SM.
  const int smem_sm = static_cast<int>(prop.sharedMemPerMultiprocessor);
  // Headroom for the per-CTA reserved shared memory (a cluster-launched
  // pair needs more slack than the arithmetic suggests: measured with the
  // former separate ingest kernel, 8 KB places every pair).
  int smem_worker = std::min<int>(static_cast<int>(prop.sharedMemPerBlockOptin) - 2048,
                                  smem_sm / cfg.workers_per_sm - 8192);
  smem_worker = std::max(smem_worker - smem_worker % 1024, 0);
  if (cfg.workers_per_sm > 1) {
    // W+1 workers must not fit.
    while ((cfg.workers_per_sm + 1) * (smem_worker + 1024) <= smem_sm) smem_worker += 1024;
  }
  d->topo.sm_count = prop.multiProcessorCount;
  d->topo.physical_tpcs = phys_tpcs;
  d->topo.logical_tpcs = cfg.logical_tpcs;
  d->topo.workers_per_sm = cfg.workers_per_sm;
  d->topo.workers_per_tpc = 2 * cfg.workers_per_sm;
  d->topo.threads_per_worker = kWorkerThreads;
  d->topo.smem_per_worker = smem_worker;
  d->grid = prop.multiProcessorCount * cfg.workers_per_sm;

  CUDA_TRY(cudaFuncSetAttribute(k_worker, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_worker));
  // Max shared carveout: operand init kernels that run beside the resident
  // dispatcher ask for the same one (csrc/tools/residency_probe.cu).
  CUDA_TRY(cudaFuncSetAttribute(k_worker, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_worker, kWorkerThreads, smem_worker));
  // The occupancy calculator reports 1 CTA/SM for any kernel that uses
  // tcgen05.alloc (it cannot see how many TMEM columns a CTA takes); two
  // workers with 256 columns each do co-reside (measured), and
  // launch_workers() verifies the real placement: exactly W per SM.
  if (per_sm > cfg.workers_per_sm)
    return fail(GPUOS_E_CONFIG, "worker occupancy is " + std::to_string(per_sm) +
                                    " CTAs/SM, expected " + std::to_string(cfg.workers_per_sm));

  CUDA_TRY(cudaStreamCreateWithFlags(&d->s_work, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&d->s_side, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreate(&d->ev_start));
  CUDA_TRY(cudaEventCreate(&d->ev_stop));

  const size_t T = static_cast<size_t>(cfg.logical_tpcs);
  CUDA_TRY(cudaMalloc(&d->atoms, sizeof(DevAtom) * cfg.atom_slots));
  CUDA_TRY(cudaMemset(d->atoms, 0, sizeof(DevAtom) * cfg.atom_slots));
  CUDA_TRY(cudaMalloc(&d->resident, sizeof(unsigned long long) * T * kResident));
  CUDA_TRY(cudaMalloc(&d->version, sizeof(unsigned) * T));
  CUDA_TRY(cudaMalloc(&d->fence, sizeof(int) * T));
  CUDA_TRY(cudaMalloc(&d->tc_busy, sizeof(unsigned) * T));
  CUDA_TRY(cudaMalloc(&d->pair_seq, sizeof(unsigned) * T));
  CUDA_TRY(cudaMalloc(&d->ctl, sizeof(DevCtl)));
  CUDA_TRY(cudaMalloc(&d->phys2log, sizeof(int) * phys_tpcs));
  CUDA_TRY(cudaMalloc(&d->gt_scratch, sizeof(unsigned long long)));
  CUDA_TRY(cudaMalloc(&d->tpc_occ, sizeof(unsigned) * T));
  CUDA_TRY(cudaMalloc(&d->tpc_busy, sizeof(unsigned long long) * T));
  CUDA_TRY(cudaMemset(d->tpc_occ, 0, sizeof(unsigned) * T));
  CUDA_TRY(cudaMemset(d->tpc_busy, 0, sizeof(unsigned long long) * T));
  std::vector<int> p2l(phys_tpcs, -1);
  for (int t = 0; t < cfg.logical_tpcs; ++t) p2l[t] = t;
  CUDA_TRY(cudaMemcpy(d->phys2log, p2l.data(), sizeof(int) * phys_tpcs, cudaMemcpyHostToDevice));

  CUDA_TRY(cudaHostAlloc(&d->ring_h, sizeof(RingEntry) * cfg.ring_entries, cudaHostAllocMapped));
  CUDA_TRY(cudaHostAlloc(&d->comp_h, sizeof(CompRec) * cfg.atom_slots, cudaHostAllocMapped));
  CUDA_TRY(cudaHostAlloc(&d->consumed_h, 128, cudaHostAllocMapped));
  CUDA_TRY(cudaHostAlloc(&d->alive_h, sizeof(unsigned) * d->grid, cudaHostAllocMapped));
  CUDA_TRY(cudaHostGetDevicePointer(&d->ring_d, d->ring_h, 0));
  CUDA_TRY(cudaHostGetDevicePointer(&d->comp_d, d->comp_h, 0));
  CUDA_TRY(cudaHostGetDevicePointer(&d->consumed_d, d->consumed_h, 0));
  CUDA_TRY(cudaHostGetDevicePointer(&d->alive_d, d->alive_h, 0));

  d->slots.assign(cfg.atom_slots, HostAtom{});
  for (int s = cfg.atom_slots - 1; s >= 0; --s) d->free_slots.push_back(static_cast<uint32_t>(s));
  d->tpc_resident.assign(T, 0);
  d->t0_ns = steady_ns();
  *out = d.release();
  return GPUOS_OK;
}

int gpuos_dev_close(gpuos_dev* d) {
  if (d == nullptr) return GPUOS_OK;
  if (d->running) {
    float ms = 0;
    gpuos_dev_stop(d, 0, &ms);
  }
  if (d->launcher.joinable()) d->launcher.join();
  cudaFree(d->atoms);
  cudaFree(d->resident);
  cudaFree(d->version);
  cudaFree(d->fence);
  cudaFree(d->tc_busy);
  cudaFree(d->pair_seq);
  cudaFree(d->ctl);
  cudaFree(d->phys2log);
  cudaFree(d->gt_scratch);
  cudaFree(d->tpc_occ);
  cudaFree(d->tpc_busy);
  cudaFreeHost(d->ring_h);
  cudaFreeHost(d->comp_h);
  cudaFreeHost(d->consumed_h);
  cudaFreeHost(d->alive_h);
  if (d->ev_start) cudaEventDestroy(d->ev_start);
  if (d->ev_stop) cudaEventDestroy(d->ev_stop);
  if (d->s_work) cudaStreamDestroy(d->s_work);
  if (d->s_side) cudaStreamDestroy(d->s_side);
  delete d;
  return GPUOS_OK;
}

int gpuos_dev_get_topology(gpuos_dev* d, gpuos_dev_topology* out) {
  if (!d || !out) return fail(GPUOS_E_CONFIG, "null argument");
  *out = d->topo;
  return GPUOS_OK;
}

int64_t gpuos_dev_now_ns(gpuos_dev* d) { return d ? steady_ns() - d->t0_ns : 0; }
int32_t gpuos_dev_in_flight(gpuos_dev* d) { return d ? d->in_flight : 0; }

int gpuos_dev_debug_dump(gpuos_dev* d, char* buf, int32_t len) {
  if (!d || !buf || len <= 0) return fail(GPUOS_E_CONFIG, "null argument");
  std::string out;
  char line[320];
  std::snprintf(line, sizeof(line), "in_flight %d, ring published %llu consumed %llu\n", d->in_flight,
                static_cast<unsigned long long>(d->ring_head),
                static_cast<unsigned long long>(__atomic_load_n(d->consumed_h, __ATOMIC_ACQUIRE)));
  out += line;
  int shown = 0;
  for (const uint32_t slot : d->live) {
    if (shown++ == 24) {
      out += "...\n";
      break;
    }
    DevAtom a{};
    // (side stream: a copy engine read while the persistent kernel runs)
    if (cudaMemcpyAsync(&a, d->atoms + slot, 128, cudaMemcpyDeviceToHost, d->s_side) != cudaSuccess ||
        cudaMemcpyAsync(&a.armed, &d->atoms[slot].armed, 4, cudaMemcpyDeviceToHost, d->s_side) != cudaSuccess ||
        cudaStreamSynchronize(d->s_side) != cudaSuccess)
      return fail(GPUOS_E_CUDA, "debug dump copy");
    const HostAtom& h = d->slots[slot];
    std::snprintf(line, sizeof(line),
                  "atom %u slot %u seq %u body %u prio %d count %u claimed %u done %u paused 0x%x armed %u "
                  "chain %u succ 0x%x pred_slot %u tpcs %d\n",
                  h.atom_id, slot, a.seq, a.body, a.prio, a.count, static_cast<unsigned>(a.claim), a.done,
                  a.paused, a.armed, a.chain, a.succ, h.pred_seq ? h.pred_slot : 0u,
                  __builtin_popcountll(a.mask[0]) + __builtin_popcountll(a.mask[1]));
    out += line;
  }
  std::snprintf(buf, static_cast<size_t>(len), "%s", out.c_str());
  return static_cast<int32_t>(out.size());
}

int gpuos_dev_start(gpuos_dev* d) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  if (d->running) return fail(GPUOS_E_STATE, "dispatcher already running");
  if (d->in_flight != 0) return fail(GPUOS_E_STATE, "atoms still in flight");
  if (d->cfg.workers_per_sm != 2)
    return fail(GPUOS_E_CONFIG, "live mode needs workers_per_sm = 2: cluster 0 hosts the ingest warp "
                                "and its TPC keeps the other worker pair (W = 1 runs batch mode only)");
  CUDA_TRY(cudaSetDevice(d->device));
  const size_t T = static_cast<size_t>(d->cfg.logical_tpcs);
  CUDA_TRY(cudaMemset(d->resident, 0, sizeof(unsigned long long) * T * kResident));
  CUDA_TRY(cudaMemset(d->version, 0, sizeof(unsigned) * T));
  CUDA_TRY(cudaMemset(d->fence, 0, sizeof(int) * T));
  CUDA_TRY(cudaMemset(d->tc_busy, 0, sizeof(unsigned) * T));
  CUDA_TRY(cudaMemset(d->pair_seq, 0, sizeof(unsigned) * T));
  CUDA_TRY(cudaMemset(d->tpc_occ, 0, sizeof(unsigned) * T));
  CUDA_TRY(cudaMemset(d->tpc_busy, 0, sizeof(unsigned long long) * T));
  std::memset(d->ring_h, 0, sizeof(RingEntry) * d->cfg.ring_entries);
  std::memset(d->comp_h, 0, sizeof(CompRec) * d->cfg.atom_slots);
  std::memset(d->alive_h, 0, sizeof(unsigned) * d->grid);
  *d->consumed_h = 0;
  d->ring_head = 0;
  d->live.clear();
  d->slot_of.clear();
  for (const auto& f : d->deferred_free) d->free_slots.push_back(f.second);
  d->deferred_free.clear();
  std::fill(d->tpc_resident.begin(), d->tpc_resident.end(), 0);

  // Calibrate device globaltimer against the host origin (+- half an RTT),
  // once per handle: later runs launch nothing but the dispatcher itself.
  if (!d->calibrated) {
    int64_t best_rtt = INT64_MAX;
    for (int i = 0; i < 5; ++i) {
      const int64_t h0 = gpuos_dev_now_ns(d);
      k_gtimer<<<1, 1, 0, d->s_work>>>(d->gt_scratch);
      unsigned long long g = 0;
      CUDA_TRY(cudaMemcpyAsync(&g, d->gt_scratch, 8, cudaMemcpyDeviceToHost, d->s_work));
      CUDA_TRY(cudaStreamSynchronize(d->s_work));
      const int64_t h1 = gpuos_dev_now_ns(d);
      if (h1 - h0 < best_rtt) {
        best_rtt = h1 - h0;
        d->gt_offset = static_cast<int64_t>(g) - (h0 + h1) / 2;
      }
    }
    d->calibrated = true;
  }
  DevCtl ctl{};
  ctl.t_enter = ctl.t_first_block = ~0ull;
  // Hang guard: every dispatcher kernel exits 30 min after start regardless.
  ctl.deadline = static_cast<unsigned long long>(d->gt_offset + gpuos_dev_now_ns(d)) +
                 1800ull * 1000000000ull;
  CUDA_TRY(cudaMemcpyAsync(d->ctl, &ctl, sizeof(DevCtl), cudaMemcpyHostToDevice, d->s_side));
  CUDA_TRY(cudaStreamSynchronize(d->s_side));

  d->params = make_params(d, true);
  d->running = true;
  d->workers_launched = false;
  if (d->cfg.flags & GPUOS_DEV_DEFER_WORKERS) return GPUOS_OK;
  return gpuos_dev_launch_workers(d);
}

int gpuos_dev_launch_workers(gpuos_dev* d) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  if (!d->running || d->workers_launched) return fail(GPUOS_E_STATE, "dispatcher not launchable now");
  if (d->launcher.joinable()) d->launcher.join();
  d->launch_rc.store(0);
  d->launch_error.clear();
  d->workers_launched = true;
  d->exit_check_ns = 0;
  // One launch, from a helper thread (see gpuos_dev::launcher). Its events
  // bracket the kernel on the work stream.
  d->launcher = std::thread([d] {
    cudaError_t e = cudaSetDevice(d->device);
    if (e == cudaSuccess) e = cudaEventRecord(d->ev_start, d->s_work);
    if (e == cudaSuccess) {
      k_worker<<<d->grid, kWorkerThreads, d->topo.smem_per_worker, d->s_work>>>(d->params);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(d->ev_stop, d->s_work);
    if (e != cudaSuccess) {
      d->launch_error = std::string("dispatcher launch: ") + cudaGetErrorString(e);
      d->launch_rc.store(-1, std::memory_order_release);
    } else {
      d->launch_rc.store(1, std::memory_order_release);
    }
  });

  // Every worker CTA must be resident, W per SM, 2W per logical TPC.
  const int64_t deadline = steady_ns() + 5'000'000'000LL;
  for (;;) {
    if (d->launch_rc.load(std::memory_order_acquire) < 0) {
      d->launcher.join();
      d->running = false;
      return fail(GPUOS_E_CUDA, d->launch_error);
    }
    int ready = 0;
    for (int i = 0; i < d->grid; ++i)
      ready += __atomic_load_n(d->alive_h + i, __ATOMIC_ACQUIRE) != 0u;
    if (ready == d->grid) break;
    if (steady_ns() > deadline) {
      std::vector<int> per_sm(d->topo.sm_count, 0);
      std::string missing;
      for (int i = 0; i < d->grid; ++i) {
        const unsigned v = __atomic_load_n(d->alive_h + i, __ATOMIC_ACQUIRE);
        if (v == 0u) missing += " cta" + std::to_string(i);
        else if ((v & 0x7fffffffu) - 1u < per_sm.size()) ++per_sm[(v & 0x7fffffffu) - 1u];
      }
      std::string sms;
      for (int s = 0; s < d->topo.sm_count; ++s)
        if (per_sm[s] != d->cfg.workers_per_sm)
          sms += " sm" + std::to_string(s) + "=" + std::to_string(per_sm[s]);
      gpuos_dev_stop(d, 0, nullptr);
      return fail(GPUOS_E_TIMEOUT, "only " + std::to_string(ready) + " of " +
                                       std::to_string(d->grid) +
                                       " worker CTAs became resident; missing:" + missing +
                                       "; short SMs:" + sms);
    }
  }
  std::vector<int> per_sm(d->topo.sm_count, 0);
  for (int i = 0; i < d->grid; ++i) {
    const unsigned sm = (d->alive_h[i] & 0x7fffffffu) - 1u;
    if (sm < per_sm.size()) ++per_sm[sm];
  }
  for (int s = 0; s < d->topo.sm_count; ++s)
    if (per_sm[s] != d->cfg.workers_per_sm) {
      std::string detail;
      for (int i = 0; i < d->grid; ++i) {
        const unsigned smi = (d->alive_h[i] & 0x7fffffffu) - 1u;
        if (static_cast<int>(smi) == s || per_sm[smi] != d->cfg.workers_per_sm)
          detail += " cta" + std::to_string(i) + "@sm" + std::to_string(smi);
      }
      gpuos_dev_stop(d, 0, nullptr);
      return fail(GPUOS_E_INVARIANT, "SM " + std::to_string(s) + " hosts " +
                                         std::to_string(per_sm[s]) + " workers (W=" +
                                         std::to_string(d->cfg.workers_per_sm) + "):" + detail);
    }
  return GPUOS_OK;
}

int gpuos_dev_consumed(gpuos_dev* d, uint64_t* consumed, uint64_t* published) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  if (consumed) *consumed = __atomic_load_n(d->consumed_h, __ATOMIC_ACQUIRE);
  if (published) *published = d->ring_head;
  return GPUOS_OK;
}

int gpuos_dev_stop(gpuos_dev* d, int drain, float* elapsed_ms) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  if (!d->running) return fail(GPUOS_E_STATE, "dispatcher not running");
  if (!d->workers_launched) {
    // Deferred dispatcher never launched: run it now so the drain completes.
    if (drain) {
      const int lrc = gpuos_dev_launch_workers(d);
      if (lrc != GPUOS_OK) return lrc;
    } else {
      d->running = false;
      d->last_elapsed_ms = 0.f;
      if (elapsed_ms) *elapsed_ms = 0.f;
      return GPUOS_OK;
    }
  }
  uint32_t data[28] = {};
  data[kFOp] = drain ? kOpDrain : kOpShutdown;
  int rc = publish(d, data);
  if (rc != GPUOS_OK) drain = 0;
  if (!drain) {
    // Abort path: also raise the quit flag directly through the side stream,
    // so workers stop even if the ingest warp is stuck.
    static const unsigned one = 1;
    cudaMemcpyAsync(&d->ctl->quit, &one, sizeof one, cudaMemcpyHostToDevice, d->s_side);
    cudaStreamSynchronize(d->s_side);
  }
  // Completions keep arriving while draining; the caller polls them after.
  const int64_t deadline = steady_ns() + (drain ? 300'000'000'000LL : 30'000'000'000LL);
  while (d->launch_rc.load(std::memory_order_acquire) == 0 ||
         cudaStreamQuery(d->s_work) == cudaErrorNotReady) {
    if (steady_ns() > deadline) {
      if (drain) {
        static const unsigned one = 1;
        cudaMemcpyAsync(&d->ctl->quit, &one, sizeof one, cudaMemcpyHostToDevice, d->s_side);
        cudaStreamSynchronize(d->s_side);
        drain = 0;
        continue;
      }
      return fail(GPUOS_E_TIMEOUT, "dispatcher did not stop");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  d->launcher.join();
  d->running = false;
  if (d->launch_rc.load() < 0) return fail(GPUOS_E_CUDA, d->launch_error);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(d->s_work));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, d->ev_start, d->ev_stop));
  d->last_elapsed_ms = ms;
  if (elapsed_ms) *elapsed_ms = ms;
  DevCtl ctl{};
  if (const int crc = collect_run(d, ms, ctl); crc != GPUOS_OK) return crc;
  d->stats.ingest_entries += static_cast<int64_t>(*d->consumed_h);
  if (ctl.fault != 0u)
    return fail(GPUOS_E_TIMEOUT, std::string("device fault: ") + fault_text(ctl));
  if (drain && ctl.outstanding != 0)
    return fail(GPUOS_E_INVARIANT, "drained with atoms outstanding");
  return GPUOS_OK;
}

// Batch mode: the host stages a whole set of atoms straight into the device
// tables (exactly the state the ingest warp would build), then launches the
// worker kernel alone with the drain flag raised. The kernel exits when the
// last atom completes, so its CUDA-event time is pure execution, and it is a
// single self-contained launch that ncu can replay.
int gpuos_dev_run_batch(gpuos_dev* d, const gpuos_atom_desc* descs, int32_t n, float* elapsed_ms) {
  if (!d || (!descs && n > 0)) return fail(GPUOS_E_CONFIG, "null argument");
  if (d->running) return fail(GPUOS_E_STATE, "dispatcher running");
  if (d->in_flight != 0) return fail(GPUOS_E_STATE, "atoms still in flight");
  if (n < 1 || n > d->cfg.atom_slots) return fail(GPUOS_E_FULL, "batch larger than the atom table");
  CUDA_TRY(cudaSetDevice(d->device));
  const int T = d->cfg.logical_tpcs;
  std::vector<DevAtom> atoms(static_cast<size_t>(n));
  std::vector<unsigned long long> resident(static_cast<size_t>(T) * kResident, 0ull);
  std::vector<int> fill(static_cast<size_t>(T), 0);
  std::vector<uint32_t> ids(static_cast<size_t>(n));
  std::vector<uint32_t> seqs(static_cast<size_t>(n));
  std::vector<int> pred(static_cast<size_t>(n), -1);  // chained: predecessor index
  const uint32_t id_base = d->next_atom_id;
  for (int i = 0; i < n; ++i) {
    const gpuos_atom_desc& a = descs[i];
    if (a.flags & ~(GPUOS_ATOM_CHAIN_HEAD | GPUOS_ATOM_NO_EARLY)) return fail(GPUOS_E_CONFIG, "unknown atom flags");
    if (a.tenant > 0xffffu) return fail(GPUOS_E_CONFIG, "tenant must be < 65536");
    if (a.after != 0) {
      // Only atoms of this batch exist: the predecessor is an earlier entry.
      const int64_t j = static_cast<int64_t>(a.after - 1u) - static_cast<int64_t>(id_base);
      if (j < 0 || j >= i) return fail(GPUOS_E_CONFIG, "predecessor must be an earlier atom of the batch");
      if (!(descs[j].flags & GPUOS_ATOM_CHAIN_HEAD))
        return fail(GPUOS_E_CONFIG, "predecessor was not submitted as a chain head");
      if (atoms[static_cast<size_t>(j)].succ != 0u)
        return fail(GPUOS_E_CONFIG, "predecessor already has a successor");
      pred[static_cast<size_t>(i)] = static_cast<int>(j);
    }
    const uint32_t parts = a.parts == 0 ? 1u : a.parts;
    if (a.lo < 0 || a.hi <= a.lo || (a.hi - a.lo) * static_cast<int64_t>(parts) > 0xfffffffeLL)
      return fail(GPUOS_E_CONFIG, "atom block range out of bounds");
    if (!known_body(a.body)) return fail(GPUOS_E_CONFIG, "unknown body kind");
    if (const std::string e = body_args_error(a); !e.empty()) return fail(GPUOS_E_CONFIG, e);
    const uint32_t seq = d->next_seq++;
    seqs[static_cast<size_t>(i)] = seq;
    const int prio = map_priority(a.priority);
    DevAtom& x = atoms[static_cast<size_t>(i)];
    std::memset(&x, 0, sizeof x);
    x.claim = static_cast<unsigned long long>(seq) << 32;
    x.count = static_cast<unsigned>((a.hi - a.lo) * parts);
    x.parts = parts;
    x.seq = seq;
    x.prio = prio;
    x.paused = a.tenant << 16;
    x.body = a.body;
    x.lo = a.lo;
    ids[static_cast<size_t>(i)] = d->next_atom_id++;
    x.chain = ((a.flags & GPUOS_ATOM_CHAIN_HEAD) ? kChainHead : 0u) |
              ((a.flags & GPUOS_ATOM_NO_EARLY) ? kNoEarly : 0u);
    x.armed = pred[static_cast<size_t>(i)] >= 0 ? 0u : 1u;
    if (pred[static_cast<size_t>(i)] >= 0) {
      x.claim |= x.count;  // unarmed until the predecessor's last block
      atoms[static_cast<size_t>(pred[static_cast<size_t>(i)])].succ = static_cast<unsigned>(i) + 1u;
    }
    std::memcpy(x.args, a.args, sizeof x.args);
    x.tag = a.tag;
    x.trace = a.trace;
    x.mask[0] = a.tpc_mask[0];
    x.mask[1] = a.tpc_mask[1];
    x.t_first = ~0ull;
    const unsigned long long key = (static_cast<unsigned long long>(prio & 0xff) << 56) |
                                   (static_cast<unsigned long long>(~seq) << 24) |
                                   static_cast<unsigned long long>(i);
    bool any = false;
    for (int t = 0; t < GPUOS_MAX_TPCS; ++t) {
      if (!((a.tpc_mask[t >> 6] >> (t & 63)) & 1ull)) continue;
      if (t >= T) return fail(GPUOS_E_CONFIG, "TPC id out of range");
      if (fill[t] >= kResident) return fail(GPUOS_E_FULL, "more than 32 atoms on one TPC");
      x.entry[t] = static_cast<unsigned char>(fill[t]);
      resident[static_cast<size_t>(t) * kResident + fill[t]++] = key;
      any = true;
    }
    if (!any) return fail(GPUOS_E_CONFIG, "atom needs a non-empty TPC set");
  }
  // Host bookkeeping: slots 0..n-1 in flight, completions consumed by poll().
  d->free_slots.clear();
  d->deferred_free.clear();
  for (int s = d->cfg.atom_slots - 1; s >= n; --s) d->free_slots.push_back(static_cast<uint32_t>(s));
  const int64_t now = gpuos_dev_now_ns(d);
  d->slot_of.clear();
  for (int i = 0; i < n; ++i) {
    HostAtom& h = d->slots[static_cast<size_t>(i)];
    h.atom_id = ids[static_cast<size_t>(i)];
    h.blocks = static_cast<uint32_t>(descs[i].hi - descs[i].lo);
    h.seq = seqs[static_cast<size_t>(i)];
    h.submit_ns = now;
    h.mask[0] = descs[i].tpc_mask[0];
    h.mask[1] = descs[i].tpc_mask[1];
    h.live = true;
    h.chain_head = (descs[i].flags & GPUOS_ATOM_CHAIN_HEAD) != 0;
    h.has_succ = atoms[static_cast<size_t>(i)].succ != 0u;
    const int j = pred[static_cast<size_t>(i)];
    h.pred_slot = j >= 0 ? static_cast<uint32_t>(j) : 0u;
    h.pred_seq = j >= 0 ? seqs[static_cast<size_t>(j)] : 0u;
    d->slot_of[h.atom_id] = static_cast<uint32_t>(i);
  }
  std::fill(d->tpc_resident.begin(), d->tpc_resident.end(), 0);
  std::memset(d->comp_h, 0, sizeof(CompRec) * d->cfg.atom_slots);
  std::memset(d->alive_h, 0, sizeof(unsigned) * d->grid);
  d->live.clear();
  for (int i = 0; i < n; ++i) d->live.push_back(static_cast<uint32_t>(i));
  d->in_flight = n;

  CUDA_TRY(cudaMemcpy(d->atoms, atoms.data(), sizeof(DevAtom) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d->resident, resident.data(), sizeof(unsigned long long) * resident.size(),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemset(d->version, 0, sizeof(unsigned) * T));
  CUDA_TRY(cudaMemset(d->fence, 0, sizeof(int) * T));
  CUDA_TRY(cudaMemset(d->tc_busy, 0, sizeof(unsigned) * T));
  CUDA_TRY(cudaMemset(d->pair_seq, 0, sizeof(unsigned) * T));
  DevCtl ctl{};
  ctl.t_enter = ctl.t_first_block = ~0ull;
  ctl.drain = 1;
  ctl.outstanding = n;
  ctl.deadline = ~0ull >> 1;
  CUDA_TRY(cudaMemcpy(d->ctl, &ctl, sizeof ctl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemset(d->tpc_occ, 0, sizeof(unsigned) * T));
  CUDA_TRY(cudaMemset(d->tpc_busy, 0, sizeof(unsigned long long) * T));

  const Params p = make_params(d, false);  // every cluster works; no ring
  CUDA_TRY(cudaEventRecord(d->ev_start, d->s_work));
  k_worker<<<d->grid, kWorkerThreads, d->topo.smem_per_worker, d->s_work>>>(p);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(d->ev_stop, d->s_work));
  CUDA_TRY(cudaStreamSynchronize(d->s_work));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, d->ev_start, d->ev_stop));
  if (elapsed_ms) *elapsed_ms = ms;
  d->last_elapsed_ms = ms;
  DevCtl after{};
  if (const int crc = collect_run(d, ms, after); crc != GPUOS_OK) return crc;
  if (after.fault != 0u)
    return fail(GPUOS_E_TIMEOUT, std::string("device fault: ") + fault_text(after));
  if (after.outstanding != 0) return fail(GPUOS_E_INVARIANT, "batch finished with atoms outstanding");
  return GPUOS_OK;
}

int gpuos_dev_submit_atom(gpuos_dev* d, const gpuos_atom_desc* a, uint32_t* atom_id) {
  if (!d || !a) return fail(GPUOS_E_CONFIG, "null argument");
  if (!d->running) return fail(GPUOS_E_STATE, "dispatcher not running");
  if (a->lo < 0 || a->hi <= a->lo) return fail(GPUOS_E_CONFIG, "atom block range out of bounds");
  const uint32_t parts = a->parts == 0 ? 1u : a->parts;
  if (parts > 4096) return fail(GPUOS_E_CONFIG, "parts must be <= 4096");
  if ((a->hi - a->lo) * static_cast<int64_t>(parts) > 0xfffffffeLL)
    return fail(GPUOS_E_CONFIG, "atom too large");
  if (!known_body(a->body)) return fail(GPUOS_E_CONFIG, "unknown body kind");
  if (const std::string e = body_args_error(*a); !e.empty()) return fail(GPUOS_E_CONFIG, e);
  const int T = d->cfg.logical_tpcs;
  bool any = false;
  for (int w = 0; w < 2; ++w) {
    const uint64_t m = a->tpc_mask[w];
    if (m == 0) continue;
    any = true;
    const int top = 64 * w + 63 - __builtin_clzll(m);
    if (top >= T) return fail(GPUOS_E_CONFIG, "TPC id out of range");
  }
  if (!any) return fail(GPUOS_E_CONFIG, "atom needs a non-empty TPC set");
  for (int t = 0; t < T; ++t)
    if (((a->tpc_mask[t >> 6] >> (t & 63)) & 1ull) && d->tpc_resident[t] >= kResident)
      return fail(GPUOS_E_FULL, "TPC " + std::to_string(t) + " already holds 32 resident atoms");
  if (!d->deferred_free.empty()) {
    const uint64_t consumed = __atomic_load_n(d->consumed_h, __ATOMIC_ACQUIRE);
    while (!d->deferred_free.empty() && d->deferred_free.front().first <= consumed) {
      d->free_slots.push_back(d->deferred_free.front().second);
      d->deferred_free.pop_front();
    }
  }
  if (d->free_slots.empty()) return fail(GPUOS_E_FULL, "atom table full");
  if (a->flags & ~(GPUOS_ATOM_CHAIN_HEAD | GPUOS_ATOM_NO_EARLY))
    return fail(GPUOS_E_CONFIG, "unknown atom flags");
  if (a->tenant > 0xffffu) return fail(GPUOS_E_CONFIG, "tenant must be < 65536");
  // Chaining: a live predecessor (not yet polled) arms this atom on the
  // device; one that already completed leaves nothing to wait for.
  uint32_t pred_slot = 0, pred_seq = 0;
  bool chained = false;
  if (a->after != 0) {
    const auto it = d->slot_of.find(a->after - 1u);
    if (it != d->slot_of.end()) {
      HostAtom& p = d->slots[it->second];
      if (!p.chain_head) return fail(GPUOS_E_CONFIG, "predecessor was not submitted as a chain head");
      if (p.has_succ) return fail(GPUOS_E_CONFIG, "predecessor already has a successor");
      pred_slot = it->second;
      pred_seq = p.seq;
      chained = true;
    } else if (a->after - 1u >= d->next_atom_id) {
      return fail(GPUOS_E_CONFIG, "predecessor atom id was never issued");
    }
  }

  const uint32_t slot = d->free_slots.front();
  d->free_slots.pop_front();
  const uint32_t id = d->next_atom_id++;
  const uint32_t seq = d->next_seq++;
  uint32_t data[28] = {};
  data[kFOp] = kOpSubmit;
  data[kFSlot] = slot;
  data[kFSeq] = seq;
  data[kFPrio] = static_cast<uint32_t>(map_priority(a->priority)) | (a->tenant << 16);
  put64(data, kFLo, static_cast<uint64_t>(a->lo));
  data[kFCount] = static_cast<uint32_t>((a->hi - a->lo) * parts);
  data[kFAux] = parts | ((a->flags & GPUOS_ATOM_CHAIN_HEAD) ? kAuxChainHead : 0u) |
                ((a->flags & GPUOS_ATOM_NO_EARLY) ? kAuxNoEarly : 0u);
  data[kFBody] = a->body;
  put64(data, kFMask0, a->tpc_mask[0]);
  put64(data, kFMask1, a->tpc_mask[1]);
  data[kFPred] = chained ? pred_slot + 1u : 0u;
  for (int k = 0; k < 5; ++k) put64(data, kFArgs + 2 * k, a->args[k]);
  put64(data, kFTag, a->tag);
  put64(data, kFTrace, reinterpret_cast<uint64_t>(a->trace));
  HostAtom& h = d->slots[slot];
  h.atom_id = id;
  h.blocks = static_cast<uint32_t>(a->hi - a->lo);
  h.seq = seq;
  h.submit_ns = gpuos_dev_now_ns(d);
  h.mask[0] = a->tpc_mask[0];
  h.mask[1] = a->tpc_mask[1];
  h.live = true;
  h.chain_head = (a->flags & GPUOS_ATOM_CHAIN_HEAD) != 0;
  h.has_succ = false;
  h.pred_slot = pred_slot;
  h.pred_seq = pred_seq;
  h.succ_ring = 0;
  const int rc = publish(d, data);
  if (rc != GPUOS_OK) {
    h.live = false;
    d->free_slots.push_front(slot);
    return rc;
  }
  if (chained) {
    // The device registers this atom on the predecessor's slot when it
    // ingests this entry: the slot must not be recycled before that.
    d->slots[pred_slot].has_succ = true;
    d->slots[pred_slot].succ_ring = d->ring_head;
  }
  d->slot_of[id] = slot;
  for (int t = 0; t < T; ++t)
    if ((a->tpc_mask[t >> 6] >> (t & 63)) & 1ull) ++d->tpc_resident[t];
  d->live.push_back(slot);
  ++d->in_flight;
  if (atom_id) *atom_id = id;
  return GPUOS_OK;
}

int gpuos_dev_set_atom_paused(gpuos_dev* d, uint32_t atom_id, int paused) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  const auto it = d->slot_of.find(atom_id);
  if (it == d->slot_of.end()) return GPUOS_OK;  // already finished: nothing to pause (device.cpp:167)
  uint32_t data[28] = {};
  data[kFOp] = paused ? kOpPause : kOpResume;
  data[kFSlot] = it->second;
  return publish(d, data);  // already finished: nothing to pause (device.cpp:167)
}

int gpuos_dev_set_tpc_fence(gpuos_dev* d, int32_t tpc, int32_t min_priority) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  if (tpc < 0 || tpc >= d->cfg.logical_tpcs) return fail(GPUOS_E_CONFIG, "TPC id out of range");
  uint32_t data[28] = {};
  data[kFOp] = kOpFence;
  data[kFAux] = static_cast<uint32_t>(tpc);
  data[kFPrio] = min_priority <= 0 ? 0u : static_cast<uint32_t>(map_priority(min_priority));
  return publish(d, data);
}

int gpuos_dev_set_fence_mask(gpuos_dev* d, const uint64_t mask[2], int32_t min_priority) {
  if (!d || !mask) return fail(GPUOS_E_CONFIG, "null argument");
  uint32_t data[28] = {};
  data[kFOp] = kOpFenceMask;
  put64(data, kFMask0, mask[0]);
  put64(data, kFMask1, mask[1]);
  data[kFPrio] = min_priority <= 0 ? 0u : static_cast<uint32_t>(map_priority(min_priority));
  return publish(d, data);
}

int gpuos_dev_set_pair_fence(gpuos_dev* d, const uint64_t mask[2], uint32_t pair_slots, int32_t min_priority) {
  if (!d || !mask) return fail(GPUOS_E_CONFIG, "null argument");
  if (pair_slots > 0xffu) return fail(GPUOS_E_CONFIG, "pair_slots is an 8-bit mask");
  uint32_t data[28] = {};
  data[kFOp] = kOpFenceMask;
  put64(data, kFMask0, mask[0]);
  put64(data, kFMask1, mask[1]);
  data[kFPrio] = (min_priority <= 0 ? 0u : static_cast<uint32_t>(map_priority(min_priority))) | (pair_slots << 8);
  return publish(d, data);
}

int gpuos_dev_set_tpc_owner(gpuos_dev* d, const uint64_t mask[2], uint32_t owner, int32_t min_priority) {
  if (!d || !mask) return fail(GPUOS_E_CONFIG, "null argument");
  if (owner > 0xffffu) return fail(GPUOS_E_CONFIG, "owner must be < 65536");
  uint32_t data[28] = {};
  data[kFOp] = kOpFenceMask;
  put64(data, kFMask0, mask[0]);
  put64(data, kFMask1, mask[1]);
  data[kFPrio] = min_priority <= 0 ? 0u : static_cast<uint32_t>(map_priority(min_priority));
  data[kFAux] = owner;
  return publish(d, data);
}

int gpuos_dev_poll(gpuos_dev* d, gpuos_completion* out, int32_t max) {
  if (!d || (!out && max > 0)) return fail(GPUOS_E_CONFIG, "null argument");
  int n = 0;
  // Each in-flight atom owns the completion record of its slot; its ticket
  // is the atom's sequence number once the device has published it.
  for (std::size_t i = 0; i < d->live.size() && n < max;) {
    const uint32_t slot = d->live[i];
    HostAtom& h = d->slots[slot];
    CompRec* rec = d->comp_h + slot;
    if (h.pred_seq != 0 && d->slots[h.pred_slot].live && d->slots[h.pred_slot].seq == h.pred_seq) {
      ++i;  // chained: reported after its predecessor (next poll)
      continue;
    }
    if (__atomic_load_n(&rec->w[15], __ATOMIC_ACQUIRE) != h.seq ||
        __atomic_load_n(&rec->w[11], __ATOMIC_ACQUIRE) != h.seq ||
        __atomic_load_n(&rec->w[7], __ATOMIC_ACQUIRE) != h.seq ||
        __atomic_load_n(&rec->w[3], __ATOMIC_ACQUIRE) != h.seq) {
      ++i;
      continue;
    }
    const volatile uint32_t* w = rec->w;
    gpuos_completion& c = out[n];
    c.atom_id = h.atom_id;
    c.blocks = w[0];
    c.tag = (uint64_t)w[1] | ((uint64_t)w[2] << 32);
    const uint64_t t_first = (uint64_t)w[4] | ((uint64_t)w[5] << 32);
    const uint64_t t_last = t_first + w[6];
    c.tpc_touched[0] = (uint64_t)w[8] | ((uint64_t)w[9] << 32);
    c.tpc_touched[1] = (uint64_t)w[10] | ((uint64_t)w[12] << 32);
    c.dev_first_start_ns = static_cast<int64_t>(t_first) - d->gt_offset;
    c.dev_ingest_ns = c.dev_first_start_ns - static_cast<int64_t>(w[13]);
    c.dev_armed_ns = c.dev_first_start_ns - static_cast<int64_t>(w[14]);
    c.dev_last_end_ns = static_cast<int64_t>(t_last) - d->gt_offset;
    c.host_complete_ns = gpuos_dev_now_ns(d);
    c.host_submit_ns = h.submit_ns;
    if (c.blocks != h.blocks)
      return fail(GPUOS_E_INVARIANT, "completion record does not match its atom");
    for (int t = 0; t < d->cfg.logical_tpcs; ++t)
      if ((h.mask[t >> 6] >> (t & 63)) & 1ull) --d->tpc_resident[t];
    h.live = false;
    d->slot_of.erase(h.atom_id);
    if (h.succ_ring > __atomic_load_n(d->consumed_h, __ATOMIC_ACQUIRE))
      d->deferred_free.emplace_back(h.succ_ring, slot);  // successor not ingested yet
    else
      d->free_slots.push_back(slot);
    d->live[i] = d->live.back();  // O(1) removal; order is irrelevant
    d->live.pop_back();
    --d->in_flight;
    ++d->stats.atoms_completed;
    ++n;
  }
  if (n == 0 && d->in_flight > 0 && d->running && d->launch_rc.load(std::memory_order_acquire) == 1) {
    // Nothing new: make sure the dispatcher still runs (a device fault or
    // the hang guard ends it early), at most once per millisecond.
    const int64_t now = steady_ns();
    if (now - d->exit_check_ns > 1'000'000) {
      d->exit_check_ns = now;
      const cudaError_t q = cudaStreamQuery(d->s_work);
      if (q != cudaErrorNotReady) {
        DevCtl c{};
        cudaMemcpy(&c, d->ctl, sizeof c, cudaMemcpyDeviceToHost);
        if (c.fault != 0u)
          return fail(GPUOS_E_TIMEOUT, std::string("dispatcher stopped on a device fault: ") + fault_text(c));
        return fail(GPUOS_E_INVARIANT, q == cudaSuccess ? "dispatcher exited with atoms in flight"
                                                        : std::string("dispatcher failed: ") + cudaGetErrorString(q));
      }
    }
  }
  return n;
}

int gpuos_dev_get_stats(gpuos_dev* d, gpuos_dev_stats* out) {
  if (!d || !out) return fail(GPUOS_E_CONFIG, "null argument");
  *out = d->stats;
  return GPUOS_OK;
}

// Workspace management runs on a side stream with the stream-ordered
// allocator: it never synchronises the device, so it is safe while the
// persistent dispatcher is resident.
int gpuos_dev_alloc(gpuos_dev* d, uint64_t bytes, void** ptr) {
  if (!d || !ptr) return fail(GPUOS_E_CONFIG, "null argument");
  CUDA_TRY(cudaSetDevice(d->device));
  CUDA_TRY(cudaMallocAsync(ptr, bytes, d->s_side));
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  return GPUOS_OK;
}

int gpuos_dev_free(gpuos_dev* d, void* ptr) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  CUDA_TRY(cudaFreeAsync(ptr, d->s_side));
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  return GPUOS_OK;
}

int gpuos_dev_copy(gpuos_dev* d, void* dst, const void* src, uint64_t bytes, int kind) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                           : kind == 2 ? cudaMemcpyDeviceToHost
                                       : cudaMemcpyDeviceToDevice;
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, k, d->s_side));
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  return GPUOS_OK;
}

int gpuos_dev_memset(gpuos_dev* d, void* dst, int value, uint64_t bytes) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  CUDA_TRY(cudaMemsetAsync(dst, value, bytes, d->s_side));
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  return GPUOS_OK;
}

int gpuos_dev_host_alloc(gpuos_dev* d, uint64_t bytes, void** ptr) {
  if (!d || !ptr) return fail(GPUOS_E_CONFIG, "null argument");
  CUDA_TRY(cudaHostAlloc(ptr, bytes, cudaHostAllocDefault));
  return GPUOS_OK;
}

int gpuos_dev_gemm_desc(gpuos_dev* d, const void* a, const void* b, void* c, int64_t m,
                        int64_t n, int64_t k, int64_t ldc, uint32_t flags, void** desc,
                        int64_t* blocks, int32_t* tile_m, int32_t* tile_n) {
  return gpuos_dev_gemm_desc_splitk(d, a, b, c, m, n, k, ldc, flags, 1, desc, blocks, tile_m, tile_n);
}

int gpuos_dev_gemm_desc_splitk(gpuos_dev* d, const void* a, const void* b, void* c, int64_t m,
                               int64_t n, int64_t k, int64_t ldc, uint32_t flags, int32_t k_splits,
                               void** desc, int64_t* blocks, int32_t* tile_m, int32_t* tile_n) {
  if (!d || !a || !b || !c || !desc) return fail(GPUOS_E_CONFIG, "null argument");
  if (m <= 0 || n <= 0 || k <= 0 || m > 0x7fffffff || n > 0x7fffffff || k > 0x7fffffff)
    return fail(GPUOS_E_CONFIG, "GEMM shape out of range");
  if (k % 8 != 0) return fail(GPUOS_E_CONFIG, "GEMM K must be a multiple of 8 (16-byte rows)");
  if (ldc < n) return fail(GPUOS_E_CONFIG, "GEMM ldc < N");
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) % 16 != 0)
    return fail(GPUOS_E_CONFIG, "GEMM operands must be 16-byte aligned");
  const unsigned cols = tmem_cols_for(d->cfg.workers_per_sm);
  if (cols < kGemmTile || d->topo.smem_per_worker < static_cast<int>(1024 + kGemmStageBytes))
    return fail(GPUOS_E_CONFIG, "workers cannot host a GEMM stage");
  // Narrow outputs (attention heads, narrow layers) take a 64- or 128-wide
  // UMMA N so the tensor cores do not compute padding columns.
  const unsigned n_tile = narrow_tile(n);

  EncodeTiledFn encode = tensor_map_encoder();
  if (!encode) return fail(GPUOS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  GemmDesc h{};
  auto make = [&](CUtensorMap* map, const void* ptr, int64_t rows, unsigned box_rows) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * 2};
    const cuuint32_t box[2] = {kGemmBK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  if (make(&h.a, a, m, kGemmHalf) != CUDA_SUCCESS || make(&h.b, b, n, n_tile / 2) != CUDA_SUCCESS)
    return fail(GPUOS_E_CONFIG, "cuTensorMapEncodeTiled rejected the GEMM operands");
  h.c = reinterpret_cast<unsigned long long>(c);
  h.m = static_cast<unsigned>(m);
  h.n = static_cast<unsigned>(n);
  h.k = static_cast<unsigned>(k);
  h.ldc = static_cast<unsigned>(ldc);
  h.m_tiles = static_cast<unsigned>((m + kGemmTile - 1) / kGemmTile);
  h.n_tiles = static_cast<unsigned>((n + n_tile - 1) / n_tile);
  h.n_tile = n_tile;
  h.flags = flags & kGemmOutBf16;
  h.timing = nullptr;
  // Split-K (wide-K, few-tile shapes such as weight gradients): K slices
  // per split rounded so every split is non-empty.
  const unsigned nk = static_cast<unsigned>((k + kGemmBK - 1) / kGemmBK);
  const unsigned want = std::clamp<unsigned>(k_splits <= 0 ? 1u : static_cast<unsigned>(k_splits), 1u, nk);
  h.tiles = h.m_tiles * h.n_tiles;
  h.k_slices_per_split = (nk + want - 1) / want;
  h.splits = (nk + h.k_slices_per_split - 1) / h.k_slices_per_split;
  if (h.splits == 1) h.k_slices_per_split = nk;
  // One allocation: descriptor, split counters and fp32 tile accumulators
  // (both zeroed; the last split of a tile re-zeroes its accumulator).
  const size_t counters_off = (sizeof(GemmDesc) + 255) & ~size_t{255};
  const size_t partial_off = (counters_off + 4ull * h.tiles + 255) & ~size_t{255};
  const size_t acc_bytes = 4ull * h.tiles * kGemmTile * static_cast<size_t>(n_tile);
  const size_t total = h.splits > 1 ? partial_off + acc_bytes : sizeof(GemmDesc);
  void* p = nullptr;
  CUDA_TRY(cudaSetDevice(d->device));
  CUDA_TRY(cudaMallocAsync(&p, total, d->s_side));
  if (h.splits > 1) {
    h.arrivals = reinterpret_cast<unsigned*>(static_cast<char*>(p) + counters_off);
    h.partial = reinterpret_cast<float*>(static_cast<char*>(p) + partial_off);
    CUDA_TRY(cudaMemsetAsync(h.arrivals, 0, 4ull * h.tiles, d->s_side));
    CUDA_TRY(cudaMemsetAsync(h.partial, 0, acc_bytes, d->s_side));
  }
  CUDA_TRY(cudaMemcpyAsync(p, &h, sizeof(GemmDesc), cudaMemcpyHostToDevice, d->s_side));
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  *desc = p;
  if (blocks) *blocks = static_cast<int64_t>(h.tiles) * h.splits;
  if (tile_m) *tile_m = static_cast<int32_t>(kGemmTile);
  if (tile_n) *tile_n = static_cast<int32_t>(n_tile);
  return GPUOS_OK;
}

int gpuos_dev_gemv_pack(gpuos_dev* d, void* dst, const void* src, int64_t n, int64_t k) {
  if (!d || !dst || !src) return fail(GPUOS_E_CONFIG, "null argument");
  if (n <= 0 || k <= 0 || n > 0x7fffffff || k > 0x7fffffff) return fail(GPUOS_E_CONFIG, "GEMV shape out of range");
  const int64_t total = gemv_packed_rows(n, k) * kGemmBK;
  CUDA_TRY(cudaSetDevice(d->device));
  k_gemv_pack<<<1184, 256, 0, d->s_side>>>(static_cast<unsigned short*>(dst),
                                            static_cast<const unsigned short*>(src), n, k, total);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  return GPUOS_OK;
}

int gpuos_dev_gemv_desc(gpuos_dev* d, const void* w, const void* x, void* y, int64_t n, int64_t k,
                        uint32_t flags, int32_t k_splits, void** desc, int64_t* blocks) {
  if (!d || !w || !x || !y || !desc) return fail(GPUOS_E_CONFIG, "null argument");
  if (n <= 0 || k <= 0 || n > 0x7fffffff || k > 0x7fffffff)
    return fail(GPUOS_E_CONFIG, "GEMV shape out of range");
  if (k % 8 != 0) return fail(GPUOS_E_CONFIG, "GEMV K must be a multiple of 8 (16-byte rows)");
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(x)) % 16 != 0)
    return fail(GPUOS_E_CONFIG, "GEMV W and x must be 16-byte aligned");
  if (tmem_cols_for(d->cfg.workers_per_sm) < kGemvN ||
      d->topo.smem_per_worker < static_cast<int>(1024 + kGemvStageBytes))
    return fail(GPUOS_E_CONFIG, "workers cannot host a GEMV stage");
  EncodeTiledFn encode = tensor_map_encoder();
  if (!encode) return fail(GPUOS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  GemvDesc h{};
  auto make = [&](CUtensorMap* map, const void* ptr, int64_t rows, unsigned box_rows) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * 2};
    const cuuint32_t box[2] = {kGemmBK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  // x is a one-row tensor read with a 16-row box: rows >= 1 are zero fill.
  // Packed W: a [rows, 64] tensor whose 128-row boxes are contiguous 16 KiB.
  const bool packed = (flags & GPUOS_GEMV_W_PACKED) != 0;
  CUresult wr;
  if (packed) {
    const int64_t prow = gemv_packed_rows(n, k);
    const cuuint64_t dims[2] = {kGemmBK, static_cast<cuuint64_t>(prow)};
    const cuuint64_t strides[1] = {kGemmBK * 2};
    const cuuint32_t box[2] = {kGemmBK, kGemmHalf};
    const cuuint32_t estr[2] = {1, 1};
    wr = encode(&h.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    wr = make(&h.w, w, n, kGemmHalf);
  }
  if (wr != CUDA_SUCCESS || make(&h.x, x, 1, kGemvXRows) != CUDA_SUCCESS)
    return fail(GPUOS_E_CONFIG, "cuTensorMapEncodeTiled rejected the GEMV operands");
  h.y = reinterpret_cast<unsigned long long>(y);
  h.n = static_cast<unsigned>(n);
  h.k = static_cast<unsigned>(k);
  const unsigned nk = static_cast<unsigned>((k + kGemmBK - 1) / kGemmBK);
  const unsigned splits = std::clamp<unsigned>(k_splits <= 0 ? 1u : static_cast<unsigned>(k_splits), 1u, nk);
  h.row_tiles = static_cast<unsigned>((n + kGemvTile - 1) / kGemvTile);
  h.k_slices_per_block = (nk + splits - 1) / splits;
  h.splits = (nk + h.k_slices_per_block - 1) / h.k_slices_per_block;
  h.blocks = h.row_tiles * h.splits;
  h.flags = flags & (kGemvOutBf16 | kGemvPacked);
  // One allocation: descriptor, then the split counters (zeroed), then the
  // partial sums; gpuos_dev_free(desc) releases all of it.
  const size_t counters_off = sizeof(GemvDesc);
  const size_t partial_off = (counters_off + 4ull * h.row_tiles + 255) & ~size_t{255};
  const size_t total = partial_off + (h.splits > 1 ? 4ull * h.splits * static_cast<size_t>(n) : 0);
  void* p = nullptr;
  CUDA_TRY(cudaSetDevice(d->device));
  CUDA_TRY(cudaMallocAsync(&p, total, d->s_side));
  h.arrivals = reinterpret_cast<unsigned*>(static_cast<char*>(p) + counters_off);
  h.partial = h.splits > 1 ? reinterpret_cast<float*>(static_cast<char*>(p) + partial_off) : nullptr;
  h.timing = nullptr;
  CUDA_TRY(cudaMemsetAsync(static_cast<char*>(p) + counters_off, 0, 4ull * h.row_tiles, d->s_side));
  CUDA_TRY(cudaMemcpyAsync(p, &h, sizeof(GemvDesc), cudaMemcpyHostToDevice, d->s_side));
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  *desc = p;
  if (blocks) *blocks = h.blocks;
  return GPUOS_OK;
}

int gpuos_dev_conv_desc(gpuos_dev* d, const void* x, const void* w, void* y, int32_t n, int32_t h,
                        int32_t wd, int32_t c, int32_t k, int32_t r, int32_t s, int32_t pad,
                        int32_t stride, uint32_t flags, void** desc, int64_t* blocks, int32_t* p_out,
                        int32_t* q_out) {
  if (!d || !x || !w || !y || !desc) return fail(GPUOS_E_CONFIG, "null argument");
  if (n <= 0 || h <= 0 || wd <= 0 || c <= 0 || k <= 0 || r <= 0 || s <= 0 || pad < 0 || stride <= 0)
    return fail(GPUOS_E_CONFIG, "conv shape out of range");
  if (c % 8 != 0) return fail(GPUOS_E_CONFIG, "conv C must be a multiple of 8 (16-byte pixels)");
  if (stride > 2) return fail(GPUOS_E_CONFIG, "conv stride must be 1 or 2");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) % 16 != 0)
    return fail(GPUOS_E_CONFIG, "conv tensors must be 16-byte aligned");
  const int P = (h + 2 * pad - r) / stride + 1, Q = (wd + 2 * pad - s) / stride + 1;
  if (P <= 0 || Q <= 0) return fail(GPUOS_E_CONFIG, "conv output is empty");
  if (tmem_cols_for(d->cfg.workers_per_sm) < kGemmTile ||
      d->topo.smem_per_worker < static_cast<int>(1024 + kGemmStageBytes))
    return fail(GPUOS_E_CONFIG, "workers cannot host a conv stage");
  if (r > 128 || s > 128 || pad > 127) return fail(GPUOS_E_CONFIG, "conv filter or padding too large");
  EncodeTiledFn encode = tensor_map_encoder();
  EncodeIm2colFn encode_im2col = im2col_map_encoder();
  if (!encode || !encode_im2col) return fail(GPUOS_E_CUDA, "cuTensorMapEncode* unavailable");
  ConvDesc hd{};
  hd.n_tile = narrow_tile(k);
  const unsigned cb = (static_cast<unsigned>(c) + kGemmBK - 1) / kGemmBK;
  {
    // im2col: the bounding box of window origins is [-pad, dim + pad - (F - 1))
    // per spatial dim ({W, H} order), walked with the conv stride.
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(wd),
                                static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 2,
                                   static_cast<cuuint64_t>(c) * 2 * wd,
                                   static_cast<cuuint64_t>(c) * 2 * wd * h};
    const int lower[2] = {-pad, -pad};
    const int upper[2] = {pad - (s - 1), pad - (r - 1)};
    const cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
    if (encode_im2col(&hd.act, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides,
                      lower, upper, kGemmBK, kGemmHalf, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(GPUOS_E_CONFIG, "cuTensorMapEncodeIm2col rejected the conv activations");
  }
  {
    const uint64_t kdim = static_cast<uint64_t>(r) * s * cb * kGemmBK;
    const cuuint64_t dims[2] = {kdim, static_cast<cuuint64_t>(k)};
    const cuuint64_t strides[1] = {kdim * 2};
    const cuuint32_t box[2] = {kGemmBK, hd.n_tile / 2};
    const cuuint32_t estr[2] = {1, 1};
    if (encode(&hd.wgt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(GPUOS_E_CONFIG, "cuTensorMapEncodeTiled rejected the conv weights");
  }
  hd.y = reinterpret_cast<unsigned long long>(y);
  hd.n = n; hd.h = h; hd.w = wd; hd.c = c; hd.k = k; hd.r = r; hd.s = s;
  hd.pad = pad; hd.stride = stride; hd.p = P; hd.q = Q;
  const uint64_t pixels = static_cast<uint64_t>(n) * P * Q;
  if (pixels > 0x7fffffffull) return fail(GPUOS_E_CONFIG, "conv output too large");
  hd.pixels = static_cast<unsigned>(pixels);
  hd.pair_tiles = static_cast<unsigned>((pixels + kGemmTile - 1) / kGemmTile);
  hd.k_tiles = (static_cast<unsigned>(k) + hd.n_tile - 1) / hd.n_tile;
  hd.c_blocks = cb;
  hd.flags = flags & kConvOutBf16;
  void* pdev = nullptr;
  CUDA_TRY(cudaSetDevice(d->device));
  CUDA_TRY(cudaMallocAsync(&pdev, sizeof(ConvDesc), d->s_side));
  CUDA_TRY(cudaMemcpyAsync(pdev, &hd, sizeof(ConvDesc), cudaMemcpyHostToDevice, d->s_side));
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  *desc = pdev;
  if (blocks) *blocks = static_cast<int64_t>(hd.pair_tiles) * hd.k_tiles;
  if (p_out) *p_out = P;
  if (q_out) *q_out = Q;
  return GPUOS_OK;
}

int gpuos_dev_fill_bf16(gpuos_dev* d, void* ptr, uint64_t count, uint64_t seed) {
  if (!d || (!ptr && count)) return fail(GPUOS_E_CONFIG, "null argument");
  if (count == 0) return GPUOS_OK;
  CUDA_TRY(cudaSetDevice(d->device));
  // Tenants register kernels (and so initialise operands) while the
  // persistent dispatcher runs: the fill CTAs must fit beside the workers,
  // which needs the same shared-memory carveout (csrc/tools/residency_probe.cu).
  static bool carveout_set = false;
  if (!carveout_set) {
    CUDA_TRY(cudaFuncSetAttribute(k_fill_bf16, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    carveout_set = true;
  }
  const unsigned long long blocks = std::min<unsigned long long>((count + 255) / 256, 4096);
  k_fill_bf16<<<static_cast<unsigned>(blocks), 256, 0, d->s_side>>>(static_cast<unsigned short*>(ptr),
                                                                    count, seed);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(d->s_side));
  return GPUOS_OK;
}

int gpuos_dev_host_free(gpuos_dev* d, void* ptr) {
  if (!d) return fail(GPUOS_E_CONFIG, "null device");
  CUDA_TRY(cudaFreeHost(ptr));
  return GPUOS_OK;
}

}  // extern "C"
