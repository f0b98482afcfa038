"""Device-level parity of the persistent sm_100a dispatcher, through the C
ABI (include/gpuos_dev.h). Checked against the CPU oracle: every block of
every atom runs exactly once, only on SMs of the atom's TPC set, and STREAM
body outputs equal oracle.policy.stream_expect bit for bit. Also the
reference engine's priority-refill, pause and revocation semantics
(device.cpp:165-206) on real hardware."""
from __future__ import annotations

import random
import time

import numpy as np
import pytest

from oracle.policy import stream_expect

pytestmark = pytest.mark.gpu


def wait_all(dev, n, timeout=30.0):
    done = []
    t0 = time.time()
    while len(done) < n:
        done += dev.poll()
        assert time.time() - t0 < timeout, f"only {len(done)}/{n} atoms completed"
    return done


def decode(trace):
    tr = trace.cpu().numpy().view(np.uint32)
    return tr >> 16, (tr & 0xFFFF).astype(np.int64) - 1


@pytest.fixture()
def torch_mod(cuda_device):
    import torch

    return torch


def test_topology_and_residency(api, cuda_device):
    with api.Device(workers_per_sm=2) as dev:
        t = dev.topology
        assert (t.sm_count, t.physical_tpcs, t.logical_tpcs) == (148, 74, 74)
        assert t.workers_per_tpc == 4
        dev.start()  # fails loudly unless every SM hosts exactly W workers
        dev.stop()
    with api.Device(workers_per_sm=1) as dev:
        with pytest.raises(api.GpuosError) as e:
            dev.start()  # live mode needs W = 2 (cluster 0 hosts the ingest warp)
        assert e.value.code == -2


@pytest.mark.parametrize("workers_per_sm", [1, 2])
def test_stream_atoms_exactly_once_placed_bit_exact(api, torch_mod, workers_per_sm):
    torch = torch_mod
    rng = random.Random(workers_per_sm)
    words, blocks = 1024, 6000
    src = torch.randint(-2**31, 2**31 - 1, (blocks * words,), dtype=torch.int32, device="cuda")
    dst = torch.zeros_like(src)
    trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    salt = 0x5EED1234
    # Random partition into atoms with random TPC sets and priorities,
    # including single-block atoms and the highest TPC ids.
    cuts = sorted(rng.sample(range(1, blocks), 60))
    ranges = list(zip([0] + cuts, cuts + [blocks]))
    specs = []
    for lo, hi in ranges:
        k = rng.choice([1, 2, 5, 20, 74])
        tpcs = sorted(rng.sample(range(74), k)) if k < 74 else list(range(74))
        if rng.random() < 0.1:
            tpcs = [73]
        specs.append((lo, hi, tpcs, rng.choice([10, 20, 30])))
    with api.Device(workers_per_sm=workers_per_sm) as dev:
        if workers_per_sm == 2:
            dev.start()  # live: ring + ingest warp (cluster 0) + workers
            for lo, hi, tpcs, prio in specs:
                dev.submit(lo, hi, tpcs, prio, api.GPUOS_BODY_STREAM,
                           [src.data_ptr(), dst.data_ptr(), words, salt, 0], trace=trace.data_ptr())
            done = wait_all(dev, len(specs))
            dev.stop()
        else:
            # W = 1 runs batch mode only (live mode's ingest cluster would
            # take a TPC's only worker pair); <= 32 atoms per TPC.
            descs = [api.Device.desc(lo, hi, tpcs, prio, api.GPUOS_BODY_STREAM,
                                     [src.data_ptr(), dst.data_ptr(), words, salt, 0], trace=trace.data_ptr())
                     for lo, hi, tpcs, prio in specs]
            dev.run_batch(descs[:30])
            done = wait_all(dev, 30)
            dev.run_batch(descs[30:])
            done += wait_all(dev, len(specs) - 30)
    counts, sm = decode(trace)
    assert (counts == 1).all(), f"{int((counts == 0).sum())} missing, {int((counts > 1).sum())} duplicated"
    for (lo, hi, tpcs, _), c in zip(specs, sorted(done, key=lambda c: c.atom_id)):
        assert set((sm[lo:hi] >> 1).tolist()) <= set(tpcs)
        assert c.blocks == hi - lo
        touched = {t for t in range(74) if (c.tpc_touched[t >> 6] >> (t & 63)) & 1}
        assert touched <= set(tpcs) and touched
        assert c.dev_last_end_ns >= c.dev_first_start_ns
    expect = stream_expect(src.cpu().numpy().view(np.uint32), salt, 0)
    assert np.array_equal(dst.cpu().numpy().view(np.uint32), expect)


def test_chunked_stream_and_block_offsets(api, torch_mod):
    """args[4] = chunks: block b works on chunk b % chunks (bounded workspace)."""
    torch = torch_mod
    words, chunks, blocks = 512, 7, 500
    src = torch.randint(-2**31, 2**31 - 1, (chunks * words,), dtype=torch.int32, device="cuda")
    dst = torch.zeros_like(src)
    trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    with api.Device() as dev:
        dev.start()
        dev.submit(100, 500, list(range(10, 30)), 20, api.GPUOS_BODY_STREAM,
                   [src.data_ptr(), dst.data_ptr(), words, 77, chunks], trace=trace.data_ptr())
        dev.submit(0, 100, [0], 30, api.GPUOS_BODY_STREAM,
                   [src.data_ptr(), dst.data_ptr(), words, 77, chunks], trace=trace.data_ptr())
        wait_all(dev, 2)
        dev.stop()
    counts, sm = decode(trace)
    assert (counts == 1).all()
    assert set((sm[100:] >> 1).tolist()) <= set(range(10, 30))
    assert set((sm[:100] >> 1).tolist()) == {0}
    assert np.array_equal(dst.cpu().numpy().view(np.uint32),
                          stream_expect(src.cpu().numpy().view(np.uint32), 77, 0))


@pytest.mark.parametrize("parts", [2, 3, 7])
def test_preemption_slices_exactly_once(api, torch_mod, parts):
    """parts > 1: every block runs as `parts` independently claimed slices;
    each slice exactly once, on the atom's TPCs, output bit-exact."""
    torch = torch_mod
    words, blocks = 4096, 700
    src = torch.randint(-2**31, 2**31 - 1, (blocks * words,), dtype=torch.int32, device="cuda")
    dst = torch.zeros_like(src)
    trace = torch.zeros(blocks * parts, dtype=torch.int32, device="cuda")
    with api.Device() as dev:
        dev.start()
        dev.submit(0, 300, list(range(0, 20)), 20, api.GPUOS_BODY_STREAM,
                   [src.data_ptr(), dst.data_ptr(), words, 5, 0], trace=trace.data_ptr(), parts=parts)
        dev.submit(300, 700, [40, 41], 30, api.GPUOS_BODY_STREAM,
                   [src.data_ptr(), dst.data_ptr(), words, 5, 0], trace=trace.data_ptr(), parts=parts)
        done = wait_all(dev, 2)
        dev.stop()
    assert sorted(c.blocks for c in done) == [300, 400]
    counts, sm = decode(trace)
    assert (counts == 1).all()
    assert set((sm[:300 * parts] >> 1).tolist()) <= set(range(20))
    assert set((sm[300 * parts:] >> 1).tolist()) <= {40, 41}
    assert np.array_equal(dst.cpu().numpy().view(np.uint32),
                          stream_expect(src.cpu().numpy().view(np.uint32), 5, 0))


def test_higher_priority_takes_freed_slots_first(api, torch_mod):
    """A late high-priority atom overtakes the waiting blocks of a resident
    low-priority atom on the same TPC (reference refill rule,
    device.cpp:188-206; test_device.cpp:101-115)."""
    with api.Device(workers_per_sm=2) as dev:
        dev.start()
        lp = dev.submit(0, 200, [0], 5, api.GPUOS_BODY_SPIN, [200_000, 0, 0, 0, 0], tag=1)
        time.sleep(0.002)
        t_hp = dev.now_ns()
        hp = dev.submit(0, 8, [0], 30, api.GPUOS_BODY_SPIN, [50_000, 0, 0, 0, 0], tag=2)
        done = {c.atom_id: c for c in wait_all(dev, 2)}
        dev.stop()
    # 4 workers on TPC 0: HP waits at most one LP block (200 us) for a slot,
    # then runs 2 waves of 50 us; LP still has ~190 blocks (~10 ms) to go.
    assert done[hp].dev_last_end_ns - t_hp < 1_000_000
    assert done[hp].dev_last_end_ns < done[lp].dev_last_end_ns - 5_000_000


def test_pause_keeps_in_flight_blocks_and_resumes(api, torch_mod):
    torch = torch_mod
    trace = torch.zeros(400, dtype=torch.int32, device="cuda")
    with api.Device() as dev:
        dev.start()
        a = dev.submit(0, 400, [3], 20, api.GPUOS_BODY_SPIN, [100_000, 0, 0, 0, 0],
                       trace=trace.data_ptr())
        time.sleep(0.001)
        dev.pause(a, True)
        time.sleep(0.003)  # let in-flight blocks finish
        before = int((decode(trace)[0] > 0).sum())
        time.sleep(0.005)
        after = int((decode(trace)[0] > 0).sum())
        assert after == before and 0 < before < 400
        dev.pause(a, False)
        wait_all(dev, 1)
        dev.stop()
    assert (decode(trace)[0] == 1).all()


def test_fence_revokes_tpcs_mid_atom(api, torch_mod):
    """Raising a TPC's fence stops a stolen (priority 10) atom from starting
    new blocks there without relaunching it: block-granular revocation."""
    torch = torch_mod
    blocks = 800
    trace = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    with api.Device() as dev:
        dev.start()
        dev.submit(0, blocks, [0, 1, 2, 3], 10, api.GPUOS_BODY_SPIN, [100_000, 0, 0, 0, 0],
                   trace=trace.data_ptr())
        time.sleep(0.001)
        dev.fence_mask([0, 1], 11)
        time.sleep(0.0005)
        frontier = int(np.nonzero(decode(trace)[0])[0].max()) + 64  # claimed before the fence took hold
        wait_all(dev, 1)
        dev.fence(0, 0)
        dev.fence(1, 0)
        dev.stop()
    counts, sm = decode(trace)
    assert (counts == 1).all()
    late = sm[frontier:] >> 1
    assert frontier < blocks - 100
    assert set(late.tolist()) <= {2, 3}


def test_tpc_owner_keeps_its_own_stolen_priority_atoms(api, torch_mod):
    """The TPC-ownership table: an owner fences its quota (TPCs 0-1) against
    other tenants' stolen-priority atoms, while its own atom -- priority 10
    because it also spans stolen TPCs 2-3 -- keeps starting blocks there."""
    torch = torch_mod
    blocks = 800
    own = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    other = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    with api.Device() as dev:
        dev.start()
        dev.set_owner([0, 1], owner=1, min_priority=11)
        time.sleep(0.0005)
        dev.submit(0, blocks, [0, 1, 2, 3], 10, api.GPUOS_BODY_SPIN, [50_000], trace=own.data_ptr(), tenant=1)
        dev.submit(0, blocks, [0, 1, 2, 3], 10, api.GPUOS_BODY_SPIN, [50_000], trace=other.data_ptr(), tenant=2)
        wait_all(dev, 2)
        dev.set_owner([0, 1], owner=0, min_priority=0)
        dev.stop()
    c_own, sm_own = decode(own)
    c_oth, sm_oth = decode(other)
    assert (c_own == 1).all() and (c_oth == 1).all()
    assert set((sm_own >> 1).tolist()) == {0, 1, 2, 3}  # the owner's atom used its quota
    assert set((sm_oth >> 1).tolist()) <= {2, 3}        # the other tenant's never did


def test_slot_recycling_many_small_atoms(api, torch_mod):
    """10k one-to-three-block atoms through a 64-slot atom table: slots are
    reused while stale resident keys are still visible; the sequence-tagged
    claim word must keep every block exactly once."""
    torch = torch_mod
    n_atoms = 10_000
    trace = torch.zeros(n_atoms * 3, dtype=torch.int32, device="cuda")
    rng = random.Random(5)
    with api.Device(atom_slots=64) as dev:
        dev.start()
        sub, got, b = 0, 0, 0
        t0 = time.time()
        while got < n_atoms:
            if sub < n_atoms:
                k = rng.randint(1, 3)
                aid = dev.try_submit(b, b + k, [rng.randrange(74)], rng.choice([10, 20, 30]),
                                     api.GPUOS_BODY_SPIN, [0, 0, 0, 0, 0], trace=trace.data_ptr())
                if aid is not None:
                    sub += 1
                    b += k
            got += len(dev.poll())
            assert time.time() - t0 < 60
        dev.stop()
    counts, _ = decode(trace)
    assert (counts[:b] == 1).all() and (counts[b:] == 0).all()


def test_residency_limit_is_enforced(api, torch_mod):
    with api.Device() as dev:
        dev.start()
        for _ in range(32):
            dev.submit(0, 1, [5], 20, api.GPUOS_BODY_SPIN, [2_000_000, 0, 0, 0, 0])
        with pytest.raises(api.GpuosError) as e:
            dev.submit(0, 1, [5], 20, api.GPUOS_BODY_SPIN, [0, 0, 0, 0, 0])
        assert e.value.code == api.GPUOS_E_FULL
        wait_all(dev, 32)
        dev.stop()


def test_bad_submissions_rejected(api, torch_mod):
    with api.Device() as dev:
        dev.start()
        for lo, hi, tpcs in [(5, 5, [0]), (-1, 3, [0]), (0, 3, []), (0, 3, [74])]:
            with pytest.raises(api.GpuosError) as e:
                dev.submit(lo, hi, tpcs, 20, api.GPUOS_BODY_SPIN, [0, 0, 0, 0, 0])
            assert e.value.code == -2
        dev.stop()


def test_batch_stream_bandwidth(api, torch_mod):
    """Full-width atomized STREAM kernel in batch mode (atoms staged, worker
    kernel launched alone): its CUDA-event time is execution only."""
    torch = torch_mod
    words, blocks = 65536, 8192  # 256 KiB per block, 2 GiB per buffer
    src = torch.randint(-2**31, 2**31 - 1, (blocks * words,), dtype=torch.int32, device="cuda")
    dst = torch.zeros_like(src)
    torch.cuda.synchronize()
    n_atoms, per = 32, blocks // 32
    descs = [api.Device.desc(i * per, (i + 1) * per, range(74), 20, api.GPUOS_BODY_STREAM,
                             [src.data_ptr(), dst.data_ptr(), words, 9, 0]) for i in range(n_atoms)]
    with api.Device() as dev:
        best = 0.0
        for _ in range(3):
            ms = dev.run_batch(descs)
            assert len(wait_all(dev, n_atoms)) == n_atoms
            best = max(best, blocks * words * 8 / (ms * 1e-3) / 1e9)
    expect = stream_expect(src.cpu().numpy().view(np.uint32), 9, 0)
    assert np.array_equal(dst.cpu().numpy().view(np.uint32), expect)
    assert best > 3000, f"{best:.0f} GB/s"


def test_batch_mode_priority_and_placement(api, torch_mod):
    torch = torch_mod
    trace = torch.zeros(3000, dtype=torch.int32, device="cuda")
    descs = [api.Device.desc(i * 100, (i + 1) * 100, [i % 74, (i * 7) % 74], 10 + 10 * (i % 3),
                             api.GPUOS_BODY_SPIN, [2000, 0, 0, 0, 0], trace=trace.data_ptr())
             for i in range(30)]
    with api.Device() as dev:
        dev.run_batch(descs)
        done = wait_all(dev, 30)
    counts, sm = decode(trace)
    assert (counts == 1).all()
    for i in range(30):
        assert set((sm[i * 100:(i + 1) * 100] >> 1).tolist()) <= {i % 74, (i * 7) % 74}
    assert sorted(c.blocks for c in done) == [100] * 30


def test_tpc_busy_sampler_matches_known_occupancy(api, cuda_device):
    """TPC utilisation with the reference's definition (device.cpp:264-275):
    the device integrates "TPCs with >= 1 running block". 10 TPCs run 1 ms
    SPIN blocks back to back (4 workers each, 20 waves) while the other 64
    stay idle: the integral is ~10 TPCs x the atom's span."""
    with api.Device(workers_per_sm=2) as dev:
        dev.start()
        before = dev.stats().tpc_busy_ns
        blocks = 10 * 4 * 20
        dev.submit(0, blocks, list(range(10, 20)), 20, api.GPUOS_BODY_SPIN, [1_000_000])
        (c,) = wait_all(dev, 1)
        dev.stop()
        busy = dev.stats().tpc_busy_ns - before
    span = c.dev_last_end_ns - c.dev_first_start_ns
    assert 19e6 <= span <= 23e6, span
    assert 0.95 * 10 * span <= busy <= 10 * span + 10 * 0.5e6, (busy, span)


def test_pair_fence_keeps_one_pair_per_tpc(api, torch_mod):
    """gpuos_dev_set_pair_fence: with pair slot 0 fenced against priority
    < 21, a priority-20 atom of 1-SM blocks on one TPC runs on the slot-1
    pair's two CTAs only (half the TPC's four workers: ~2x the span), while
    a priority-30 atom still uses all four; lifting the fence restores it."""
    torch = torch_mod
    blocks, spin_ns = 16, 100_000

    ideal = blocks * spin_ns / 1e3 / 4  # four workers

    def span(dev, tpc, prio):
        aid = dev.submit(0, blocks, [tpc], prio, api.GPUOS_BODY_SPIN, [spin_ns])
        c = [x for x in wait_all(dev, 1) if x.atom_id == aid][0]
        return (c.dev_last_end_ns - c.dev_first_start_ns) / 1e3

    with api.Device() as dev:
        dev.start()
        # (the TPC hosting the ingest warp has one worker pair: skip it)
        tpc = next(t for t in (40, 41, 42) if span(dev, t, 20) < 1.3 * ideal)
        free = span(dev, tpc, 20)
        dev.set_pair_fence([tpc], 1, 21)
        time.sleep(0.0005)
        fenced = span(dev, tpc, 20)
        hp = span(dev, tpc, 30)
        dev.set_pair_fence([tpc], 1, 0)
        time.sleep(0.0005)
        lifted = span(dev, tpc, 20)
        dev.stop()
    assert free < 1.3 * ideal and lifted < 1.3 * ideal, (free, lifted, ideal)
    assert hp < 1.3 * ideal, (hp, ideal)
    assert 1.8 * ideal < fenced < 2.6 * ideal, (fenced, ideal)
