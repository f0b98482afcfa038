"""Kernel chaining on the persistent dispatcher (gpuos_atom_desc::after).

A chained atom is armed on the device by its predecessor's last block, so a
dependent kernel starts without a host round trip. Checked here:
  * data dependence: a chain of STREAM atoms where atom k reads what atom
    k - 1 wrote equals the CPU oracle applied k times (an early start would
    read unfinished words);
  * ordering: every atom's first block starts after its predecessor's last
    block ends (device clock), and poll() reports the chain in order;
  * both arming paths -- successor registered before the predecessor ends
    (the finisher arms it) and after (the ingest warp arms it) -- and a
    successor whose predecessor was already polled (runs at once);
  * batch mode chains and the argument errors;
  * early start: a chained GEMV whose x is its predecessor's output streams
    W before the predecessor ends and reads x only when its gate opens.
"""
from __future__ import annotations

import random
import time

import numpy as np
import pytest

from oracle.policy import stream_expect

pytestmark = pytest.mark.gpu

WORDS = 4096          # u32 words per STREAM block
BLOCKS = 96


def wait_all(dev, n, timeout=60.0):
    done = []
    t0 = time.time()
    while len(done) < n:
        done += dev.poll()
        assert time.time() - t0 < timeout, f"only {len(done)}/{n} atoms completed"
    return done


def chain_buffers(torch, links, seed=1):
    g = torch.Generator(device="cpu").manual_seed(seed)
    src = torch.randint(-2**31, 2**31 - 1, (BLOCKS * WORDS,), generator=g, dtype=torch.int32)
    bufs = [src.cuda()] + [torch.zeros(BLOCKS * WORDS, dtype=torch.int32, device="cuda")
                           for _ in range(links)]
    return src.numpy().view(np.uint32), bufs


def expect_chain(src, salts):
    x = src
    for s in salts:
        x = stream_expect(x, s, 0)
    return x


def check_order(done, ids):
    by_id = {c.atom_id: c for c in done}
    assert [c.atom_id for c in done if c.atom_id in set(ids)] == ids, "poll order broke the chain"
    for a, b in zip(ids, ids[1:]):
        assert by_id[b].dev_first_start_ns >= by_id[a].dev_last_end_ns, (a, b)


@pytest.mark.parametrize("gap_us", [0, 30])
def test_chain_of_dependent_streams(api, cuda_device, gap_us):
    """gap 0: successors registered while the predecessor runs (finisher
    arms); gap 30 us: often registered after it ended (ingest arms)."""
    import torch

    links = 24
    src, bufs = chain_buffers(torch, links)
    rng = random.Random(gap_us)
    salts = [rng.randrange(1, 2**32) for _ in range(links)]
    with api.Device(workers_per_sm=2) as dev:
        dev.start()
        ids = []
        for k in range(links):
            tpcs = sorted(rng.sample(range(74), rng.choice([2, 8, 37, 74])))
            ids.append(dev.submit(0, BLOCKS, tpcs, 30, api.GPUOS_BODY_STREAM,
                                  [bufs[k].data_ptr(), bufs[k + 1].data_ptr(), WORDS, salts[k], 0],
                                  after=ids[-1] if ids else None, chain_head=k + 1 < links))
            if gap_us:
                time.sleep(gap_us * 1e-6 * rng.random())
        done = wait_all(dev, links)
        dev.stop()
    check_order(done, ids)
    got = bufs[-1].cpu().numpy().view(np.uint32)
    assert np.array_equal(got, expect_chain(src, salts))


def test_successor_of_a_polled_atom_runs_at_once(api, cuda_device):
    import torch

    src, bufs = chain_buffers(torch, 2, seed=5)
    with api.Device(workers_per_sm=2) as dev:
        dev.start()
        a = dev.submit(0, BLOCKS, range(74), 30, api.GPUOS_BODY_STREAM,
                       [bufs[0].data_ptr(), bufs[1].data_ptr(), WORDS, 11, 0], chain_head=True)
        wait_all(dev, 1)
        b = dev.submit(0, BLOCKS, range(74), 30, api.GPUOS_BODY_STREAM,
                       [bufs[1].data_ptr(), bufs[2].data_ptr(), WORDS, 12, 0], after=a)
        (c,) = wait_all(dev, 1)
        assert c.atom_id == b
        dev.stop()
    assert np.array_equal(bufs[2].cpu().numpy().view(np.uint32), expect_chain(src, [11, 12]))


def test_chains_beside_unchained_traffic(api, cuda_device):
    """Two interleaved chains (HP) and independent BE atoms on shared TPCs."""
    import torch

    links = 10  # 3 resident atoms per link on TPCs 30-39 (32 per TPC at most)
    s1, b1 = chain_buffers(torch, links, seed=2)
    s2, b2 = chain_buffers(torch, links, seed=3)
    words_be, be_blocks = 2048, 300
    be_src = torch.randint(-2**31, 2**31 - 1, (be_blocks * words_be,), dtype=torch.int32, device="cuda")
    be_dst = torch.zeros_like(be_src)
    with api.Device(workers_per_sm=2) as dev:
        dev.start()
        ids1, ids2, n = [], [], 0
        for k in range(links):
            ids1.append(dev.submit(0, BLOCKS, range(0, 40), 30, api.GPUOS_BODY_STREAM,
                                   [b1[k].data_ptr(), b1[k + 1].data_ptr(), WORDS, 100 + k, 0],
                                   after=ids1[-1] if ids1 else None, chain_head=True))
            ids2.append(dev.submit(0, BLOCKS, range(30, 74), 25, api.GPUOS_BODY_STREAM,
                                   [b2[k].data_ptr(), b2[k + 1].data_ptr(), WORDS, 200 + k, 0],
                                   after=ids2[-1] if ids2 else None, chain_head=True))
            lo, hi = k * be_blocks // links, (k + 1) * be_blocks // links
            dev.submit(lo, hi, range(74), 20, api.GPUOS_BODY_STREAM,
                       [be_src.data_ptr(), be_dst.data_ptr(), words_be, 7, 0])
            n += 3
        done = wait_all(dev, n)
        dev.stop()
    check_order(done, ids1)
    check_order(done, ids2)
    assert np.array_equal(b1[-1].cpu().numpy().view(np.uint32), expect_chain(s1, [100 + k for k in range(links)]))
    assert np.array_equal(b2[-1].cpu().numpy().view(np.uint32), expect_chain(s2, [200 + k for k in range(links)]))
    assert np.array_equal(be_dst.cpu().numpy().view(np.uint32),
                          stream_expect(be_src.cpu().numpy().view(np.uint32), 7, 0))


def test_batch_chain(api, cuda_device):
    import torch

    links = 12
    src, bufs = chain_buffers(torch, links, seed=9)
    with api.Device(workers_per_sm=2) as dev:
        base = None
        descs = []
        for k in range(links):
            descs.append(api.Device.desc(0, BLOCKS, range(74), 30, api.GPUOS_BODY_STREAM,
                                         [bufs[k].data_ptr(), bufs[k + 1].data_ptr(), WORDS, 50 + k, 0],
                                         chain_head=True))
        # Atom ids of a batch are consecutive from the handle's next id:
        # learn it from a first one-atom batch.
        dev.run_batch([api.Device.desc(0, 1, [0], 30, api.GPUOS_BODY_SPIN, [0])])
        (c,) = wait_all(dev, 1)
        base = c.atom_id + 1
        for k in range(1, links):
            descs[k].after = base + k - 1 + 1
        dev.run_batch(descs)
        done = wait_all(dev, links)
    check_order(done, [base + k for k in range(links)])
    assert np.array_equal(bufs[-1].cpu().numpy().view(np.uint32),
                          expect_chain(src, [50 + k for k in range(links)]))


def test_chain_argument_errors(api, cuda_device):
    with api.Device(workers_per_sm=2) as dev:
        dev.start()
        a = dev.submit(0, 1, [0], 30, api.GPUOS_BODY_SPIN, [200_000])  # not a chain head
        with pytest.raises(api.GpuosError):
            dev.submit(0, 1, [0], 30, api.GPUOS_BODY_SPIN, [0], after=a)
        h = dev.submit(0, 1, [1], 30, api.GPUOS_BODY_SPIN, [200_000], chain_head=True)
        dev.submit(0, 1, [1], 30, api.GPUOS_BODY_SPIN, [0], after=h)
        with pytest.raises(api.GpuosError):  # one successor per head
            dev.submit(0, 1, [1], 30, api.GPUOS_BODY_SPIN, [0], after=h)
        with pytest.raises(api.GpuosError):  # never issued
            dev.submit(0, 1, [1], 30, api.GPUOS_BODY_SPIN, [0], after=10_000_000)
        wait_all(dev, 3)
        dev.stop()


def test_chain_removes_the_host_round_trip(api, cuda_device):
    """200 one-block kernels back to back: chained on the device vs each
    submitted when the host sees its predecessor complete."""
    n = 200
    with api.Device(workers_per_sm=2) as dev:
        dev.start()
        t0 = time.perf_counter()
        for _ in range(n):
            dev.submit(0, 1, [3], 30, api.GPUOS_BODY_SPIN, [1000])
            wait_all(dev, 1)
        serial = (time.perf_counter() - t0) / n
        ids, done = [], []
        for k in range(n):
            while len(ids) - len(done) >= 24:  # 32 resident atoms per TPC at most
                done += dev.poll()
            ids.append(dev.submit(0, 1, [3], 30, api.GPUOS_BODY_SPIN, [1000],
                                  after=ids[-1] if ids else None, chain_head=True))
        done += wait_all(dev, n - len(done))
        dev.stop()
    check_order(done, ids)
    by_id = {c.atom_id: c for c in done}
    gaps = [by_id[b].dev_first_start_ns - by_id[a].dev_last_end_ns for a, b in zip(ids, ids[1:])]
    med = float(np.median(gaps))
    print(f"serial host round trip {serial * 1e6:.1f} us/kernel; chained gap median {med / 1e3:.2f} us")
    assert med < 0.5 * (serial * 1e9 - 1000)


@pytest.mark.parametrize("n1,k,n2,splits", [(8192, 4096, 4096, 4), (2048, 1024, 28672, 1)])
def test_early_started_gemv_reads_its_predecessors_output(api, cuda_device, n1, k, n2, splits):
    """y1 = W1 x (bf16 out) then y2 = W2 y1, chained: y2 must equal the
    product with the y1 the device wrote (y1 starts as NaN, so an x read
    before the gate opened shows up)."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(n1 + n2)
    w1 = (torch.rand(n1, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    x = (torch.rand(k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w2 = (torch.rand(n2, n1, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    y1 = torch.full((n1,), float("nan"), device="cuda", dtype=torch.bfloat16)
    y2 = torch.full((n2,), float("nan"), device="cuda")
    with api.Device(workers_per_sm=2) as dev:
        d1, b1 = dev.gemv_desc(w1.data_ptr(), x.data_ptr(), y1.data_ptr(), n1, k, bf16_out=True, k_splits=splits)
        d2, b2 = dev.gemv_desc(w2.data_ptr(), y1.data_ptr(), y2.data_ptr(), n2, n1, k_splits=splits)
        for rep in range(3):
            # (no torch kernel can run beside the resident dispatcher: fill
            # and check between runs)
            y1.fill_(float("nan"))
            y2.fill_(float("nan"))
            torch.cuda.synchronize()
            dev.start()
            a = dev.submit(0, b1, range(74), 30, api.GPUOS_BODY_GEMV_BF16, [d1], chain_head=True)
            b = dev.submit(0, b2, range(74), 30, api.GPUOS_BODY_GEMV_BF16, [d2], after=a)
            done = wait_all(dev, 2)
            dev.stop()
            assert [c.atom_id for c in done] == [a, b]
            y1h = y1.double().cpu()
            ref = (w2.double().cpu() @ y1h).float()
            assert not torch.isnan(y1h).any()
            err = ((y2.cpu() - ref).abs().max() / ref.abs().max()).item()
            assert err < 1e-3, (rep, err)
        dev.free(d1)
        dev.free(d2)


def test_early_started_gemm_and_conv_read_their_predecessors_output(api, cuda_device):
    """C1 = A B1^T (bf16) then C2 = C1 B2^T; X1 = conv(X0) (bf16 NHWC) then
    X2 = conv(X1): each second kernel chained and started early (weights
    first); the intermediates start as NaN."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(11)
    m, k, n1, n2 = 1024, 512, 768, 640
    a = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    b1 = (torch.rand(n1, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    b2 = (torch.rand(n2, n1, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    c1 = torch.full((m, n1), float("nan"), device="cuda", dtype=torch.bfloat16)
    c2 = torch.full((m, n2), float("nan"), device="cuda")
    nb, hw, ch = 4, 14, 128
    x0 = (torch.rand(nb, hw, hw, ch, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    wa = (torch.rand(ch, 3, 3, ch, device="cuda", generator=g) * 0.2 - 0.1).to(torch.bfloat16)
    wb = (torch.rand(ch, 3, 3, ch, device="cuda", generator=g) * 0.2 - 0.1).to(torch.bfloat16)
    x1 = torch.full((nb, hw, hw, ch), float("nan"), device="cuda", dtype=torch.bfloat16)
    x2 = torch.full((nb, hw, hw, ch), float("nan"), device="cuda")
    torch.cuda.synchronize()
    with api.Device(workers_per_sm=2) as dev:
        g1, gb1, _, _ = dev.gemm_desc(a.data_ptr(), b1.data_ptr(), c1.data_ptr(), m, n1, k, bf16_out=True)
        g2, gb2, _, _ = dev.gemm_desc(c1.data_ptr(), b2.data_ptr(), c2.data_ptr(), m, n2, n1)
        v1, vb1, _, _ = dev.conv_desc(x0.data_ptr(), wa.data_ptr(), x1.data_ptr(), nb, hw, hw, ch, ch, 3, 3, 1, 1,
                                      bf16_out=True)
        v2, vb2, _, _ = dev.conv_desc(x1.data_ptr(), wb.data_ptr(), x2.data_ptr(), nb, hw, hw, ch, ch, 3, 3, 1, 1)
        dev.start()
        ga = dev.submit(0, gb1, range(74), 30, api.GPUOS_BODY_GEMM_BF16, [g1], chain_head=True)
        gb = dev.submit(0, gb2, range(74), 30, api.GPUOS_BODY_GEMM_BF16, [g2], after=ga)
        ca = dev.submit(0, vb1, range(74), 30, api.GPUOS_BODY_CONV_BF16, [v1], chain_head=True)
        cb = dev.submit(0, vb2, range(74), 30, api.GPUOS_BODY_CONV_BF16, [v2], after=ca)
        done = wait_all(dev, 4)
        dev.stop()
        for d in (g1, g2, v1, v2):
            dev.free(d)
    order = [c.atom_id for c in done]
    assert order.index(ga) < order.index(gb) and order.index(ca) < order.index(cb)
    c1h = c1.double().cpu()
    assert not torch.isnan(c1h).any()
    ref = c1h @ b2.double().cpu().T
    err = ((c2.double().cpu() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-3, err
    x1h = x1.double().cpu()
    assert not torch.isnan(x1h).any()
    refx = torch.nn.functional.conv2d(x1h.permute(0, 3, 1, 2), wb.double().cpu().permute(0, 3, 1, 2),
                                      padding=1).permute(0, 2, 3, 1)
    errx = ((x2.double().cpu() - refx).abs().max() / refx.abs().max()).item()
    assert errx < 1e-3, errx


def test_no_early_keeps_a_chained_gemv_behind_its_predecessor(api, cuda_device):
    """GPUOS_ATOM_NO_EARLY: the chained GEMV is armed only when its
    predecessor completes (no block starts before the predecessor's last
    ends), and still reads the predecessor's output."""
    import torch

    n1, k, n2 = 8192, 4096, 4096
    g = torch.Generator(device="cuda").manual_seed(5)
    w1 = (torch.rand(n1, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    x = (torch.rand(k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w2 = (torch.rand(n2, n1, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    y1 = torch.full((n1,), float("nan"), device="cuda", dtype=torch.bfloat16)
    y2 = torch.full((n2,), float("nan"), device="cuda")
    torch.cuda.synchronize()
    with api.Device(workers_per_sm=2) as dev:
        d1, b1 = dev.gemv_desc(w1.data_ptr(), x.data_ptr(), y1.data_ptr(), n1, k, bf16_out=True, k_splits=4)
        d2, b2 = dev.gemv_desc(w2.data_ptr(), y1.data_ptr(), y2.data_ptr(), n2, n1, k_splits=4)
        dev.start()
        a = dev.submit(0, b1, range(74), 30, api.GPUOS_BODY_GEMV_BF16, [d1], chain_head=True)
        b = dev.submit(0, b2, range(74), 30, api.GPUOS_BODY_GEMV_BF16, [d2], after=a, no_early=True)
        done = wait_all(dev, 2)
        dev.stop()
        dev.free(d1)
        dev.free(d2)
    check_order(done, [a, b])
    by_id = {c.atom_id: c for c in done}
    # Not armed early: no block of b starts before a's last block ends.
    assert by_id[b].dev_first_start_ns >= by_id[a].dev_last_end_ns, (
        by_id[b].dev_first_start_ns, by_id[a].dev_last_end_ns)
    ref = (w2.double().cpu() @ y1.double().cpu()).float()
    err = ((y2.cpu() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-3, err


def test_look_ahead_races_the_successors_own_finisher(api, cuda_device):
    """Chains alternating GEMV -> one-block STREAM -> GEMV ...: a GEMV's
    finisher arms the STREAM and looks ahead to arm the next GEMV behind a
    gate, while the STREAM -- on a TPC the finisher is not on, so another
    worker runs it -- may finish first and arm that GEMV itself. Exactly one
    of them may arm it (kSuccLook / the finisher's swap): arming it twice
    re-opened its claims behind a gate nobody would open again (a stall a
    config-#3 run hit once in ~12). Many short chains must all complete, in
    chain order, every block once."""
    import torch

    n, k = 1024, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    w = (torch.rand(n, k, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    x = (torch.rand(k, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    y = torch.zeros(n, device="cuda")
    src = torch.randint(-2**31, 2**31 - 1, (WORDS,), dtype=torch.int32, device="cuda")
    dst = torch.zeros_like(src)
    torch.cuda.synchronize()
    chains, length = 40, 12
    with api.Device(workers_per_sm=2) as dev:
        d, blocks = dev.gemv_desc(w.data_ptr(), x.data_ptr(), y.data_ptr(), n, k, k_splits=2)
        dev.start()
        ids = []
        for c in range(chains):
            prev = None
            chain = []
            for j in range(length):
                head = j + 1 < length
                if j % 2 == 0:
                    aid = dev.submit(0, blocks, list(range(8, 74)), 30, api.GPUOS_BODY_GEMV_BF16, [d],
                                     after=prev, chain_head=head)
                else:
                    aid = dev.submit(0, 1, [c % 8], 30, api.GPUOS_BODY_STREAM,
                                     [src.data_ptr(), dst.data_ptr(), WORDS, 5, 1], after=prev, chain_head=head)
                chain.append(aid)
                prev = aid
            ids.append(chain)
            if c % 4 == 3:  # keep the atom table and resident lists from filling
                wait_all(dev, 4 * length, timeout=30.0)
        rest = chains % 4
        if rest:
            wait_all(dev, rest * length, timeout=30.0)
        dev.stop()
        dev.free(d)
