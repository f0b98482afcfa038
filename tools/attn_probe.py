"""Decode attention body timing: one atom of attn_decode_bf16 on all 74 TPCs,
per-block stamps (args[3] bit 63): start, loads issued, partials written,
end -- and the atom's device span."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402

ctx, chunk = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1024, 32)
chunks = -(-ctx // chunk)
blocks = chunks * 8
q = (torch.rand(32, 128, device="cuda") - 0.5).to(torch.bfloat16)
kv = (torch.rand(2, ctx, 8, 128, device="cuda") - 0.5).to(torch.bfloat16)
ws_bytes = 8448 + 32 * chunks * 130 * 4 + 32 * blocks
ws = torch.zeros(ws_bytes // 4 + 8, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
body = api.body_id("attn_decode_bf16")
args = [q.data_ptr(), kv.data_ptr(), ws.data_ptr(), ctx | (chunk << 32) | (1 << 63), api.grid(chunks, 8)]
spans, phases = [], []
with api.Device() as dev:
    dev.start()
    for rep in range(30):
        aid = dev.submit(0, blocks, list(range(74)), 30, body, args)
        got = None
        while got is None:
            for c in dev.poll():
                got = c
        if rep >= 5:
            spans.append((got.dev_last_end_ns - got.dev_first_start_ns) / 1e3)
            st = ws[(8448 + 32 * chunks * 130 * 4) // 4:].cpu().view(torch.int64)[:4 * blocks].view(blocks, 4).double()
            t0 = st[:, 0].min()
            phases.append([(st[:, 0].max() - t0).item(), (st[:, 1] - st[:, 0]).median().item(),
                           (st[:, 2] - st[:, 1]).median().item(), (st[:, 3] - st[:, 2]).median().item(),
                           (st[:, 3] - st[:, 2]).max().item(), (st[:, 3].max() - t0).item()])
    dev.stop()
med = [statistics.median(p[i] for p in phases) / 1e3 for i in range(6)]
print(f"attn ctx {ctx} chunk {chunk} ({blocks} blocks): span p50 {statistics.median(spans):.2f} us | start skew {med[0]:.2f}"
      f" prologue {med[1]:.2f} compute+partials {med[2]:.2f} merge(p50) {med[3]:.2f} merge(max) {med[4]:.2f}"
      f" first start->last end {med[5]:.2f} us")
