"""One batch-mode launch of the dispatcher's worker kernel executing a
full-width atomized STREAM kernel (the bench's roofline workload), for ncu:

  ncu --set full --clock-control none --import-source on -k regex:k_worker \
      -c 1 -o gpurun_out/prof python tools/ncu_batch.py

Batch mode stages every atom before the launch, so the kernel is a single
self-contained launch that ncu can replay."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_15465_b200 import api  # noqa: E402

words = int(sys.argv[1]) if len(sys.argv) > 1 else 550000  # bench saturation shape (> L2 with 256 chunks)
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 2160
src = torch.randint(-2**31, 2**31 - 1, (256 * words,), dtype=torch.int32, device="cuda")
dst = torch.empty_like(src)
torch.cuda.synchronize()
per = blocks // 16
descs = [api.Device.desc(i * per, (i + 1) * per, range(74), 20, api.GPUOS_BODY_STREAM,
                         [src.data_ptr(), dst.data_ptr(), words, 7, 256]) for i in range(16)]
with api.Device() as dev:
    for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
        ms = dev.run_batch(descs)
        while dev.in_flight():
            dev.poll()
        print(f"batch {blocks} blocks x {words * 8} B: {ms:.3f} ms, "
              f"{blocks * words * 8 / ms / 1e6:.0f} GB/s", flush=True)
