"""Time ted_adam_step (the standalone AdamW kernel) on an expert-family-sized range."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_06318_b200 as ted  # noqa: E402

for n in (33_562_624, 64 << 20):
    f32 = [torch.zeros(n, device="cuda") for _ in range(3)]
    p = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    g = torch.randn(n, device="cuda").bfloat16()
    for i in range(3):
        ted.adam_step(*f32, p, g, 0, n, i + 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        ted.adam_step(*f32, p, g, 0, n, i + 4)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"n={n} {ms:.4f} ms {n * 26 / ms / 1e9:.1f} GB/s")
