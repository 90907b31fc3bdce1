"""Time ted_gate_forward (transpose + tcgen05 gate) at a given shape with CUDA events.
usage: python tools/gate_time.py [n h E reps]  -> prints us/call and the HBM GB/s of the
token read (n*h*2 B) + logits/probs/expert/prob writes."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_06318_b200 as ted  # noqa: E402

n, h, E, reps = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (32768, 4096, 16, 50)
g = torch.Generator(device="cuda")
g.manual_seed(1)
a = torch.randn(n, h, device="cuda", generator=g).bfloat16()
wg = (torch.randn(h, E, device="cuda", generator=g) * 0.02).bfloat16()
lg = torch.empty(n, E, device="cuda")
for _ in range(3):
    ted.gate_forward(a, wg, logits=lg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ted.gate_forward(a, wg, logits=lg)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
byts = n * h * 2 + n * (8 * E + 8)
print(f"gate n={n} h={h} E={E}: {us:.1f} us/call, {byts / us / 1e3:.0f} GB/s")
