"""One C2 MoE-layer training step after 3 warm-up steps (for ncu captures: run with
TED_GRAPH=0 so every kernel is a plain launch)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_06318_b200 as ted  # noqa: E402

# argv: [steps] [tokens hidden experts]  (default C2: 16384 1024 8)
n, h, E = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (16384, 1024, 8)
L = ted.MoeLayer(ted.MoeModelConfig(1, h, E, n, 0), ted.TedConfig(), capacity_factor=1.25)
L.init_params(1234)
g = torch.Generator(device="cuda")
g.manual_seed(1000)
a = torch.randn(n, h, device="cuda", generator=g).bfloat16()
y, da = torch.empty_like(a), torch.empty_like(a)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    L.step(a, y, da)
torch.cuda.synchronize()
print("ok", L.loss())
L.close()
