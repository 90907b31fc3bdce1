"""MoE-layer training steps (default C2); the last one inside cudaProfilerStart/Stop so
`ncu --profile-from-start off` captures exactly one step (run with TED_GRAPH=0 so every
kernel is a plain launch)."""
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
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for i in range(steps):
    if i == steps - 1:  # ncu --profile-from-start off: only the last step is captured
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    L.step(a, y, da)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", L.loss())
L.close()
