"""Generate tests/golden/golden.npz from the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/libtedsim_ref.so (the unmodified tedsim sources + ref_shim.cpp)
and records the reference's outputs on small seeded inputs, so the parity suite can pin
the oracle (and, through it, the GPU path) on machines without /root/reference.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "golden.npz")


def main():
    O.build(ref=True)
    R = O.ref()
    g = {}
    # tensor.cpp: mix_seed / seeded_init
    tags = ["batch", "layer0.gate.w", "layer0.expert3.w1", "x"]
    g["mix_seed_tags"] = np.array(tags)
    g["mix_seed_vals"] = np.array([R.ref_mix_seed(s, t.encode()) for s in (1, 7) for t in tags],
                                  np.uint64)
    x = np.empty(4096)
    R.ref_seeded_init(x, 4096, 12345, 0.5)
    g["seeded_init_12345"] = x
    # test_moe.cpp:133-153 gate KAT and :155-161 tie
    a = np.array([[1, 0], [0, 1], [1, 1]], np.float64)
    w = np.array([[1.0, 0.2, -0.5], [0.1, 0.85, 0.3]])
    ex = np.empty(3, np.int32)
    ch = np.empty(3)
    pr = np.empty((3, 3))
    assert R.ref_gate_forward(a, w, 3, 2, 3, ex, ch, pr) == 0
    g["gate_kat_expert"], g["gate_kat_chosen"], g["gate_kat_probs"] = ex, ch, pr
    dc = np.array([0.7, -1.3, 0.4])
    dw = np.empty((2, 3))
    di = np.empty((3, 2))
    assert R.ref_gate_backward(a, w, 3, 2, 3, dc, dw, di) == 0
    g["gate_kat_dweight"], g["gate_kat_dinput"] = dw, di
    # gelu (nn.cpp:92-106)
    xs = np.linspace(-4, 4, 81)
    g["gelu_x"] = xs
    g["gelu_y"] = np.array([R.ref_gelu(v) for v in xs])
    g["gelu_dy"] = np.array([R.ref_gelu_grad(v) for v in xs])
    # MoE sublayer on seeded, bf16-rounded inputs (composed from the reference's public
    # free functions: gate_forward, linear_*, gelu_*, gate_backward)
    for tag, (S, n, h, f, E, seed) in {"small": (2, 64, 16, 64, 4, 7),
                                       "c1ish": (2, 128, 32, 128, 4, 1)}.items():
        inp = O.make_layer_inputs(S, n, h, f, E, seed, bf16=True)
        N = S * n
        dy = O.bf16_round(O.seeded_init(N * h, 99, 0.01).reshape(N, h))
        r = {k: np.empty(s) for k, s in dict(y=(N, h), da=(N, h), dwg=(h, E), dw1=(E, h, f),
                                             db1=(E, f), dw2=(E, f, h), db2=(E, h)).items()}
        assert R.ref_moe_sublayer(N, h, f, E, inp["a"], inp["wg"], inp["w1"], inp["b1"],
                                  inp["w2"], inp["b2"], dy, r["y"], r["da"], r["dwg"], r["dw1"],
                                  r["db1"], r["dw2"], r["db2"], 1) == 0
        for k, v in inp.items():
            g[f"moe_{tag}_in_{k}"] = v
        g[f"moe_{tag}_dy"] = dy
        for k, v in r.items():
            g[f"moe_{tag}_out_{k}"] = v
        g[f"moe_{tag}_dims"] = np.array([S, n, h, f, E, seed])
    # optimizer.cpp: AdamW KAT (test_optimizer.cpp:59-75) + 3 tiled steps
    fam = 1000
    vals = O.seeded_init(fam, 41, 0.5)
    grads = np.concatenate([O.seeded_init(fam, 100 + s, 0.5) for s in range(3)])
    out = np.empty(fam)
    ms, m1, m2 = np.empty(fam), np.empty(fam), np.empty(fam)
    peak = np.zeros(1, np.uint64)
    import ctypes as C
    pk = C.c_uint64()
    assert R.ref_adam(fam, vals, 1, 0, 1e-4, 0.9, 0.999, 1e-8, 0.01, 1, 7, 3, grads, out, ms,
                      m1, m2, C.byref(pk)) == 0
    g["adam_vals"], g["adam_grads"], g["adam_out"] = vals, grads.reshape(3, fam), out
    g["adam_m1"], g["adam_m2"], g["adam_upcast"] = m1, m2, np.array([pk.value], np.uint64)
    # shard_range (optimizer.cpp:12-28)
    sr = []
    for total in (0, 1, 7, 64, 1000, 101):
        for parts in (1, 2, 3, 7, 16):
            for i in range(parts):
                b, e = C.c_int64(), C.c_int64()
                R.ref_shard_range(total, parts, i, C.byref(b), C.byref(e))
                sr.append((total, parts, i, b.value, e.value))
    g["shard_range"] = np.array(sr, np.int64)
    # derive_config (topology.cpp:10-37)
    dcfg = []
    for world, tp, ex in [(8, 2, 4), (8, 2, 2), (4, 2, 2), (8, 1, 8), (16, 2, 4), (8, 2, 16),
                          (1, 1, 8), (4, 2, 4)]:
        o5 = np.zeros(5, np.int32)
        rc = R.ref_derive_config(world, tp, ex, o5)
        dcfg.append([world, tp, ex, rc] + list(o5))
    g["derive_config"] = np.array(dcfg, np.int64)
    # predict_comm_volume (cost_model.cpp:346-416): fwd A2A / AG / AR payload bytes
    pc = []
    for (world, tp, ex, h, n) in [(4, 2, 2, 256, 1024), (8, 2, 4, 4096, 8192)]:
        for dtd in (0, 1):
            o3 = np.zeros(3, np.uint64)
            assert R.ref_predict_comm(1, h, ex, n, world, tp, dtd, 0, 0, o3) == 0
            pc.append([world, tp, ex, h, n, dtd] + [int(v) for v in o3])
    g["predict_comm"] = np.array(pc, np.int64)
    # SerialModel losses (moe.cpp:899-1121), 2 layers, 3 steps
    losses = np.empty(3)
    assert R.ref_serial_step(2, 8, 2, 8, 7, 2, 3, losses) == 0
    g["serial_losses"] = losses
    # SerialModel losses for the model-stack parity tests (layers, h, E, n, seed, shards)
    stacks = [(2, 256, 4, 128, 1, 1), (4, 256, 4, 128, 5, 1), (2, 256, 4, 128, 3, 2),
              (2, 256, 4, 128, 3, 1)]
    # the reference's verify sweep shape (harness.cpp:254-278: hidden 8, 8 tokens per
    # shard, 1 layer) for every (experts, data shards) a 1-4 GPU layout produces, and a
    # 2-layer variant
    stacks += [(1, 8, e, 8, 1, s) for e in (1, 2, 4) for s in (1, 2, 4)]
    stacks += [(2, 8, 2, 8, 7, 1), (2, 8, 2, 8, 7, 2)]
    sl = []
    for (L_, h_, E_, n_, s_, S_) in stacks:
        ls = np.empty(3)
        assert R.ref_serial_step(L_, h_, E_, n_, s_, S_, 3, ls) == 0
        sl.append([L_, h_, E_, n_, s_, S_] + list(ls))
    g["stack_serial_losses"] = np.array(sl, np.float64)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, len(g), "arrays")


if __name__ == "__main__":
    main()
