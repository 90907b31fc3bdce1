"""The MoE branch composed from the single-rank C-ABI operators (ted_gate_forward ->
ted_dispatch_forward -> ted_expert_ffn_forward -> ted_combine_forward, and back through
ted_combine_backward -> ted_expert_ffn_backward -> ted_gate_backward_dlogits) against the
fp64 oracle, the way SerialModel::forward_layer / backward_layer compose the reference's
free functions (moe.cpp:989-1064).  Same tolerances as the layer tests (rel-L2 <= 1e-2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from tests._util import from_dev, rel_l2, to_dev_bf16  # noqa: E402

TOL = 1e-2  # measured worst 4.5e-3 over the 1-GPU parity suite (tools: TED_TOL_REPORT)


@pytest.mark.parametrize("n,h,E,cf,seed", [(1024, 256, 4, 0.0, 1), (1024, 256, 4, 1.25, 11),
                                           (768, 512, 16, 1.0, 3)])
def test_operator_chain_matches_oracle(n, h, E, cf, seed):
    import paper_2303_06318_b200 as ted
    f = 4 * h
    inp = O.make_layer_inputs(1, n, h, f, E, seed, bf16=True)
    a = to_dev_bf16(inp["a"])
    wg = to_dev_bf16(inp["wg"])
    w1, b1 = to_dev_bf16(inp["w1"]), to_dev_bf16(inp["b1"])
    w2, b2 = to_dev_bf16(inp["w2"]), to_dev_bf16(inp["b2"])
    cap = ted.capacity(cf, n, E) if cf > 0 else 0

    expert, prob, probs, _ = ted.gate_forward(a, wg)
    x, pos, seg, kept, slot = ted.dispatch_forward(a, expert, E, cap)
    z, hh, fa = ted.expert_ffn_forward(x, seg, w1, b1, w2, b2)
    y = ted.combine_forward(fa, pos, prob)
    dy = (y.float() / n).bfloat16()  # the synthetic objective sum(y^2)/2N (moe.cpp:379-391)
    df, dl = ted.combine_backward(fa, pos, prob, probs, expert, dy, seg, kept)
    dx, dw1, db1, dw2, db2 = ted.expert_ffn_backward(x, z, hh, df, seg, w1, w2)
    dwg, da = ted.gate_backward_dlogits(a, wg, dl, dispatch_grad=dx, pos=pos)
    da_dispatch = ted.dispatch_backward(dx, pos, n)
    torch.cuda.synchronize()

    o = O.moe_layer(1, n, h, f, E, cf if cf > 0 else 0.0, **inp)
    np.testing.assert_array_equal(expert.cpu().numpy(), o["expert"])
    # capacity bookkeeping: the reference's append order, kept = slot < C
    sl, keep, counts = O.route_capacity(expert.cpu().numpy(), E, O.capacity(cf, n, E))
    np.testing.assert_array_equal(slot.cpu().numpy(), sl)
    np.testing.assert_array_equal(pos.cpu().numpy() >= 0, keep.astype(bool))
    np.testing.assert_array_equal(kept.cpu().numpy(), counts.reshape(-1))
    so = seg.cpu().numpy()
    assert so[0] == 0 and np.all(np.diff(so) % 128 == 0)
    assert rel_l2(from_dev(y), o["y"]) < TOL
    assert rel_l2(from_dev(da), o["da"]) < TOL
    assert rel_l2(from_dev(dwg), o["dwg"]) < TOL
    for e in range(E):
        if np.abs(o["dw1"][e]).sum() == 0:
            assert torch.count_nonzero(dw1[e]) == 0
            continue
        assert rel_l2(from_dev(dw1[e]), o["dw1"][e]) < TOL
        assert rel_l2(from_dev(db1[e]), o["db1"][e]) < TOL
        assert rel_l2(from_dev(dw2[e]), o["dw2"][e]) < TOL
        assert rel_l2(from_dev(db2[e]), o["db2"][e]) < TOL
    # the un-permute alone: dropped tokens get zero rows
    dd = from_dev(da_dispatch)
    p = pos.cpu().numpy()
    assert np.all(dd[p < 0] == 0)
    np.testing.assert_array_equal(dd[p >= 0], from_dev(dx)[p[p >= 0]])


def test_operator_chain_equals_the_layer():
    """The operators are the layer's kernels: the chain's forward output is bit-identical to
    ted_layer_forward on the same parameters and tokens."""
    import paper_2303_06318_b200 as ted
    n, h, E, cf, seed = 1024, 256, 8, 1.25, 5
    f = 4 * h
    inp = O.make_layer_inputs(1, n, h, f, E, seed, bf16=True)
    L = ted.MoeLayer(ted.MoeModelConfig(1, h, E, n, seed), ted.TedConfig(), capacity_factor=cf)
    L.set_param("layer0.gate.w", inp["wg"])
    for e in range(E):
        for k in ("w1", "b1", "w2", "b2"):
            L.set_param(f"layer0.expert{e}.{k}", inp[k][e])
    a = to_dev_bf16(inp["a"])
    y_layer = torch.empty_like(a)
    L.forward(a, y_layer)
    expert, prob, probs, _ = ted.gate_forward(a, to_dev_bf16(inp["wg"]))
    x, pos, seg, kept, _ = ted.dispatch_forward(a, expert, E, ted.capacity(cf, n, E))
    _, _, fa = ted.expert_ffn_forward(x, seg, to_dev_bf16(inp["w1"]), to_dev_bf16(inp["b1"]),
                                      to_dev_bf16(inp["w2"]), to_dev_bf16(inp["b2"]))
    y = ted.combine_forward(fa, pos, prob)
    torch.cuda.synchronize()
    assert torch.equal(y, y_layer)
    L.close()


def test_operator_config_errors_are_status_2():
    import paper_2303_06318_b200 as ted
    a = torch.zeros(64, 100, device="cuda", dtype=torch.bfloat16)  # hidden not a multiple of 8
    e = torch.zeros(64, device="cuda", dtype=torch.int32)
    with pytest.raises(ted.InvalidConfigError):
        ted.dispatch_forward(a, e, 4)
    x = torch.zeros(128, 200, device="cuda", dtype=torch.bfloat16)  # hidden % 256 != 0
    seg = torch.tensor([0, 128], device="cuda", dtype=torch.int32)
    w1 = torch.zeros(1, 200, 800, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ted.InvalidConfigError):
        ted.expert_ffn_forward(x, seg, w1, w1[:, 0], w1.transpose(1, 2), w1[:, :, 0])


def test_operator_edge_cases():
    """Empty and tiny inputs (the reference's tests cover empty shards and single tokens):
    no tokens, one token, one expert, every token dropped (capacity 1 with all tokens on one
    expert)."""
    import paper_2303_06318_b200 as ted
    h, E = 256, 4
    # one token, one expert
    a = torch.randn(1, h, device="cuda").bfloat16()
    e = torch.zeros(1, device="cuda", dtype=torch.int32)
    x, pos, seg, kept, slot = ted.dispatch_forward(a, e, 1)
    torch.cuda.synchronize()
    assert pos.item() == 0 and kept.item() == 1 and seg.tolist() == [0, 128]
    assert torch.equal(x[0], a[0]) and torch.count_nonzero(x[1:128]) == 0
    # 64 tokens on expert 2 with capacity 1: one kept, the rest dropped (pos -1, zero y)
    a = torch.randn(64, h, device="cuda").bfloat16()
    e = torch.full((64,), 2, device="cuda", dtype=torch.int32)
    x, pos, seg, kept, slot = ted.dispatch_forward(a, e, E, cap=1)
    torch.cuda.synchronize()
    assert kept.tolist() == [0, 0, 1, 0] and int((pos >= 0).sum()) == 1 and pos[0].item() == 0
    assert slot.tolist() == list(range(64))
    prob = torch.rand(64, device="cuda")
    y = ted.combine_forward(x, pos, prob)
    torch.cuda.synchronize()
    assert torch.count_nonzero(y[1:]) == 0
    da = ted.dispatch_backward(x, pos, 64)
    torch.cuda.synchronize()
    assert torch.count_nonzero(da[1:]) == 0 and torch.equal(da[0], x[0])
    # no tokens: nothing to do, no error
    a0 = torch.empty(0, h, device="cuda").bfloat16()
    e0 = torch.empty(0, device="cuda", dtype=torch.int32)
    x0, pos0, seg0, kept0, _ = ted.dispatch_forward(a0, e0, E)
    torch.cuda.synchronize()
    assert kept0.tolist() == [0] * E and seg0.tolist() == [0] * (E + 1)
