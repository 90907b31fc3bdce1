"""Gate / routing parity on the GPU (ted_gate_forward, ted_gate_route_logits, ted_route,
ted_gate_backward) against the CPU oracle (oracle/ted_oracle.c, itself pinned to the
reference in tests/test_oracle.py).

Bars: routing indices, capacity slots, keep masks and kept counts
are BIT-EXACT given identical fp32 logits; chosen/softmax probabilities rel <= 1e-6 vs
fp64 on the same fp32 logits; GPU-computed logits vs fp64 logits on the same bf16
inputs rel <= 1e-5; gate-backward bf16 outputs rel-L2 <= 1e-2."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402  (test infrastructure: the checker)
from tests._util import rel_l2  # noqa: E402


def _ted():
    import paper_2303_06318_b200 as ted
    return ted


def test_gate_known_answer_test_moe_133():
    """test_moe.cpp:133-153 (Gate.PicksArgmaxAndNormalizesProbs) on exact fp32 logits."""
    ted = _ted()
    a = np.array([[1, 0], [0, 1], [1, 1]], np.float64)
    w = np.array([[1.0, 0.2, -0.5], [0.1, 0.85, 0.3]])
    L = (a @ w).astype(np.float32)
    expert, prob, probs = ted.gate_route_logits(torch.from_numpy(L).cuda())
    assert expert.cpu().tolist() == [0, 1, 0]
    gold = np.load(O.HERE + "/../tests/golden/golden.npz")
    np.testing.assert_allclose(prob.cpu().numpy(), gold["gate_kat_chosen"], rtol=1e-6)
    np.testing.assert_allclose(probs.cpu().numpy().sum(1), 1.0, rtol=1e-6)


def test_gate_tie_breaks_toward_lowest_index_test_moe_155():
    ted = _ted()
    L = torch.tensor([[1.0, 1.0]], device="cuda")
    expert, prob, _ = ted.gate_route_logits(L)
    assert expert.item() == 0 and abs(prob.item() - 0.5) < 1e-7


@pytest.mark.parametrize("E", [2, 4, 8, 16, 32, 33, 64])
def test_route_logits_bit_exact_with_ties_and_nans(E):
    ted = _ted()
    rng = np.random.default_rng(E)
    n = 4096 + 77
    L = rng.integers(-3, 4, size=(n, E)).astype(np.float32) * 0.5  # many exact ties
    L[5, 0] = np.nan          # NaN at j=0 pins expert 0 (moe.cpp:167-174)
    L[6, E - 1] = np.nan      # NaN elsewhere never wins
    L[7, :] = -np.inf if E > 1 else L[7, :]
    expert, prob, probs = ted.gate_route_logits(torch.from_numpy(L).cuda())
    oe, oc, op = O.gate_route_logits(L.astype(np.float64))
    np.testing.assert_array_equal(expert.cpu().numpy(), oe)
    ok = ~np.isnan(oc)
    np.testing.assert_allclose(prob.cpu().numpy()[ok], oc[ok], rtol=1e-6)
    okp = ~np.isnan(op)
    np.testing.assert_allclose(probs.cpu().numpy()[okp], op[okp], rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("n,h,E", [(2048, 256, 4), (16384, 1024, 8), (3000, 512, 16),
                                   (1024, 4096, 16), (777, 256, 64)])
def test_gate_forward_matches_oracle(n, h, E):
    ted = _ted()
    rng = np.random.default_rng(n + E)
    a = O.bf16_round(rng.standard_normal((n, h)))
    wg = O.bf16_round(rng.standard_normal((h, E)) / np.sqrt(h))
    ad = torch.from_numpy(a.astype(np.float32)).cuda().bfloat16()
    wd = torch.from_numpy(wg.astype(np.float32)).cuda().bfloat16()
    expert, prob, probs, logits = ted.gate_forward(ad, wd)
    Lg = logits.cpu().numpy().astype(np.float64)
    Lo = a @ wg
    assert np.max(np.abs(Lg - Lo)) <= 1e-5 * max(1.0, np.max(np.abs(Lo)))
    # routing is bit-exact given the GPU's own fp32 logits
    oe, oc, op = O.gate_route_logits(Lg)
    np.testing.assert_array_equal(expert.cpu().numpy(), oe)
    np.testing.assert_allclose(prob.cpu().numpy(), oc, rtol=1e-6)
    np.testing.assert_allclose(probs.cpu().numpy(), op, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("cf", [0.0, 1.0, 1.25, 1.5, 2.0])
@pytest.mark.parametrize("T", [1, 2, 4])
@pytest.mark.parametrize("E,skew", [(8, 0.0), (16, 1.5), (64, 3.0)])
def test_capacity_slots_bit_exact(cf, T, E, skew):
    """Routing stress (C5): Zipf-biased logits, capacity factor sweep, DTD chunking."""
    ted = _ted()
    rng = np.random.default_rng(int(cf * 100) + T + E)
    n = 8192
    bias = skew * (1.0 / np.arange(1, E + 1) ** 1.2)
    L = (rng.standard_normal((n, E)) + bias).astype(np.float32)
    expert, _, _ = ted.gate_route_logits(torch.from_numpy(L).cuda())
    ex = expert.cpu().numpy()
    cap = ted.capacity(cf, n, E)
    slot, keep, kc = ted.route(expert, E, cap, T)
    os_, ok, okc = O.route_capacity(ex, E, O.capacity(cf, n, E), T)
    np.testing.assert_array_equal(slot.cpu().numpy(), os_)
    np.testing.assert_array_equal(keep.cpu().numpy(), ok)
    np.testing.assert_array_equal(kc.cpu().numpy(), okc)


def test_gate_backward_matches_oracle():
    ted = _ted()
    rng = np.random.default_rng(5)
    n, h, E = 4096, 512, 8
    a = O.bf16_round(rng.standard_normal((n, h)))
    wg = O.bf16_round(rng.standard_normal((h, E)) / np.sqrt(h))
    ad = torch.from_numpy(a.astype(np.float32)).cuda().bfloat16()
    wd = torch.from_numpy(wg.astype(np.float32)).cuda().bfloat16()
    expert, prob, probs, logits = ted.gate_forward(ad, wd)
    dchosen = rng.standard_normal(n).astype(np.float32)
    dwg, dinput = ted.gate_backward(ad, wd, probs, expert, torch.from_numpy(dchosen).cuda())
    dwo = np.empty((h, E))
    dio = np.empty((n, h))
    O.lib().o_gate_backward(a, wg, probs.cpu().numpy().astype(np.float64),
                            expert.cpu().numpy(), dchosen.astype(np.float64), n, h, E, dwo, dio)
    assert rel_l2(dwg.float().cpu().numpy(), dwo) < 1e-2
    assert rel_l2(dinput.float().cpu().numpy(), dio) < 1e-2


def test_placement_verdict_kernel():
    """The DTD placement verdict (moe.cpp:537-556) computed on the device from a dispatch's
    row records: the right chunk passes, the chunk corrupt_drop sends (test_moe.cpp:388-414)
    fails, and the sticky verdict stays failed."""
    import paper_2303_06318_b200 as ted
    rng = np.random.default_rng(4)
    n, T = 1024, 2
    chunk = n // T
    home = np.where(rng.random(n) < 0.8, np.arange(n), -1).astype(np.int32)  # 20 % dropped

    def sent_by(c):
        s = np.full(n, -1, np.int32)
        idx = [k for k in range(c * chunk, (c + 1) * chunk) if home[k] >= 0]
        s[idx] = np.arange(len(idx), dtype=np.int32)
        return s

    ph = torch.from_numpy(home).cuda()
    v = torch.ones(2, dtype=torch.int32, device="cuda")
    ted.placement_verdict(torch.from_numpy(sent_by(1)).cuda(), ph, T, 1, v)
    assert v.tolist() == [1, 1]
    ted.placement_verdict(torch.from_numpy(sent_by(0)).cuda(), ph, T, 1, v)  # wrong chunk
    assert v.tolist() == [0, 0]
    ted.placement_verdict(torch.from_numpy(sent_by(1)).cuda(), ph, T, 1, v)
    assert v.tolist() == [1, 0]  # this forward fine, the rank's record stays failed
    all_kept = np.where(home >= 0, home, -1).astype(np.int32)  # no DTD: every kept token
    ted.placement_verdict(torch.from_numpy(all_kept).cuda(), ph, 1, -1, v)
    assert v[0].item() == 1
    miss = all_kept.copy()
    miss[np.nonzero(home >= 0)[0][5]] = -1  # a kept token that was never sent
    ted.placement_verdict(torch.from_numpy(miss).cuda(), ph, 1, -1, v)
    assert v[0].item() == 0
