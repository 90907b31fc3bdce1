"""Tiled AdamW on the GPU (ted_adam_step) vs OptimizerShard::step_owned.

Reference tests restated: SingleElementStepMatchesHandRolledAdamW (test_optimizer.cpp:59-75),
TilingAtAnySizeIsBitwiseIdenticalToUntiled (:77-99), UpcastPeakIsTileBound (:101-127),
LargeFamilyUpcastPeakIsCappedByTileSize (:129-143), ShardedStepsReassemble (:145-173).
Tolerance: fp32 master/moments vs fp64 reference math rel <= 1e-6 (atol 1e-9)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402


def _ted():
    import paper_2303_06318_b200 as ted
    return ted


def _run(vals, grads, begin, end, tile, steps=None):
    ted = _ted()
    fam = vals.shape[0]
    owned = end - begin
    master = torch.from_numpy(vals[begin:end].astype(np.float32)).cuda()
    m1 = torch.zeros(owned, device="cuda")
    m2 = torch.zeros(owned, device="cuda")
    param = torch.from_numpy(vals.astype(np.float32)).cuda().bfloat16()
    peak = 0
    for s, g in enumerate(grads):
        gd = torch.from_numpy(g.astype(np.float32)).cuda().bfloat16()
        peak = ted.adam_step(master, m1, m2, param, gd, begin, end, s + 1,
                             tiles=ted.TileConfig(True, tile))
    torch.cuda.synchronize()
    return (master.cpu().numpy().astype(np.float64), m1.cpu().numpy(), m2.cpu().numpy(),
            param.float().cpu().numpy(), peak)


def test_single_element_matches_hand_rolled_adamw():
    vals = np.array([1.0])
    master, _, _, _, _ = _run(vals, [np.array([0.5])], 0, 1, 1_800_000)
    lr, b1, b2, eps, wd = 1e-4, 0.9, 0.999, 1e-8, 0.01
    g = 0.5
    mhat = (1 - b1) * g / (1 - b1)
    vhat = (1 - b2) * g * g / (1 - b2)
    expect = 1.0 - lr * (mhat / (np.sqrt(vhat) + eps) + wd * 1.0)
    assert abs(master[0] - expect) <= 1e-7


@pytest.mark.parametrize("tile", [1, 7, 1_800_000])
def test_three_steps_match_oracle_and_golden(tile):
    gold = np.load(O.HERE + "/../tests/golden/golden.npz")
    vals, grads = gold["adam_vals"], gold["adam_grads"]
    gb = [O.bf16_round(g) for g in grads]  # the GPU consumes bf16 gradients
    master, m1, m2, param, peak = _run(vals, gb, 0, vals.shape[0], tile)
    om, o1, o2 = vals.copy(), np.zeros_like(vals), np.zeros_like(vals)
    for s, g in enumerate(gb):
        opeak = O.adam_step_owned(0, vals.shape[0], s + 1, g, om, o1, o2, tile_size=tile)
    np.testing.assert_allclose(master, om, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(m1, o1, rtol=1e-5, atol=2e-8)  # fp32 cancellation
    np.testing.assert_allclose(m2, o2, rtol=1e-5, atol=1e-10)
    assert peak == opeak
    if tile == 7:
        assert peak == int(gold["adam_upcast"][0])
        # against the reference's own output on unrounded gradients
        np.testing.assert_allclose(master, gold["adam_out"], rtol=0, atol=2e-6)
    np.testing.assert_array_equal(param, O.bf16_round(master))


def test_sharded_steps_reassemble_to_replicated():
    vals = O.seeded_init(101, 51, 0.5)
    grads = [O.bf16_round(O.seeded_init(101, 200 + s, 0.5)) for s in range(3)]
    whole = _run(vals, grads, 0, 101, 1_800_000)[0]
    parts = []
    for i in range(4):
        b, e = O.shard_range(101, 4, i)
        parts.append(_run(vals, grads, b, e, 1_800_000)[0])
    np.testing.assert_array_equal(np.concatenate(parts), whole)


def test_large_family_upcast_peak_capped_by_tile():
    n = 5_000_000
    vals = np.full(n, 0.125)
    grads = [np.full(n, 0.25)]
    master, _, _, _, peak = _run(vals, grads, 0, n, 1_800_000)
    assert peak == 7_200_000
    assert master[0] == master[1_800_000] == master[n - 1]
