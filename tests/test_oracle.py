"""Pin the CPU oracle (oracle/ted_oracle.c) to the reference: against the committed golden
vectors generated from the compiled reference (tests/golden/make_golden.py), and live
against oracle/_ref/libtedsim_ref.so when it is present.  CPU only."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

GOLD = np.load(O.HERE + "/../tests/golden/golden.npz")


def test_mix_seed_and_seeded_init_match_reference():
    tags = [str(t) for t in GOLD["mix_seed_tags"]]
    got = [O.mix_seed(s, t) for s in (1, 7) for t in tags]
    np.testing.assert_array_equal(np.array(got, np.uint64), GOLD["mix_seed_vals"])
    np.testing.assert_array_equal(O.seeded_init(4096, 12345, 0.5), GOLD["seeded_init_12345"])


def test_gate_known_answer_and_backward():
    """test_moe.cpp:133-195 values, produced by the reference."""
    a = np.array([[1, 0], [0, 1], [1, 1]], np.float64)
    w = np.array([[1.0, 0.2, -0.5], [0.1, 0.85, 0.3]])
    lg = np.empty((3, 3))
    ex = np.empty(3, np.int32)
    ch = np.empty(3)
    pr = np.empty((3, 3))
    O.lib().o_gate_forward(a, w, 3, 2, 3, lg, ex, ch, pr)
    np.testing.assert_array_equal(ex, GOLD["gate_kat_expert"])
    np.testing.assert_allclose(ch, GOLD["gate_kat_chosen"], rtol=1e-15)
    np.testing.assert_allclose(pr, GOLD["gate_kat_probs"], rtol=1e-15)
    dw, di = np.empty((2, 3)), np.empty((3, 2))
    O.lib().o_gate_backward(a, w, pr, ex, np.array([0.7, -1.3, 0.4]), 3, 2, 3, dw, di)
    np.testing.assert_allclose(dw, GOLD["gate_kat_dweight"], rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(di, GOLD["gate_kat_dinput"], rtol=1e-13, atol=1e-16)


def test_gate_tie_and_nan_rules():
    e, c, _ = O.gate_route_logits(np.array([[1.0, 1.0], [np.nan, 5.0], [1.0, np.nan]]))
    assert e.tolist() == [0, 0, 0]
    assert c[0] == 0.5


def test_gelu_matches_reference():
    x = GOLD["gelu_x"]
    np.testing.assert_allclose([O.lib().o_gelu(v) for v in x], GOLD["gelu_y"], rtol=1e-14,
                               atol=1e-16)
    np.testing.assert_allclose([O.lib().o_gelu_grad(v) for v in x], GOLD["gelu_dy"],
                               rtol=1e-14, atol=1e-16)


@pytest.mark.parametrize("tag", ["small", "c1ish"])
def test_moe_layer_matches_reference_sublayer(tag):
    S, n, h, f, E, seed = (int(v) for v in GOLD[f"moe_{tag}_dims"])
    inp = {k: GOLD[f"moe_{tag}_in_{k}"] for k in ("a", "wg", "w1", "b1", "w2", "b2")}
    o = O.moe_layer(S, n, h, f, E, 0.0, dy=GOLD[f"moe_{tag}_dy"], **inp)
    for k in ("y", "da", "dwg", "dw1", "db1", "dw2", "db2"):
        ref = GOLD[f"moe_{tag}_out_{k}"]
        np.testing.assert_allclose(o[k], ref, rtol=1e-9, atol=1e-13, err_msg=k)


def test_adam_matches_reference_bitwise_shapes():
    vals, grads = GOLD["adam_vals"], GOLD["adam_grads"]
    fam = vals.shape[0]
    master, m1, m2 = vals.copy(), np.zeros(fam), np.zeros(fam)
    out = np.zeros(fam)
    for s in range(3):
        peak = O.adam_step_owned(0, fam, s + 1, grads[s], master, m1, m2, out, tile_size=7)
    np.testing.assert_allclose(out, GOLD["adam_out"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(m1, GOLD["adam_m1"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(m2, GOLD["adam_m2"], rtol=1e-15, atol=0)
    assert peak == int(GOLD["adam_upcast"][0]) == 28


def test_shard_range_matches_reference():
    for total, parts, i, b, e in GOLD["shard_range"]:
        assert O.shard_range(int(total), int(parts), int(i)) == (b, e)


def test_capacity_semantics():
    rng = np.random.default_rng(0)
    ex = rng.integers(0, 8, 4096).astype(np.int32)
    # cf <= 0 -> reference semantics: everyone kept, slots are per-expert ranks
    slot, keep, kc = O.route_capacity(ex, 8, O.capacity(0.0, 4096, 8), T=2)
    assert keep.all() and kc.sum() == 4096
    for e in range(8):
        np.testing.assert_array_equal(slot[ex == e], np.arange((ex == e).sum()))
    cap = O.capacity(1.0, 4096, 8)
    assert cap == 512
    slot, keep, kc = O.route_capacity(ex, 8, cap, T=2)
    for e in range(8):
        assert keep[ex == e].sum() == min(cap, (ex == e).sum())
    assert kc.sum() == keep.sum()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_live_against_compiled_reference_random_sizes():
    R = O.ref()
    rng = np.random.default_rng(3)
    for (n, h, f, E) in [(97, 8, 32, 3), (256, 16, 64, 8), (64, 32, 128, 5)]:
        a = rng.standard_normal((n, h))
        wg = rng.standard_normal((h, E))
        w1 = rng.standard_normal((E, h, f)) / np.sqrt(h)
        b1 = rng.standard_normal((E, f)) * 0.1
        w2 = rng.standard_normal((E, f, h)) / np.sqrt(f)
        b2 = rng.standard_normal((E, h)) * 0.1
        dy = rng.standard_normal((n, h))
        r = {k: np.empty(s) for k, s in dict(y=(n, h), da=(n, h), dwg=(h, E), dw1=(E, h, f),
                                             db1=(E, f), dw2=(E, f, h), db2=(E, h)).items()}
        assert R.ref_moe_sublayer(n, h, f, E, a, wg, w1, b1, w2, b2, dy, r["y"], r["da"],
                                  r["dwg"], r["dw1"], r["db1"], r["dw2"], r["db2"], 1) == 0
        o = O.moe_layer(1, n, h, f, E, 0.0, a, wg, w1, b1, w2, b2, dy=dy)
        for k in r:
            np.testing.assert_allclose(o[k], r[k], rtol=1e-9, atol=1e-12, err_msg=k)
        ex = np.empty(n, np.int32)
        ch = np.empty(n)
        pr = np.empty((n, E))
        R.ref_gate_forward(a, wg, n, h, E, ex, ch, pr)
        np.testing.assert_array_equal(o["expert"], ex)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_live_adam_against_reference():
    R = O.ref()
    fam = 333
    vals = O.seeded_init(fam, 5, 0.5)
    grads = np.concatenate([O.seeded_init(fam, 50 + s, 0.5) for s in range(4)])
    out, ms, m1, m2 = (np.empty(fam) for _ in range(4))
    pk = C.c_uint64()
    for parts in (1, 3):
        for pos in range(parts):
            b, e = O.shard_range(fam, parts, pos)
            own = e - b
            rm, r1, r2 = np.empty(own), np.empty(own), np.empty(own)
            assert R.ref_adam(fam, vals, parts, pos, 1e-4, 0.9, 0.999, 1e-8, 0.01, 1, 5, 4, grads,
                              out, rm, r1, r2, C.byref(pk)) == 0
            master, o1, o2 = vals[b:e].copy(), np.zeros(own), np.zeros(own)
            for s in range(4):
                O.adam_step_owned(b, e, s + 1, grads[s * fam:(s + 1) * fam], master, o1, o2,
                                  tile_size=5)
            np.testing.assert_allclose(master, rm, rtol=1e-15)
