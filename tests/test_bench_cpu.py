"""bench.py's host-side bookkeeping on CPU: the workload per GPU count (BASELINE configs,
SURVEY §8(d) C3 = TP2 x EP4 on 8 GPUs), the roofline arithmetic (26 B per parameter + 2 B
per operand element for the fused wgrad + AdamW launch; 2 rows h f/T FLOP per expert GEMM)
and the parity verdict."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("n,tp,ep", [(1, 1, 1), (2, 2, 1), (4, 2, 2), (8, 2, 4)])
def test_workload_layouts(bench, n, tp, ep):
    w = bench.workload(n, dtd=True)
    assert (w["tp"], w["ep"]) == (tp, ep)
    assert (w["hidden"], w["experts"], w["tokens"], w["cf"]) == (4096, 16, 32768, 1.25)
    assert w["dtd"] == (tp > 1)  # DTD needs a TP group
    assert w["name"] == f"C3 MoE layer TP={tp}xEP={ep}"
    c2 = bench.workload(1, dtd=False, which="c2")
    assert (c2["hidden"], c2["experts"], c2["tokens"]) == (1024, 8, 16384)


def test_roofline_arithmetic(bench):
    w = bench.workload(1, dtd=False)
    h, f, E = 4096, 16384, 16
    kept = [2048] * E
    rows = 33792  # assembled rows incl. the 128-row padding of each group
    stages = {"gemm1_fwd": 4.0, "gemm2_fwd": 3.5, "dgrad2": 3.7, "dgrad1": 3.6,
              "wgrad1": 6.5, "wgrad2": 6.7}
    stats = {"kept_per_expert": kept, "asm_rows": rows}
    roof, extra = bench.rooflines(w, stages, stats, T=1, P=1, D=1, world=1)
    pk = bench.peaks()
    params = E * h * f
    wg_bytes = 26.0 * params + 2.0 * rows * (h + f)
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s"
    assert roof["bytes_per_launch"] == pytest.approx(wg_bytes)
    assert roof["ms_per_launch"] == pytest.approx(6.6)
    assert roof["achieved"] == pytest.approx(wg_bytes / 6.6e-3 / 1e9)
    assert roof["frac"] == pytest.approx(roof["achieved"] / pk["hbm_gbs"])
    g = extra["roofline_gemm"]
    flops = 8.0 * sum(kept) * h * f  # four GEMMs of 2 rows h f each
    assert g["flops_per_launch"] == pytest.approx(flops / 4)
    assert g["achieved"] == pytest.approx(flops / (14.8e-3) / 1e12)
    assert g["frac"] == pytest.approx(g["achieved"] / pk["bf16_tflops_sustained"])
    # ZeRO-sharded expert family (D > 1): AdamW is not fused, only the GEMM roofline
    roof2, extra2 = bench.rooflines(w, stages, stats, T=1, P=1, D=2, world=1)
    assert roof2["bound"] == "tensor" and extra2 == {}


def test_parity_verdict(bench):
    good = {"routing_bit_exact_all_tokens": True, "y_rel_l2_sampled": 2e-3,
            "y_err_vs_terms": 3e-5, "condition": 70.0, "tokens_sampled": 8}
    v = bench.parity_verdict(good, dict(good, y_rel_l2_sampled=1.9e-3))
    assert v["pass"] and v["tolerance"] == 1e-2
    assert not bench.parity_verdict(good, dict(good, y_rel_l2_sampled=2e-2))["pass"]
    assert not bench.parity_verdict(dict(good, routing_bit_exact_all_tokens=False), good)["pass"]
