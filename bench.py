#!/usr/bin/env python
"""bench.py -- MoE-layer tokens/s (fwd + bwd + tiled AdamW step) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--dtd 0|1]
                  [--workload c3|c2|c4] [--layers L] [--no-cpu-baseline] [--no-dtd-compare]

Workload (all N): configs[2] of BASELINE.json, the layer the north-star target is quoted on
-- d=4096, ffn=16384, 16 experts top-1, 32768 tokens in total, capacity factor 1.25 --
partitioned TP=2 x EP=N/2 (N=1: TP=EP=1, all 16 experts on one GPU; N=8: exactly TP=2 x
EP=4, 4 data shards of 8192 tokens).  Total work is fixed, so the 1/2/4/8 series is strong
scaling of one layer.  DTD on by default for TP>1 (--dtd 0 for the off arm); at N>1 the
line also carries a DTD on/off comparison measured in the same run.  At N=1 the line adds
configs[1] (d=1024, ffn=4096, 8 experts, 16384 tokens) as `c2_single_gpu`
(--workload c2 makes it the headline).

A step = one pass of the MoE layer over one batch: gate, capacity routing, dispatch,
[EP all-to-all, DTD all-gathers, TP all-reduce], expert FFN fwd (tcgen05 GEMMs), combine,
synthetic loss sum(y^2)/2N, the whole backward, gradient sync and AdamW.
`value` times K steps with inputs resident in HBM (CUDA events, max over ranks);
`e2e` repeats it through the public API with the step's tokens copied from pinned host
memory (double-buffered on a copy stream: step i+1's copy runs under step i) and the loss
read back every step.  `roofline` is the dominant kernel (the wgrad GEMMs with the fused
AdamW, HBM-bound); `roofline_gemm` the forward / dgrad GEMMs against the tensor peak.
--workload c4 runs configs[3] instead: a layer stack (attention stand-in + MoE / dense FFN)
through the Trainer-level model API, TP=2 x EP=2 x DP=N/4, ZeRO-1.

--impl reference times the reference's own CPU implementation (oracle/_ref/
libtedsim_ref.so, the unmodified tedsim sources) on a bounded token sample of the same
workload with one rank-thread per expert, the reference's own concurrency model.
"""
from __future__ import annotations

import argparse
import glob
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "MoE-layer tokens/sec fwd+bwd at 1/2/4/8 B200; all-to-all bytes & time w/ DTD"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


def workload(n_gpus: int, dtd: bool, which: str = "c3"):
    if which == "c2":
        return dict(name="C2 single-GPU MoE layer", hidden=1024, experts=8, tokens=16384,
                    tp=1, ep=1, cf=1.25, dtd=False)
    tp = 2 if n_gpus % 2 == 0 else 1
    ep = n_gpus // tp
    return dict(name=f"C3 MoE layer TP={tp}xEP={ep}", hidden=4096, experts=16,
                tokens=32768, tp=tp, ep=ep, cf=1.25, dtd=dtd and tp > 1)


def rooflines(w, stage_avg_ms, stats, T, P, D, world):
    """(roofline, extra) of the step's dominant kernels from the per-stage CUDA-event times.
    With the expert family unsharded (D = 1) AdamW runs inside the two wgrad GEMMs and that
    kernel dominates the step (HBM-bound on the optimizer state: 26 B per parameter + the
    operands once); the four forward / dgrad GEMMs are reported beside it against the
    sustained tensor-core peak (algorithmic FLOPs 2 x rows x h x f/T per GEMM).  `traffic`
    comes from a committed ncu --set full capture of the same workload (profiles/)."""
    pk = peaks()

    def st(k):
        return stage_avg_ms.get(k, 0.0)
    Eloc = max(1, w["experts"] // P)
    kept_rows = sum(stats["kept_per_expert"][:Eloc])
    f_t = 4 * w["hidden"] // T
    h_ = w["hidden"]
    tc_ms = sum(st(k) for k in ["gemm1_fwd", "gemm2_fwd", "dgrad2", "dgrad1"])
    tc_flops = 8.0 * kept_rows * h_ * f_t
    tc_ach = tc_flops / (tc_ms / 1e3) / 1e12 if tc_ms > 0 else None
    peak_tc = pk["bf16_tflops_sustained"]
    tj = None
    for tp in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_gemm_traffic*.json"))):
        with open(tp) as f:
            cand = json.load(f)
        if cand.get("workload") == w["name"] and cand.get("n_gpus", 1) == world:
            tj = cand
    roof_tc = {"bound": "tensor", "kernel": "expert FFN fwd + dgrad tcgen05 GEMMs (4/step)",
               "achieved": tc_ach, "peak": peak_tc, "unit": "TFLOP/s",
               "frac": (tc_ach / peak_tc) if tc_ach else None,
               "traffic": tj.get("tc_per_launch") if tj else None,
               "flops_per_launch": tc_flops / 4, "ms_per_launch": tc_ms / 4,
               "peak_source": pk["source"] + " bf16_tflops_sustained"}
    if D != 1:
        return roof_tc, {}
    wg_ms = (st("wgrad1") + st("wgrad2")) / 2
    params = Eloc * h_ * f_t
    rows = int(stats["asm_rows"])
    wg_bytes = 26.0 * params + 2.0 * rows * (h_ + f_t)
    wg_ach = wg_bytes / (wg_ms / 1e3) / 1e9 if wg_ms > 0 else None
    roofline = {"bound": "hbm", "kernel": "wgrad GEMM + fused AdamW (2/step)",
                "achieved": wg_ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": (wg_ach / pk["hbm_gbs"]) if wg_ach else None,
                "traffic": tj.get("wgrad_per_launch") if tj else None,
                "bytes_per_launch": wg_bytes, "ms_per_launch": wg_ms,
                "unit_work": "26 B per parameter + 2 B per operand element",
                "peak_source": pk["source"] + " hbm_gbs (copy)"}
    return roofline, {"roofline_gemm": roof_tc}


def sampled_parity(L, a, w, T, P, tokens=8, seed=0):
    """A parity check at the benched configuration (one GPU): one forward on the benched
    tokens, then, in fp64 numpy on the layer's current bf16 parameters (MoeRank's MoE
    branch, moe.cpp:435-563, restated here -- bench.py does not run the test oracle on this
    path): the routing of EVERY token must equal the argmax of the GPU's own fp32 logits
    (lowest index on ties), and y of `tokens` sampled kept tokens must match
    p * (gelu(a W1_e + b1_e) W2_e + b2_e) (bf16 storage of X, Z, H, F; fp32 accumulation).

    Two error figures: `y_rel_l2_sampled` = ||y - ref|| / ||ref||, and `y_err_vs_terms` =
    ||y - ref|| / ||p (|H| |W2_e| + |b2_e|)||, the error against the magnitude of the terms
    summed into y; `condition` = ||terms|| / ||ref|| (about sqrt(ffn) for random weights;
    thousands on the batch the layer was trained on, where y cancels)."""
    import numpy as np
    import torch
    y = torch.empty_like(a)
    L.forward(a, y)
    torch.cuda.synchronize()
    r = L.routing()
    lg = r["logits"]
    exp_route = np.argmax(lg, axis=1)  # numpy argmax: first maximum = lowest index
    routing_ok = bool(np.array_equal(exp_route, r["expert"]))
    h, f = w["hidden"], 4 * w["hidden"]
    kept = np.nonzero(r["pos_home"] >= 0)[0]
    rng = np.random.default_rng(seed)
    pick = rng.choice(kept, size=min(tokens, len(kept)), replace=False)
    av = a.float().cpu().numpy().astype(np.float64)
    yv = y.float().cpu().numpy().astype(np.float64)

    def bf16(x):
        return torch.from_numpy(np.asarray(x, np.float32)).bfloat16().float().numpy().astype(np.float64)
    cache, num, den, scl = {}, 0.0, 0.0, 0.0
    for k in sorted(pick, key=lambda k: r["expert"][k]):
        e = int(r["expert"][k])
        if e not in cache:
            cache.clear()
            cache[e] = {nm: L.get_param(f"layer0.expert{e}.{nm}").astype(np.float64)
                        for nm in ("w1", "b1", "w2", "b2")}
        W = cache[e]
        z = av[k] @ W["w1"].reshape(h, f) + W["b1"]  # (the epilogue applies GELU before rounding)
        g = bf16(0.5 * z * (1 + np.tanh(0.7978845608028654 * (z + 0.044715 * z ** 3))))
        fo = bf16(g @ W["w2"].reshape(f, h) + W["b2"])
        ref = r["prob"][k] * fo
        terms = r["prob"][k] * (np.abs(g) @ np.abs(W["w2"].reshape(f, h)) + np.abs(W["b2"]))
        num += float(np.sum((yv[k] - ref) ** 2))
        den += float(np.sum(ref ** 2))
        scl += float(np.sum(terms ** 2))
    rel = (num / max(den, 1e-300)) ** 0.5
    return {"routing_bit_exact_all_tokens": routing_ok, "y_rel_l2_sampled": rel,
            "y_err_vs_terms": (num / max(scl, 1e-300)) ** 0.5,
            "condition": (scl / max(den, 1e-300)) ** 0.5, "tokens_sampled": int(len(pick))}


def parity_verdict(before, after):
    """`before`: the check on the initialised parameters and the benched tokens (ahead of the
    warm-up steps); `after`: the same check once the timed steps have trained the
    parameters, on a fresh batch of tokens (training on one fixed batch cancels y on that
    batch -- the objective is sum(y^2)/2N -- which only inflates the relative error there:
    see `condition`).  Pass = routing bit-exact and y rel-L2 <= 1e-2, both times."""
    ok = all(r["routing_bit_exact_all_tokens"] and r["y_rel_l2_sampled"] < 1e-2
             for r in (before, after))
    return {"before_steps": before, "after_steps": after, "tolerance": 1e-2, "pass": bool(ok),
            "check": "routing of all tokens vs argmax of the GPU logits; y of sampled kept "
                     "tokens vs fp64 numpy on the layer's bf16 parameters (rel-L2), on the "
                     "initialised parameters and, after the timed steps, on fresh tokens"}


def quick_layer_bench(w, steps: int, warmup: int):
    """ms/step of one more single-GPU workload in the same process (graph-replayed step,
    CUDA events), plus its per-stage times from an eager timed pass."""
    import torch

    import paper_2303_06318_b200 as ted
    model = ted.MoeModelConfig(1, w["hidden"], w["experts"], w["tokens"], 0)
    L = ted.MoeLayer(model, ted.derive_config(1, 1, 1), ted.RunFlags(dtd=False),
                     capacity_factor=w["cf"])
    L.init_params(1234)
    g = torch.Generator(device="cuda")
    g.manual_seed(1000)
    a = torch.randn(w["tokens"], w["hidden"], device="cuda", generator=g).bfloat16()
    y, da = torch.empty_like(a), torch.empty_like(a)
    for _ in range(warmup):
        L.step(a, y, da)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        L.step(a, y, da)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    L.timing(True)
    k = max(1, min(steps, 20))
    for _ in range(k):
        L.step(a, y, da)
    torch.cuda.synchronize()
    raw = L.timing_read()
    st = {kk: round(v[0] / k, 4) for kk, v in sorted(raw.items())}
    roof, extra = rooflines(w, {kk: v[0] / k for kk, v in raw.items()}, L.stats(), 1, 1, 1, 1)
    L.close()
    return {"workload": w["name"], "hidden": w["hidden"], "ffn": 4 * w["hidden"],
            "experts": w["experts"], "tokens": w["tokens"], "capacity_factor": w["cf"],
            "ms_per_step": ms, "tokens_per_s": w["tokens"] / (ms / 1e3), "steps": steps,
            "stage_ms": st, "roofline": roof, **extra}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.samples, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("BENCH_SMI_MS", "100")], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()),
                 default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm (CPU)

def host_info():
    """The box's host CPU, for the CPU baselines."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"nproc": os.cpu_count(), "usable_cpus": usable, "cpu_model": model}


class pinned:
    """Pin this process (and the reference's rank threads it spawns) to the first k usable
    CPUs for one measurement (the taskset of BASELINE.md section 3)."""

    def __init__(self, k):
        self.k = k

    def __enter__(self):
        try:
            self.old = os.sched_getaffinity(0)
            cpus = sorted(self.old)[:max(1, self.k)]
            os.sched_setaffinity(0, cpus)
            self.cpus = cpus
        except (AttributeError, OSError):
            self.old, self.cpus = None, None
        return self

    def __exit__(self, *a):
        if self.old is not None:
            os.sched_setaffinity(0, self.old)


def ref_sample_plan(w, threads_wanted):
    """(experts = threads, token counts of the two timed runs) of the bounded CPU sample.
    Top-1 routing makes the per-token cost independent of the expert count, so wide layers
    are sampled with few experts (host memory: 4 fp64 weight / gradient tensors each)."""
    h = w["hidden"]
    cap = 4 if h > 1024 else w["experts"]
    threads = max(1, min(threads_wanted, cap, w["experts"]))
    per = 2 if h > 1024 else 16
    return threads, per * threads, 4 * per * threads


def reference_tokens_per_s(w, threads: int, k_lo: int, k_hi: int):
    """Time the unmodified reference (oracle/_ref) on a bounded sample of the layer: the
    MoE branch (gate_forward + per-expert linear/gelu fwd+bwd + gate_backward, one thread
    per expert, the reference's rank-thread model) on k_lo and on k_hi tokens over `threads`
    experts; the marginal time per token (the slope, free of the per-expert fixed costs) +
    OptimizerShard::step_owned over the layer's parameter count (a 4 M-element probe,
    scaled) amortised over the full batch."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as O
    R = O.ref()
    h, E = w["hidden"], threads
    f = 4 * h
    rng = np.random.default_rng(0)
    wg = rng.standard_normal((h, E)) / np.sqrt(h)
    w1 = rng.uniform(-1, 1, (E, h, f)) / np.sqrt(h)
    b1 = rng.uniform(-0.1, 0.1, (E, f))
    w2 = rng.uniform(-1, 1, (E, f, h)) / np.sqrt(f)
    b2 = rng.uniform(-0.1, 0.1, (E, h))
    dwg, dw1, db1 = np.empty((h, E)), np.empty((E, h, f)), np.empty((E, f))
    dw2, db2 = np.empty((E, f, h)), np.empty((E, h))
    times = {}
    for k in (k_lo, k_hi):
        a = rng.standard_normal((k, h))
        dy = rng.standard_normal((k, h)) / (k * 8)
        y, da = np.empty((k, h)), np.empty((k, h))
        t0 = time.perf_counter()
        rc = R.ref_moe_sublayer(k, h, f, E, a, wg, w1, b1, w2, b2, dy, y, da, dwg, dw1, db1,
                                dw2, db2, threads)
        times[k] = time.perf_counter() - t0
        assert rc == 0, R.ref_last_error()
    per_token_layer = max(times[k_hi] - times[k_lo], 1e-9) / (k_hi - k_lo)
    params = w["experts"] * (2 * h * f + f + h) + h * w["experts"]
    t_probe, probe = ref_step_owned(min(params, 4_000_000))
    t_adam = t_probe * params / probe
    per_token = per_token_layer + t_adam / w["tokens"]
    return 1.0 / per_token, {"layer_s": times, "per_token_layer_s": per_token_layer,
                             "adam_s_extrapolated": t_adam, "adam_probe_elems": probe}


def ref_step_owned(elems: int):
    """OptimizerShard::step_owned (optimizer.cpp:58-104) over `elems` owned elements, tile
    1.8 M (TileConfig default), 1 thread: seconds."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as O
    R = O.ref()
    rng = np.random.default_rng(1)
    vals = rng.standard_normal(elems)
    grads = rng.standard_normal(elems)
    out, m, m1, m2 = (np.empty(elems) for _ in range(4))
    pk = C.c_uint64()
    t0 = time.perf_counter()
    R.ref_adam(elems, vals, 1, 0, 1e-4, 0.9, 0.999, 1e-8, 0.01, 1, 1_800_000, 1, grads, out, m,
               m1, m2, C.byref(pk))
    return time.perf_counter() - t0, elems


def reference_entry_points():
    """the reference's own entry points on this host, each pinned to
    as many CPUs as it has rank threads -- SerialModel::step at C1 (1 thread), Trainer::step
    at the reference-expressible (8,2,4) and (4,2,2) layouts (world-size threads, DTD on),
    OptimizerShard::step_owned at 16.8 M elements."""
    import numpy as np

    from oracle import oracle as O
    R = O.ref()
    out = {}
    losses = np.zeros(1)
    with pinned(1) as pn:
        t0 = time.perf_counter()
        assert R.ref_serial_step(1, 256, 4, 1024, 1, 2, 1, losses) == 0, R.ref_last_error()
        dt = time.perf_counter() - t0
    out["serial_model_c1"] = {"config": "SerialModel::step, d=256, ffn=1024, E=4, 2 shards x "
                                        "1024 tokens, 1 MoE layer", "threads": 1,
                              "cpus": pn.cpus, "s_per_step": dt, "tokens_per_s": 2048 / dt}
    for world, tp, ep, n in ((8, 2, 4, 512), (4, 2, 2, 1024)):
        for dtd in (1,):
            a2a, ag = O.C.c_uint64(), O.C.c_uint64()
            with pinned(world) as pn:
                t0 = time.perf_counter()
                rc = R.ref_trainer_step(1, 256, ep, n, 1, world, tp, dtd, 0, 0, 1, losses,
                                        O.C.byref(a2a), O.C.byref(ag))
                dt = time.perf_counter() - t0
            assert rc == 0, R.ref_last_error()
            tokens = n * (world // tp)
            out[f"trainer_{world}_{tp}_{ep}_dtd{dtd}"] = {
                "config": f"Trainer::step world {world}, T={tp}, E={ep}, {n} tokens/shard, "
                          f"d=256, DTD {'on' if dtd else 'off'}", "threads": world,
                "cpus": pn.cpus, "s_per_step": dt, "tokens_per_s": tokens / dt,
                "ledger_a2a_bytes_fwd": a2a.value, "ledger_ag_bytes_fwd": ag.value}
    with pinned(1) as pn:
        t, el = ref_step_owned(16_800_000)
    out["step_owned"] = {"elements": el, "tile": 1_800_000, "threads": 1, "cpus": pn.cpus,
                         "s": t, "melem_per_s": el / t / 1e6}
    return out


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    hi = host_info()
    threads, k_lo, k_hi = ref_sample_plan(w, hi["usable_cpus"] or 1)
    tps, det = reference_tokens_per_s(w, threads, k_lo, k_hi)
    ms = w["tokens"] / tps * 1e3
    entry = reference_entry_points() if not args.no_entry_points else None
    line = {
        "metric": METRIC, "value": tps, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": w["name"], "hidden": w["hidden"], "ffn": 4 * w["hidden"],
                   "experts": w["experts"], "tokens": w["tokens"], "capacity_factor": None},
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "host": hi,
                         "sample": f"extrapolated: the reference MoE branch on {k_lo} and "
                                   f"{k_hi} tokens over {threads} experts ({threads} expert "
                                   f"threads; {det['layer_s'][k_lo]:.2f} s / "
                                   f"{det['layer_s'][k_hi]:.2f} s, marginal "
                                   f"{det['per_token_layer_s']:.3f} s per token) + step_owned "
                                   f"over the layer's parameters ({det['adam_s_extrapolated']:.1f}"
                                   f" s, from a {det['adam_probe_elems']}-element probe) "
                                   f"amortised over {w['tokens']} tokens"},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if entry is not None:
        line["reference_entry_points"] = entry
    print(json.dumps(line), flush=True)


def nvlink_bytes(gpu: int):
    """(tx, rx) NVLink data bytes of this GPU so far (NVML throughput counters, all links), or
    None when NVML does not expose them.  Read outside the timed regions (before the barrier
    that starts them): a slow query on one rank would otherwise skew the ranks' start."""
    try:
        import pynvml as N
        N.nvmlInit()
        hd = N.nvmlDeviceGetHandleByIndex(gpu)
        vals = N.nvmlDeviceGetFieldValues(hd, [N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                               N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
        if all(v.nvmlReturn == 0 for v in vals):
            out = tuple(int(v.value.ullVal) * 1024 for v in vals)  # KiB counters
            return out if any(out) else None
    except Exception:
        pass
    return None


def ted_switches():
    """The TED_* environment switches in effect (A/B knobs that change code paths)."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("TED_")}


# ------------------------------------------------------------------ our arm

def run_ours(args, w, rank, world, local_rank, dist):
    import numpy as np
    import torch

    import paper_2303_06318_b200 as ted

    torch.cuda.set_device(local_rank)
    ted.set_device(local_rank)
    T, P = w["tp"], w["ep"]
    D = world // (T * P)
    nshards = P * D
    n = w["tokens"] // nshards
    model = ted.MoeModelConfig(1, w["hidden"], w["experts"], n, 0)
    topo = ted.derive_config(world, T, P)
    uid = None
    if world > 1:
        obj = [ted.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    L = ted.MoeLayer(model, topo, ted.RunFlags(dtd=w["dtd"]), capacity_factor=w["cf"],
                     rank=rank, nccl_uid=uid)
    L.init_params(1234)
    # this rank's shard of tokens (replicated over the TP group): data shard index d*EP + e
    t_coord, e_coord, d_coord = rank % T, (rank // T) % P, rank // (T * P)
    g = torch.Generator(device="cuda")
    g.manual_seed(1000 + d_coord * P + e_coord)
    a = torch.randn(n, w["hidden"], device="cuda", generator=g).bfloat16()
    y = torch.empty_like(a)
    da = torch.empty_like(a)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    do_parity = world == 1 and not args.no_parity
    parity0 = sampled_parity(L, a, w, T, P) if do_parity else None
    for _ in range(args.warmup):
        L.step(a, y, da)
    torch.cuda.synchronize()
    nv0 = nvlink_bytes(local_rank) if world > 1 else None
    barrier()
    torch.cuda.synchronize()
    launches0 = ted.kernel_launches()
    with ClockSampler(local_rank) as clk:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            L.step(a, y, da)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # enqueue cost per step
        ev1.record(stream)
        torch.cuda.synchronize()
    nv1 = nvlink_bytes(local_rank) if world > 1 else None
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = (ted.kernel_launches() - launches0) // max(args.steps, 1)
    # per-stage CUDA events (event nodes inside the captured step on one GPU) for the
    # roofline of the dominant kernels; a separate pass so the headline loop carries no
    # timing overhead
    barrier()
    nprof = max(1, min(args.steps, 30))
    L.timing(True)
    for _ in range(nprof):
        L.step(a, y, da)
    torch.cuda.synchronize()
    stages = L.timing_read()
    L.timing(False)
    barrier()
    ms = max_over_ranks(ms)
    stats = L.stats()
    loss = L.loss()
    parity = None
    if do_parity:
        g2 = torch.Generator(device="cuda")
        g2.manual_seed(7777)
        a_new = torch.randn(n, w["hidden"], device="cuda", generator=g2).bfloat16()
        parity = parity_verdict(parity0, sampled_parity(L, a_new, w, T, P))
        del a_new

    # e2e through the public API: every step's tokens are copied from pinned host memory
    # (on a copy stream into one of two device buffers, so step i+1's H2D runs under step
    # i -- an input pipeline) and every step's loss is read back to the host.
    a_host = a.cpu().pin_memory()
    bufs = [a, torch.empty_like(a)]
    copy_s = torch.cuda.Stream()
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    free = [torch.cuda.Event(), torch.cuda.Event()]

    def h2d(i):
        with torch.cuda.stream(copy_s):
            copy_s.wait_event(free[i % 2])  # the step that last read this buffer is done
            bufs[i % 2].copy_(a_host, non_blocking=True)
            ready[i % 2].record(copy_s)

    # every step's loss is copied to pinned host memory on the stream (D2H inside the timed
    # region) and read on the host one step later, after that step's event -- the loop never
    # drains the GPU to read a result
    losses = torch.zeros(2, dtype=torch.float64).pin_memory()
    done = [torch.cuda.Event(), torch.cuda.Event()]
    seen = []

    def e2e_steps(k):
        for e in free:
            e.record(stream)
        h2d(0)
        for i in range(k):
            if i + 1 < k:
                h2d(i + 1)
            stream.wait_event(ready[i % 2])
            if i >= 2:
                done[i % 2].synchronize()  # step i-2's loss has landed in slot i % 2
                seen.append(float(losses[i % 2]))
            L.step(bufs[i % 2], y, da)
            free[i % 2].record(stream)
            L.loss_async(losses[i % 2:])  # (the current stream: the step's)
            done[i % 2].record(stream)
        torch.cuda.current_stream().synchronize()
        for i in range(max(0, k - 2), k):
            seen.append(float(losses[i % 2]))

    e2e_steps(3)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_steps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    # DTD on vs off, on both exchange implementations, on the same workload: step time,
    # the all-to-all and the DTD all-gather times separately (the peer exchange's fused
    # scatter is split into its two parts in the timed pass), the reference's ledger bytes
    # and the NVLink bytes NVML counts (rank 0)
    dtd_cmp = None
    if world > 1 and T > 1 and not args.no_dtd_compare:
        L.close()
        L = None
        kx = max(3, min(args.steps, 10))
        exchanges = ["peer"] + (["nccl"] if args.exchange_compare else [])
        saved = os.environ.get("TED_EXCHANGE")

        def arm(ex, dtd_flag):
            os.environ["TED_EXCHANGE"] = ex
            obj = [ted.nccl_unique_id() if rank == 0 else None]  # a fresh id per layer
            dist.broadcast_object_list(obj, src=0)
            Lx = ted.MoeLayer(model, topo, ted.RunFlags(dtd=dtd_flag), capacity_factor=w["cf"],
                              rank=rank, nccl_uid=obj[0])
            Lx.init_params(1234)
            for _ in range(3):
                Lx.step(a, y, da)
            torch.cuda.synchronize()
            nv0 = nvlink_bytes(local_rank)
            Lx.ledger(reset=True)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(kx):
                Lx.step(a, y, da)
            e1.record(stream)
            torch.cuda.synchronize()
            nv1 = nvlink_bytes(local_rank)
            led = Lx.ledger(reset=True)
            ms_x = max_over_ranks(e0.elapsed_time(e1) / kx)
            barrier()
            Lx.timing(True)
            for _ in range(kx):
                Lx.step(a, y, da)
            torch.cuda.synchronize()
            stx = {k: v[0] / kx for k, v in Lx.timing_read().items()}
            Lx.timing(False)
            barrier()
            Lx.close()

            def g(*keys):
                return round(sum(stx.get(k, 0.0) for k in keys), 4)
            if ex == "peer":
                a2a, ag = g("dispatch_a2a"), g("dispatch_ag")
                ret = g("combine_pull")
                total = g("dispatch_a2a", "dispatch_ag", "combine_pull", "combine_bwd", "gate_dx",
                          "barrier", "count_exchange")
            else:
                a2a, ag = g("a2a_fwd"), g("ag_fwd")
                ret = g("tp_allreduce_fwd", "a2a_ret_fwd", "ag_home_fwd")
                total = g("count_exchange", "a2a_fwd", "ag_fwd", "tp_allreduce_fwd", "a2a_ret_fwd",
                          "ag_home_fwd", "a2a_bwd", "ag_bwd", "tp_allreduce_bwd", "a2a_ret_bwd",
                          "ag_home_bwd")

            def per_step(key):
                return led.get(key, {}).get("payload_bytes", 0) // kx
            return {
                "ms_per_step": ms_x, "tokens_per_s": w["tokens"] / (ms_x / 1e3),
                "a2a_ms_fwd_rank0": a2a, "dtd_allgather_ms_fwd_rank0": ag,
                "return_ms_fwd_rank0": ret, "exchange_ms_total_rank0": total,
                "ledger_bytes_per_step_rank0": {
                    "a2a_fwd": per_step("forward.all_to_all"),
                    "allgather_fwd": per_step("forward.all_gather"),
                    "allreduce_fwd": per_step("forward.all_reduce"),
                    "a2a_bwd": per_step("backward.all_to_all")},
                "nvlink_tx_bytes_per_step_rank0_nvml":
                    (nv1[0] - nv0[0]) // kx if nv0 and nv1 else None,
                "stage_ms_rank0": {k: round(v, 4) for k, v in sorted(stx.items())}}

        arms = {}
        try:
            for ex in exchanges:
                for dtd_flag in (True, False):
                    arms[f"{ex}_dtd_{'on' if dtd_flag else 'off'}"] = arm(ex, dtd_flag)
        finally:
            if saved is None:
                os.environ.pop("TED_EXCHANGE", None)
            else:
                os.environ["TED_EXCHANGE"] = saved
        for ex in exchanges:
            on, off = arms[f"{ex}_dtd_on"], arms[f"{ex}_dtd_off"]
            arms[f"{ex}_dtd_ratio_off_over_on"] = {
                "a2a_ms_fwd": round(off["a2a_ms_fwd_rank0"] / on["a2a_ms_fwd_rank0"], 3)
                if on["a2a_ms_fwd_rank0"] else None,
                "a2a_ledger_bytes": round(off["ledger_bytes_per_step_rank0"]["a2a_fwd"] /
                                          max(1, on["ledger_bytes_per_step_rank0"]["a2a_fwd"]), 3),
                "step_ms": round(off["ms_per_step"] / on["ms_per_step"], 3)}
        dtd_cmp = arms
    if rank != 0:
        if L is not None:
            L.close()
        return
    tokens_global = w["tokens"]
    value = tokens_global / (ms / 1e3)
    pk = peaks()
    roofline, extra_roof = rooflines(w, {k: v[0] / nprof for k, v in stages.items()}, stats, T, P,
                                     D, world)
    stage_ms = {k: round(v[0] / nprof, 4) for k, v in sorted(stages.items())}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": w["name"], "hidden": w["hidden"], "ffn": 4 * w["hidden"],
                   "experts": w["experts"], "tokens": tokens_global, "tokens_per_shard": n,
                   "capacity_factor": w["cf"], "tp": T, "ep": P, "dp": D, "dtd": w["dtd"],
                   "step": "fwd+bwd+grad-sync+AdamW",
                   "l2": "no flush: per-step working set (weights+AdamW state+activations) "
                         "> 126 MB L2"},
        "roofline": roofline,
        **extra_roof,
        "stage_ms": stage_ms,
        "gpu_launches": int(launches),
        "host_enqueue_ms_per_step": host_ms,
        "e2e": {"value": tokens_global / (ms_e2e / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(a.numel() * 2), "d2h_bytes_per_step": 8,
                "h2d": "pinned host -> one of two device buffers on a copy stream (next "
                       "step's tokens copied under this step); every step's loss copied to "
                       "pinned host memory on the stream and read on the host one step later",
                "losses_finite": bool(all(math.isfinite(v) for v in seen))},
        "routing": {"dropped_tokens_rank0": stats["dropped"], "loss_rank0": loss},
        "clocks": clk.summary(),
        "switches": ted_switches(),
    }
    if parity is not None:
        line["parity"] = parity
    if dtd_cmp is not None:
        line["dtd_compare"] = dtd_cmp
    if world > 1:
        line["comm"] = {"a2a_bytes_fwd_rank0": stats["a2a_bytes_fwd"],
                        "nvlink_bytes_fwd_rank0": stats["peer_bytes_fwd"],
                        "peer_exchange": bool(stats["peer_exchange"]),
                        "a2a_rows_offrank_rank0": stats["a2a_rows_offrank"],
                        "ag_bytes_fwd_rank0": stats["ag_bytes_fwd"],
                        "ar_bytes_fwd_rank0": stats["ar_bytes_fwd"],
                        "nvlink_tx_bytes_per_step_rank0_nvml":
                            (nv1[0] - nv0[0]) // args.steps if nv0 and nv1 else None,
                        "nvlink_rx_bytes_per_step_rank0_nvml":
                            (nv1[1] - nv0[1]) // args.steps if nv0 and nv1 else None}
    if not args.no_cpu_baseline and world == 1:
        # a single reference rank-thread on a bounded sample (the reference arm,
        # --impl reference, uses the host's cores)
        threads, k_lo, k_hi = ref_sample_plan(w, 1)
        with pinned(threads):
            tps, det = reference_tokens_per_s(w, threads, k_lo, k_hi)
        line["cpu_baseline"] = {
            "value": tps, "unit": "tokens/s", "cores": threads, "kind": "reference",
            "host": host_info(),
            "sample": f"extrapolated: the reference MoE branch on {k_lo} and {k_hi} tokens "
                      f"over {threads} expert(s) ({det['layer_s'][k_lo]:.2f} s / "
                      f"{det['layer_s'][k_hi]:.2f} s: marginal {det['per_token_layer_s']:.3f} s "
                      f"per token, {threads} thread(s) pinned) + step_owned over the layer's "
                      f"parameters ({det['adam_s_extrapolated']:.1f} s from a "
                      f"{det['adam_probe_elems']}-element probe) amortised over "
                      f"{w['tokens']} tokens"}
    if world == 1 and w["name"].startswith("C3") and not args.no_c2:
        line["c2_single_gpu"] = quick_layer_bench(workload(1, False, "c2"), 200, 10)
    print(json.dumps(line), flush=True)
    if L is not None:
        L.close()


def run_model_stack(args, rank, world, local_rank, dist):
    """configs[3] (C4): a full training step of a layer stack (attention stand-in + MoE on
    even layers / dense FFN on odd layers, ted_model_*) with the tiled AdamW and ZeRO-1,
    16 experts, d=4096, 32768 tokens in total, TP=2 x EP=2 x DP=N/4 (fewer GPUs: TP first,
    then EP).  A side measurement: the headline bench is the C3 layer."""
    import torch

    import paper_2303_06318_b200 as ted
    torch.cuda.set_device(local_rank)
    ted.set_device(local_rank)
    T = 2 if world % 2 == 0 else 1
    P = 2 if world % 4 == 0 else 1
    D = world // (T * P)
    h, E, tokens, layers = 4096, 16, 32768, args.layers
    n = tokens // (P * D)
    model = ted.MoeModelConfig(layers, h, E, n, 0)
    uid = None
    if world > 1:
        obj = [ted.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    M = ted.TedModel(model, ted.derive_config(world, T, P), ted.RunFlags(dtd=T > 1),
                     capacity_factor=1.25, shard_optimizer=True, rank=rank, nccl_uid=uid)
    M.init_params(1234)
    g = torch.Generator(device="cuda")
    g.manual_seed(1000 + rank // T)
    batch = torch.randn(n, h, device="cuda", generator=g).bfloat16()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        M.step(batch)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ted.kernel_launches()
    with ClockSampler(local_rank) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            M.step(batch)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t_ = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms = float(t_.item())
    loss = M.loss()
    M.close()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": tokens / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": f"C4 model stack, {layers} layers", "hidden": h,
                       "ffn": 4 * h, "experts": E, "tokens": tokens, "tokens_per_shard": n,
                       "capacity_factor": 1.25, "tp": T, "ep": P, "dp": D, "dtd": T > 1,
                       "zero1": True, "step": "Trainer::step: fwd+loss+bwd+grad-sync+AdamW"},
            "gpu_launches": int((ted.kernel_launches() - launches0) // max(args.steps, 1)),
            "loss_rank0": loss, "clocks": clk.summary()}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtd", type=int, default=1)
    ap.add_argument("--no-entry-points", action="store_true",
                    help="reference arm: skip BASELINE.md section 3's entry points (~1 min)")
    ap.add_argument("--exchange-compare", type=int, default=1,
                    help="N>1: also time the NCCL send/recv exchange (DTD on and off)")
    ap.add_argument("--workload", default="c3", choices=["c3", "c2", "c4"])
    ap.add_argument("--layers", type=int, default=2, help="c4: layers of the stack")
    ap.add_argument("--no-c2", action="store_true", help="skip the configs[1] side line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the sampled parity check")
    ap.add_argument("--no-dtd-compare", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        world = args.gpus if world == 1 else world
    if args.workload == "c2" and world > 1:
        raise SystemExit("--workload c2 is the single-GPU configuration")
    if args.workload == "c4" and args.impl == "ours":
        dist = None
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        run_model_stack(args, rank, world, local_rank, dist)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    w = workload(world, bool(args.dtd), "c3" if args.workload == "c4" else args.workload)
    dist = None
    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    run_ours(args, w, rank, world, local_rank, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
