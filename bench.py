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
    st = {kk: round(v[0] / k, 4) for kk, v in sorted(L.timing_read().items())}
    L.close()
    return {"workload": w["name"], "hidden": w["hidden"], "ffn": 4 * w["hidden"],
            "experts": w["experts"], "tokens": w["tokens"], "capacity_factor": w["cf"],
            "ms_per_step": ms, "tokens_per_s": w["tokens"] / (ms / 1e3), "steps": steps,
            "stage_ms": st}


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
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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

def ref_sample_plan(w, sample_tokens):
    """(tokens, experts) of the bounded CPU sample: top-1 routing makes the per-token cost
    independent of the expert count, so wide layers are sampled with fewer experts (host
    memory: 4 fp64 weight/gradient tensors per expert) and fewer tokens (10-30 s)."""
    h = w["hidden"]
    if sample_tokens <= 0:
        sample_tokens = 256 if h <= 1024 else 24
    return sample_tokens, (w["experts"] if h <= 1024 else min(w["experts"], 2))


def reference_tokens_per_s(w, sample_tokens: int, experts: int, reps: int = 1):
    """Time the unmodified reference (oracle/_ref) on a bounded sample: the MoE branch
    (gate_forward + per-expert linear/gelu fwd+bwd + gate_backward, one thread per expert)
    on `sample_tokens` tokens routed over `experts` experts (`reps` timed repetitions,
    mean), plus OptimizerShard::step_owned on the layer's full parameter count amortised
    over the full batch."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as O
    R = O.ref()
    h, E = w["hidden"], experts
    threads = experts
    f = 4 * h
    rng = np.random.default_rng(0)
    a = rng.standard_normal((sample_tokens, h))
    wg = rng.standard_normal((h, E)) / np.sqrt(h)
    w1 = rng.uniform(-1, 1, (E, h, f)) / np.sqrt(h)
    b1 = rng.uniform(-0.1, 0.1, (E, f))
    w2 = rng.uniform(-1, 1, (E, f, h)) / np.sqrt(f)
    b2 = rng.uniform(-0.1, 0.1, (E, h))
    dy = rng.standard_normal((sample_tokens, h)) / (sample_tokens * 8)
    y, da = np.empty((sample_tokens, h)), np.empty((sample_tokens, h))
    dwg, dw1, db1 = np.empty((h, E)), np.empty((E, h, f)), np.empty((E, f))
    dw2, db2 = np.empty((E, f, h)), np.empty((E, h))
    t_layer = 0.0
    for _ in range(max(1, reps)):
        t0 = time.perf_counter()
        rc = R.ref_moe_sublayer(sample_tokens, h, f, E, a, wg, w1, b1, w2, b2, dy, y, da, dwg,
                                dw1, db1, dw2, db2, threads)
        t_layer += time.perf_counter() - t0
        assert rc == 0, R.ref_last_error()
    t_layer /= max(1, reps)
    # optimizer over a slice of the family, scaled to the layer's parameter count
    params = w["experts"] * (2 * h * f + f + h) + h * w["experts"]
    probe = min(params, 4_000_000)
    vals = rng.standard_normal(probe)
    grads = rng.standard_normal(probe)
    out, m, m1, m2 = (np.empty(probe) for _ in range(4))
    pk = C.c_uint64()
    t0 = time.perf_counter()
    R.ref_adam(probe, vals, 1, 0, 1e-4, 0.9, 0.999, 1e-8, 0.01, 1, 1_800_000, 1, grads, out, m,
               m1, m2, C.byref(pk))
    t_adam = (time.perf_counter() - t0) * params / probe
    per_token = t_layer / sample_tokens + t_adam / w["tokens"]
    return 1.0 / per_token, t_layer, t_adam


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    sample, threads = ref_sample_plan(w, args.ref_sample)
    # one bounded sample per timed step, capped so the whole run stays within minutes
    reps = max(1, min(args.steps, 3 if w["hidden"] > 1024 else 5))
    tps, t_layer, t_adam = reference_tokens_per_s(w, sample, threads, reps)
    ms = w["tokens"] / tps * 1e3
    line = {
        "metric": METRIC, "value": tps, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": w["name"], "hidden": w["hidden"], "ffn": 4 * w["hidden"],
                   "experts": w["experts"], "tokens": w["tokens"], "capacity_factor": None},
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "sample": f"{sample} tokens through the reference MoE branch "
                                   f"({t_layer:.2f} s mean of {reps} timed repetitions, "
                                   f"{threads} expert threads) + "
                                   f"step_owned over the layer's parameters ({t_adam:.2f} s, "
                                   f"1 thread) amortised over {w['tokens']} tokens"},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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

    for _ in range(args.warmup):
        L.step(a, y, da)
    torch.cuda.synchronize()
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

    def e2e_steps(k):
        for e in free:
            e.record(stream)
        h2d(0)
        for i in range(k):
            if i + 1 < k:
                h2d(i + 1)
            stream.wait_event(ready[i % 2])
            L.step(bufs[i % 2], y, da)
            free[i % 2].record(stream)
            L.loss()  # D2H of the result (synchronises the stream)

    e2e_steps(3)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_steps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    # DTD on vs off on the same workload (all-to-all bytes and time reported separately)
    dtd_cmp = None
    if world > 1 and T > 1 and not args.no_dtd_compare:
        def exch_ms(st):
            keys = ["dispatch_peer", "combine_pull", "combine_bwd", "gate_dx", "barrier", "count_exchange",
                    "a2a_fwd", "ag_fwd", "a2a_ret_fwd", "ag_home_fwd", "a2a_bwd", "ag_bwd",
                    "a2a_ret_bwd", "ag_home_bwd", "tp_allreduce_fwd", "tp_allreduce_bwd"]
            return {k: round(v, 4) for k, v in st.items() if k in keys}
        arms = {}
        for dtd_flag in (w["dtd"], not w["dtd"]):
            if dtd_flag == w["dtd"]:
                Lx, stx, ms_x = L, stages, ms
            else:
                L.close()
                obj = [ted.nccl_unique_id() if rank == 0 else None]  # a fresh id per communicator
                dist.broadcast_object_list(obj, src=0)
                Lx = ted.MoeLayer(model, topo, ted.RunFlags(dtd=dtd_flag), capacity_factor=w["cf"],
                                  rank=rank, nccl_uid=obj[0])
                Lx.init_params(1234)
                for _ in range(3):
                    Lx.step(a, y, da)
                torch.cuda.synchronize()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                kx = max(1, min(args.steps, 10))
                e0.record(stream)
                for _ in range(kx):
                    Lx.step(a, y, da)
                e1.record(stream)
                torch.cuda.synchronize()
                ms_x = max_over_ranks(e0.elapsed_time(e1) / kx)
                Lx.timing(True)
                for _ in range(kx):
                    Lx.step(a, y, da)
                torch.cuda.synchronize()
                stx = {k: v[0] / kx for k, v in Lx.timing_read().items()}
                Lx.timing(False)
                barrier()
            if dtd_flag == w["dtd"]:
                stx = {k: v[0] / nprof for k, v in stx.items()}
            sx = Lx.stats()
            ex = exch_ms(stx)
            arms["dtd_on" if dtd_flag else "dtd_off"] = {
                "ms_per_step": ms_x, "tokens_per_s": w["tokens"] / (ms_x / 1e3),
                "a2a_bytes_fwd_rank0_ledger": sx["a2a_bytes_fwd"],
                "a2a_rows_offrank_rank0": sx["a2a_rows_offrank"],
                "dtd_allgather_bytes_fwd_rank0_ledger": sx["ag_bytes_fwd"],
                "nvlink_bytes_fwd_rank0": sx["peer_bytes_fwd"],
                "exchange_ms_rank0": ex, "exchange_ms_total_rank0": round(sum(ex.values()), 4),
                "stage_ms_rank0": {k: round(v, 4) for k, v in sorted(stx.items())}}
            if Lx is not L:
                Lx.close()
        dtd_cmp = arms
        L = None
    if rank != 0:
        if L is not None:
            L.close()
        return
    tokens_global = w["tokens"]
    value = tokens_global / (ms / 1e3)
    pk = peaks()
    # roofline.  With the expert family unsharded (D = 1) AdamW runs inside the two wgrad
    # GEMMs and that kernel dominates the step (47 % of the GPU time at C3, N=1,
    # profiles/r02_ncu_summary.md): it is HBM-bound on the optimizer state.  The four
    # forward / dgrad GEMMs are reported beside it against the tensor-core peak.
    def st(k):
        return stages.get(k, (0.0, 0))[0] / nprof
    Eloc = max(1, w["experts"] // P)
    kept_rows = sum(stats["kept_per_expert"][:Eloc])
    f_t = 4 * w["hidden"] // T
    h_ = w["hidden"]
    tc_names = ["gemm1_fwd", "gemm2_fwd", "dgrad2", "dgrad1"]
    tc_ms = sum(st(k) for k in tc_names)
    tc_flops = 8.0 * kept_rows * h_ * f_t  # 4 GEMMs x 2 flops x rows x h x f/T, algorithmic
    tc_ach = tc_flops / (tc_ms / 1e3) / 1e12 if tc_ms > 0 else None
    peak_tc = pk["bf16_tflops_sustained"]
    tj = None
    for tp in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_gemm_traffic*.json"))):
        with open(tp) as f:  # from a committed ncu --set full capture of this workload
            cand = json.load(f)
        if cand.get("workload") == w["name"] and cand.get("n_gpus", 1) == world:
            tj = cand
    roof_tc = {"bound": "tensor", "kernel": "expert FFN fwd + dgrad tcgen05 GEMMs (4/step)",
               "achieved": tc_ach, "peak": peak_tc, "unit": "TFLOP/s",
               "frac": (tc_ach / peak_tc) if tc_ach else None,
               "traffic": (sum(tj["per_launch"][i] for i in (0, 1, 2, 4)) / 4) if tj else None,
               "flops_per_launch": tc_flops / 4, "ms_per_launch": tc_ms / 4,
               "peak_source": pk["source"] + " bf16_tflops_sustained"}
    if D == 1:
        wg_ms = (st("wgrad1") + st("wgrad2")) / 2
        params = Eloc * h_ * f_t
        rows = int(stats["asm_rows"])
        # 26 B per parameter (fp32 master/m/v read + write, bf16 parameter write) + the
        # wgrad operands read once (rows x (h + f/T) bf16)
        wg_bytes = 26.0 * params + 2.0 * rows * (h_ + f_t)
        wg_ach = wg_bytes / (wg_ms / 1e3) / 1e9 if wg_ms > 0 else None
        roofline = {"bound": "hbm", "kernel": "wgrad GEMM + fused AdamW (2/step)",
                    "achieved": wg_ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": (wg_ach / pk["hbm_gbs"]) if wg_ach else None,
                    "traffic": (sum(tj["per_launch"][i] for i in (3, 5)) / 2) if tj else None,
                    "bytes_per_launch": wg_bytes, "ms_per_launch": wg_ms,
                    "unit_work": "26 B per parameter + 2 B per operand element",
                    "peak_source": pk["source"] + " hbm_gbs (copy)"}
        extra_roof = {"roofline_gemm": roof_tc}
    else:
        roofline, extra_roof = roof_tc, {}
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
                       "step's tokens copied under this step); loss read back every step"},
        "routing": {"dropped_tokens_rank0": stats["dropped"], "loss_rank0": loss},
        "clocks": clk.summary(),
    }
    if dtd_cmp is not None:
        line["dtd_compare"] = dtd_cmp
    if world > 1:
        line["comm"] = {"a2a_bytes_fwd_rank0": stats["a2a_bytes_fwd"],
                        "nvlink_bytes_fwd_rank0": stats["peer_bytes_fwd"],
                        "peer_exchange": bool(stats["peer_exchange"]),
                        "a2a_rows_offrank_rank0": stats["a2a_rows_offrank"],
                        "ag_bytes_fwd_rank0": stats["ag_bytes_fwd"],
                        "ar_bytes_fwd_rank0": stats["ar_bytes_fwd"]}
    if not args.no_cpu_baseline and world == 1:
        sample, nexp = ref_sample_plan(w, args.ref_sample)
        tps, t_layer, t_adam = reference_tokens_per_s(w, sample, nexp)
        line["cpu_baseline"] = {"value": tps, "unit": "tokens/s", "cores": nexp,
                                "kind": "reference",
                                "sample": f"{sample} tokens over {nexp} experts through the "
                                          f"reference MoE branch ({t_layer:.2f} s, {nexp} "
                                          f"expert threads) + step_owned over the layer's "
                                          f"{w['experts']} experts' parameters "
                                          f"({t_adam:.2f} s) amortised over {w['tokens']} tokens"}
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
    ap.add_argument("--ref-sample", type=int, default=0, help="0: automatic (10-30 s)")
    ap.add_argument("--workload", default="c3", choices=["c3", "c2", "c4"])
    ap.add_argument("--layers", type=int, default=2, help="c4: layers of the stack")
    ap.add_argument("--no-c2", action="store_true", help="skip the configs[1] side line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
