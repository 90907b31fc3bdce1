"""ted-b200: B200-native TED (arXiv 2303.06318) MoE-layer hot path.

Python face of ``libted_b200.so`` (the C ABI in ``include/ted.h``), mirroring the
reference's configuration and operator API (tedsim: ``MoeModelConfig``, ``TedConfig``,
``RunFlags``, ``AdamConfig``, ``TileConfig``, ``gate_forward`` / ``gate_backward``,
``OptimizerShard::step_owned``, ``MoeRank``'s MoE branch).

Device buffers are passed as ``torch`` tensors (torch is only the allocator / stream
plumbing here); every compute call goes through the CUDA library.  There is no CPU
fallback: importing works anywhere, but calls raise ``TedRuntimeError`` without an
sm_100 device, and a missing ``libted_b200.so`` raises at import time.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
# TED_LIB: load another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("TED_LIB") or os.path.join(HERE, "libted_b200.so")
PLAN_PATH = os.path.join(HERE, "libted_plan.so")

TED_OK, TED_ERR_RUNTIME, TED_ERR_CONFIG = 0, 1, 2


class TedError(RuntimeError):
    pass


class TedRuntimeError(TedError):
    """ProtocolError / TimeoutError / CUDA / NCCL failure (status 1)."""


class InvalidConfigError(TedError, ValueError):
    """InvalidConfigError / InvalidGroupError (status 2)."""


def build(verbose: bool = False) -> None:
    """Compile libted_b200.so / libted_plan.so in-tree (nvcc, sm_100a)."""
    import subprocess

    subprocess.run(["make", "-C", os.path.join(HERE, "csrc"), "-j8"] + ([] if verbose else ["-s"]),
                   check=True)


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run paper_2303_06318_b200.build() "
                      "(the TED hot path has no CPU fallback)")

def _preload_nccl() -> None:
    """libted_b200.so needs libnccl.so.2.  If torch's bundled NCCL (newer, ABI-compatible)
    exists, load it first so that torch and this library share one NCCL whatever the
    import order (otherwise the system 2.27 copy would shadow the symbols torch needs)."""
    import importlib.util

    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        spec = None
    for base in (spec.submodule_search_locations if spec else []) or []:
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            C.CDLL(cand, mode=C.RTLD_GLOBAL)
            return


_preload_nccl()
_lib = C.CDLL(LIB_PATH)
_vp, _i64, _i32, _u64, _dbl = C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_double


class ModelCfg(C.Structure):
    _fields_ = [("layers", C.c_int), ("hidden", C.c_int), ("experts", C.c_int),
                ("tokens_per_shard", C.c_int), ("seed", C.c_uint64)]


class TopoCfg(C.Structure):
    _fields_ = [("world_size", C.c_int), ("tensor_parallel", C.c_int), ("experts", C.c_int),
                ("expert_data_parallel", C.c_int), ("nonexpert_data_parallel", C.c_int)]


class FlagsC(C.Structure):
    _fields_ = [("dtd", C.c_int), ("cac", C.c_int), ("ckpt", C.c_int),
                ("track_tokens", C.c_int), ("corrupt_drop", C.c_int)]


class AdamC(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double)]


class TileC(C.Structure):
    _fields_ = [("enabled", C.c_int), ("tile_size", C.c_int64)]


class LayerStats(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("dropped", C.c_int64), ("send_rows", C.c_int64),
                ("a2a_rows_offrank", C.c_int64), ("a2a_bytes_fwd", C.c_int64),
                ("ag_bytes_fwd", C.c_int64), ("ar_bytes_fwd", C.c_int64),
                ("asm_rows", C.c_int64), ("placement_ok", C.c_int),
                ("kept_per_expert", C.c_int64 * 64), ("peer_bytes_fwd", C.c_int64),
                ("peer_exchange", C.c_int), ("placement_ok_all", C.c_int)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("ted_last_error", C.c_char_p, [])
_sig("ted_version", C.c_char_p, [])
_sig("ted_set_device", _i32, [_i32])
_sig("ted_default_configs", None, [C.POINTER(ModelCfg), C.POINTER(TopoCfg), C.POINTER(FlagsC),
                                   C.POINTER(AdamC), C.POINTER(TileC)])
_sig("ted_derive_config", _i32, [_i32, _i32, _i32, C.POINTER(TopoCfg)])
_sig("ted_shard_range", _i32, [_i64, _i32, _i32, C.POINTER(_i64), C.POINTER(_i64)])
_sig("ted_gate_forward", _i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp])
_sig("ted_gate_route_logits", _i32, [_vp, _i64, _i32, _vp, _vp, _vp, _vp])
_sig("ted_route", _i32, [_vp, _i64, _i32, _i64, _i32, _vp, _vp, _vp, _vp])
_sig("ted_gate_backward", _i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp])
_sig("ted_grouped_gemm", _i32, [_i32, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _i64, _i32,
                                _vp, _i64, _i64, _i32, _vp, _i64, _i64, _vp, _i64, _vp, _i64,
                                _vp])
_sig("ted_adam_step", _i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, C.POINTER(AdamC),
                             C.POINTER(TileC), C.POINTER(_u64), _vp])
_sig("ted_nccl_unique_id", _i32, [C.c_char_p])
_sig("ted_placement_verdict", _i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp])
_sig("ted_layer_create", _i32, [C.POINTER(ModelCfg), C.POINTER(TopoCfg), C.POINTER(FlagsC),
                                C.POINTER(AdamC), C.POINTER(TileC), _dbl, _i32, _i32,
                                C.c_char_p, C.POINTER(_vp)])
_sig("ted_layer_destroy", None, [_vp])
_sig("ted_layer_set_param", _i32, [_vp, C.c_char_p, _vp])
_sig("ted_layer_get_param", _i32, [_vp, C.c_char_p, _vp, C.POINTER(_i64)])
_sig("ted_layer_get_grad", _i32, [_vp, C.c_char_p, _vp, C.POINTER(_i64)])
_sig("ted_layer_init_params", _i32, [_vp, _u64])
_sig("ted_layer_keep_grads", _i32, [_vp, _i32])
_sig("ted_layer_forward", _i32, [_vp, _vp, _vp, _vp])
_sig("ted_layer_backward", _i32, [_vp, _vp, _vp, _vp])
_sig("ted_layer_optimizer_step", _i32, [_vp, _vp])
_sig("ted_layer_step", _i32, [_vp, _vp, _vp, _vp, _vp])
_sig("ted_layer_loss", _i32, [_vp, C.POINTER(_dbl), _vp])
_sig("ted_layer_set_timeout", _i32, [_vp, _dbl])
_sig("ted_layer_loss_async", _i32, [_vp, _vp, _vp])
_sig("ted_layer_ledger", _i32, [_vp, _vp, _i32])
_sig("ted_model_ledger", _i32, [_vp, _vp, _i32])
_sig("ted_ops_reserve", _i32, [C.c_size_t, _vp])
_sig("ted_ops_release", _i32, [])
_sig("ted_dispatch_rows_bound", _i64, [_i64, _i32, _i64])
_sig("ted_dispatch_forward", _i32, [_vp, _vp, _i64, _i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp,
                                    _vp])
_sig("ted_dispatch_backward", _i32, [_vp, _vp, _i64, _i32, _vp, _vp])
_sig("ted_combine_forward", _i32, [_vp, _vp, _vp, _i64, _i32, _vp, _vp])
_sig("ted_combine_backward", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp,
                                    _vp, _vp, _vp])
_sig("ted_gate_backward_dlogits", _i32, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp,
                                         _vp])
_sig("ted_expert_ffn_forward", _i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _i64, _vp, _i64,
                                      _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp])
_sig("ted_expert_ffn_backward", _i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp,
                                       _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64,
                                       _vp, _i64, _vp])
_sig("ted_model_set_timeout", _i32, [_vp, _dbl])
_sig("ted_layer_get_stats", _i32, [_vp, C.POINTER(LayerStats)])
_sig("ted_layer_get_routing", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp])
_sig("ted_layer_timing", _i32, [_vp, _i32])
_sig("ted_layer_timing_read", _i32, [_vp, C.c_char_p, _i32])
_sig("ted_kernel_launches", C.c_ulonglong, [])
_sig("ted_model_create", _i32, [C.POINTER(ModelCfg), C.POINTER(TopoCfg), C.POINTER(FlagsC),
                                C.POINTER(AdamC), C.POINTER(TileC), _dbl, _i32, _i32,
                                C.c_char_p, C.POINTER(_vp)])
_sig("ted_model_destroy", None, [_vp])
_sig("ted_model_set_param", _i32, [_vp, C.c_char_p, _vp])
_sig("ted_model_get_param", _i32, [_vp, C.c_char_p, _vp, C.POINTER(_i64)])
_sig("ted_model_get_grad", _i32, [_vp, C.c_char_p, _vp, C.POINTER(_i64)])
_sig("ted_model_init_params", _i32, [_vp, _u64])
_sig("ted_model_keep_grads", _i32, [_vp, _i32])
_sig("ted_model_step", _i32, [_vp, _vp, _vp])
_sig("ted_model_forward", _i32, [_vp, _vp, _vp])
_sig("ted_model_backward", _i32, [_vp, _vp])
_sig("ted_model_optimizer_step", _i32, [_vp, _vp])
_sig("ted_model_loss", _i32, [_vp, C.POINTER(_dbl), _vp])
_sig("ted_model_output", _i32, [_vp, _vp, _vp])
_sig("ted_model_memory", _i32, [_vp, C.POINTER(_i64)])

EXPORTED = [
    "ted_default_configs", "ted_last_error", "ted_version", "ted_derive_config",
    "ted_shard_range", "ted_gate_forward", "ted_gate_route_logits", "ted_route",
    "ted_gate_backward", "ted_grouped_gemm", "ted_adam_step", "ted_placement_verdict", "ted_layer_create",
    "ted_layer_destroy", "ted_nccl_unique_id", "ted_layer_set_param", "ted_layer_get_param",
    "ted_layer_get_grad", "ted_layer_keep_grads", "ted_layer_init_params", "ted_layer_forward", "ted_layer_backward",
    "ted_layer_optimizer_step", "ted_layer_step", "ted_layer_loss", "ted_layer_loss_async",
    "ted_layer_set_timeout",
    "ted_layer_get_stats",
    "ted_layer_get_routing", "ted_layer_timing", "ted_layer_timing_read", "ted_kernel_launches",
    "ted_set_device", "ted_model_create", "ted_model_destroy", "ted_model_set_param",
    "ted_model_get_param", "ted_model_get_grad", "ted_model_init_params", "ted_model_keep_grads", "ted_model_step",
    "ted_model_forward", "ted_model_backward", "ted_model_optimizer_step", "ted_model_loss",
    "ted_model_set_timeout", "ted_layer_ledger", "ted_model_ledger", "ted_ops_reserve", "ted_ops_release", "ted_dispatch_rows_bound",
    "ted_dispatch_forward", "ted_dispatch_backward", "ted_combine_forward", "ted_combine_backward",
    "ted_gate_backward_dlogits", "ted_expert_ffn_forward", "ted_expert_ffn_backward",
    "ted_model_output", "ted_model_memory"]


LEDGER_PHASES = ("forward", "recompute", "backward", "grad_sync", "optim")  # types.hpp:32
LEDGER_OPS = ("all_reduce", "all_gather", "all_to_all")  # types.hpp:39


def _ledger(fn, h, reset):
    buf = (C.c_uint64 * 30)()
    _check(fn(h, C.cast(buf, _vp), int(reset)))
    out = {}
    for ph, pn in enumerate(LEDGER_PHASES):
        for op, on in enumerate(LEDGER_OPS):
            calls, byts = buf[(ph * 3 + op) * 2], buf[(ph * 3 + op) * 2 + 1]
            if calls or byts:
                out[f"{pn}.{on}"] = {"calls": int(calls), "payload_bytes": int(byts)}
    return out


def lib():
    return _lib


def _check(rc: int) -> None:
    if rc == TED_OK:
        return
    msg = (_lib.ted_last_error() or b"").decode()
    if rc == TED_ERR_CONFIG:
        raise InvalidConfigError(msg)
    raise TedRuntimeError(msg)


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(stream)


# ------------------------------------------------------------------ config mirror

@dataclass
class MoeModelConfig:  # moe.hpp:24-30
    layers: int = 1
    hidden: int = 8
    experts: int = 2
    tokens_per_shard: int = 8
    seed: int = 1

    def c(self):
        return ModelCfg(self.layers, self.hidden, self.experts, self.tokens_per_shard, self.seed)


@dataclass
class TedConfig:  # topology.hpp:22-28 (experts = expert-parallel degree)
    world_size: int = 1
    tensor_parallel: int = 1
    experts: int = 1
    expert_data_parallel: int = 1
    nonexpert_data_parallel: int = 1

    def c(self):
        return TopoCfg(self.world_size, self.tensor_parallel, self.experts,
                       self.expert_data_parallel, self.nonexpert_data_parallel)


@dataclass
class RunFlags:  # moe.hpp:40-46 (ckpt / cac: the model stack (TedModel); a single MoeLayer rejects them)
    dtd: bool = False
    cac: bool = False
    ckpt: bool = False
    track_tokens: bool = False
    corrupt_drop: bool = False

    def c(self):
        return FlagsC(int(self.dtd), int(self.cac), int(self.ckpt), int(self.track_tokens),
                      int(self.corrupt_drop))


@dataclass
class AdamConfig:  # optimizer.hpp:17-23
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01

    def c(self):
        return AdamC(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay)


@dataclass
class TileConfig:  # optimizer.hpp:36-39
    enabled: bool = True
    tile_size: int = 1_800_000

    def c(self):
        return TileC(int(self.enabled), self.tile_size)


def derive_config(world_size: int, tensor_parallel: int, experts: int) -> TedConfig:
    """topology.cpp:10-37; `experts` is the expert-parallel degree."""
    out = TopoCfg()
    _check(_lib.ted_derive_config(world_size, tensor_parallel, experts, C.byref(out)))
    return TedConfig(out.world_size, out.tensor_parallel, out.experts, out.expert_data_parallel,
                     out.nonexpert_data_parallel)


def shard_range(total: int, parts: int, index: int):
    b, e = _i64(), _i64()
    _check(_lib.ted_shard_range(total, parts, index, C.byref(b), C.byref(e)))
    return b.value, e.value


def capacity(cf: float, n: int, E: int) -> int:
    """C = ceil(cf * n / E) on the full pre-drop shard; cf <= 0 -> unlimited (n)."""
    if cf <= 0:
        return n
    return min(n, int(math.ceil(cf * n / E)))


# ------------------------------------------------------------------ operators (torch tensors)

def gate_forward(a, wg, logits=None, stream=None):
    """gate_forward (moe.cpp:158-186).  a [n,h] bf16, wg [h,E] bf16 (CUDA tensors).
    Returns (expert int32 [n], prob fp32 [n], probs fp32 [n,E], logits fp32 [n,E])."""
    import torch
    n, h = a.shape
    E = wg.shape[1]
    dev = a.device
    expert = torch.empty(n, dtype=torch.int32, device=dev)
    prob = torch.empty(n, dtype=torch.float32, device=dev)
    probs = torch.empty(n, E, dtype=torch.float32, device=dev)
    if logits is None:
        logits = torch.empty(n, E, dtype=torch.float32, device=dev)
    _check(_lib.ted_gate_forward(_p(a), _p(wg), n, h, E, _p(logits), _p(probs), _p(expert),
                                 _p(prob), _stream(stream)))
    return expert, prob, probs, logits


def gate_route_logits(logits, stream=None):
    import torch
    n, E = logits.shape
    dev = logits.device
    expert = torch.empty(n, dtype=torch.int32, device=dev)
    prob = torch.empty(n, dtype=torch.float32, device=dev)
    probs = torch.empty(n, E, dtype=torch.float32, device=dev)
    _check(_lib.ted_gate_route_logits(_p(logits), n, E, _p(probs), _p(expert), _p(prob),
                                      _stream(stream)))
    return expert, prob, probs


def route(expert, E: int, cap: int, T: int = 1, stream=None):
    """Capacity slots: returns (slot int32 [n], keep uint8 [n], kept_counts int32 [T,E])."""
    import torch
    n = expert.shape[0]
    dev = expert.device
    slot = torch.empty(n, dtype=torch.int32, device=dev)
    keep = torch.empty(n, dtype=torch.uint8, device=dev)
    kc = torch.empty(T, E, dtype=torch.int32, device=dev)
    _check(_lib.ted_route(_p(expert), n, E, cap, T, _p(slot), _p(keep), _p(kc),
                          _stream(stream)))
    return slot, keep, kc


def gate_backward(a, wg, probs, expert, dchosen, stream=None):
    import torch
    n, h = a.shape
    E = wg.shape[1]
    dwg = torch.empty(h, E, dtype=torch.bfloat16, device=a.device)
    dinput = torch.empty(n, h, dtype=torch.bfloat16, device=a.device)
    _check(_lib.ted_gate_backward(_p(a), _p(wg), _p(probs), _p(expert), _p(dchosen), n, h, E,
                                  _p(dwg), _p(dinput), _stream(stream)))
    return dwg, dinput


# ---- the MoE branch as single-rank operators (moe.cpp:440-563 / :587-686 on one rank)

def ops_reserve(nbytes: int, stream=None):
    _check(_lib.ted_ops_reserve(int(nbytes), _stream(stream)))


def dispatch_forward(a, expert, E: int, cap: int = 0, stream=None):
    """Dispatch pack: returns (x_asm [R,h] bf16, pos int32 [n], seg_off int32 [E+1],
    kept int32 [E], slot int32 [n]); R = dispatch_rows_bound(n, E, cap)."""
    import torch
    n, h = a.shape
    R = int(_lib.ted_dispatch_rows_bound(n, E, cap))
    dev = a.device
    x = torch.empty(R, h, dtype=torch.bfloat16, device=dev)
    pos = torch.empty(n, dtype=torch.int32, device=dev)
    slot = torch.empty(n, dtype=torch.int32, device=dev)
    seg = torch.empty(E + 1, dtype=torch.int32, device=dev)
    kept = torch.empty(E, dtype=torch.int32, device=dev)
    _check(_lib.ted_dispatch_forward(_p(a), _p(expert), n, h, E, cap, _p(slot), _p(pos), _p(x),
                                     _p(seg), _p(kept), _stream(stream)))
    return x, pos, seg, kept, slot


def dispatch_backward(dx_asm, pos, n: int, stream=None):
    import torch
    h = dx_asm.shape[1]
    da = torch.empty(n, h, dtype=torch.bfloat16, device=dx_asm.device)
    _check(_lib.ted_dispatch_backward(_p(dx_asm), _p(pos), n, h, _p(da), _stream(stream)))
    return da


def combine_forward(f_asm, pos, prob, stream=None):
    import torch
    n, h = pos.shape[0], f_asm.shape[1]
    y = torch.empty(n, h, dtype=torch.bfloat16, device=f_asm.device)
    _check(_lib.ted_combine_forward(_p(f_asm), _p(pos), _p(prob), n, h, _p(y), _stream(stream)))
    return y


def combine_backward(f_asm, pos, prob, probs, expert, dy, seg_off=None, kept=None, stream=None):
    """Returns (df_asm like f_asm, dlogits fp32 [n,E])."""
    import torch
    n, E = probs.shape
    h = f_asm.shape[1]
    df = torch.empty_like(f_asm)
    dl = torch.empty(n, E, dtype=torch.float32, device=f_asm.device)
    _check(_lib.ted_combine_backward(_p(f_asm), _p(pos), _p(prob), _p(probs), _p(expert), _p(dy),
                                     n, h, E, _p(seg_off), _p(kept), _p(df), _p(dl),
                                     _stream(stream)))
    return df, dl


def gate_backward_dlogits(a, wg, dlogits, dispatch_grad=None, pos=None, stream=None):
    """Returns (dWg [h,E] bf16, da [n,h] bf16 = dlogits Wg^T (+ dispatch_grad[pos]))."""
    import torch
    n, h = a.shape
    E = wg.shape[1]
    dwg = torch.empty(h, E, dtype=torch.bfloat16, device=a.device)
    da = torch.empty(n, h, dtype=torch.bfloat16, device=a.device)
    _check(_lib.ted_gate_backward_dlogits(_p(a), _p(wg), _p(dlogits), n, h, E, _p(dwg), _p(da),
                                          _p(dispatch_grad), _p(pos), _stream(stream)))
    return dwg, da


def expert_ffn_forward(x_asm, seg_off, w1, b1, w2, b2, stream=None):
    """w1 [E,h,f], b1 [E,f], w2 [E,f,h], b2 [E,h] bf16.  Returns (Z, H, F)."""
    import torch
    R, h = x_asm.shape
    E, _, f = w1.shape
    z = torch.empty(R, f, dtype=torch.bfloat16, device=x_asm.device)
    hh = torch.empty_like(z)
    fo = torch.empty(R, h, dtype=torch.bfloat16, device=x_asm.device)
    _check(_lib.ted_expert_ffn_forward(_p(x_asm), _p(seg_off), R, E, h, f, _p(w1), h * f, _p(b1),
                                       f, _p(w2), f * h, _p(b2), h, _p(z), _p(hh), _p(fo),
                                       _stream(stream)))
    return z, hh, fo


def expert_ffn_backward(x_asm, z, hact, df_asm, seg_off, w1, w2, stream=None):
    """z is overwritten with dZ.  Returns (dX, dW1, db1, dW2, db2)."""
    import torch
    R, h = x_asm.shape
    E, _, f = w1.shape
    dev = x_asm.device
    dx = torch.empty(R, h, dtype=torch.bfloat16, device=dev)
    dw1 = torch.empty(E, h, f, dtype=torch.bfloat16, device=dev)
    db1 = torch.empty(E, f, dtype=torch.bfloat16, device=dev)
    dw2 = torch.empty(E, f, h, dtype=torch.bfloat16, device=dev)
    db2 = torch.empty(E, h, dtype=torch.bfloat16, device=dev)
    _check(_lib.ted_expert_ffn_backward(_p(x_asm), _p(z), _p(hact), _p(df_asm), _p(seg_off), R,
                                        E, h, f, _p(w1), h * f, _p(w2), f * h, _p(dx), _p(dw1),
                                        h * f, _p(db1), f, _p(dw2), f * h, _p(db2), h,
                                        _stream(stream)))
    return dx, dw1, db1, dw2, db2


GEMM_ROWS, GEMM_KDIM = 0, 1
EPI_STORE, EPI_BIAS, EPI_BIAS_GELU, EPI_DGELU = 0, 1, 2, 3


def grouped_gemm(mode, epi, groups, M, N, K, seg_off, max_rows, A, lda, a_mn, B, ldb,
                 b_group_stride, b_mn, Cm, ldc, c_group_stride=0, bias=None,
                 bias_group_stride=0, aux=None, ld_aux=0, stream=None):
    _check(_lib.ted_grouped_gemm(mode, epi, groups, M, N, K, _p(seg_off), max_rows, _p(A), lda,
                                 int(a_mn), _p(B), ldb, b_group_stride, int(b_mn), _p(Cm), ldc,
                                 c_group_stride, _p(bias), bias_group_stride, _p(aux), ld_aux,
                                 _stream(stream)))


def adam_step(master, m1, m2, param, grad, begin, end, step, adam=None, tiles=None,
              stream=None) -> int:
    """OptimizerShard::step_owned on device; returns the up-cast peak bytes accounted."""
    adam = adam or AdamConfig()
    tiles = tiles or TileConfig()
    peak = _u64()
    a, t = adam.c(), tiles.c()
    _check(_lib.ted_adam_step(_p(master), _p(m1), _p(m2), _p(param), _p(grad), begin, end, step,
                              C.byref(a), C.byref(t), C.byref(peak), _stream(stream)))
    return peak.value


def placement_verdict(pos_send, pos_home, T: int, slot_chunk: int, verdict, stream=None):
    """DTD placement verdict (moe.cpp:537-556) on device int32 row records; verdict is a
    device int32[2] ([0] this call, [1] &= it)."""
    _check(_lib.ted_placement_verdict(_p(pos_send), _p(pos_home), pos_send.numel(), T,
                                      slot_chunk, _p(verdict), _stream(stream)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.ted_nccl_unique_id(buf))
    return buf.raw


def set_device(dev: int) -> None:
    _check(_lib.ted_set_device(dev))


def kernel_launches() -> int:
    return int(_lib.ted_kernel_launches())


# ------------------------------------------------------------------ the layer (MoeRank)

class MoeLayer:
    """One rank's TED MoE layer (MoeRank's MoE branch, moe.cpp:418-741)."""

    def __init__(self, model: MoeModelConfig, topo: TedConfig, flags: RunFlags | None = None,
                 adam: AdamConfig | None = None, tiles: TileConfig | None = None,
                 capacity_factor: float = 0.0, shard_optimizer: bool = True, rank: int = 0,
                 nccl_uid: bytes | None = None):
        self.model, self.topo = model, topo
        self.flags = flags or RunFlags()
        self.adam = adam or AdamConfig()
        self.tiles = tiles or TileConfig()
        self.capacity_factor = capacity_factor
        self.rank = rank
        h = _vp()
        m, t, f, a, ti = model.c(), topo.c(), self.flags.c(), self.adam.c(), self.tiles.c()
        _check(_lib.ted_layer_create(C.byref(m), C.byref(t), C.byref(f), C.byref(a),
                                     C.byref(ti), capacity_factor, int(shard_optimizer), rank,
                                     nccl_uid, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.ted_layer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_param(self, name: str, full):
        import numpy as np
        arr = np.ascontiguousarray(full, dtype=np.float32)
        _check(_lib.ted_layer_set_param(self._h, name.encode(), arr.ctypes.data_as(_vp)))

    def _get(self, name, grad):
        import numpy as np
        n = _i64()
        fn = _lib.ted_layer_get_grad if grad else _lib.ted_layer_get_param
        _check(fn(self._h, name.encode(), None, C.byref(n)))
        out = np.empty(n.value, np.float32)
        _check(fn(self._h, name.encode(), out.ctypes.data_as(_vp), C.byref(n)))
        return out

    def get_param(self, name):
        return self._get(name, False)

    def get_grad(self, name):
        return self._get(name, True)

    def init_params(self, seed: int = 0):
        _check(_lib.ted_layer_init_params(self._h, seed))

    def keep_grads(self, keep: bool = True):
        """step() fuses AdamW into the wgrad GEMMs; keep=True also stores the expert
        w1/w2 gradients there (else get_grad of those fails after a fused step)."""
        _check(_lib.ted_layer_keep_grads(self._h, int(keep)))

    def forward(self, a, y, stream=None):
        _check(_lib.ted_layer_forward(self._h, _p(a), _p(y), _stream(stream)))

    def backward(self, dy, da, stream=None):
        _check(_lib.ted_layer_backward(self._h, _p(dy), _p(da), _stream(stream)))

    def optimizer_step(self, stream=None):
        _check(_lib.ted_layer_optimizer_step(self._h, _stream(stream)))

    def step(self, a, y, da, stream=None):
        _check(_lib.ted_layer_step(self._h, _p(a), _p(y), _p(da), _stream(stream)))

    def loss(self, stream=None) -> float:
        v = _dbl()
        _check(_lib.ted_layer_loss(self._h, C.byref(v), _stream(stream)))
        return v.value

    def ledger(self, reset: bool = False) -> dict:
        """This rank's CommLedger entries {"<phase>.<op>": {calls, payload_bytes}}."""
        return _ledger(_lib.ted_layer_ledger, self._h, reset)

    def loss_async(self, dst_pinned, stream=None):
        """Copy the last forward's loss into element 0 of a pinned float64 host tensor,
        stream-ordered, without waiting."""
        _check(_lib.ted_layer_loss_async(self._h, C.c_void_p(dst_pinned.data_ptr()),
                                         _stream(stream)))

    def set_timeout(self, seconds: float):
        """collective_timeout (moe.hpp:96): a stalled peer raises TedRuntimeError
        ("TimeoutError: ...") at the next call instead of hanging or trapping."""
        _check(_lib.ted_layer_set_timeout(self._h, float(seconds)))

    def stats(self) -> dict:
        s = LayerStats()
        _check(_lib.ted_layer_get_stats(self._h, C.byref(s)))
        d = {k: getattr(s, k) for k, _ in LayerStats._fields_ if k != "kept_per_expert"}
        d["kept_per_expert"] = list(s.kept_per_expert)
        return d

    def timing(self, enable: bool = True):
        _check(_lib.ted_layer_timing(self._h, int(enable)))

    def timing_read(self) -> dict:
        import json
        buf = C.create_string_buffer(1 << 16)
        _check(_lib.ted_layer_timing_read(self._h, buf, len(buf)))
        return {k: (v[0], v[1]) for k, v in json.loads(buf.value.decode()).items()}

    def routing(self):
        import numpy as np
        n, E = self.model.tokens_per_shard, self.model.experts
        ex = np.empty(n, np.int32)
        pr = np.empty(n, np.float32)
        sl = np.empty(n, np.int32)
        ph = np.empty(n, np.int32)
        ps = np.empty((n, E), np.float32)
        lg = np.empty((n, E), np.float32)
        _check(_lib.ted_layer_get_routing(self._h, *(x.ctypes.data_as(_vp)
                                                     for x in (ex, pr, sl, ph, ps, lg))))
        return dict(expert=ex, prob=pr, slot=sl, pos_home=ph, probs=ps, logits=lg)


# ------------------------------------------------------------------ the model (Trainer)

def param_names(model: MoeModelConfig) -> list:
    """enumerate_params order (moe.cpp:115-147): attention block, then the gate and experts
    on even layers or the dense FFN block on odd layers."""
    out = []
    for l in range(model.layers):
        out += [f"layer{l}.attn.{k}" for k in ("w1", "b1", "w2", "b2")]
        if l % 2 == 0:
            out.append(f"layer{l}.gate.w")
            for e in range(model.experts):
                out += [f"layer{l}.expert{e}.{k}" for k in ("w1", "b1", "w2", "b2")]
        else:
            out += [f"layer{l}.ffn.{k}" for k in ("w1", "b1", "w2", "b2")]
    return out


def param_shape(model: MoeModelConfig, name: str) -> tuple:
    h = model.hidden
    leaf = name.rsplit(".", 1)[1]
    if name.endswith("gate.w"):
        return (h, model.experts)
    return {"w1": (h, 4 * h), "b1": (4 * h,), "w2": (4 * h, h), "b2": (h,)}[leaf]


class TedModel:
    """One rank of the reference's Trainer over a layer stack (MoeRank, moe.cpp:334-415):
    attention stand-in block + MoE branch (even layers) or dense FFN (odd layers)."""

    def __init__(self, model: MoeModelConfig, topo: TedConfig, flags: RunFlags | None = None,
                 adam: AdamConfig | None = None, tiles: TileConfig | None = None,
                 capacity_factor: float = 0.0, shard_optimizer: bool = True, rank: int = 0,
                 nccl_uid: bytes | None = None):
        self.model, self.topo = model, topo
        self.flags = flags or RunFlags()
        self.adam = adam or AdamConfig()
        self.tiles = tiles or TileConfig()
        h = _vp()
        m, t, f, a, ti = model.c(), topo.c(), self.flags.c(), self.adam.c(), self.tiles.c()
        _check(_lib.ted_model_create(C.byref(m), C.byref(t), C.byref(f), C.byref(a),
                                     C.byref(ti), capacity_factor, int(shard_optimizer), rank,
                                     nccl_uid, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.ted_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_param(self, name: str, full):
        import numpy as np
        arr = np.ascontiguousarray(full, dtype=np.float32)
        _check(_lib.ted_model_set_param(self._h, name.encode(), arr.ctypes.data_as(_vp)))

    def _get(self, name, grad):
        import numpy as np
        n = _i64()
        fn = _lib.ted_model_get_grad if grad else _lib.ted_model_get_param
        _check(fn(self._h, name.encode(), None, C.byref(n)))
        out = np.empty(n.value, np.float32)
        _check(fn(self._h, name.encode(), out.ctypes.data_as(_vp), C.byref(n)))
        return out

    def get_param(self, name):
        return self._get(name, False)

    def get_grad(self, name):
        return self._get(name, True)

    def init_params(self, seed: int = 0):
        _check(_lib.ted_model_init_params(self._h, seed))

    def keep_grads(self, keep: bool = True):
        _check(_lib.ted_model_keep_grads(self._h, int(keep)))

    def step(self, batch, stream=None):
        _check(_lib.ted_model_step(self._h, _p(batch), _stream(stream)))

    def forward(self, batch, stream=None):
        _check(_lib.ted_model_forward(self._h, _p(batch), _stream(stream)))

    def backward(self, stream=None):
        _check(_lib.ted_model_backward(self._h, _stream(stream)))

    def optimizer_step(self, stream=None):
        _check(_lib.ted_model_optimizer_step(self._h, _stream(stream)))

    def loss(self, stream=None) -> float:
        v = _dbl()
        _check(_lib.ted_model_loss(self._h, C.byref(v), _stream(stream)))
        return v.value

    def set_timeout(self, seconds: float):
        _check(_lib.ted_model_set_timeout(self._h, float(seconds)))

    def ledger(self, reset: bool = False) -> dict:
        return _ledger(_lib.ted_model_ledger, self._h, reset)

    def output(self, y, stream=None):
        _check(_lib.ted_model_output(self._h, _p(y), _stream(stream)))

    def memory(self) -> dict:
        out = (_i64 * 4)()
        _check(_lib.ted_model_memory(self._h, out))
        return dict(params_grads_optimizer=out[0], activations=out[1], checkpoint=out[2],
                    cac_stash=out[3])
