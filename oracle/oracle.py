"""TEST INFRASTRUCTURE ONLY -- ctypes face of the CPU oracle.

Two libraries live under ``oracle/``:

* ``liboracle.so``  -- our plain-C fp64 restatement of the reference hot path
  (``ted_oracle.c``; every function cites the reference file:line it follows);
* ``_ref/libtedsim_ref.so`` -- the UNMODIFIED reference (tedsim) compiled from
  ``/root/reference/proj/core/src`` plus ``ref_shim.cpp`` (built here, travels to
  the GPU box as a prebuilt file; git-ignored).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or the
timed reference arm -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE = None
_REF = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def _opt(ptr_type):
    """ndpointer that also accepts None."""

    class _P(ptr_type):  # type: ignore[misc, valid-type]
        @classmethod
        def from_param(cls, obj):
            if obj is None:
                return None
            return super().from_param(obj)

    return _P


_dpo, _ipo, _upo = _opt(_dp), _opt(_ip), _opt(_up)


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and the reference lib when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj/core/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def lib():
    global _ORACLE
    if _ORACLE is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.o_mix_seed.restype = C.c_uint64
        L.o_mix_seed.argtypes = [C.c_uint64, C.c_char_p]
        L.o_seeded_init.argtypes = [_dp, C.c_int64, C.c_uint64, C.c_double]
        L.o_gate_route_logits.argtypes = [_dp, C.c_int64, C.c_int, _ip, _dp, _dp]
        L.o_gate_forward.argtypes = [_dp, _dp, C.c_int64, C.c_int, C.c_int, _dp, _ip, _dp, _dp]
        L.o_gate_backward.argtypes = [_dp, _dp, _dp, _ip, _dp, C.c_int64, C.c_int, C.c_int,
                                      _dpo, _dpo]
        L.o_capacity.restype = C.c_int64
        L.o_capacity.argtypes = [C.c_double, C.c_int64, C.c_int]
        L.o_route_capacity.argtypes = [_ip, C.c_int64, C.c_int, C.c_int64, C.c_int, _ipo, _upo,
                                       _ipo]
        L.o_gelu.restype = C.c_double
        L.o_gelu.argtypes = [C.c_double]
        L.o_gelu_grad.restype = C.c_double
        L.o_gelu_grad.argtypes = [C.c_double]
        L.o_moe_layer.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double,
                                  _dp, _dp, _dp, _dp, _dp, _dp, _dpo, _dpo,
                                  C.POINTER(C.c_double), _dpo, _dpo, _dpo, _dpo, _dpo, _dpo,
                                  _ipo, _ipo, _upo, _dpo, _dpo]
        L.o_shard_range.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64)]
        L.o_adam_step_owned.restype = C.c_uint64
        L.o_adam_step_owned.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                        C.c_double, C.c_double, C.c_double, C.c_int, C.c_int64,
                                        _dp, _dp, _dp, _dp, _dpo]
        _ORACLE = L
    return _ORACLE


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libtedsim_ref.so"))


def ref():
    """The compiled reference (raises if it was never built)."""
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libtedsim_ref.so")
        if not os.path.exists(path):
            build(ref=True)
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_char_p]
        L.ref_seeded_init.argtypes = [_dp, C.c_int64, C.c_uint64, C.c_double]
        L.ref_gate_forward.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, _ip, _dp, _dp]
        L.ref_gate_backward.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_gelu.restype = C.c_double
        L.ref_gelu.argtypes = [C.c_double]
        L.ref_gelu_grad.restype = C.c_double
        L.ref_gelu_grad.argtypes = [C.c_double]
        L.ref_moe_sublayer.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp,
                                       _dp, _dp, _dpo, _dpo, _dpo, _dpo, _dpo, _dpo, _dpo, _dpo,
                                       C.c_int]
        L.ref_adam.argtypes = [C.c_int64, _dp, C.c_int, C.c_int, C.c_double, C.c_double,
                               C.c_double, C.c_double, C.c_double, C.c_int, C.c_int64, C.c_int,
                               _dp, _dp, _dpo, _dpo, _dpo, C.POINTER(C.c_uint64)]
        L.ref_shard_range.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]
        L.ref_derive_config.argtypes = [C.c_int, C.c_int, C.c_int, _ip]
        L.ref_serial_step.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                      C.c_int, _dp]
        L.ref_trainer_step.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_predict_comm.argtypes = [C.c_int] * 9 + [np.ctypeslib.ndpointer(np.uint64)]
        _REF = L
    return _REF


# --------------------------------------------------------------------------- helpers

def seeded_init(n: int, seed: int, scale: float) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().o_seeded_init(out, n, seed, scale)
    return out


def mix_seed(seed: int, tag: str) -> int:
    return int(lib().o_mix_seed(seed, tag.encode()))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float64 (exactly representable)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp64 -> bf16 bit patterns (uint16), round-to-nearest-even."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF).astype(np.uint16)


def bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def gate_route_logits(logits: np.ndarray):
    n, E = logits.shape
    L = np.ascontiguousarray(logits, np.float64)
    expert = np.empty(n, np.int32)
    chosen = np.empty(n, np.float64)
    probs = np.empty((n, E), np.float64)
    lib().o_gate_route_logits(L, n, E, expert, chosen, probs)
    return expert, chosen, probs


def route_capacity(expert: np.ndarray, E: int, cap: int, T: int = 1):
    n = expert.shape[0]
    slot = np.empty(n, np.int32)
    keep = np.empty(n, np.uint8)
    counts = np.empty((T, E), np.int32)
    lib().o_route_capacity(np.ascontiguousarray(expert, np.int32), n, E, cap, T, slot, keep,
                           counts)
    return slot, keep, counts


def capacity(cf: float, n: int, E: int) -> int:
    return int(lib().o_capacity(cf, n, E))


def moe_layer(S, n, h, f, E, cf, a, wg, w1, b1, w2, b2, dy=None, backward=True):
    """fp64 oracle of the MoE branch; returns a dict of numpy arrays."""
    N = S * n
    out = dict(
        y=np.empty((N, h)), expert=np.empty(N, np.int32), slot=np.empty(N, np.int32),
        keep=np.empty(N, np.uint8), logits=np.empty((N, E)), probs=np.empty((N, E)))
    if backward:
        out.update(da=np.empty((N, h)), dwg=np.empty((h, E)), dw1=np.empty((E, h, f)),
                   db1=np.empty((E, f)), dw2=np.empty((E, f, h)), db2=np.empty((E, h)))
    loss = C.c_double(0.0)
    c = lambda x: None if x is None else np.ascontiguousarray(x, np.float64)  # noqa: E731
    g = out.get
    lib().o_moe_layer(S, n, h, f, E, cf, c(a), c(wg), c(w1), c(b1), c(w2), c(b2), c(dy),
                      out["y"], C.byref(loss), g("da"), g("dwg"), g("dw1"), g("db1"), g("dw2"),
                      g("db2"), out["expert"], out["slot"], out["keep"], out["logits"],
                      out["probs"])
    out["loss"] = loss.value
    return out


def make_layer_inputs(S, n, h, f, E, seed, bf16=True):
    """Inputs generated exactly like the reference (seeded_init + mix_seed over the
    parameter names of enumerate_params, moe.cpp:115-156, batch moe.cpp:266-267),
    optionally rounded to bf16 so GPU and oracle see identical values."""
    rnd = bf16_round if bf16 else (lambda x: x)
    sin, sout = 1.0 / np.sqrt(h), 1.0 / np.sqrt(f)
    a = seeded_init(S * n * h, mix_seed(seed, "batch"), 1.0).reshape(S * n, h)
    wg = seeded_init(h * E, mix_seed(seed, "layer0.gate.w"), sin).reshape(h, E)
    w1 = np.stack([seeded_init(h * f, mix_seed(seed, f"layer0.expert{e}.w1"), sin).reshape(h, f)
                   for e in range(E)])
    b1 = np.stack([seeded_init(f, mix_seed(seed, f"layer0.expert{e}.b1"), 0.1) for e in range(E)])
    w2 = np.stack([seeded_init(f * h, mix_seed(seed, f"layer0.expert{e}.w2"), sout).reshape(f, h)
                   for e in range(E)])
    b2 = np.stack([seeded_init(h, mix_seed(seed, f"layer0.expert{e}.b2"), 0.1) for e in range(E)])
    return dict(a=rnd(a), wg=rnd(wg), w1=rnd(w1), b1=rnd(b1), w2=rnd(w2), b2=rnd(b2))


def adam_step_owned(begin, end, step, grad_full, master, m1, m2, out_full=None, lr=1e-4,
                    b1=0.9, b2=0.999, eps=1e-8, wd=0.01, tiles_enabled=True,
                    tile_size=1_800_000):
    return int(lib().o_adam_step_owned(begin, end, step, lr, b1, b2, eps, wd,
                                       int(tiles_enabled), tile_size, grad_full, master, m1, m2,
                                       out_full))


def shard_range(total, parts, index):
    b, e = C.c_int64(), C.c_int64()
    lib().o_shard_range(total, parts, index, C.byref(b), C.byref(e))
    return b.value, e.value
