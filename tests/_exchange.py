"""Host-side TED exchange, driven by the product's planner (libted_plan.so, the same
ted_plan.h compiled into libted_b200.so), with numpy buffers.  Used by the CPU tests to
check the multi-rank dispatch / DTD / return bookkeeping against an independent
restatement of the reference's ordering rules (moe.cpp:454-556)."""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_PLAN = None


def plan_lib():
    global _PLAN
    if _PLAN is None:
        path = os.path.join(ROOT, "paper_2303_06318_b200", "libted_plan.so")
        L = C.CDLL(path)
        L.ted_plan_build.restype = C.c_int
        L.ted_plan_last_error.restype = C.c_char_p
        _PLAN = L
    return _PLAN


def build_plan(P, T, E, dtd, my_ep, my_t, cnt):
    """cnt: int32 [P][Tc][E].  Returns a dict mirroring ted::LayerPlan."""
    Eloc = E // P if E % P == 0 else 1
    dtd = bool(dtd) and T > 1
    Tc = T if dtd else 1
    cap = 4 * (P * Eloc + T * Eloc + T) + 8
    seg_off = np.zeros(Eloc + 1, np.int32)
    seg_rows = np.zeros(Eloc, np.int32)
    chunk_row = np.zeros(Tc + 1, np.int64)
    send_off = np.zeros(E, np.int64)
    lists = np.zeros((6, cap, 3), np.int64)
    counts = np.zeros(6, np.int32)
    totals = np.zeros(4, np.int64)
    cnt = np.ascontiguousarray(cnt, np.int32)
    rc = plan_lib().ted_plan_build(
        P, T, E, int(dtd), my_ep, my_t, cnt.ctypes.data_as(C.c_void_p),
        seg_off.ctypes.data_as(C.c_void_p), seg_rows.ctypes.data_as(C.c_void_p),
        chunk_row.ctypes.data_as(C.c_void_p), send_off.ctypes.data_as(C.c_void_p),
        lists.ctypes.data_as(C.c_void_p), cap, counts.ctypes.data_as(C.c_void_p),
        totals.ctypes.data_as(C.c_void_p))
    if rc != 0:
        raise ValueError(plan_lib().ted_plan_last_error().decode())
    names = ["a2a_send", "a2a_recv", "ag_asm_send", "ag_asm_recv", "ag_home_send", "ag_home_recv"]
    out = {nm: [tuple(int(v) for v in lists[i, j]) for j in range(counts[i])]
           for i, nm in enumerate(names)}
    out.update(seg_off=seg_off, seg_rows=seg_rows, chunk_row=chunk_row, send_off=send_off,
               asm_rows=int(totals[0]), send_rows=int(totals[1]), a2a_offrank=int(totals[2]),
               a2a_total=int(totals[3]), Eloc=Eloc, Tc=Tc, dtd=dtd)
    return out


def route_shard(expert, E, cap, Tc):
    """Independent numpy restatement of slot / keep / kept counts / home positions."""
    n = expert.shape[0]
    slot = np.zeros(n, np.int64)
    seen = np.zeros(E, np.int64)
    for k in range(n):
        slot[k] = seen[expert[k]]
        seen[expert[k]] += 1
    keep = slot < cap
    chunk = (np.arange(n) // (n // Tc)).clip(max=Tc - 1)
    kc = np.zeros((Tc, E), np.int64)
    for k in range(n):
        if keep[k]:
            kc[chunk[k], expert[k]] += 1
    # home layout: chunk-major, experts ascending, ascending tokens
    pos_home = -np.ones(n, np.int64)
    base = 0
    for c in range(Tc):
        for e in range(E):
            ks = [k for k in range(n) if chunk[k] == c and expert[k] == e and keep[k]]
            for i, k in enumerate(ks):
                pos_home[k] = base + i
            base += len(ks)
    return slot, keep, chunk, kc, pos_home


def send_rows_of(a, expert, keep, chunk, my_c, E, dtd):
    rows = []
    for e in range(E):
        for k in range(a.shape[0]):
            if keep[k] and expert[k] == e and (not dtd or chunk[k] == my_c):
                rows.append(a[k])
    return np.array(rows).reshape(-1, a.shape[1])


def expected_expert_rows(shards, e, Tc, P):
    """Reference order of expert e's input rows: DTD member (chunk) major, then source
    member, then ascending token (moe.cpp:465-489)."""
    out = []
    for c in range(Tc):
        for s in range(P):
            a, expert, keep, chunk = shards[s]
            for k in range(a.shape[0]):
                if keep[k] and expert[k] == e and chunk[k] == c:
                    out.append(a[k])
    return np.array(out).reshape(-1, shards[0][0].shape[1])
