"""Multi-rank host logic on CPU: the exchange planner that drives the NCCL calls
(ted_plan.h via libted_plan.so), simulated over a whole TED world in-process (the
reference's own testing model: ranks as in-process peers, fabric.cpp) and over real
gloo process groups (world size 2 and 4).

Checks, against an independent numpy restatement of the reference's ordering rules:
  * each expert's assembled input rows = kept tokens in (DTD member, source member,
    ascending token) order (moe.cpp:465-489; test_moe.cpp:201-286);
  * DTD keeps the same row SET per expert and cuts dispatch all-to-all rows by exactly T
    (acceptance_test.cpp:166-195);
  * the return trip + home all-gather puts each token's expert output at the position
    the GPU combine kernel reads (pos_home), dropped tokens nowhere (moe.cpp:504-556);
  * ledger bytes equal the reference's predict_comm_volume (cost_model.cpp:346-416).
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import _exchange as X


def _world(T, P, E, n, h, cf, dtd, seed):
    rng = np.random.default_rng(seed)
    Tc = T if (dtd and T > 1) else 1
    shards = []
    cnt = np.zeros((P, Tc, E), np.int32)
    homes = []
    cap = O.capacity(cf, n, E)
    for s in range(P):
        a = rng.standard_normal((n, h))
        logits = rng.standard_normal((n, E)) + np.linspace(1.0, 0.0, E) * (seed % 3)
        expert, _, _ = O.gate_route_logits(logits)
        slot, keep, chunk, kc, pos_home = X.route_shard(expert, E, cap, Tc)
        # the oracle's capacity routing agrees with the restatement
        os_, ok, okc = O.route_capacity(expert, E, cap, Tc)
        np.testing.assert_array_equal(os_, slot)
        np.testing.assert_array_equal(okc, kc)
        cnt[s] = kc
        shards.append((a, expert, keep, chunk))
        homes.append(pos_home)
    return shards, cnt, homes, Tc


def _simulate(T, P, E, n, h, cf, dtd, seed):
    shards, cnt, homes, Tc = _world(T, P, E, n, h, cf, dtd, seed)
    Eloc = E // P
    ranks = [(t, ep) for ep in range(P) for t in range(T)]
    plans = {r: X.build_plan(P, T, E, dtd, r[1], r[0], cnt) for r in ranks}
    sendbuf, asm = {}, {}
    for (t, ep) in ranks:
        a, expert, keep, chunk = shards[ep]
        pl = plans[(t, ep)]
        sendbuf[(t, ep)] = X.send_rows_of(a, expert, keep, chunk, t, E, pl["dtd"])
        assert sendbuf[(t, ep)].shape[0] == pl["send_rows"]
        asm[(t, ep)] = np.zeros((max(pl["asm_rows"], 1), h))
    # EP all-to-all: k-th send to peer m matches k-th recv from me at m (NCCL p2p order)
    for (t, ep) in ranks:
        sends = {}
        for peer, row, rows in plans[(t, ep)]["a2a_send"]:
            sends.setdefault(peer, []).append(sendbuf[(t, ep)][row:row + rows])
        for m, msgs in sends.items():
            recvs = [x for x in plans[(t, m)]["a2a_recv"] if x[0] == ep]
            assert len(recvs) == len(msgs)
            for (pp, row, rows), msg in zip(recvs, msgs):
                assert msg.shape[0] == rows
                asm[(t, m)][row:row + rows] = msg
    # DTD all-gather-v over the TP group
    if Tc > 1:
        snap = {r: asm[r].copy() for r in ranks}
        for (t, ep) in ranks:
            for peer, row, rows in plans[(t, ep)]["ag_asm_recv"]:
                src = [x for x in plans[(peer, ep)]["ag_asm_send"] if x[0] == t]
                got = [x for x in plans[(t, ep)]["ag_asm_recv"] if x[0] == peer]
                for (p2, srow, srows), (p3, drow, drows) in zip(src, got):
                    assert srows == drows
                    asm[(t, ep)][drow:drow + drows] = snap[(peer, ep)][srow:srow + srows]
    # expert inputs in the reference order, pads zero, identical on TP peers
    for (t, ep) in ranks:
        pl = plans[(t, ep)]
        assert all(v % 128 == 0 for v in pl["seg_off"])
        for le in range(Eloc):
            e = ep * Eloc + le
            lo, rows = pl["seg_off"][le], pl["seg_rows"][le]
            want = X.expected_expert_rows([shards[s] for s in range(P)], e, Tc, P)
            np.testing.assert_array_equal(asm[(t, ep)][lo:lo + rows], want)
            assert not asm[(t, ep)][lo + rows:pl["seg_off"][le + 1]].any()
        np.testing.assert_array_equal(asm[(t, ep)], asm[(0, ep)])
    # return trip: expert "output" f(x) = 3x + 1 on the rows this rank received
    home = {r: np.zeros((n, h)) for r in ranks}
    for (t, ep) in ranks:
        pl = plans[(t, ep)]
        out = 3 * asm[(t, ep)] + 1
        my_c = t if pl["dtd"] else 0
        for src, row, rows in pl["a2a_recv"]:  # goes back to source `src` (same t)
            recvs = [x for x in plans[(t, src)]["a2a_send"] if x[0] == ep]
            sends = [x for x in pl["a2a_recv"] if x[0] == src]
            for (p1, srow, srows), (p2, drow, drows) in zip(sends, recvs):
                base = plans[(t, src)]["chunk_row"][my_c]
                home[(t, src)][base + drow:base + drow + drows] = out[srow:srow + srows]
    if Tc > 1:
        snap = {r: home[r].copy() for r in ranks}
        for (t, ep) in ranks:
            for peer, row, rows in plans[(t, ep)]["ag_home_recv"]:
                home[(t, ep)][row:row + rows] = snap[(peer, ep)][row:row + rows]
    for (t, ep) in ranks:
        a, expert, keep, chunk = shards[ep]
        ph = homes[ep]
        for k in range(n):
            if keep[k]:
                np.testing.assert_array_equal(home[(t, ep)][ph[k]], 3 * a[k] + 1)
            else:
                assert ph[k] == -1
    return plans, cnt


@pytest.mark.parametrize("T,P,E,dtd", [(1, 1, 4, False), (2, 1, 4, True), (1, 2, 4, False),
                                       (2, 2, 4, True), (2, 2, 4, False), (2, 4, 16, True),
                                       (2, 4, 16, False), (4, 2, 8, True), (1, 8, 64, False)])
@pytest.mark.parametrize("cf", [0.0, 1.25])
def test_world_exchange_matches_reference_order(T, P, E, dtd, cf):
    _simulate(T, P, E, n=64, h=4, cf=cf, dtd=dtd, seed=T * 10 + P + E)


def test_dtd_cuts_dispatch_rows_by_T_and_keeps_row_sets():
    """acceptance_test.cpp:166-195: DTD all-to-all bytes are exactly 1/T."""
    for T, P, E in [(2, 4, 16), (2, 2, 4), (4, 2, 8)]:
        p_off, _ = _simulate(T, P, E, 64, 4, 0.0, False, 5)
        p_on, _ = _simulate(T, P, E, 64, 4, 0.0, True, 5)
        off = sum(p["a2a_total"] for p in p_off.values())
        on = sum(p["a2a_total"] for p in p_on.values())
        assert off == T * on


def test_ledger_bytes_match_predict_comm_volume():
    """Our per-rank payload accounting summed over ranks == the reference's closed form
    (tests/golden: predict_comm_volume at world 4 (T=2,E=2) h=256 n=1024 and world 8
    (T=2,E=4) h=4096 n=8192, DTD off/on, forward phase)."""
    gold = np.load(O.HERE + "/../tests/golden/golden.npz")
    for world, tp, ex, h, n, dtd, a2a, ag, ar in gold["predict_comm"]:
        P, T = int(ex), int(tp)
        rng = np.random.default_rng(1)
        Tc = T if dtd else 1
        cnt = np.zeros((P, Tc, P), np.int32)
        for s in range(P):  # any routing: payload is routing-independent (cost_model.cpp:363)
            ex_ = rng.integers(0, P, int(n)).astype(np.int32)
            _, _, kc = O.route_capacity(ex_, P, int(n), Tc)
            cnt[s] = kc
        a2a_sum = ag_sum = 0
        for ep in range(P):
            for t in range(T):
                pl = X.build_plan(P, T, P, bool(dtd), ep, t, cnt)
                a2a_sum += 2 * pl["a2a_total"] * h * 2  # dispatch + return, self included
                ag_sum += sum(x[2] for x in pl["ag_asm_send"] + pl["ag_home_send"]) * h * 2
        assert a2a_sum == a2a
        assert ag_sum == ag
        assert ar == 2 * world * n * h * 2  # attention + expert TP all-reduce sites


def test_planner_rejects_bad_config():
    with pytest.raises(ValueError):
        X.build_plan(3, 1, 4, False, 0, 0, np.zeros((3, 1, 4), np.int32))


# ------------------------------------------------------------------ gloo, real processes

def _gloo_worker(rank, world, T, P, E, dtd, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n, h, cf = 64, 8, 1.25
        t, ep = rank % T, rank // T
        Tc = T if (dtd and T > 1) else 1
        rng = np.random.default_rng(100 + ep)  # shard ep's tokens, replicated over TP
        a = rng.standard_normal((n, h)).astype(np.float32)
        expert, _, _ = O.gate_route_logits(rng.standard_normal((n, E)))
        cap = O.capacity(cf, n, E)
        slot, keep, chunk, kc, pos_home = X.route_shard(expert, E, cap, Tc)
        # count exchange over the EP group (all-gather of [Tc][E] counts)
        mine = torch.from_numpy(kc.astype(np.int32).reshape(-1))
        allc = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allc, mine)
        cnt = np.stack([allc[t + T * s].numpy().reshape(Tc, E) for s in range(P)])
        pl = X.build_plan(P, T, E, dtd, ep, t, cnt)
        send = X.send_rows_of(a, expert, keep, chunk, t, E, pl["dtd"]).astype(np.float32)
        asm = torch.zeros(max(pl["asm_rows"], 1), h)
        # grouped p2p exactly as layer.cu issues it (sends then recvs, per peer order)
        reqs = []
        for peer, row, rows in pl["a2a_send"]:
            dst = t + T * peer
            if dst == rank:
                continue
            reqs.append(dist.isend(torch.from_numpy(send[row:row + rows].copy()), dst))
        selfq = [(r, rr) for (p, r, rr) in pl["a2a_send"] if p == ep]
        recvbufs = []
        for peer, row, rows in pl["a2a_recv"]:
            src = t + T * peer
            if src == rank:
                srow, srows = selfq.pop(0)
                asm[row:row + rows] = torch.from_numpy(send[srow:srow + srows])
                continue
            buf = torch.zeros(rows, h)
            reqs.append(dist.irecv(buf, src))
            recvbufs.append((row, buf))
        for r in reqs:
            r.wait()
        for row, buf in recvbufs:
            asm[row:row + buf.shape[0]] = buf
        if pl["dtd"]:
            reqs, bufs = [], []
            for peer, row, rows in pl["ag_asm_send"]:
                reqs.append(dist.isend(asm[row:row + rows].clone(), peer + T * ep))
            for peer, row, rows in pl["ag_asm_recv"]:
                buf = torch.zeros(rows, h)
                reqs.append(dist.irecv(buf, peer + T * ep))
                bufs.append((row, buf))
            for r in reqs:
                r.wait()
            for row, buf in bufs:
                asm[row:row + buf.shape[0]] = buf
        # gather every shard's routing to build the expected rows on this rank
        allx = [None] * world
        dist.all_gather_object(allx, (a, expert, keep, chunk))
        shards = [allx[0 + T * s] for s in range(P)]
        Eloc = E // P
        for le in range(Eloc):
            e = ep * Eloc + le
            lo, rows = pl["seg_off"][le], pl["seg_rows"][le]
            want = X.expected_expert_rows(shards, e, Tc, P)
            np.testing.assert_array_equal(asm[lo:lo + rows].numpy(), want)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover - reported through the queue
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world,T,P,E,dtd", [(2, 1, 2, 4, False), (2, 2, 1, 4, True),
                                             (4, 2, 2, 8, True)])
def test_gloo_exchange(world, T, P, E, dtd):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, T, P, E, dtd, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


@pytest.mark.parametrize("P,T,E,dtd", [(2, 2, 4, 1), (4, 2, 16, 1), (4, 2, 16, 0), (1, 2, 8, 1),
                                       (4, 1, 8, 0), (2, 4, 8, 1)])
def test_device_plan_matches_host_planner(P, T, E, dtd):
    """The peer path's device plan (peer_plan_expert, run by plan_peer_kernel; here through
    its CPU build) places every rank's rows exactly where the host planner's assembled
    layout puts them (build_plan's blk_row / seg_off, the layout the NCCL path and the
    reference ordering tests use)."""
    L = X.plan_lib()
    Tc = T if (dtd and T > 1) else 1
    Eloc = E // P
    rng = np.random.default_rng(P * 100 + T * 10 + E + dtd)
    cnt = rng.integers(0, 300, (P, Tc, E)).astype(np.int32)
    plane = np.zeros((P * T, Tc, E), np.int32)  # member t + T*ep; TP peers agree
    for ep in range(P):
        for t in range(T):
            plane[t + T * ep] = cnt[ep]
    blocks = {}
    for ep2 in range(P):
        br = np.zeros(Eloc * Tc * P, np.int64)
        bc = np.zeros(Eloc * Tc * P, np.int32)
        assert L.ted_plan_blocks(P, T, E, dtd, ep2, 0, cnt.ctypes.data_as(C.c_void_p),
                                 br.ctypes.data_as(C.c_void_p), bc.ctypes.data_as(C.c_void_p)) == 0
        blocks[ep2] = br.reshape(Eloc, Tc, P)
    for ep in range(P):
        for t in range(T):
            my_c = t if Tc > 1 else 0
            seg = np.zeros(2 * Eloc + 1, np.int32)
            disp = np.zeros(E, np.int64)
            pull = np.zeros(Tc * E, np.int64)
            assert L.ted_plan_peer_tables(T, P, E, Tc, ep, my_c, plane.ctypes.data_as(C.c_void_p),
                                          seg.ctypes.data_as(C.c_void_p),
                                          disp.ctypes.data_as(C.c_void_p),
                                          pull.ctypes.data_as(C.c_void_p)) == 0
            pull = pull.reshape(Tc, E)
            for e in range(E):
                ep2, le = divmod(e, Eloc)
                for c in range(Tc):
                    assert pull[c, e] == blocks[ep2][le, c, ep]
                assert disp[e] == blocks[ep2][le, my_c, ep]
            pl = X.build_plan(P, T, E, dtd, ep, t, cnt)
            np.testing.assert_array_equal(seg[:Eloc + 1], pl["seg_off"])
            np.testing.assert_array_equal(seg[Eloc + 1:], pl["seg_rows"])
