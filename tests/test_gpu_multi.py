"""Multi-GPU parity (TP x EP with and without DTD) through torchrun; skipped unless the
box exposes enough GPUs.  See tests/mgpu_layer_check.py."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(nproc, *args, env=None, script="mgpu_layer_check.py", timeout=600):
    for _attempt in range(3):  # a freshly probed port can be taken before torchrun binds it
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
               os.path.join(HERE, script), *args]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout,
                               env=dict(os.environ, **(env or {})))
        except subprocess.TimeoutExpired as e:
            out = (e.stdout or b"").decode(errors="replace") if isinstance(e.stdout, bytes) else (e.stdout or "")
            err = (e.stderr or b"").decode(errors="replace") if isinstance(e.stderr, bytes) else (e.stderr or "")
            raise AssertionError(f"timed out after {timeout} s\n" + out[-4000:] + err[-4000:])
        if "EADDRINUSE" not in r.stderr + r.stdout:
            break
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "MGPU-OK" in r.stdout, r.stdout[-4000:]
    rep = os.environ.get("TED_MGPU_REPORT")  # collect the parity reports (worst_rel, ledger)
    if rep:
        with open(rep, "a") as f:
            for line in r.stdout.splitlines():
                if line.startswith("MGPU-OK "):
                    f.write(line[8:] + "\n")
    return r.stdout


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
@pytest.mark.parametrize("tp,ep,dtd", [(2, 1, 1), (2, 1, 0), (1, 2, 0)])
def test_two_gpus(tp, ep, dtd, exchange):
    """exchange=peer: NVLink peer-memory scatter/pull kernels; nccl: grouped send/recv."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, "--tp", str(tp), "--ep", str(ep), "--dtd", str(dtd),
         env={"TED_EXCHANGE": exchange})


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
@pytest.mark.parametrize("tp,ep,dtd,E", [(2, 2, 1, 8), (2, 2, 0, 8), (1, 4, 0, 16), (2, 1, 1, 4)])
def test_four_gpus(tp, ep, dtd, E, exchange):
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "--tp", str(tp), "--ep", str(ep), "--dtd", str(dtd), "--experts", str(E),
         env={"TED_EXCHANGE": exchange})


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_four_gpus_corrupt_drop_is_detected(exchange):
    """Fault injection (test_moe.cpp:388-414): dispatching the wrong DTD chunk fails the
    placement verdict every rank computes on the device (moe.cpp:537-556) and breaks the
    layer output, on both exchange implementations."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "--tp", "2", "--ep", "2", "--dtd", "1", "--corrupt", "1", "--cf", "0",
         env={"TED_EXCHANGE": exchange})


def test_two_gpus_corrupt_drop_is_detected():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, "--tp", "2", "--ep", "1", "--dtd", "1", "--corrupt", "1", "--cf", "0",
         "--experts", "4")


@pytest.mark.parametrize("nproc,tp,ep,E", [(2, 2, 1, 2), (4, 2, 2, 4)])
def test_wide_layer_h4096(nproc, tp, ep, E):
    """The north-star width (d=4096, ffn=16384, TP-sharded to 8192) over TP x EP with DTD,
    128 tokens per shard so the fp64 oracle over all shards stays within minutes."""
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    _run(nproc, "--tp", str(tp), "--ep", str(ep), "--dtd", "1", "--experts", str(E),
         "--hidden", "4096", "--tokens", "128")


@pytest.mark.parametrize("nproc,tp,ep,zero", [(2, 2, 1, 1), (2, 1, 2, 1), (2, 1, 1, 1),
                                              (4, 2, 2, 1), (4, 2, 1, 1), (4, 2, 1, 0)])
def test_model_stack_matches_reference(nproc, tp, ep, zero):
    """Whole model (attention stand-in + MoE / dense FFN, 2 layers) over TP x EP x DP, with
    and without ZeRO-1, against the reference SerialModel losses (tests/mgpu_model_check.py)."""
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    _run(nproc, "--tp", str(tp), "--ep", str(ep), "--zero", str(zero),
         script="mgpu_model_check.py")


@pytest.mark.parametrize("dtd", [0, 1])
def test_four_gpus_ledger_matches_predict_comm_volume(dtd):
    """E = EP = 2, TP = 2, h = 256, n = 1024, no capacity drops: the forward all-to-all and
    DTD all-gather payload bytes the layer accounts on the real exchange path, summed over
    ranks, equal the reference's predict_comm_volume (tests/golden)."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "--tp", "2", "--ep", "2", "--dtd", str(dtd), "--experts", "2", "--hidden", "256",
         "--tokens", "1024", "--cf", "0", "--ledger", "1")


@pytest.mark.parametrize("ckpt,cac", [(1, 0), (1, 1)])
def test_model_stack_checkpointing_four_gpus(ckpt, cac):
    """Activation checkpointing, live and with CAC replay of the recorded exchange and
    all-reduce outputs, over TP2 x EP2: the reference SerialModel's losses."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "--tp", "2", "--ep", "2", "--ckpt", str(ckpt), "--cac", str(cac),
         script="mgpu_model_check.py")


@pytest.mark.parametrize("E,cf", [(64, 1.0), (32, 1.5), (64, 2.0)])
def test_four_gpus_routing_stress(E, cf):
    """configs[4] (C5) at 4 GPUs: skewed gate (Zipf-like column scales), 32-64 experts,
    capacity factor 1.0-2.0 with heavy drops on the popular experts, TP2 x EP2 with DTD:
    outputs and gradients against the oracle run serially over all shards."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "--tp", "2", "--ep", "2", "--dtd", "1", "--experts", str(E), "--cf", str(cf),
         "--skew", "3.0", "--tokens", "1024")


@pytest.mark.parametrize("nproc,tp,ep,dtd", [(2, 2, 1, 1), (4, 2, 2, 1), (4, 2, 2, 0)])
def test_step_graph_matches_separate_calls(nproc, tp, ep, dtd):
    """ted_layer_step on the peer path (device-side exchange plan, fused AdamW, replayed
    CUDA graph) leaves the same parameters as forward / backward / optimizer_step."""
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    out = _run(nproc, "--tp", str(tp), "--ep", str(ep), "--dtd", str(dtd), "--experts", "8",
               "--step-check", "1")
    assert "step-check" in out


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_two_gpus_stalled_peer_times_out(exchange):
    """A peer that never reaches the backward: rank 0 gets TimeoutError (status 1) after the
    collective timeout instead of a hang or a trapped context (fabric.cpp:65-96)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    out = _run(2, "--tp", "2", "--ep", "1", "--dtd", "1", "--experts", "4", "--stall", "1",
               env={"TED_EXCHANGE": exchange, "NCCL_DEBUG": "WARN"}, timeout=180)
    assert "TimeoutError" in out


# The reference's verify sweep (harness.cpp:254-278): every valid (tensor, experts) split of
# worlds 2 and 4 at hidden 8, 8 tokens per shard, 1 layer, DTD when T > 1, with
# checkpointing + CAC -- losses against the reference SerialModel (the shapes run
# zero-padded to the 256 tensor-core tile).
SWEEP = [(w, t, e) for w in (2, 4) for t in range(1, w + 1) if w % t == 0
         for e in range(1, min(w // t, 4) + 1) if (w // t) % e == 0]


@pytest.mark.parametrize("world,tp,ep", SWEEP)
def test_verify_sweep_small_shapes(world, tp, ep):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    _run(world, "--tp", str(tp), "--ep", str(ep), "--dtd", str(int(tp > 1)), "--ckpt", "1",
         "--cac", "1", "--layers", "1", "--hidden", "8", "--experts", str(ep), "--tokens", "8",
         "--seed", "1", script="mgpu_model_check.py")
