"""C-ABI checks that need no GPU: the library loads, exports every entry point declared in
include/ted.h, mirrors the reference's config validation (derive_config, shard_range,
status 2 = InvalidConfigError), and refuses compute without an sm_100 device (no CPU
fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2303_06318_b200 as ted
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ted.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ted_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", ted.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ted_[a-z0-9_]+)$", out, flags=re.M))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    assert len(_declared()) >= 25


def test_python_mirror_binds_every_symbol():
    for s in _declared():
        assert hasattr(ted.lib(), s), s
    assert set(ted.EXPORTED) <= set(_declared())


def test_defaults_mirror_the_reference():
    m, t, f, a, ti = ted.ModelCfg(), ted.TopoCfg(), ted.FlagsC(), ted.AdamC(), ted.TileC()
    import ctypes as C
    ted.lib().ted_default_configs(C.byref(m), C.byref(t), C.byref(f), C.byref(a), C.byref(ti))
    assert (m.layers, m.hidden, m.experts, m.tokens_per_shard, m.seed) == (1, 8, 2, 8, 1)
    assert (a.lr, a.beta1, a.beta2, a.eps, a.weight_decay) == (1e-4, 0.9, 0.999, 1e-8, 0.01)
    assert (ti.enabled, ti.tile_size) == (1, 1_800_000)


def test_derive_config_matches_reference_table():
    gold = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    for world, tp, ex, rc, *vals in gold["derive_config"]:
        if rc == 0:
            got = ted.derive_config(int(world), int(tp), int(ex))
            assert [got.world_size, got.tensor_parallel, got.experts, got.expert_data_parallel,
                    got.nonexpert_data_parallel] == [int(v) for v in vals]
        else:
            with pytest.raises(ted.InvalidConfigError):
                ted.derive_config(int(world), int(tp), int(ex))


def test_shard_range_matches_reference_and_rejects_bad_args():
    gold = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    for total, parts, i, b, e in gold["shard_range"]:
        assert ted.shard_range(int(total), int(parts), int(i)) == (b, e)
    for args in [(10, 0, 0), (10, 2, 2), (10, 2, -1), (-1, 2, 0)]:
        with pytest.raises(ted.InvalidConfigError):
            ted.shard_range(*args)


def test_capacity_formula():
    assert ted.capacity(0.0, 2048, 4) == 2048
    assert ted.capacity(1.25, 1024, 4) == 320 == O.capacity(1.25, 1024, 4)
    assert ted.capacity(1.0, 16384, 8) == 2048


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    rc = ted.lib().ted_gate_forward(None, None, 16, 256, 8, None, None, None, None, None)
    assert rc == ted.TED_ERR_RUNTIME
    assert b"no CUDA device" in ted.lib().ted_last_error()
    with pytest.raises(ted.TedRuntimeError):
        ted.MoeLayer(ted.MoeModelConfig(1, 256, 4, 64, 1), ted.TedConfig())
    import ctypes as C
    a, t, pk = ted.AdamConfig().c(), ted.TileConfig().c(), C.c_uint64()
    rc = ted.lib().ted_adam_step(None, None, None, None, None, 0, 4, 1, C.byref(a), C.byref(t),
                                 C.byref(pk), None)
    assert rc == ted.TED_ERR_RUNTIME
    with pytest.raises(ted.TedRuntimeError):  # the whole model: no CPU path either
        ted.TedModel(ted.MoeModelConfig(2, 256, 4, 64, 1), ted.TedConfig())


def test_model_config_errors_are_config_status():
    """Model-level configuration errors map to InvalidConfigError (status 2) before any
    device work, like the reference's validate_model (moe.cpp:100-113)."""
    with pytest.raises(ted.InvalidConfigError, match="layers must be >= 1"):
        ted.TedModel(ted.MoeModelConfig(0, 256, 4, 64, 1), ted.TedConfig())
    with pytest.raises(ted.InvalidConfigError, match="tensor_parallel"):
        ted.TedModel(ted.MoeModelConfig(2, 1, 8, 64, 1), ted.derive_config(8, 8, 1))


def test_plan_library_loads():
    from tests import _exchange as X
    pl = X.build_plan(2, 2, 4, True, 0, 1, np.ones((2, 2, 4), np.int32))
    assert pl["seg_off"][-1] % 128 == 0


def _build_example(tmp_path):
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / "layer_step")
    cmd = ["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(root, "examples", "layer_step.c"),
           "-L", os.path.join(root, "paper_2303_06318_b200"), "-lted_b200",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,--allow-shlib-undefined", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe, root


def test_c_example_compiles_and_links(tmp_path):
    """include/ted.h is plain C: a C11 host program (the reference-side integration
    sketch of INTEGRATION.md) compiles with -Wall -Werror and links against the library."""
    _build_example(tmp_path)
