"""Reference-identical inputs for the model-stack parity tests: every parameter of
enumerate_params (moe.cpp:115-147) from seeded_init(shape, mix_seed(seed, name), scale)
(tensor.cpp:113-129; scales moe.cpp:119-121) and the batch seeded_init({N_global, h},
mix_seed(seed, "batch"), 1.0) (moe.cpp:266-267).  Golden losses: SerialModel
(moe.cpp:899-1121) through the compiled reference, tests/golden/make_golden.py."""
import os

import numpy as np

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


def golden_losses(layers, h, E, n, seed, shards):
    g = np.load(GOLDEN)["stack_serial_losses"]
    for row in g:
        if tuple(int(v) for v in row[:6]) == (layers, h, E, n, seed, shards):
            return row[6:]
    raise KeyError((layers, h, E, n, seed, shards))


def scale_of(name, h):
    f = 4 * h
    leaf = name.rsplit(".", 1)[1]
    if name.endswith("gate.w") or leaf == "w1":
        return 1.0 / np.sqrt(h)
    if leaf == "w2":
        return 1.0 / np.sqrt(f)
    return 0.1


def stack_params(ted, model):
    out = {}
    for nm in ted.param_names(model):
        shape = ted.param_shape(model, nm)
        size = int(np.prod(shape))
        out[nm] = O.seeded_init(size, O.mix_seed(model.seed, nm),
                                scale_of(nm, model.hidden)).reshape(shape)
    return out


def stack_batch(model, shards):
    n, h = model.tokens_per_shard, model.hidden
    a = O.seeded_init(shards * n * h, O.mix_seed(model.seed, "batch"), 1.0)
    return a.reshape(shards * n, h)
