"""Seeded random layer configurations through the full GPU forward, each
checked stage by stage against the oracle exactly like the named cases of
test_forward_gpu.py (routing / permutation bit-exact, FFN rows, combine and
end-to-end tokens within tolerance): expert counts 2-128, top-k 1-4, d_model
and d_ff multiples of 256 (bf16) or 64 (fp32), resident subsets of every
size, both CTA groups, both activations and weight modes, ragged T."""
import numpy as np
import pytest

import test_forward_gpu as fw

pytestmark = pytest.mark.gpu


def random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    dtype = "fp32" if seed % 5 == 4 else "bf16"
    E = int(rng.choice([2, 4, 8, 16, 32, 64, 128]))
    k = int(rng.integers(1, min(4, E) + 1))
    act = "swiglu" if rng.random() < 0.6 else "relu"
    wm = "topk_softmax" if rng.random() < 0.5 else "full_softmax"
    if dtype == "bf16":
        d = int(rng.choice([256, 512, 768, 1024]))
        f = int(rng.choice([256, 512, 1024, 1536]))
    else:
        d = int(rng.choice([128, 256, 512]))
        f = int(rng.choice([256, 512, 768]))
    slots = int(rng.integers(1, E + 1))
    resident = sorted(rng.choice(E, slots, replace=False).tolist())
    T = int(rng.integers(1, 2500))
    cg = int(rng.choice([0, 1, 2])) if dtype == "bf16" else 0
    return (E, d, f, k, dtype, act, wm, slots, resident, T, cg)


@pytest.mark.parametrize("seed", range(40))
def test_random_layer_parity(seed, port):
    name = f"random_{seed}"
    fw.CASES[name] = random_case(seed)
    try:
        c = fw.run_case(name, port)
        fw.check_case(c, port)
        c["layer"].close()
    finally:
        del fw.CASES[name]
