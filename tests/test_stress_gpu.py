"""Soak test of the layer under interleaved operations: forwards of random
size (device and async host-buffer), expert swaps started mid-stream
(evictions at load start, loads resident at completion, polled without
blocking by the next forward), score updates.  After every forward the
residency that forward used is mirrored onto a reference layer with the
same weights (blocking loads) and the outputs must be bit-identical: the
side-stream loads never race the compute that reads the slot pool."""
import numpy as np
import pytest
import torch

from helpers import build_layer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1])
def test_interleaved_forwards_loads_and_host_calls(seed):
    E, d, f, k, L = 8, 512, 1024, 2, 4
    rng = np.random.default_rng(seed)
    a, _, _ = build_layer(E, d, f, k, "bf16", "swiglu", "topk_softmax", L, [0, 1, 2, 3], max_tokens=4096)
    b, _, _ = build_layer(E, d, f, k, "bf16", "swiglu", "topk_softmax", L, [0, 1, 2, 3], max_tokens=4096)
    g = torch.Generator().manual_seed(seed)
    checked = 0
    for step in range(40):
        op = rng.random()
        if op < 0.3:  # start a swap of 1-2 experts; it completes while later forwards run
            res = np.flatnonzero(a.residency())
            non = np.flatnonzero(a.residency() == 0)
            n = int(rng.integers(1, 3))
            ev = sorted(rng.choice(res, n, replace=False).tolist())
            ld = sorted(rng.choice(non, n, replace=False).tolist())
            try:
                a.begin_load(ev, ld)
            except Exception:
                a.poll_loads(blocking=True)  # a previous plan still pending: plans apply in order
                continue
        elif op < 0.4:
            sc = rng.random(E)
            a.set_scores(sc)
            b.set_scores(sc)
        else:
            T = int(rng.integers(1, 4096))
            x = torch.randn(T, d, generator=g).to(torch.bfloat16)
            if op < 0.7:
                y = a.forward(x.cuda()).cpu()
            else:
                xh = x.pin_memory()
                yh = torch.empty_like(xh).pin_memory()
                a.forward_host_async(xh, yh)
                a.wait_host()
                y = yh.clone()
            used = a.residency()
            b.load_initial(np.flatnonzero(used).tolist())
            y_ref = b.forward(x.cuda()).cpu()
            assert torch.equal(y, y_ref), f"step {step}: output differs from a layer with the same residency"
            checked += 1
    a.poll_loads(blocking=True)
    assert checked >= 15
    a.close()
    b.close()
