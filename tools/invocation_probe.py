"""Latency of one predictor invocation (emoe_invocation_host: predict ->
per-task modulation -> Eq. 2 -> loading_targets -> plan_loading) for the
config-5 shape (32 layers, E = 8) and the Switch shape (1 layer, E = 128),
host wall time per call with the inputs prepared once."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2503_06823_b200 as emoe  # noqa: E402
from paper_2503_06823_b200 import _lib  # noqa: E402
from paper_2503_06823_b200.moesim import _p, _sets_array, check  # noqa: E402


def probe(m, E, k, L, P_train, T, n_req, reps=50):
    shape = emoe.ModelShape(m, E, k)
    trace = emoe.gen_routing_trace(shape, 0.6, 0.8, 0, 17, P_train, T)
    pred = emoe.moesim._Pred(m, E, k, 2, 0.01)
    tr = torch.from_numpy(trace).cuda()
    tid = torch.tensor([p % 2 for p in range(P_train)], dtype=torch.int32, device="cuda")
    import ctypes as C
    check(_lib.lib.emoe_hist_update(pred.h, C.c_void_p(tr.data_ptr()), P_train, T, C.c_void_p(tid.data_ptr()), None))
    torch.cuda.synchronize()
    _, sets = emoe.prompt_expert_sets(trace, P_train - 1)
    arr, sizes = _sets_array(sets, k)
    wo = np.array([16.0, 256.0])
    sens = np.ones((2, m), np.int32).reshape(-1)
    has = np.ones(2, np.uint8)
    rt = np.array([i % 2 for i in range(n_req)], np.int32)
    rn = np.full(n_req, T, np.int32)
    res = np.zeros((m, E), np.uint8)
    res[:, :L] = 1
    budgets = np.full(m, L, np.int32)
    agg = np.zeros((m, E))
    ev = np.full((m, E), -1, np.int32)
    ld = np.full((m, E), -1, np.int32)
    ne = np.zeros(m, np.int32)
    nl = np.zeros(m, np.int32)
    de = np.zeros(1)
    args = (pred.h, 0, _p(arr), _p(sizes), 2, _p(wo), _p(sens), _p(has), n_req, _p(rt), _p(rn), 1, _p(res),
            _p(budgets), 0.0, _p(agg), _p(ev), _p(ne), _p(ld), _p(nl), _p(de))
    for _ in range(5):
        check(_lib.lib.emoe_invocation_host(*args))
    t0 = time.perf_counter()
    for _ in range(reps):
        check(_lib.lib.emoe_invocation_host(*args))
    return (time.perf_counter() - t0) / reps * 1e6


if __name__ == "__main__":
    print(f"config 5 shape (m=32, E=8):   {probe(32, 8, 2, 4, 60, 256, 40):.1f} us per invocation")
    print(f"Switch shape (m=1, E=128):    {probe(1, 128, 1, 26, 200, 256, 32):.1f} us per invocation")
