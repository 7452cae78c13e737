"""Measure the reference CostModel on this GPU.

Builds the config-5 stack (m Mixtral-shaped layers, phi = 0.5, routing-driven
from the reference trace), runs serving.profile_cost_model and prints the
reference scenario's "cost" object (scenario.cpp:252-260) -- drop it into a
moesim scenario JSON to run the reference engine / scheduler with B200 costs.

    python tools/profile_cost_model.py --layers 32 > profiles/r01_cost_model.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_06823_b200 as emoe  # noqa: E402
from paper_2503_06823_b200.serving import (MoEStack, StreamConfig, TaskSpec, moesim_prompt_sets,  # noqa: E402
                                           profile_cost_model)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--tokens", type=int, default=8192)
    args = ap.parse_args()
    m, E, k, L, d, f, T, p = args.layers, 8, 2, 4, 4096, 14336, args.tokens, 40
    device = torch.device("cuda", 0)
    tasks = {"cls": TaskSpec(16.0, [0] * m), "conv": TaskSpec(256.0, [1] * m)}
    cfg = StreamConfig(m=m, E=E, k=k, L=L, d=d, f=f, tokens_per_prompt=T, period=p, mode=0, tasks=tasks)
    P_train = 60
    trace = emoe.gen_routing_trace(emoe.ModelShape(m, E, k), 0.6, 0.8, 0, 17, P_train + 1, T)
    prompt_tasks = ["conv" if q % 2 else "cls" for q in range(P_train + 1)]
    g = torch.Generator(device=device).manual_seed(1234)
    host = [tuple((torch.randn(*s, generator=g, device=device) / s[1] ** 0.5).to(torch.bfloat16).cpu().pin_memory()
                  for s in ((f, d), (f, d), (d, f))) for _ in range(E)]
    stack = MoEStack(cfg, host, [torch.zeros(E, d, dtype=torch.bfloat16) for _ in range(m)])
    trace_dev = torch.from_numpy(trace).to(device)
    stack.fit(trace_dev[:P_train].contiguous(), prompt_tasks[:P_train])
    _, sets = moesim_prompt_sets(trace_dev, P_train - 1)
    requests = [("conv", T)] * p
    ops, _, _ = stack.invocation(sets, requests)
    stack.apply(ops)
    for layer in stack.layers:
        layer.poll_loads(blocking=True)
    lg = torch.rand(m, T, E, generator=g, device=device) * 8.0 - 4.0
    ch = trace_dev[P_train].long()
    for r in range(k):
        lg.scatter_(2, ch[:, :, r:r + 1], 8.0 - r)
    x = torch.randn(T, d, generator=g, device=device).to(torch.bfloat16)
    cost = profile_cost_model(stack, x, lg, sets, requests)
    expert_bytes = 3 * d * f * 2
    print(json.dumps(dict(cost=cost, model=dict(num_moe_layers=m, experts_per_layer=E, top_k=k,
                                                expert_bytes=expert_bytes),
                          measured_on=torch.cuda.get_device_name(0), tokens_per_prompt=T,
                          expert_transfer_seconds=cost["per_expert_transfer"] + expert_bytes / cost["hd_bandwidth"]),
                     indent=1))
    stack.close()


if __name__ == "__main__":
    main()
