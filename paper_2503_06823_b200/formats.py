"""On-disk formats shared with the reference.

* Routing traces as NDJSON (report.cpp:260-306): a header line
  {"schema_version":1,"num_layers":m,"top_k":k} followed by one prompt per line,
  experts[l][t][r].  GPU routing from the layer workspace (topk_idx) can be
  written in this format and read by the reference's `load_trace`.
* Predictor state as the reference model JSON (predictor.cpp:240-274): the
  TransitionModel tallies, keys in nlohmann::json (sorted) order, indent 2.
Both writers produce the reference's bytes (tests/test_formats.py).
"""
from __future__ import annotations

import json
from pathlib import Path
from typing import Union

import numpy as np

from .moesim import TransitionModel, ValidationError


def save_trace(trace: np.ndarray, path: Union[str, Path]) -> None:
    """trace: [P][m][T][k] int routing choices (rank 0 = top)."""
    trace = np.asarray(trace)
    P, m, T, k = trace.shape
    with open(path, "w") as f:
        f.write(json.dumps({"schema_version": 1, "num_layers": int(m), "top_k": int(k)}, separators=(",", ":")))
        f.write("\n")
        for p in range(P):
            f.write(json.dumps(trace[p].tolist(), separators=(",", ":")))
            f.write("\n")


def load_trace(path: Union[str, Path]) -> np.ndarray:
    lines = Path(path).read_text().splitlines()
    if not lines:
        raise ValidationError(f"{path}: empty trace file")
    try:
        header = json.loads(lines[0])
    except json.JSONDecodeError as e:
        raise ValidationError(f"{path}:1: bad trace header: {e}")
    if header.get("schema_version", 0) != 1:
        raise ValidationError(f"{path}: trace schema_version: expected 1")
    m, k = int(header["num_layers"]), int(header["top_k"])
    prompts = []
    for i, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        prompt = json.loads(line)
        if len(prompt) != m:
            raise ValidationError(f"{path}:{i}: prompt has wrong layer count")
        if any(len(tok) != k for layer in prompt for tok in layer):
            raise ValidationError(f"{path}:{i}: token without top_k experts")
        prompts.append(prompt)
    if not prompts:
        return np.zeros((0, m, 0, k), np.int32)
    return np.asarray(prompts, np.int32)


def routing_to_trace(topk_idx: np.ndarray, prompts: int) -> np.ndarray:
    """A layer's routed gate choices [P*T][k] (workspace topk_idx) as a
    one-layer trace [P][1][T][k]."""
    topk_idx = np.asarray(topk_idx, np.int32)
    n, k = topk_idx.shape
    return topk_idx.reshape(prompts, 1, n // prompts, k)


def _num(v: float):
    return float(v)


def save_model(model: TransitionModel, path: Union[str, Path]) -> None:
    m, E = model.num_layers, model.num_experts
    j = {
        "layer_counts": [[[_num(v) for v in row] for row in mat] for mat in np.asarray(model.layer_counts).reshape(
            max(m - 1, 0), E, E)],
        "num_experts": int(E),
        "num_layers": int(m),
        "prompt_counts": [[[_num(v) for v in row] for row in mat] for mat in model.prompt_counts],
        "schema_version": 1,
        "smoothing": float(model.smoothing),
        "task_token_counts": {t: [[_num(v) for v in row] for row in model.task_counts[i]]
                              for i, t in enumerate(model.task_ids)},
        "top_k": int(model.top_k),
    }
    Path(path).write_text(json.dumps(j, indent=2) + "\n")


def load_model(path: Union[str, Path]) -> TransitionModel:
    try:
        j = json.loads(Path(path).read_text())
        m, E = int(j["num_layers"]), int(j["num_experts"])
        names = sorted(j["task_token_counts"])
        tc = np.array([j["task_token_counts"][n] for n in names], np.float64).reshape(len(names), m, E)
        model = TransitionModel(m, E, int(j["top_k"]), float(j["smoothing"]),
                                np.array(j["layer_counts"], np.float64).reshape(max(m - 1, 0), E, E),
                                np.array(j["prompt_counts"], np.float64).reshape(m, E, E), names, tc)
    except (OSError, KeyError, ValueError, TypeError) as e:
        raise ValidationError(f"model file: {e}")
    return model
