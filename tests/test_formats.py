"""Trace NDJSON and model JSON written by paper_2503_06823_b200.formats are
byte-identical to the reference's save_trace / save_model (report.cpp:260-267,
predictor.cpp:240-252) and round-trip."""
import numpy as np
import pytest

from paper_2503_06823_b200 import formats
from paper_2503_06823_b200.moesim import TransitionModel


@pytest.mark.parametrize("case", [(2, 8, 2, 5, 16), (1, 8, 2, 3, 64), (3, 16, 1, 4, 9)])
def test_trace_ndjson_bytes_and_round_trip(case, ref, tmp_path):
    m, E, k, P, T = case
    tr = ref.gen_routing_trace(m, E, k, 0.6, 0.8, 0, 17, P, T)
    ours, theirs = tmp_path / "ours.ndjson", tmp_path / "ref.ndjson"
    formats.save_trace(tr, ours)
    ref.save_trace(tr, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    assert np.array_equal(formats.load_trace(theirs), tr)


def test_model_json_bytes_and_round_trip(ref, port, tmp_path):
    tr = ref.gen_routing_trace(4, 6, 2, 0.5, 0.8, 1, 77, 60, 8)
    names = ["chat", "qa"]
    tids = np.array([p % 2 for p in range(60)], np.int32)
    theirs = tmp_path / "ref.json"
    ref.fit_and_save_model(tr, tids, names, 0.01, 6, theirs)
    f = port.fit(tr, tids, 2, 6)
    model = TransitionModel(4, 6, 2, 0.01, f["layer_counts"], f["prompt_counts"], names, f["task_counts"])
    ours = tmp_path / "ours.json"
    formats.save_model(model, ours)
    assert ours.read_bytes() == theirs.read_bytes()
    back = formats.load_model(theirs)
    assert np.array_equal(back.layer_counts, model.layer_counts)
    assert np.array_equal(back.prompt_counts, model.prompt_counts)
    assert np.array_equal(back.task_counts, model.task_counts) and back.task_ids == names
