"""Host logic of the serving loop (no GPU): the on-demand baseline's per-layer
target rule (engine.cpp:469-497 dynamic_transfers)."""
import numpy as np

from paper_2503_06823_b200.serving import dynamic_targets


def test_dynamic_targets_keep_top_demand_with_index_ties():
    demand = np.array([5, 0, 3, 3, 1, 0, 0, 9])
    resident = np.array([1, 1, 0, 0, 0, 0, 0, 1], np.uint8)
    # ranked by demand: 7 (9), 0 (5), 2 (3), 3 (3: loses the tie to 2), 4 (1)
    assert dynamic_targets(demand, resident, 3) == ([1], [2])
    assert dynamic_targets(demand, resident, 5) == ([1], [2, 3, 4])


def test_dynamic_targets_never_keeps_undemanded_experts():
    demand = np.array([0, 4, 0, 0])
    resident = np.array([1, 0, 1, 0], np.uint8)
    assert dynamic_targets(demand, resident, 3) == ([0, 2], [1])
    assert dynamic_targets(demand, np.array([0, 1, 0, 0], np.uint8), 2) == ([], [])
