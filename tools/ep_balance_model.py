"""Load model of expert parallelism on the config-2/4 routing (host only).

For the config-2/4 workload (reference Markov trace, 4 predicted-resident of
8 experts per layer, 32 x 2048 tokens per GPU) this counts, per world size W,
the rows each rank's grouped FFN receives under ep.plan_destinations
(resident experts sharded in contiguous blocks, or replicated in groups of L
ranks when L < W).  The FFN-bound EP step is set by the busiest rank, so the
scaling efficiency of EP over W independent GPUs is mean(rows) / max(rows)
(exchange time ignored).  Replicas (every GPU holds the resident set) are
balanced by construction.

python tools/ep_balance_model.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def served_counts(choices: np.ndarray, resident: np.ndarray, E: int) -> np.ndarray:
    """Rows per expert under the k-slot served set: the resident
    gate choices in rank order, else route_token's fallback (smallest
    resident expert when no scores are set)."""
    hit = resident[choices]                      # [T, k]
    counts = np.zeros(E, np.int64)
    for r in range(choices.shape[1]):
        np.add.at(counts, choices[hit[:, r], r], 1)
    none = ~hit.any(axis=1)
    counts[np.flatnonzero(resident)[0]] += int(none.sum())
    return counts


def main():
    import paper_2503_06823_b200 as emoe
    from paper_2503_06823_b200.ep import plan_destinations

    E, k, P, Tp, P_train = 8, 2, 32, 2048, 200
    resident_set = [0, 5, 6, 7]   # the config-2 predicted set (bench.py)
    resident = np.zeros(E, bool)
    resident[resident_set] = True
    trace = emoe.gen_routing_trace(emoe.ModelShape(1, E, k), 0.6, 0.8, 0, 17, P_train + 8 * P, Tp)
    print("rows per expert for one GPU's batch:", served_counts(trace[P_train:P_train + P].reshape(-1, k),
                                                                 resident, E).tolist())
    for W in (1, 2, 4, 8):
        # the planner's load estimate: rows per expert summed over all W
        # sources' batches (on the GPUs: the ranks' Eq. 2 aggregates, one
        # E-float all-reduce before planning; one source alone is a poor
        # estimate because the trace drifts between prompt segments)
        est = sum(served_counts(trace[P_train + s * P: P_train + (s + 1) * P].reshape(-1, k), resident, E)
                  for s in range(W))
        for name, loads in (("equal", None), ("load-aware", est)):
            dest = plan_destinations(resident_set, E, W, loads)
            rows = np.zeros(W, np.int64)
            for src in range(W):
                ch = trace[P_train + src * P: P_train + (src + 1) * P].reshape(-1, k)
                c = served_counts(ch, resident, E)
                for e in resident_set:
                    rows[dest[src, e]] += c[e]
            print(f"W={W} {name:10s}: FFN rows per rank {rows.tolist()}  "
                  f"EP efficiency (mean/max) {rows.mean() / rows.max():.2f}")


if __name__ == "__main__":
    main()
