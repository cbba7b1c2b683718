"""Golden vectors for the baseline sparsifiers, produced by
the UNMODIFIED reference's topk_select / hard_threshold_select
(baselines.cpp:26-46) through oracle/_ref/libsparsim_ref.so.

    python tests/golden/make_golden_baselines.py   # needs /root/reference

Cases: the known answers of test_baselines.cpp:27-71, random Laplace vectors
of ragged lengths, and tie-heavy vectors (values from a small set, signed
zeros) where the lower-index tie rule decides.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402


def main():
    rng = np.random.default_rng(20240213)
    cases = []

    def add(acc, ks, deltas, tag):
        acc = np.asarray(acc, np.float64)
        cases.append({
            "tag": tag, "acc": acc.tolist(),
            "topk": [{"k": int(k), "idx": O.ref_topk_select(acc, int(k)).tolist()} for k in ks],
            "hard": [{"delta": float(d), "idx": O.ref_hard_threshold_select(acc, float(d)).tolist()}
                     for d in deltas],
        })

    # test_baselines.cpp:27-37, 66-71
    add([0.1, -0.5, 0.3], [2, 3], [], "test_baselines.cpp:27-31")
    add([0.5, 0.5, 0.1], [1, 2], [], "test_baselines.cpp:33-37")
    add([0.1, 0.4], [], [0.3, 0.05, 9.0], "test_baselines.cpp:66-71")
    for n in (1, 31, 4097):
        acc = rng.laplace(size=n).astype(np.float32).astype(np.float64)
        ks = sorted({1, max(1, n // 100), max(1, n // 3), n})
        add(acc, ks, [0.0, 0.5, 2.0, 50.0], f"laplace n={n}")
    for n in (64, 4500):
        acc = rng.choice([0.0, -0.0, 0.25, -0.25, 1.0, -1.0, 3.0], size=n)
        ks = sorted({1, 2, n // 7, n // 2, n - 1, n})
        add(acc, ks, [0.25, 1.0, 3.0, 0.0], f"ties n={n}")
    with open(os.path.join(HERE, "baselines_golden.json"), "w") as f:
        json.dump({"source": "reference topk_select / hard_threshold_select (baselines.cpp:26-46)",
                   "cases": cases}, f, separators=(",", ":"))
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
