"""Band-survey fixtures from the reference itself (oracle/_ref = the
reference's own sources): sweep_band TSVs (proj/src/pipeline.cpp:181-208)
for the grids its tests use plus a paper-scale grid, and the reference's
generate_synthetic bytes for a few SynthParams.

    python tests/golden/make_sweep_golden.py    (needs oracle/_ref)
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle_py import Ref  # noqa: E402

CASES = [
    # test_pipeline.cpp:137
    {"length": 120, "xs": [1, 4, 9], "ps": [1.0, 0.6], "seed": 7, "source": "test_pipeline.cpp:137"},
    # acceptance.cpp:282-290 (criterion 3)
    {"length": 2000, "xs": [5, 10, 15, 20], "ps": [1.0 - i / 9.0 for i in range(10)], "seed": 93,
     "source": "acceptance.cpp:282-290"},
    # acceptance.cpp:256-263 (criterion 2: L=20000, p=0.9, X=15, default seed)
    {"length": 20000, "xs": [15], "ps": [0.9], "seed": 42, "source": "acceptance.cpp:256-263"},
    # the paper's band figure at its scale (PAPER.md band survey, L=20000)
    {"length": 20000, "xs": [5, 10, 15, 20, 30, 50], "ps": [0.70, 0.75, 0.80, 0.85, 0.90, 0.95, 1.0],
     "seed": 42, "source": "paper-scale grid"},
    # edges: X = 0, always mutate (p = 0)
    {"length": 500, "xs": [0, 3], "ps": [0.0, 0.5], "seed": 11, "source": "edges"},
]

SYNTH = [(3, 1000, 0.9, 17, 42, False), (2, 500, 0.0, 17, 5, True), (4, 300, 1.0, 5, 9, True),
         (1, 17, 0.5, 17, 3, False)]


def main():
    R = Ref()
    for c in CASES:
        c["tsv"] = R.sweep_band(c["length"], c["xs"], c["ps"], c["seed"])
    synth = []
    for pairs, length, p, k, seed, uni in SYNTH:
        sym, off, tasks = R.generate_synthetic(pairs, length, p, k, seed, uni)
        synth.append({"pairs": pairs, "length": length, "p_match": p, "k": k, "seed": seed,
                      "uniform_seed": uni, "symbols_sha256": hashlib.sha256(sym.tobytes()).hexdigest(),
                      "offsets": off.tolist(), "tasks": tasks.tolist()})
    json.dump({"sweeps": CASES, "synth": synth}, open(os.path.join(HERE, "sweep_band.json"), "w"),
              indent=1)
    for c in CASES:
        print(c["source"], c["tsv"].count("\n") - 1, "rows")


if __name__ == "__main__":
    main()
