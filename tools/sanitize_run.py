"""Small end-to-end runs of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): n = 1 and a 2-rank loopback,
each compressor, Adam / LANS / NAG, checked against the oracle.

usage (GPU box): compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from gpu_harness import run_parity  # noqa: E402
from workloads import (LINEAR_DITHER, NATURAL_DITHER, NONE, RANDOM_K, SCALED_SIGN, TOP_K, Comp,  # noqa: E402
                       Config)

SHAPES = (1000, 70000, 262147, 5)   # raw, raw, two units with a ragged tail, tiny
CASES = [
    ("onebit", Comp(SCALED_SIGN, use_ef=1), "adam"),
    ("topk_f16", Comp(TOP_K, 1, 1000, use_ef=1, f16=1), "adam"),
    ("randk", Comp(RANDOM_K, 1, 32, use_ef=1), "adam"),
    ("ldither", Comp(LINEAR_DITHER, bits=7, use_ef=0), "adam"),
    ("ndither", Comp(NATURAL_DITHER, bits=3, use_ef=0), "adam"),
    ("none", Comp(NONE, use_ef=1), "adam"),
    ("onebit_lans", Comp(SCALED_SIGN, use_ef=1), "lans"),
    ("topk_lans", Comp(TOP_K, 1, 1000, use_ef=1), "lans"),
    ("onebit_nag", Comp(SCALED_SIGN, use_ef=1), "nag"),
]

if __name__ == "__main__":
    n_list = [int(a) for a in sys.argv[1:]] or [1, 2]
    for name, comp, opt in CASES:
        for n in n_list:
            w = Config("san", "custom", comp, numels=SHAPES, optimizer=opt)
            run_parity(w, n, steps=2, label=f"{name} n={n}")
            print(f"ok {name} n={n}", flush=True)
    print("SANITIZE RUN OK")
