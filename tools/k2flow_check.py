"""Small K2-flow check: apply a small oracle factorization to 64 / 70 RHS on
the device and compare with the oracle (debug aid, run under
compute-sanitizer)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
import oracle as O  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402
from helpers import cvec, oracle_factorization, rel, saved  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
X = O.grid2d(n)
K, Fo = oracle_factorization(O.KIND_FIO2D, X, X, 64, 30, 1e-9)
path = saved(Fo)
plan = M.DevicePlan.load(path, directions=3)
os.unlink(path)
for nrhs in (64, 70, 3):
    F = cvec(n * n, 16, cols=nrhs)
    print(nrhs, "fwd", rel(plan.apply(F), Fo.apply(F)), flush=True)
    print(nrhs, "tr", rel(plan.apply(F, transpose=True), Fo.apply_transpose(F)), flush=True)
