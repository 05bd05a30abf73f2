"""Loop the nufft3d flag-switch sequence of tests/test_gpu_apply.py
(variants, identity compression) and report non-finite / mismatching
results per step.  Usage: python tools/repro_nan.py [iters] [graph 0/1]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import paper_1908_09376_b200 as M  # noqa: E402
from helpers import cases, cvec, oracle_factorization, saved  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
graph = bool(int(sys.argv[2])) if len(sys.argv) > 2 else True
name, kind, X, Om, n0, k, eps = [c for c in cases() if c[0] == os.environ.get("CASE", "nufft3d")][0]
K, Fo = oracle_factorization(kind, X, Om, n0, k, eps)
plan = M.DevicePlan.load(saved(Fo), directions=3)
f, g = cvec(Fo.ncols, 24), cvec(Fo.nrows, 25)
F48 = cvec(Fo.ncols, 26, cols=48)
wf, wg = Fo.apply(f), Fo.apply_transpose(g)
print("stages F", plan.stages(), "flow bytes", plan.flow_bytes(), flush=True)
nbad = 0
for it in range(iters):
    for step, kw in enumerate([dict(variant=0), dict(variant=1), dict(flow=False), dict(),
                               dict(variant=0), dict(variant=0, compress=False), dict(variant=0, lite=True),
                               dict(variant=1), dict(variant=1, compress=False), dict(variant=1, lite=True)]):
        plan.set_flags(graph=graph, **kw)
        a = plan.apply(f)
        b = plan.apply(g, transpose=True)
        if step in (4, 7):
            plan.apply(F48)
        for tag, v, w in (("F", a, wf), ("T", b, wg)):
            bad = np.flatnonzero(~np.isfinite(v) | (np.abs(v - w) > 1e-9 * np.abs(w).max()))
            if bad.size:
                nbad += 1
                print(f"it {it} step {step} {kw} {tag}: {bad.size} bad rows {bad[:12].tolist()} "
                      f"nonfinite {int((~np.isfinite(v)).sum())}", flush=True)
plan.set_flags()
print("done, bad results:", nbad)
