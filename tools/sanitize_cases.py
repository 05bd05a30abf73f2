"""Small workload for compute-sanitizer (memcheck / synccheck / racecheck):
every kernel family once on tiny cases — K3 + K5 (device-sampled
factorization), K1 k1_flow in both layouts, compressed and dense-only, both
directions, K2 k2_flow (8 and 70 RHS), the per-stage fallbacks, K4 direct
sum — each checked against the oracle so a sanitizer run also proves the
results.  Usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402
from helpers import cvec, integer_grid, rel, saved, unit_grid  # noqa: E402


def run(name, kind, X, Om, n0, k):
    K = M.Kernel(kind, X=X, Omega=Om)
    F = M.idbf_factorize(K, n0, k=k, eps=1e-9, sampler="device")  # K3 + K5
    path = saved(F)
    Fo = O.load(path)
    plan = M.DevicePlan.load(path, directions=3)
    os.unlink(path)
    worst = 0.0
    f, g = cvec(Fo.ncols, 1), cvec(Fo.nrows, 2)
    for kw in (dict(variant=0, lite=False), dict(variant=1, lite=False), dict(variant=0, lite=True),
               dict(flow=False), dict(), dict(chain=False), dict(coop=True), dict(coop=True, chain=False)):
        plan.set_flags(**kw)
        for _ in range(3):  # consecutive applies alternate the stage-buffer parity sets
            worst = max(worst, rel(plan.apply(f), Fo.apply(f)),
                        rel(plan.apply(g, transpose=True), Fo.apply_transpose(g)))
    for nrhs in (8, 70):
        Xm = cvec(Fo.ncols, 3, cols=nrhs)
        worst = max(worst, rel(plan.apply(Xm), Fo.apply(Xm)))
    plan.set_flags(dmma_flow=False)
    Xm = cvec(Fo.ncols, 4, cols=16)
    worst = max(worst, rel(plan.apply(Xm), Fo.apply(Xm)))
    plan.reset_flags()
    rows = np.arange(0, len(X), 7, dtype=np.int64)
    gd = K.direct_sum(f, rows)  # K4
    go = O.Kernel(kind, X=X, Omega=Om).direct_sum(f, rows)
    worst = max(worst, rel(gd, go))
    print(f"{name}: worst rel vs oracle {worst:.2e}", flush=True)
    assert worst <= 1e-12


run("fio2d_n16", M.KIND_FIO2D, O.grid2d(16), integer_grid(16), 16, 12)
run("fio2d_n32", M.KIND_FIO2D, O.grid2d(32), O.grid2d(32), 64, 30)
run("fio3d_n8", M.KIND_FIO3D, unit_grid(8, 3), integer_grid(8, 3), 64, 64)
print("sanitize cases ok")
