import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import oracle as O, paper_1908_09376_b200 as M
from helpers import cases, cvec, oracle_factorization, rel, saved
for c in cases():
    name, kind, X, Om, n0, k, eps = c
    K, Fo = oracle_factorization(kind, X, Om, n0, k, eps)
    plan = M.DevicePlan.load(saved(Fo), directions=3)
    f, g = cvec(Fo.ncols, 19), cvec(Fo.nrows, 20)
    wf, wg = Fo.apply(f), Fo.apply_transpose(g)
    for v in (0, 1):
        for comp, lite in ((True, False), (False, False), (True, True)):
            plan.set_flags(variant=v, compress=comp, lite=lite)
            for tr in (False, True):
                res = []
                for rep in range(int(os.environ.get("REPS","200"))):
                    a = plan.apply(g if tr else f, transpose=tr)
                    w = wg if tr else wf
                    bad = np.where(~np.isfinite(a) | (np.abs(a - w) > 1e-9 * np.abs(w).max()))[0]
                    if len(bad): res.append((rep, rel(a, w), len(bad), bad[:6].tolist(), a[bad[:3]].tolist()))
                print(name, "v", v, "comp", comp, "lite", lite, "T" if tr else "F", res, flush=True)
    plan.set_flags()
