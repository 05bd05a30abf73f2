"""Device IDs (K5) vs host IDs: structure, accuracy, fallbacks, timing."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
import oracle as O  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402
from helpers import cvec, integer_grid, rel, unit_grid  # noqa: E402


def case(name, K, n0, k, N, direct=True):
    out = {}
    for ids in ("device", "host"):
        t0 = time.perf_counter()
        F = M.idbf_factorize(K, n0, k=k, eps=1e-9, ids=ids)
        dt = time.perf_counter() - t0
        f = cvec(N, 5)
        g = F.apply(f)
        out[ids] = (F, g, dt)
    Fd, gd_, td = out["device"]
    Fh, gh_, th = out["host"]
    st = Fd.id_stats()
    line = f"{name}: nnz dev {Fd.total_nnz} host {Fh.total_nnz}  t dev {td:.3f}s host {th:.3f}s  ids {st}  dev-vs-host {rel(gd_, gh_):.2e}"
    if direct:
        ref = K.direct_sum(cvec(N, 5), np.arange(min(N, 512)))
        line += f"  err dev {rel(gd_[:min(N,512)], ref):.2e} host {rel(gh_[:min(N,512)], ref):.2e}"
    print(line, flush=True)


for n in (16, 32, 64):
    X = O.grid2d(n)
    case(f"fio_unit_n{n}", M.Kernel(M.KIND_FIO2D, X=X, Omega=X), 64, 30, n * n)
X = O.grid2d(64)
case("fio_int_n64_k20", M.Kernel(M.KIND_FIO2D, X=X, Omega=integer_grid(64)), 64, 20, 4096)
rng = np.random.default_rng(2)
X2, O2 = rng.random((300, 2)), rng.random((300, 2))
case("const", M.Kernel(M.KIND_CONST, X=X2, Omega=O2, const=1.5 - 0.5j), 32, 5, 300, direct=False)
case("cfg1", M.Kernel(M.KIND_FIO2D, X=unit_grid(256, 2), Omega=integer_grid(256, 2)), 64, 30, 65536, direct=False)
case("cfg1_unitxi", M.Kernel(M.KIND_FIO2D, X=unit_grid(256, 2), Omega=unit_grid(256, 2)), 64, 30, 65536)
