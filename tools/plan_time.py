"""Time MIDBF001 -> device plan (host repack + upload) at cfg1 / cfg2 sizes."""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_1908_09376_b200 as M  # noqa: E402
from helpers import integer_grid, unit_grid  # noqa: E402

for n in (256, 512):
    K = M.Kernel(M.KIND_FIO2D, X=unit_grid(n, 2), Omega=integer_grid(n, 2))
    F = M.idbf_factorize(K, 64, k=30, eps=1e-9)
    fd, path = tempfile.mkstemp(suffix=".midbf")
    os.close(fd)
    t0 = time.perf_counter()
    F.save(path)
    t_save = time.perf_counter() - t0
    for dirs in (1, 3):
        t0 = time.perf_counter()
        P = M.DevicePlan.load(path, directions=dirs)
        t_load = time.perf_counter() - t0
        del P
        print(f"n={n} nnz={F.total_nnz} save {t_save:.3f}s  plan load dirs={dirs} {t_load:.3f}s", flush=True)
    t0 = time.perf_counter()
    P = F.plan(1)
    print(f"n={n} F.plan(1) from the in-memory factorization {time.perf_counter() - t0:.3f}s", flush=True)
    os.unlink(path)
