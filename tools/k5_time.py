"""Factorize cfg1 with device IDs once (launch-list helper for ncu)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_1908_09376_b200 as M  # noqa: E402
from helpers import integer_grid, unit_grid  # noqa: E402

K = M.Kernel(M.KIND_FIO2D, X=unit_grid(256, 2), Omega=integer_grid(256, 2))
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t0 = time.perf_counter()
    F = M.idbf_factorize(K, 64, k=30, eps=1e-9, ids="device")
    print("factorize", time.perf_counter() - t0, F.id_stats(), F.sample_stats(), flush=True)
