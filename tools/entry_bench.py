"""Throughput of the entry kernels on B200: K3 (batched exp(2*pi*i*Phi)
blocks feeding the IDs) and K4 (direct O(N^2) sums), at BASELINE shapes.

    python tools/entry_bench.py            # one JSON line per measurement

Times are wall-clock around the C-ABI call (K3 includes the id upload and the
D2H copy of every sampled block, as the factorization uses it); the kernel
times and FP64 pipe utilisation come from ncu (profiles/).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_09376_b200 as M  # noqa: E402


def grids(n, dim):
    ax = np.arange(n, dtype=np.float64)
    g = np.stack(np.meshgrid(*([ax] * dim), indexing="ij"), -1).reshape(-1, dim)
    return g / n, g - n // 2


def k3(name, K, nrows, ncols, ntasks=4096, nr=64, nc=150, reps=3):
    rng = np.random.default_rng(0)
    rows = [rng.integers(0, nrows, nr) for _ in range(ntasks)]
    cols = [rng.integers(0, ncols, nc) for _ in range(ntasks)]
    K.sample(rows[:8], cols[:8])
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        K.sample(rows, cols)
        best = min(best, time.perf_counter() - t0)
    ent = ntasks * nr * nc
    print(json.dumps({"kernel": "k3_sample", "workload": name, "entries": ent, "seconds": best,
                      "entries_per_s": ent / best, "note": "wall clock incl. id upload + D2H of the blocks"}))


def k4(name, K, nrows, ncols, nsel, reps=3):
    f = np.random.default_rng(1).standard_normal(ncols) + 0j
    rows = np.arange(min(nsel, nrows), dtype=np.int64)
    K.direct_sum(f, rows[:16])
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        K.direct_sum(f, rows)
        best = min(best, time.perf_counter() - t0)
    ent = len(rows) * ncols
    print(json.dumps({"kernel": "k4_direct", "workload": name, "entries": ent, "seconds": best,
                      "entries_per_s": ent / best}))


def main():
    X, Om = grids(256, 2)
    K = M.Kernel(M.KIND_FIO2D, X=X, Omega=Om)
    k3("cfg1 FIO-2D integer xi", K, len(X), len(Om))
    k4("cfg1 FIO-2D, 256 sampled rows (eps_b)", K, len(X), len(Om), 256)
    k4("cfg1 FIO-2D, 8192 rows", K, len(X), len(Om), 8192)
    X3, O3 = grids(32, 3)
    K3 = M.Kernel(M.KIND_FIO3D, X=X3, Omega=O3)
    k3("cfg3 FIO-3D", K3, len(X3), len(O3), nc=320)
    A = np.random.default_rng(2).standard_normal((65536, 8))
    B = np.random.default_rng(3).standard_normal((65536, 8)) * 30
    KL = M.Kernel(M.KIND_LOWRANK, A=A, B=B)
    k3("low-rank r=8", KL, 65536, 65536)
    k4("low-rank r=8, 8192 rows", KL, 65536, 65536, 8192)


if __name__ == "__main__":
    main()
