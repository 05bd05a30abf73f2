"""Device throughput of K3 (entry sampling inside a real factorization) and
K4 (direct sums) at BASELINE shapes, one JSON line each.

    python tools/k3_bench.py [cfg1 cfg2 cfg3 ...]

K3 figures are the factorization's own CUDA-event times of its k3_sample*
launches (Factorization.kernel_stats()); K4 is wall time around a large
direct sum (kernel-dominated).  FP64 flops per entry come from ncu SASS
counters (tools/gpu_k3_prof.sh -> profiles/), not from this script.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402


def k3(cfg):
    K, X, Om, fk, nrhs, desc = bench.workload(cfg)
    for _ in range(2):
        F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, t=5, seed=M.chain(0, 0x666163), sampler="device")
    ks = F.kernel_stats()
    n_dev, n_host, id_s, fac_s = F.id_stats()
    print(json.dumps({"kernel": "k3", "workload": cfg, **ks,
                      "k3_entries_per_s": ks["k3_entries"] / max(ks["k3_seconds"], 1e-12),
                      "ids_on_gpu": n_dev, "ids_on_host": n_host, "factorize_seconds": fac_s}), flush=True)
    return K, len(X), len(Om)


def k4(name, K, ncols, nsel, reps=3):
    f = M.random_coefficients(ncols, 5)
    rows = np.arange(nsel, dtype=np.int64)
    K.direct_sum(f, rows[:64])
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        K.direct_sum(f, rows)
        best = min(best, time.perf_counter() - t0)
    ent = nsel * ncols
    print(json.dumps({"kernel": "k4", "workload": name, "entries": ent, "seconds": best,
                      "entries_per_s": ent / best}), flush=True)


def main():
    cfgs = sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]
    for c in cfgs:
        K, nr, nc = k3(c)
        k4(c + " 8192 rows", K, nc, min(8192, nr))


if __name__ == "__main__":
    main()
