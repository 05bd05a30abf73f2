"""cfg1 factorize wall time with and without torch imported first (OpenMP
runtime interplay check)."""
import os
import sys
import time

if len(sys.argv) > 1 and sys.argv[1] == "torch":
    import torch  # noqa: F401
    torch.cuda.set_device(0)
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_1908_09376_b200 as M  # noqa: E402
from helpers import integer_grid, unit_grid  # noqa: E402

K = M.Kernel(M.KIND_FIO2D, X=unit_grid(256, 2), Omega=integer_grid(256, 2))
for _ in range(3):
    t0 = time.perf_counter()
    F = M.idbf_factorize(K, 64, k=30, eps=1e-9)
    print(sys.argv[1:] or ["plain"], f"wall {time.perf_counter() - t0:.3f}s internal {F.id_stats()[3]:.3f}s", flush=True)
