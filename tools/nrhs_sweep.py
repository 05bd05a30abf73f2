"""Device-timed apply vs number of right-hand sides at cfg1 (CUDA events,
operands resident, graph replays)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402

K, X, Om, fk, _, _ = bench.workload("cfg1")
F = M.idbf_factorize(K, 64, k=30, eps=1e-9, seed=M.chain(0, 0x666163))
plan = F.plan(1)
if len(sys.argv) > 1:  # raw plan flags (timing experiments)
    M.lib().midbf_plan_set_flags(plan._h, int(sys.argv[1]))
sizes = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else (1, 2, 4, 5, 6, 8, 16, 24, 32, 48, 64, 96, 128)
s = torch.cuda.current_stream()
for nrhs in sizes:
    f = torch.randn(F.ncols * nrhs, dtype=torch.complex128, device="cuda")
    g = torch.empty(F.nrows * nrhs, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        plan.apply_ptr(f.data_ptr(), g.data_ptr(), nrhs, False, s.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record(s)
    for _ in range(reps):
        plan.apply_ptr(f.data_ptr(), g.data_ptr(), nrhs, False, s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    tf = 8.0 * F.total_nnz * nrhs / (us * 1e-6) / 1e12
    print(f"nrhs {nrhs:4d}: {us:8.1f} us/apply  {nrhs / us * 1e6:10.0f} matvecs/s  {tf:6.2f} TFLOP/s  launches {plan.launches(nrhs)}",
          flush=True)
