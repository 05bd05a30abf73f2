"""Interleaved A/B timing of k1_flow flag sets on one plan (one process, one
factorization): each round times every flag set over `reps` graph-replayed
applies with CUDA events; prints the median per-apply time per flag set.

    python tools/flow_ab.py config flagsA flagsB [...] [--rounds R] [--reps N]
e.g. flags 63 (default) vs 575 (bit 9: dense panels, no identity compression).
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("flags", nargs="+", type=int)
    ap.add_argument("--rounds", type=int, default=15)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--transpose", action="store_true")
    ap.add_argument("--nrhs", type=int, default=1)
    a = ap.parse_args()
    K, X, Om, fk, nrhs, desc = bench.workload(a.config)
    F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, seed=M.chain(0, 0x666163))
    plan = F.plan(3)
    nin, nout = (F.nrows, F.ncols) if a.transpose else (F.ncols, F.nrows)
    f = torch.randn(nin * a.nrhs, dtype=torch.complex128, device="cuda")
    g = torch.empty(nout * a.nrhs, dtype=torch.complex128, device="cuda")
    s = torch.cuda.current_stream()
    ref = None
    times = {fl: [] for fl in a.flags}
    for fl in a.flags:  # warm every graph / variant once, check agreement
        M.lib().midbf_plan_set_flags(plan._h, fl)
        for _ in range(3):
            plan.apply_ptr(f.data_ptr(), g.data_ptr(), a.nrhs, a.transpose, s.cuda_stream)
        torch.cuda.synchronize()
        if ref is None:
            ref = g.clone()
        else:
            err = (torch.linalg.vector_norm(g - ref) / torch.linalg.vector_norm(ref)).item()
            print(f"flags {fl}: rel diff vs flags {a.flags[0]} = {err:.2e}")
    for _ in range(a.rounds):
        for fl in a.flags:
            M.lib().midbf_plan_set_flags(plan._h, fl)
            plan.apply_ptr(f.data_ptr(), g.data_ptr(), a.nrhs, a.transpose, s.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.reps):
                plan.apply_ptr(f.data_ptr(), g.data_ptr(), a.nrhs, a.transpose, s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            times[fl].append(e0.elapsed_time(e1) * 1e3 / a.reps)
    for fl in a.flags:
        t = np.array(times[fl])
        M.lib().midbf_plan_set_flags(plan._h, fl)
        mb = sum(plan.flow_bytes(a.transpose)) / 1e6
        print(f"{a.config} flags {fl:6d}: median {np.median(t):7.2f} us  min {t.min():7.2f}  max {t.max():7.2f}"
              f"  streamed {mb:.1f} MB")


if __name__ == "__main__":
    main()
