"""Time the K1 apply kernels on synthetic single-stage plans with uniform
strips (h x n panels, `nseg` panels per strip), ~358 MB of payload like
cfg1, to separate kernel mechanics from cfg1's strip shapes.

    python tools/flow_probe.py      (needs a B200)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_09376_b200 as M  # noqa: E402


def synthetic_plan(h, n, nseg, total_bytes=358 << 20):
    """One factor: strips of h rows, each fed by nseg blocks h x n reading
    disjoint input segments (a U-type group)."""
    per_strip = h * n * nseg * 16
    nstrip = max(1, total_bytes // per_strip)
    rows, cols = nstrip * h, nstrip * nseg * n
    blocks, mats = [], []
    rng = np.random.default_rng(0)
    M0 = (rng.standard_normal((h, n)) + 1j * rng.standard_normal((h, n))).astype(np.complex128)
    for s in range(nstrip):
        for j in range(nseg):
            blocks.append((s * h, (s * nseg + j) * n, h, n))
            mats.append(M0)
    groups = [(s * nseg, (s + 1) * nseg) for s in range(nstrip)]
    factor = (rows, cols, np.array(blocks), np.array(groups), mats)
    plan = M.DevicePlan.from_tables(rows, cols, np.arange(rows), np.arange(cols), [factor])
    return plan, rows, cols


def time_apply(plan, rows, cols, flags, reps=30):
    """flags: midbf_plan_set_flags bits (15 = flow kernel, 7 = stage kernels,
    15|128 = flow kernel streaming the payload only, a timing experiment)."""
    M.lib().midbf_plan_set_flags(plan._h, flags)
    f = torch.randn(cols, dtype=torch.complex128, device="cuda")
    g = torch.empty(rows, dtype=torch.complex128, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        plan.apply_ptr(f.data_ptr(), g.data_ptr(), 1, False, s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        plan.apply_ptr(f.data_ptr(), g.data_ptr(), 1, False, s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    for (h, n, nseg) in [(32, 128, 1), (32, 32, 4), (32, 30, 4), (30, 120, 1), (32, 120, 1), (32, 256, 1),
                         (32, 512, 1), (32, 64, 1), (32, 30, 1)]:
        plan, rows, cols = synthetic_plan(h, n, nseg)
        nbytes = plan.total_nnz * 16
        out = []
        for name, fl in [("flow", 15), ("stream", 15 | 2 << 6), ("compute", 15 | 3 << 6), ("no-fma", 15 | 4 << 6),
                         ("stage", 7)]:
            us = time_apply(plan, rows, cols, fl)
            out.append(f"{name} {us:7.1f} us {nbytes / us / 1e3:7.1f} GB/s")
        print(f"h={h:2d} n={n:3d} nseg={nseg} strips={rows // h:6d}: " + " | ".join(out), flush=True)


if __name__ == "__main__":
    main()
