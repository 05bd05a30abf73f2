"""Per-stage timeline of one k1_flow apply (flag bit 12 builds): for every
stage, when its strips got their context, had x staged and stored their rows
(us from the first CTA's entry; min / median / p90 / max).

    python tools/flow_timeline.py [flags] [config]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402

BASE = 1024 * 64 * 16


def main():
    flags = int(sys.argv[1]) if len(sys.argv) > 1 else 15
    config = sys.argv[2] if len(sys.argv) > 2 else "cfg1"
    K, X, Om, fk, nrhs, desc = bench.workload(config)
    F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, seed=M.chain(0, 0x666163))
    plan = F.plan(1)
    M.lib().midbf_plan_set_flags(plan._h, flags | 4096)
    f = torch.randn(F.ncols, dtype=torch.complex128, device="cuda")
    g = torch.empty(F.nrows, dtype=torch.complex128, device="cuda")
    for _ in range(5):
        plan.apply_ptr(f.data_ptr(), g.data_ptr(), 1, False, 0)
    torch.cuda.synchronize()
    stages = plan.stages()
    ns = sum(s[0] for s in stages)
    n = BASE + 3 * ns
    out = np.zeros(n, dtype=np.int64)
    M.lib().midbf_plan_flow_profile(plan._h, out.ctypes.data_as(C.POINTER(C.c_int64)), C.c_int64(n))
    warps = out[:BASE].reshape(-1, 16)
    ent = warps[:, 14]
    t0 = ent[ent > 0].min()
    ends = warps[:, 11]
    print(f"{config} flags {flags}: last warp end {(ends.max() - t0) / 1e3:.2f} us, streamed "
          f"{sum(plan.flow_bytes()) / 1e6:.1f} MB")
    ts = (out[BASE:BASE + 3 * ns].reshape(ns, 3) - t0) / 1e3
    s0 = 0
    q = lambda v: f"{v.min():6.2f} {np.median(v):6.2f} {np.percentile(v, 90):6.2f} {v.max():6.2f}"
    print("stage strips  MB    | ctx: min med p90 max        | x staged: min med p90 max   | stored: min med p90 max")
    for si, (cnt, pb, _, _) in enumerate(stages):
        t = ts[s0:s0 + cnt]
        s0 += cnt
        print(f"{si:5d} {cnt:6d} {plan.flow_bytes()[si] / 1e6:6.1f} | {q(t[:, 0])} | {q(t[:, 1])} | {q(t[:, 2])}")


if __name__ == "__main__":
    main()
