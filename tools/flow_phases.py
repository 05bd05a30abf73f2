"""Phase breakdown of k1_flow at cfg1 (flag bit 12 phase timers).

    python tools/flow_phases.py [flags] [config]
Prints, per warp role, the mean cycles per apply spent in each phase.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402

NAMES = ["P: wait ctx", "P: wait empty slot", "C: wait ctx", "X: wait ctx", "C: wait x staged",
         "C: strip setup", "C: epilogue (sums, identity)", "C: y store", "C: wait full slot", "C: FMA loop", "total", "-",
         "X: wait x buffer free", "X: gather+poll"]


def main():
    flags = int(sys.argv[1]) if len(sys.argv) > 1 else 31
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
    fw = {15: 4, 31: 8, 47: 6}[flags & 63]
    grid = 148
    dual = bool(flags & (1 << 25))  # two consumers per pair (4-pair layout): warps 3fw..4fw
    nw = (3 if fw <= 4 else 2) * fw + (fw if dual else 0)  # consumers, producers (+ x stagers when fw <= 4)
    n = grid * nw * 16
    out = np.zeros(n, dtype=np.int64)
    M.lib().midbf_plan_flow_profile(plan._h, out.ctypes.data_as(C.POINTER(C.c_int64)), C.c_int64(n))
    t = out.reshape(grid, nw, 16)
    cons, prod = t[:, :fw, :].reshape(-1, 16), t[:, fw:2 * fw, :].reshape(-1, 16)
    roles = [("consumer", cons), ("producer", prod)]
    if fw <= 4:
        roles.append(("x stager", t[:, 2 * fw:3 * fw, :].reshape(-1, 16)))
    if dual:
        roles.append(("consumer 1", t[:, 3 * fw:, :].reshape(-1, 16)))
    clk = 1.965e3  # cycles per us
    ent, pro, end = t[:, :, 14], t[:, :, 15], t[:, :, 11]
    base = ent[ent > 0].min()
    print(f"== launch (global timer, us from the first CTA's entry): entry spread {(ent.max() - base) / 1e3:.2f}, "
          f"prologue done median {(np.median(pro) - base) / 1e3:.2f} max {(pro.max() - base) / 1e3:.2f}, "
          f"warp ends median {(np.median(end) - base) / 1e3:.2f} max {(end.max() - base) / 1e3:.2f}")
    for role, arr in roles:
        print(f"== {role} warps ({len(arr)}), mean over warps, us")
        for i, name in enumerate(NAMES):
            if name != "-" and arr[:, i].any():
                v = arr[:, i].mean()
                print(f"  {name:28s} {v / clk if i != 11 else v:9.2f}   (max {arr[:, i].max() / (clk if i != 11 else 1):.2f})")


if __name__ == "__main__":
    main()
