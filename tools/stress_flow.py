"""Race hunt for k1_flow: alternate two inputs over many device applies per
(variant, compressed/dense-only, direction) and compare every result
bitwise with the first result of the same input (the apply is run-to-run
bitwise deterministic).  Usage: python tools/stress_flow.py cfg1 cfg3 ..."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1908_09376_b200 as M  # noqa: E402

REPS = int(os.environ.get("REPS", "2000"))
for name in sys.argv[1:]:
    K, X, Om, fk, nrhs, desc = bench.workload(name)
    F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, t=5, seed=M.chain(0, 0x666163), sampler="device")
    plan = F.plan(3)
    sp = torch.cuda.current_stream().cuda_stream
    for tr in (False, True):
        nin, nout = (F.nrows, F.ncols) if tr else (F.ncols, F.nrows)
        fs = [torch.from_numpy(M.random_coefficients(nin, s)).to("cuda") for s in (1, 2)]
        for v in (0, 1):
            for lite in (False, True):
                plan.set_flags(variant=v, lite=lite)
                outs = [torch.empty(nout, dtype=torch.complex128, device="cuda") for _ in range(8)]
                ref = []
                for i in range(2):
                    r = torch.empty(nout, dtype=torch.complex128, device="cuda")
                    plan.apply_ptr(fs[i].data_ptr(), r.data_ptr(), 1, tr, sp)
                    ref.append(r)
                bad, nan = 0, 0
                for rep in range(REPS):
                    o = outs[rep % 8]
                    plan.apply_ptr(fs[rep & 1].data_ptr(), o.data_ptr(), 1, tr, sp)
                    if rep % 8 == 7:
                        for j in range(8):
                            if not torch.equal(outs[j], ref[(rep - 7 + j) & 1]):
                                bad += 1
                                nan += int(torch.isnan(outs[j].real).sum().item())
                torch.cuda.synchronize()
                print(name, "T" if tr else "F", "variant", v, "lite", lite, "bad", bad, "nan", nan,
                      "finite_ref", bool(torch.isfinite(ref[0].real).all()), flush=True)
    plan.set_flags()
