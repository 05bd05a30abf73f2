"""Race hunt for the single-RHS dataflow kernel (k1_flow) inside the GPU
suite: many back-to-back device applies per (layout variant, compressed /
dense-only records, direction), alternating two inputs, every result
compared bitwise with the first result of the same input (the apply is
run-to-run bitwise deterministic: fixed summation order per strip, no
atomics).  A leaked stage-buffer sentinel or a torn read shows up as a
mismatch or a NaN.  Reference behaviour matched: src/butterfly.cpp:624-667
(the output equals the serial fixed-order apply)."""
import os

import numpy as np
import pytest

import paper_1908_09376_b200 as M
from helpers import cases, cvec, integer_grid, oracle_factorization, rel, saved, unit_grid

import oracle as O

pytestmark = pytest.mark.gpu
REPS = int(os.environ.get("MIDBF_STRESS_REPS", "64"))
PICK = ("fio_n32", "cfg0_intxi_n64", "scattered_odd", "nufft3d", "fio3d_n8")


@pytest.fixture(scope="module", params=[c for c in cases() if c[0] in PICK] + [
    ("fio3d_n16_wide", O.KIND_FIO3D, unit_grid(16, 3), integer_grid(16, 3), 64, 64, 1e-9)], ids=lambda c: c[0])
def plan_case(request, gpu):
    name, kind, X, Om, n0, k, eps = request.param
    K, Fo = oracle_factorization(kind, X, Om, n0, k, eps)
    path = saved(Fo)
    plan = M.DevicePlan.load(path, directions=3)
    os.unlink(path)
    return Fo, plan


@pytest.mark.parametrize("transpose", [False, True], ids=["fwd", "tr"])
def test_back_to_back_applies_are_bitwise_stable(plan_case, transpose):
    torch = pytest.importorskip("torch")
    Fo, plan = plan_case
    nin, nout = (Fo.nrows, Fo.ncols) if transpose else (Fo.ncols, Fo.nrows)
    host = [cvec(nin, s) for s in (101, 102)]
    want = [Fo.apply_transpose(f) if transpose else Fo.apply(f) for f in host]
    fs = [torch.from_numpy(f).cuda() for f in host]
    sp = torch.cuda.current_stream().cuda_stream
    total = 0
    try:
        for kw in (dict(variant=0, lite=False), dict(variant=1, lite=False), dict(variant=0, lite=True),
                   dict(variant=1, lite=True), dict(), dict(chain=False), dict(chain=False, variant=1, lite=False),
                   dict(coop=True), dict(coop=True, chain=False), dict(variant=0, prologue=True),
                   dict(variant=0, lite=True, chain=False)):
            plan.set_flags(**kw)
            ref = [torch.empty(nout, dtype=torch.complex128, device="cuda") for _ in range(2)]
            for i in range(2):
                plan.apply_ptr(fs[i].data_ptr(), ref[i].data_ptr(), 1, transpose, sp)
            torch.cuda.synchronize()
            for i in range(2):
                assert rel(ref[i].cpu().numpy(), want[i]) <= 1e-12, (kw, i)
            outs = [torch.empty(nout, dtype=torch.complex128, device="cuda") for _ in range(8)]
            bad = []
            for rep in range(REPS):
                plan.apply_ptr(fs[rep & 1].data_ptr(), outs[rep % 8].data_ptr(), 1, transpose, sp)
                total += 1
                if rep % 8 == 7:
                    for j in range(8):
                        if not torch.equal(outs[j], ref[(rep - 7 + j) & 1]):
                            bad.append((rep - 7 + j, int(torch.isnan(outs[j].real).sum().item())))
            torch.cuda.synchronize()
            assert not bad, (kw, bad[:8])
    finally:
        plan.reset_flags()
    assert total >= 11 * REPS
