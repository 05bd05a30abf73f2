"""Regenerate the committed golden fixtures (run from the repo root, in the
container where /root/reference exists):

    python tests/golden/make_golden.py

Provenance: every fixture is produced by the REFERENCE's own code —
/root/reference/proj/src compiled unmodified against the Eigen stand-in in
oracle/shim/ (oracle/ref.mk -> oracle/_ref/libmidbf_ref.so, C ABI in
oracle/ref_capi.cpp):
  <name>.midbf  bf::idbf_factorize (src/butterfly.cpp:708-769) with the
                reference's entry evaluators (ker::make_accessor scenario 1,
                src/kernels.cpp:228-245; metrics::phase_entry_fn,
                src/metrics.cpp:18-24), Exec::Serial, saved by
                bf::save_factorization (src/butterfly_io.cpp:63-101);
  <name>.npz    the seeded inputs f, ft (the oracle's restatement of the
                experiment's generator, src/experiment.cpp:75-81 — inputs
                only), g = bf::apply(F, f), gt = bf::apply_transpose(F, ft),
                gd = the direct sum through the reference's evaluator in the
                loop order of src/metrics.cpp:40-43, ref_eps_b =
                metrics::eps_b(F, K, f, 256, seed) (src/metrics.cpp:26-53),
                and the factorization parameters.
The only non-reference arithmetic is the stand-in's: Eigen3 is unpinned in
the reference (proj/CMakeLists.txt:29), so the summation order inside its
GEMV / norms is the shim's documented plain order.  The CPU tests require
the oracle and the product's host factorize to reproduce these bytes
exactly; the GPU tests require the device path to match them to 1e-12.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))
import oracle as O  # noqa: E402  (input generator only)
import ref as R  # noqa: E402
from helpers import integer_grid, unit_grid  # noqa: E402


def _lowrank():
    rng = np.random.default_rng(7)
    return rng.standard_normal((256, 8)) * 0.25, rng.standard_normal((256, 8)) * 0.25


CASES = {
    # name: (kind, X, Omega, A, B, n0, k, eps, seed)
    "fio16_unitxi": (R.KIND_FIO2D, lambda: R.grid2d(16), lambda: R.grid2d(16), None, None, 64, 30, 1e-9, 0),
    "fio16_intxi": (R.KIND_FIO2D, lambda: R.grid2d(16), lambda: integer_grid(16), None, None, 64, 20, 1e-9, 0),
    "scattered256": (R.KIND_FIO2D, lambda: np.random.default_rng(5).random((256, 2)),
                     lambda: np.random.default_rng(6).random((256, 2)), None, None, 16, 12, 1e-9, 1),
    "lowrank16": (R.KIND_LOWRANK, lambda: R.grid2d(16), lambda: R.grid2d(16), lambda: _lowrank()[0],
                  lambda: _lowrank()[1], 16, 12, 1e-9, 2),
    "nufft3d_n8": (R.KIND_NUFFT, lambda: unit_grid(8, 3), lambda: unit_grid(8, 3) * 4.0, None, None, 64, 24, 1e-9,
                   3),
}
KINDS = {R.KIND_FIO2D: O.KIND_FIO2D, R.KIND_LOWRANK: O.KIND_LOWRANK, R.KIND_NUFFT: O.KIND_NUFFT}


def problem(name):
    kind, mx, mo, ma, mb, n0, k, eps, seed = CASES[name]
    X, Om = mx(), mo()
    A = ma() if ma else None
    B = mb() if mb else None
    return R.Problem(kind, X, Om, A=A, B=B), (n0, k, eps, seed)


def main():
    for name in CASES:
        P, (n0, k, eps, seed) = problem(name)
        path = os.path.join(HERE, f"{name}.midbf")
        P.factorize(n0, k=k, eps=eps, seed=seed, parallel=False, path=path)
        f = O.random_coefficients(len(P.Omega), O.chain(seed, 0x66))
        g = R.apply(path, f)
        ft = O.random_coefficients(len(P.X), O.chain(seed, 0x67))
        gt = R.apply(path, ft, transpose=True)
        gd = P.direct_sum(f)
        e = P.eps_b(path, f, 256, O.chain(seed, 0x657062))
        inf = R.info(path)
        extra = {} if P.A is None else {"A": P.A, "B": P.B}
        np.savez(os.path.join(HERE, f"{name}.npz"), X=P.X, Omega=P.Omega, f=f, g=g, ft=ft, gt=gt, gd=gd, ref_eps_b=e,
                 total_nnz=inf["total_nnz"], kind=P.kind, n0=n0, k=k, eps=eps, seed=seed, **extra)
        print(name, inf["total_nnz"], os.path.getsize(path), f"eps_b={e:.3e}")


if __name__ == "__main__":
    main()
