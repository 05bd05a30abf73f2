"""Regenerate the committed golden fixtures (run from the repo root):

    python tests/golden/make_golden.py

Each case stores a MIDBF001 container built by the CPU oracle plus an .npz
with a seeded input f, the oracle's apply g = F f, transpose apply F^T f and
the direct sum K f.  The reference itself cannot run here (DESIGN.md
"Oracle"), so these fixtures freeze the oracle's outputs: the CPU tests
check the oracle still reproduces them bit for bit, the GPU tests check the
device path against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))
import oracle as O  # noqa: E402
from helpers import integer_grid  # noqa: E402

CASES = {
    # name: (X, Omega, n0, k, eps, seed)
    "fio16_unitxi": (lambda: O.grid2d(16), lambda: O.grid2d(16), 64, 30, 1e-9, 0),
    "fio16_intxi": (lambda: O.grid2d(16), lambda: integer_grid(16), 64, 20, 1e-9, 0),
    "scattered256": (lambda: np.random.default_rng(5).random((256, 2)), lambda: np.random.default_rng(6).random((256, 2)),
                     16, 12, 1e-9, 1),
}


def build(name):
    mk_x, mk_o, n0, k, eps, seed = CASES[name]
    X, Om = mk_x(), mk_o()
    K = O.Kernel(O.KIND_FIO2D, X=X, Omega=Om)
    F = O.factorize(K, X, Om, n0, k=k, eps=eps, seed=seed, parallel=False)
    f = O.random_coefficients(len(Om), O.chain(seed, 0x66))
    return X, Om, K, F, f


def main():
    for name in CASES:
        X, Om, K, F, f = build(name)
        F.save(os.path.join(HERE, f"{name}.midbf"))
        np.savez(os.path.join(HERE, f"{name}.npz"), X=X, Omega=Om, f=f, g=F.apply(f, parallel=False),
                 gt=F.apply_transpose(f, parallel=False), gd=K.direct_sum(f), total_nnz=F.total_nnz)
        print(name, F.total_nnz, os.path.getsize(os.path.join(HERE, f"{name}.midbf")))


if __name__ == "__main__":
    main()
