"""Committed golden fixtures (tests/golden/, made by make_golden.py): the CPU
oracle and the product host factorization must reproduce them exactly; the
device apply / direct sum must match them to rel-L2 <= 1e-12."""
import filecmp
import os
import tempfile

import numpy as np
import pytest

import oracle as O
import paper_1908_09376_b200 as M
from helpers import rel

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["fio16_unitxi", "fio16_intxi", "scattered256"]
PARAMS = {"fio16_unitxi": (64, 30, 1e-9, 0), "fio16_intxi": (64, 20, 1e-9, 0), "scattered256": (16, 12, 1e-9, 1)}


def fixture(name):
    return os.path.join(GOLD, f"{name}.midbf"), dict(np.load(os.path.join(GOLD, f"{name}.npz")))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name):
    path, io = fixture(name)
    F = O.load(path)
    assert F.total_nnz == int(io["total_nnz"])
    assert np.array_equal(F.apply(io["f"], parallel=False), io["g"])
    assert np.array_equal(F.apply(io["f"], parallel=True), io["g"])  # group order fixed (test_butterfly.cpp:275)
    assert np.array_equal(F.apply_transpose(io["f"], parallel=False), io["gt"])
    K = O.Kernel(O.KIND_FIO2D, X=io["X"], Omega=io["Omega"])
    assert np.array_equal(K.direct_sum(io["f"]), io["gd"])


@pytest.mark.parametrize("name", NAMES)
def test_factorizations_reproduce_golden_containers(name):
    path, io = fixture(name)
    n0, k, eps, seed = PARAMS[name]
    with tempfile.TemporaryDirectory() as d:
        Fo = O.factorize(O.Kernel(O.KIND_FIO2D, X=io["X"], Omega=io["Omega"]), io["X"], io["Omega"], n0, k=k,
                         eps=eps, seed=seed, parallel=False)
        Fo.save(os.path.join(d, "o.midbf"))
        assert filecmp.cmp(path, os.path.join(d, "o.midbf"), shallow=False)
        Fm = M.idbf_factorize(M.Kernel(M.KIND_FIO2D, X=io["X"], Omega=io["Omega"]), n0, k=k, eps=eps, seed=seed,
                              parallel=False, sampler="host")
        Fm.save(os.path.join(d, "m.midbf"))
        assert filecmp.cmp(path, os.path.join(d, "m.midbf"), shallow=False)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_matches_golden(gpu, name):
    path, io = fixture(name)
    plan = M.DevicePlan.load(path, directions=3)
    assert rel(plan.apply(io["f"]), io["g"]) <= 1e-12
    assert rel(plan.apply(io["f"], transpose=True), io["gt"]) <= 1e-12
    K = M.Kernel(M.KIND_FIO2D, X=io["X"], Omega=io["Omega"])
    assert rel(K.direct_sum(io["f"]), io["gd"]) <= 1e-12
