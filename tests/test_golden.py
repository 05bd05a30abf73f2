"""Committed golden fixtures (tests/golden/, made by make_golden.py from the
REFERENCE's own code compiled in oracle/_ref): the CPU oracle and the
product's host factorization must reproduce them exactly (container bytes,
apply, transpose apply, direct sum); the device apply / direct sum must
match them to rel-L2 <= 1e-12 (north_star)."""
import filecmp
import os
import tempfile

import numpy as np
import pytest

import oracle as O
import paper_1908_09376_b200 as M
from helpers import rel

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["fio16_unitxi", "fio16_intxi", "scattered256", "lowrank16", "nufft3d_n8"]


def fixture(name):
    return os.path.join(GOLD, f"{name}.midbf"), dict(np.load(os.path.join(GOLD, f"{name}.npz")))


def kernel(mod, io):
    kind = int(io["kind"])  # oracle / ref / product share the kind numbering
    if "A" in io:  # low-rank phase: entries from A, B; trees from X, Omega
        return mod.Kernel(kind, X=io["X"], Omega=io["Omega"], A=io["A"], B=io["B"])
    return mod.Kernel(kind, X=io["X"], Omega=io["Omega"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name):
    path, io = fixture(name)
    F = O.load(path)
    assert F.total_nnz == int(io["total_nnz"])
    assert np.array_equal(F.apply(io["f"], parallel=False), io["g"])
    assert np.array_equal(F.apply(io["f"], parallel=True), io["g"])  # group order fixed (test_butterfly.cpp:275)
    assert np.array_equal(F.apply_transpose(io["ft"], parallel=False), io["gt"])
    assert np.array_equal(kernel(O, io).direct_sum(io["f"]), io["gd"])
    # metrics::eps_b on the same rows / seed (src/metrics.cpp:26-53)
    e = kernel(O, io).eps_b(F.apply(io["f"]), io["f"], 256, O.chain(int(io["seed"]), 0x657062))
    assert e == float(io["ref_eps_b"])


@pytest.mark.parametrize("name", NAMES)
def test_factorizations_reproduce_golden_containers(name):
    path, io = fixture(name)
    n0, k, eps, seed = int(io["n0"]), int(io["k"]), float(io["eps"]), int(io["seed"])
    with tempfile.TemporaryDirectory() as d:
        Fo = O.factorize(kernel(O, io), io["X"], io["Omega"], n0, k=k, eps=eps, seed=seed, parallel=False)
        Fo.save(os.path.join(d, "o.midbf"))
        assert filecmp.cmp(path, os.path.join(d, "o.midbf"), shallow=False)
        Fm = M.idbf_factorize(kernel(M, io), n0, k=k, eps=eps, seed=seed, parallel=False, sampler="host")
        Fm.save(os.path.join(d, "m.midbf"))
        assert filecmp.cmp(path, os.path.join(d, "m.midbf"), shallow=False)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_matches_golden(gpu, name):
    path, io = fixture(name)
    plan = M.DevicePlan.load(path, directions=3)
    assert rel(plan.apply(io["f"]), io["g"]) <= 1e-12
    assert rel(plan.apply(io["ft"], transpose=True), io["gt"]) <= 1e-12
    assert rel(kernel(M, io).direct_sum(io["f"]), io["gd"]) <= 1e-12
