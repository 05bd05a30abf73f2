"""The drop-in boundary: libmidbf_b200.so loads and exports every entry point
include/midbf_b200.h declares; device entry points fail loudly (no CPU
fallback) when no sm_100 device is visible."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1908_09376_b200 as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "midbf_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(midbf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for need in ("midbf_plan_create", "midbf_plan_load", "midbf_apply", "midbf_sample", "midbf_direct_sum",
                 "midbf_factorize", "midbf_fact_save", "midbf_fact_load", "midbf_last_error"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", M.LIB_PATH], capture_output=True, text=True, check=True)
    exported = set(re.findall(r"\bT (midbf_[a-z0-9_]+)", out.stdout))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = M.lib()
    for s in declared_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", M.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_device_calls_fail_loudly_without_gpu():
    if M.device_count() > 0:
        pytest.skip("a device is visible")
    X = np.random.default_rng(0).random((64, 2))
    K = M.Kernel(M.KIND_FIO2D, X=X, Omega=X)
    with pytest.raises(M.MidbfCudaError):
        M.idbf_factorize(K, 16, sampler="device")
    with pytest.raises(M.MidbfCudaError):
        K.direct_sum(np.ones(64, complex))
    F = M.idbf_factorize(K, 16, sampler="host")  # host IDs + host entries work on CPU
    with pytest.raises(M.MidbfCudaError):
        F.apply(np.ones(64, complex))  # ...but the apply has no CPU path


def test_error_classes_follow_the_reference():
    X = np.random.default_rng(1).random((64, 2))
    K = M.Kernel(M.KIND_FIO2D, X=X, Omega=X)
    with pytest.raises(ValueError):  # rank cap must be positive (src/butterfly.cpp:303)
        M.idbf_factorize(K, 16, k=0, sampler="host")
    with pytest.raises(ValueError):  # sampling oversize must be positive (:304)
        M.idbf_factorize(K, 16, t=0, sampler="host")
    with pytest.raises(ValueError):  # build_tree: n0 must be positive (src/tree.cpp:36)
        M.idbf_factorize(K, 0, sampler="host")
    with pytest.raises(RuntimeError):  # missing container (src/butterfly_io.cpp:105)
        M.load_factorization("/nonexistent/midbf.bin")


def test_new_entry_points_fail_loudly_without_gpu():
    """K5 batched IDs, low-rank phase sampling and eps_K need the device."""
    if M.device_count() > 0:
        pytest.skip("a device is visible")
    with pytest.raises(M.MidbfCudaError):
        M.cid_batch([np.eye(4, dtype=complex)], 2, 1e-9)
    X = np.random.default_rng(2).random((64, 2))
    K = M.Kernel(M.KIND_FIO2D, X=X, Omega=X)
    with pytest.raises(M.MidbfCudaError):
        M.lowrank_phase(K, 2, 2, seed=1)
    with pytest.raises(M.MidbfCudaError):
        M.eps_K(K, np.zeros((64, 1)), np.zeros((64, 1)), 8, 1)


def test_host_linear_algebra_argument_errors():
    """rsvd / pinv / thin_q are host-only and reject bad arguments like the
    reference (std::invalid_argument -> ValueError)."""
    A = np.random.default_rng(3).standard_normal((10, 8))
    with pytest.raises(ValueError):  # sample index out of range
        M.rsvd_dense(A, [0, 11], [0, 1], 1, 0)
    with pytest.raises(ValueError):  # R0 / C0 of different sizes
        M.rsvd_dense(A, [0, 1, 2], [0, 1], 1, 0)
    P, cond = M.pinv(A)
    assert P.shape == (8, 10) and np.isfinite(cond)
    assert M.thin_q(A).shape == (10, 8)
