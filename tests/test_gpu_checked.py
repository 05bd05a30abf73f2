"""The checked build (libmidbf_b200_checked.so: the same sources with
device-side bounds assertions on every table-driven access of the apply
kernels, csrc/device/common.cuh MIDBF_DCHECK) runs the small parity workload
of tools/sanitize_cases.py — every kernel family, both directions, every
single-RHS kernel and layout, multi-RHS, direct sums — and must finish with
every result within 1e-12 of the oracle and no assertion firing.  This pool
closes compute-sanitizer; this is the memcheck stand-in."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1908_09376_b200", "libmidbf_b200_checked.so")

pytestmark = pytest.mark.gpu


def test_checked_build_runs_the_parity_cases_clean(gpu):
    assert os.path.exists(CHECKED), "build the checked library: make -C paper_1908_09376_b200 checked"
    env = dict(os.environ, MIDBF_LIB=CHECKED)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], capture_output=True,
                       text=True, timeout=900, env=env, cwd=ROOT)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert "MIDBF_CHECKED violation" not in out
    assert "sanitize cases ok" in p.stdout


def test_checked_library_is_the_one_loaded(gpu):
    env = dict(os.environ, MIDBF_LIB=CHECKED)
    code = "import paper_1908_09376_b200 as M; print(M.LIB_PATH)"
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)
    assert p.stdout.strip() == CHECKED
