"""The drop-in C++ API as a user compiles it: tests/cpp/consumer.cpp built
against include/midbf/*.hpp and linked to libmidbf_b200.so (reference API
proj/include/midbf/butterfly.hpp:117-126, butterfly_io.hpp:24-28).  Building
and linking is checked on the CPU; running it needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "consumer.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "consumer")
LIBDIR = os.path.join(ROOT, "paper_1908_09376_b200")


def build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(SRC),
                                                           os.path.getmtime(os.path.join(LIBDIR, "libmidbf_b200.so"))):
        return
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", OUT,
                    "-L", LIBDIR, "-l:libmidbf_b200.so", f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_consumer_compiles_and_links_against_the_headers():
    build()
    syms = subprocess.run(["nm", "-C", "-u", OUT], capture_output=True, text=True).stdout
    for s in ("midbf::bf::apply(", "midbf::bf::apply_transpose(", "midbf::bf::idbf_factorize(",
              "midbf::bf::save_factorization(", "midbf::bf::load_factorization(", "midbf::tree::build_tree("):
        assert s in syms, s


@pytest.mark.gpu
def test_consumer_runs(gpu, tmp_path):
    build()
    p = subprocess.run([OUT, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "consumer ok" in p.stdout
