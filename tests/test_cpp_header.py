"""The C++ drop-in header (include/sparsegate/ffn_exec.hpp) compiles against the
C ABI and behaves like the reference API (tests/cpp/header_check.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2603_14110_b200")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "header_check")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "header_check.cpp"), "-L" + PKG, "-lsparsegate_b200",
           "-Wl,-rpath," + PKG, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_header_host_entry_points(binary):
    r = subprocess.run([binary, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_header_executor_known_answers(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


REF_BIN = os.path.join(ROOT, "tests", "cpp", "_ref_tests", "ffn_exec_tests")


@pytest.mark.gpu
def test_reference_ffn_exec_tests_unmodified():
    """/root/reference/proj/tests/ffn_exec_tests.cpp, compiled UNMODIFIED against this
    repo's drop-in headers (include/sparsegate/{common,types,ffn_exec,factorization}.hpp
    over libsparsegate_b200.so; tests/cpp/Makefile, built by __graft_entry__.build()
    where /root/reference exists), runs every TEST_CASE / SECTION on the B200."""
    assert os.path.exists(REF_BIN), f"{REF_BIN} was not built (make -C tests/cpp)"
    r = subprocess.run([REF_BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " 0 failed" in r.stdout
