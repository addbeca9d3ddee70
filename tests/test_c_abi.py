"""The C ABI from plain C (include/pgx.h is the drop-in boundary: extern "C",
plain pointers and sizes).  The CPU part compiles and links a C99 consumer
against the header and libpgx.so; the GPU part runs it."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "abi_smoke.c")
LIB_DIR = os.path.join(ROOT, "paper_2605_20816_b200", "lib")


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    if not os.path.exists(os.path.join(LIB_DIR, "libpgx.so")):
        pytest.skip("libpgx.so not built")
    exe = str(tmp_path / "abi_smoke")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(ROOT, "include"),
           SRC, "-L", LIB_DIR, "-lpgx", "-lm", f"-Wl,-rpath,{LIB_DIR}", "-o", exe]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    assert proc.returncode == 0, proc.stderr
    return exe


def test_c_consumer_compiles_and_links(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [0, 1, 2])  # PGX_PREC_EXACT / FP64 / TC
def test_c_consumer_runs(tmp_path, prec):
    exe = _build(tmp_path)
    proc = subprocess.run([exe, str(prec)], capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stdout + proc.stderr
    assert f"path {(0, 1, 2)[prec]}" in proc.stdout, proc.stdout
