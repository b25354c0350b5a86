"""A compiled C program calls libodyssey_b200.so through include/odyssey_b200.h -- the
reference's own kind of caller (odyssey.h consumers: the CLI, test_capi.cpp) -- built
with gcc against the header and linked to the in-tree library (tests/c_caller/)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2311_09550_b200")


def _build(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    if not os.path.exists(os.path.join(LIBDIR, "libodyssey_b200.so")):
        pytest.skip("libodyssey_b200.so not built")
    exe = str(tmp_path / "capi_example")
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_caller", "capi_example.c"), "-L" + LIBDIR, "-lodyssey_b200",
                    "-Wl,-rpath," + LIBDIR, "-lm", "-o", exe], check=True, capture_output=True, text=True)
    return exe


def test_c_caller_builds_and_links(tmp_path):
    """No GPU needed: the header compiles as C11, every referenced symbol resolves, and the
    GPU-free calls (tensor handles, EINVAL on NULL / NaN, thread-local messages) behave."""
    exe = _build(tmp_path)
    r = subprocess.run([exe, "--link-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok" in r.stdout


@pytest.mark.gpu
def test_c_caller_runs_the_reference_capi_flow(tmp_path):
    """ref test_capi.cpp:121-165 (FAST vs matmul_f32 of the dequantized operands <= 1e-4
    rel, counters) and every engine, from C."""
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi_example: ok" in r.stdout
