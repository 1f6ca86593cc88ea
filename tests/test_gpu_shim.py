"""GPU: the C++ drop-in (include/hkkt_gpu.hpp) running restatements of the
reference's own hybrid-solver tests against the linked reference
(tests/cpp/test_gpu_shim.cpp; built by tests/cpp/Makefile from the
__graft_entry__.build() step where /root/reference exists)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tests" / "cpp" / "_build" / "test_gpu_shim"


@pytest.mark.gpu
def test_cpp_dropin_shim_runs_reference_cases():
    if not BIN.exists():
        pytest.fail(f"{BIN} not built (run __graft_entry__.build() where /root/reference exists)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "0 failed cases" in r.stdout


def test_cpp_dropin_header_compiles_against_reference():
    """CPU: hkkt_gpu.hpp compiles against the reference headers."""
    ref = Path("/root/reference/proj/core/include")
    if not ref.exists():
        pytest.skip("reference headers not present (GPU box)")
    src = '#include "hkkt_gpu.hpp"\nint main() { return 0; }\n'
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", f"-I{ref}",
                        f"-I{ROOT / 'include'}", "-x", "c++", "-"], input=src, capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
