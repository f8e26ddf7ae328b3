"""Drop-in: the ACTUAL reference (every object of /root/reference/proj/core unchanged, solver.cpp compiled
through oracle/dropin/solver_gpu.cpp with INTEGRATION.md's binding) running apply_operator and gmres_solve
on the GPU, against the reference's own CPU implementations of the same functions in the same binary.
The binary is built where /root/reference exists (oracle/Makefile, target `dropin`; __graft_entry__.build())
and travels to the GPU box under oracle/_ref/."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_test")
needs_binary = pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/dropin_test not built (no /root/reference here)")


@needs_binary
def test_patched_reference_refuses_without_a_device(gpu_available):
    if gpu_available:
        pytest.skip("a GPU is present: covered by the gpu test")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 3 and "no CUDA device" in r.stdout     # loud failure, no CPU fallback
    assert "reference system:" in r.stdout                         # the reference's own setup ran on the host


@needs_binary
@pytest.mark.gpu
@pytest.mark.parametrize("args", [[], ["16", "10", "4.0"]], ids=["504-unknowns-k2.5", "864-unknowns-k4"])
def test_patched_reference_runs_its_solver_on_the_gpu(args):
    # sphere mesh, build_system (CPU correction builders), assemble_rhs: the reference's; apply_operator and
    # gmres_solve: the binding.  Checks: operator 1e-5, GMRES iteration count +-1 with and without block-Jacobi
    r = subprocess.run([EXE] + args, capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
