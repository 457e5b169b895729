"""The C-ABI library builds for sm_100a, loads, and exports every symbol that
include/dot_b200.h declares (no GPU needed); host-only utilities work."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dot_b200.h")


@pytest.fixture(scope="module")
def libpath():
    from paper_1706_05586_b200 import build
    return build.build()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dot_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_paper_calls():
    names = declared_functions()
    for n in ("dot_set_params", "dot_misfit", "dot_jacobian", "dot_optimize_directions"):
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}\b", out), n


def test_library_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_binding_loads_and_reports_version(libpath):
    import paper_1706_05586_b200 as dot
    assert "sm_100a" in dot.version()


def test_host_sym_eig_matches_definition(libpath):
    """dot_sym_eig (used for the Table 1 SVDs through Lemma 3.2): A Z = Z diag(w),
    Z orthogonal, eigenvalues descending -- checked from the definition."""
    import paper_1706_05586_b200 as dot
    rng = np.random.default_rng(0)
    for n in (1, 2, 3, 7, 40, 130):
        M = rng.standard_normal((n, n + 3))
        A = M @ M.T
        w, Z = dot.sym_eig(A)
        assert np.all(np.diff(w) <= 1e-12 * max(1.0, abs(w[0])))
        assert np.abs(Z.T @ Z - np.eye(n)).max() < 1e-12
        assert np.abs(A @ Z - Z * w).max() < 1e-11 * np.abs(A).max()
    # repeated eigenvalues / diagonal / zero matrix
    w, Z = dot.sym_eig(np.diag([3.0, 1.0, 3.0, 2.0]))
    assert np.allclose(w, [3, 3, 2, 1])
    w, Z = dot.sym_eig(np.zeros((4, 4)))
    assert np.allclose(w, 0) and np.abs(Z.T @ Z - np.eye(4)).max() < 1e-14


def test_problem_without_gpu_fails_loudly(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1706_05586_b200 as dot
    with pytest.raises(RuntimeError):
        dot.DOTProblem((4, 4, 4), (1, 1, 1), 0.03, 0.15, 0.05, 2.2e10, [0.0], [0], [60], 1, 0.01, 0.1, 0.15)
