"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
no GPU compute is called here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "phmat_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(phm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(ph):
    lib = ctypes.CDLL(ph.library_path())
    syms = header_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header(ph):
    assert sorted(ph.SIGNATURES) == header_symbols()


def test_no_device_fails_loudly_without_gpu(ph):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ph.CudaError):
        ph.Context(0)


def test_library_is_sm100a(ph):
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    out = subprocess.run(["cuobjdump", "--list-elf", ph.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_defaults(ph):
    assert ph.lib().phm_version() == 1
    c = ph.PHConfig().to_c(ph.Format.H2)
    # reference defaults, phmatrix.hpp:20-35
    assert (c.l_max, c.p_s, c.p_theta[0], c.eps, c.r_max_far, c.r_max_near) == (2, 15, 27, 1e-5, 120, 150)
