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


def test_cpp_facade_compiles_and_links(ph, tmp_path):
    """include/phmat_b200.hpp (reference-named C++ facade) compiles against
    the C ABI and links; without a GPU the context throws runtime_error and
    the host-only structure build works."""
    import shutil
    import subprocess

    if not shutil.which("g++"):
        pytest.skip("no g++")
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include "phmat_b200.hpp"
#include <cstdio>
int main() {
  std::vector<double> pts(2 * 256);
  phm_generate_points(256, 2, 3, pts.data());
  phmat_b200::PHConfig cfg;
  cfg.spec = phmat_b200::default_kernel_spec(phmat_b200::KernelFamily::SquaredExponential);
  cfg.l_max = 2; cfg.p_s = 4; cfg.p_theta = 5; cfg.eps = 1e-3;
  const phm_config cc = cfg.to_c(PHM_FORMAT_H2);
  phm_matrix m = nullptr;
  phmat_b200::check(phm_matrix_build_host(pts.data(), 256, 2, &cc, &m));
  phm_info info; phmat_b200::check(phm_matrix_info(m, &info));
  std::printf("near=%lld far=%lld\n", (long long)info.n_near, (long long)info.n_far);
  phm_matrix_destroy(m);
  try { phmat_b200::Context ctx(0); std::printf("gpu\n"); }
  catch (const std::runtime_error& e) { std::printf("nogpu\n"); }
  // the reference-shaped API: PHConfig / StageCounters / offline_h2 over a
  // row-major point matrix (no Eigen here: the facade's own Matrix type)
  phmat_b200::Matrix P(256, 2);
  for (int i = 0; i < 256; ++i) { P(i, 0) = pts[2 * i]; P(i, 1) = pts[2 * i + 1]; }
  phmat_b200::PHConfig rc;
  rc.spec = phmat_b200::default_kernel_spec(phmat_b200::KernelFamily::SquaredExponential);
  rc.l_max = 2; rc.p_s = 4; rc.p_theta = 5; rc.eps = 1e-3;
  phmat_b200::StageCounters counters;
  try { auto pm = phmat_b200::offline_h2(P, rc, counters); std::printf("built\n"); }
  catch (const std::runtime_error&) { std::printf("nogpu-build\n"); }
  try { std::vector<double> th{3.0}; phm_instance i; phmat_b200::check(phm_instantiate(nullptr, th.data(), 1, &i)); }
  catch (const std::invalid_argument&) { std::printf("invalid\n"); }
  return 0;
}
''')
    exe = tmp_path / "t"
    libdir = os.path.dirname(ph.library_path())
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                    "-L", libdir, "-lphmat_b200", f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert "near=" in out and "invalid" in out


def test_version_and_defaults(ph):
    assert ph.lib().phm_version() == 1
    c = ph.PHConfig().to_c(ph.Format.H2)
    # reference defaults, phmatrix.hpp:20-35
    assert (c.l_max, c.p_s, c.p_theta[0], c.eps, c.r_max_far, c.r_max_near) == (2, 15, 27, 1e-5, 120, 150)
