"""The drop-in boundary: C ABI exports, C++ headers, no CPU fallback (runs on any host)."""
from __future__ import annotations

import ctypes as C
import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2008_12559_b200" / "libpft_b200.so"
HEADER = ROOT / "include" / "pft_capi.h"


def declared_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(pft_[A-Za-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(pft):
    names = declared_functions()
    assert len(names) >= 40
    lib = C.CDLL(str(LIB))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and nothing in the ctypes layer refers to an undeclared symbol
    from paper_2008_12559_b200 import _capi
    assert set(_capi.SIGNATURES) <= set(names)


def test_exported_symbols_are_c_linkage():
    nm = shutil.which("nm")
    if nm is None:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (pft_[A-Za-z0-9_]+)$", out, flags=re.M))
    assert set(declared_functions()) <= exported


def test_version_and_status_strings(pft):
    lib = pft.lib()
    assert b"sm_100a" in lib.pft_version()
    assert lib.pft_status_string(0) == b"ok"
    assert lib.pft_status_string(7) == b"non-finite input entries"


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(pft):
    """Without a GPU the transform fails loudly instead of computing on the CPU."""
    plan = pft.build_plan(4096, 32, 0, None, 1e-12)
    with pytest.raises(pft.PftDeviceError) as e:
        pft.execute(plan, [0j] * 4096)
    assert e.value.status == 10  # PFT_ERR_NO_DEVICE


def test_length_mismatch_is_a_value_error(pft):
    plan = pft.build_plan(4096, 32, 0, None, 1e-12)
    with pytest.raises(ValueError):
        pft.execute(plan, [0j] * 4095)


def _compile(args, out):
    res = subprocess.run(args + ["-o", str(out)], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


def test_types_header_compiles_with_gcc_and_nvcc(tmp_path):
    """include/pft/types.hpp is source compatible with the reference header (same names,
    members, semantics) and compiles -- the reference's does not (types.hpp:72)."""
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include "pft/types.hpp"
#include <cassert>
#include <cstdio>
int main() {
    using namespace pft;
    assert(mod_index(-12345, 6220800) == 6208455);   // SURVEY.md a2 (probed)
    assert(mod_index(7, 4) == 3 && mod_index(-1, 4) == 3);
    TargetRange R{37, 16};
    assert(R.count() == 33 && R.first() == 21 && R.last() == 53 && R.slot(21) == 0);
    bool threw = false;
    try { (void)R.slot(54); } catch (const std::out_of_range&) { threw = true; }
    assert(threw);
    PartialSpectrum s{R, ComplexVec(R.count(), cplx(1.0, 2.0)), 7};
    assert(s.at(40) == cplx(1.0, 2.0));
    PartialSpectrum2d s2{TargetRect{TargetRange{0, 1}, TargetRange{0, 2}}, ComplexVec(15), 0};
    s2.values[1 * 5 + 3] = 5.0;
    assert(s2.at(0, 1) == cplx(5.0, 0.0));
    ComplexMatrix m(3, 4);
    m.at(2, 3) = 1.0;
    assert(m.row(2)[3] == cplx(1.0, 0.0));
    assert(l1_norm(ComplexVec{cplx(3, 4), cplx(0, 1)}) == 6.0);
    const TargetRange a{1, 2}, b2{1, 2};
    assert(a == b2);
    std::puts("types ok");
}
''')
    exe = tmp_path / "t"
    _compile(["g++", "-std=c++20", "-I", str(ROOT / "include"), str(src)], exe)
    assert subprocess.run([str(exe)], capture_output=True, text=True).stdout.strip() == "types ok"
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    res = subprocess.run([nvcc, "-std=c++20", "-gencode", "arch=compute_100a,code=sm_100a", "-x", "cu", "-c",
                          "-I", str(ROOT / "include"), str(src), "-o", str(tmp_path / "t.o")],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


def _demo(tmp_path):
    exe = tmp_path / "demo"
    cuda = Path(shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc").resolve().parents[1]
    _compile(["g++", "-std=c++20", "-Wall", "-Werror", "-pthread", "-I", str(ROOT / "include"), "-I",
              str(cuda / "include"), str(ROOT / "examples" / "cpp_api_demo.cpp"), "-L", str(LIB.parent),
              "-lpft_b200", "-L", str(cuda / "lib64"), "-lcudart", f"-Wl,-rpath,{LIB.parent}",
              f"-Wl,-rpath,{cuda / 'lib64'}"], exe)
    return exe


def test_cpp_api_demo_builds_and_runs(tmp_path, pft):
    """examples/cpp_api_demo.cpp uses the reference's interface from C++ (pft/pft.hpp)."""
    exe = _demo(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert '"p": 32768' in res.stdout
    assert "device p = 16384, r = 8" in res.stdout  # pft_select_divisor_device at C2b


@pytest.mark.gpu
def test_cpp_api_demo_executes_on_the_gpu(tmp_path, pft):
    """The C++ drop-in path end to end on the B200: pft::execute (host vectors, the plan's staging
    pool), 4 threads x 3 executes sharing one plan, non-finite input -> std::invalid_argument.
    --require-gpu turns a pft::DeviceError into a failure (exit 6)."""
    exe = _demo(tmp_path)
    res = subprocess.run([str(exe), "--require-gpu"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "4 threads x 3 executes on one plan" in res.stdout
    assert "execute_sharded (1 rank)" in res.stdout
