"""Build libpft_b200.so in-tree (host C++20 + sm_100a CUDA), with incremental rebuilds.

    python -m paper_2008_12559_b200.build [--force] [--verbose]

Host sources (csrc/host/*.cpp) are compiled with g++ and OpenMP; device sources
(csrc/device/*.cu) with nvcc for sm_100a only (-gencode arch=compute_100a,code=sm_100a)
and -lineinfo so ncu's source page maps to the kernels.  The CUDA runtime is linked
statically so the library loads on a machine without a GPU (planning works, device
calls return PFT_ERR_NO_DEVICE).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
LIB = PKG / "libpft_b200.so"
CLI = PKG / "pft"  # the command-line surface (SPEC.md cli module), linked against LIB
TABLE = PKG / "data" / "scope_table_v1.pftt"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
# /usr/bin/g++ first: the image's /opt/gcc wrapper cannot locate libgomp when linking
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# x86-64-v3 (AVX2/FMA): the library is built here and executed on the GPU box's host.
CUDA_INC = os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(NVCC))), "include")
HOST_FLAGS = ["-std=c++20", "-O3", "-march=x86-64-v3", "-fPIC", "-fopenmp", "-Wall", "-Wextra",
              "-Wno-unused-parameter", "-I", CUDA_INC]
NVCC_FLAGS = ["-std=c++20", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-fopenmp",
              "-Xptxas", "-O3", "--expt-relaxed-constexpr"]


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(map(str, cmd)), flush=True)
    res = subprocess.run([str(c) for c in cmd], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(map(str, cmd[:3]))} ...")
    if verbose and (res.stdout.strip() or res.stderr.strip()):
        print(res.stdout + res.stderr, flush=True)


def _write_table_blob() -> Path | None:
    gen = BUILD / "gen"
    gen.mkdir(parents=True, exist_ok=True)
    inc = gen / "table_blob.inc"
    if not TABLE.exists():
        if inc.exists():
            inc.unlink()
        return None
    data = TABLE.read_bytes()
    lines = ["// generated from data/scope_table_v1.pftt by build.py -- do not edit",
             "static const unsigned char kPftTableBlob[] = {"]
    for i in range(0, len(data), 20):
        lines.append("    " + ", ".join(str(b) for b in data[i:i + 20]) + ",")
    lines.append("};")
    text = "\n".join(lines) + "\n"
    if not inc.exists() or inc.read_text() != text:
        inc.write_text(text)
    return inc


def _deps_hash(src: Path) -> str:
    h = hashlib.sha256()
    h.update(src.read_bytes())
    for d in sorted((CSRC / "host").glob("*.hpp")) + sorted((CSRC / "common").glob("*.h")) + \
            sorted((CSRC / "device").glob("*.cuh")) + sorted(INCLUDE.rglob("*.h*")):
        h.update(d.read_bytes())
    blob = BUILD / "gen" / "table_blob.inc"
    if src.name == "table_default.cpp" and blob.exists():
        h.update(blob.read_bytes())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    """checked=True: the bounds-checked flavour (-DPFT_CHECKED: every computed workspace / output /
    input index is checked and traps) as libpft_b200_checked.so, for the GPU check runs
    (PFT_LIB=... python tools/sanitize.py / pytest); the product library is unchanged."""
    global BUILD, LIB
    if checked:
        BUILD, LIB = PKG / "build" / "checked", PKG / "libpft_b200_checked.so"
    BUILD.mkdir(parents=True, exist_ok=True)
    _write_table_blob()
    objs: list[Path] = []
    jobs: list[list] = []
    incs = ["-I", INCLUDE, "-I", CSRC, "-I", BUILD / "gen"]
    for src in sorted((CSRC / "host").glob("*.cpp")):
        obj = BUILD / f"host_{src.stem}_{_deps_hash(src)}.o"
        if force or not obj.exists():
            jobs.append([CXX, *HOST_FLAGS, *incs, "-c", src, "-o", obj])
        objs.append(obj)
    for src in sorted((CSRC / "device").glob("*.cu")):
        obj = BUILD / f"dev_{src.stem}_{_deps_hash(src)}.o"
        if force or not obj.exists():
            jobs.append([NVCC, *NVCC_FLAGS, *(["-DPFT_CHECKED"] if checked else []), *incs, "-c", src, "-o", obj])
        objs.append(obj)
    # translation units compile concurrently (the kernel instantiations dominate)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_run, j, verbose) for j in jobs]:
            f.result()
    stamp = "".join(sorted(o.name for o in objs))
    stamp_file = BUILD / "link.stamp"
    if force or not LIB.exists() or not stamp_file.exists() or stamp_file.read_text() != stamp:
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, "-shared", *ARCH, "-o", tmp, *objs, "-Xcompiler", "-fopenmp", "-lgomp", "-ldl"], verbose)
        os.replace(tmp, LIB)
        stamp_file.write_text(stamp)
    # the CLI (host code compiled by nvcc: it times with CUDA events), rpath'd to the library
    cli_src = CSRC / "cli" / "pft_cli.cu"
    cli_stamp = BUILD / "cli.stamp"
    cli_key = _deps_hash(cli_src) + LIB.stat().st_mtime_ns.__str__() if cli_src.exists() else ""
    if not checked and cli_src.exists() and (force or not CLI.exists() or not cli_stamp.exists() or
                                              cli_stamp.read_text() != cli_key):
        tmp = CLI.with_suffix(".tmp")
        _run([NVCC, "-std=c++20", "-O2", *ARCH, "-I", INCLUDE, cli_src, "-o", tmp, "-L", PKG, "-lpft_b200",
              "-Xlinker", "-rpath,$ORIGIN", "-ldl"], verbose)
        os.replace(tmp, CLI)
        cli_stamp.write_text(cli_key)
    # drop stale objects
    live = {o.name for o in objs}
    for o in BUILD.glob("*.o"):
        if o.name not in live:
            o.unlink()
    lib = LIB
    if checked:
        BUILD, LIB = PKG / "build", PKG / "libpft_b200.so"
    return lib


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--checked", action="store_true", help="bounds-checked flavour (libpft_b200_checked.so)")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, checked=a.checked))


if __name__ == "__main__":
    main()
