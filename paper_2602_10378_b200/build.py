"""In-tree build of libfkde_b200.so for sm_100a.

    python -m paper_2602_10378_b200.build

Compiles csrc/fkde_gpu.cu (which includes every kernel header) with nvcc
``-gencode arch=compute_100a,code=sm_100a -lineinfo``.  The .so lands next
to this file, is git-ignored, and travels to the GPU box with the repo.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libfkde_b200.so")
SOURCES = ["fkde_gpu.cu", "host_fixtures.cpp", "host_io.cpp"]
HEADERS = ["ptx.cuh", "layout.cuh", "pairwise_tc.cuh", "prep_kernels.cuh", "direct_rows.cuh",
           "spatial_order.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-shared",
]


def nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.isabs(p) and os.path.exists(p) or not os.path.isabs(p)):
            return p
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "fkde_gpu.h"))
    deps.append(os.path.join(HERE, "..", "include", "fkde_io.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Build the library (``out``; extra ``-D`` ``defines`` for tool variants,
    e.g. ``FKDE_ENABLE_TRACE`` for the clock64 trace build used by tools/)."""
    if out == OUT and not defines and not force and not _stale():
        return OUT
    cmd = [nvcc()] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
        ["-D" + d for d in defines] + ["-I", json_include()] + \
        ["-o", out] + [os.path.join(CSRC, s) for s in SOURCES] + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libfkde_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    return out


CLI_SRC = os.path.join(HERE, "cli", "fkde_cli.cpp")
CLI_OUT = os.path.join(HERE, "bin", "fkde-b200")


def json_include() -> str:
    """Directory holding nlohmann's single-header json.hpp (vendored in the image
    under cudnn_frontend's third-party tree); the CLI's only external header."""
    import sysconfig
    cands = [os.environ.get("FKDE_JSON_INCLUDE", "")]
    for base in {sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]}:
        cands.append(os.path.join(base, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
    for c in cands:
        if c and os.path.exists(os.path.join(c, "json.hpp")):
            return c
    raise RuntimeError("nlohmann/json.hpp not found (set FKDE_JSON_INCLUDE)")


def build_cli(force: bool = False) -> str:
    """g++ build of the fkde-b200 command-line tool (cli/fkde_cli.cpp) against
    libfkde_b200.so (rpath $ORIGIN/..)."""
    lib = build()
    if (not force and os.path.exists(CLI_OUT)
            and os.path.getmtime(CLI_OUT) >= max(os.path.getmtime(CLI_SRC), os.path.getmtime(lib))):
        return CLI_OUT
    os.makedirs(os.path.dirname(CLI_OUT), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(HERE, "..", "include"),
           "-I", json_include(), CLI_SRC, "-L", HERE, "-l:libfkde_b200.so",
           "-Wl,-rpath,$ORIGIN/..", "-o", CLI_OUT]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building fkde-b200")
    return CLI_OUT


if __name__ == "__main__":
    if "--trace" in sys.argv:   # python -m paper_2602_10378_b200.build --trace ab/lib_trace.so
        print(build(out=os.path.abspath(sys.argv[sys.argv.index("--trace") + 1]),
                    defines=["FKDE_ENABLE_TRACE"]))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
        print(build_cli(force="--force" in sys.argv))
