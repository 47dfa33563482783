"""Builds libtilefield_gpu.so in-tree (sm_100a only; nvcc cross-compiles here).

Translation units that carry the bit-exact contract (K1 sampler, K5 Adam, the
host-side camera/crop code) are compiled with -fmad=false / -ffp-contract=off.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libtilefield_gpu.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-ffp-contract=off",
    "-I", os.path.join(HERE, "..", "include"),
]
# (source, extra flags)
UNITS = [
    ("k_sampler.cu", ["-fmad=false"]),
    ("k_adam.cu", ["-fmad=false"]),
    ("tfg_api.cu", ["-fmad=false"]),
    ("tfg_io.cu", ["-fmad=false"]),
    ("tfg_eval.cu", ["-fmad=false"]),
    ("k_field.cu", []),
    ("k_field_tc.cu", []),
    ("k_composite.cu", []),
    ("k_eval.cu", ["-fmad=false"]),
    ("tfg_comm.cu", []),
]


def _newer(src_files, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_files)


def build(verbose: bool = False, force: bool = False, defines: list[str] | None = None,
          out: str | None = None, build_dir: str | None = None) -> str:
    """Compiles every unit for sm_100a and links the C-ABI library.  `defines`
    / `out` / `build_dir` build an A/B variant (tools/variants.py)."""
    lib_out = out or OUT
    bdir = build_dir or BUILD
    dflags = [f"-D{d}" for d in (defines or [])]
    os.makedirs(bdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "tilefield_gpu.h"))
    objs = []
    procs = []
    for src, extra in UNITS:
        s = os.path.join(CSRC, src)
        o = os.path.join(bdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer([s] + headers, o):
            cmd = [NVCC] + COMMON + extra + dflags + ["-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose and out:
            sys.stdout.write(out.decode())
    if force or procs or not os.path.exists(lib_out):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib_out] + objs + ["-cudart", "static", "-lpthread", "-ldl", "-lrt"]
        subprocess.check_call(cmd)
    return lib_out


def build_examples() -> str:
    """The C++ host programs against the C-ABI: the example trainer
    (examples/train_window.cpp) and the drop-in batch-operator caller of the
    adapter test (tests/cpp/field_adapter.cpp, include/tilefield_gpu_field.hpp)."""
    lib = build()
    out_dir = os.path.join(HERE, "bin")
    os.makedirs(out_dir, exist_ok=True)
    inc = os.path.join(HERE, "..", "include")
    hdrs = [os.path.join(inc, f) for f in os.listdir(inc)]
    exe = os.path.join(out_dir, "train_window")
    for name, src in (("train_window", os.path.join(HERE, "..", "examples", "train_window.cpp")),
                      ("field_adapter", os.path.join(HERE, "..", "tests", "cpp", "field_adapter.cpp"))):
        out = os.path.join(out_dir, name)
        if _newer([src, lib] + hdrs, out):
            subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-I", inc, "-o", out, src, "-L", HERE,
                                   "-ltilefield_gpu", "-Wl,-rpath,$ORIGIN/.."])
    return exe


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    build_examples()
    print(OUT)
