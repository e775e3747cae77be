"""Builds libmggcn.so in-tree (nvcc, sm_100a). Used by __graft_entry__.build() and the tests.

    python -m paper_2110_08688_b200.build        # or: python paper_2110_08688_b200/build.py
"""
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmggcn.so")
LIB_RC = os.path.join(PKG, "libmggcn_rc.so")
SOURCES = ["mg_host.cpp", "mg_io.cpp", "mg_timeline.cpp", "mg_json.cpp", "mg_synth_rank.cpp", "mg_device.cu", "mg_tc_gemm.cu", "mg_prepare_dev.cu"]
HEADERS = ["mg_internal.hpp", "mg_kernels.cuh", "mg_tc_gemm.cuh", "mg_epi.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "mggcn.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, racecheck=False):
    """racecheck=True: libmggcn_rc.so, the compute-sanitizer racecheck variant (MG_RACECHECK_PLAIN_COPIES:
    the EXACT hub-row SpMM's cp.async copies become plain loads / stores with the same ring protocol)."""
    lib_out = LIB_RC if racecheck else LIB
    if not racecheck and not force and not needs_build():
        return LIB
    objs = []
    bdir = os.path.join(PKG, "build_rc" if racecheck else "build")
    os.makedirs(bdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    if racecheck:
        common += ["-DMG_RACECHECK_PLAIN_COPIES"]
    procs = []
    for src in SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = [nvcc(), *ARCH, "-lineinfo", *common, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + out)
        if verbose and out:
            print(out)
    tmp = lib_out + ".tmp"
    link = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lnccl", "-lpthread"]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed: " + " ".join(link) + "\n" + r.stdout)
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, racecheck="--racecheck" in sys.argv))
