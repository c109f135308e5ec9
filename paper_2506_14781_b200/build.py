"""Build the sm_100a engine library in-tree (paper_2506_14781_b200/libtempergrid_b200.so).

    python -m paper_2506_14781_b200.build          # engine only
    python -m paper_2506_14781_b200.build --all    # engine + oracle checkers

nvcc cross-compiles for sm_100a without a GPU.  The .so is git-ignored but
travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtempergrid_b200.so")
SOURCES = ["kernels.cu", "capi.cu", "host_common.cu", "host_plane.cu", "host_slot.cu",
           "host_run.cu", "host_extras.cu", "host_ckpt.cu", "plane_sweep.cu", "plane_tpw.cu", "plane_c5.cu", "plane_cl.cu", "slot_engine.cu", "slot_fast.cu", "prep.cu"]
HEADERS = ["engine.cuh", "kernels.cuh", "philox.cuh", "philox_plane.cuh", "plane_device.cuh", "plane_round.cuh",
           "host.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_engine(force: bool = False, verbose: bool = False) -> str:
    """Compile each translation unit to an object in parallel, then link."""
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "tempergrid_b200.h"))
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    units = [("kernels.cu", "kernels.o", []), ("capi.cu", "capi.o", []),
             ("host_common.cu", "host_common.o", []), ("host_plane.cu", "host_plane.o", []),
             ("host_slot.cu", "host_slot.o", []), ("host_run.cu", "host_run.o", []),
             ("host_extras.cu", "host_extras.o", []), ("host_ckpt.cu", "host_ckpt.o", []),
             ("plane_sweep.cu", "plane_r0.o", ["-DTG_PLANE_RULE=0"]),
             ("plane_sweep.cu", "plane_r1.o", ["-DTG_PLANE_RULE=1"]),
             ("plane_tpw.cu", "tpw_r0.o", ["-DTG_PLANE_RULE=0"]),
             ("plane_tpw.cu", "tpw_r1.o", ["-DTG_PLANE_RULE=1"]),
             ("plane_c5.cu", "plane_c5.o", []),
             ("plane_cl.cu", "plane_cl.o", []),
             ("slot_engine.cu", "slot_engine.o", []), ("slot_fast.cu", "slot_fast.o", []),
             ("prep.cu", "prep.o", [])]
    procs = []
    for src, obj, extra in units:
        cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v",
               "-Xcompiler", "-fPIC", *extra, "-c", os.path.join(CSRC, src),
               "-o", os.path.join(objdir, obj)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
    log = []
    ok = True
    for cmd, pr in procs:
        out, err = pr.communicate()
        log.append(" ".join(cmd) + "\n" + out + err)
        ok &= pr.returncode == 0
    with open(os.path.join(PKG, "build_ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if not ok:
        sys.stderr.write("\n".join(log))
        raise RuntimeError("nvcc failed building %s" % LIB)
    link = [nvcc(), *ARCH, "-shared", "-o", LIB,
            *[os.path.join(objdir, u[1]) for u in units], "-ldl"]
    subprocess.run(link, check=True)
    if verbose:
        sys.stdout.write("\n".join(log))
    return LIB


def build_oracle() -> None:
    targets = ["port"]
    if os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), *targets], check=True)


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    force = "--force" in argv
    build_engine(force=force, verbose="-v" in argv)
    if "--all" in argv:
        build_oracle()
    print(LIB)
    return 0


if __name__ == "__main__":
    sys.exit(main())
