"""Build the helmsweep C-ABI shared library for sm_100a, in-tree.

    python -m paper_2408_11929_b200.build        (or __graft_entry__.build())

Produces paper_2408_11929_b200/libhelmsweep.so from csrc/*.cu with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3``.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhelmsweep.so")
SOURCES = ["assemble.cu", "strip_setup.cu", "sweep_apply.cu", "sweep_fast.cu", "sweep_dual.cu", "krylov.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "helmsweep.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, prof=False):
    """prof=True builds libhelmsweep_prof.so with the kernels' cycle counters
    (-DHELM_DUAL_PROF; load it with HELM_LIB=... for tools/prof_sweep.py)."""
    lib = LIB.replace(".so", "_prof.so") if prof else LIB
    if not force and not prof and not needs_build():
        return LIB
    objs = []
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
             "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3"]
    if prof:
        flags.append("-DHELM_DUAL_PROF")
    def compile_one(src):
        obj = os.path.join(CSRC, src.replace(".cu", "_prof.o" if prof else ".o"))
        cmd = [NVCC, "-c", os.path.join(CSRC, src), "-o", obj] + flags
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, "-shared", "-o", tmp] + objs + ["-gencode", "arch=compute_100a,code=sm_100a", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, prof="--prof" in sys.argv))
