"""Build libtat.so in-tree for sm_100a with nvcc (no torch involvement).

    python -m paper_2510_24687_b200.build_lib        # or: from ... import build; build()
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libtat.so")
SOURCES = ["tat_api.cu", "kernels.cu", "kernels_fft.cu", "kernels_ring.cu", "kernels_ring2.cu", "kernels_dct.cu",
           "kernels_col.cu", "kernels_util.cu", "kernels_inv.cu", "kernels_dense.cu",
           "plan_host.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "tat.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every translation unit and link libtat.so (or `out`, with extra -D `defines`:
    tuning variants, e.g. python -m paper_2510_24687_b200.build_lib --out /tmp/v.so -DX=1)."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    nvcc = _nvcc()
    objdir = os.path.join(HERE, "build") if out is None else out + ".objs"
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:   # compile the translation units concurrently
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               *defines, "-I", INCLUDE, "-I", CSRC, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        else:
            cmd[1:1] = ["-x", "c++"]
        procs.append((src, subprocess.Popen(cmd)))
        objs.append(obj)
    bad = [src for src, p in procs if p.wait() != 0]
    if bad:
        raise RuntimeError(f"nvcc failed for {bad}")
    tmp = target + ".tmp"
    subprocess.run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"], check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                defines=[a for a in sys.argv[1:] if a.startswith("-D")], out=out))
