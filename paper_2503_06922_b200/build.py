"""In-tree build of the sm_100a library (libaccfem.so) with nvcc."""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libaccfem.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-shared",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))] + [
        os.path.join(HERE, "..", "include", "accfem.h")]


def stale():
    if not os.path.exists(SO):
        return True
    return os.path.getmtime(SO) < max(os.path.getmtime(p) for p in sources())


def build(force=False, verbose=False, profile=False):
    """Compile csrc/accfem.cu -> libaccfem.so when any source is newer.

    profile=True builds the development variant libaccfem_prof.so with the
    per-phase clock counters (-DACCFEM_PROFILE); the package never loads it.
    """
    so = SO.replace(".so", "_prof.so") if profile else SO
    if not force and os.path.exists(so) and os.path.getmtime(so) >= max(os.path.getmtime(p) for p in sources()):
        return so
    extra = ["-DACCFEM_PROFILE"] if profile else []
    cmd = [NVCC, *FLAGS, *extra, "-o", so + ".tmp", os.path.join(CSRC, "accfem.cu"), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if not profile:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
            fh.write(res.stderr)
    os.replace(so + ".tmp", so)
    if verbose:
        print(res.stderr)
    return so


if __name__ == "__main__":
    print(build(force=True))
