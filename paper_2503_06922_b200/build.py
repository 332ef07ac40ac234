"""In-tree build of the sm_100a library (libaccfem.so) with nvcc.

The translation units (csrc/accfem.cu: host ABI + small kernels;
csrc/ksolve_<NW>.cu: the persistent solve kernel per team width) are
compiled in parallel and linked into one shared library.
"""

import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libaccfem.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))] + [
        os.path.join(HERE, "..", "include", "accfem.h")]


def units():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cu")]


def stale():
    if not os.path.exists(SO):
        return True
    return os.path.getmtime(SO) < max(os.path.getmtime(p) for p in sources())


def build(force=False, verbose=False, profile=False):
    """Compile csrc/*.cu -> libaccfem.so when any source is newer.

    profile=True builds the development variant libaccfem_prof.so with the
    per-phase clock counters (-DACCFEM_PROFILE); the package never loads it.
    """
    so = SO.replace(".so", "_prof.so") if profile else SO
    if not force and os.path.exists(so) and os.path.getmtime(so) >= max(os.path.getmtime(p) for p in sources()):
        return so
    extra = ["-DACCFEM_PROFILE"] if profile else []
    with tempfile.TemporaryDirectory() as tmp:
        procs = []
        for cu in units():
            obj = os.path.join(tmp, os.path.basename(cu) + ".o")
            cmd = [NVCC, *FLAGS, *extra, "-c", "-o", obj, cu]
            procs.append((cu, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        log = []
        for cu, obj, p in procs:
            out, err = p.communicate()
            if p.returncode != 0:
                raise RuntimeError(f"nvcc failed on {cu}:\n{out}\n{err}")
            log.append(f"== {os.path.basename(cu)}\n{err}")
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", so + ".tmp",
               *[obj for _, obj, _ in procs], "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    if not profile:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
            fh.write("\n".join(log))
    os.replace(so + ".tmp", so)
    if verbose:
        print("\n".join(log))
    return so


if __name__ == "__main__":
    print(build(force=True))
