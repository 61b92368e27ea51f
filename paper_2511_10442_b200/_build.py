"""Build the sm_100a CUDA library in-tree (no JIT cache, no pip install).

``python -m paper_2511_10442_b200._build`` or ``__graft_entry__.build()``
compiles ``csrc/*.cu`` with nvcc into ``paper_2511_10442_b200/libfastgraph_b200.so``
(C ABI declared in ``include/fastgraph_b200.h``).  The .so is git-ignored but
travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_NAME = "libfastgraph_b200.so"
LIB_PATH = os.path.join(PKG, LIB_NAME)
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def needs_rebuild() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(ROOT, "include", "fastgraph_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile csrc/*.cu; ``defines``/``out`` build an experimental variant."""
    target = out or LIB_PATH
    if not force and not defines and out is None and not needs_rebuild():
        return LIB_PATH
    objs = []
    tmp = os.path.join(PKG, "build" if not defines else "build_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(tmp, exist_ok=True)
    procs = []
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    hdrs.append(os.path.join(ROOT, "include", "fastgraph_b200.h"))
    t_hdr = max(os.path.getmtime(h) for h in hdrs)
    for src in sources():
        obj = os.path.join(tmp, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        # incremental (not force): an object newer than its source and every header is reused
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), t_hdr)):
            continue
        cmd = [nvcc(), ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               *(["-Xptxas", "-v"] if verbose else []),
               *["-D" + d for d in defines],
               "-I" + os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp_lib = target + ".tmp"
    subprocess.run([nvcc(), ARCH, "-shared", "-o", tmp_lib, *objs], check=True)
    os.replace(tmp_lib, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
