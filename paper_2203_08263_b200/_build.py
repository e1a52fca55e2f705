"""In-tree build of libnbody_b200.so for sm_100a (nvcc, no JIT cache).

The shared library lands next to this file so it travels with the repository
snapshot to the GPU box; ``_native`` loads it from there.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libnbody_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-I", os.path.join(REPO, "include"), "-I", CSRC]
SOURCES = ["nbody_force.cu", "nbody_update.cu", "nbody_capi.cu"]


def source_files() -> list:
    """Every file the library is compiled from (sorted)."""
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    files.append(os.path.join(REPO, "include", "nbody_b200.h"))
    return sorted(files)


def source_digest() -> str:
    """First 16 hex digits of SHA-256 over (relative path, content) of the
    sources; compiled into nb_version() and checked by _native.verify_build."""
    import hashlib
    h = hashlib.sha256()
    for f in source_files():
        h.update(os.path.relpath(f, REPO).encode() + b"\0")
        with open(f, "rb") as fh:
            h.update(fh.read())
        h.update(b"\0")
    return h.hexdigest()[:16]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), lib: str = LIB, objdir: str = OBJ) -> str:
    """Compile the sources for sm_100a and link ``lib``; ``defines`` (e.g.
    ["NB_CHECK"]) produce a variant build in its own ``objdir``."""
    OBJ_ = objdir
    os.makedirs(OBJ_, exist_ok=True)
    digest = source_digest()
    stamp = os.path.join(OBJ_, "digest.txt")
    try:
        with open(stamp) as f:
            built_from = f.read().strip()
    except OSError:
        built_from = None
    # the digest is compiled into every object: a source change anywhere rebuilds all
    spec = digest + " " + " ".join(defines)
    if built_from != spec:
        force = True
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(REPO, "include", "nbody_b200.h"))
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ_, src.replace(".cu", ".o"))
        if force or _stale(o, [s] + headers):
            dflags = [f"-D{d}" for d in defines] + [f'-DNB_SRC_DIGEST="{digest}"']
            cmd = [NVCC, *ARCH, *FLAGS, *dflags, "-Xptxas", "-v", "-c", s, "-o", o] if verbose else \
                  [NVCC, *ARCH, *FLAGS, *dflags, "-c", s, "-o", o]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for log in ex.map(run, jobs):
            if verbose and log:
                sys.stderr.write(log)
    objs = [os.path.join(OBJ_, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _stale(lib, objs):
        link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-ldl"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}\n{r.stderr}")
    with open(stamp, "w") as f:
        f.write(spec + "\n")
    if lib == LIB:
        build_hostpath(force)
    return lib


def build_hostpath(force: bool = False) -> str:
    """The CPython binding of simulate()'s single-GPU path (csrc/hostpath.c,
    gcc against this interpreter's headers), next to the package."""
    import sysconfig
    src = os.path.join(CSRC, "hostpath.c")
    out = os.path.join(PKG, "_hostpath" + sysconfig.get_config_var("EXT_SUFFIX"))
    if force or _stale(out, [src]):
        cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-Wall", "-I", sysconfig.get_paths()["include"],
               src, "-o", out]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"gcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return out


def build_checked() -> str:
    """Bounds-checked build (NB_CHECK: device traps on any out-of-range index)."""
    return build(defines=("NB_CHECK",), lib=os.path.join(PKG, "libnbody_b200_check.so"),
                 objdir=os.path.join(PKG, "build_check"))


if __name__ == "__main__":
    if "--check" in sys.argv:
        print(build_checked())
    else:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
