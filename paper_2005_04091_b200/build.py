"""Build libspconv.so (all CUDA sources, sm_100a) in-tree with nvcc.

Each translation unit compiles to its own object in parallel (kernel_pipe.cu
dominates), then nvcc links the shared library.  ``defines`` / ``out`` build an
A/B variant of the same ABI (e.g. ``-DSPC_DISPATCH_VARIANT=1`` into
``ab/libspconv_v1.so``), loaded through ``SPCONV_LIB``.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libspconv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "--expt-relaxed-constexpr", "-Xcompiler", "-Wall"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = (sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.inc"))
            + glob.glob(os.path.join(CSRC, "*.py")) + glob.glob(os.path.join(INCLUDE, "*.h")))
    return any(os.path.getmtime(d) > t for d in deps)


def generate() -> None:
    """Regenerate the inline-PTX dispatcher include when its generator changed."""
    for inc_name, gen_name in (("dispatch_gen.inc", "gen_dispatch.py"), ("dispatch2_gen.inc", "gen_dispatch2.py")):
        inc = os.path.join(CSRC, inc_name)
        gen = os.path.join(CSRC, gen_name)
        if not os.path.exists(inc) or os.path.getmtime(inc) < os.path.getmtime(gen):
            subprocess.check_call([sys.executable, gen, inc])


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    generate()
    lib = out or LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tag = f"{os.getpid()}_{abs(hash((lib,) + tuple(defines))) % 10**8}"
    objdir = os.path.join(os.path.dirname(lib), f".obj_{tag}")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src: str):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *CFLAGS, *defines, "-I", INCLUDE, "-I", CSRC, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, sources()))
    log = []
    for src, obj, r in results:
        log.append(f"== {os.path.basename(src)}\n{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed compiling {src}")
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *[o for _, o, _ in results], "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libspconv.so")
    for _, o, _ in results:
        os.remove(o)
    os.rmdir(objdir)
    if verbose:
        sys.stderr.write("".join(log))
    if out is None:
        with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
            f.write("".join(log))
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    outp = None
    defs = tuple(a for a in args if a.startswith("-D"))
    for a in args:
        if a.startswith("--out="):
            outp = os.path.abspath(a.split("=", 1)[1])
    build(force="--force" in args, verbose="--verbose" in args, out=outp, defines=defs)
