"""Build the in-tree native libraries (no JIT cache, no site-packages):

* paper_2012_09646_b200/libdagrt.so  -- scheduler core + sm_100a product kernels
* paper_2012_09646_b200/libdagrt_exp.so -- experimental kernel variants
  (csrc/exp/), loaded only on request (dagrt.load_experimental())
* synth/libsynth.so                  -- GPU twin of the seeded input generator

Every CUDA file is compiled with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo``; cudart is linked statically so the .so loads on a GPU-less box.
Usage: ``python -m paper_2012_09646_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _needs(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, obj, includes, extra=()):
    cmd = [nvcc()] + NVCC_FLAGS + list(extra) + [f"-I{i}" for i in includes] + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return r.stderr


def _lib(name, srcs, headers, includes, out, verbose=False, link=()):
    os.makedirs(BUILD, exist_ok=True)
    objs, jobs = [], []
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for s in srcs:
            o = os.path.join(BUILD, name + "_" + os.path.basename(s) + ".o")
            objs.append(o)
            if _needs(o, [s] + headers):
                jobs.append(ex.submit(_compile, s, o, includes))
        for j in jobs:
            msg = j.result()
            if verbose and msg.strip():
                print(msg, file=sys.stderr)
    if _needs(out, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-Xlinker",
                                 "-soname=" + os.path.basename(out), "-o", out] + objs + \
              list(link) + ["-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed for {out}:\n{r.stderr}")
    return out


def build(verbose=False):
    srcs = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "dagrt.h"))
    lib = _lib("dagrt", srcs, headers, [CSRC, os.path.join(ROOT, "include")],
               os.path.join(HERE, "libdagrt.so"), verbose)
    # experimental variants: their own library over libdagrt.so's registry
    edir = os.path.join(CSRC, "exp")
    esrcs = sorted(os.path.join(edir, f) for f in os.listdir(edir) if f.endswith(".cu"))
    eheaders = headers + [os.path.join(edir, f) for f in os.listdir(edir) if f.endswith(".cuh")]
    _lib("dagrt_exp", esrcs, eheaders, [CSRC, edir], os.path.join(HERE, "libdagrt_exp.so"), verbose,
         link=["-L" + HERE, "-ldagrt", "-Xlinker", "-rpath=$ORIGIN"])
    sdir = os.path.join(ROOT, "synth", "csrc")
    ssrcs = [os.path.join(sdir, f) for f in sorted(os.listdir(sdir)) if f.endswith(".cu")]
    slib = _lib("synth", ssrcs, [], [sdir], os.path.join(ROOT, "synth", "libsynth.so"), verbose)
    ext = build_fastcall(lib, verbose)
    return lib, slib, ext


def build_fastcall(lib, verbose=False):
    """CPython METH_FASTCALL module over libdagrt.so (pyext/dagrt_fastcall.c):
    the per-step calls of the Python binding without ctypes' marshalling."""
    import sysconfig
    src = os.path.join(HERE, "pyext", "dagrt_fastcall.c")
    out = os.path.join(HERE, "_dagrt_fastcall" + sysconfig.get_config_var("EXT_SUFFIX"))
    if not _needs(out, [src, lib, os.path.join(ROOT, "include", "dagrt.h")]):
        return out
    cmd = ["gcc", "-O2", "-shared", "-fPIC", f"-I{sysconfig.get_paths()['include']}",
           f"-I{os.path.join(ROOT, 'include')}", src, "-o", out, f"-L{HERE}", "-ldagrt",
           "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"gcc failed for {src}:\n{r.stderr}")
    return out


if __name__ == "__main__":
    print(build(verbose=True))
