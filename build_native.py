"""Native build for the repo: the product library and the test infrastructure.

* ``build_leyenda()`` — ``paper_1909_08006_b200/libleyenda.so`` from ``paper_1909_08006_b200/csrc``
  (nvcc, ``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``), linked against NCCL from the
  torch-bundled wheel. This is the product.
* ``build_oracle()`` — ``oracle/liboracle.so`` (g++ -O2 -fopenmp). Test infrastructure.
* ``build_gen_host()`` / ``build_gen_cuda()`` — the seeded input generator and its CUDA twin.

Everything is built in-tree so the ``.so`` files travel to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1909_08006_b200")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as _n  # type: ignore

        base = list(_n.__path__)[0]
    except Exception:  # pragma: no cover
        base = os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                            "site-packages", "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _run(cmd, cwd=ROOT):
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} (exit {r.returncode})")
    return r


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_oracle(force=False):
    src = os.path.join(ROOT, "oracle", "oracle.cpp")
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, [src]):
        _run(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-o", out + ".tmp", src])
        os.replace(out + ".tmp", out)
    return out


def build_gen_host(force=False):
    srcs = [os.path.join(ROOT, "gen", f) for f in ("gen.cpp", "gen_core.h")]
    out = os.path.join(ROOT, "gen", "libleygen_host.so")
    if force or _stale(out, srcs):
        _run(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-o", out + ".tmp", srcs[0]])
        os.replace(out + ".tmp", out)
    return out


def build_gen_cuda(force=False):
    srcs = [os.path.join(ROOT, "gen", f) for f in ("gen_cuda.cu", "gen.cpp", "gen_core.h")]
    out = os.path.join(ROOT, "gen", "libleygen_cuda.so")
    if force or _stale(out, srcs):
        _run([NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp", "-shared", "-o", out + ".tmp",
              srcs[0], srcs[1], "-lgomp"])
        os.replace(out + ".tmp", out)
    return out


def leyenda_sources():
    csrc = os.path.join(PKG, "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cpp")))
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.h")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))
    return srcs, hdrs


def build_leyenda(force=False, jobs=8):
    """Compile every CUDA/C++ source of the product into libleyenda.so (sm_100a)."""
    srcs, hdrs = leyenda_sources()
    out = os.path.join(PKG, "libleyenda.so")
    if not (force or _stale(out, srcs + hdrs)):
        return out
    nccl_inc, nccl_lib = _nccl_dirs()
    objdir = os.path.join(ROOT, "build", "leyenda")
    os.makedirs(objdir, exist_ok=True)
    common = ["-std=c++17", "-O3", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc"),
              "-I", nccl_inc]
    objs, procs = [], []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(o)
        if s.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", *common,
                   "-c", s, "-o", o]
        else:
            cmd = ["g++", "-fPIC", "-Wall", *common, "-I", os.path.join(CUDA_HOME, "include"), "-c", s, "-o", o]
        procs.append((cmd, subprocess.Popen(cmd, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
    failed = []
    for cmd, p in procs:
        txt = p.communicate()[0]
        if p.returncode != 0:
            failed.append((cmd, txt))
    if failed:
        for cmd, txt in failed:
            sys.stderr.write(" ".join(cmd) + "\n" + txt + "\n")
        raise RuntimeError("libleyenda build failed")
    nccl_so = os.path.join(nccl_lib, "libnccl.so.2")
    link = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out + ".tmp", *objs,
            "-L", nccl_lib, "-l:libnccl.so.2",
            "-Xlinker", f"-rpath,{nccl_lib}", "-Xlinker", f"-rpath,{os.path.join(CUDA_HOME, 'lib64')}"]
    _run(link)
    os.replace(out + ".tmp", out)
    return out


def build_all(force=False):
    build_oracle(force)
    build_gen_host(force)
    build_gen_cuda(force)
    build_leyenda(force)


def clean():
    for p in [os.path.join(ROOT, "build")]:
        shutil.rmtree(p, ignore_errors=True)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built")
