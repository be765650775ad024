"""Build the in-tree CUDA library liblorpc.so for sm_100a (nvcc, no torch types)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liblorpc.so")
SOURCES = ["basis.cpp", "mesh.cu", "operator.cu", "lor.cu", "schwarz.cu", "vcycle.cu", "vcycle_t.cu", "vcycle_w.cu", "single.cu", "pcg.cu", "dg.cu", "dist.cu", "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr"] + \
    os.environ.get("LORPC_NVCC_EXTRA", "").split()


def nccl_dir():
    """The NCCL torch loads (pip nvidia-nccl, 2.28.x in this image): headers and library
    for dist.cu, so the process holds one NCCL (SURVEY §7 hard part 10); None falls back
    to the system one."""
    try:
        import nvidia.nccl as nn
        for d in nn.__path__:
            if os.path.exists(os.path.join(d, "include", "nccl.h")) and \
                    os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
                return d
    except ImportError:
        pass
    return None


def build(force=False, verbose=False):
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in ("common.h", "device.cuh", "patch.cuh")] + \
        [os.path.join(HERE, "..", "include", "lorpc.h")]
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(p) for p in deps):
        return OUT
    nd = nccl_dir()
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in srcs:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if os.path.exists(obj) and not force and os.path.getmtime(obj) >= max(
                [os.path.getmtime(src)] + [os.path.getmtime(os.path.join(CSRC, h)) for h in ("common.h", "device.cuh", "patch.cuh")]
                + [os.path.getmtime(os.path.join(HERE, "..", "include", "lorpc.h"))]):
            continue
        cmd = [NVCC] + FLAGS + (["-I", os.path.join(nd, "include")] if nd else []) + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed on {src}")
        elif verbose and out.strip():
            print(out)
    if nd:
        link = ["-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    else:
        link = ["-lnccl"]
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT] + objs + ["-lcudart"] + link
    subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
