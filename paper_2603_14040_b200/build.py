"""Compile libstokes_b200.so in-tree for sm_100a (nvcc; no torch extension machinery)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstokes_b200.so")
SOURCES = ["kernels.cu", "stream.cu", "gcr.cu", "aa.cu", "ras.cu", "driver.cu", "dist.cu", "markers.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    """NCCL headers + library of the torch-bundled nvidia-nccl wheel (same lib torch loads)."""
    try:
        import nvidia.nccl as n
        return os.path.dirname(n.__file__) if n.__file__ else list(n.__path__)[0]
    except Exception:
        return "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xcompiler", "-fvisibility=hidden",
         "-I", os.path.join(NCCL, "include")]
LIBS = ["-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "stokes.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, out=None, defs=()):
    """nvcc every source to an object in parallel (no cross-file device code), then link.
    out / defs: an experimental variant (-D knobs of csrc/, e.g. "RR_NS=4") built elsewhere."""
    out = out or LIB
    if out == LIB and not defs and not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    tag = "main" if out == LIB else os.path.splitext(os.path.basename(out))[0]
    odir = os.path.join(HERE, "..", "build", "obj_" + tag)
    os.makedirs(odir, exist_ok=True)
    dflags = [f"-D{d}" for d in defs]
    objs = [os.path.join(odir, s.replace(".cu", ".o")) for s in SOURCES]
    comp = [FL for FL in FLAGS if FL != "-shared"]

    def one(k):
        cmd = [NVCC, *comp, *dflags, "-c", "-o", objs[k], os.path.join(CSRC, SOURCES[k])]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd, cwd=CSRC)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(one, range(len(SOURCES))))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, *LIBS]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=CSRC)
    return out


if __name__ == "__main__":
    build(force=True, verbose=True)
