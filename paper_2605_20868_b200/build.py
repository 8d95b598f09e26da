"""In-tree build of libcertkv_b200.so for sm_100a (nvcc, no JIT cache).

Every ``csrc/*.cu`` is compiled to an object in parallel (the kernels of one
file never call device code of another), then the objects are linked into the
shared library next to this file."""

import glob
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libcertkv_b200.so")
OBJ = os.path.join(HERE, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + \
        [os.path.join(ROOT, "include", "certkv_b200.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    import fcntl
    # one builder at a time (e.g. every rank of a torchrun job calling build())
    with open(LIB + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not needs_build():  # another process built it meanwhile
            return LIB
        nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
        extra = os.environ.get("CKV_NVCC_EXTRA", "").split()  # experiments only (e.g. -DPA_MINB=4)
        os.makedirs(OBJ, exist_ok=True)
        tag = os.getpid()

        def compile_one(src):
            obj = os.path.join(OBJ, os.path.basename(src)[:-3] + f".{tag}.o")
            cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", src,
                   "-o", obj]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
            return obj

        with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            objs = list(ex.map(compile_one, sources()))
        tmp = f"{LIB}.{tag}.tmp"
        subprocess.run([nvcc, *ARCH, "-shared", *objs, "-o", tmp], check=True)
        for o in objs:
            os.remove(o)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
