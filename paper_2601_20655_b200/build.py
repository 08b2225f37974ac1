"""Build the in-tree C-ABI library libb200ring.so for sm_100a with nvcc."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libb200ring.so")
SOURCES = ["host.cu", "put.cu", "get.cu", "clock.cu", "stage.cu", "fanin.cu"]
HEADERS = ["ring_internal.h", "ring_copy.cuh"] + [os.path.join("..", "..", "include", h) for h in ("b200ring.h", "b200ring_layout.cuh", "b200ring_device.cuh")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-cudart", "static", "--expt-relaxed-constexpr"]


STAMP = LIB + ".flags"


def _extra() -> list:
    return os.environ.get("B200RING_NVCC_DEFINES", "").split()   # experiments only


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    # a library built with other experiment defines is stale too
    try:
        with open(STAMP) as f:
            if f.read() != " ".join(_extra()):
                return True
    except OSError:
        if _extra():
            return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        extra = _extra()
        cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
        objs.append(obj)
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, check=True), cmds):
            pass
    tmp = LIB + ".tmp"
    subprocess.run([NVCC, "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
                    *objs, "-Xlinker", "--no-undefined", "-o", tmp], check=True)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(" ".join(_extra()))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
