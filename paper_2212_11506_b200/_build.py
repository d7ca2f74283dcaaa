"""Build libbhtsne_b200.so in-tree with nvcc for sm_100a (no JIT cache)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(REPO, "include")
OBJ = os.path.join(REPO, "build", "obj")
LIB = os.path.join(HERE, "libbhtsne_b200.so")
SOURCES = ["abi.cu", "points.cu", "sort.cu", "tree.cu", "forces.cu", "engine.cu",
           "forces_f64.cu", "affinity.cu", "knn.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
         "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE,
         "-Xptxas", "-warn-spills"]


def _rpath():
    """Resolve libcudart.so.12 like torch does (venv wheel), else the toolkit."""
    dirs = ["/usr/local/cuda/lib64"]
    try:
        import nvidia.cuda_runtime as cr  # the wheel torch itself loads
        dirs.insert(0, os.path.join(list(cr.__path__)[0], "lib"))
    except Exception:
        pass
    return [f"-Xlinker=-rpath={d}" for d in dirs]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
               if f.endswith(".cuh")] + [os.path.join(INCLUDE, "bhtsne_b200.h")]
    objs, procs = [], []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [NVCC, *FLAGS, "-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                stderr=subprocess.STDOUT)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode()}")
        if verbose and out:
            print(out.decode(), file=sys.stderr)
    if force or _stale(LIB, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
               "-o", LIB, *objs, "-lcudart", *_rpath()]
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
