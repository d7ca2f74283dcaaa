"""Build an A/B variant of libbhtsne_b200.so (tuning aid, not the product).

    python tools/build_variant.py OUT.so [--src forces.cu=path] [-DNAME=V ...]

Compiles every source like _build.py, replacing any `--src name=path` file
and adding the -D defines, then links OUT.so.  Run the variant with
`BH_LIB=OUT.so python tools/microbench.py`.
"""

from __future__ import annotations

import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2212_11506_b200 import _build as B  # noqa: E402


def main(argv):
    out = os.path.abspath(argv[0])
    subs, defs = {}, []
    for a in argv[1:]:
        if a.startswith("--src="):
            name, path = a[len("--src="):].split("=", 1)
            subs[name] = os.path.abspath(path)
        elif a.startswith("-D"):
            defs.append(a)
    tag = os.path.splitext(os.path.basename(out))[0]
    odir = os.path.join(REPO, "build", "var", tag)
    os.makedirs(odir, exist_ok=True)
    objs, procs = [], []
    for src in B.SOURCES:
        path = subs.get(src, os.path.join(B.CSRC, src))
        obj = os.path.join(odir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [B.NVCC, *B.FLAGS, "-I" + B.CSRC, *defs, "-c", path, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT)))
    for src, p in procs:
        msg, _ = p.communicate()
        if p.returncode != 0:
            raise SystemExit(f"nvcc failed on {src}:\n{msg.decode()}")
        if b"spill" in msg:
            print(f"{src}: spills\n{msg.decode()}", file=sys.stderr)
    subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a",
                    "-shared", "-o", out, *objs, "-lcudart", *B._rpath()],
                   check=True)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1:])
