"""Per-source-line instruction and stall shares of one kernel in an ncu
report (tuning aid): maps the report's SASS rows to source lines through
nvdisasm -g of the locally built object (same sources, same nvcc).

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX OBJ.o MANGLED_SUBSTR SRC.cu [N]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, kregex, obj, mangled, src, top=30):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d,
                       check=True, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)],
                             capture_output=True, text=True).stdout.split("\n")
    st = [i for i, l in enumerate(dis) if l.startswith(".text.") and mangled in l][0]
    cur, seq = None, []
    for l in dis[st + 1:]:
        if l.startswith(".text.") or l.startswith("//-----"):
            if seq:
                break
        m = re.search(r"line (\d+)", l)
        if "//##" in l and m:
            cur = int(m.group(1))
        if re.search(r"/\*[0-9a-f]{4,}\*/", l) and ";" in l:
            seq.append(cur)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                          "--print-source", "sass", "-k", f"regex:{kregex}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_ex = hdr.index("Instructions Executed")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[i_ex] or 0), int(r[i_s] or 0)) for r in rows[2:]
            if len(r) > i_ex and (r[i_ex] or "0").isdigit()][:len(seq)]
    agg = {}
    for ln, (e, s) in zip(seq, data):
        a = agg.setdefault(ln, [0, 0])
        a[0] += e
        a[1] += s
    te = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    text = open(src).read().split("\n")
    print(f"sass {len(seq)} rows {len(data)}; instructions {te}, samples {ts}")
    for ln, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"L{ln} inst {e / te * 100:5.1f}% stall {s / ts * 100:5.1f}%  "
              f"{text[ln - 1].strip()[:80] if ln else ''}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(*a[:5], *(int(x) for x in a[5:6]))
