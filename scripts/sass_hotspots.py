"""Per-source-line warp-stall hotspots of one kernel from an ncu report.

usage: python scripts/sass_hotspots.py <report.ncu-rep> <lib.so> <kernel-substring> [top]
Joins `ncu --page source --print-source sass` samples with the line table of
`nvdisasm -g` on the cubin extracted from the library (build with -lineinfo).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, lib, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ai, si = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    cols = {c: hdr.index(c) for c in ("stall_long_sb", "stall_barrier", "stall_short_sb", "stall_lg",
                                      "stall_wait", "stall_membar")}
    samples = []
    for r in rows[2:]:
        try:
            samples.append((int(r[ai], 16), int(r[si] or 0), {c: int(r[i] or 0) for c, i in cols.items()}))
        except (ValueError, IndexError):
            pass
    base = samples[0][0]
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    sass = ""
    for f in os.listdir(d):
        t = subprocess.run(["nvdisasm", "-g", os.path.join(d, f)], capture_output=True, text=True).stdout
        if kname in t:
            sass = t
    lines = sass.split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kname in l)
    a2l, cur = {}, None
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith("\t.section") or l.startswith(".section"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            a2l[int(m.group(1), 16)] = cur
    agg, per = collections.Counter(), collections.defaultdict(collections.Counter)
    tot = 0
    for a, s, st in samples:
        k = a2l.get(a - base, ("?", 0))
        agg[k] += s
        tot += s
        for c, v in st.items():
            per[k][c] += v
    srcdir = os.path.join(os.path.dirname(os.path.abspath(lib)), "..", "csrc")
    cache = {}
    print(f"total samples {tot}")
    for k, v in agg.most_common(top):
        if k[0] not in cache:
            p = os.path.join(srcdir, k[0])
            cache[k[0]] = open(p).read().split("\n") if os.path.exists(p) else []
        txt = cache[k[0]][k[1] - 1].strip()[:70] if k[1] and len(cache[k[0]]) >= k[1] else ""
        st = " ".join(f"{c[6:]}={per[k][c] / tot * 100:.1f}" for c in ("stall_long_sb", "stall_barrier")
                      if per[k][c])
        print(f"{v / tot * 100:5.1f}% [{st}] {k[0]}:{k[1]}  {txt}")


if __name__ == "__main__":
    main()
