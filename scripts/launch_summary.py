"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import re
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        name = re.sub(r"\(.*", "", re.sub(r".*::", "", r[ki].split("(")[0] if "<" not in r[ki] else r[ki]))
        name = re.sub(r".*\)::", "", r[ki])
        name = re.sub(r"^(void )?", "", name)
        name = re.sub(r"\(ocmb.*", "", name)
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:32s} launches={c:5d} total_us={t / 1e3:9.1f} avg_us={t / c / 1e3:8.2f} share={t / tot:.3f}")
    return "\n".join(out) + f"\nTOTAL_us={tot / 1e3:.1f}"


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
