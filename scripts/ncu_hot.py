"""Per-source-line executed warp instructions, thread efficiency and stall samples
from an ncu --set full report (needs --import-source on and a -lineinfo build), plus
the totals per enclosing function.

usage: python scripts/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [top_n]
"""
import csv
import io
import re
import subprocess
import sys


def main(rep, kernel, top=40):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
           "--kernel-name-base", "demangled", "-k", f"regex:{kernel}"]
    txt = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    agg, srcs, cur_file = {}, {}, None
    for row in csv.reader(io.StringIO(txt)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Line No" or len(row) < 9:
            continue
        if row[0]:  # source line (aggregated over its SASS rows)
            try:
                ln = int(row[0])
                num = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
                vals = (num(row[4]), num(row[7]), num(row[8]))
            except ValueError:  # a source line whose quotes confuse the CSV
                continue
            srcs[(cur_file, ln)] = row[1]
            agg[(cur_file, ln)] = vals
    # enclosing function of each line: the last `__device__ ... name(` above it
    func_of, cur = {}, {}
    for (f, ln) in sorted(srcs):
        m = re.search(r"(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", srcs[(f, ln)])
        if m:
            cur[f] = m.group(1)
        func_of[(f, ln)] = cur.get(f, "?")
    ts = sum(v[0] for v in agg.values()) or 1.0
    ti = sum(v[1] for v in agg.values()) or 1.0
    print(f"total warp instructions {ti:.4g}, stall samples {ts:.0f}")
    print("\n-- by function (instructions, samples, thread efficiency) --")
    fa = {}
    for k, (s, i, t) in agg.items():
        a = fa.setdefault((k[0], func_of.get(k, "?")), [0, 0, 0])
        a[0] += s; a[1] += i; a[2] += t
    for (f, fn), (s, i, t) in sorted(fa.items(), key=lambda kv: -kv[1][1])[:30]:
        eff = t / (32 * i) if i else 0
        print(f"{i / ti:6.1%} {s / ts:6.1%}  eff {eff:4.2f}  {f}:{fn}")
    print("\n-- top lines by instructions --")
    for k, (s, i, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        eff = t / (32 * i) if i else 0
        print(f"{i / ti:6.1%} {s / ts:6.1%}  eff {eff:4.2f}  {k[0]}:{k[1]}  {srcs[k].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
