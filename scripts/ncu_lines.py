"""Per-source-line warp-stall samples and executed instructions from an ncu report.

usage: python scripts/ncu_lines.py REPORT.ncu-rep [top_n] [kernel_regex]
Needs a capture made with --import-source on and a -lineinfo build.
"""
import csv
import io
import subprocess
import sys


def main(rep, top=25, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["--kernel-name-base", "demangled", "-k", f"regex:{kernel}"]
    txt = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    agg, cur_file, cur_line, cur_src, hdr = {}, None, None, "", None
    for row in csv.reader(io.StringIO(txt)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) < 8:
            continue
        if row[0]:
            cur_line, cur_src = row[0], row[1]
            continue
        num = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
        samples, inst = num(row[4]), num(row[7])
        k = (cur_file, cur_line)
        a = agg.setdefault(k, [0.0, 0.0, cur_src])
        a[0] += samples
        a[1] += inst
    ts = sum(v[0] for v in agg.values()) or 1.0
    ti = sum(v[1] for v in agg.values()) or 1.0
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{s / ts:6.1%} {i / ti:6.1%}  {f}:{ln}  {src.strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         sys.argv[3] if len(sys.argv) > 3 else None)
