"""Markdown summary of an `ncu --set full --import-source on` capture (profiles/).

usage: python scripts/ncu_report_md.py REPORT.ncu-rep OUT.md [title]

Sections: per-kernel headline metrics (duration, DRAM bytes, registers,
occupancy, issue activity), the warp-stall breakdown, and the source lines with
the most stall samples (needs a -lineinfo build).
"""
import csv
import io
import subprocess
import sys

HEAD = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("launch__registers_per_thread", "registers"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("smsp__inst_executed.sum", "warp instructions"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
        ("sass__inst_executed_local_loads", "local loads"),
        ("sass__inst_executed_local_stores", "local stores")]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main(rep, out, title=None):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# {title or rep}", "", f"Source: `{rep}` (ncu --set full, --clock-control none).", ""]
    for r in data:
        kname = r[hdr.index("Kernel Name")].split("(")[0]
        lines += [f"## {kname}", "", "| metric | value |", "|---|---|"]
        for key, label in HEAD:
            if key in hdr:
                lines.append(f"| {label} | {r[hdr.index(key)]} {units[hdr.index(key)]} |")
        st = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), k.split("stalled_")[1]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        lines += ["", "Warp-stall samples:", "", "| reason | share |", "|---|---|"]
        for v, k in sorted(st, reverse=True)[:10]:
            lines.append(f"| {k} | {v / tot:.1%} |")
        lines.append("")
        try:
            src = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kname.split('::')[-1]}")
        except subprocess.CalledProcessError:
            continue
        agg, cur, h2 = {}, None, None
        fname = "?"
        for row in csv.reader(io.StringIO(src)):
            if not row:
                continue
            if row[0] in ("File Name", "File Path"):
                fname = row[1].rsplit("/", 1)[-1]
                continue
            if row[0] == "Line No":
                h2 = row
                continue
            if h2 is None or len(row) < 8:
                continue
            if row[0]:
                cur = (fname, row[0], row[1].strip()[:70])
                continue
            try:
                smp = float(row[h2.index("Warp Stall Sampling (All Samples)")] or 0)
                ins = float(row[h2.index("Instructions Executed")] or 0)
            except ValueError:
                continue
            a = agg.setdefault(cur, [0.0, 0.0])
            a[0] += smp
            a[1] += ins
        ts = sum(v[0] for v in agg.values()) or 1.0
        ti = sum(v[1] for v in agg.values()) or 1.0
        lines += ["Hottest source lines (share of stall samples / of executed warp instructions):",
                  "", "| samples | instructions | line | source |", "|---|---|---|---|"]
        for (f, ln, code), (smp, ins) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]:
            code = code.replace("|", "\\|")
            lines.append(f"| {smp / ts:.1%} | {ins / ti:.1%} | {f}:{ln} | `{code}` |")
        lines.append("")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print(f"wrote {out}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
