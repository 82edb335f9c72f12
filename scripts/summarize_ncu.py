"""Summarize an ncu --set full report into profiles/ (kernel -> key metrics)."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "launch__grid_size": "grid",
    "launch__occupancy_limit_registers": "occupancy_limit_registers",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "Kbyte/s": 1e3}


def main(rep, out, tag):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {}
    for r in data:
        parts = r[hdr.index("Kernel Name")].split("(")[0].split("::")
        name = "::".join(parts[-2:]) if len(parts) > 2 else parts[-1]  # e.g. dense::sim_kernel
        d = {}
        for k, short in WANT.items():
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    val = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    continue
                d[short] = val
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d["dram_write"]
        d["units_note"] = "bytes, seconds"
        d["source"] = tag
        base, n = name, 2
        while name in res:  # a second launch of the same kernel (e.g. the dense wave)
            name = f"{base}_{n}"
            n += 1
        res[name] = d
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1])
