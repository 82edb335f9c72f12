"""Command line (reference: pkg/src/frontier_sim/cli.py:155-365).

    python -m paper_2508_03148_b200.cli run <config> [--seed N] [--out DIR]
    python -m paper_2508_03148_b200.cli sweep <config> --grid <gridfile> [--out DIR]
    python -m paper_2508_03148_b200.cli validate-config <config>

Exit codes follow the reference: 0 success, 1 configuration problem,
2 runtime failure. Both run and sweep execute on the GPU engine.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys

from .config import ParseError, ValidationError, load_config
from .topology import TopologyError
from .workload import WorkloadError

CONFIG_ERRORS = (ParseError, ValidationError, TopologyError, WorkloadError, FileNotFoundError)


def write_run_artifacts(result: dict, out_dir: str) -> dict[str, str]:
    """trace.log (body + `#hash=` footer), metrics.json, summary.csv (cli.py:121-141)."""
    import csv
    import io
    from .metrics import SUMMARY_CSV_HEADER, summary_csv_row
    from .sweep import _atomic_write
    paths = {"trace": os.path.join(out_dir, "trace.log"),
             "metrics": os.path.join(out_dir, "metrics.json"),
             "summary": os.path.join(out_dir, "summary.csv")}
    trace = result["trace"]
    body = trace.body_bytes()
    _atomic_write(paths["trace"], body + f"#hash={trace.hash}\n".encode("utf-8"))
    doc = result["metrics"].to_dict()
    doc.update(config_hash=result["config_hash"], seed=result["config"].seed,
               mode=result["config"].mode)
    _atomic_write(paths["metrics"], (json.dumps(doc, sort_keys=True, indent=2) + "\n").encode("utf-8"))
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(SUMMARY_CSV_HEADER)
    w.writerow(summary_csv_row(result["metrics"], result["config_hash"]))
    _atomic_write(paths["summary"], buf.getvalue().encode("utf-8"))
    return paths


def cmd_run(args) -> int:
    from .api import run_one
    config = load_config(args.config)
    if args.seed is not None:
        wl = config.workload
        if wl is not None and wl.seed == config.seed:
            wl = dataclasses.replace(wl, seed=args.seed)
        config = dataclasses.replace(config, seed=args.seed, workload=wl)
    out_dir = args.out or config.output_dir
    result = run_one(config)
    write_run_artifacts(result, out_dir)
    s = result["metrics"].workload_summary
    print("batch_size,avg_input,output,throughput_tokens_per_s_per_gpu")
    print(f"{s['batch_size']},{s['avg_input_tokens']:g},{s['avg_output_tokens']:g},"
          f"{s['throughput_tokens_per_s_per_gpu']:.3f}")
    return 0


def cmd_sweep(args) -> int:
    from .sweep import cmd_sweep as run
    return run(args.config, args.grid, args.out)


def cmd_validate(args) -> int:
    config = load_config(args.config)
    print(f"ok: {config.mode} deployment, hash {config.config_hash()}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="frontier-b200")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("run")
    p.add_argument("config")
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--out", default=None)
    p.set_defaults(func=cmd_run)
    p = sub.add_parser("sweep")
    p.add_argument("config")
    p.add_argument("--grid", required=True)
    p.add_argument("--out", default=None)
    p.set_defaults(func=cmd_sweep)
    p = sub.add_parser("validate-config")
    p.add_argument("config")
    p.set_defaults(func=cmd_validate)
    args = ap.parse_args(argv)
    try:
        return args.func(args)
    except CONFIG_ERRORS as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except Exception as exc:  # runtime failures
        print(f"runtime error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
