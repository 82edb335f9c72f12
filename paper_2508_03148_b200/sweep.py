"""Design-space sweeps on the GPU (reference: pkg/src/frontier_sim/cli.py:167-275).

Same semantics as `frontier-sim sweep`: the grid is the cartesian product of
its dotted-key value lists (keys sorted), every point gets the seed
`sha256(f"{master}:{canonical overrides}")[:4]` (a workload seed that merely
mirrored the master seed follows it), point failures become
`failed: {Type}: {msg}` rows, and the Pareto frontier (throughput up, p90 TPOT
down) is written next to `sweep.csv`. Differences:

* all points are simulated in ONE batched engine call (`api.simulate_rows`), not
  a thread pool of per-point Python runs (which the GIL serialises);
  the CSV and frontier need only each point's fixed-size metric row;
* dotted keys may index lists: `clusters.0.parallelism.tp` addresses the first
  cluster (the reference replaces the list with a dict and the point fails to
  parse); `clusters.1.num_replicas` etc.; an override that cannot
  be applied fails its point only;
* with torch.distributed initialised (world > 1, e.g. under torchrun), points are
  LPT-sharded across ranks by `api.config_cost`, each rank simulates its shard on
  its own GPU, the metric rows are all-gathered (NCCL) and rank 0 writes the files.
"""

from __future__ import annotations

import copy
import csv
import hashlib
import io
import json
import os
import tempfile

from .api import Failure, process_group, simulate_rows
from .config import DeploymentConfig, ParseError, load_config
from .metrics import SUMMARY_CSV_HEADER, pareto_frontier, summary_csv_row


def grid_points(grid: dict[str, list]) -> list[dict]:
    points: list[dict] = [{}]
    for key in sorted(grid):
        values = grid[key]
        if not isinstance(values, list) or not values:
            raise ParseError(f"grid.{key}: expected a non-empty array")
        points = [dict(p, **{key: v}) for p in points for v in values]
    return points


def apply_overrides(document: dict, overrides: dict) -> dict:
    """Deep-copy `document` and set each dotted key; integer parts index lists."""
    doc = copy.deepcopy(document)
    for dotted, value in overrides.items():
        parts = dotted.split(".")
        node = doc
        for part in parts[:-1]:
            if isinstance(node, list) and part.isdigit() and int(part) < len(node):
                node = node[int(part)]
                continue
            if not isinstance(node, dict):
                raise ParseError(f"override {dotted!r}: {part!r} does not address an object")
            if part not in node or not isinstance(node[part], (dict, list)):
                node[part] = {}
            node = node[part]
        last = parts[-1]
        if isinstance(node, list) and last.isdigit() and int(last) < len(node):
            node[int(last)] = value
        elif isinstance(node, dict):
            node[last] = value
        else:
            raise ParseError(f"override {dotted!r}: cannot set {last!r}")
    return doc


def point_seed(master_seed: int, overrides: dict) -> int:
    canonical = json.dumps(overrides, sort_keys=True, separators=(",", ":"))
    digest = hashlib.sha256(f"{master_seed}:{canonical}".encode("utf-8")).digest()
    return int.from_bytes(digest[:4], "big")


def point_documents(document: dict, points: list[dict], master_seed: int) -> list:
    """One config document per point, or a Failure for a point whose overrides
    cannot be applied (the reference records it as a failed row)."""
    docs: list = []
    for ov in points:
        try:
            d = apply_overrides(document, ov)
        except Exception as exc:
            docs.append(Failure(exc))
            continue
        d["seed"] = point_seed(master_seed, ov)
        wl = d.get("workload", {})
        if wl.get("seed") == master_seed:
            del wl["seed"]
        docs.append(d)
    return docs


def _atomic_write(path: str, data: bytes) -> None:
    directory = os.path.dirname(path) or "."
    os.makedirs(directory, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".tmp-")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def run_sweep(config: DeploymentConfig, grid: dict, out_dir: str, base_dir: str = ".",
              engine=None, distributed: bool | None = None) -> dict:
    """Simulate every grid point; write sweep.csv and frontier.json to out_dir
    (rank 0 only when sharded over ranks)."""
    document = config.to_document()
    points = grid_points(grid)
    docs = point_documents(document, points, config.seed)
    sr = simulate_rows(docs, engine=engine, base_dir=base_dir, distributed=distributed)
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(["point", "overrides", "status"] + SUMMARY_CSV_HEADER)
    ok = []
    for idx, ov in enumerate(points):
        ov_json = json.dumps(ov, sort_keys=True)
        if idx in sr.failed:
            w.writerow([idx, ov_json, f"failed: {sr.failed[idx]}"] + [""] * len(SUMMARY_CSV_HEADER))
        else:
            b = sr.bundle(idx)
            w.writerow([idx, ov_json, "ok"] + summary_csv_row(b, sr.config_hash[idx]))
            ok.append((idx, b))
    dist = process_group(distributed)
    if dist is not None and dist.get_rank() != 0:
        front = pareto_frontier(ok)
        return {"points": len(points), "ok": len(ok), "frontier": len(front)}
    _atomic_write(os.path.join(out_dir, "sweep.csv"), buf.getvalue().encode("utf-8"))
    front = pareto_frontier(ok)
    front_doc = [{"point": idx, "overrides": points[idx],
                  "throughput_tokens_per_s_per_gpu": b.throughput_tokens_per_s_per_gpu,
                  "tpot_p90_s": b.tpot["p90"] if b.tpot else None} for idx, b in front]
    _atomic_write(os.path.join(out_dir, "frontier.json"),
                  (json.dumps(front_doc, sort_keys=True, indent=2) + "\n").encode("utf-8"))
    return {"points": len(points), "ok": len(ok), "frontier": len(front_doc)}


def cmd_sweep(config_path: str, grid_path: str, out: str | None = None, engine=None) -> int:
    config = load_config(config_path)
    base_dir = os.path.dirname(os.path.abspath(config_path))
    with open(grid_path, encoding="utf-8") as fh:
        grid_doc = json.load(fh)
    grid = grid_doc.get("grid")
    if not isinstance(grid, dict) or not grid:
        raise ParseError(f"{grid_path}: expected an object with a 'grid' mapping")
    summary = run_sweep(config, grid, out or config.output_dir, base_dir, engine)
    print(f"sweep: {summary['ok']}/{summary['points']} points succeeded, "
          f"{summary['frontier']} on the frontier")
    return 0 if summary["ok"] else 2
