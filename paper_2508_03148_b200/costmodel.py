"""Operator cost models: learned-model files and the batched GPU cost kernels.

Model files use the reference's portable format (reference:
pkg/src/frontier_sim/costmodel/model.py:140-182): a JSON document with
`format`, `schema`, `operator`, `trees[].nodes[]` and a sha256 `hash` over
the canonical body. `load_model_file` checks format, hash and schema exactly
as the reference does, then packs the trees into flat node arrays
(`ForestSet`) that the engine stages in HBM. Inference itself (feature
vectors, tree walks, the sorted-leaf mean) runs only on the device.
"""

from __future__ import annotations

import gzip
import hashlib
import json
from dataclasses import dataclass, field

import numpy as np

MODEL_FILE_FORMAT = "frontier-sim-operator-model"
SCHEMAS = {
    "attention_v1": 17,
    "grouped_gemm_v1": 12,
    "attention_sqrt_proxy_v1": 1,
}


from .errors import ModelFileError, SchemaMismatch  # noqa: E402,F401


def _document_hash(body: dict) -> str:
    canonical = json.dumps({k: v for k, v in body.items() if k != "hash"},
                           sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(canonical.encode("utf-8")).hexdigest()


@dataclass
class LearnedModel:
    """A loaded model file: operator, schema and the packed trees."""

    operator: str
    schema: str
    path: str
    n_trees: int
    tree_root: np.ndarray     # int64, local node index of each tree root (0 per tree + offset)
    feature: np.ndarray       # int32, -1 = leaf
    threshold: np.ndarray     # float64
    left: np.ndarray          # int32, forest-local node index
    right: np.ndarray         # int32
    value: np.ndarray         # float64

    @property
    def n_features(self) -> int:
        return SCHEMAS[self.schema]


def load_model_file(path: str) -> LearnedModel:
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        doc = json.load(fh)
    return model_from_document(doc, path)


def as_learned_model(model) -> LearnedModel | None:
    """A LearnedModel from one of ours or from the reference's LearnedOperatorModel
    (its portable document, costmodel/model.py:140-152)."""
    if model is None or isinstance(model, LearnedModel):
        return model
    return model_from_document(model.to_document(), f"<{model.operator} model>")


def model_from_document(doc: dict, path: str = "<document>") -> LearnedModel:
    """Pack a model document (load_model_file's checks, model.py:169-182)."""
    if doc.get("format") != MODEL_FILE_FORMAT:
        raise ModelFileError(f"{path}: not a {MODEL_FILE_FORMAT} file")
    if doc.get("hash") != _document_hash(doc):
        raise ModelFileError(f"{path}: hash footer does not match document body")
    if doc["schema"] not in SCHEMAS:
        raise SchemaMismatch(f"{path}: unknown schema {doc['schema']!r}")
    feats, thrs, lefts, rights, vals, roots = [], [], [], [], [], []
    base = 0
    for tree in doc["trees"]:
        nodes = tree["nodes"]
        roots.append(base)
        for nd in nodes:
            if "value_us" in nd:
                feats.append(-1)
                thrs.append(0.0)
                lefts.append(-1)
                rights.append(-1)
                vals.append(float(nd["value_us"]))
            else:
                feats.append(int(nd["feature_index"]))
                thrs.append(float(nd["threshold"]))
                lefts.append(base + int(nd["left"]))
                rights.append(base + int(nd["right"]))
                vals.append(0.0)
        base += len(nodes)
    n_feat = SCHEMAS[doc["schema"]]
    feat = np.asarray(feats, dtype=np.int64)
    inner = feat >= 0
    kids = np.concatenate([np.asarray(lefts)[inner], np.asarray(rights)[inner]])
    if (feat[inner] >= n_feat).any() or (kids < 0).any() or (kids >= base).any():
        raise ModelFileError(f"{path}: node feature or child index out of range")
    return LearnedModel(
        operator=doc["operator"], schema=doc["schema"], path=path, n_trees=len(roots),
        tree_root=np.asarray(roots, dtype=np.int64), feature=np.asarray(feats, dtype=np.int32),
        threshold=np.asarray(thrs, dtype=np.float64), left=np.asarray(lefts, dtype=np.int32),
        right=np.asarray(rights, dtype=np.int32), value=np.asarray(vals, dtype=np.float64))


_CACHE: dict[tuple, LearnedModel] = {}


def load_model_cached(path: str) -> LearnedModel:
    """load_model_file, memoised on (path, size, mtime): a sweep's points share files."""
    import os
    st = os.stat(path)
    key = (os.path.abspath(path), st.st_size, st.st_mtime_ns)
    m = _CACHE.get(key)
    if m is None:
        m = _CACHE[key] = load_model_file(path)
    return m


def check_model_slots(attention_model: LearnedModel | None,
                      grouped_gemm_model: LearnedModel | None) -> None:
    """CostModel.__post_init__ (costmodel/model.py:305-309): operator per slot."""
    if attention_model is not None and attention_model.operator != "attention":
        raise SchemaMismatch("attention slot needs an attention-operator model")
    if grouped_gemm_model is not None and grouped_gemm_model.operator != "grouped_gemm":
        raise SchemaMismatch("grouped_gemm slot needs a grouped_gemm-operator model")


def check_model_slots_engine(attention_model: LearnedModel | None,
                             grouped_gemm_model: LearnedModel | None) -> None:
    """check_model_slots plus the engine's forest size limit."""
    if attention_model is None and grouped_gemm_model is None:
        return
    from .abi import MAX_FOREST_TREES
    from .errors import EngineCapacityError
    check_model_slots(attention_model, grouped_gemm_model)
    for m in (attention_model, grouped_gemm_model):
        if m is not None and m.n_trees > MAX_FOREST_TREES:
            raise EngineCapacityError(f"{m.path}: {m.n_trees} trees exceed {MAX_FOREST_TREES}")


def forest_slot(forests: "ForestSet", model: LearnedModel | None, schema: str) -> int:
    """fs_instance_desc.attn_forest / gg_forest: -1 analytic, -2 a model whose
    schema the slot rejects at its first prediction (model.py:315-327)."""
    if model is None:
        return -1
    if model.schema != schema:
        return -2
    return forests.add(model)


@dataclass
class ForestSet:
    """Several models concatenated for the engine (node indices made global)."""

    models: list[LearnedModel] = field(default_factory=list)

    def add(self, model: LearnedModel) -> int:
        for i, m in enumerate(self.models):
            if m is model:
                return i
        self.models.append(model)
        return len(self.models) - 1

    def arrays(self):
        from . import abi
        descs = np.zeros(len(self.models), dtype=abi.FOREST_DESC)
        roots, feat, thr, left, right, val = [], [], [], [], [], []
        node_base, tree_base = 0, 0
        for i, m in enumerate(self.models):
            descs[i] = (m.n_trees, m.n_features, tree_base)
            roots.append(m.tree_root + node_base)
            feat.append(m.feature)
            thr.append(m.threshold)
            left.append(np.where(m.left >= 0, m.left + node_base, -1).astype(np.int32))
            right.append(np.where(m.right >= 0, m.right + node_base, -1).astype(np.int32))
            val.append(m.value)
            node_base += len(m.feature)
            tree_base += m.n_trees
        cat = lambda xs, dt: np.ascontiguousarray(np.concatenate(xs).astype(dt))  # noqa: E731
        return (descs, cat(roots, np.int64), cat(feat, np.int32), cat(thr, np.float64),
                cat(left, np.int32), cat(right, np.int32), cat(val, np.float64))


def forest_set_struct(fs: ForestSet | None):
    """ctypes fs_forest_set over the arrays of `fs` (arrays kept alive on the struct)."""
    from . import abi
    c = abi.ForestSetC()
    if fs is None or not fs.models:
        return c
    arrs = fs.arrays()
    c._keep = arrs
    descs, roots, feat, thr, left, right, val = arrs
    c.forests, c.n_forests = abi.ptr(descs), len(descs)
    c.tree_root, c.n_trees = abi.ptr(roots), len(roots)
    c.feature, c.threshold = abi.ptr(feat), abi.ptr(thr)
    c.left, c.right, c.value = abi.ptr(left), abi.ptr(right), abi.ptr(val)
    c.n_nodes = len(feat)
    return c


# -- GPU entry points mirroring the reference's pure functions ---------------------------

def route_tokens_uniform(tokens, seeds, num_experts: int, top_k: int, engine=None):
    """route_tokens(T, E, k, "uniform", seed).counts for many calls (routing.py:65-113)."""
    from .engine import default_engine
    from .errors import STATUS_EXCEPTIONS
    eng = engine or default_engine()
    counts, st = eng.route_uniform(tokens, seeds, num_experts, top_k)
    bad = np.flatnonzero(st)
    if len(bad):
        raise STATUS_EXCEPTIONS.get(int(st[bad[0]]), RuntimeError)(f"call {int(bad[0])}")
    return counts


def attention_cost_batches(q_lens, kv_lens, offsets, is_decode, num_query_heads, num_kv_heads,
                           head_dim, hardware, dtype_bytes: int = 2, model: LearnedModel | None = None,
                           engine=None) -> np.ndarray:
    """CostModel.predict_attention over CSR batches (model.py:313-321): analytic
    roofline, or the learned forest when `model` is given."""
    from .engine import attn_params, default_engine
    eng = engine or default_engine()
    prm = attn_params(num_query_heads, num_kv_heads, head_dim, dtype_bytes, hardware.peak_flops,
                      hardware.mem_bw, hardware.kernel_overhead_us)
    if model is None:
        out, st = eng.attention_cost(q_lens, kv_lens, offsets, is_decode, prm)
        if (st != 0).any():
            raise ValueError(f"{int((st != 0).sum())} batches failed AttentionFeatures validation")
        return out
    if model.operator != "attention":
        raise SchemaMismatch("attention slot needs an attention-operator model")
    if model.schema != "attention_v1":
        raise SchemaMismatch(f"attention predictor uses schema {model.schema!r}; expected attention_v1")
    fs = ForestSet([model])
    out = eng.attention_forest(fs, 0, q_lens, kv_lens, offsets, is_decode, prm)
    if np.isnan(out).any():
        raise ValueError(f"{int(np.isnan(out).sum())} batches failed AttentionFeatures validation")
    return out
