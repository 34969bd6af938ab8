"""Multi-GPU sharding for the stitched path.

Every BASELINE config is independent along its batch (token-row) axis, and the
column-reduction config along its column axis, so N GPUs run N independent
shard graphs -- one process per GPU, each with its own plan (shapes change,
so plans are recomputed per shard and parity-checked per shard), its own
CUDA Graph, and no collective on the data path.  NCCL (torch.distributed over
NVLink) is used only after timing, to gather shard outputs on rank 0 for
verification against the full-graph oracle.

A ShardRule rewrites the graph text for one shard and maps full-graph
tensors to shard tensors (and back), so the gathered shard outputs equal the
full graph's outputs element for element.
"""
from __future__ import annotations

import re
from dataclasses import dataclass
from typing import Dict, List

import numpy as np


@dataclass(frozen=True)
class ShardRule:
    full: int               # extent of the sharded axis in the full graph
    token: str              # regex matching that extent inside shape annotations
    axis_of: Dict[str, int]  # tensor -> sharded axis (tensors absent are replicated)

    def shard_size(self, n: int) -> int:
        if self.full % n:
            raise ValueError("extent %d does not split into %d shards" % (self.full, n))
        return self.full // n

    def graph_text(self, text: str, n: int) -> str:
        return self.extent_text(text, self.shard_size(n))

    def extent_text(self, text: str, b: int) -> str:
        """the graph with the sharded axis set to extent b (any 1 <= b <= full)"""
        if not 1 <= b <= self.full:
            raise ValueError("extent %d outside [1, %d]" % (b, self.full))
        return re.sub(self.token, lambda m: m.group(0).replace(str(self.full), str(b)), text)

    def slice_inputs(self, inputs: Dict[str, np.ndarray], n: int, rank: int) -> Dict[str, np.ndarray]:
        b = self.shard_size(n)
        out = {}
        for name, a in inputs.items():
            ax = self.axis_of.get(name)
            if ax is None:
                out[name] = a
            else:
                idx = [slice(None)] * a.ndim
                idx[ax] = slice(rank * b, (rank + 1) * b)
                out[name] = np.ascontiguousarray(a[tuple(idx)])
        return out

    def concat_outputs(self, parts: List[Dict[str, np.ndarray]]) -> Dict[str, np.ndarray]:
        out = {}
        for name in parts[0]:
            ax = self.axis_of.get(name)
            out[name] = parts[0][name] if ax is None else np.concatenate([p[name] for p in parts], axis=ax)
        return out


# shape-token rules for the BASELINE config graphs (paper_2009_10924_b200/graphs)
RULES = {
    "attn_softmax": ShardRule(32, r"\[32,", {"x": 0, "mask": 0, "y": 0}),
    "ln_4096x768": ShardRule(4096, r"\[4096[,\]]", {"x": 0, "y": 0}),
    "ln2pass_4096x768": ShardRule(4096, r"\[4096[,\]]", {"x": 0, "y": 0}),
    "bert_gelu": ShardRule(4096, r"\[4096,", {"ffn1": 0, "gl": 0}),
    "bert_resln": ShardRule(4096, r"\[4096[,\]]", {"h": 0, "ffn2": 0, "y": 0}),
    "bert_cut": ShardRule(4096, r"\[4096[,\]]", {"h": 0, "ffn1": 0, "ffn2": 0, "gl": 0, "y": 0}),
    # DIEN AUGRU (batch 256): every per-step tensor is batch-leading.  Shape
    # rewriting only (CPU-baseline timing on host threads): the opaque
    # placeholders average over their whole operands, so shards are NOT
    # equivalent to the full graph -- no tensor mapping, no gather
    "dien_T10": ShardRule(256, r"\[256[,\]]", {}),
    "bert_layer": ShardRule(4096, r"\[4096[,\]]", {}),
    "dien_T20": ShardRule(256, r"\[256[,\]]", {}),
    # column reductions: shard the kept (column) axis; each GPU reduces all rows
    "colreduce": ShardRule(1024, r"1024\]", {"dy": 1, "xhat": 1, "dbias": 0, "dgamma": 0}),
}
