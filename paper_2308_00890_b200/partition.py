"""Destination-row partitioning of a graph across ranks.

Host-side only, no arithmetic of the method: rank r owns the contiguous node block
[starts[r], starts[r+1]) and holds the in-CSR rows (its destinations' in-edges)
and the out-CSR rows (its sources' out-edges, the reversed graph of ⑤′) of that
block, with GLOBAL node ids in the index arrays.  Edge tensors of the owned in-CSR rows are the
slice [in_ptr[rb], in_ptr[re]) of the global in-CSR edge order, so concatenating the ranks'
edge tensors in rank order gives the single-GPU edge order.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition_rows(g, nranks: int) -> list[int]:
    """Contiguous node ranges balanced by in-edges + one unit per row.  Returns nranks+1 starts."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    cum = g.in_ptr.astype(np.float64) + np.arange(g.n + 1)
    starts = [0]
    for r in range(1, nranks):
        starts.append(max(starts[-1], int(np.searchsorted(cum, cum[-1] * r / nranks))))
    starts.append(g.n)
    return starts


@dataclass
class LocalGraph:
    """One rank's block of a graph: rows [row_begin, row_end) of the in- and out-CSR."""
    n_global: int
    row_begin: int
    row_end: int
    in_ptr: np.ndarray    # int64 [n_local + 1], rebased to 0
    in_src: np.ndarray    # int32 [e_in], global source ids
    out_ptr: np.ndarray   # int64 [n_local + 1], rebased to 0
    out_dst: np.ndarray   # int32 [e_out], global destination ids
    out_eid: np.ndarray | None  # int32 [e_out] global in-CSR edge ids (only for the full graph)
    in_edge0: int         # global in-CSR id of this block's first in-edge

    @property
    def n(self) -> int:
        return self.row_end - self.row_begin

    @property
    def e(self) -> int:
        return int(self.in_src.shape[0])

    @property
    def e_out(self) -> int:
        return int(self.out_dst.shape[0])


def local_graph(g, row_begin: int = 0, row_end: int | None = None, keep_eid: bool | None = None) -> LocalGraph:
    """Slice rows [row_begin, row_end) of g (inputs.Graph).  out_eid is kept only when the block
    is the whole graph (a partitioned source pass cannot address other ranks' edge arrays),
    unless keep_eid forces it (tests)."""
    row_end = g.n if row_end is None else row_end
    if not (0 <= row_begin <= row_end <= g.n):
        raise ValueError(f"bad row range [{row_begin}, {row_end}) for n = {g.n}")
    ib, ie = int(g.in_ptr[row_begin]), int(g.in_ptr[row_end])
    ob, oe = int(g.out_ptr[row_begin]), int(g.out_ptr[row_end])
    full = row_begin == 0 and row_end == g.n
    keep = full if keep_eid is None else keep_eid
    return LocalGraph(
        n_global=g.n, row_begin=row_begin, row_end=row_end,
        in_ptr=np.ascontiguousarray(g.in_ptr[row_begin:row_end + 1] - ib, dtype=np.int64),
        in_src=np.ascontiguousarray(g.in_src[ib:ie], dtype=np.int32),
        out_ptr=np.ascontiguousarray(g.out_ptr[row_begin:row_end + 1] - ob, dtype=np.int64),
        out_dst=np.ascontiguousarray(g.out_dst[ob:oe], dtype=np.int32),
        out_eid=np.ascontiguousarray(g.out_eid[ob:oe], dtype=np.int32) if keep else None,
        in_edge0=ib)


def block_sizes(starts: list[int]) -> list[int]:
    return [starts[r + 1] - starts[r] for r in range(len(starts) - 1)]
