"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no quantization, no GEMM, no
softmax, no aggregation).  It only draws graphs and dense tensors and lays the
graph out as CSR, so that the CPU oracle (``oracle/``) and the CUDA path
(``paper_2308_00890_b200``) can be fed identical inputs while sharing no code.

Graph recipe:
  * Chung-Lu draws (power-law or lognormal expected degrees) with a random node
    relabelling, then graph augmentation as in PAPER.md §4.1: add the
    reverse of every edge and one self-loop per node; duplicates removed.
  * In-CSR: rows = destination, sources ascending  (edge ids = in-CSR positions).
  * Out-CSR: rows = source, destinations ascending, with ``out_eid`` = position
    of each out-edge in the in-CSR (DS3/DS4 of SURVEY.md §2.3).

Seeds: graph 0, features 1, params 2, gradients 3, relabel 4.
"""
from __future__ import annotations

import dataclasses
import numpy as np

SEED_GRAPH, SEED_FEAT, SEED_PARAM, SEED_GRAD, SEED_RELABEL = 0, 1, 2, 3, 4
SR_SEED = 0x7A4E60  # stochastic-rounding key, SURVEY.md §8(d)


@dataclasses.dataclass
class Graph:
    """A directed graph in in-CSR + out-CSR form (global node ids)."""
    n: int
    in_ptr: np.ndarray    # int64 [n+1]
    in_src: np.ndarray    # int32 [e]   (sorted by dst, then src)
    out_ptr: np.ndarray   # int64 [n+1]
    out_dst: np.ndarray   # int32 [e]   (sorted by src, then dst)
    out_eid: np.ndarray   # int32 [e]   position of each out-edge in the in-CSR

    @property
    def e(self) -> int:
        return int(self.in_src.shape[0])

    def in_dst(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int32), np.diff(self.in_ptr))

    def degree_stats(self) -> dict:
        d = np.diff(self.in_ptr)
        if d.size == 0:
            return {"max": 0, "mean": 0.0, "p99": 0.0}
        return {"max": int(d.max()), "mean": float(d.mean()), "p99": float(np.percentile(d, 99))}


def build_csr(n: int, src: np.ndarray, dst: np.ndarray) -> Graph:
    """Lay out a list of unique directed edges (src -> dst) as in-CSR + out-CSR."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    order = np.argsort(dst * n + src, kind="stable")
    in_src = src[order]
    in_dst = dst[order]
    in_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(in_dst, minlength=n), out=in_ptr[1:])
    order2 = np.argsort(in_src * n + in_dst, kind="stable")
    out_dst = in_dst[order2]
    out_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(in_src, minlength=n), out=out_ptr[1:])
    return Graph(n=n, in_ptr=in_ptr, in_src=in_src.astype(np.int32),
                 out_ptr=out_ptr, out_dst=out_dst.astype(np.int32),
                 out_eid=order2.astype(np.int32))


def augment(n: int, src: np.ndarray, dst: np.ndarray, self_loops: bool = True):
    """PAPER.md §4.1: add reverse edges and self-loops; drop duplicates."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    keep = src != dst
    s = np.concatenate([src[keep], dst[keep]])
    d = np.concatenate([dst[keep], src[keep]])
    if self_loops:
        loop = np.arange(n, dtype=np.int64)
        s = np.concatenate([s, loop])
        d = np.concatenate([d, loop])
    key = np.unique(d * n + s)
    return key % n, key // n


def _chung_lu_pairs(n, m, weights, rng):
    cdf = np.cumsum(weights / weights.sum())
    cdf[-1] = 1.0
    a = np.searchsorted(cdf, rng.random(m), side="right")
    b = np.searchsorted(cdf, rng.random(m), side="right")
    return np.minimum(a, n - 1), np.minimum(b, n - 1)


def _clip_weights(w, m, dmax):
    """Cap expected degree 2m*w/sum(w) at dmax (fixed-point on the cap)."""
    w = w.astype(np.float64).copy()
    for _ in range(20):
        cap = dmax * w.sum() / (2.0 * m)
        if w.max() <= cap * (1 + 1e-9):
            break
        w = np.minimum(w, cap)
    return w


def chung_lu_graph(n: int, m: int, gamma: float | None = None, *, lognormal_sigma: float | None = None,
                   dmax: int | None = None, seed: int = SEED_GRAPH, relabel_seed: int = SEED_RELABEL,
                   self_loops: bool = True) -> Graph:
    """Power-law (gamma) or lognormal Chung-Lu graph with m undirected draws, augmented."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if lognormal_sigma is not None:
        w = rng.lognormal(0.0, lognormal_sigma, size=n)
    else:
        i = np.arange(n, dtype=np.float64)
        w = (i + 1.0) ** (-1.0 / (gamma - 1.0))
    if dmax is not None:
        w = _clip_weights(w, m, dmax)
    perm = np.random.Generator(np.random.PCG64(relabel_seed)).permutation(n)
    w = w[perm]
    a, b = _chung_lu_pairs(n, m, w, rng)
    s, d = augment(n, a, b, self_loops=self_loops)
    return build_csr(n, s, d)


def random_graph(n: int, draws: int, seed: int = SEED_GRAPH, self_loops: bool = True) -> Graph:
    """Small Chung-Lu graph for parity cases (config C0b): draws directed pairs, augmented."""
    return chung_lu_graph(n, draws, gamma=2.5, seed=seed, relabel_seed=seed + 100, self_loops=self_loops)


def toy_graph() -> Graph:
    """The paper's running example (§2.1 Fig.1).

    e0: v1->v0, e1: v3->v1 (reading A19), e2: v1->v2, e3: v0->v3, e4: v2->v3.
    No self-loops. Edge ids equal in-CSR positions.
    """
    src = np.array([1, 3, 1, 0, 2])
    dst = np.array([0, 1, 2, 3, 3])
    return build_csr(4, src, dst)


# ----------------------------------------------------------------------------------------------
# Named workloads (BASELINE.json configs; shapes per SURVEY.md §8 table and readings A16/A18)
# ----------------------------------------------------------------------------------------------
WORKLOADS = {
    # name: (graph kwargs, F, H, D)
    "c0b": (dict(n=64, m=256, gamma=2.5), 16, 2, 8),
    "cora": (dict(n=2708, m=5278, gamma=2.5, dmax=168), 1433, 1, 128),
    "arxiv": (dict(n=169_343, m=1_166_243, gamma=2.1, dmax=13_000), 128, 4, 128),
    "reddit": (dict(n=232_965, m=57_307_946, lognormal_sigma=1.0, dmax=21_000), 602, 4, 128),
    "products": (dict(n=2_449_029, m=61_859_140, gamma=2.1, dmax=17_500), 100, 4, 128),
}


def workload_graph(name: str, order: str = "random") -> Graph:
    """order "random": the seeded random relabelling of the recipe; "degree": the same graph with
    nodes renumbered by descending in-degree (a locality relabelling)."""
    kw, _, _, _ = WORKLOADS[name]
    g = chung_lu_graph(**kw)
    return relabel_by_degree(g) if order == "degree" else g


def relabel_by_degree(g: Graph) -> Graph:
    """Renumber nodes by descending in-degree (stable), keeping the edge set."""
    deg = np.diff(g.in_ptr)
    perm = np.argsort(-deg, kind="stable")          # new id i <- old id perm[i]
    new_of = np.empty(g.n, dtype=np.int64)
    new_of[perm] = np.arange(g.n, dtype=np.int64)
    src = new_of[g.in_src.astype(np.int64)]
    dst = new_of[g.in_dst().astype(np.int64)]
    return build_csr(g.n, src, dst)


def features(n: int, f: int, seed: int = SEED_FEAT) -> np.ndarray:
    """Node features H ~ N(0,1), float32 [n][f]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((n, f), dtype=np.float32)


def gat_params(f: int, heads: int, head_dim: int, seed: int = SEED_PARAM):
    """Glorot-uniform W [f][H*D], a_src [H*D], a_dst [H*D] (float32)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    hd = heads * head_dim
    lim = np.sqrt(6.0 / (f + hd))
    W = rng.uniform(-lim, lim, size=(f, hd)).astype(np.float32)
    lim_a = np.sqrt(6.0 / (head_dim + 1))
    a_src = rng.uniform(-lim_a, lim_a, size=hd).astype(np.float32)
    a_dst = rng.uniform(-lim_a, lim_a, size=hd).astype(np.float32)
    return W, a_src, a_dst


def gcn_params(f: int, out: int, seed: int = SEED_PARAM) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    lim = np.sqrt(6.0 / (f + out))
    return rng.uniform(-lim, lim, size=(f, out)).astype(np.float32)


def grad_out(n: int, cols: int, seed: int = SEED_GRAD) -> np.ndarray:
    """Upstream gradient dH_out ~ N(0,1), float32 [n][cols]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((n, cols), dtype=np.float32)


# ----------------------------------------------------------------------------------------------
# NEXT-1 (training step) inputs: labels and the parameters of a multi-layer GAT
# ----------------------------------------------------------------------------------------------
SEED_LABEL = 5
ARXIV_CLASSES, ARXIV_TRAIN_FRAC = 40, 90_941 / 169_343   # ogbn-arxiv: 40 classes, 53.7 % train split


def labels(n: int, classes: int, train_frac: float = 1.0, seed: int = SEED_LABEL) -> np.ndarray:
    """Class ids int32 [n] uniform in [0, classes); rows outside a seeded train subset get -1."""
    rng = np.random.Generator(np.random.PCG64(seed))
    y = rng.integers(0, classes, size=n).astype(np.int32)
    if train_frac < 1.0:
        y[rng.random(n) >= train_frac] = -1
    return y


def gat_model_params(f: int, heads: int, head_dim: int, layers: int, classes: int, out_heads: int | None = None,
                     bias_scale: float = 0.0, seed: int = SEED_PARAM):
    """(hidden, out) parameter dicts of an L-layer GAT: L-1 hidden layers f -> heads*head_dim
    (concatenated) and a final layer -> out_heads x classes (averaged).  Glorot W / a; biases
    N(0, bias_scale) (0 = zeros, DGL's default)."""
    hidden = []
    fin = f
    for l in range(layers - 1):
        W, a_s, a_d = gat_params(fin, heads, head_dim, seed=seed + 10 * l)
        rng = np.random.Generator(np.random.PCG64(seed + 10 * l + 1))
        b = (rng.standard_normal(heads * head_dim) * bias_scale).astype(np.float32)
        hidden.append(dict(W=W, a_src=a_s, a_dst=a_d, b=b, heads=heads, head_dim=head_dim))
        fin = heads * head_dim
    oh = out_heads or heads
    W, a_s, a_d = gat_params(fin, oh, classes, seed=seed + 10 * (layers - 1))
    rng = np.random.Generator(np.random.PCG64(seed + 10 * (layers - 1) + 1))
    b = (rng.standard_normal(classes) * bias_scale).astype(np.float32)
    out = dict(W=W, a_src=a_s, a_dst=a_d, b=b, heads=oh, classes=classes)
    return hidden, out


CORA_CLASSES = 7


def gcn_model_params(f: int, hidden_dim: int, layers: int, classes: int, bias_scale: float = 0.0,
                     seed: int = SEED_PARAM):
    """(hidden, out) of an L-layer GCN: L-1 hidden layers -> hidden_dim and the final layer -> classes.
    Glorot W, biases N(0, bias_scale)."""
    hidden, fin = [], f
    for l in range(layers - 1):
        W = gcn_params(fin, hidden_dim, seed=seed + 10 * l)
        rng = np.random.Generator(np.random.PCG64(seed + 10 * l + 1))
        hidden.append(dict(W=W, b=(rng.standard_normal(hidden_dim) * bias_scale).astype(np.float32)))
        fin = hidden_dim
    W = gcn_params(fin, classes, seed=seed + 10 * (layers - 1))
    rng = np.random.Generator(np.random.PCG64(seed + 10 * (layers - 1) + 1))
    return hidden, dict(W=W, b=(rng.standard_normal(classes) * bias_scale).astype(np.float32))
