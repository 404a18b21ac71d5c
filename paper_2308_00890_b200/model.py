"""The training step around the quantized layer: a multi-layer GAT whose
hidden layers are Tango's quantized layer (tango_gat_layer_fwd/bwd) and whose final layer runs in
full precision (tango_gat_out_fwd/bwd), with bias + ReLU between layers, cross-entropy
and the FP32 master-weight update (Eq.6).

Orchestration only: every step is a C-ABI call into libtango.so; all buffers are allocated once,
so a whole step can be captured in a CUDA graph.  The oracle counterpart is
oracle.oracle.gat_model_step (same layer order, layer ids and Philox tags).
"""
from __future__ import annotations

import torch

from . import tango as T
from .inputs import SR_SEED


class GATModel:
    """hidden: list of dicts {W, a_src, a_dst, b, heads, head_dim} (CUDA fp32 masters, updated in place);
    out: dict {W, a_src, a_dst, b, heads, classes}.  Layer l (1-based) of the hidden stack uses
    Philox layer_id = l."""

    def __init__(self, graph: T.DeviceGraph, hidden, out, slope=0.2, bits=8, seed=SR_SEED):
        self.graph, self.seed = graph, seed
        self.hidden, self.outp = hidden, out
        n = graph.n_local
        dev = "cuda"
        f32 = dict(dtype=torch.float32, device=dev)
        self.layers = [T.GATLayer(graph, p["W"], p["a_src"], p["a_dst"], p["heads"], p["head_dim"], slope=slope,
                                  bits=bits) for p in hidden]
        self.out = T.GATOutLayer(graph, out["W"], out["a_src"], out["a_dst"], out["b"], out["heads"], out["classes"],
                                 slope=slope)
        hd = [p["heads"] * p["head_dim"] for p in hidden]
        self.pre = [torch.empty((n, c), **f32) for c in hd]          # H_out of each quantized layer
        self.act = [torch.empty((n, c), **f32) for c in hd]          # ReLU(H_out + b)
        self.dact = [torch.empty((n, c), **f32) for c in hd]         # ∂ w.r.t. act
        self.dpre = [torch.empty((n, c), **f32) for c in hd]         # ∂ w.r.t. H_out
        self.scal = [torch.zeros(3, **f32) for _ in hidden]           # [amax pre, amax act, amax dpre]
        self.grads = []
        for p in hidden:
            self.grads.append(dict(W=torch.empty_like(p["W"]), a_src=torch.empty_like(p["a_src"]),
                                   a_dst=torch.empty_like(p["a_dst"]), b=torch.empty_like(p["b"])))
        self.out_grads = dict(W=torch.empty_like(out["W"]), a_src=torch.empty_like(out["a_src"]),
                              a_dst=torch.empty_like(out["a_dst"]), b=torch.empty_like(out["b"]))
        self.logits = torch.empty((n, out["classes"]), **f32)
        self.dlogits = torch.empty_like(self.logits)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = max([T.load().tango_colsum_workspace_bytes(n, c) for c in hd] + [4])
        self.ws = torch.empty(ws, dtype=torch.uint8, device=dev)
        self.pairs = []
        for p, g in zip(hidden + [out], self.grads + [self.out_grads]):
            for k in ("W", "a_src", "a_dst", "b"):
                self.pairs.append((p[k], g[k]))

    def forward(self, X, step=0):
        """Logits of the model (no loss); returns the logits buffer."""
        h, hint = X, None
        for l, layer in enumerate(self.layers):
            sc = self.scal[l]
            layer.forward(h, seed=self.seed, step=step, layer_id=l + 1, amax_hint=hint, out=self.pre[l],
                          amax_out=sc[0:1])
            T.bias_act_fwd(self.pre[l], self.hidden[l]["b"], out=self.act[l], amax_out=sc[1:2])
            h, hint = self.act[l], sc[1:2]
        self.out.forward(h, out=self.logits)
        return self.logits

    def step(self, X, labels, n_labeled, lr, step=0):
        """One full-batch training step: forward, loss, backward, SGD.  Returns the device loss (f64)."""
        self.forward(X, step)
        T.cross_entropy(self.logits, labels, n_labeled, dlogits=self.dlogits, loss=self.loss, status=self.status)
        nh = len(self.layers)
        h_last = self.act[-1] if nh else X
        og = self.out_grads
        self.out.backward(h_last, self.dlogits, outs=(self.dact[-1] if nh else None, og["W"], og["a_src"],
                                                      og["a_dst"], og["b"]))
        for l in range(nh - 1, -1, -1):
            sc, g = self.scal[l], self.grads[l]
            T.bias_act_bwd(self.act[l], self.dact[l], dx=self.dpre[l], dbias=g["b"], amax_out=sc[2:3],
                           workspace=self.ws)
            self.layers[l].backward(self.dpre[l], seed=self.seed, step=step, layer_id=l + 1, amax_hint=sc[2:3],
                                    outs=(self.dact[l - 1] if l > 0 else None, g["W"], g["a_src"], g["a_dst"]))
        T.sgd_update(self.pairs, lr)
        return self.loss

    def check_status(self):
        for layer in self.layers:
            layer.check_status()
        st = int(self.status.item())
        if st != 0:
            raise T.TangoError(st, "device status (cross_entropy)")


class GCNModel:
    """hidden: list of dicts {W, b} (CUDA fp32 masters, updated in place); out: {W, b}.  Hidden layers are
    the quantized GCN layer (tango_gcn_layer_fwd/bwd, layer_id = l) + bias + ReLU; the final layer is
    FP32 (tango_gcn_out_fwd/bwd).  Oracle counterpart: oracle.oracle.gcn_model_step."""

    def __init__(self, graph: T.DeviceGraph, hidden, out, bits=8, seed=SR_SEED):
        self.graph, self.seed, self.hidden, self.outp = graph, seed, hidden, out
        n = graph.n_local
        f32 = dict(dtype=torch.float32, device="cuda")
        self.layers = [T.GCNLayer(graph, p["W"], bits=bits) for p in hidden]
        self.out = T.GCNOutLayer(graph, out["W"], out["b"])
        widths = [p["W"].shape[1] for p in hidden]
        self.pre = [torch.empty((n, c), **f32) for c in widths]
        self.act = [torch.empty((n, c), **f32) for c in widths]
        self.dact = [torch.empty((n, c), **f32) for c in widths]
        self.dpre = [torch.empty((n, c), **f32) for c in widths]
        self.scal = [torch.zeros(3, **f32) for _ in hidden]
        self.grads = [dict(W=torch.empty_like(p["W"]), b=torch.empty_like(p["b"])) for p in hidden]
        self.out_grads = dict(W=torch.empty_like(out["W"]), b=torch.empty_like(out["b"]))
        self.logits = torch.empty((n, out["W"].shape[1]), **f32)
        self.dlogits = torch.empty_like(self.logits)
        self.loss = torch.zeros(1, dtype=torch.float64, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        ws = max([T.load().tango_colsum_workspace_bytes(n, c) for c in widths] + [4])
        self.ws = torch.empty(ws, dtype=torch.uint8, device="cuda")
        self.pairs = [(p[k], g[k]) for p, g in zip(hidden + [out], self.grads + [self.out_grads]) for k in ("W", "b")]

    def forward(self, X, step=0):
        h, hint = X, None
        for l, layer in enumerate(self.layers):
            sc = self.scal[l]
            layer.forward(h, seed=self.seed, step=step, layer_id=l + 1, amax_hint=hint, out=self.pre[l],
                          amax_out=sc[0:1])
            T.bias_act_fwd(self.pre[l], self.hidden[l]["b"], out=self.act[l], amax_out=sc[1:2])
            h, hint = self.act[l], sc[1:2]
        self.out.forward(h, out=self.logits)
        return self.logits

    def step(self, X, labels, n_labeled, lr, step=0):
        self.forward(X, step)
        T.cross_entropy(self.logits, labels, n_labeled, dlogits=self.dlogits, loss=self.loss, status=self.status)
        nh = len(self.layers)
        og = self.out_grads
        self.out.backward(self.act[-1] if nh else X, self.dlogits, outs=(self.dact[-1] if nh else None, og["W"],
                                                                         og["b"]))
        for l in range(nh - 1, -1, -1):
            sc, g = self.scal[l], self.grads[l]
            T.bias_act_bwd(self.act[l], self.dact[l], dx=self.dpre[l], dbias=g["b"], amax_out=sc[2:3],
                           workspace=self.ws)
            self.layers[l].backward(self.dpre[l], seed=self.seed, step=step, layer_id=l + 1,
                                    outs=(self.dact[l - 1] if l > 0 else None, g["W"]))
        T.sgd_update(self.pairs, lr)
        return self.loss

    def check_status(self):
        for layer in self.layers:
            layer.check_status()
        st = int(self.status.item())
        if st != 0:
            raise T.TangoError(st, "device status (cross_entropy)")
