"""One rank of the partitioned GAT dataflow, emulated with oracle primitives over gloo.

Launched by tests/test_multigpu_cpu.py as
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 ... dist_gat_worker.py
It follows the multi-GPU dataflow of DESIGN.md §8 (the one api.cu runs over NCCL): destination-row
blocks from partition.partition_rows, AllReduce-MAX of every amax (reading R28), quantization of
the owned rows with GLOBAL Philox counters (g0 = row_begin * cols), all-gather of the node tensors
the sparse steps read (q_H′, q_S, q_G), the sparse steps on the owned in-CSR / out-CSR rows, and
an int64 AllReduce-SUM of the ∂W partials.  Every per-rank result must equal the corresponding
rows / edges of the single-process oracle bit for bit.  Row-local dense steps (GEMM rows, the ∂H′
chain rule) are taken from the single-process oracle, not re-derived.
"""
import argparse
import os
import sys
from types import SimpleNamespace

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_2308_00890_b200 import inputs  # noqa: E402
from paper_2308_00890_b200.partition import local_graph, partition_rows  # noqa: E402

ROLE = dict(H=1, W=2, HP=3, S=4, D=5, G=6, DHP=7)


def amax_all(x):
    t = torch.tensor([float(np.abs(x).max()) if x.size else 0.0], dtype=torch.float32)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return np.float32(t.item())


def gather_rows(local, counts):
    """All-gather blocks of rows of different sizes (pad to the largest, trim)."""
    mx = max(counts)
    pad = np.zeros((mx,) + local.shape[1:], local.dtype)
    pad[:local.shape[0]] = local
    t = torch.from_numpy(pad.view(np.uint8) if local.dtype == np.int8 else pad)
    parts = [torch.empty_like(t) for _ in counts]
    dist.all_gather(parts, t)
    out = [p.numpy()[:c] for p, c in zip(parts, counts)]
    out = np.concatenate(out, axis=0)
    return out.view(np.int8) if local.dtype == np.int8 else out


def eq(name, got, want, rank):
    got, want = np.asarray(got), np.asarray(want)
    if got.shape != want.shape or not np.array_equal(got, want):
        bad = np.argwhere(got != want) if got.shape == want.shape else "shape"
        raise AssertionError(f"rank {rank}: {name} differs ({got.shape} vs {want.shape}; {bad[:3] if len(bad) else bad})")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=400)
    ap.add_argument("--draws", type=int, default=3000)
    ap.add_argument("--gamma", type=float, default=2.1)
    ap.add_argument("--F", type=int, default=24)
    ap.add_argument("--heads", type=int, default=2)
    ap.add_argument("--hd", type=int, default=16)
    ap.add_argument("--chunk", type=int, default=7)
    a = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    orc.set_threads(1)

    gr = inputs.chung_lu_graph(a.n, a.draws, a.gamma, dmax=a.n // 2, seed=5)
    F, heads, hd, chunk, slope, step, L = a.F, a.heads, a.hd, a.chunk, 0.2, 3, 1
    HD = heads * hd
    seed = inputs.SR_SEED
    H = inputs.features(gr.n, F, seed=41)
    W, a_src, a_dst = inputs.gat_params(F, heads, hd, seed=42)
    dH = inputs.grad_out(gr.n, HD, seed=43)
    f = orc.gat_fwd(gr, H, W, a_src, a_dst, heads, hd, slope=slope, bits=8, seed=seed, step=step, layer_id=L,
                    chunk=chunk)
    b = orc.gat_bwd(gr, f, H, W, a_src, a_dst, dH)

    starts = partition_rows(gr, world)
    counts = [starts[r + 1] - starts[r] for r in range(world)]
    rb, re = starts[rank], starts[rank + 1]
    lg = local_graph(gr, rb, re)
    ib, ie = lg.in_edge0, lg.in_edge0 + lg.e
    ecounts = [int(gr.in_ptr[starts[r + 1]] - gr.in_ptr[starts[r]]) for r in range(world)]
    Q = lambda x, role, cols, amax: orc.quantize(x, 8, seed, step, (L << 8) | role, g0=rb * cols, amax=amax)

    # F1 Q(H) on the owned rows; F2 Q(W) replicated
    qH, sH, _ = Q(H[rb:re], ROLE["H"], F, amax_all(H[rb:re]))
    eq("qH", qH, f["qH"][rb:re], rank)
    eq("sH", sH, f["sH"][0], rank)
    # F4 Q(H′), Q(S), Q(D) of the owned rows (H′, S, D rows are row-local GEMM results)
    Hp, S, D = f["Hp"][rb:re], f["S"][rb:re], f["Dd"][rb:re]
    qHp, sHp, _ = Q(Hp, ROLE["HP"], HD, amax_all(Hp))
    qS, sS, _ = Q(S, ROLE["S"], heads, amax_all(S))
    qD, sD, _ = Q(D, ROLE["D"], heads, amax_all(D))
    eq("qHp", qHp, f["qHp"][rb:re], rank)
    eq("qS", qS, f["qS"][rb:re], rank)
    eq("qD", qD, f["qD"][rb:re], rank)
    qHp_all, qS_all = gather_rows(qHp, counts), gather_rows(qS, counts)
    eq("qHp_all", qHp_all, f["qHp"], rank)
    # F5/F6 on the owned in-CSR rows
    e_pre, el = orc.sddmm_add(lg, heads, orc.qref(q=qS_all, s=sS), orc.qref(q=qD, s=sD), slope, chunk)
    m, den, alpha = orc.edge_softmax(lg, heads, el, chunk)
    Hout = orc.spmm_alpha(lg, 0, heads, HD, alpha, orc.qref(q=qHp_all, s=sHp), chunk)
    eq("e_pre", e_pre, f["e_pre"][ib:ie], rank)
    eq("m", m, f["m"][rb:re], rank)
    eq("den", den, f["den"][rb:re], rank)
    eq("alpha", alpha, f["alpha"][ib:ie], rank)
    eq("Hout", Hout, f["Hout"][rb:re], rank)

    # B1 Q(∂H_out); B2-B4 on the owned in-CSR rows
    qG, sG, _ = Q(dH[rb:re], ROLE["G"], HD, amax_all(dH[rb:re]))
    eq("qG", qG, b["qG"][rb:re], rank)
    qG_all = gather_rows(qG, counts)
    dalpha = orc.sddmm_dot(lg, heads, HD, orc.qref(q=qG, s=sG), orc.qref(q=qHp_all, s=sHp), chunk)
    P, _, dEp = orc.softmax_bwd(lg, heads, alpha, dalpha, e_pre, slope, chunk)
    dD = orc.edge_sum(lg, 0, heads, dEp, chunk)
    eq("dalpha", dalpha, b["dalpha"][ib:ie], rank)
    eq("P", P, b["P"][rb:re], rank)
    eq("dE_pre", dEp, b["dE_pre"][ib:ie], rank)
    eq("dD", dD, b["dD"][rb:re], rank)
    # B5/B6 on the owned out-CSR rows, with the per-edge α / ∂E_pre of every rank gathered
    alpha_all, dEp_all = gather_rows(alpha, ecounts), gather_rows(dEp, ecounts)
    ob, oe = int(gr.out_ptr[rb]), int(gr.out_ptr[re])
    eids = gr.out_eid[ob:oe]
    og = SimpleNamespace(n=lg.n, e=lg.e_out, in_ptr=lg.out_ptr, in_src=lg.out_dst)
    agg = orc.spmm_alpha(og, 0, heads, HD, alpha_all[eids], orc.qref(q=qG_all, s=sG), chunk)
    dS = orc.edge_sum(og, 0, heads, dEp_all[eids], chunk)
    eq("dHp_agg", agg, b["dHp_agg"][rb:re], rank)
    eq("dS", dS, b["dS"][rb:re], rank)
    # B8 Q(∂H′) of the owned rows (the chain rule B7 is row-local); B9 ∂W int64 partials summed
    dHp = b["dHp"][rb:re]
    qdHp, sdHp, _ = Q(dHp, ROLE["DHP"], HD, amax_all(dHp))
    eq("qdHp", qdHp, b["qdHp"][rb:re], rank)
    eq("sdHp", sdHp, b["sdHp"][0], rank)
    part, _ = orc.gemm(orc.qref(q=qH), orc.qref(q=qdHp), F, HD, lg.n, F, HD, transA=True)
    t = torch.from_numpy(part.copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    full, _ = orc.gemm(orc.qref(q=f["qH"]), orc.qref(q=b["qdHp"]), F, HD, gr.n, F, HD, transA=True)
    eq("dW_acc", t.numpy(), full, rank)
    dist.barrier()
    print(f"OK rank{rank} rows [{rb},{re}) edges [{ib},{ie})", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
