"""Multi-rank path on CPU: partition logic and a world-size-2
gloo run of the partitioned dataflow (tests/dist_gat_worker.py), checked bit-exact against the
single-process oracle.  The NCCL transport itself needs GPUs; this covers the host-side logic
and the partition-independence of every step (global Philox counters, per-row canonical sums).
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2308_00890_b200 import inputs
from paper_2308_00890_b200.partition import block_sizes, local_graph, partition_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
def test_partition_covers_and_balances(nranks):
    g = inputs.chung_lu_graph(3000, 20000, 2.1, dmax=1500, seed=9)
    starts = partition_rows(g, nranks)
    assert starts[0] == 0 and starts[-1] == g.n and len(starts) == nranks + 1
    assert all(b >= 0 for b in block_sizes(starts))
    blocks = [local_graph(g, starts[r], starts[r + 1]) for r in range(nranks)]
    # concatenating the blocks gives back the global in- and out-CSR
    assert np.array_equal(np.concatenate([b.in_src for b in blocks]), g.in_src)
    assert np.array_equal(np.concatenate([b.out_dst for b in blocks]), g.out_dst)
    e0 = 0
    for b in blocks:
        assert b.in_edge0 == e0
        assert np.array_equal(b.in_ptr + b.in_edge0, g.in_ptr[b.row_begin:b.row_end + 1])
        e0 += b.e
    # balance: each block's (edges + rows) within one max-degree row of the ideal share
    load = [b.e + b.n for b in blocks]
    ideal = (g.e + g.n) / nranks
    maxdeg = int(np.diff(g.in_ptr).max())
    assert max(load) <= ideal + maxdeg + 1
    # out_eid only for the whole graph
    assert (blocks[0].out_eid is not None) == (nranks == 1)


def test_partition_degenerate():
    g = inputs.random_graph(5, 4, seed=1)
    starts = partition_rows(g, 8)           # more ranks than rows: empty blocks are allowed
    assert starts[-1] == g.n and sorted(starts) == starts
    empty = [local_graph(g, starts[r], starts[r + 1]) for r in range(8) if starts[r] == starts[r + 1]]
    assert empty and all(b.e == 0 and b.e_out == 0 and b.in_ptr.tolist() == [0] for b in empty)
    with pytest.raises(ValueError):
        local_graph(g, 3, 2)
    with pytest.raises(ValueError):
        partition_rows(g, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("args", [["--chunk", "7"], ["--chunk", "256", "--heads", "4", "--hd", "8", "--F", "40"]],
                         ids=["chunk7", "chunk256_h4"])
def test_gloo_world2_partitioned_gat_matches_single_process(orc, args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_gat_worker.py"), *args]
    env = dict(os.environ, OMP_NUM_THREADS="1", PYTHONPATH=ROOT)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "OK rank0" in out and "OK rank1" in out, out[-2000:]
