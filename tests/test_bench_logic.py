"""CPU checks of bench.py's measurement bookkeeping (no GPU): gather passes are timed as the sum of
their launches, and every pass / kernel the roofline can pick has a bytes model."""
import bench


def test_pass_profile_merges_launches():
    prof = {"gat_bwd_src": (2.0, 10), "gat_bwd_src_hub": (1.0, 10), "gat_bwd_src_combine": (0.25, 10),
            "quantize": (2.5, 60), "gat_fwd_agg": (1.5, 10)}
    r = bench.pass_profile(prof)
    assert r["gat_bwd_src"] == (3.25, 10)
    assert "gat_bwd_src_hub" not in r and "gat_bwd_src_combine" not in r
    assert r["quantize"] == (2.5, 60) and r["gat_fwd_agg"] == (1.5, 10)


def test_models_cover_the_roofline_candidates():
    for name in list(bench.PASSES) + ["quantize", "absmax"]:
        m = bench.kernel_model(name, 1000, 100, 128, 4, 512, {}, 1965.0)
        assert m is not None and m[0] > 0 and m[1] > 0
    assert bench.kernel_model("gat_bwd_src_hub", 1000, 100, 128, 4, 512, {}, 1965.0) is None
    # the pass model counts every edge: bytes grow with E at the per-edge rate of each dataflow
    for df, per_edge in ((1, 8 + 8 * 4 + 512), (2, 4 + 512 + 13 * 4)):
        b1 = bench.kernel_model("gat_bwd_src", 1000, 100, 128, 4, 512, {}, 1965.0, df)[0]
        b2 = bench.kernel_model("gat_bwd_src", 2000, 100, 128, 4, 512, {}, 1965.0, df)[0]
        assert b2 - b1 == 1000 * per_edge
    # v6 passes merge their launches; the ALU peak follows the unit counts (148 SMs x 128 lanes x clock)
    r = bench.pass_profile({"gat_bwd_dst": (1.0, 5), "gat_bwd_dst2": (0.5, 5), "gat_fwd_stats": (0.2, 5),
                            "gat_fwd_stats1": (0.1, 5)})
    assert r == {"gat_bwd_dst": (1.5, 5), "gat_fwd_stats": (0.30000000000000004, 5)}
    assert abs(bench.alu_peak(1965.0) - 148 * 128 * 1.965e9) < 1


def test_pass_bound_follows_the_l2():
    # gather passes are issue-bound while the gathered int8 table fits in L2 (Reddit: 233 K x 512 B)
    assert bench.pass_bound("gat_fwd_agg", 232_965 * 512) == "alu"
    assert bench.pass_bound("gat_bwd_src", 2_449_029 * 512) == "hbm"     # products: 1.25 GB table
    assert bench.pass_bound("gat_bwd_dst", 1000) == "hbm"
    assert bench.ncu_traffic("no-such-workload", "gat_bwd_src") is None


def test_relabel_by_degree_is_a_permutation():
    import numpy as np
    from paper_2308_00890_b200 import inputs
    g = inputs.random_graph(300, 1500, seed=9)
    h = inputs.relabel_by_degree(g)
    dg, dh = np.diff(g.in_ptr), np.diff(h.in_ptr)
    assert h.e == g.e and np.all(np.diff(dh) <= 0)                      # degrees now descending
    assert np.array_equal(np.sort(dg), np.sort(dh))                      # same degree multiset
    assert np.array_equal(np.sort(np.diff(g.out_ptr)), np.sort(np.diff(h.out_ptr)))
    # CSR invariants of the relabelled graph: sources ascending within each row
    for v in range(h.n):
        row = h.in_src[h.in_ptr[v]:h.in_ptr[v + 1]]
        assert np.all(np.diff(row) > 0)
