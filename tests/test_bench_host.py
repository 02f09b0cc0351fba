"""CPU checks of bench.py's accounting: the per-launch timeline is grouped into
the kernel classes the bench line reports (the dropout masks generated beside
the scans apart from the site applies), the GEMM-only roofline counts 2MNK per
launch, and the HBM classes use the algorithmic bytes of DESIGN.md §4.3."""

import bench


def _timeline():
    return [
        ("gemm 6400x4096x1024 t256x2", 0.06), ("lstm_fwd_tm_pair", 0.40), ("dropout_mask_kernel", 0.03),
        ("dropout_apply_kernel", 0.01), ("dropout_fwd_kernel4", 0.03), ("ce_stats_kernel", 0.15),
        ("ce_grad_kernel", 0.22), ("colsum_v8_kernel", 0.02), ("sumsq_partial_kernel", 0.1),
        ("clip_scale_kernel", 0.01), ("sgd_dense_kernel", 0.3), ("attn_tc_softmax", 0.01), ("gather_rows_kernel", 0.02),
    ]


def test_step_breakdown_classes():
    bd = bench.step_breakdown(_timeline())
    sh = bd["shares"]
    tot = sum(ms for _, ms in _timeline())
    assert abs(sh["serialized_step_ms"] - tot) < 1e-9
    assert abs(sh["dropout masks (beside the scans in the timed step)"] - round(0.03 / tot, 4)) < 1e-9
    assert abs(sh["dropout"] - round(0.04 / tot, 4)) < 1e-9  # apply + fused kernels
    assert abs(sh["recurrent scans"] - round(0.40 / tot, 4)) < 1e-9
    assert abs(sh["CE + column sums"] - round(0.39 / tot, 4)) < 1e-9
    assert abs(sh["SGD + norm"] - round(0.41 / tot, 4)) < 1e-9
    assert bd["gemms"] == [(6400, 4096, 1024, 0.06)]


def test_gemm_roofline_counts_2mnk():
    bd = bench.step_breakdown(_timeline())
    r = bench.gemm_roofline(bd, 1000.0)
    flops = 2.0 * 6400 * 4096 * 1024
    assert abs(r["flops_per_step"] - flops) < 1.0
    assert abs(r["achieved"] - flops / 0.06e-3 / 1e12) < 1e-6
    assert abs(r["frac"] - r["achieved"] / 1000.0) < 1e-12


def test_hbm_class_bytes():
    V, E, H, L, B, S, T = bench.CONFIGS["c3"]
    out = bench.hbm_classes(_timeline(), bench.CONFIGS["c3"], 6551.0)
    NS, NT = S * B, T * B
    ce = out["CE (ce_stats + ce_grad)"]
    assert ce["bytes"] == 3 * 2.0 * NT * V and abs(ce["ms"] - 0.37) < 1e-9
    ap = out["dropout apply (7 sites)"]
    # enc.l2's site reads y_f and y_b, H_o's reads fp32; the others read bf16
    assert ap["bytes"] == float(H) * (NS * (7 + 5 * (L - 2)) + NT * 5 * (L - 1) + NT * 7)
    assert "dropout fused (7 sites)" in out
    assert abs(out["norm + SGD (dense)"]["ms"] - 0.41) < 1e-9
