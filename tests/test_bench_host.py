"""Host-side measurement logic of bench.py (CPU): the usable-rate queueing computation and
the gather random-access model."""
import numpy as np

import bench
import coldgen


def test_usable_rate_bounds_and_monotone():
    """A FIFO server with service time D: the usable rate never exceeds the stability bound 1/mean(S),
    grows with the latency limit, and is 0 when the limit is below the service time itself."""
    s = np.full(4000, 0.1)   # ms
    r1 = bench.usable_rate(s, 0.15)
    r2 = bench.usable_rate(s, 1.0)
    r3 = bench.usable_rate(s, 10.0)
    assert 0 < r1 < r2 < r3 < 1e4   # 1 / 0.1 ms = 10^4 requests/s
    assert bench.usable_rate(s, 0.05) == 0.0


def test_usable_rate_md1_light_load():
    """M/D/1 at utilisation rho: P(wait > 0) = rho. With rho = 0.005 fewer than 1% of requests queue at all,
    so a limit just above the service time admits at least that rate."""
    s = np.full(20000, 0.1)
    assert bench.usable_rate(s, 0.1 + 1e-9) >= 0.005 / 0.1e-3 * 0.9


def test_gather_access_model_paper_schema():
    """S-paper, 16-chunk span: ad_id, user_id x cate and gender_age x ad_id (10^7 rows, 320 MB each) are
    random DRAM rows; the other 58 rows per ad (61 in total) are L2-served."""
    sch = coldgen.schema_paper()
    m = bench.gather_access_model(sch, 151552 * 16, 2, 6500.0)
    assert m["dram_random_rows_per_ad"] == 3
    assert m["l2_rows_per_ad"] == 58
    assert m["ceiling_ads_per_s_serial"] < m["ceiling_ads_per_s_overlapped"]
    # a short span gives every 10^6-row table too few touches to stay in L2
    m4 = bench.gather_access_model(sch, 151552, 2, 6500.0)
    assert m4["dram_random_rows_per_ad"] > m["dram_random_rows_per_ad"]


def test_gather_access_model_tiny_tables_all_l2():
    sch = coldgen.schema_tiny()
    m = bench.gather_access_model(sch, 10**6, 4, 6500.0)
    assert m["dram_random_rows_per_ad"] == 0
    assert m["l2_rows_per_ad"] > 0


def test_usable_rate_more_servers_more_rate():
    """S servers with the same service times sustain more load, at most S times the one-server bound."""
    s = np.full(3000, 0.1)
    r1 = bench.usable_rate(s, 1.0)
    r4 = bench.usable_rate(s, 1.0, servers=4)
    assert r1 < r4 < 4 * 1e4


def test_kernel_classes_attribute_mixed_chain_and_gemm_steps():
    """A step whose big chunks ran the chain and whose last chunk ran the layer-by-layer GEMMs: every
    class gets its own launches' time and FLOPs (counted by the library from the rows each launch
    covered), so no class can read above the peak because another kernel's work landed on it."""
    from paper_2007_16122_b200.cold import PROF_CHAIN, PROF_FC, PROF_KINDS, PROF_TAIL
    sch = coldgen.schema_paper()
    ms = np.zeros(PROF_KINDS)
    n = np.zeros(PROF_KINDS, np.int64)
    fl = np.zeros(PROF_KINDS)
    f123 = 2 * (256 * 1024 + 1024 * 512 + 512 * 256)
    ms[PROF_CHAIN], n[PROF_CHAIN], fl[PROF_CHAIN] = 10 * 0.27, 10, 10 * 151552 * f123
    ms[PROF_FC], n[PROF_FC], fl[PROF_FC] = 0.01, 1, 2 * 256 * 1024 * 4000          # fc1 GEMM, 4000 rows
    ms[PROF_FC + 1], n[PROF_FC + 1], fl[PROF_FC + 1] = 0.012, 1, 2 * 1024 * 512 * 4000
    ms[PROF_TAIL], n[PROF_TAIL], fl[PROF_TAIL] = 11 * 0.024, 11, 2 * (256 * 128 + 128 * 64 + 64 * 2) * (10 * 151552 + 4000)
    cls = bench.kernel_classes(sch, ms, n, fl)
    assert set(cls) == {"chain (fc1+fc2+fc3)", "gemm fc1", "gemm fc2", "tail (fc4+fc5+head)"}
    assert abs(cls["chain (fc1+fc2+fc3)"]["tflops"] - 151552 * f123 / 0.27e-3 / 1e12) < 1e-6
    assert abs(cls["gemm fc1"]["tflops"] - 2 * 256 * 1024 * 4000 / 0.01e-3 / 1e12) < 1e-6
    peaks = {"bf16_tflops": 1627.7, "bf16_tflops_sustained": 1362.4, "clocks_under_load": {"sm_mhz_median": 1237.0}}
    r = bench.fc_roofline(cls, peaks, "measured", {"sm_mhz": 1665.0}, {})
    assert r["kernel"] == "chain (fc1+fc2+fc3)" and r["peak"] == 1627.7
    assert abs(r["frac"] - r["achieved"] / 1627.7) < 1e-12 and abs(r["frac_sustained"] - r["achieved"] / 1362.4) < 1e-12
    assert abs(r["frac_sustained_at_run_clock"] - r["achieved"] / (1362.4 * 1665 / 1237)) < 1e-12
    assert "suspect" not in r
    ms[PROF_CHAIN] = 0.001                                                            # impossible rate: flagged
    r = bench.fc_roofline(bench.kernel_classes(sch, ms, n, fl), peaks, "measured", None, {})
    assert "suspect" in r
