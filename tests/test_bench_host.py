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
