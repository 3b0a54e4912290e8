"""Pins for the oracle (CPU only): each part of oracle/cold_oracle.c is checked against
something other than itself — the paper's closed forms, the hand-computed worked
example (tests/golden/), hash known answers, torch fp64 library routines, brute
force and the independent pure-Python twin oracle/mini.py.
"""
import dataclasses
import math

import numpy as np
import pytest

import coldgen
import oracle
from oracle import mini
from tests.fixtures import bag_schema, load_golden, small_case, worked_example


# ---- P-1 linear_log (Eq. eq:log) --------------------------------

def test_linear_log_closed_forms():
    for x, want in load_golden("linear_log_values.json")["points"]:
        assert oracle.linear_log(x) == pytest.approx(want, rel=1e-14, abs=1e-15)


def test_linear_log_odd_monotone_c1():
    xs = np.concatenate([-np.logspace(-6, 30, 400), np.linspace(-3, 3, 601), np.logspace(-6, 30, 400)])
    xs.sort()
    ys = np.array([oracle.linear_log(x) for x in xs])
    assert np.all(np.diff(ys) >= 0) and np.all(np.diff(ys)[np.diff(xs) > 0] > 0)   # strictly increasing
    for x in xs:
        assert oracle.linear_log(-x) == -oracle.linear_log(x)                      # odd
    assert max(abs(y) for y in ys) <= 71.0                                         # range compression
    eps = 1e-6                                                                     # C^1 at |x| = 1
    for c in (1.0, -1.0):
        left = (oracle.linear_log(c) - oracle.linear_log(c - eps)) / eps
        right = (oracle.linear_log(c + eps) - oracle.linear_log(c)) / eps
        assert abs(left - right) <= 2 * eps


# ---- P-2 sigma --------------------------------------------------------

def test_sigmoid():
    assert oracle.sigmoid(0.0) == 0.5
    assert oracle.sigmoid(40.0) >= 1 - 1e-15
    for z in np.linspace(-50, 50, 201):
        assert oracle.sigmoid(-z) == pytest.approx(1 - oracle.sigmoid(z), abs=3e-16)
        assert oracle.sigmoid(z) == pytest.approx(mini.sigmoid(z), rel=1e-15)
    assert oracle.sigmoid(-800.0) == 0.0 and oracle.sigmoid(800.0) == 1.0


# ---- P-3 cross-feature hash (AMB-9) ----------------------------------------------------

def test_cross_hash_known_answers():
    kat = load_golden("cross_hash_kat.json")
    for k, v in kat["fmix64"]:
        assert oracle.fmix64(k) == int(v, 16)
    for g, x, y, card, want in kat["cross_row"]:
        assert oracle.cross_row(g, x, y, card) == want
        assert mini.cross_row(g, x, y, card) == want


def test_cross_hash_properties():
    rng = np.random.default_rng(5)
    xs = rng.integers(0, 2**31 - 1, 100000)
    ys = rng.integers(0, 2**31 - 1, 100000)
    counts = np.zeros(1000, np.int64)
    for x, y in zip(xs[:100000], ys[:100000]):
        counts[oracle.cross_row(3, int(x), int(y), 1000)] += 1
    assert counts.max() <= 3 * counts.mean()
    for x, y in zip(xs[:200], ys[:200]):
        assert oracle.cross_row(9, int(x), int(y), 1) == 0    # cardinality 1 -> row 0
        r = oracle.cross_row(9, int(x), int(y), 12345)
        assert 0 <= r < 12345 and r == oracle.cross_row(9, int(x), int(y), 12345)


# ---- P-4 worked example ----------------------------------------------------------------

@pytest.mark.parametrize("head", ["one", "two"])
def test_worked_example(head):
    schema, params, batch, exp = worked_example(head)
    m = oracle.Model(schema, params)
    p, z = oracle.score(m, batch)
    if head == "one":
        assert p[0] == pytest.approx(exp["adA_p_one_wide"], abs=1e-14)
        assert p[1] == pytest.approx(exp["adB_p_one_wide"], abs=1e-14)
        assert z[0] == pytest.approx(exp["adA_z_one_wide"], abs=1e-14)
        assert z[1] == pytest.approx(exp["adB_z_one_wide"], abs=1e-14)
        idx, _ = oracle.topk(p, 1)
        assert idx[0] == exp["top1_one_wide"]
        p_off, _ = oracle.score(oracle.Model(schema, params, linear_log=False), batch)
        assert p_off[0] == pytest.approx(exp["adA_p_one_wide_ll_off"], abs=1e-14)
        assert p_off[1] == pytest.approx(exp["adB_p_one_wide_ll_off"], abs=1e-14)
    else:
        assert p[0] == pytest.approx(exp["adA_p_two_wide"], abs=1e-14)
        assert p[1] == pytest.approx(exp["adB_p_two_wide"], abs=1e-14)
        idx, _ = oracle.topk(p, 1)
        assert idx[0] == exp["top1_two_wide"]


def test_worked_example_features():
    """ê (after LL) and s for ad A: x = [s_g * ê_g]."""
    schema, params, batch, exp = worked_example("one")
    m = oracle.Model(schema, params)
    x = oracle.features(m, batch)[0]
    eh = np.asarray(exp["adA_features_ll_on"])
    s = np.repeat(exp["adA_se_ll_on"], 2)
    np.testing.assert_allclose(x, s * eh, rtol=1e-14, atol=1e-15)


# ---- SE importance weights and feature-group selection (F3) ---------------

def test_se_gates_worked_example():
    """s_g of ad A in the hand-computed worked example (P-4 golden values)."""
    schema, params, batch, exp = worked_example("one")
    s = oracle.se_gates(oracle.Model(schema, params), batch)
    np.testing.assert_allclose(s[0], exp["adA_se_ll_on"], rtol=1e-14)


def test_se_gates_planted_closed_form_and_selection():
    """w_g = 0, b_g = 3 - 0.5 g: s_g = sigma(b_g) for every ad (P-11 closed form), so ranking by
    mean s_g selects the first K groups of the schema; every s_g lies in (0, 1)."""
    sch = coldgen.scaled_schema(coldgen.schema_full(), 2000)
    params = coldgen.make_params(sch, seed=5, precision="f16", se="planted")
    batch = coldgen.make_batch(sch, 2, [40, 25], seed=6)
    s = oracle.se_gates(oracle.Model(sch, params), batch)
    b = 3.0 - 0.5 * np.arange(len(sch.groups))
    np.testing.assert_allclose(s, np.broadcast_to(1.0 / (1.0 + np.exp(-b)), s.shape), rtol=1e-15)
    for K in (1, 8, 20, 32):
        assert oracle.select_groups(s.mean(0), K) == list(range(K))


def test_se_gates_planted_noisy_ranking():
    """|w_g . ê_g| <= 16 * 0.01 * LL(8) < 0.5 = the b-gaps, so the empirical ranking keeps schema
    order (P-11 empirical run) and the gates stay within their bounds."""
    sch = coldgen.scaled_schema(coldgen.schema_full(), 2000)
    params = coldgen.make_params(sch, seed=7, precision="f16", se="planted_noisy")
    batch = coldgen.make_batch(sch, 3, [60, 60, 60], seed=8)
    s = oracle.se_gates(oracle.Model(sch, params), batch)
    assert np.all((s > 0) & (s < 1))
    assert oracle.select_groups(s.mean(0), 12) == list(range(12))
    b = 3.0 - 0.5 * np.arange(len(sch.groups))
    lo, hi = 1 / (1 + np.exp(-(b - 0.5))), 1 / (1 + np.exp(-(b + 0.5)))
    assert np.all((s >= lo) & (s <= hi))


def test_select_groups_ties_and_range():
    assert oracle.select_groups([0.5, 0.7, 0.5, 0.7], 3) == [0, 1, 3]
    assert oracle.select_groups([0.1, 0.2], 2) == [0, 1]
    with pytest.raises(oracle.OracleError):
        oracle.select_groups([0.1, 0.2], 3)


# ---- P-6 reduction to library routines (torch fp64) ---------------------------------

def test_reduces_to_torch_embedding_bag_mlp():
    """LL off and SE pinned to s = 1 (w = 0, b = +40): the model is
    MLP(concat(embedding_bag_sum)). Rows for cross groups come from the pinned twin hash."""
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F
    sch, params, batch = small_case("tiny", R=3, n_ads=(6, 11, 2), precision="f32", se="identity")
    m = oracle.Model(sch, params, linear_log=False)
    p, z = oracle.score(m, batch)
    feats = []
    for g, grp in enumerate(sch.groups):
        bags = []
        for r in range(batch.R):
            for a in range(batch.ad_offsets[r], batch.ad_offsets[r + 1]):
                bags.append(mini.rows(sch, batch, g, r, a))
        flat = torch.tensor([x for b in bags for x in b], dtype=torch.long)
        offs = torch.tensor(np.cumsum([0] + [len(b) for b in bags[:-1]]), dtype=torch.long)
        T = torch.tensor(params.table_f64(g))
        feats.append(F.embedding_bag(flat, T, offs, mode="sum"))
    h = torch.cat(feats, 1)
    L = len(params.fc_w)
    for l in range(L):
        h = F.linear(h, torch.tensor(params.fc_w[l], dtype=torch.float64), torch.tensor(params.fc_b[l], dtype=torch.float64))
        if l < L - 1:
            h = F.relu(h)
    zt = h[:, 0] if h.shape[1] == 1 else h[:, 1] - h[:, 0]
    np.testing.assert_allclose(z, zt.numpy(), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(p, torch.sigmoid(zt).numpy(), rtol=1e-12, atol=1e-14)


def test_zero_fcn_scores_sigma_of_bias():
    sch, params, batch = small_case("tiny", R=2, n_ads=(9, 4), init="zero")
    p, _ = oracle.score(oracle.Model(sch, params), batch)
    np.testing.assert_allclose(p, mini.sigmoid(float(params.fc_b[-1][-1])), rtol=1e-15)


# ---- P-12 the two oracles agree --------------------------------------------------------

@pytest.mark.parametrize("case", ["tiny_f32", "tiny_f16_zipf", "paper_bf16", "bags", "bags_2req_empty"])
def test_c_oracle_matches_python_twin(case):
    if case == "tiny_f32":
        sch, params, batch = small_case("tiny", R=2, n_ads=(7, 5))
    elif case == "tiny_f16_zipf":
        sch, params, batch = small_case("tiny", R=2, n_ads=(3, 9), precision="f16", dist="zipf")
    elif case == "paper_bf16":
        sch, params, batch = small_case("paper", R=1, n_ads=(4,), precision="bf16", cap=5000)
    else:
        sch = bag_schema()
        params = coldgen.make_params(sch, seed=3, precision="f32")
        batch = coldgen.make_batch(sch, 3, [4, 0, 6] if case == "bags_2req_empty" else [5, 3, 6], seed=11)
    for sel in (None, [0, 2, 4, 5, 6] if sch.M >= 7 else None):
        d_in = (len(sel) if sel else sch.M) * sch.k
        if d_in != params.fc_w[0].shape[1]:
            params = coldgen.make_params(sch, seed=3, precision=params.precision, d_in=d_in,
                                         table_dtype=params.table_dtype)
        p, z = oracle.score(oracle.Model(sch, params, selected=sel), batch)
        pm, zm = mini.score(sch, params, batch, selected=sel)
        np.testing.assert_allclose(p, pm, rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(z, zm, rtol=1e-13, atol=1e-14)


def test_rows_match_twin_and_definition():
    sch = bag_schema()
    params = coldgen.make_params(sch, seed=3, precision="f32")
    batch = coldgen.make_batch(sch, 3, [5, 3, 6], seed=12)
    m = oracle.Model(sch, params)
    for r in range(batch.R):
        for a in range(batch.ad_offsets[r], batch.ad_offsets[r + 1]):
            for g in range(sch.M):
                got = oracle.rows(m, batch, g, a).tolist()
                assert got == mini.rows(sch, batch, g, r, a)
            # cross g=4 is the x-major product of user bag x ad bag: count = |x| * |y|
            ub = batch.ids[1][batch.offs[1][r]:batch.offs[1][r + 1]]
            ab = batch.ids[3][batch.offs[3][a]:batch.offs[3][a + 1]]
            assert len(oracle.rows(m, batch, 4, a)) == len(ub) * len(ab)
            assert oracle.rows(m, batch, 6, a).tolist() == [0] * len(ub)    # card 1


# ---- invariants ------------------------------------------------------------------------

def test_permuting_ads_permutes_scores():
    sch, params, batch = small_case("tiny", R=1, n_ads=(23,))
    p, _ = oracle.score(oracle.Model(sch, params), batch)
    perm = np.random.default_rng(0).permutation(23)
    b2 = coldgen.Batch(batch.R, batch.ad_offsets, [None if v is None else (v[perm] if batch.offs[g] is None else v)
                                                   for g, v in enumerate(batch.ids)], batch.offs, None, batch.req_ids)
    p2, _ = oracle.score(oracle.Model(sch, params), b2)
    np.testing.assert_array_equal(p2, p[perm])


def test_request_independence_and_sampling():
    """Scores of a request do not depend on the other requests in the batch,
    and scoring a sample of ads equals scoring all of them."""
    sch, params, batch = small_case("tiny", R=4, n_ads=(5, 8, 3, 6))
    m = oracle.Model(sch, params)
    p, _ = oracle.score(m, batch)
    for r in range(batch.R):
        sb = coldgen.sub_batch(batch, [r])
        pr, _ = oracle.score(m, sb)
        np.testing.assert_array_equal(pr, p[batch.ad_offsets[r]:batch.ad_offsets[r + 1]])
    ads = np.array([21, 0, 7, 13, 13])
    ps, _ = oracle.score(m, batch, ad_list=ads)
    np.testing.assert_array_equal(ps, p[ads])


def test_row_order_equals_column_order():
    """column-based computation reorders work, not results."""
    sch = bag_schema()
    params = coldgen.make_params(sch, seed=4, precision="f32")
    batch = coldgen.make_batch(sch, 3, [5, 2, 7], seed=13)
    m = oracle.Model(sch, params)
    np.testing.assert_array_equal(oracle.features(m, batch, order=0), oracle.features(m, batch, order=1))


def test_user_broadcast_equals_per_pair():
    """Hoisting the user side is exact: user-group features are identical for all ads of a
    request, and equal those of a one-ad request of the same user."""
    sch, params, batch = small_case("tiny", R=2, n_ads=(6, 4))
    m = oracle.Model(sch, params)
    x = oracle.features(m, batch)
    k = sch.k
    ucols = np.concatenate([np.arange(g * k, (g + 1) * k) for g in sch.side_indices(coldgen.USER)])
    for r in range(batch.R):
        blk = x[batch.ad_offsets[r]:batch.ad_offsets[r + 1]][:, ucols]
        assert np.all(blk == blk[0])


def test_se_weights_in_unit_interval():
    sch, params, batch = small_case("tiny", R=1, n_ads=(30,))
    m = oracle.Model(sch, params)
    x = oracle.features(m, batch)
    xe = oracle.features(oracle.Model(sch, coldgen.make_params(sch, seed=7, precision="f32", se="identity")), batch)
    k = sch.k
    for g in range(sch.M):
        cols = slice(g * k, (g + 1) * k)
        nz = np.abs(xe[:, cols]) > 1e-12
        s = x[:, cols][nz] / xe[:, cols][nz]
        assert np.all((s > 0) & (s < 1))


def test_dense_se_block_diagonal_equals_per_group():
    """AMB-1: Doc B's dense SE with a block-diagonal W is Doc A's per-group SE."""
    sch, params, batch = small_case("tiny", R=2, n_ads=(4, 5))
    M, k = sch.M, sch.k
    Wd = np.zeros((M, M * k))
    for g in range(M):
        Wd[g, g * k:(g + 1) * k] = params.se_w[g]
    p1, _ = oracle.score(oracle.Model(sch, params), batch)
    p2, _ = oracle.score(oracle.Model(sch, params, se_dense=(Wd, params.se_b.astype(np.float64))), batch)
    np.testing.assert_allclose(p1, p2, rtol=1e-15)


def test_dense_se_cross_group_gate_closed_form():
    """AMB-1, Doc B: under the dense reading the gate of group j may read another group's
    embedding. With one nonzero per row, W[j, (j+1 mod M) k + d_j] = c_j, the gate is the closed form
    s_j = sigma(c_j * ê_{j+1}[d_j] + b_j); check x = s ê against the identity-gate features (x = ê) of the
    same batch. A transposed W, a wrong column order or a dropped bias fails this."""
    sch, params, batch = small_case("tiny", R=2, n_ads=(6, 3))
    M, k = sch.M, sch.k
    rng = np.random.default_rng(11)
    W = np.zeros((M, M * k))
    c = rng.uniform(-1.5, 1.5, M)
    dj = rng.integers(0, k, M)
    for j in range(M):
        W[j, ((j + 1) % M) * k + dj[j]] = c[j]
    b = rng.uniform(-1, 1, M)
    x = oracle.features(oracle.Model(sch, params, se_dense=(W, b)), batch)
    e = oracle.features(oracle.Model(sch, coldgen.make_params(sch, seed=7, precision="f32", se="identity")), batch)
    for j in range(M):
        src = e[:, ((j + 1) % M) * k + dj[j]]
        s = 1.0 / (1.0 + np.exp(-(c[j] * src + b[j])))
        np.testing.assert_allclose(x[:, j * k:(j + 1) * k], s[:, None] * e[:, j * k:(j + 1) * k], rtol=1e-12, atol=1e-15)


def test_ll_order_variants_agree_when_gate_is_one():
    sch, params, batch = small_case("tiny", R=1, n_ads=(9,), se="identity")
    a = oracle.features(oracle.Model(sch, params), batch)
    b = oracle.features(oracle.Model(sch, params, ll_after_se=True), batch)
    np.testing.assert_allclose(a, b, rtol=1e-15)


def test_ll_order_variants_closed_form_with_constant_gate():
    """AMB-3 ("put a linear_log operator in the first layer"; P:229-235 SE): with w_g = 0 the gate
    is the constant s_g = sigma(b_g) != 1, so the two orders have closed forms over the raw pooled sums e
    (LL off, gate 1): default (LL before SE) x = s_g * LL(e); ll_after_se x = LL(s_g * e). LL is pinned
    by its own closed forms (P-1). A swapped order, or LL applied twice / not at all, fails one side."""
    sch, p_id, batch = small_case("paper", R=2, n_ads=(7, 4), se="identity", cap=2000)
    raw = oracle.features(oracle.Model(sch, p_id, linear_log=False), batch)   # x = e (s = 1 exactly)
    assert np.abs(raw).max() > 1.5 and np.abs(raw).min() < 1.0   # both LL branches are hit
    b = np.linspace(-2.0, 1.5, sch.M)
    s = np.array([oracle.sigmoid(x) for x in b])
    assert np.all(np.abs(s - 1.0) > 0.1)
    params = coldgen.Params(tables=p_id.tables, table_dtype=p_id.table_dtype, se_w=np.zeros_like(p_id.se_w),
                            se_b=b, fc_w=p_id.fc_w, fc_b=p_id.fc_b, precision=p_id.precision, init=p_id.init,
                            seed=p_id.seed)
    k = sch.k
    scol = np.repeat(s, k)[None, :]
    ll = np.vectorize(oracle.linear_log)
    default = oracle.features(oracle.Model(sch, params), batch)
    after = oracle.features(oracle.Model(sch, params, ll_after_se=True), batch)
    np.testing.assert_allclose(default, scol * ll(raw), rtol=1e-14, atol=1e-300)
    np.testing.assert_allclose(after, ll(scol * raw), rtol=1e-14, atol=1e-300)
    assert np.abs(default - after).max() > 1e-3                               # the orders really differ


def test_pooled_f32_mode():
    """fp32-ordered gather: single ids are exact copies; pooled sums equal a sequential
    float32 sum over the twin's rows in bag order."""
    sch = bag_schema()
    params = coldgen.make_params(sch, seed=4, precision="f32")
    batch = coldgen.make_batch(sch, 2, [5, 4], seed=14)
    m = oracle.Model(sch, params)
    got = oracle.pooled_f32(m, batch)
    for r in range(batch.R):
        for a in range(batch.ad_offsets[r], batch.ad_offsets[r + 1]):
            for g in range(sch.M):
                acc = np.zeros(sch.k, np.float32)
                for row in mini.rows(sch, batch, g, r, a):
                    acc = (acc + params.tables[g][row]).astype(np.float32)
                np.testing.assert_array_equal(got[a, g], acc)


def test_id_out_of_range_raises():
    sch, params, batch = small_case("tiny", R=1, n_ads=(4,))
    batch.ids[3][2] = sch.groups[3].card
    with pytest.raises(oracle.OracleError) as e:
        oracle.score(oracle.Model(sch, params), batch)
    assert e.value.code == oracle.ORC_ERR_ID_RANGE


# ---- top-K ---------------------------------------------------------------------

def test_topk_brute_force_ties_nan():
    rng = np.random.default_rng(1)
    for n in (1, 2, 7, 100, 1000):
        keys = np.round(rng.random(n), 2)                 # many ties
        keys[rng.random(n) < 0.05] = np.nan
        for K in sorted({1, max(1, n // 3), n}):
            idx, kv = oracle.topk(keys, K)
            want = mini.topk(list(keys), K)
            assert idx.tolist() == want
            assert all((math.isnan(a) and math.isnan(b)) or a == b for a, b in zip(kv, keys[want]))
    with pytest.raises(oracle.OracleError):
        oracle.topk(np.zeros(5), 6)
    with pytest.raises(oracle.OracleError):
        oracle.topk(np.zeros(5), 0)


def test_ecpm_key():
    """eCPM = pCTR * bid (PAPER.md L155 footnote, L332) reorders the top-K."""
    p = np.array([0.5, 0.1, 0.3])
    bid = np.array([1.0, 10.0, 1.0])
    assert oracle.topk(p, 1)[0][0] == 0
    assert oracle.topk(p * bid, 1)[0][0] == 1


# ---- F4: the vector-product based model COLD is compared with -------------

def test_vps_worked_example():
    gd = load_golden("vps_example.json")
    p = oracle.vps_score(np.asarray(gd["ad_table"], np.float32), "f32", np.asarray(gd["user_vecs"]),
                         gd["ad_offsets"], gd["ad_ids"])
    np.testing.assert_allclose(p, gd["expected_p"], rtol=1e-15)


def test_vps_closed_forms():
    """Orthogonal vectors score sigma(0) = 1/2; v_a = c v_u scores sigma(c |v_u|^2); 16-bit storage of
    exactly representable values equals fp32 storage; ids out of range raise."""
    u = np.array([[1.0, -2.0, 0.5, 4.0]])
    tab = np.array([[2.0, 1.0, 0.0, 0.0], [0.5, -1.0, 0.25, 2.0], [-1, 2, -0.5, -4]], np.float32)
    p = oracle.vps_score(tab, "f32", u, [0, 3], [0, 1, 2])
    sq = float((u[0] ** 2).sum())
    np.testing.assert_allclose(p, [0.5, 1 / (1 + math.exp(-0.5 * sq)), 1 / (1 + math.exp(sq))], rtol=1e-15)
    p16 = oracle.vps_score(tab.astype(np.float16).view(np.uint16), "f16", u, [0, 3], [0, 1, 2])
    np.testing.assert_array_equal(p16, p)
    with pytest.raises(oracle.OracleError):
        oracle.vps_score(tab, "f32", u, [0, 1], [3])


# ---- F2: batch norm of the network input (P:276's alternative to linear_log) ----------

def test_input_norm_folds_into_fc1():
    """x <- x * scale + shift before FC1 equals FC1 with W1' = W1 diag(scale), b1' = b1 + W1 shift (an
    algebraic invariant between two parameterisations of the oracle); identity scale/shift is a no-op."""
    sch, params, batch = small_case("paper", R=2, n_ads=(17, 9), precision="f32", cap=3000, seed=12)
    rng = np.random.default_rng(3)
    d = params.fc_w[0].shape[1]
    scale, shift = rng.uniform(0.2, 1.5, d), rng.uniform(-0.5, 0.5, d)
    p_bn, _ = oracle.score(oracle.Model(sch, params, linear_log=False, in_norm=(scale, shift)), batch)
    W1 = np.asarray(params.fc_w[0], np.float64)
    folded = dataclasses.replace(params, fc_w=[W1 * scale[None, :]] + list(params.fc_w[1:]),
                                 fc_b=[np.asarray(params.fc_b[0], np.float64) + W1 @ shift] + list(params.fc_b[1:]))
    p_fold, _ = oracle.score(oracle.Model(sch, folded, linear_log=False), batch)
    np.testing.assert_allclose(p_bn, p_fold, rtol=1e-11)
    p_id, _ = oracle.score(oracle.Model(sch, params, in_norm=(np.ones(d), np.zeros(d))), batch)
    p_none, _ = oracle.score(oracle.Model(sch, params), batch)
    np.testing.assert_array_equal(p_id, p_none)


# ---- F2 PReLU hidden activation (the paper never names the activation, AMB-6) ----

def _prelu_torch_reference(sch, params, batch, slopes):
    """LL off, SE pinned to s = 1: MLP(concat(embedding_bag_sum)) with torch's F.prelu between layers."""
    import torch
    import torch.nn.functional as F
    feats = []
    for g, grp in enumerate(sch.groups):
        bags = []
        for r in range(batch.R):
            for a in range(batch.ad_offsets[r], batch.ad_offsets[r + 1]):
                bags.append(mini.rows(sch, batch, g, r, a))
        flat = torch.tensor([x for b in bags for x in b], dtype=torch.long)
        offs = torch.tensor(np.cumsum([0] + [len(b) for b in bags[:-1]]), dtype=torch.long)
        feats.append(F.embedding_bag(flat, torch.tensor(params.table_f64(g)), offs, mode="sum"))
    h = torch.cat(feats, 1)
    L = len(params.fc_w)
    for l in range(L):
        h = F.linear(h, torch.tensor(params.fc_w[l], dtype=torch.float64), torch.tensor(params.fc_b[l], dtype=torch.float64))
        if l < L - 1:
            h = F.prelu(h, torch.tensor(np.asarray(slopes[l], np.float64)))
    return (h[:, 0] if h.shape[1] == 1 else h[:, 1] - h[:, 0]).numpy()


def test_prelu_reduces_to_torch_prelu_mlp():
    """P-6 style reduction with the PReLU variant: the oracle equals torch's embedding_bag + linear +
    F.prelu (per-channel slopes) + sigmoid; a slope applied to the wrong channel or layer fails it."""
    pytest.importorskip("torch")
    sch, params, batch = small_case("tiny", R=3, n_ads=(6, 11, 2), precision="f32", se="identity")
    slopes = coldgen.prelu_slopes(sch, seed=9)
    p, z = oracle.score(oracle.Model(sch, params, linear_log=False, prelu=slopes), batch)
    zt = _prelu_torch_reference(sch, params, batch, slopes)
    np.testing.assert_allclose(z, zt, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(p, 1.0 / (1.0 + np.exp(-zt)), rtol=1e-12, atol=1e-14)
    p_relu, _ = oracle.score(oracle.Model(sch, params, linear_log=False), batch)
    assert np.abs(p - p_relu).max() > 1e-4                       # the negative branch is exercised


def test_prelu_special_slopes():
    """Slope 0 is ReLU exactly; slope 1 makes every hidden layer the identity, so the network is the
    affine map z = W_L (... (W_1 x + b_1) ...) + b_L of the (separately pinned) features x."""
    sch, params, batch = small_case("paper", R=2, n_ads=(5, 3), precision="f32", cap=2000, seed=13)
    m_relu = oracle.Model(sch, params)
    p_relu, z_relu = oracle.score(m_relu, batch)
    zeros = [np.zeros(w.shape[0]) for w in params.fc_w[:-1]]
    p0, z0 = oracle.score(oracle.Model(sch, params, prelu=zeros), batch)
    np.testing.assert_array_equal(z0, z_relu)
    ones = [np.ones(w.shape[0]) for w in params.fc_w[:-1]]
    _, z1 = oracle.score(oracle.Model(sch, params, prelu=ones), batch)
    h = oracle.features(m_relu, batch).T
    for W, b in zip(params.fc_w, params.fc_b):
        h = W.astype(np.float64) @ h + b.astype(np.float64)[:, None]
    za = h[1] - h[0] if h.shape[0] == 2 else h[0]
    np.testing.assert_allclose(z1, za, rtol=1e-10, atol=1e-12)


def test_prelu_c_oracle_matches_python_twin():
    sch, params, batch = small_case("tiny", R=2, n_ads=(7, 5), seed=17)
    slopes = coldgen.prelu_slopes(sch, seed=18)
    p, z = oracle.score(oracle.Model(sch, params, prelu=slopes), batch)
    pm, zm = mini.score(sch, params, batch, prelu=slopes)
    np.testing.assert_allclose(p, pm, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(z, zm, rtol=1e-13, atol=1e-14)
