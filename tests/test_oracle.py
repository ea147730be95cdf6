"""Pins of the CPU oracle against the paper and against mathematics (not against itself).

Each test names what fixes the expected value: a value printed in PAPER.md (golden fixture), a
closed form, an invariant the paper states, a textbook routine, or brute force on tiny inputs.
"""
import json
import os

import numpy as np
import pytest

from oracle import bbc_oracle as O
from oracle import bruteforce as BF

GOLD = os.path.join(os.path.dirname(__file__), "golden")
F32 = np.float32


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- values printed in the paper
def test_fig3_walkthrough():
    """tau 5 -> 4 and relaxed threshold 6 -> 5 when object 9 (4.9) arrives.
    Also pins the Update comparison as '>=' (Alg. 1 l.9 prints 's > k', reading R1)."""
    g = _gold("fig3_walkthrough.json")
    rb = O.ResultBuffer(g["codebook"])
    for oid, dist in g["objects"]:
        rb.push(oid, dist)
    rb.tau = rb.update(g["k"])
    assert rb.tau == g["expect_tau_before"]
    assert rb.relaxed_threshold() == g["expect_relaxed_threshold_before"]
    oid, dist = g["insert"]
    assert rb.bucket(dist) == g["expect_bucket_of_insert"]
    rb.push(oid, dist)
    rb.tau = rb.update(g["k"])
    assert rb.tau == g["expect_tau_after"]
    assert rb.relaxed_threshold() == g["expect_relaxed_threshold_after"]
    # Collect returns the exact top-k of what was pushed
    allp = sorted([(d, i) for i, d in g["objects"]] + [(dist, oid)])
    assert sorted(rb.collect(g["k"])) == allp[: g["k"]]


def test_fig3_strict_reading_contradicts_text():
    """Under the literal 's > k' the threshold before the insert would be infinity, which the
    text (bucket 5 is the threshold bucket) rules out -- the reason for reading R1."""
    g = _gold("fig3_walkthrough.json")
    counts = np.zeros(9, int)
    for _, dist in g["objects"]:
        counts[int(dist)] += 1
    cum = np.cumsum(counts)
    assert not np.any(cum > g["k"])                       # '>' never fires: tau = inf
    assert int(np.flatnonzero(cum >= g["k"])[0]) == g["expect_tau_before"]


def test_eq3_bucket_counts():
    g = _gold("eq3_num_buckets.json")
    for c in g["cases"]:
        m = O.eq3_num_buckets(c["d"], c["d"] // 4, g["bits"], g["l1_bytes"])
        assert m == c["m"], c
    nd = g["not_pinned"]
    assert O.eq3_num_buckets(nd["d"], nd["d"] // 4, g["bits"], g["l1_bytes"]) == nd["eq3_gives"]


# ---------------------------------------------------------------- O1 coarse probe
def test_coarse_d2_matches_fp64(rng):
    Q = rng.standard_normal((7, 33)).astype(F32)
    C = rng.standard_normal((50, 33)).astype(F32)
    d = O.coarse_d2(Q, C)
    ref = ((Q[:, None, :].astype(np.float64) - C[None].astype(np.float64)) ** 2).sum(2)
    np.testing.assert_allclose(d, ref, rtol=1e-5)


def test_probe_is_textbook_sort_and_prefix_monotone(rng):
    Q = rng.standard_normal((5, 16)).astype(F32)
    C = rng.standard_normal((40, 16)).astype(F32)
    C[7] = C[3]                                         # exact tie: smaller id first
    d = O.coarse_d2(Q, C)
    pr, rq = O.probe(Q, C, 40)
    for i in range(5):
        ref = sorted(range(40), key=lambda j: (float(d[i, j]), j))
        assert list(pr[i]) == ref
        assert np.all(np.diff(rq[i]) >= 0)
    p10, _ = O.probe(Q, C, 10)
    assert np.array_equal(p10, pr[:, :10])


# ---------------------------------------------------------------- O2/O3 PQ
def test_lut_identity(c1t):
    """sum_m LUT[m][code_m] == ||q - decode(code)||^2."""
    cfg, ix, Q, _ = c1t
    books = np.asarray(ix["codebooks"])
    codes = np.asarray(ix["codes"][:500])
    for q in Q[:3]:
        est = O.pq_est(O.pq_lut(q, books), codes)
        dec = np.concatenate([books[m][codes[:, m]] for m in range(books.shape[0])], axis=1)
        ref = ((dec.astype(np.float64) - q.astype(np.float64)) ** 2).sum(1)
        np.testing.assert_allclose(est, ref, rtol=1e-5)


def test_pq_est_zero_at_decoded_query(c1t):
    """q = decode(c) makes every LUT term (q_t - C_t)^2 exactly 0."""
    cfg, ix, Q, _ = c1t
    books = np.asarray(ix["codebooks"])
    code = np.asarray(ix["codes"][17:18])
    q = np.concatenate([books[m][code[0, m]] for m in range(books.shape[0])])
    assert O.pq_est(O.pq_lut(q, books), code)[0] == 0.0


# ---------------------------------------------------------------- O4-O8 result buffer
def _probed_est(ix, q, nprobe):
    pr, rq = O.probe(q[None], ix["centroids"], nprobe)
    off = np.asarray(ix["list_offsets"])
    lut = O.pq_lut(q, np.asarray(ix["codebooks"]))
    sizes = off[pr[0] + 1] - off[pr[0]]
    pos = np.concatenate([np.arange(off[L], off[L + 1]) for L in pr[0]])
    return O.pq_est(lut, np.asarray(ix["codes"][pos])), sizes, pos


def test_cells_monotone_and_clamped(rng):
    x = np.sort(rng.uniform(-1, 12, 200_000).astype(F32))
    c = O.cells(x, F32(0.5), F32(9.25))
    assert np.all(np.diff(c) >= 0)
    assert c.min() == 0 and c.max() == 255
    assert np.all(c[x > F32(9.25)] == 255) and np.all(c[x <= F32(9.25)] <= 254)
    assert np.all(c[x < F32(0.5)] == 0)
    assert np.all(O.cells(x, F32(3.0), F32(3.0))[x <= 3.0] == 0)


def test_threshold_invariants(c1t):
    """tau = cell(budget-th smallest estimate) (closed form; cell() is monotone), and
    sum_{c<tau} H < budget <= sum_{c<=tau} H (Alg. 1 Update)."""
    cfg, ix, Q, _ = c1t
    for q in Q[:4]:
        est, sizes, _ = _probed_est(ix, q, cfg.nprobe)
        budget = cfg.budget
        s = O.sample_lists(sizes, budget)
        ns = int(sizes[:s].sum())
        dmin, dmax = O.edges(est[:ns], budget)
        c = O.cells(est, dmin, dmax)
        H = np.bincount(c, minlength=256)
        tau = O.threshold(H, budget)
        kth = np.sort(est)[budget - 1]
        assert tau == O.cells(np.array([kth]), dmin, dmax)[0]
        assert H[:tau].sum() < budget <= H[: tau + 1].sum()
        assert tau <= 254


def test_sample_and_edges(c1t):
    """d_max >= the budget-th smallest estimate over everything probed (P:L899's claim), d_min is
    the sample minimum, and the sample is the shortest probe-order prefix of >= min(8, nprobe)
    lists holding >= budget objects (reading R5)."""
    cfg, ix, Q, _ = c1t
    for q in Q[:4]:
        for nprobe, budget in ((cfg.nprobe, cfg.budget), (cfg.nlist, 2 * cfg.budget), (12, 350)):
            est, sizes, _ = _probed_est(ix, q, nprobe)
            s = O.sample_lists(sizes, budget)
            if sizes.sum() <= budget:
                assert s == 0
                continue
            assert s >= min(8, nprobe) and sizes[:s].sum() >= budget
            if s > min(8, nprobe):
                assert sizes[: s - 1].sum() < budget
            ns = int(sizes[:s].sum())
            dmin, dmax = O.edges(est[:ns], budget)
            assert dmin == est[:ns].min()
            assert dmax >= np.sort(est)[budget - 1]
            assert dmax == np.sort(est[:ns])[budget - 1]


def test_superset_invariants(c1t):
    """|S*| >= budget; S* contains the top-budget by estimate; every member lies at or below the
    threshold bucket's upper edge (BASELINE.json north_star invariants); threshold gap small
    (Exp-4: 'on the order of 1e-2 or smaller')."""
    cfg, ix, Q, _ = c1t
    for q in Q:
        est, sizes, _ = _probed_est(ix, q, 16)
        budget = cfg.budget
        s = O.sample_lists(sizes, budget)
        ns = int(sizes[:s].sum())
        dmin, dmax = O.edges(est[:ns], budget)
        c = O.cells(est, dmin, dmax)
        tau = O.threshold(np.bincount(c, minlength=256), budget)
        sup = np.flatnonzero(c <= tau)
        assert len(sup) >= budget
        top = np.lexsort((np.arange(len(est)), est))[:budget]
        assert set(top) <= set(sup)
        upper = float(dmin) + (tau + 1) * (float(dmax) - float(dmin)) / 255.0
        assert np.all(est[sup].astype(np.float64) <= upper * (1 + 1e-6))
        kth = float(np.sort(est)[budget - 1])
        assert (upper - kth) / kth <= 5e-2


def test_alg1_literal_equals_one_shot(c1t):
    """Alg. 1 run cluster by cluster (Push drops j > tau, Update after every cluster) keeps
    exactly the one-shot superset {cell <= tau_final} (reading R17)."""
    cfg, ix, Q, _ = c1t
    est, sizes, _ = _probed_est(ix, Q[0], 16)
    budget = 900
    s = O.sample_lists(sizes, budget)
    dmin, dmax = O.edges(est[: int(sizes[:s].sum())], budget)
    c = O.cells(est, dmin, dmax)
    tau = O.threshold(np.bincount(c, minlength=256), budget)
    rb = O.ResultBuffer(np.arange(1, 258))            # bucket j = [j, j+1) holds cell j-1
    pos = 0
    for n in sizes:
        for i in range(pos, pos + n):
            rb.push(i, float(c[i]) + 1.5)
        rb.tau = rb.update(budget)
        pos += n
    assert rb.tau - 1 == tau
    kept = {oid for j in range(1, rb.tau + 1) for _, oid in rb.B[j]}
    assert kept == set(np.flatnonzero(c <= tau))


# ---------------------------------------------------------------- O9
def test_exact_d2_and_select_textbook(rng):
    q = rng.standard_normal(40).astype(F32)
    X = rng.standard_normal((300, 40)).astype(F32)
    d = O.exact_d2(q, X)
    ref = np.linalg.norm(X.astype(np.float64) - q.astype(np.float64), axis=1) ** 2
    np.testing.assert_allclose(d, ref, rtol=1e-6)
    ids = rng.permutation(1000)[:300].astype(np.int64)
    d[5] = d[9]                                           # a tie: smaller id first
    oi, od = O.select_topk(d, ids, 50)
    ref = sorted(zip(d.tolist(), ids.tolist()))[:50]
    assert list(oi) == [r[1] for r in ref]
    oi, od = O.select_topk(d[:3], ids[:3], 5)             # short: padded
    assert list(oi[3:]) == [-1, -1] and np.all(np.isinf(od[3:]))


def test_u8_exact_distances_are_integers(rng):
    q = rng.integers(0, 256, 128).astype(F32)
    X = rng.integers(0, 256, (100, 128)).astype(np.uint8)
    d = O.exact_d2(q, X)
    ref = ((X.astype(np.int64) - q.astype(np.int64)) ** 2).sum(1)
    assert np.array_equal(d.astype(np.int64), ref)


# ---------------------------------------------------------------- end to end
def test_full_probe_unlimited_budget_is_brute_force(c1t):
    """nprobe = nlist and budget >= N reproduce brute force exactly (BASELINE.json north_star)."""
    cfg, ix, Q, _ = c1t
    raw = np.asarray(ix["raw"])
    X = np.empty_like(raw)
    X[np.asarray(ix["ids"])] = raw
    ids, d2 = O.search(ix, Q[:4], cfg.k, cfg.nlist, cfg.N)
    gi, gd = BF.ground_truth(Q[:4], X, cfg.k)
    assert np.array_equal(ids, gi)
    np.testing.assert_allclose(d2, gd, rtol=1e-6)


def test_tiny_brute_force_all_parameters(rng):
    """Tiny index built by the builder: with every list probed and budget >= N the result is the
    brute-force top-k for every k."""
    import datagen
    from datagen import build_index, configs
    cfg = configs.get("C1t").replace(name="tiny", N=700, nlist=8, nq=3, k=20, nprobe=8, budget=700,
                                     M=8, kmeans_iters=3, pq_train=700, pq_iters=3)
    from datagen import synth
    X = synth.generate_data(cfg)
    ix = build_index.build(cfg, X=X)
    Q = synth.generate_queries(cfg)
    for k in (1, 7, 20, 700):
        ids, d2 = O.search(ix, Q, k, cfg.nlist, max(k, cfg.N))
        gi, gd = BF.ground_truth(Q, X, k)
        assert np.array_equal(ids, gi)


def test_short_results_padded(c1t):
    cfg, ix, Q, _ = c1t
    off = np.asarray(ix["list_offsets"])
    ids, d2, dbg = O.search(ix, Q[:2], 5000, 1, 5000, want_debug=True)
    for i in range(2):
        n_o = dbg[i]["n_o"]
        assert dbg[i]["tau"] == O.TAU_INF and n_o < 5000
        assert np.all(ids[i, n_o:] == -1) and np.all(np.isinf(d2[i, n_o:]))
        assert len(set(ids[i, :n_o])) == n_o


def test_recall_and_relative_error_hand_examples():
    gt = np.array([[1, 2, 3, 4]])
    gd = np.array([[1.0, 4.0, 9.0, 16.0]])
    res = np.array([[1, 2, 9, 8]])
    rd = np.array([[1.0, 4.0, 16.0, 25.0]])
    assert BF.recall(res, rd, gt, gd) == 0.75              # id 9 ties the 4th GT distance
    assert abs(BF.relative_error(np.array([[1.0, 4.0, 9.0, 16.0 * 1.1025]]), gd) - 0.0125) < 1e-12


# ---------------------------------------------------------------- RaBitQ
def test_rabitq_estimator_bound_and_closed_form(c3s):
    """<x_bar, q'> from (c1, c2, c3) equals sum_i x_bar_i * (v_l + delta * qbar_i) exactly (up to
    fp32 rounding), and differs from <x_bar, q'> by at most sqrt(D)*delta/2 (the 4-bit query
    quantisation bound); q = a database vector gives est d^2 within that bound of 0."""
    cfg, ix, Q, _ = c3s
    off = np.asarray(ix["list_offsets"])
    P = np.asarray(ix["P"])
    D = P.shape[0]
    L = 5
    sl = slice(off[L], off[L + 1])
    bits = np.asarray(ix["bits"][sl])
    fac = np.asarray(ix["factors"][sl])
    raw = np.asarray(ix["raw"][sl])
    b = np.unpackbits(bits, axis=1, bitorder="little").astype(np.float64)
    xbar = (2 * b - 1) / np.sqrt(D)
    for q in (Q[0], raw[3]):
        rq2 = O.coarse_d2(q[None], np.asarray(ix["centroids"][L:L + 1]))[0, 0]
        u = O.rabitq_rotate(q, P)
        qbar, (c1, c2, c3), r = O.rabitq_query_code(u, np.asarray(ix["wL"][L]), rq2)
        qp = (u.astype(np.float64) - ix["wL"][L]) / float(r)
        vl = qp.min()
        delta = (qp.max() - vl) / 15
        ip = (b * qbar).sum(1)
        est_ip = c1 * ip + c2 * b.sum(1) + c3
        deq = (xbar * (vl + delta * qbar)).sum(1)
        np.testing.assert_allclose(est_ip, deq, atol=1e-4)
        exact_ip = xbar @ qp
        assert np.all(np.abs(est_ip - exact_ip) <= np.sqrt(D) * delta / 2 + 1e-5)
    # q = raw[3]: true d^2 = 0 for that object
    est = O.rabitq_est(bits, fac, qbar, (c1, c2, c3), r, rq2)
    ro, go = float(fac[3, 0]), float(fac[3, 1])
    bound = 2 * ro * float(r) * (np.sqrt(D) * delta / 2 + 1e-5) / go
    assert abs(float(est[3])) <= bound + 1e-3


def test_rabitq_factors_and_unbiased(c3s):
    """g_o in (0, 1], mean ~ sqrt(2/pi) (RaBitQ), rotation orthogonal; the estimator of <o, q>
    is unbiased and its error is covered by eps0 * sqrt((1-g^2)/g^2)/sqrt(D-1) for most pairs
    with eps0 = 1.9."""
    cfg, ix, Q, _ = c3s
    P = np.asarray(ix["P"]).astype(np.float64)
    assert np.abs(P.T @ P - np.eye(len(P))).max() < 1e-5
    fac = np.asarray(ix["factors"])
    assert np.all(fac[:, 1] > 0) and np.all(fac[:, 1] <= 1.0 + 1e-6)
    assert abs(fac[:, 1].mean() - np.sqrt(2 / np.pi)) < 0.02
    off = np.asarray(ix["list_offsets"])
    D = P.shape[0]
    errs, cover = [], []
    for qi in range(6):
        q = Q[qi]
        for L in range(0, 40, 3):
            sl = slice(off[L], off[L + 1])
            c = np.asarray(ix["centroids"][L])
            rq2 = O.coarse_d2(q[None], c[None])[0, 0]
            u = O.rabitq_rotate(q, np.asarray(ix["P"]))
            qbar, cs, r = O.rabitq_query_code(u, np.asarray(ix["wL"][L]), rq2)
            est = O.rabitq_est(np.asarray(ix["bits"][sl]), np.asarray(ix["factors"][sl]), qbar, cs,
                               r, rq2).astype(np.float64)
            raw = np.asarray(ix["raw"][sl]).astype(np.float64)
            ro = fac[sl, 0].astype(np.float64)
            g = fac[sl, 1].astype(np.float64)
            true_ip = ((raw - c) @ (q - c)) / (ro * np.sqrt(rq2))
            est_ip = (ro ** 2 + rq2 - est) / (2 * ro * np.sqrt(rq2))
            errs.append(est_ip - true_ip)
            cover.append(np.abs(est_ip - true_ip) <= 1.9 * np.sqrt((1 - g * g) / (g * g)) / np.sqrt(D - 1))
    e = np.concatenate(errs)
    assert abs(e.mean()) < 3 * e.std() / np.sqrt(len(e)) + 2e-3
    assert np.concatenate(cover).mean() > 0.85


def test_rabitq_full_probe_is_brute_force(c3s):
    cfg, ix, Q, _ = c3s
    raw = np.asarray(ix["raw"])
    X = np.empty_like(raw)
    X[np.asarray(ix["ids"])] = raw
    ids, d2 = O.search(ix, Q[:2], 50, cfg.nlist, cfg.N)
    gi, gd = BF.ground_truth(Q[:2], X, 50)
    assert np.array_equal(ids, gi)


# ---------------------------------------------------------------- f4 inner-product metric
def _tiny_ip(n=900, nlist=8, M=8):
    """Tiny unit-norm (cosine = inner product) PQ index from the C4 generator, IP metric."""
    from datagen import build_index, configs, synth
    cfg = configs.get("C4ip_s").replace(name="tiny_ip", N=n, nlist=nlist, nq=3, k=20, nprobe=nlist,
                                        budget=n, M=M, kmeans_iters=3, pq_train=n, pq_iters=3)
    X = synth.generate_data(cfg)
    ix = build_index.build(cfg, X=X)
    return cfg, ix, X, synth.generate_queries(cfg)


def test_ip_lut_identity_and_probe_sort():
    """Inner product: sum_m LUT[m][code_m] == -<q, decode(code)> (fp64 within
    fp32 rounding) and the probe order is the textbook sort of -<q, c_j> with ties by id."""
    cfg, ix, X, Q = _tiny_ip()
    books = np.asarray(ix["codebooks"])
    codes = np.asarray(ix["codes"])
    for q in Q:
        est = O.pq_est(O.pq_lut(q, books, "ip"), codes)
        dec = np.concatenate([books[m][codes[:, m]] for m in range(books.shape[0])], axis=1)
        ref = -(dec.astype(np.float64) @ q.astype(np.float64))
        np.testing.assert_allclose(est, ref, rtol=1e-5, atol=1e-6)
    C = np.asarray(ix["centroids"])
    pr, rq = O.probe(Q, C, cfg.nlist, "ip")
    sim = Q.astype(np.float64) @ C.astype(np.float64).T
    for i in range(len(Q)):
        np.testing.assert_allclose(rq[i], -sim[i][pr[i]], rtol=1e-5, atol=1e-6)
        assert np.all(np.diff(rq[i]) >= 0)


def test_ip_full_probe_is_brute_force_mips():
    """IP index, every list probed, budget >= N: the result is the brute-force maximum inner
    product top-k for every k (keys -<q, x>, ties by id)."""
    cfg, ix, X, Q = _tiny_ip()
    for k in (1, 7, 20, cfg.N):
        ids, key = O.search(ix, Q, k, cfg.nlist, max(k, cfg.N))
        gi, gd = BF.ground_truth(Q, X, k, metric="ip")
        assert np.array_equal(ids, gi)
        np.testing.assert_allclose(key, gd, rtol=1e-5, atol=1e-6)


def test_ip_index_file_roundtrip(tmp_path):
    from datagen import index_file
    cfg, ix, X, Q = _tiny_ip(n=300, nlist=4)
    p = str(tmp_path / "ip.bbcivf")
    index_file.write(p, ix)
    back = index_file.read(p, mmap=False)
    assert back["metric"] == "ip"
    a, _ = O.search(ix, Q, 5, 4, 300)
    b, _ = O.search(back, Q, 5, 4, 300)
    assert np.array_equal(a, b)


def test_bucket_count_closed_forms(c1t):
    """B regular buckets (Eq. 6): B = 1 puts every object <= d_max in bucket 0, so tau = 0 and
    S* = {est <= d_max}; for every B, tau is the bucket of the budget-th smallest estimate and the
    superset shrinks (weakly) as the grid refines by doubling within rounding."""
    cfg, ix, Q, _ = c1t
    q = Q[0]
    est, sizes, pos = _probed_est(ix, q, cfg.nprobe)
    s = O.sample_lists(sizes, cfg.budget)
    dmin, dmax = O.edges(est[: int(sizes[:s].sum())], cfg.budget)
    c1 = O.cells(est, dmin, dmax, 1)
    assert set(np.unique(c1)) <= {0, 255}
    assert np.array_equal(c1 == 0, ~(est > dmax))
    assert O.threshold(np.bincount(c1, minlength=256), cfg.budget) == 0
    kth = np.sort(est)[cfg.budget - 1]
    sizes_S = []
    for B in (1, 2, 4, 8, 16, 32, 64, 128, 255):
        c = O.cells(est, dmin, dmax, B)
        tau = O.threshold(np.bincount(c, minlength=256), cfg.budget)
        assert tau == O.cells(np.array([kth], dtype=np.float32), dmin, dmax, B)[0]
        sizes_S.append(int(np.count_nonzero(c <= tau)))
        assert sizes_S[-1] >= cfg.budget
    assert all(a >= b - 2 for a, b in zip(sizes_S[:-2], sizes_S[1:-1]))   # doubling B: nested up to rounding
    with pytest.raises(ValueError):
        O.cells(est, dmin, dmax, 0)


# ---------------------------------------------------------------------------------------------
# 4-bit PQ ("M = d/4 ... 4 bits per sub-vector"; FastScan P:L1798):
# the 8-bit quantised lookup table and its estimate (reading R20)
# ---------------------------------------------------------------------------------------------
def test_pq4_lut_hand_example():
    """A 2 x 16 LUT worked by hand: row 0 spans [1, 3.55] (span 2.55, the largest), row 1 is
    [10, 10.51].  delta = 2.55 / 255 = 0.01; row 0 maps 1 + 0.01 c' to c', row 1's 10.51 to 51."""
    lut = np.full((2, 16), 0.0, dtype=np.float32)
    lut[0] = np.float32(1.0) + np.float32(0.17) * np.arange(16, dtype=np.float32)   # 1 .. 3.55
    lut[1] = np.float32(10.0)
    lut[1][7] = np.float32(10.51)
    Q, delta, bias = O.pq4_fastscan_lut(lut)
    assert abs(float(delta) - 0.01) < 1e-8
    assert abs(float(bias) - 11.0) < 1e-6
    assert list(Q[0]) == [17 * c for c in range(16)]      # 0.17 c / 0.01 = 17 c
    assert Q[1][7] == 51 and Q[1].sum() == 51
    est = O.pq4_est(Q, delta, bias, np.array([[15, 7], [0, 0]]))
    assert abs(float(est[0]) - (3.55 + 10.51)) < 1e-5 and abs(float(est[1]) - 11.0) < 1e-6


def test_pq4_lut_invariants_and_error_bound(rng):
    """Row minima map to 0, the widest row's maximum to 255, every entry dequantises to within
    delta/2 of the fp32 LUT, and the estimate is within M*delta/2 (+ rounding) of pq_est."""
    for trial in range(20):
        M = int(rng.integers(1, 40))
        lut = (rng.random((M, 16)) * rng.random() * 50 + rng.normal() * 10).astype(np.float32)
        Q, delta, bias = O.pq4_fastscan_lut(lut)
        lo = lut.min(axis=1)
        assert np.all(Q.min(axis=1) == 0)
        assert Q.max() == 255
        deq = lo[:, None].astype(np.float64) + float(delta) * Q.astype(np.float64)
        assert np.all(np.abs(deq - lut) <= float(delta) * 0.5 * (1 + 1e-5) + 1e-6)
        codes = rng.integers(0, 16, (500, M))
        e4 = O.pq4_est(Q, delta, bias, codes).astype(np.float64)
        e = O.pq_est(lut, codes).astype(np.float64)
        tol = M * float(delta) * 0.5 * (1 + 1e-5) + 1e-5 * (np.abs(e) + M * np.abs(lut).max())
        assert np.all(np.abs(e4 - e) <= tol)


def test_pq4_degenerate_lut():
    """All entries of every row equal: delta = 0, codes 0, the estimate is the bias exactly."""
    lut = np.tile(np.arange(5, dtype=np.float32)[:, None], (1, 16))
    Q, delta, bias = O.pq4_fastscan_lut(lut)
    assert delta == 0 and not Q.any() and bias == np.float32(10.0)
    assert np.all(O.pq4_est(Q, delta, bias, np.zeros((3, 5), dtype=int)) == np.float32(10.0))


def test_pq4_full_probe_is_brute_force(rng):
    """A tiny 4-bit PQ index from the builder: every list probed and budget >= N give the
    brute-force top-k (the estimate only decides buckets; re-rank distances are exact)."""
    from datagen import build_index, configs, synth
    cfg = configs.get("C2q4s").replace(name="tiny_q4", N=800, nlist=8, nq=3, k=25, nprobe=8,
                                      budget=800, kmeans_iters=3, pq_train=800, pq_iters=3)
    X = synth.generate_data(cfg)
    ix = build_index.build(cfg, X=X)
    assert ix["nbits"] == 4 and ix["codebooks"].shape == (cfg.M, 16, cfg.d // cfg.M)
    assert int(np.asarray(ix["codes"]).max()) <= 15
    Q = synth.generate_queries(cfg)
    for k in (1, 25):
        ids, d2 = O.search(ix, Q, k, cfg.nlist, cfg.N)
        gi, gd = BF.ground_truth(Q, X, k)
        assert np.array_equal(ids, gi)


# ---------------------------------------------------------------------------------------------
# n_ew -> m equal-depth remap (Eq. 6 with map P:L922-932; reading R6)
# ---------------------------------------------------------------------------------------------
def test_equal_depth_map_hand_example():
    """Sample histogram 4, 0, 2, 2 (T = 8) into m = 2 buckets: the first bucket closes after
    cell 0 (4 of 8 = half); cells 1..254 form the second; the overflow cell stays 255."""
    H0 = np.zeros(256, dtype=np.int64)
    H0[:4] = [4, 0, 2, 2]
    mp = O.equal_depth_map(H0, 2)
    assert mp[0] == 0 and np.all(mp[1:255] == 1) and mp[255] == 255
    # m = 4: bucket b closes at the first cell where the running count reaches 2 (b + 1),
    # at most one bucket per cell: after cells 0 (4), 1 (4), 2 (6)
    mp4 = O.equal_depth_map(H0, 4)
    assert list(mp4[:5]) == [0, 1, 2, 3, 3]


def test_equal_depth_map_invariants(rng):
    """Nondecreasing, starts at 0, at most m buckets, and every bucket but the last closes as
    soon as the running sample count reaches its share (the greedy equal-depth rule)."""
    for trial in range(30):
        H0 = np.zeros(256, dtype=np.int64)
        nz = rng.integers(1, 255)
        H0[:255] = rng.integers(0, 50, 255) * (rng.random(255) < nz / 255)
        H0[0] += 1
        m = int(rng.integers(1, 60))
        mp = O.equal_depth_map(H0, m)
        assert mp[0] == 0 and np.all(np.diff(mp[:255]) >= 0) and mp[:255].max() <= m - 1
        assert np.all(np.diff(mp[:255]) <= 1)
        T = H0[:255].sum()
        run = np.cumsum(H0[:255])
        for c in range(1, 255):
            if mp[c] > mp[c - 1]:                      # bucket mp[c-1] closed after cell c-1
                assert run[c - 1] * m >= (mp[c - 1] + 1) * T
                assert c - 1 == 0 or mp[c - 2] < mp[c - 1] or run[c - 2] * m < (mp[c - 1] + 1) * T


def test_remap_identity_reduces_to_threshold(rng):
    """One sample object per cell and m = 255: the map is the identity, so the remapped
    threshold is the equal-width one."""
    H0 = np.zeros(256, dtype=np.int64)
    H0[:255] = 1
    mp = O.equal_depth_map(H0, 255)
    assert np.array_equal(mp[:255], np.arange(255))
    for trial in range(20):
        H = rng.integers(0, 100, 256)
        budget = int(rng.integers(1, H[:255].sum() + 50))
        assert O.remap_threshold(H, mp, budget, 255) == O.threshold(H[:255], budget)


def test_remap_superset_contains_equal_width(c1t):
    """Equal-depth buckets are unions of equal-width cells: the remapped superset contains the
    equal-width one for every m, and m = 1 takes every object within d_max."""
    cfg, ix, Q, _ = c1t
    for m in (1, 4, 16, 64):
        _, _, d0 = O.search(ix, Q[:3], cfg.k, cfg.nprobe, cfg.budget, want_debug=True)
        _, _, d1 = O.search(ix, Q[:3], cfg.k, cfg.nprobe, cfg.budget, want_debug=True, remap_m=m)
        for a, b in zip(d0, d1):
            if a["tau"] == O.TAU_INF:
                continue
            assert b["tau"] >= a["tau"]
            assert set(a["sup_pos"].tolist()) <= set(b["sup_pos"].tolist())
            if m == 1:
                assert b["tau"] == 254 and len(b["sup_pos"]) == int((b["cell"] < 255).sum())


# ---------------------------------------------------------------- f1: bound-aware RaBitQ re-rank
def _valid_bounds(rng, n, spread=0.3):
    ex = rng.uniform(1.0, 2.0, n).astype(np.float32)
    lb = (ex - spread * rng.random(n)).astype(np.float32)
    ub = (ex + spread * rng.random(n)).astype(np.float32)
    return ex, lb, ub


def test_rabitq_bounds_closed_forms_and_coverage(c3s):
    """rabitq_bounds (reading R21): lb <= est <= ub; g_o = 1 gives a zero-width interval (the
    code is the vector: no estimation error); and the interval with eps0 = 1.9 holds the
    exact d^2 for most (query, object) pairs -- the 'high probability' of P:L962."""
    cfg, ix, Q, _ = c3s
    fac = np.array([[1.5, 1.0], [2.0, 0.8], [0.5, 0.6]], dtype=np.float32)
    est = np.array([3.0, 4.0, 5.0], dtype=np.float32)
    lb, ub = O.rabitq_bounds(est, fac, np.float32(2.0), 960)
    assert lb[0] == est[0] == ub[0]
    assert np.all(lb <= est) and np.all(est <= ub)
    # hand value for object 1: delta = (2*2.0*2.0) * (sqrt(1 - 0.64)/0.8 * 1.9/sqrt(959))
    want = 8.0 * (0.6 / 0.8 * 1.9 / np.sqrt(959.0))
    assert abs(float(ub[1] - est[1]) - want) < 1e-5
    off = np.asarray(ix["list_offsets"])
    D = int(ix["D"])
    cover = []
    for qi in range(4):
        pr, rq = O.probe(Q[qi:qi + 1], np.asarray(ix["centroids"]), 6)
        u = O.rabitq_rotate(Q[qi], np.asarray(ix["P"]))
        for j, L in enumerate(pr[0]):
            sl = slice(off[L], off[L + 1])
            qbar, cs, r = O.rabitq_query_code(u, np.asarray(ix["wL"][L]), rq[0, j])
            e = O.rabitq_est(np.asarray(ix["bits"][sl]), np.asarray(ix["factors"][sl]), qbar, cs, r, rq[0, j])
            lo, hi = O.rabitq_bounds(e, np.asarray(ix["factors"][sl]), r, D)
            ex = O.exact_d2(Q[qi], np.asarray(ix["raw"][sl]))
            cover.append((ex >= lo) & (ex <= hi))
    assert np.concatenate(cover).mean() > 0.85


def test_alg2_minimal_rerank_exact_under_valid_bounds(rng):
    """Algorithm 2 with valid bounds (lb <= exact <= ub) returns the exact top-k
    and re-ranks every object of Observation 1's minimal set {[lb, ub] contains Dist_k}."""
    for n, k in ((400, 1), (400, 37), (1000, 250)):
        ex, lb, ub = _valid_bounds(rng, n)
        top, vis = O.minimal_rerank_alg2(lb, ub, lambda i: ex[i], k)
        want = sorted(np.argsort(ex, kind="stable")[:k].tolist())
        assert top == want
        dk = np.sort(ex)[k - 1]
        minimal = set(np.flatnonzero((lb <= dk) & (ub >= dk)).tolist())
        assert minimal - {want[np.argmax(ex[want])]} <= vis | set(want)
        assert len(vis) < n                              # it does skip objects


def test_alg3_under_valid_bounds_exact_up_to_threshold_bucket(rng):
    """Algorithm 3 with valid bounds: k results; every object it misses or adds
    against the exact top-k has its exact distance in the final threshold bucket or beyond
    (bucket-granularity greediness, 'near-minimal'); it re-ranks fewer objects than all."""
    for n, k in ((800, 10), (2000, 300)):
        ex, lb, ub = _valid_bounds(rng, n, spread=0.05)
        dmin, dmax = np.float32(lb.min()), np.float32(np.sort(ex)[min(n - 1, 3 * k)])
        top, rer, j = O.bounded_rerank_alg3(lb, ub, lambda i: ex[i], k, dmin, dmax)
        assert len(top) == k and set(top) <= rer
        want = set(np.argsort(ex, kind="stable")[:k].tolist())
        edge_j = dmin + j * (dmax - dmin) / 255.0
        for o in set(top) ^ want:
            assert ex[o] >= edge_j - 1e-5, (o, ex[o], edge_j)
        assert len(rer) < n


def test_alg3_wide_bounds_is_full_rerank_and_zero_width_is_exact(rng):
    """Limits of Algorithm 3: bounds wider than the data (every object ambiguous) re-rank every
    in-range object and return the exact top-k; zero-width bounds (lb = ub = exact) re-rank only
    the threshold bucket and still return the exact top-k up to ties inside that bucket."""
    n, k = 1200, 50
    ex = rng.uniform(1.0, 2.0, n).astype(np.float32)
    dmin, dmax = np.float32(0.5), np.float32(2.5)
    lb = np.full(n, 0.5, np.float32)
    ub = np.full(n, 2.4, np.float32)
    top, rer, _ = O.bounded_rerank_alg3(lb, ub, lambda i: ex[i], k, dmin, dmax)
    assert sorted(top) == sorted(np.argsort(ex, kind="stable")[:k].tolist())
    assert len(rer) == n
    top0, rer0, j0 = O.bounded_rerank_alg3(ex, ex, lambda i: ex[i], k, dmin, dmax)
    cells = O.cells(ex, dmin, dmax)
    assert rer0 <= set(np.flatnonzero(cells <= j0).tolist())
    assert len(rer0) < n // 4
    assert set(top0) == set(np.argsort(ex, kind="stable")[:k].tolist())


# ---------------------------------------------------------------- f2: Algorithm 4
def test_alg4_predicted_threshold_hand_example():
    """tau_pred by hand: sample estimates 0..99, |O| = 1000, n_cand = 200: rank
    floor(200 * 100 / 1000) = 20 -> the 20th smallest = 19.0; codebook [0, 51] with 255 cells of
    width 0.2 -> bucket floor(19 / 0.2) = 95.  Rank below 1 is taken as 1 (the sample minimum:
    bucket 0); a rank beyond the sample as its last element."""
    v = np.arange(100, dtype=np.float32)[::-1].copy()
    assert O.predicted_threshold(v, 1000, 200, np.float32(0), np.float32(51)) == 95
    assert O.predicted_threshold(v, 100000, 200, np.float32(0), np.float32(51)) == 0
    assert O.predicted_threshold(v, 100, 200, np.float32(0), np.float32(51)) == 255   # 99 > d_max
    # the whole set as the sample: the n_cand-th distance's bucket, i.e. Algorithm 1's closed-form tau
    x = np.random.default_rng(5).uniform(0, 1, 5000).astype(np.float32)
    dmin, dmax = O.edges(x, 700)
    c = O.cells(x, dmin, dmax)
    assert O.predicted_threshold(x, len(x), 700, dmin, dmax) == O.threshold(np.bincount(c, minlength=256), 700)


def test_alg4_hand_example():
    """Ten objects, the first four the sample; cells 0 1 3 2 | 0 1 2 3 4 255, tau = 2, tau_pred = 2:
    the buffer takes cells <= 2 (positions 0 1 3 4 5 6); of the objects after the sample those with
    a cell < 2 (positions 4, 5) get their exact distance early, position 6 (cell 2) and the sample's
    0, 1, 3 at the end; the result is the k smallest exact distances of those six."""
    cell = np.array([0, 1, 3, 2, 0, 1, 2, 3, 4, 255])
    est = np.arange(10, dtype=np.float32)
    exact = np.array([5, 1, 0.5, 7, 3, 9, 2, 0.1, 0.2, 0.3], dtype=np.float32)
    calls = []

    def fn(i):
        calls.append(i)
        return exact[i]

    ids = np.arange(100, 110)
    out_ids, out_d2, early = O.early_rerank_alg4(est, 4, cell, 2, 2, fn, ids, 3)
    assert early.tolist() == [4, 5]
    assert calls == [4, 5, 0, 1, 3, 6]                 # early ones first, each object once
    assert out_ids.tolist() == [101, 106, 104] and out_d2.tolist() == [1.0, 2.0, 3.0]
    # tau_pred = 0: nothing early; tau_pred above tau: every candidate after the sample is early
    assert len(O.early_rerank_alg4(est, 4, cell, 2, 0, fn, ids, 3)[2]) == 0
    assert O.early_rerank_alg4(est, 4, cell, 2, 200, fn, ids, 3)[2].tolist() == [4, 5, 6]


def test_alg4_equals_alg1_and_early_set_invariants(c1t):
    """Algorithm 4 changes when an exact distance is computed, not which objects are re-ranked
    ("we cannot reduce the number of objects to be re-ranked"): its result equals
    Algorithm 1's (`search`) exactly; the early objects lie after the sample, in buckets below
    tau_pred and at or below tau, and they are all of those."""
    cfg, ix, Q, _ = c1t
    k, nprobe, budget = 300, 16, 900
    ids1, d1, dbg = O.search(ix, Q[:6], k, nprobe, budget, want_debug=True)
    ids4, d4, info = O.search_early_alg4(ix, Q[:6], k, nprobe, budget)
    assert np.array_equal(ids1, ids4) and np.array_equal(d1, d4)
    some = 0
    for g, f in zip(dbg, info):
        assert f["tau"] == g["tau"]
        c = g["cell"]
        want = np.flatnonzero((np.arange(len(c)) >= f["n_sample"]) & (c < f["tau_pred"]) & (c <= f["tau"]))
        assert np.array_equal(f["early_pos"], want)
        assert set(f["early_ids"].tolist()) <= set(g["sup_ids"].tolist())
        some += len(want)
    assert some > 0
