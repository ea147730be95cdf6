"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element.

Tolerances (BASELINE.json north_star): probe lists, sample counts, edges,
estimates, histograms, thresholds and superset ids bit-exact (canonical fp32 order on both
sides); exact d^2 within 1e-5 relative; final id sets identical except ids whose oracle d^2 is
within 1e-5 relative of the oracle's k-th d^2; recall equal within 0.001.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _index(path):
    from paper_2604_01960_b200 import Index
    return Index(path)


_IDX = {}
_LOAD = {}


@pytest.fixture(autouse=True)
def _bind_loader(load):
    _LOAD["f"] = load


def gpu_index(name):
    cfg, ix, Q, path = _LOAD["f"](name)
    if name not in _IDX:
        _IDX[name] = _index(path)
    return cfg, ix, Q, _IDX[name]


def integer_exact(cfg):
    """Integer-valued data and queries (C2: integers 0-255 stored as fp32; C5: uint8) under L2:
    every partial sum of an exact d^2 is an integer < 2^24, so fp32 and fp64 exact distances are
    identical and the final (d^2, id) selection is compared exactly."""
    return cfg.gen in ("C2", "C5") and cfg.metric == "l2"


def compare(cfg, ix, Q, gidx, k, nprobe, budget, want_est=True, check_final=True, nbuckets=255,
            remap_m=0, sel=None, cand_stride=None):
    """GPU search of all of Q in one call; the oracle's intermediates of the queries `sel`
    (default: all) compared element by element.  Rows are selected on the device before any copy
    (full-size debug buffers are gigabytes)."""
    from oracle import bbc_oracle as O
    q = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    gidx.set_buckets(nbuckets)
    gidx.set_remap(remap_m)
    try:
        ids, d2, t = gidx.search_debug(q, k, nprobe, budget, want_est=want_est, cand_stride=cand_stride)
        torch.cuda.synchronize()
    finally:
        gidx.set_buckets(255)
        gidx.set_remap(0)
    sel = np.arange(len(Q)) if sel is None else np.asarray(sel)
    si = torch.from_numpy(sel).cuda()
    t = {a: b[si].cpu().numpy() for a, b in t.items()}
    ids, d2 = ids[si].cpu().numpy(), d2[si].cpu().numpy()
    del si
    oi, od, dbg = O.search(ix, np.ascontiguousarray(Q[sel]), k, nprobe, budget, want_debug=True,
                           nbuckets=nbuckets, remap_m=remap_m)
    exact = integer_exact(cfg)
    cs = t["cand_ids"].shape[1]
    for i, g in enumerate(dbg):
        qi = int(sel[i])
        assert np.array_equal(t["probe"][i], g["probe"]), f"q{qi} probe"
        assert np.array_equal(t["rq2"][i].view(np.uint32), g["rq2"].view(np.uint32)), f"q{qi} rq2"
        assert t["n_probed"][i] == g["n_o"], f"q{qi} n_o"
        assert t["nsample"][i] == g["s"], f"q{qi} sample lists"
        if want_est:
            ge = t["est"][i][: g["n_o"]]
            assert np.array_equal(ge.view(np.uint32), g["est"].view(np.uint32)), \
                f"q{qi} est: {np.count_nonzero(ge != g['est'])} differ"
        if g["s"] > 0:
            assert t["edges"][i][0] == g["d_min"] and t["edges"][i][1] == g["d_max"], f"q{qi} edges"
            assert np.array_equal(t["hist"][i][:255], g["H"][:255]), f"q{qi} hist"
            assert t["tau"][i] == g["tau"], f"q{qi} tau"
        else:
            assert t["tau"][i] == O.TAU_INF
        nc = t["n_cand"][i]
        assert nc == len(g["sup_ids"]), f"q{qi} |S*|"
        assert nc <= cs, f"q{qi}: |S*| {nc} exceeds the debug stride {cs}"
        assert np.array_equal(t["cand_ids"][i][:nc], g["sup_ids"]), f"q{qi} superset ids"
        if exact:
            assert np.array_equal(t["cand_d2"][i][:nc], g["sup_d2"]), f"q{qi} exact d2 (integer data)"
        else:
            np.testing.assert_allclose(t["cand_d2"][i][:nc], g["sup_d2"], rtol=1e-5, atol=1e-6)
        if check_final:
            # the GPU row is exactly the k smallest (GPU d^2, id) of its own candidates ...
            check_final_self(ids[i], d2[i], t["cand_ids"][i][:nc], t["cand_d2"][i][:nc], k)
            # ... and the oracle's: identical (integer data), else up to ties within 1e-5
            if exact:
                assert np.array_equal(np.sort(ids[i]), np.sort(oi[i])), f"q{qi} final ids"
            else:
                check_final_ids(ids[i], d2[i], oi[i], od[i], k)
    return ids, d2, t


def check_final_self(gi, gd, cand_ids, cand_d2, k):
    """The (d^2, id) tie-break of k_final_select, exactly: the row is the k smallest (d^2, id) of
    the candidate set (ids and d^2 as the GPU computed them), padded with (-1, inf)."""
    order = np.lexsort((cand_ids, cand_d2))[:k]
    want = np.sort(cand_ids[order])
    got = gi[gi >= 0]
    assert np.array_equal(np.sort(got), want), "final selection is not the (d2, id) top-k"
    assert len(got) == min(k, len(cand_ids))
    assert (gi[len(got):] == -1).all() and np.isinf(gd[len(got):]).all()
    pos = {int(x): j for j, x in enumerate(cand_ids)}
    assert all(gd[j] == cand_d2[pos[int(x)]] for j, x in enumerate(got[:64])), "d2 of the selected ids"


def check_final_ids(gi, gd, oi, od, k):
    """Same id set except at ties of the k-th distance (within 1e-5 relative)."""
    valid = oi >= 0
    assert np.count_nonzero(gi >= 0) == np.count_nonzero(valid)
    if not valid.any():
        return
    kth = od[valid].max()
    tol = 1e-5 * max(abs(kth), 1e-30)
    go, oo = set(gi[gi >= 0].tolist()), set(oi[valid].tolist())
    for x in go ^ oo:
        # the differing id must sit at the boundary distance
        if x in oo:
            dx = od[oi == x][0]
        else:
            dx = gd[gi == x][0]
        assert abs(dx - kth) <= tol, f"id {x} d2 {dx} vs kth {kth}"
    assert len(go) == len(gi[gi >= 0])                   # no duplicates


@pytest.mark.parametrize("name", ["C1t", "C1s", "C2s", "C2f", "C3s", "C4s", "C5s", "C4ip_s", "C2q4s",
                                  "C3d1024s", "C3d64s", "C3d200s", "C2m64s", "C4m24s", "C4m8s"])
def test_parity_config_point(name):
    cfg, ix, Q, g = gpu_index(name)
    compare(cfg, ix, Q, g, cfg.k, cfg.nprobe, cfg.budget)


def _pairs_per_list(ix, Q, nprobe, nsamp_lists=None):
    from oracle import bbc_oracle as O
    pr, _ = O.probe(Q, np.asarray(ix["centroids"]), nprobe)
    return np.bincount(pr.ravel(), minlength=int(ix["nlist"]))


@pytest.mark.parametrize("name,stride", [("C3mt", 1), ("C3mt960", 4)])
def test_parity_rabitq_multitile(name, stride):
    """The tensor-core RaBitQ GEMM with >= 5 query tiles of kRbN = 96 pairs per list (Push pass):
    both TMEM accumulators, the wrap of the two B stages and of the 4-deep records ring, and the
    producer's loop past the first stages.  The whole batch runs in one call; every `stride`-th
    query is compared with the oracle (estimates, edges, histogram, tau, superset, results)."""
    cfg, ix, Q, g = gpu_index(name)
    per_list = _pairs_per_list(ix, Q, cfg.nprobe)
    assert per_list.max() >= 5 * 96, per_list            # the configuration reaches the paths
    g.set_scan_mode(g.SCAN_TENSOR)
    compare(cfg, ix, Q, g, cfg.k, cfg.nprobe, cfg.budget, sel=np.arange(0, len(Q), stride))


@pytest.mark.parametrize("name", ["C2s", "C4s", "C5s"])
def test_parity_code_load_modes(name):
    """The PQ scan with its code loads streamed past L1 (BBC_CODES_STREAM, the instantiation the
    full-size C4/C5 codes take) and cached (BBC_CODES_CACHED): both equal the oracle bit for bit."""
    cfg, ix, Q, g = gpu_index(name)
    try:
        for mode in (g.CODES_STREAM, g.CODES_CACHED):
            g.set_code_loads(mode)
            compare(cfg, ix, Q, g, cfg.k, cfg.nprobe, cfg.budget)
    finally:
        g.set_code_loads(g.CODES_AUTO)


@pytest.mark.parametrize("name,nprobe", [("C2s", None), ("C4s", None), ("C5s", None), ("C4ip_s", None),
                                         ("C2f", 1500)])
def test_parity_scan_orders(name, nprobe):
    """The 8-bit PQ scan in sweep order (BBC_ORDER_SWEEP: each query's lists by ascending id,
    work items sorted by their first list -- the order full-size C4/C5 take) and in probe order
    (BBC_ORDER_PROBE): both equal the oracle bit for bit (estimates, histograms, superset, results).
    C2f at nprobe 1,500 runs the order kernel's two-keys-per-thread sort."""
    cfg, ix, Q, g = gpu_index(name)
    npr = nprobe or cfg.nprobe
    q = Q if nprobe is None else Q[:4]
    try:
        for order in (g.ORDER_SWEEP, g.ORDER_PROBE):
            g.set_scan_order(order)
            compare(cfg, ix, q, g, cfg.k, npr, cfg.budget)
            st = g.last_stats()                      # the sample pass covers the sample (and, in
            assert st["sample_pass"] >= st["sampled"]   # sweep order, the lists filling its item)
    finally:
        g.set_scan_order(g.ORDER_AUTO)


@pytest.mark.parametrize("nprobe", [1025, 1500, 2048])
def test_parity_probe_sets_past_1024(nprobe):
    """Probe sets of 1,025-2,048 lists (C3's operating point has 2,048): the probe selection's
    two-keys-per-thread sort, and every list probed at 2,048."""
    cfg, ix, Q, g = gpu_index("C2f")
    compare(cfg, ix, Q[:4], g, cfg.k, nprobe, cfg.budget)


@pytest.mark.parametrize("name", ["C1t", "C2s", "C3s", "C4ip_s", "C2q4s"])
def test_parity_parameter_grid(name):
    cfg, ix, Q, g = gpu_index(name)
    for nprobe, bm in ((1, 1), (3, 2), (cfg.nprobe * 2, 1), (min(cfg.nlist, 64), 3)):
        nprobe = min(nprobe, cfg.nlist)
        for k in (1, 17, cfg.k):
            compare(cfg, ix, Q[:6], g, k, nprobe, max(k, int(bm * k)), want_est=False)


def test_full_probe_unlimited_budget_is_brute_force():
    from oracle import bruteforce as BF
    cfg, ix, Q, g = gpu_index("C1t")
    raw = np.asarray(ix["raw"])
    X = np.empty_like(raw)
    X[np.asarray(ix["ids"])] = raw
    q = torch.from_numpy(Q).cuda()
    ids, d2 = g.search(q, cfg.k, cfg.nlist, cfg.N)
    gi, gd = BF.ground_truth(Q, X, cfg.k)
    ids = ids.cpu().numpy()
    d2 = d2.cpu().numpy()
    for i in range(len(Q)):
        check_final_ids(ids[i], d2[i], gi[i], gd[i].astype(np.float32), cfg.k)


def test_edge_cases_sweep_order():
    """Degenerate passes in the scan's sweep order: a main pass with no lists (nprobe = 1: the
    sample is every probed list), tau = infinity (no sample), k = budget = 1, a single list after
    the sample, and every list probed."""
    cfg, ix, Q, g = gpu_index("C1t")
    try:
        g.set_scan_order(g.ORDER_SWEEP)
        compare(cfg, ix, Q[:3], g, 5000, 1, 5000)
        compare(cfg, ix, Q[:1], g, 1, 4, 1)
        compare(cfg, ix, Q[:2], g, 250, 9, 250)
        compare(cfg, ix, Q[:2], g, 300, cfg.nlist, 600)
    finally:
        g.set_scan_order(g.ORDER_AUTO)


def test_edge_cases():
    from paper_2604_01960_b200.bbc import BBCError
    cfg, ix, Q, g = gpu_index("C1t")
    q = torch.from_numpy(Q).cuda()
    # n_o < k: padded rows (tau = infinity)
    ids, d2, t = compare(cfg, ix, Q[:3], g, 5000, 1, 5000)
    assert (ids[:, -1] == -1).all() and np.isinf(d2[:, -1]).all()
    # budget == k, k == 1, single query, empty batch
    compare(cfg, ix, Q[:1], g, 1, 4, 1)
    compare(cfg, ix, Q[:2], g, 250, 6, 250)
    e = torch.empty((0, cfg.d), dtype=torch.float32, device="cuda")
    g.search(e, 10, 4, 20)
    # errors
    for k, nprobe, budget in ((0, 4, 10), (10, 0, 10), (10, cfg.nlist + 1, 10), (10, 4, 9),
                              (cfg.N + 1, 4, cfg.N + 1)):
        with pytest.raises(BBCError):
            g.search(q, k, nprobe, budget)


def test_degenerate_identical_vectors(tmp_path):
    """All database vectors equal: every estimate is equal, d_max == d_min, every object lands in
    cell 0 and the final selection is decided by id alone."""
    from datagen import build_index, configs, index_file, synth
    cfg = configs.get("C1t").replace(name="degen", N=1500, nlist=8, M=16, kmeans_iters=2,
                                     pq_train=1500, pq_iters=2)
    X = np.repeat(synth.generate_data(cfg)[:1], cfg.N, axis=0)
    idx = build_index.build(cfg, X=X)
    p = str(tmp_path / "degen.bbcivf")
    index_file.write(p, idx)
    ix = index_file.read(p)
    g = _index(p)
    Q = synth.generate_queries(cfg)[:3]
    ids, d2, t = compare(cfg, ix, Q, g, 100, 8, 300)
    for i in range(3):
        assert sorted(ids[i].tolist()) == list(range(100))


def test_final_select_large_tie_bins(tmp_path):
    """Final selection where the k-th distance is shared by thousands of candidates: two distinct
    database vectors (15,000 + 5,000 copies) give two keys; k inside either key's run is decided
    by id alone, and the result is the (d^2, id) top-k."""
    from datagen import build_index, configs, index_file, synth
    cfg = configs.get("C1t").replace(name="ties2", N=20000, nlist=4, M=16, kmeans_iters=2,
                                     pq_train=2000, pq_iters=2)
    base = synth.generate_data(cfg)[:2]
    X = np.concatenate([np.repeat(base[:1], 15000, axis=0), np.repeat(base[1:], 5000, axis=0)])
    X = X[np.random.default_rng(7).permutation(len(X))]
    idx = build_index.build(cfg, X=np.ascontiguousarray(X))
    p = str(tmp_path / "ties2.bbcivf")
    index_file.write(p, idx)
    ix = index_file.read(p)
    g = _index(p)
    Q = synth.generate_queries(cfg)[:2]
    d0 = ((Q[:, None, :].astype(np.float64) - base[None].astype(np.float64)) ** 2).sum(-1)
    for k in (10000, 17000):
        ids, d2, t = compare(cfg, ix, Q, g, k, cfg.nlist, cfg.N)
        for i in range(len(Q)):
            near = np.argmin(d0[i])
            first = np.flatnonzero((X == base[near]).all(1))
            second = np.flatnonzero((X == base[1 - near]).all(1))
            want = np.sort(first)[:k] if k <= len(first) else \
                np.concatenate([first, np.sort(second)[:k - len(first)]])
            assert np.array_equal(np.sort(ids[i]), np.sort(want)), (k, i)


def test_microbatching_matches_one_batch():
    cfg, ix, Q, g = gpu_index("C2s")
    q = torch.from_numpy(Q).cuda()
    a_ids, a_d2 = g.search(q, cfg.k, cfg.nprobe, cfg.budget)
    _, mn = g.workspace_size(len(Q), cfg.k, cfg.nprobe, cfg.budget)
    ws = torch.empty(mn + (mn // 3), dtype=torch.uint8, device="cuda")   # one query per batch
    b_ids, b_d2 = g.search(q, cfg.k, cfg.nprobe, cfg.budget, workspace=ws)
    assert torch.equal(a_ids, b_ids) and torch.equal(a_d2, b_d2)
    assert g.last_stats()["microbatches"] == len(Q)


def test_host_api_matches_device_api():
    cfg, ix, Q, g = gpu_index("C2s")
    q = torch.from_numpy(Q).cuda()
    a_ids, a_d2 = g.search(q, cfg.k, cfg.nprobe, cfg.budget)
    h_ids, h_d2 = g.search_host(Q, cfg.k, cfg.nprobe, cfg.budget)
    assert np.array_equal(a_ids.cpu().numpy(), h_ids)
    assert np.array_equal(a_d2.cpu().numpy(), h_d2)


@pytest.mark.parametrize("order", ["auto", "sweep"])
def test_host_api_pipelined_microbatches(order):
    """Host path with >= 4 micro-batches (device->host copies on a second stream, double-buffered
    staging) returns the device path's results bit for bit, also on a short last batch; in the
    scan's default order and in sweep order (the order the full-size C4/C5 host paths take)."""
    from datagen import configs, synth
    cfg, ix, Q, g = gpu_index("C2s")
    Qm = np.ascontiguousarray(synth.generate_queries(cfg, 1100))
    q = torch.from_numpy(Qm).cuda()
    a_ids, a_d2 = g.search(q, 200, cfg.nprobe, 400)
    try:
        if order == "sweep":
            g.set_scan_order(g.ORDER_SWEEP)
        h_ids, h_d2 = g.search_host(Qm, 200, cfg.nprobe, 400)
    finally:
        g.set_scan_order(g.ORDER_AUTO)
    assert g.last_stats()["microbatches"] >= 4
    assert np.array_equal(a_ids.cpu().numpy(), h_ids)
    assert np.array_equal(a_d2.cpu().numpy(), h_d2)


def test_host_api_large_k_relative_to_capacity():
    """with k large against the per-query capacity (few probed lists, padded rows) the
    host path's pipelined micro-batches must not overwrite an output staging buffer the copy
    stream still reads (the staging buffers sit at fixed workspace offsets): host results equal
    the device path's bit for bit over >= 4 micro-batches of shrinking size."""
    from datagen import synth
    cfg, ix, Q, g = gpu_index("C2s")
    Qm = np.ascontiguousarray(synth.generate_queries(cfg, 1300))
    q = torch.from_numpy(Qm).cuda()
    k, nprobe, budget = 3000, 10, 3000
    a_ids, a_d2 = g.search(q, k, nprobe, budget)
    h_ids, h_d2 = g.search_host(Qm, k, nprobe, budget)
    assert g.last_stats()["microbatches"] >= 3
    assert np.array_equal(a_ids.cpu().numpy(), h_ids)
    assert np.array_equal(a_d2.cpu().numpy().view(np.uint32), h_d2.view(np.uint32))


def test_binding_rejects_mismatched_arrays():
    """The binding checks what the C ABI cannot (it takes no d): queries of the wrong width, dtype
    or device, and caller-supplied outputs of the wrong shape or dtype, raise BBCError."""
    from paper_2604_01960_b200.bbc import BBCError
    cfg, ix, Q, g = gpu_index("C1t")
    q = torch.from_numpy(Q).cuda()
    for bad in (q[:, :-4].contiguous(), q.double(), q.cpu(), q[None]):
        with pytest.raises(BBCError):
            g.search(bad, 10, 4, 20)
    with pytest.raises(BBCError):
        g.search(q, 10, 4, 20, out=(torch.empty((len(Q), 9), dtype=torch.int64, device="cuda"),
                                    torch.empty((len(Q), 10), dtype=torch.float32, device="cuda")))
    with pytest.raises(BBCError):
        g.search_host(Q[:, :-4], 10, 4, 20)


def test_recall_matches_oracle():
    from oracle import bbc_oracle as O
    from oracle import bruteforce as BF
    cfg, ix, Q, g = gpu_index("C1s")
    raw = np.asarray(ix["raw"])
    X = np.empty_like(raw)
    X[np.asarray(ix["ids"])] = raw
    q = torch.from_numpy(Q).cuda()
    ids, d2 = g.search(q, cfg.k, cfg.nprobe, cfg.budget)
    ids = ids.cpu().numpy()
    oi, od = O.search(ix, Q, cfg.k, cfg.nprobe, cfg.budget)
    gi, gd = BF.ground_truth(Q, X, cfg.k)
    ex = lambda R: np.stack([BF.exact_all(Q[i], X)[np.maximum(R[i], 0)] for i in range(len(Q))])
    r_gpu = BF.recall(ids, ex(ids), gi, gd)
    r_orc = BF.recall(oi, ex(oi), gi, gd)
    assert abs(r_gpu - r_orc) <= 1e-3


@pytest.mark.slow
@pytest.mark.parametrize("name,nprobe,budget,nq,nsel", [
    ("C2", 768, 20000, 1000, 16),        # bench.py's C2 operating point, the whole batch in one call
    ("C2", 128, 20000, 1000, 8),         # BASELINE.json's C2 point
    ("C3", 2048, 20000, 500, 10),        # C3's operating point, 500 queries (~250 pairs per list:
                                         #   several query tiles of the RaBitQ GEMM per list)
    ("C4", 768, 85000, 2500, 12),        # C4's operating point, one micro-batch of bench.py's run
    ("C4", 512, 75000, 1000, 6),         # BASELINE.json's C4 point
    pytest.param("C5", 1024, 30000, 1000, 6, marks=pytest.mark.skipif(
        os.environ.get("BBC_FULL_C5") != "1",
        reason="C5's 100M-row index takes ~9 min to build: opt-in with BBC_FULL_C5=1 "
               "(run and logged in profiles/r02_parity_c5_full.log)")),
])
def test_full_size_sampled_parity(name, nprobe, budget, nq, nsel):
    """BASELINE.json configs at full size, at the operating points bench.py times, with the batch
    size of one bench micro-batch: `nsel` sampled queries compared with the oracle element by
    element (probe, estimates, edges, histogram, tau, superset ids and exact d^2, final ids), and
    every query's row checked for k distinct valid ids."""
    cfg, ix, Q, g = gpu_index(name)
    Q = np.ascontiguousarray(Q[:nq])
    sel = np.sort(np.random.default_rng(7).choice(nq, nsel, replace=False))
    ids, _, _ = compare(cfg, ix, Q, g, cfg.k, nprobe, budget, sel=sel, cand_stride=3 * budget)
    a, _ = g.search(torch.from_numpy(Q).cuda(), cfg.k, nprobe, budget)
    a = a.sort(dim=1).values
    assert bool((a >= 0).all())
    assert bool((a[:, 1:] != a[:, :-1]).all()), "duplicate ids in a row"


# ------------------------------------------------------------------ list-sharded path (8(e))
def _sorted_by_id(ids, d2):
    o = np.argsort(ids, axis=1, kind="stable")
    return np.take_along_axis(ids, o, 1), np.take_along_axis(d2, o, 1)


@pytest.mark.parametrize("name,G", [("C1t", 2), ("C2s", 3), ("C3s", 2), ("C5s", 4)])
def test_sharded_group_equals_single(name, G):
    """Lists sharded over G shards (greedy by size, as ivf_load does on G GPUs), the exchange
    steps (MIN/histogram all-reduces, radix passes, result gather) done by the single-process
    group: results equal the ORACLE's (oracle/bbc_oracle.py: the sharded algebra reproduces the
    unsharded search, tests/test_sharded_gloo.py) -- identical ids for integer data, up to ties
    within 1e-5 otherwise -- and are bit-identical to the unsharded CUDA search."""
    from oracle import bbc_oracle as O
    from paper_2604_01960_b200 import Index
    from paper_2604_01960_b200.bbc import search_group
    cfg, ix, Q, g = gpu_index(name)
    path = _LOAD["f"](name)[3]
    shards = [Index(path, rank=r, world=G) for r in range(G)]
    assert sum(s.info.n_local for s in shards) == cfg.N
    q = torch.from_numpy(Q).cuda()
    for k, nprobe, budget in ((cfg.k, cfg.nprobe, cfg.budget), (17, 3, 40), (cfg.k, 1, cfg.k)):
        a_ids, a_d2 = g.search(q, k, nprobe, budget)
        b_ids, b_d2 = search_group(shards, q, k, nprobe, budget)
        oi, od = O.search(ix, Q, k, nprobe, budget)
        bi, bd = b_ids.cpu().numpy(), b_d2.cpu().numpy()
        for i in range(len(Q)):
            if integer_exact(cfg):
                assert np.array_equal(np.sort(bi[i]), np.sort(oi[i])), f"q{i} sharded ids vs oracle"
            else:
                check_final_ids(bi[i], bd[i], oi[i], od[i], k)
        a = _sorted_by_id(a_ids.cpu().numpy(), a_d2.cpu().numpy())
        b = _sorted_by_id(bi, bd)
        assert np.array_equal(a[0], b[0])
        assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


@pytest.mark.parametrize("name,G", [("C2s", 2), ("C5s", 3)])
def test_sharded_group_sweep_order(name, G):
    """The list-sharded group search with every shard's PQ scan in sweep order (each shard sorts
    its own probed lists and work items): results equal the unsharded search bit for bit."""
    from paper_2604_01960_b200 import Index
    from paper_2604_01960_b200.bbc import search_group
    cfg, ix, Q, g = gpu_index(name)
    path = _LOAD["f"](name)[3]
    shards = [Index(path, rank=r, world=G) for r in range(G)]
    for s in shards:
        s.set_scan_order(s.ORDER_SWEEP)
    q = torch.from_numpy(Q).cuda()
    a_ids, a_d2 = g.search(q, cfg.k, cfg.nprobe, cfg.budget)
    b_ids, b_d2 = search_group(shards, q, cfg.k, cfg.nprobe, cfg.budget)
    a = _sorted_by_id(a_ids.cpu().numpy(), a_d2.cpu().numpy())
    b = _sorted_by_id(b_ids.cpu().numpy(), b_d2.cpu().numpy())
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


def test_nccl_path_world1_equals_single():
    """bbc_search through the sharded code path with a real (1-rank) NCCL communicator."""
    from paper_2604_01960_b200 import Index
    from paper_2604_01960_b200.bbc import nccl_unique_id
    cfg, ix, Q, g = gpu_index("C2s")
    path = _LOAD["f"]("C2s")[3]
    h = Index(path)
    h.comm_init(nccl_unique_id(), 0, 1)
    q = torch.from_numpy(Q).cuda()
    a_ids, a_d2 = g.search(q, cfg.k, cfg.nprobe, cfg.budget)
    b_ids, b_d2 = h.search(q, cfg.k, cfg.nprobe, cfg.budget)
    a = _sorted_by_id(a_ids.cpu().numpy(), a_d2.cpu().numpy())
    b = _sorted_by_id(b_ids.cpu().numpy(), b_d2.cpu().numpy())
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("name", ["C1t", "C2s", "C3s", "C4s", "C5s"])
def test_probe_modes_identical(name):
    """Tensor-core shortlist probe (default) and the SIMT canonical probe give the same probe
    lists, rq2 and results, and both equal the oracle's probe (a1)."""
    from oracle import bbc_oracle as O
    cfg, ix, Q, g = gpu_index(name)
    q = torch.from_numpy(Q).cuda()
    outs = {}
    for mode in (g.PROBE_SIMT, g.PROBE_TENSOR):
        g.set_probe_mode(mode)
        ids, d2, t = g.search_debug(q, cfg.k, cfg.nprobe, cfg.budget)
        torch.cuda.synchronize()
        outs[mode] = (ids.cpu().numpy(), d2.cpu().numpy(), t["probe"].cpu().numpy(),
                      t["rq2"].cpu().numpy())
    g.set_probe_mode(g.PROBE_AUTO)
    a, b = outs[g.PROBE_SIMT], outs[g.PROBE_TENSOR]
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))
    lists, rq = O.probe(Q, np.asarray(ix["centroids"]), cfg.nprobe)
    assert np.array_equal(b[2], lists)
    assert np.array_equal(b[3].view(np.uint32), np.asarray(rq, dtype=np.float32).view(np.uint32))


def test_probe_tensor_large_nprobe_and_ties():
    """Tensor-core probe at nprobe = nlist (every list shortlisted) and with duplicated queries."""
    cfg, ix, Q, g = gpu_index("C2s")
    Q2 = np.ascontiguousarray(np.concatenate([Q[:4], Q[:4]]))
    q = torch.from_numpy(Q2).cuda()
    res = []
    for mode in (g.PROBE_SIMT, g.PROBE_TENSOR):
        g.set_probe_mode(mode)
        _, _, t = g.search_debug(q, cfg.k, cfg.nlist, cfg.budget)
        torch.cuda.synchronize()
        res.append(t["probe"].cpu().numpy())
    g.set_probe_mode(g.PROBE_AUTO)
    assert np.array_equal(res[0], res[1])


@pytest.mark.parametrize("nprobe_mult", [1, 4])
def test_rabitq_scan_modes_identical(nprobe_mult):
    """RaBitQ estimates from the list-major tensor-core GEMM (default) and from the popcount
    kernel are bit-identical (exact integer code/query inner products), and so are every
    downstream intermediate and the results."""
    cfg, ix, Q, g = gpu_index("C3s")
    q = torch.from_numpy(Q).cuda()
    nprobe = min(cfg.nlist, cfg.nprobe * nprobe_mult)
    outs = []
    for mode in (g.SCAN_SIMT, g.SCAN_TENSOR):
        g.set_scan_mode(mode)
        ids, d2, t = g.search_debug(q, cfg.k, nprobe, cfg.budget, want_est=True)
        torch.cuda.synchronize()
        outs.append({"ids": ids.cpu().numpy(), "d2": d2.cpu().numpy(),
                     **{k_: v.cpu().numpy() for k_, v in t.items()}})
    g.set_scan_mode(g.SCAN_TENSOR)
    a, b = outs
    valid = {"est": "n_probed", "cand_ids": "n_cand", "cand_d2": "n_cand"}
    for key in a:
        if key in valid:                               # rows are valid up to their count only
            for i in range(len(Q)):
                n = int(a[valid[key]][i])
                assert np.array_equal(a[key][i][:n].view(np.uint8), b[key][i][:n].view(np.uint8)), key
        else:
            assert np.array_equal(a[key].view(np.uint8), b[key].view(np.uint8)), key


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C2s", "C2f", "C3s", "C4s", "C5s", "C4ip_s", "C2q4s"])
def test_rerank_orders_identical(name):
    """The list-major re-rank (segments ordered by inverted list), its shared-memory tiled form
    (rows of a list tile staged once per CTA) and the query-major one compute every candidate's
    exact distance identically: candidate distances, ids and results are bit-identical, at the
    config's nprobe and with every list probed."""
    cfg, ix, Q, g = gpu_index(name)
    q = torch.from_numpy(Q).cuda()
    for nprobe in (cfg.nprobe, cfg.nlist):
        outs = []
        orders = (g.RERANK_QUERY, g.RERANK_LIST) + ((g.RERANK_TILE,) if cfg.raw_dtype == "f32" and cfg.d * 4 <= 512 else ())
        for order in orders:
            g.set_rerank_order(order)
            ids, d2, t = g.search_debug(q, cfg.k, nprobe, cfg.budget)
            torch.cuda.synchronize()
            outs.append({"ids": ids.cpu().numpy(), "d2": d2.cpu().numpy(),
                         **{k_: v.cpu().numpy() for k_, v in t.items()}})
        g.set_rerank_order(g.RERANK_AUTO)
        a = outs[0]
        assert int(a["n_cand"].sum()) > 0
        for b in outs[1:]:
            for key in ("ids", "d2"):
                assert np.array_equal(a[key].view(np.uint8), b[key].view(np.uint8)), key
            for i in range(len(Q)):
                n = int(a["n_cand"][i])
                assert n == int(b["n_cand"][i])
                for key in ("cand_ids", "cand_d2"):
                    assert np.array_equal(a[key][i][:n].view(np.uint8), b[key][i][:n].view(np.uint8)), key


def test_ip_full_probe_unlimited_budget_is_brute_force_mips():
    """Inner-product index (f4): every list probed and budget >= N give the brute-force maximum
    inner product top-k, keys -<q, x> within 1e-5 relative (ids up to key ties)."""
    from oracle import bruteforce as BF
    cfg, ix, Q, g = gpu_index("C4ip_s")
    assert g.info.metric == 1
    raw = np.asarray(ix["raw"])
    X = np.empty_like(raw)
    X[np.asarray(ix["ids"])] = raw
    Qs = np.ascontiguousarray(Q[:3])
    k = 50
    ids, key = g.search(torch.from_numpy(Qs).cuda(), k, cfg.nlist, cfg.N)
    torch.cuda.synchronize()
    gi, gd = BF.ground_truth(Qs, X, k, metric="ip")
    for i in range(len(Qs)):
        check_final_ids(ids[i].cpu().numpy(), key[i].cpu().numpy(), gi[i], gd[i].astype(np.float32), k)
        np.testing.assert_allclose(np.sort(key[i].cpu().numpy()), gd[i], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("name", ["C2s", "C3s"])
@pytest.mark.parametrize("nbuckets", [1, 15, 100])
def test_parity_bucket_counts(name, nbuckets):
    """B regular buckets (Eq. 6; Table 4 sweep): histograms, tau, supersets and results equal the
    oracle's for coarse bucket grids too (PQ and the tensor-core RaBitQ path)."""
    cfg, ix, Q, g = gpu_index(name)
    compare(cfg, ix, Q[:8], g, cfg.k, cfg.nprobe, cfg.budget, want_est=False, nbuckets=nbuckets)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C2s", "C3s", "C2q4s"])
@pytest.mark.parametrize("m", [1, 8, 56, 255])
def test_parity_equal_depth_remap(name, m):
    """The n_ew -> m equal-depth remap (reading R6): thresholds, supersets and results equal the
    oracle's for m buckets (56 = the paper's Wiki setting), also with B = 100 cells."""
    cfg, ix, Q, g = gpu_index(name)
    compare(cfg, ix, Q[:8], g, cfg.k, cfg.nprobe, cfg.budget, want_est=False, remap_m=m)
    if m == 56:
        compare(cfg, ix, Q[:8], g, cfg.k, cfg.nprobe, cfg.budget, want_est=False, remap_m=m,
                nbuckets=100)


@pytest.mark.parametrize("name,mult", [("C2s", 4), ("C3s", 8), ("C5s", 4), ("C4ip_s", 2)])
def test_workspace_bounds_respected(name, mult):
    """The search stays inside the workspace bbc_workspace_size asks for: a guard region placed
    right after exactly that many bytes is left untouched (one micro-batch and the minimum)."""
    cfg, ix, Q, g = gpu_index(name)
    q = torch.from_numpy(Q).cuda()
    nprobe = min(cfg.nlist, cfg.nprobe * mult)
    want, mn = g.workspace_size(len(Q), cfg.k, nprobe, cfg.budget)
    ref_ids, ref_d2 = g.search(q, cfg.k, nprobe, cfg.budget)
    for size in (want, mn):
        guard = 1 << 20
        buf = torch.full((size + guard,), 0xA5, dtype=torch.uint8, device="cuda")
        ids, d2 = g.search(q, cfg.k, nprobe, cfg.budget, workspace=buf[:size])
        torch.cuda.synchronize()
        assert bool((buf[size:] == 0xA5).all()), f"workspace overflow ({size} bytes)"
        assert torch.equal(ids, ref_ids) and torch.equal(d2, ref_d2)


def test_search_captures_into_a_cuda_graph():
    """bbc_search enqueues only stream-ordered work (no host synchronisation, no allocation) on
    the single-shard device path, so a caller can capture it into a CUDA graph once and replay it
    (launch-bound small batches); the replays return the eager results bit for bit."""
    cfg, ix, Q, g = gpu_index("C1t")
    q = torch.from_numpy(Q).cuda()
    k, nprobe, budget = cfg.k, cfg.nprobe, cfg.budget
    ws = g.workspace(len(Q), k, nprobe, budget)
    ref_ids, ref_d2 = g.search(q, k, nprobe, budget, workspace=ws)
    out = (torch.empty_like(ref_ids), torch.empty_like(ref_d2))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):                          # warm the kernels' attributes outside capture
        g.search(q, k, nprobe, budget, out=out, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        g.search(q, k, nprobe, budget, out=out, workspace=ws)
    for _ in range(3):
        out[0].fill_(-7)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out[0], ref_ids) and torch.equal(out[1], ref_d2)
