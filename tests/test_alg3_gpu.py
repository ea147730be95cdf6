"""f1 on the GPU: Algorithm 3, the bound-aware IVF+RaBitQ re-rank (DESIGN.md reading
R21), through the C ABI (bbc_set_bound_rerank + bbc_search_debug) against the oracle's literal
`bounded_rerank_alg3`, element by element.

The oracle side: O.search's per-query estimates, rq2 and sample edges (Algorithm 1's codebook,
P:L898), O.rabitq_bounds per probed list, O.cells of lb/ub, O.threshold of the upper-bound
histogram at k, O.exact_d2 as the exact distance, and O.bounded_rerank_alg3's re-ranked set
B_exact; the final result is the k smallest (exact d^2, id) of B_exact (O.select_topk, the
path's Collect l.22-23 order).  Integer-valued data (C3a3: C2's generator in fp32; C3a3u8: C5's
uint8 rows) makes every exact d^2 exact in fp32, so the exact distances' buckets that steer the
loop agree and everything is compared bit for bit: tau, the upper-bound histogram, the candidate
set {a_lb <= tau}, the re-ranked set, its distances, the final ids and distances, and the
rows-re-ranked counter.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

_IDX = {}


def gidx(load, name):
    from paper_2604_01960_b200 import Index
    cfg, ix, Q, path = load(name)
    if name not in _IDX:
        _IDX[name] = Index(path)
    return cfg, ix, Q, _IDX[name]


def oracle_alg3(ix, Q, k, nprobe, budget, eps0, nbuckets=255):
    """Per query: dict(tau, hist, cand (ids of a_lb <= tau), rer (ids of B_exact), rer_d2 by id,
    top ids / d2) from the oracle only."""
    from oracle import bbc_oracle as O
    _, _, dbg = O.search(ix, Q, k, nprobe, budget, want_debug=True)
    fac = np.asarray(ix["factors"])
    off = np.asarray(ix["list_offsets"])
    raw = np.asarray(ix["raw"])
    ids_all = np.asarray(ix["ids"])
    out = []
    for i, g in enumerate(dbg):
        pos = g["pos"]
        lb = np.empty(len(pos), np.float32)
        ub = np.empty(len(pos), np.float32)
        o = 0
        for j, L in enumerate(g["probe"]):
            n = int(off[L + 1] - off[L])
            lb[o:o + n], ub[o:o + n] = O.rabitq_bounds(g["est"][o:o + n], fac[pos[o:o + n]],
                                                       np.sqrt(np.float32(g["rq2"][j])), int(ix["D"]),
                                                       eps0)
            o += n
        a_lb = O.cells(lb, g["d_min"], g["d_max"], nbuckets)
        a_ub = O.cells(ub, g["d_min"], g["d_max"], nbuckets)
        H = np.bincount(a_ub, minlength=256)
        tau = O.threshold(H[:255], k)
        tc = 254 if tau == O.TAU_INF else tau
        ex = O.exact_d2(Q[i], raw[pos])
        _, rer, _ = O.bounded_rerank_alg3(lb, ub, lambda t: ex[t], k, g["d_min"], g["d_max"], nbuckets)
        rer = np.array(sorted(rer), dtype=np.int64)
        rid = ids_all[pos[rer]]
        top_ids, top_d2 = O.select_topk(ex[rer], rid, k)
        out.append(dict(tau=tau, hist=H[:255], cand=np.sort(ids_all[pos[a_lb <= tc]]),
                        rer=np.sort(rid), rer_d2=dict(zip(rid.tolist(), ex[rer].tolist())),
                        top_ids=top_ids, top_d2=top_d2))
    return out


def run_and_compare(load, name, eps0, nprobe=None, budget=None, k=None, scan=None, nq=None, gathers="list",
                    nbuckets=255):
    cfg, ix, Q, g = gidx(load, name)
    nprobe = cfg.nprobe if nprobe is None else nprobe
    budget = cfg.budget if budget is None else budget
    k = cfg.k if k is None else k
    Q = np.ascontiguousarray(Q[:nq] if nq else Q)
    if scan is not None:
        g.set_scan_mode(scan)
    g.set_bound_rerank(True, eps0, gathers)
    g.set_buckets(nbuckets)
    try:
        q = torch.from_numpy(Q).cuda()
        ids, d2, t = g.search_debug(q, k, nprobe, budget)
        torch.cuda.synchronize()
        st = g.last_stats()
    finally:
        g.set_bound_rerank(False)
        g.set_scan_mode(g.SCAN_TENSOR)
        g.set_buckets(255)
    ids, d2 = ids.cpu().numpy(), d2.cpu().numpy()
    t = {a: b.cpu().numpy() for a, b in t.items()}
    exp = oracle_alg3(ix, Q, k, nprobe, budget, np.float32(eps0), nbuckets)
    n_rer = n_cand = 0
    for i, e in enumerate(exp):
        assert t["tau"][i] == e["tau"], f"q{i} tau {t['tau'][i]} vs {e['tau']}"
        assert np.array_equal(t["hist"][i][:255], e["hist"]) and t["hist"][i][255] == 0, f"q{i} ub histogram"
        nc = int(t["n_cand"][i])
        assert nc == len(e["cand"]), f"q{i} n_cand {nc} vs {len(e['cand'])}"
        cids, cd2 = t["cand_ids"][i][:nc], t["cand_d2"][i][:nc]
        assert np.array_equal(np.sort(cids), e["cand"]), f"q{i} candidate set"
        done = np.isfinite(cd2)
        assert np.array_equal(np.sort(cids[done]), e["rer"]), f"q{i} re-ranked set"
        want = np.array([e["rer_d2"][c] for c in cids[done].tolist()], dtype=np.float32)
        assert np.array_equal(cd2[done], want), f"q{i} exact d2 of B_exact"
        assert np.all(np.isposinf(cd2[~done])), f"q{i} non-re-ranked not +inf"
        o = np.lexsort((ids[i], d2[i]))                   # results leave unsorted (bbc.h)
        assert np.array_equal(ids[i][o], e["top_ids"]), f"q{i} final ids"
        assert np.array_equal(d2[i][o], e["top_d2"]), f"q{i} final d2"
        n_rer += len(e["rer"])
        n_cand += nc
    # rows gathered: B_exact's (query mode) or every candidate's (list mode)
    assert st["candidates"] == (n_rer if gathers == "query" else n_cand)
    return t, exp


# eps0 1.9 (the paper's) leaves tau = infinity for most queries of these small indexes (wide
# bounds against the sample's range); 0.6 and 1.2 keep tau finite, and at 1.2 the loop stops
# before re-ranking every candidate (B_exact strictly inside {a_lb <= tau})
@pytest.mark.parametrize("name,eps0,scan", [
    ("C3a3", 1.9, "tensor"), ("C3a3", 1.2, "simt"), ("C3a3", 1.2, "tensor"), ("C3a3", 0.6, "tensor"),
    ("C3a3u8", 0.6, "tensor"), ("C3a3u8", 1.2, "simt"), ("C3a3u8d512", 0.6, "tensor"),
    ("C3a3u8d512", 0.6, "simt")])
@pytest.mark.parametrize("gathers", ["list", "query"])
def test_alg3_parity(load, name, eps0, scan, gathers):
    from paper_2604_01960_b200 import Index
    mode = Index.SCAN_TENSOR if scan == "tensor" else Index.SCAN_SIMT
    t, exp = run_and_compare(load, name, eps0, scan=mode, gathers=gathers)
    assert any(e["tau"] != (1 << 30) for e in exp)           # the threshold is finite somewhere
    if eps0 == 1.2:                                            # the loop stopped early somewhere
        assert any(len(e["rer"]) < len(e["cand"]) for e in exp)


@pytest.mark.parametrize("gathers", ["list", "query"])
def test_alg3_tau_infinity(load, gathers):
    """eps0 so wide that fewer than k upper bounds fall below d_max: tau = infinity, every object
    with a_lb <= 254 is re-ranked (R21)."""
    t, exp = run_and_compare(load, "C3a3", 60.0, nq=8, gathers=gathers)
    assert all(e["tau"] == (1 << 30) for e in exp)


@pytest.mark.parametrize("gathers", ["list", "query"])
def test_alg3_no_sample(load, gathers):
    """budget >= the probed objects: no sample (Alg. 1 l.11), every bound in bucket 0, tau = 0 and
    all of B_u[0] re-ranked as the threshold bucket's leftovers."""
    t, exp = run_and_compare(load, "C3a3", 1.9, nprobe=3, budget=10 ** 6, nq=8, gathers=gathers)
    assert all(e["tau"] == 0 for e in exp)


@pytest.mark.parametrize("gathers", ["list", "query"])
def test_alg3_narrow_bound(load, gathers):
    """eps0 -> 0: lb = ub = est (up to rounding), Algorithm 3 becomes Algorithm 1 with budget k
    plus the threshold bucket."""
    run_and_compare(load, "C3a3", 1e-4, nq=12, gathers=gathers)


@pytest.mark.parametrize("gathers", ["list", "query"])
def test_alg3_host_path_and_microbatches(load, gathers):
    """The pipelined host path (micro-batches) gives the device path's results under Algorithm 3."""
    cfg, ix, Q, g = gidx(load, "C3a3")
    g.set_bound_rerank(True, 1.2, gathers)
    try:
        q = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
        a_ids, a_d2 = g.search(q, cfg.k, cfg.nprobe, cfg.budget)
        torch.cuda.synchronize()
        h_ids, h_d2 = g.search_host(np.ascontiguousarray(Q), cfg.k, cfg.nprobe, cfg.budget)
        ws_min = g.workspace_size(len(Q), cfg.k, cfg.nprobe, cfg.budget)[1]
        ws = torch.empty(ws_min, dtype=torch.uint8, device="cuda")       # one query per micro-batch
        m_ids, m_d2 = g.search(q, cfg.k, cfg.nprobe, cfg.budget, workspace=ws)
        torch.cuda.synchronize()
    finally:
        g.set_bound_rerank(False)
    def srt(i_, d_):                       # Algorithm 3's candidate order is unspecified
        i_, d_ = np.asarray(i_), np.asarray(d_)
        o = np.array([np.lexsort((a, b)) for a, b in zip(i_, d_)])
        return np.take_along_axis(i_, o, 1), np.take_along_axis(d_, o, 1)
    ai, ad = srt(a_ids.cpu().numpy(), a_d2.cpu().numpy())
    for bi, bd in ((h_ids, h_d2), (m_ids.cpu().numpy(), m_d2.cpu().numpy())):
        bi, bd = srt(bi, bd)
        assert np.array_equal(ai, bi) and np.array_equal(ad, bd)


def test_alg3_argument_errors(load, c1t):
    from paper_2604_01960_b200 import Index
    from paper_2604_01960_b200.bbc import BBCError
    _, _, _, g = gidx(load, "C3a3")
    with pytest.raises(BBCError):
        g.set_bound_rerank(True, 0.0)
    with pytest.raises(BBCError):
        g.set_bound_rerank(True, float("nan"))
    with pytest.raises(BBCError):
        g.set_bound_rerank(True, 1.9, "rows")
    g.set_remap(8)
    try:
        with pytest.raises(BBCError):
            g.set_bound_rerank(True, 1.9)
    finally:
        g.set_remap(0)
    pq = Index(c1t[3])
    try:
        with pytest.raises(BBCError):
            pq.set_bound_rerank(True, 1.9)
        pq.set_bound_rerank(False)
    finally:
        pq.close()


@pytest.mark.slow
def test_alg3_full_size_c3_sampled(load):
    """Full-size C3 (1M x 960 fp32) at bench.py's operating point (nprobe 2,048, budget 20,000,
    k 5,000) with eps0 = 1.3 (Algorithm 3's recall-0.95 point), a batch of 200
    queries, 3 sampled queries against the oracle.  Everything the exact distances do not decide is
    bit-exact: tau, the upper-bound histogram, the candidate set {a_lb <= tau}.  fp32 data: the
    GPU's exact d^2 (fp32, FMA order of the warp split) and the oracle's (fp64 rounded once) differ
    by ~1e-6 relative, which can move an exact distance across a bucket edge and so steer the loop
    by a few objects; the re-ranked sets must agree to 0.1 %, the shared distances to 1e-5 relative,
    and the final ids to 0.1 % of k."""
    cfg, ix, Q, g = gidx(load, "C3")
    nprobe, budget, k, eps0 = 2048, 20000, cfg.k, 1.3
    Q = np.ascontiguousarray(Q[:200])
    sel = np.array([3, 101, 177])
    g.set_bound_rerank(True, eps0)
    try:
        ids, d2, t = g.search_debug(torch.from_numpy(Q).cuda(), k, nprobe, budget, cand_stride=60000)
        torch.cuda.synchronize()
    finally:
        g.set_bound_rerank(False)
    si = torch.from_numpy(sel).cuda()
    t = {a: b[si].cpu().numpy() for a, b in t.items()}
    ids, d2 = ids[si].cpu().numpy(), d2[si].cpu().numpy()
    exp = oracle_alg3(ix, np.ascontiguousarray(Q[sel]), k, nprobe, budget, np.float32(eps0))
    for i, e in enumerate(exp):
        assert t["tau"][i] == e["tau"] and e["tau"] != (1 << 30), f"q{sel[i]} tau"
        assert np.array_equal(t["hist"][i][:255], e["hist"]), f"q{sel[i]} ub histogram"
        nc = int(t["n_cand"][i])
        assert nc == len(e["cand"]) and nc <= 60000, f"q{sel[i]} n_cand"
        cids, cd2 = t["cand_ids"][i][:nc], t["cand_d2"][i][:nc]
        assert np.array_equal(np.sort(cids), e["cand"]), f"q{sel[i]} candidate set"
        done = np.isfinite(cd2)
        g_rer = set(cids[done].tolist())
        o_rer = set(e["rer"].tolist())
        assert len(g_rer ^ o_rer) <= 0.001 * len(o_rer), f"q{sel[i]} re-ranked sets {len(g_rer ^ o_rer)}"
        both = [c for c in cids[done].tolist() if c in o_rer]
        gd = dict(zip(cids[done].tolist(), cd2[done].tolist()))
        a = np.array([gd[c] for c in both])
        b = np.array([e["rer_d2"][c] for c in both])
        assert np.all(np.abs(a - b) <= 1e-5 * np.abs(b)), f"q{sel[i]} exact d2"
        common = len(set(ids[i].tolist()) & set(e["top_ids"].tolist()))
        assert common >= k - max(1, k // 1000), f"q{sel[i]} final ids {common}/{k}"


@pytest.mark.parametrize("gathers", ["list", "query"])
@pytest.mark.parametrize("nbuckets", [1, 40, 120])
def test_alg3_bucket_counts(load, gathers, nbuckets):
    """B < 255 equal-width buckets (bbc_set_buckets) for both of Algorithm 3's buffers and B_exact."""
    run_and_compare(load, "C3a3", 1.2, nq=12, gathers=gathers, nbuckets=nbuckets)
