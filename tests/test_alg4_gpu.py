"""f2 on the GPU: Algorithm 4, the early re-ranking of IVF+PQ (DESIGN.md reading
R22), through the C ABI (bbc_set_early_rerank + bbc_search_debug) against the oracle.

Two comparisons per case.  (1) Everything Algorithm 1's parity test compares (probe, estimates,
edges, histogram, tau, superset ids in probe order, exact d^2 of every candidate, final ids) must
still hold with the early re-rank on: Algorithm 4 changes when an exact distance is computed, not
the result (`test_gpu_parity.compare` against `O.search`).  (2) What Algorithm 4 adds is compared
with `O.search_early_alg4`: tau_pred per query, the set of candidates whose distance was computed
early (ids), the final ids and distances, and the counter of early candidates.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def run_case(load, name, nprobe=None, budget=None, k=None, order=None, rerank=None, nq=None, nbuckets=255,
             expect_early=True):
    import test_gpu_parity as P
    from oracle import bbc_oracle as O
    P._LOAD["f"] = load
    cfg, ix, Q, g = P.gpu_index(name)
    nprobe = cfg.nprobe if nprobe is None else nprobe
    budget = cfg.budget if budget is None else budget
    k = cfg.k if k is None else k
    Q = np.ascontiguousarray(Q[:nq] if nq else Q)
    g.set_early_rerank(True)
    if order is not None:
        g.set_scan_order(order)
    if rerank is not None:
        g.set_rerank_order(rerank)
    try:
        ids, d2, t = P.compare(cfg, ix, Q, g, k, nprobe, budget, nbuckets=nbuckets)     # (1)
        stats = g.last_stats()
    finally:
        g.set_early_rerank(False)
        g.set_scan_order(g.ORDER_AUTO)
        g.set_rerank_order(g.RERANK_AUTO)
    oi, od, info = O.search_early_alg4(ix, Q, k, nprobe, budget, nbuckets=nbuckets)      # (2)
    exact = P.integer_exact(cfg)
    total = 0
    for i, f in enumerate(info):
        assert t["tau_pred"][i] == f["tau_pred"], f"q{i} tau_pred"
        nc = t["n_cand"][i]
        got = t["cand_ids"][i][:nc][t["cand_early"][i][:nc] != 0]
        assert np.array_equal(np.sort(got), np.sort(f["early_ids"])), f"q{i} early set"
        total += len(got)
        if exact:
            assert np.array_equal(np.sort(ids[i]), np.sort(oi[i])), f"q{i} final ids"
            assert np.array_equal(np.sort(d2[i]), np.sort(od[i])), f"q{i} final d2"
        else:                                            # GPU rows are not sorted by distance
            P.check_final_ids(ids[i], d2[i], oi[i], od[i], k)
            np.testing.assert_allclose(np.sort(d2[i]), np.sort(od[i]), rtol=1e-5, atol=1e-6)
    assert stats["early_candidates"] == total
    assert stats["early_objects"] >= total          # objects below tau_pred but above tau: computed, unused
    if expect_early:
        assert total > 0, "the case exercises no early object"
    return total


@pytest.mark.parametrize("name", ["C1t", "C2s", "C4s", "C5s", "C4ip_s", "C2m64s", "C4m8s"])
def test_alg4_parity_config_point(load, name):
    run_case(load, name, expect_early=False)


@pytest.mark.parametrize("name,nprobe,frac", [("C2s", 12, 0.6), ("C4s", 16, 0.5), ("C5s", 12, 0.7),
                                              ("C4ip_s", 16, 0.5), ("C1t", 10, 0.5)])
def test_alg4_many_early_objects(load, name, nprobe, frac):
    """A budget that is a large share of the probed objects puts tau_pred high: a large part of
    the candidates after the sample gets its exact distance in the scan."""
    import test_gpu_parity as P
    P._LOAD["f"] = load
    cfg, ix, Q, g = P.gpu_index(name)
    off = np.asarray(ix["list_offsets"])
    mean_list = float(off[-1]) / (len(off) - 1)
    budget = max(cfg.k, int(frac * nprobe * mean_list))
    total = run_case(load, name, nprobe=nprobe, budget=budget, nq=8)
    assert total > 8 * 20


@pytest.mark.parametrize("order", ["probe", "sweep"])
@pytest.mark.parametrize("rerank", ["list", "query"])
def test_alg4_scan_and_rerank_orders(load, order, rerank):
    import test_gpu_parity as P
    P._LOAD["f"] = load
    _, _, _, g = P.gpu_index("C2s")
    run_case(load, "C2s", nprobe=16, budget=3_000, order=g.ORDER_PROBE if order == "probe" else g.ORDER_SWEEP,
             rerank=g.RERANK_LIST if rerank == "list" else g.RERANK_QUERY, nq=10)


def test_alg4_degenerate_cases(load):
    """tau = infinity (budget >= probed objects: no sample, nothing early), fewer buckets, and the
    host path and micro-batches returning the same rows as the device path."""
    import test_gpu_parity as P
    P._LOAD["f"] = load
    cfg, ix, Q, g = P.gpu_index("C1t")
    run_case(load, "C1t", nprobe=6, budget=5_999, k=300, expect_early=False)
    run_case(load, "C1t", nbuckets=40, expect_early=False)
    q = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    g.set_early_rerank(True)
    try:
        a_ids, a_d2 = g.search(q, cfg.k, 10, 1_500)
        _, mn = g.workspace_size(len(Q), cfg.k, 10, 1_500)
        ws = torch.empty(mn + mn // 3, dtype=torch.uint8, device="cuda")   # one query per micro-batch
        b_ids, b_d2 = g.search(q, cfg.k, 10, 1_500, workspace=ws)
        assert g.last_stats()["microbatches"] == len(Q)
        h_ids, h_d2 = g.search_host(np.ascontiguousarray(Q), cfg.k, 10, 1_500)
        torch.cuda.synchronize()
    finally:
        g.set_early_rerank(False)
    assert torch.equal(a_ids, b_ids) and torch.equal(a_d2, b_d2)
    assert np.array_equal(a_ids.cpu().numpy(), h_ids) and np.array_equal(a_d2.cpu().numpy(), h_d2)


def test_alg4_rejected_configurations(load):
    import test_gpu_parity as P
    from paper_2604_01960_b200 import BBCError
    P._LOAD["f"] = load
    _, _, _, r = P.gpu_index("C3s")
    with pytest.raises(BBCError):
        r.set_early_rerank(True)                        # RaBitQ
    _, _, _, q4 = P.gpu_index("C2q4s")
    with pytest.raises(BBCError):
        q4.set_early_rerank(True)                       # 4-bit PQ
    _, _, _, g = P.gpu_index("C1t")
    g.set_early_rerank(True)
    try:
        with pytest.raises(BBCError):
            g.set_remap(16)
    finally:
        g.set_early_rerank(False)
