"""f1: is the bound-aware RaBitQ re-rank (Algorithm 3) worth building
on the GPU for C3?  The oracle's literal Algorithm 3 (reading R21) against Algorithm 1's candidate
superset S* at bench.py's C3 operating point (nprobe 2048, budget 20,000, k 5,000), on sampled
queries of the full-size index.  Measured per query: rows Algorithm 1 re-ranks (|S*|), rows
Algorithm 3 re-ranks, the rows ANY bound-based re-rank must gather to return exact distances
(objects with lb <= Dist_k: the certainly-in plus Observation 1's ambiguous set), the
bound's coverage at eps0 = 1.9 and both results' recall; plus rows/recall of Algorithm 3 at eps0 1.0/1.3/1.6
(the bound scaled around the estimate) and of Algorithm 1 at budgets 15k/25k/30k.  The numbers go to
gpurun_out/r2_alg3_c3.json (copied to profiles/); DESIGN.md section 8 reads them.  Marked gpu/slow:
it runs where the full-size C3 index is built (the GPU box), but computes on the CPU."""
import json
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_alg3_against_alg1_on_c3(load):
    from oracle import bbc_oracle as O
    from oracle import bruteforce as BF
    cfg, ix, Q, _ = load("C3")
    nprobe, budget, k, nsel = 2048, 20000, cfg.k, 6
    sel = np.random.default_rng(11).choice(len(Q), nsel, replace=False)
    Qs = np.ascontiguousarray(Q[sel])
    oi, od, dbg = O.search(ix, Qs, k, nprobe, budget, want_debug=True)
    pr = O.probe(Qs, np.asarray(ix["centroids"]), nprobe)
    alg1 = {b: O.search(ix, Qs, k, nprobe, b, want_debug=True, probe_result=pr)
            for b in (15000, 25000, 30000)}
    raw = np.asarray(ix["raw"])
    ids_all = np.asarray(ix["ids"])
    X = np.empty_like(raw)
    X[ids_all] = raw
    gi, gd = BF.ground_truth(Qs, X, k)
    fac_all = np.asarray(ix["factors"])
    off = np.asarray(ix["list_offsets"])
    rows = []
    for i, g in enumerate(dbg):
        pos = g["pos"]
        sizes = off[g["probe"] + 1] - off[g["probe"]]
        lb = np.empty(len(pos), np.float32)
        ub = np.empty(len(pos), np.float32)
        o = 0
        for j, L in enumerate(g["probe"]):                 # per probed list: r = sqrt(rq2)
            n = int(sizes[j])
            lb[o:o + n], ub[o:o + n] = O.rabitq_bounds(g["est"][o:o + n], fac_all[pos[o:o + n]],
                                                       np.sqrt(np.float32(g["rq2"][j])), int(ix["D"]))
            o += n
        ex = O.exact_d2(Qs[i], raw[pos])
        top, rer, j = O.bounded_rerank_alg3(lb, ub, lambda o: ex[o], k, g["d_min"], g["d_max"])
        # recall against rows at other bound widths (Alg. 3) and budgets (Alg. 1)
        curve = {}
        for e0 in (1.0, 1.3, 1.6):
            lb2, ub2 = g["est"] - (g["est"] - lb) * np.float32(e0 / 1.9), g["est"] + (ub - g["est"]) * np.float32(e0 / 1.9)
            t2, r2, _ = O.bounded_rerank_alg3(lb2.astype(np.float32), ub2.astype(np.float32), lambda o: ex[o], k,
                                              g["d_min"], g["d_max"])
            rid2 = ids_all[pos[np.asarray(t2)]]
            curve[f"alg3_eps{e0}"] = (int(len(r2)), float(np.mean(np.isin(rid2, gi[i]) | (ex[np.asarray(t2)] <= gd[i, -1]))))
        for b_, (oi2, od2, dbg2) in alg1.items():
            curve[f"alg1_budget{b_}"] = (int(len(dbg2[i]["sup_ids"])),
                                         float(np.mean(np.isin(oi2[i], gi[i]) | (od2[i] <= gd[i, -1]))))
        dk = np.sort(ex)[k - 1]
        rid = ids_all[pos[np.asarray(top)]]
        rec3 = float(np.mean(np.isin(rid, gi[i]) | (ex[np.asarray(top)] <= gd[i, -1])))
        rec1 = float(np.mean(np.isin(oi[i], gi[i]) | (od[i] <= gd[i, -1])))
        assert len(top) == k
        rows.append({"query": int(sel[i]), "probed": int(len(pos)), "alg1_rows": int(len(g["sup_ids"])),
                     "alg3_rows": int(len(rer)), "rows_lb_below_distk": int(np.sum(lb <= dk)),
                     "observation1_ambiguous": int(np.sum((lb <= dk) & (ub >= dk))),
                     "certainly_in": int(np.sum(ub < dk)),
                     "bound_coverage": float(np.mean((ex >= lb) & (ex <= ub))),
                     "recall_alg1": rec1, "recall_alg3": rec3,
                     **{f"{key}_rows": v[0] for key, v in curve.items()},
                     **{f"{key}_recall": v[1] for key, v in curve.items()}})
    out = {"workload": "C3", "nprobe": nprobe, "budget": budget, "k": k, "eps0": 1.9, "queries": rows,
           "mean": {key: float(np.mean([r_[key] for r_ in rows])) for key in rows[0] if key != "query"}}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "r2_alg3_c3.json"), "w") as f:
        json.dump(out, f, indent=1)
