"""CPU oracle of the BBC large-k IVF query path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference` leg
may import this module.  The product path (`paper_2604_01960_b200`) never imports it, and this
module imports nothing from the product.  It shares no code with the CUDA path: the only common
dependency is the seeded-input layer `datagen/` (generators, index file), which holds none of the
method's arithmetic.

What it computes (steps O1-O9; "P:Lnnn" = line of PAPER.md):

  O1 coarse probe      d^2(q, c_j) for all lists, keep the nprobe smallest by (d^2, j)
                       (route; nearest-first order)
  O2 query tables      PQ: LUT[m][c] = sum_t (q_t - C[m][c][t])^2   ("pre-compute distances
                       between the query and the codebook vectors")
                       RaBitQ: u = P^T q, per probed list the 4-bit query code (B_q = 4)
  O3 estimate          PQ: est = sum_m LUT[m][code_m] ("use these pre-computed distances to
                       efficiently estimate"); 4-bit PQ: the FastScan estimate from the
                       8-bit quantised LUT (reading R20);
                       RaBitQ: unbiased inner-product estimator
  O4 sample            codebook generation from the nearest clusters
  O5 edges             d_min = smallest, d_max = budget-th smallest estimate of the sample
                       ("partial sort ... derive d_min and d_max from the local top-k")
                       equal-width cells, Eq. 6 with an explicit overflow cell
  O6 histogram         Push: bucket id of every probed object (Alg. 1 l.1-4)
  O7 threshold         Update: first bucket whose cumulative count reaches the budget
                       (Alg. 1 l.5-11; ">=" per Fig. 3)
  O8 superset          Collect l.19-21: all objects in buckets <= tau (superset P:L209)
  O9 re-rank, select   exact distance of every superset object and the k
                       smallest by (d^2, id)

Floating-point conventions.  Every quantity that feeds a discrete
decision (probe order, LUT, estimate, bucket) is evaluated in fp32 in the fixed order written
below, with each +,-,*,/ rounded separately (no fused multiply-add): that is the kernel's
precision, and both sides take the decision in it.  Exact re-rank distances are accumulated in
fp64 and rounded to fp32 once.

Metrics (the result buffer "applies to ... cosine
similarity and inner product").  Squared L2 is the default.  For an inner-product index
(ix["metric"] == "ip", PQ only) every key is the negated similarity, so "smaller is better"
everywhere: probe key -<q, c_j>, LUT[m][c] = -<q_m, C[m][c]>, estimate = sum of LUT entries,
exact key -<q, x>; the sample, buckets, threshold, superset and selection are unchanged.

Parity pins (tests/test_oracle.py): brute force on tiny inputs, the LUT identity, the closed form
tau = cell(budget-th smallest estimate), the superset invariants, Fig. 3 of the paper, Eq. 3, the
RaBitQ closed forms and error bound, and full-probe/unlimited-budget == brute force.
"""
from __future__ import annotations

import numpy as np

F32 = np.float32
TAU_INF = 1 << 30          # "tau = infinity" (Alg. 1 l.11): every probed object is a candidate
NCELL = 256                # 255 regular equal-width cells + 1 overflow cell (reading R3)
SAMPLE_MIN_LISTS = 8       # "5-10 nearest clusters", reading R5


# ----------------------------------------------------------------------------------------------
# O1  coarse probe
# ----------------------------------------------------------------------------------------------
def coarse_d2(Q: np.ndarray, C: np.ndarray, metric: str = "l2") -> np.ndarray:
    """Probe keys [nq x nlist].  L2: acc = 0; for t ascending: diff = q_t - c_t;
    acc = acc + diff*diff.  IP: acc = 0; for t ascending: acc = acc + q_t*c_t; key = -acc."""
    Q = np.asarray(Q, dtype=F32)
    C = np.asarray(C, dtype=F32)
    acc = np.zeros((len(Q), len(C)), dtype=F32)
    for t in range(Q.shape[1]):
        if metric == "ip":
            acc = acc + Q[:, t, None] * C[None, :, t]
        else:
            diff = Q[:, t, None] - C[None, :, t]
            acc = acc + diff * diff
    return -acc if metric == "ip" else acc


def probe(Q: np.ndarray, C: np.ndarray, nprobe: int, metric: str = "l2"):
    """The nprobe nearest lists per query (smallest keys), ties by list id.
    -> (probe i32, rq2 f32 = the probe keys)."""
    d2 = coarse_d2(Q, C, metric)
    nq, nlist = d2.shape
    pr = np.empty((nq, nprobe), dtype=np.int32)
    rq = np.empty((nq, nprobe), dtype=F32)
    j = np.arange(nlist)
    for i in range(nq):
        order = np.lexsort((j, d2[i]))[:nprobe]
        pr[i] = order
        rq[i] = d2[i][order]
    return pr, rq


# ----------------------------------------------------------------------------------------------
# O2/O3  PQ
# ----------------------------------------------------------------------------------------------
def pq_lut(q: np.ndarray, books: np.ndarray, metric: str = "l2") -> np.ndarray:
    """LUT[m][c] = sum_{t < dsub} (q[m*dsub + t] - C[m][c][t])^2, t ascending, fp32 [M x 256];
    inner product: LUT[m][c] = -(sum_t q[m*dsub + t] * C[m][c][t]), t ascending."""
    M, K, ds = books.shape
    qs = np.asarray(q, dtype=F32).reshape(M, ds)
    acc = np.zeros((M, K), dtype=F32)
    for t in range(ds):
        if metric == "ip":
            acc = acc + qs[:, t, None] * books[:, :, t]
        else:
            diff = qs[:, t, None] - books[:, :, t]
            acc = acc + diff * diff
    return -acc if metric == "ip" else acc


def pq_est(lut: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """est = LUT[0][c_0] + LUT[1][c_1] + ... + LUT[M-1][c_{M-1}], left to right, fp32."""
    acc = lut[0][codes[:, 0]]
    for m in range(1, lut.shape[0]):
        acc = acc + lut[m][codes[:, m]]
    return acc


def pq4_fastscan_lut(lut: np.ndarray):
    """The 8-bit quantised lookup table of 4-bit PQ (FastScan, P:L1798 with the paper's 4-bit PQ
    setting P:L1440; reading R20), from the fp32 LUT [M x 16] of pq_lut:
        lo_m  = min_c LUT[m][c]
        span  = max_m (max_c LUT[m][c] - lo_m)            (fp32 subtraction)
        delta = span / 255                                  (fp32 division)
        Q[m][c] = min(255, floor((LUT[m][c] - lo_m) / delta + 0.5))   (0 when delta = 0)
        bias  = lo_0 + lo_1 + ... + lo_{M-1}                (fp32, left to right)
    Returns (Q uint8 [M x 16], delta fp32, bias fp32)."""
    lut = np.asarray(lut, dtype=F32)
    lo = lut.min(axis=1)
    span = F32(0.0)
    for m in range(lut.shape[0]):
        span = max(span, F32(lut[m].max() - lo[m]))
    delta = F32(span / F32(255.0))
    if delta > 0:
        t = ((lut - lo[:, None]) / delta).astype(F32)
        qt = np.minimum(F32(255.0), np.floor((t + F32(0.5)).astype(F32))).astype(np.uint8)
    else:
        qt = np.zeros(lut.shape, dtype=np.uint8)
    bias = F32(0.0)
    for m in range(lut.shape[0]):
        bias = F32(bias + lo[m])
    return qt, delta, bias


def pq4_est(qlut: np.ndarray, delta: F32, bias: F32, codes: np.ndarray) -> np.ndarray:
    """est = delta * S + bias (fp32, multiply then add) with S = sum_m Q[m][code_m], an exact
    integer (<= 255 M): the FastScan estimate of the PQ distance, within M * delta / 2 of the
    fp32 LUT sum up to rounding."""
    codes = np.asarray(codes)
    S = np.zeros(len(codes), dtype=np.int64)
    for m in range(qlut.shape[0]):
        S += qlut[m][codes[:, m]]
    return (F32(delta) * S.astype(F32)).astype(F32) + F32(bias)


# ----------------------------------------------------------------------------------------------
# O2/O3  RaBitQ (1-bit codes, B_q = 4-bit query, estimator of gao2024rabitq)
# ----------------------------------------------------------------------------------------------
def rabitq_rotate(q: np.ndarray, P: np.ndarray) -> np.ndarray:
    """u = P^T q: u_i = sum_t P[t][i] q_t, t ascending over the d real dims (the zero padding
    up to D adds +-0 and cannot change a sum), fp32."""
    q = np.asarray(q, dtype=F32)
    acc = np.zeros(P.shape[1], dtype=F32)
    for t in range(len(q)):
        acc = acc + P[t] * q[t]
    return acc


def rabitq_query_code(u: np.ndarray, wL: np.ndarray, rq2: F32):
    """Per (query, list): q' = (u - w_L) * (1/r), 4-bit scalar quantisation of q' (round half
    up): qbar = clamp(floor((q' - v_l) * (1/delta) + 1/2), 0, 15).  The reciprocals 1/r and
    1/delta are single fp32 divisions per pair (canonical arithmetic, R12).

    Returns (qbar int [D], consts (c1, c2, c3) fp32, r fp32).  With D the padded dimension,
    <x_bar, q'> ~= c1 * <b, qbar> + c2 * popcount(b) + c3 where x_bar = (2b - 1)/sqrt(D):
      c1 = (2 delta)/sqrt(D), c2 = (2 v_l)/sqrt(D), c3 = -((delta * sum qbar)/sqrt(D)) - sqrt(D) v_l.
    """
    D = len(u)
    r = np.sqrt(F32(rq2))
    if r > 0:
        rinv = F32(1.0) / r
        qp = (u - wL) * rinv
    else:
        qp = np.zeros(D, dtype=F32)
    vl = qp.min()
    vr = qp.max()
    delta = (vr - vl) / F32(15.0)
    if delta > 0:
        dinv = F32(1.0) / delta
        qbar = np.floor((qp - vl) * dinv + F32(0.5))
        qbar = np.clip(qbar, 0, 15).astype(np.int64)
    else:
        qbar = np.zeros(D, dtype=np.int64)
    sq = F32(int(qbar.sum()))
    sD = np.sqrt(F32(D))
    c1 = (F32(2.0) * delta) / sD
    c2 = (F32(2.0) * vl) / sD
    c3 = (-((delta * sq) / sD)) - sD * vl
    return qbar, (F32(c1), F32(c2), F32(c3)), F32(r)


def rabitq_est(bits: np.ndarray, fac: np.ndarray, qbar: np.ndarray, consts, r: F32,
               rq2: F32) -> np.ndarray:
    """est d^2 = r_o^2 + r_q^2 - 2 r_o r_q <o,q>_est, <o,q>_est = <x_bar,q'>_est / g_o.

    Evaluation order (fp32, each op rounded): t1 = c2*p; t2 = t1 + c3; t3 = c1*ip; oq = t3 + t2;
    e = oq * (1/g_o); a = r_o*r_o; s = a + rq2; f = (2*r_o)*r; est = s - f*e, with 1/g_o one fp32
    division per object.
    """
    c1, c2, c3 = consts
    b = np.unpackbits(bits, axis=1, bitorder="little").astype(np.int64)
    ip = (b * qbar[None, :]).sum(1)
    p = b.sum(1)
    t1 = c2 * p.astype(F32)
    t2 = t1 + c3
    t3 = c1 * ip.astype(F32)
    oq = t3 + t2
    ginv = F32(1.0) / fac[:, 1]
    e = oq * ginv
    ro = fac[:, 0]
    a = ro * ro
    s = a + F32(rq2)
    f = (F32(2.0) * ro) * F32(r)
    return (s - f * e).astype(F32)


def rabitq_bounds(est: np.ndarray, fac: np.ndarray, r: F32, D: int, eps0: float = 1.9):
    """Lower / upper bounds of the exact d^2 around a RaBitQ estimate (the bound property the
    paper's IVF+RaBitQ re-ranking exploits; eps0 = 1.9): the estimator of
    <o, q> errs by at most eps0 * sqrt((1 - g_o^2) / g_o^2) / sqrt(D - 1) with high probability
    (gao2024rabitq), and d^2 = r_o^2 + r^2 - 2 r_o r <o, q>, so
        delta = ((2 r_o) r) * (t_o * eps),  t_o = sqrt(1 - g_o g_o) * (1 / g_o),
        eps = eps0 / sqrt(D - 1),            lb = est - delta,  ub = est + delta
    in fp32, each operation rounded (reading R21)."""
    ro = fac[:, 0].astype(F32)
    g = fac[:, 1].astype(F32)
    t = np.sqrt(F32(1.0) - g * g) * (F32(1.0) / g)
    eps = F32(F32(eps0) / np.sqrt(F32(D - 1)))
    delta = ((F32(2.0) * ro) * F32(r)) * (t * eps)
    est = np.asarray(est, dtype=F32)
    return (est - delta).astype(F32), (est + delta).astype(F32)


def minimal_rerank_alg2(lb: np.ndarray, ub: np.ndarray, exact_fn, k: int):
    """Algorithm 2, the minimal re-ranking solution, literally: H_u = max-heap of
    the k smallest upper bounds, H_l = min-heap of the objects whose lower bound is below the
    top of H_u; then re-rank the object with the smaller lower bound of the two heap tops until
    H_u.top_ub <= H_l.top_lb.  Objects are indices 0..n-1; exact_fn(i) -> exact distance.
    Ties in a heap are broken by object index.  Returns (sorted top-k indices, re-ranked set)."""
    import heapq
    Hu = []                                   # max-heap by ub: entries (-ub, -i, lb)
    Hl = []                                   # min-heap by lb: entries (lb, i)
    for i in range(len(lb)):
        top_ub = -Hu[0][0] if len(Hu) >= k else np.inf
        if ub[i] < top_ub:
            heapq.heappush(Hu, (-float(ub[i]), -i, float(lb[i])))
            if len(Hu) > k:
                nub, ni, nlb = heapq.heappop(Hu)
                heapq.heappush(Hl, (nlb, -ni))
        elif lb[i] < top_ub:
            heapq.heappush(Hl, (float(lb[i]), i))
    vis = set()
    exact = {}
    while Hu and Hl and -Hu[0][0] > Hl[0][0]:
        # the object with the smaller lower bound among the two tops
        u_lb, u_i = Hu[0][2], -Hu[0][1]
        if Hl[0][0] < u_lb or u_i in vis:
            lbv, i = heapq.heappop(Hl)
            if i in vis:
                continue
        else:
            _, ni, _ = heapq.heappop(Hu)
            i = -ni
        d = float(exact_fn(i))
        exact[i] = d
        vis.add(i)
        heapq.heappush(Hu, (-d, -i, d))
        if len(Hu) > k:
            nub, ni, nlb = heapq.heappop(Hu)
            if -ni not in vis:
                heapq.heappush(Hl, (nlb, -ni))
    return sorted(-e[1] for e in Hu), vis


def bounded_rerank_alg3(lb: np.ndarray, ub: np.ndarray, exact_fn, k: int, d_min: F32, d_max: F32,
                        nbuckets: int = 255):
    """Algorithm 3, IVF+RaBitQ with two result buffers B_u (keyed on the upper
    bound's bucket) and B_l (keyed on the lower bound's) sharing the codebook of the sample
    (d_min, d_max; Eq. 6 cells), in the one-shot form of reading R17 and with DESIGN.md reading
    R21 for the points the paper leaves open:
      tau   = Update(B_u, k): the first bucket whose cumulative upper-bound count reaches k
      B_u   = {o : a_ub <= tau}            (line 7, "<=" as reading R2)
      B_l   = {o : a_ub > tau, a_lb <= tau} (line 8-9), then every object of B_u too (line 11)
      loop  (lines 12-21) i = first non-empty B_l bucket, j = tau; while i < j: exact distances
            of B_l[i] and B_u[j] into B_exact (an object is re-ranked once and leaves both
            buffers); j = first bucket where the counts of B_u (by a_ub) and B_exact (by the
            exact distance's bucket) reach k; i = next non-empty B_l bucket
      result the k smallest (exact d^2, index) of B_exact plus the objects left in B_u[j] (line
            22: "B_u u B_exact"; the threshold bucket's leftovers get exact distances too).
    If tau is infinity (fewer than k upper bounds below d_max) every object with a_lb <= 254 is
    re-ranked.  Returns (top-k indices sorted by (exact, index), re-ranked index set, j)."""
    n = len(lb)
    a_lb = cells(lb, d_min, d_max, nbuckets)
    a_ub = cells(ub, d_min, d_max, nbuckets)
    tau = threshold(np.bincount(a_ub, minlength=NCELL)[:255], k)
    exact = {}
    if tau == TAU_INF:
        for i in np.flatnonzero(a_lb < 255):
            exact[int(i)] = float(exact_fn(int(i)))
        j = TAU_INF
    else:
        Bu = {c: set(np.flatnonzero(a_ub == c).tolist()) for c in range(tau + 1)}
        Bl = {c: set() for c in range(tau + 1)}
        for i in np.flatnonzero((a_ub > tau) & (a_lb <= tau)):
            Bl[int(a_lb[i])].add(int(i))
        for c in range(tau + 1):                       # line 11: B_u's objects into B_l
            for i in Bu[c]:
                Bl[int(a_lb[i])].add(i)
        He = np.zeros(NCELL, dtype=np.int64)

        def first_nonempty():
            for c in range(tau + 1):
                if Bl[c]:
                    return c
            return TAU_INF

        i, j = first_nonempty(), tau
        while i < j:
            for o in sorted(Bl[i] | Bu.get(j, set())):
                d = float(exact_fn(o))
                exact[o] = d
                He[int(cells(np.array([d], dtype=F32), d_min, d_max, nbuckets)[0])] += 1
                Bl[int(a_lb[o])].discard(o)
                if int(a_ub[o]) in Bu:
                    Bu[int(a_ub[o])].discard(o)
            Hu = np.zeros(NCELL, dtype=np.int64)
            for c, objs in Bu.items():
                Hu[c] += len(objs)
            j = threshold((Hu + He)[:255], k)
            i = first_nonempty()
        if j != TAU_INF and j in Bu:                   # the threshold bucket's leftovers
            for o in sorted(Bu[j]):
                exact[o] = float(exact_fn(o))
    keys = sorted((d, o) for o, d in exact.items())[:k]
    return sorted(o for _, o in keys), set(exact), j


# ----------------------------------------------------------------------------------------------
# O4-O8  the bucket-based result buffer
# ----------------------------------------------------------------------------------------------
def sample_lists(sizes_in_probe_order: np.ndarray, budget: int) -> int:
    """Number s of probe-order lists forming D_sample: the smallest s >= min(8, nprobe) whose
    lists hold >= budget objects (reading R5).  Returns 0 when n_o <= budget (tau = infinity)."""
    cum = np.cumsum(sizes_in_probe_order)
    if cum[-1] <= budget:
        return 0
    s0 = min(SAMPLE_MIN_LISTS, len(sizes_in_probe_order))
    s = int(np.searchsorted(cum, budget, side="left")) + 1     # first prefix with cum >= budget
    return max(s, s0)


def edges(sample_est: np.ndarray, budget: int):
    """(d_min, d_max): smallest and budget-th smallest estimate of the sample."""
    v = np.asarray(sample_est, dtype=F32)
    return F32(v.min()), F32(np.partition(v, budget - 1)[budget - 1])


def cells(x: np.ndarray, d_min: F32, d_max: F32, nbuckets: int = 255) -> np.ndarray:
    """Bucket id (Eq. 6, reading R3) with B = nbuckets regular equal-width buckets
    over [d_min, d_max] (1 <= B <= 255; the paper's m, Eq. 3 / Table 4): 255 for x > d_max;
    otherwise clamp(floor((x - d_min) * inv), 0, B - 1) with inv = B/(d_max - d_min) in fp32;
    0 when d_max == d_min (or inv is not finite)."""
    if not 1 <= nbuckets <= 255:
        raise ValueError("nbuckets must be in [1, 255]")
    x = np.asarray(x, dtype=F32)
    out = np.full(len(x), 255, dtype=np.int64)
    inb = ~(x > d_max)
    width = F32(d_max - d_min)
    inv = F32(nbuckets) / width if width > 0 else F32(np.inf)
    if not np.isfinite(inv):
        out[inb] = 0
        return out
    t = (x[inb] - d_min) * inv
    out[inb] = np.clip(np.floor(t), 0, nbuckets - 1).astype(np.int64)
    return out


def threshold(H: np.ndarray, budget: int) -> int:
    """Update (Alg. 1 l.5-11): the first bucket whose cumulative count reaches the budget."""
    cum = np.cumsum(H)
    hit = np.flatnonzero(cum >= budget)
    return int(hit[0]) if len(hit) else TAU_INF


def equal_depth_map(H0: np.ndarray, m: int, nbuckets: int = 255) -> np.ndarray:
    """The n_ew -> m remap ("first computes n_ew equal-width buckets and then reassigns
    these buckets into m equal-depth buckets, where a lookup table map is used", Eq. 6 with map,
    P:L922-932; reading R6): walk the equal-width cells c = 0 .. nbuckets-1 accumulating the
    sample histogram H0; cell c goes to the current bucket b, and b advances after c once the
    running count reaches (b+1)/m of the sample total (exact integer test run*m >= (b+1)*T),
    b <= m-1.  Cells >= nbuckets (incl. the overflow cell 255) map to 255 (never a candidate)."""
    if not 1 <= m <= 255:
        raise ValueError("m must be in [1, 255]")
    H0 = np.asarray(H0, dtype=np.int64)
    T = int(H0[:nbuckets].sum())
    mp = np.full(256, 255, dtype=np.int64)
    b, run = 0, 0
    for c in range(nbuckets):
        mp[c] = b
        run += int(H0[c])
        if b < m - 1 and run * m >= (b + 1) * T:
            b += 1
    return mp


def remap_threshold(H: np.ndarray, mp: np.ndarray, budget: int, m: int) -> int:
    """Update over the m equal-depth buckets: the first bucket tau_b whose cumulative count
    (cells mapped to it) reaches the budget; returned as the last cell mapped to a bucket
    <= tau_b, so that {map[cell] <= tau_b} = {cell <= returned} (map is nondecreasing)."""
    Hb = np.zeros(m, dtype=np.int64)
    for c in range(255):
        if mp[c] < m:
            Hb[mp[c]] += int(H[c])
    tb = threshold(Hb, budget)
    if tb == TAU_INF:
        return TAU_INF
    return int(np.flatnonzero(mp[:255] <= tb).max())


# ----------------------------------------------------------------------------------------------
# O9  exact re-rank and final selection
# ----------------------------------------------------------------------------------------------
def exact_d2(q: np.ndarray, rows: np.ndarray, metric: str = "l2") -> np.ndarray:
    """||q - x||^2 (inner product: -<q, x>) accumulated in fp64, rounded to fp32 once."""
    if metric == "ip":
        return (-(rows.astype(np.float64) @ np.asarray(q, dtype=np.float64))).astype(F32)
    diff = rows.astype(np.float64) - np.asarray(q, dtype=np.float64)[None, :]
    return (diff * diff).sum(1).astype(F32)


def select_topk(d2: np.ndarray, ids: np.ndarray, k: int):
    """The k smallest by (d^2, id); pads with (-1, +inf) when fewer than k exist."""
    order = np.lexsort((ids, d2))[:k]
    out_ids = np.full(k, -1, dtype=np.int64)
    out_d2 = np.full(k, np.inf, dtype=F32)
    out_ids[:len(order)] = ids[order]
    out_d2[:len(order)] = d2[order]
    return out_ids, out_d2


# ----------------------------------------------------------------------------------------------
# the whole path
# ----------------------------------------------------------------------------------------------
def search(ix: dict, Q: np.ndarray, k: int, nprobe: int, budget: int, want_debug: bool = False,
           probe_result=None, nbuckets: int = 255, remap_m: int = 0):
    """BBC search of every query in Q over the index dict `ix` (datagen.index_file.read).

    Returns (ids int64 [nq x k], d2 fp32 [nq x k]) -- rows sorted by (d^2, id) -- and, when
    want_debug, a list of per-query dicts with every intermediate of O1-O9.
    """
    if not (1 <= k <= ix["N"]):
        raise ValueError("k out of range")
    if not (1 <= nprobe <= ix["nlist"]):
        raise ValueError("nprobe out of range")
    if budget < k:
        raise ValueError("budget < k")
    Q = np.asarray(Q, dtype=F32)
    nq = len(Q)
    off = np.asarray(ix["list_offsets"])
    ids_all = ix["ids"]
    raw = ix["raw"]
    metric = ix.get("metric", "l2")
    if metric == "ip" and ix["kind"] != "pq":
        raise ValueError("the inner-product metric is defined for PQ indexes only")
    pr, rq = probe(Q, ix["centroids"], nprobe, metric) if probe_result is None else probe_result
    out_ids = np.empty((nq, k), dtype=np.int64)
    out_d2 = np.empty((nq, k), dtype=F32)
    dbg = []
    for i in range(nq):
        lists = pr[i]
        sizes = off[lists + 1] - off[lists]
        pos = np.concatenate([np.arange(off[L], off[L + 1]) for L in lists])  # probe order
        if ix["kind"] == "pq" and ix.get("nbits", 8) == 4:
            qlut, delta, bias = pq4_fastscan_lut(pq_lut(Q[i], ix["codebooks"], metric))
            est = pq4_est(qlut, delta, bias, np.asarray(ix["codes"][pos]))
        elif ix["kind"] == "pq":
            lut = pq_lut(Q[i], ix["codebooks"], metric)
            est = pq_est(lut, np.asarray(ix["codes"][pos]))
        else:
            u = rabitq_rotate(Q[i], ix["P"])
            parts = []
            for j, L in enumerate(lists):
                qbar, cs, r = rabitq_query_code(u, ix["wL"][L], rq[i, j])
                sl = slice(off[L], off[L + 1])
                parts.append(rabitq_est(np.asarray(ix["bits"][sl]), np.asarray(ix["factors"][sl]),
                                        qbar, cs, r, rq[i, j]))
            est = np.concatenate(parts) if parts else np.zeros(0, F32)
        n_o = len(pos)
        s = sample_lists(sizes, budget)
        if s == 0:
            tau = TAU_INF
            dmin = dmax = F32(np.nan)
            cell = np.zeros(n_o, dtype=np.int64)       # no buckets are formed (Alg. 1 l.11)
            H = np.zeros(NCELL, dtype=np.int64)
            sup = np.arange(n_o)
        else:
            ns = int(sizes[:s].sum())
            dmin, dmax = edges(est[:ns], budget)
            cell = cells(est, dmin, dmax, nbuckets)
            H = np.bincount(cell, minlength=NCELL)
            if remap_m:                                # equal-depth buckets (reading R6)
                H0 = np.bincount(cell[:ns], minlength=NCELL)
                tau = remap_threshold(H, equal_depth_map(H0, remap_m, nbuckets), budget, remap_m)
            else:
                tau = threshold(H, budget)
            sup = np.flatnonzero(cell <= tau)
        spos = pos[sup]
        sid = np.asarray(ids_all[spos])
        d2 = exact_d2(Q[i], np.asarray(raw[spos]), metric)
        out_ids[i], out_d2[i] = select_topk(d2, sid, k)
        if want_debug:
            dbg.append(dict(probe=lists, rq2=rq[i], n_o=n_o, s=s, d_min=dmin, d_max=dmax, H=H,
                            tau=tau, est=est, cell=cell, pos=pos, sup_pos=spos, sup_ids=sid,
                            sup_d2=d2))
    return (out_ids, out_d2, dbg) if want_debug else (out_ids, out_d2)


# ----------------------------------------------------------------------------------------------
# f2  Algorithm 4: early re-ranking of IVF+PQ
# ----------------------------------------------------------------------------------------------
def predicted_threshold(sample_est: np.ndarray, n_o: int, budget: int, d_min: F32, d_max: F32,
                        nbuckets: int = 255) -> int:
    """Alg. 4 l.2-4: "we use the bucket containing the (|O_sample|/|O| x n_cand)-th
    quantized distance as the predicted threshold bucket tau_pred".  |O_sample| = objects of the
    sample lists, |O| = n_o, the objects the query probes (the same sentence's update rule ends
    at the n_cand-th distance once everything is scanned), n_cand = budget; the rank is the
    integer floor((budget * |O_sample|) / n_o), at least 1 (reading R22)."""
    v = np.asarray(sample_est, dtype=F32)
    r = max(1, (int(budget) * len(v)) // int(n_o))
    r = min(r, len(v))
    x = np.partition(v, r - 1)[r - 1]
    return int(cells(np.array([x], dtype=F32), d_min, d_max, nbuckets)[0])


def early_rerank_alg4(est: np.ndarray, n_sample: int, cell: np.ndarray, tau: int, tau_pred: int,
                      exact_fn, ids: np.ndarray, k: int):
    """Algorithm 4 for one query, in the one-shot form of readings R17/R22: the
    codebook (cells), tau and tau_pred are those of the whole pass; objects are visited in probe
    order, nearest cluster first (l.5).
      l.8   a_i <= tau ("<" in the listing; "<=" as reading R2): the object enters the buffer B
      l.9   a_i < tau_pred: its exact distance is computed now (l.10-11, "immediately")
            -- only for objects scanned after the sample: the sample's estimates (l.2) exist
            before tau_pred does (l.4)
      l.13  otherwise its quantized distance is inserted
      l.15  "Re-rank remaining candidates in B": exact distance of every entry still holding a
            quantized one
      l.16  the k smallest (exact d^2, id)
    exact_fn(i) = exact d^2 (fp32) of probe-order position i.  Returns (ids [k], d2 [k], early)
    with `early` the probe-order positions whose exact distance was computed at l.10."""
    B = {}
    early = []
    for i in range(len(est)):
        a = int(cell[i])
        if a <= tau:
            if i >= n_sample and a < tau_pred:
                B[i] = (F32(exact_fn(i)), True)
                early.append(i)
            else:
                B[i] = (F32(est[i]), False)
    for i in list(B):
        if not B[i][1]:
            B[i] = (F32(exact_fn(i)), True)
    pos = np.fromiter(B.keys(), dtype=np.int64, count=len(B))
    d2 = np.array([B[int(i)][0] for i in pos], dtype=F32)
    out_ids, out_d2 = select_topk(d2, np.asarray(ids)[pos], k)
    return out_ids, out_d2, np.asarray(early, dtype=np.int64)


def search_early_alg4(ix: dict, Q: np.ndarray, k: int, nprobe: int, budget: int, nbuckets: int = 255):
    """IVF+PQ search with Algorithm 4: steps O1-O7 as `search` (probe, LUT, estimates, sample,
    codebook, Push, Update), then `predicted_threshold` and `early_rerank_alg4` in place of
    O8-O9.  Returns (ids, d2, per-query dicts with tau_pred, early positions, tau, n_sample)."""
    if ix["kind"] != "pq" or ix.get("nbits", 8) != 8:
        raise ValueError("Algorithm 4 is defined for IVF+PQ (8-bit codes here)")
    Q = np.asarray(Q, dtype=F32)
    metric = ix.get("metric", "l2")
    off = np.asarray(ix["list_offsets"])
    pr, _ = probe(Q, ix["centroids"], nprobe, metric)
    out_ids = np.empty((len(Q), k), dtype=np.int64)
    out_d2 = np.empty((len(Q), k), dtype=F32)
    info = []
    for i in range(len(Q)):
        lists = pr[i]
        sizes = off[lists + 1] - off[lists]
        pos = np.concatenate([np.arange(off[L], off[L + 1]) for L in lists])
        est = pq_est(pq_lut(Q[i], ix["codebooks"], metric), np.asarray(ix["codes"][pos]))
        n_o = len(pos)
        s = sample_lists(sizes, budget)
        if s == 0:                                     # no codebook: nothing can be predicted
            ns, tau, tpred = 0, TAU_INF, 0
            cell = np.zeros(n_o, dtype=np.int64)
        else:
            ns = int(sizes[:s].sum())
            dmin, dmax = edges(est[:ns], budget)
            cell = cells(est, dmin, dmax, nbuckets)
            tau = threshold(np.bincount(cell, minlength=NCELL), budget)
            tpred = predicted_threshold(est[:ns], n_o, budget, dmin, dmax, nbuckets)

        def exact_fn(j, _q=Q[i], _pos=pos):
            return exact_d2(_q, np.asarray(ix["raw"][_pos[j]:_pos[j] + 1]), metric)[0]

        out_ids[i], out_d2[i], early = early_rerank_alg4(est, ns, cell, tau, tpred, exact_fn,
                                                         np.asarray(ix["ids"][pos]), k)
        info.append(dict(tau=tau, tau_pred=tpred, n_sample=ns, early_pos=early,
                         early_ids=np.asarray(ix["ids"][pos[early]]) if len(early) else np.zeros(0, np.int64)))
    return out_ids, out_d2, info


# ----------------------------------------------------------------------------------------------
# paper-literal pieces used as pins
# ----------------------------------------------------------------------------------------------
class ResultBuffer:
    """Algorithm 1 written out literally over an explicit codebook C (Eq. 1-2):
    bucket B[i] = [c_i, c_{i+1}), i = 1..m; Push appends when j <= tau; Update returns the first
    bucket whose cumulative size reaches k (">=", reading R1); Collect returns B[1..tau-1] plus
    the top-s of B[tau].  Buckets are numbered from 1 as in Eq. 2."""

    def __init__(self, codebook):
        self.c = [float(v) for v in codebook]          # c_1 .. c_{m+1}
        self.m = len(self.c) - 1
        self.B = {i: [] for i in range(1, self.m + 1)}
        self.tau = float("inf")

    def bucket(self, dist: float) -> int:
        for i in range(1, self.m + 1):
            if self.c[i - 1] <= dist < self.c[i]:
                return i
        return 1 if dist < self.c[0] else self.m       # Eq. 6 clamp at both ends

    def push(self, oid, dist: float) -> None:
        j = self.bucket(dist)
        if j <= self.tau:
            self.B[j].append((dist, oid))

    def update(self, k: int):
        s = 0
        for i in range(1, self.m + 1):
            s += len(self.B[i])
            if s >= k:
                return i
        return float("inf")

    def relaxed_threshold(self) -> float:
        return self.c[self.tau] if self.tau != float("inf") else float("inf")

    def collect(self, k: int):
        res = []
        last = self.m if self.tau == float("inf") else self.tau
        for i in range(1, last):
            res.extend(self.B[i])
        s = k - len(res)
        res.extend(sorted(self.B[last], key=lambda p: (p[0], p[1]))[:max(s, 0)])
        return res


def eq3_num_buckets(d: int, n_sub: int, bits: int, l1_bytes: int = 32768) -> float:
    """Eq. 3: m = (C_L1 - C_quant - C_lut)/256 with C_quant = 2*32*n_sub*(B/8) and
    C_lut = n_sub * 2^B bytes, where n_sub (the paper's "d/M") is the number of sub-vectors."""
    c_quant = 2 * 32 * n_sub * bits / 8
    c_lut = n_sub * (2 ** bits)
    return (l1_bytes - c_quant - c_lut) / 256
