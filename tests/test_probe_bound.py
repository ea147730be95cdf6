"""The tensor-core probe's shortlist rests on |d~ - d^2| <= E(q) (DESIGN.md 5,
paper_2604_01960_b200/csrc/bbc_probe_tc.cuh).  This checks the bound on the workloads' own
centroids and queries with a numpy emulation of the 3xTF32 product (tf32 = fp32 with the low 13
mantissa bits cleared, hi/lo split, fp32 accumulation in two different orders) against the
canonical fp32 d^2 -- the arithmetic the GPU kernel performs, not the oracle's."""
import numpy as np
import pytest

F32 = np.float32


def tf32(x):
    return (np.asarray(x, dtype=F32).view(np.uint32) & np.uint32(0xFFFFE000)).view(F32)


def canonical_d2(Q, C):
    acc = np.zeros((len(Q), len(C)), dtype=F32)
    for t in range(Q.shape[1]):
        df = Q[:, None, t] - C[None, :, t]
        acc = acc + df * df
    return acc


def approx_d2(Q, C, mu, reverse=False):
    qp = (Q - mu).astype(F32)
    cp = (C - mu).astype(F32)
    qh, ch = tf32(qp), tf32(cp)
    ql, cl = tf32(qp - qh), tf32(cp - ch)
    terms = [qh[:, None, :] * ch[None, :, :], qh[:, None, :] * cl[None, :, :],
             ql[:, None, :] * ch[None, :, :]]
    prod = (terms[0] + terms[1] + terms[2]).astype(F32)
    order = range(Q.shape[1] - 1, -1, -1) if reverse else range(Q.shape[1])
    dot = np.zeros((len(Q), len(C)), dtype=F32)
    for t in order:
        dot = dot + prod[:, :, t]
    qn = (qp * qp).sum(1, dtype=F32)
    cn = (cp.astype(np.float64) ** 2).sum(1).astype(F32)
    return qn[:, None] + cn[None, :] - F32(2) * dot, qn, cn


def _synthetic(kind, rng):
    """Small centroid/query sets shaped like the BASELINE configs the CPU suite does not build."""
    if kind == "int255":                               # C2/C5-like: integer-valued, offset
        C = np.minimum(255, np.floor(rng.exponential(20, (256, 128)))).astype(F32)
        Q = np.minimum(255, np.floor(rng.exponential(20, (6, 128)))).astype(F32)
    else:                                              # C4-like: unit norm, d = 96
        C = rng.standard_normal((256, 96)).astype(F32)
        C /= np.linalg.norm(C, axis=1, keepdims=True)
        Q = (C[:6] + 0.06 * rng.standard_normal((6, 96))).astype(F32)
        Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    return C, Q


@pytest.mark.parametrize("name", ["C1t", "C3s", "int255", "sphere96"])
def test_tensor_probe_error_bound(load, name):
    if name.startswith("C"):
        cfg, ix, Q, _ = load(name)
        Call = np.asarray(ix["centroids"], dtype=F32)
        Qs = np.asarray(Q, dtype=F32)[:6]
    else:
        Call, Qs = _synthetic(name, np.random.default_rng(7))
    C = Call[:256]
    mu = Call.astype(np.float64).mean(0).astype(F32)
    ref = canonical_d2(Qs, C).astype(np.float64)
    cmax = float(np.sqrt(((Call.astype(np.float64) - mu) ** 2).sum(1).max())) * (1 + 1e-6)
    for rev in (False, True):
        d_approx, qn, _ = approx_d2(Qs, C, mu, reverse=rev)
        qn = qn.astype(np.float64) * (1 + 2 ** -10)
        E = 2.0 ** -12 * np.sqrt(qn) * cmax + 2.0 ** -11 * (qn + cmax * cmax)
        err = np.abs(d_approx.astype(np.float64) - ref)
        assert (err <= E[:, None]).all(), float((err / E[:, None]).max())
        # the bound is not vacuous: it is far below the spread of the distances
        assert E.max() < 1e-2 * (ref.max() - ref.min())
