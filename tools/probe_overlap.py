"""How much do the probe sets of neighbouring queries overlap?  (Design data for multi-query
scan tiling.)  For the first nq queries of a workload, the nprobe nearest
lists (torch fp32 GEMM distances: statistics only), queries in the scan's locality order (region of
the nearest list, as k_qperm), and for windows of w consecutive queries the ratio
sum of probed objects / objects of the union of their lists (the reuse a code byte read once per
window could get)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from datagen import configs, index_file, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C4")
ap.add_argument("--nprobe", type=int, default=1024)
ap.add_argument("--nq", type=int, default=2500)
a = ap.parse_args()
cfg = configs.get(a.workload)
ix = index_file.read(datagen.ensure_index(cfg))
C = torch.from_numpy(np.asarray(ix["centroids"])).cuda()
Q = torch.from_numpy(synth.generate_queries(cfg)[:a.nq]).cuda()
sizes = torch.from_numpy(np.diff(np.asarray(ix["list_offsets"]))).cuda()
d2 = (Q * Q).sum(1, keepdim=True) + (C * C).sum(1)[None] - 2 * Q @ C.T
P = torch.topk(d2, a.nprobe, dim=1, largest=False).indices          # [nq, nprobe]
nlist = C.shape[0]
npiv = min(256, nlist)
piv = C[torch.arange(npiv, device="cuda") * nlist // npiv]
region = torch.argmin(((C[:, None, :] - piv[None]) ** 2).sum(-1), dim=1)
first = P[:, 0]
order = torch.argsort(region[first].long() * nlist + first.long())
P = P[order]
M = torch.zeros((a.nq, nlist), dtype=torch.bool, device="cuda")
M.scatter_(1, P, True)
objs = (M.float() @ sizes.float())                                     # probed objects per query
print(f"{cfg.name} nprobe {a.nprobe} nq {a.nq}: mean probed objects {objs.mean().item():.0f}")
for w in (2, 4, 8, 16, 32, 64, 148):
    n = a.nq // w * w
    U = M[:n].view(-1, w, nlist).any(1).float() @ sizes.float()
    S = objs[:n].view(-1, w).sum(1)
    pair = (M[:n].view(-1, w, nlist).all(1).float() @ sizes.float()) / objs[:n].view(-1, w).mean(1)
    print(f"  window {w:4d}: sum/union objects = {(S / U).mean().item():6.2f}   "
          f"objects in every query's set / mean = {pair.mean().item():.3f}")
