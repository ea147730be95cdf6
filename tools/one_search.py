"""One bbc_search of a workload at a given (nprobe, budget) -- a short command for ncu captures."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from datagen import configs, synth  # noqa: E402
from paper_2604_01960_b200 import Index  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--workload", default="C2")
p.add_argument("--nprobe", type=int, default=768)
p.add_argument("--budget", type=int, default=20000)
p.add_argument("--reps", type=int, default=2)
p.add_argument("--nq", type=int, default=0, help="first nq queries (0: the config's batch)")
p.add_argument("--rerank", choices=("auto", "query", "list", "tile"), default="auto")
a = p.parse_args()
cfg = configs.get(a.workload)
path = datagen.ensure_index(cfg)
g = Index(path)
g.set_rerank_order({"auto": g.RERANK_AUTO, "query": g.RERANK_QUERY, "list": g.RERANK_LIST,
                    "tile": g.RERANK_TILE}[a.rerank])
Q = synth.generate_queries(cfg)
q = torch.from_numpy(Q[:a.nq] if a.nq else Q).contiguous().cuda()
for _ in range(a.reps):
    ids, d2 = g.search(q, cfg.k, a.nprobe, a.budget)
torch.cuda.synchronize()
print("ok", ids.shape)
