"""Per-stage device times of bbc_search on a workload (timed like bench.py: L2 flushed between
steps), for kernel tuning runs."""
import argparse
import json
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
p.add_argument("--steps", type=int, default=5)
p.add_argument("--tag", default="")
p.add_argument("--probe-simt", action="store_true")
p.add_argument("--scan-simt", action="store_true")
p.add_argument("--probe-tc", action="store_true", help="force the tensor-core probe")
p.add_argument("--nq", type=int, default=0, help="first nq queries only (0: all)")
p.add_argument("--ws-gb", type=float, default=48.0, help="workspace cap (GiB)")
p.add_argument("--rerank", choices=("auto", "query", "list", "tile"), default="auto", help="re-rank order")
p.add_argument("--bound-rerank", type=float, default=None, help="Algorithm 3 with this eps0 (RaBitQ)")
p.add_argument("--gathers", choices=("list", "query"), default="list", help="Algorithm 3's gathers")
p.add_argument("--order", choices=("auto", "probe", "sweep"), default="auto", help="8-bit PQ scan order")
a = p.parse_args()
cfg = configs.get(a.workload)
path = datagen.ensure_index(cfg)
g = Index(path)
if a.probe_simt:
    g.set_probe_mode(g.PROBE_SIMT)
if a.probe_tc:
    g.set_probe_mode(g.PROBE_TENSOR)
if a.scan_simt:
    g.set_scan_mode(g.SCAN_SIMT)
g.set_rerank_order({"auto": g.RERANK_AUTO, "query": g.RERANK_QUERY, "list": g.RERANK_LIST,
                    "tile": g.RERANK_TILE}[a.rerank])
g.set_scan_order({"auto": g.ORDER_AUTO, "probe": g.ORDER_PROBE, "sweep": g.ORDER_SWEEP}[a.order])
if a.bound_rerank is not None:
    g.set_bound_rerank(True, a.bound_rerank, a.gathers)
q = torch.from_numpy(synth.generate_queries(cfg)).cuda()
if a.nq:
    q = q[:a.nq].contiguous()
ws = g.workspace(len(q), cfg.k, a.nprobe, a.budget, max_bytes=int(a.ws_gb * (1 << 30)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ids, d2 = g.search(q, cfg.k, a.nprobe, a.budget, workspace=ws)
torch.cuda.synchronize()
g.get_timing()
g.set_timing(True)
tot = 0.0
for _ in range(a.steps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.search(q, cfg.k, a.nprobe, a.budget, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
g.set_timing(False)
st, _ = g.get_timing()
stats = g.last_stats()
print(json.dumps({"tag": a.tag, "workload": a.workload, "ms_per_step": tot / a.steps,
                  **{k: round(v / a.steps, 4) for k, v in st.items()},
                  **{k: v / len(q) for k, v in stats.items() if k != "microbatches"}}), flush=True)
