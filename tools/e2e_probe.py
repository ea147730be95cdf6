import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import datagen
from datagen import configs, synth
from paper_2604_01960_b200 import Index
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "C4"); path = datagen.ensure_index(cfg); g = Index(path)
Q = synth.generate_queries(cfg); nq = len(Q); k = cfg.k
nprobe, budget = {"C4": (768, 85000), "C2": (768, 20000), "C3": (2048, 20000)}[cfg.name]
qh = torch.from_numpy(Q).pin_memory().numpy()
oh = (torch.empty((nq, k), dtype=torch.int64).pin_memory().numpy(), torch.empty((nq, k), dtype=torch.float32).pin_memory().numpy())
q = torch.from_numpy(Q).cuda()
for gb in (96,):
    ws = torch.empty(int(gb * (1 << 30)), dtype=torch.uint8, device="cuda")
    g.search(q, k, nprobe, budget, workspace=ws); torch.cuda.synchronize()
    t = time.time(); g.search(q, k, nprobe, budget, workspace=ws); torch.cuda.synchronize(); td = time.time() - t
    g.search_host(qh, k, nprobe, budget, out=oh, workspace=ws)
    ts = []
    for _ in range(3):
        t = time.time(); g.search_host(qh, k, nprobe, budget, out=oh, workspace=ws); ts.append(time.time() - t)
    print(f"ws {gb} GB: device {td*1e3:.1f} ms, host path {np.median(ts)*1e3:.1f} ms, microbatches {g.last_stats()['microbatches']}", flush=True)
    del ws; torch.cuda.empty_cache()
