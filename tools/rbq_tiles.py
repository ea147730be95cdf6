"""Count the RaBitQ GEMM tile-iterations (object tiles x query tiles per list) of a C3 search."""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import datagen
from datagen import configs, synth, index_file
from paper_2604_01960_b200 import Index
cfg = configs.get("C3")
path = datagen.ensure_index(cfg)
ix = index_file.read(path)
off = np.asarray(ix["list_offsets"]); sizes = np.diff(off)
g = Index(path)
q = torch.from_numpy(synth.generate_queries(cfg)).cuda()[:1000]
ids, d2, t = g.search_debug(q, cfg.k, 2048, 20000)
probe = t["probe"].cpu().numpy()
cnt = np.bincount(probe.ravel(), minlength=len(sizes))
ot = (sizes + 127) // 128
qt = (cnt + 31) // 32
print("tile-iterations", int((ot * qt).sum()), "ctas with work", int(((ot > 0) & (cnt > 0)).sum() and (ot * (cnt > 0)).sum()), "pairs", int(cnt.sum()))
print("per SM", (ot * qt).sum() / 148)
