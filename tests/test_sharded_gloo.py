"""The list-sharded exchange algebra on CPU with torch.distributed (gloo, world size 2 and 3):
each rank runs oracle/sharded.py on its own lists and talks to the others only through
all-reduces and one all-gather of the selected (d^2, id) pairs; the result equals the unsharded oracle exactly (ids and d^2).  The GPU path
implements the same exchange steps (tests/test_gpu_parity.py::test_sharded_group_equals_single
checks it against the unsharded CUDA search)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, params, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import datagen
    from datagen import configs, index_file, synth
    from oracle import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allreduce(a, op):
        t = torch.from_numpy(np.ascontiguousarray(a))
        if t.dtype == torch.uint64:
            t = t.to(torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MIN)
        return t.numpy().astype(a.dtype)

    def allgather(a):
        out = [None] * world
        dist.all_gather_object(out, np.ascontiguousarray(a))
        return out

    cfg = configs.get(name)
    ix = index_file.read(datagen.ensure_index(cfg))
    Q = synth.generate_queries(cfg)[:5]
    for j, (k, nprobe, budget) in enumerate(params):
        ids, d2 = sharded.search(ix, Q, k, nprobe, budget, rank, world, allreduce, allgather)
        np.savez(os.path.join(outdir, f"r{rank}_{j}.npz"), ids=ids, d2=d2)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("C1t", 2), ("C1t", 3), ("C3s", 2)])
def test_sharded_oracle_equals_unsharded(tmp_path, name, world, load):
    from oracle import bbc_oracle as O
    cfg, ix, Q, _ = load(name)
    params = [(cfg.k, cfg.nprobe, cfg.budget), (7, 3, 20), (cfg.k, 1, cfg.k)]
    mp.spawn(_worker, args=(world, _port(), name, params, str(tmp_path)), nprocs=world, join=True)
    for j, (k, nprobe, budget) in enumerate(params):
        oi, od = O.search(ix, Q[:5], k, nprobe, budget)
        for r in range(world):
            z = np.load(os.path.join(tmp_path, f"r{r}_{j}.npz"))
            ids, d2 = z["ids"], z["d2"]
            for i in range(5):            # same set, same d^2 per id (output order is rank-major)
                a = np.argsort(oi[i], kind="stable")
                b = np.argsort(ids[i], kind="stable")
                assert np.array_equal(oi[i][a], ids[i][b])
                assert np.array_equal(od[i][a], d2[i][b])


def test_assignment_balances_lists():
    from oracle.sharded import assign_lists
    sizes = np.array([5, 9, 1, 9, 3, 0, 7])
    own = assign_lists(sizes, 2)
    load = [sizes[own == r].sum() for r in range(2)]
    assert abs(load[0] - load[1]) <= sizes.max()
    # exact greedy rule: (size desc, id asc) -> least loaded rank, ties to lowest rank
    order = sorted(range(len(sizes)), key=lambda L: (-sizes[L], L))
    ld = [0, 0]
    for L in order:
        r = 0 if ld[0] <= ld[1] else 1
        assert own[L] == r
        ld[r] += sizes[L]
