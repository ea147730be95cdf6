#!/usr/bin/env python
"""Benchmark of the B200 BBC query path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl bbc|reference]

A step = one bbc_search over the workload's whole query batch (all steps a1-a8 of DESIGN.md
section 1) with queries already resident in HBM; L2 is flushed (256 MB write) between timed steps,
outside the timed events.  `value` = queries/s of the whole job (all ranks), timed with CUDA
events on the search stream, max over ranks.  `e2e` = the same through bbc_search_host with the
host->device query copy and the device->host result copy inside the timed region.

Multi-GPU (torchrun), --shard lists (default for N > 1): the index is sharded by IVF list, every
rank runs the same `nq` queries and the exchange steps (histogram all-reduces, result
all-gather) are NCCL collectives inside libbbc.so ("scaling": "strong": the job's work is fixed).
--shard queries: each rank runs its own batch of `nq` queries on a replicated index (independent
problems, no data-path collective, "scaling": "weak").

--impl reference times the CPU oracle (oracle/, test infrastructure) on every host core (one
single-threaded process per core) on a bounded sample of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from datagen import configs, groundtruth, index_file, synth  # noqa: E402

# Operating points (nprobe, budget) per workload where GPU recall@k >= 0.95 on the first 100
# queries (sweep: `python bench.py --sweep`).  None = use the config point.
# C4: profiles/r02_sweep_c4.jsonl and r02_sweep_c4_fine.jsonl: 768 / 85,000 -> 0.9515 at 92.7k QPS
# (768 / 82,500: 0.9505, too close to the target; 1024 / 75,000: 0.961 at 76k); C2:
# profiles/r02_sweep_c2.jsonl confirms 768 / 20,000 (0.957).  C4ip: profiles/r02_sweep_c4ip_fine.jsonl:
# 832 / 85,000 -> 0.954 at 96.3k (768: 0.947; round 1's 1024 / 75,000: 0.967 at 86.3k).
RECALL95 = {"C2": (768, 20000), "C3": (2048, 20000), "C4": (768, 85000), "C5": (1024, 25000), "C4ip": (832, 85000),
            "C2q4": (1024, 60000)}
METRIC = "queries/sec at recall@k=0.95 (k=5k\u201350k); scan+rerank HBM GB/s vs peak"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="bbc", choices=["bbc", "reference"])
    p.add_argument("--workload", default="C4",
                   help="C4 (default): BASELINE.json configs[3], the largest configuration quoted "
                        "at 1 GPU that the metric's k range covers; C2, C3, C5, C4ip, C2q4 also")
    p.add_argument("--nprobe", type=int, default=None)
    p.add_argument("--budget", type=int, default=None)
    p.add_argument("--recall-queries", type=int, default=100)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--sweep", action="store_true", help="recall/QPS over an (nprobe, budget) grid")
    p.add_argument("--sweep-nprobe", default="", help="comma-separated nprobe multipliers of the sweep")
    p.add_argument("--sweep-budget", default="", help="comma-separated budget multipliers (x k)")
    p.add_argument("--profile-steps", action="store_true", help="no warm-up/recall/cpu (ncu runs)")
    p.add_argument("--shard", default=None, choices=["queries", "lists"],
                   help="multi-GPU partitioning: lists (default for --gpus > 1: the north_star's "
                        "IVF-list sharding with NCCL exchanges) or queries (replicas)")
    p.add_argument("--cpu-workers", type=int, default=0,
                   help="processes of the oracle baseline (0: every host core)")
    p.add_argument("--buckets", type=int, default=255, help="B regular buckets (Eq. 6)")
    p.add_argument("--bound-rerank", type=float, default=None, metavar="EPS0",
                   help="RaBitQ: Algorithm 3's bound-aware re-rank with this eps0 (1.9 in the paper) "
                        "instead of Algorithm 1's superset (f1; measurement, not the headline)")
    p.add_argument("--early-rerank", action="store_true",
                   help="f2: Algorithm 4 (early re-ranking of IVF+PQ, 8-bit codes): objects in buckets below "
                        "tau_pred get their exact distance straight after the scan pass")
    p.add_argument("--bound-rerank-gathers", choices=("list", "query"), default="list",
                   help="Algorithm 3's exact distances: every candidate's in list order, or B_exact's per query")
    p.add_argument("--bucket-sweep", action="store_true",
                   help="QPS, |S*|/budget and recall over B (Table 4 analog) at the operating point")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def tensor_peak_tops(dtype: str) -> float:
    """Dense tensor peak in TOP/s: measured bf16 (MEASURED_PEAKS.json) x the nominal ratio of
    the dtype to bf16 (tf32 0.5, int8 2)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16 = float(json.load(f)["bf16_tflops"])
    except Exception:
        bf16 = 2250.0
    return bf16 * {"bf16": 1.0, "tf32": 0.5, "i8": 2.0}[dtype]


def measured_traffic(workload, nprobe, budget, kernel):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of `kernel`'s launches in one
    step of the same workload and operating point, summed over every launch of the step, from the
    committed ncu capture (profiles/traffic.json, tools/traffic_from_ncu.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t[f"{workload}/{nprobe}/{budget}"][kernel]
        return {"dram_bytes_per_step": e["dram_bytes_per_step"], "launches_per_step": e["launches"],
                "dram_bytes_per_launch": e["dram_bytes_per_step"] / max(1, e["launches"]),
                "source": e["source"]}
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def operating_point(cfg, args):
    op = RECALL95.get(cfg.name)
    nprobe = args.nprobe or (op[0] if op else cfg.nprobe)
    budget = args.budget or (op[1] if op else cfg.budget)
    return nprobe, budget


def load_workload(name: str):
    cfg = configs.get(name)
    path = datagen.ensure_index(cfg)
    return cfg, path


def database_in_id_order(path):
    ix = index_file.read(path)
    raw = np.asarray(ix["raw"])
    X = np.empty_like(raw)
    X[np.asarray(ix["ids"])] = raw
    return X


# ------------------------------------------------------------------------------------ CPU oracle
# The oracle (oracle/bbc_oracle.py, test infrastructure) as it stands, timed on every host core:
# queries are independent, so a pool of single-threaded worker processes (fork; the index file is
# memory-mapped and shared through the page cache) each answers a slice of the sample.

_ORC = {}


def _orc_init(path):
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    from oracle import bbc_oracle as O
    _ORC["O"] = O
    _ORC["ix"] = index_file.read(path)


def _orc_run(job):
    Q, k, nprobe, budget = job
    _ORC["O"].search(_ORC["ix"], Q, k, nprobe, budget)
    return len(Q)


def host_cpu():
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return cores, model


class OraclePool:
    """`workers` single-threaded oracle processes (default: every host core)."""

    def __init__(self, path, workers=0):
        import multiprocessing as mp
        self.cores, self.model = host_cpu()
        self.workers = workers or self.cores
        self.pool = mp.get_context("fork").Pool(self.workers, initializer=_orc_init, initargs=(path,))

    def run(self, Q, k, nprobe, budget):
        """Answers the queries of Q (one per task, round-robin over the workers); wall seconds."""
        jobs = [(Q[i:i + 1], k, nprobe, budget) for i in range(len(Q))]
        t0 = time.perf_counter()
        n = sum(self.pool.map(_orc_run, jobs, chunksize=1))
        assert n == len(Q)
        return time.perf_counter() - t0

    def per_query_s(self, Q, k, nprobe, budget):
        """Single-core seconds per query (one query on each worker, warm)."""
        w = min(self.workers, len(Q))
        el = self.run(Q[:w], k, nprobe, budget)
        return el                                       # w queries in parallel ~ one query's time

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg, path = load_workload(args.workload)
    nprobe, budget = operating_point(cfg, args)
    Q = synth.generate_queries(cfg)
    pool = OraclePool(path, args.cpu_workers)
    per_q = max(1e-3, pool.per_query_s(Q, cfg.k, nprobe, budget))
    # each step a bounded sample: the whole run stays within a few minutes
    budget_s = 150.0 / max(1, args.steps + args.warmup)
    ns = int(max(pool.workers, min(cfg.nq, pool.workers * budget_s / per_q)))
    ns = min(ns, cfg.nq)
    for w in range(args.warmup):
        pool.run(Q[:ns], cfg.k, nprobe, budget)
    tot = 0.0
    for s in range(args.steps):
        lo = (s * ns) % cfg.nq
        sl = np.concatenate([Q[lo:], Q[:lo]])[:ns]
        tot += pool.run(sl, cfg.k, nprobe, budget)
    pool.close()
    qps = ns * args.steps / tot
    line = {"impl": "reference", "metric": json.loads('"' + METRIC + '"'),
            "value": qps, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": cfg.name, "nq": cfg.nq, "k": cfg.k, "nprobe": nprobe,
                       "budget": budget},
            "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": pool.workers,
                             "host_cores": pool.cores, "cpu_model": pool.model, "kind": "oracle",
                             "sample": f"{ns} of {cfg.nq} {cfg.name} queries per step, one "
                                       f"single-threaded numpy oracle process per core"},
            "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, path, nprobe, budget, seconds, workers=0):
    """The oracle on every host core over a bounded sample (~`seconds` of wall time)."""
    Q = synth.generate_queries(cfg)
    pool = OraclePool(path, workers)
    try:
        per_q = max(1e-3, pool.per_query_s(Q, cfg.k, nprobe, budget))
        ns = int(max(pool.workers, min(cfg.nq, pool.workers * seconds / per_q)))
        ns = min(ns, cfg.nq)
        el = pool.run(Q[:ns], cfg.k, nprobe, budget)
    finally:
        pool.close()
    return {"value": ns / el, "unit": "queries/s", "cores": pool.workers, "host_cores": pool.cores,
            "cpu_model": pool.model, "kind": "oracle",
            "sample": f"first {ns} of {cfg.nq} {cfg.name} queries (nprobe={nprobe}, "
                      f"budget={budget}), one single-threaded numpy oracle process per core, "
                      f"{el:.1f} s wall"}


# ------------------------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2604_01960_b200 import Index, launch_count
    from paper_2604_01960_b200.bbc import measure_l2_read_gbs, measure_smem_lookups

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.get(args.workload)
    if rank == 0:
        path = datagen.ensure_index(cfg, verbose=True)
    if world > 1:
        dist.barrier()
    path = datagen.index_path(cfg)
    nprobe, budget = operating_point(cfg, args)
    k = cfg.k

    shard = args.shard or ("lists" if world > 1 else "queries")
    lists = shard == "lists" and world > 1
    if lists:
        from paper_2604_01960_b200.bbc import nccl_unique_id
        g = Index(path, rank=rank, world=world, device=local)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        g.comm_init(obj[0], rank, world)
    else:
        g = Index(path, device=local)
    g.set_buckets(args.buckets)
    if args.bound_rerank is not None:
        g.set_bound_rerank(True, args.bound_rerank, args.bound_rerank_gathers)
    if args.early_rerank:
        g.set_early_rerank(True)
    if args.sweep:
        global args_sweep_nprobe, args_sweep_budget
        if args.sweep_nprobe:
            args_sweep_nprobe = tuple(float(x) for x in args.sweep_nprobe.split(","))
        if args.sweep_budget:
            args_sweep_budget = tuple(float(x) for x in args.sweep_budget.split(","))
        return sweep(cfg, path, g, rank)
    if args.bucket_sweep:
        return bucket_sweep(cfg, path, g, *operating_point(cfg, args))
    if lists:                                            # same queries on every rank
        Qh = np.ascontiguousarray(synth.generate_queries(cfg))
    else:
        Qall = synth.generate_queries(cfg, cfg.nq * world)
        Qh = np.ascontiguousarray(Qall[rank * cfg.nq:(rank + 1) * cfg.nq])
    nq = len(Qh)
    q = torch.from_numpy(Qh).cuda()
    # workspace: up to 96 GB (half of a B200; larger micro-batches, fewer wave tails: C4 at 48 GB
    # 108.0 ms/step, at 96 GB 106.4)
    import torch as _t
    ws_cap = min(96 << 30, int(0.55 * _t.cuda.get_device_properties(local).total_memory))
    ws = g.workspace(nq, k, nprobe, budget, max_bytes=ws_cap)
    out = (torch.empty((nq, k), dtype=torch.int64, device="cuda"),
           torch.empty((nq, k), dtype=torch.float32, device="cuda"))
    st = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    for _ in range(max(args.warmup, 0 if args.profile_steps else 3)):
        g.search(q, k, nprobe, budget, out=out, workspace=ws)
    torch.cuda.synchronize()

    # ---------------- timed region: K steps, device time per step, L2 flushed between steps
    g.get_timing()
    g.set_timing(True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = launch_count()
    with Clocks(local) as clk:
        for s in range(args.steps):
            flush.zero_()
            evs[s][0].record(st)
            g.search(q, k, nprobe, budget, out=out, workspace=ws)
            evs[s][1].record(st)
        torch.cuda.synchronize()
    launches = launch_count() - l0
    if world > 1:
        dist.barrier()
    g.set_timing(False)
    stage_ms, calls = g.get_timing()
    stats = g.last_stats()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    jobq = nq if lists else world * nq                   # queries answered by the whole job
    value = jobq * args.steps / (ms_max / 1e3)

    # ---------------- e2e through the host API (pinned host buffers); skipped under
    # --profile-steps so that an ncu capture holds exactly the K timed searches
    if args.profile_steps:
        if rank == 0:
            print(json.dumps({"profile_steps": args.steps, "ms_per_step": ms_max / args.steps,
                              "stage_ms_per_step": {k_: v / args.steps for k_, v in stage_ms.items()},
                              "stats": stats}), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    qh = torch.from_numpy(Qh).pin_memory()
    oh = (torch.empty((nq, k), dtype=torch.int64).pin_memory(),
          torch.empty((nq, k), dtype=torch.float32).pin_memory())
    qn, on = qh.numpy(), (oh[0].numpy(), oh[1].numpy())
    g.search_host(qn, k, nprobe, budget, out=on, workspace=ws)
    e2e_ms = 0.0
    for s in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        g.search_host(qn, k, nprobe, budget, out=on, workspace=ws)
        b.record(st)
        torch.cuda.synchronize()
        e2e_ms += a.elapsed_time(b)
    te = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = jobq * args.steps / (float(te.item()) / 1e3)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel (algorithmic work / event-timed duration)
    # Per step (the counters of the last timed search): the main scan estimates the probed
    # objects outside the sample, M LUT lookups each (PQ); the re-rank gathers |S*| raw rows.
    info = g.info
    code_bytes = info.m if info.kind == 1 else info.dpad // 8 + 8
    row_bytes = info.d * (1 if info.raw_u8 else 4)
    # (in sweep order the sample pass also estimates the lists filling its last work item)
    main_objs = stats["probed"] - max(stats["sampled"], stats.get("sample_pass", 0))
    peak, peak_src = peaks()
    scan_ms = stage_ms["scan"] / args.steps
    rr_ms = stage_ms["rerank"] / args.steps
    # the scan's second roofline: its M LUT reads per object are conflict-free shared-memory
    # loads, bounded by the measured lookup rate (bbc_measure_smem_lookups, best of 3)
    lds_peak = max(measure_smem_lookups(0) for _ in range(3))
    lookups = main_objs * (info.m if info.kind == 1 else 0)
    per = {
        # SURVEY 8(d) / north_star: algorithmic code bytes (M per object of the main pass) over
        # the scan's event-timed duration, against the measured HBM copy peak
        "scan": {"ms": scan_ms, "bound": "hbm", "bytes": main_objs * code_bytes, "peak_GBs": peak,
                 "lds_view": {"lookups": lookups, "peak_Glookups": lds_peak,
                              "Glookups": lookups / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else None,
                              "peak_source": "measured: bbc_measure_smem_lookups (conflict-free "
                                             "LDS.32 + FADD, 32 warps/SM, best of 3)"}},
        "rerank": {"ms": rr_ms, "bound": "hbm", "bytes": stats["candidates"] * row_bytes,
                   "peak_GBs": peak},
    }
    if per["scan"]["lds_view"]["Glookups"]:
        per["scan"]["lds_view"]["frac"] = per["scan"]["lds_view"]["Glookups"] / lds_peak
    if stats.get("rerank_list_batches", 0) > 0:
        # list-order re-rank: the rows a list's queries share are read from L2, so the bound is
        # the L2 -> SM read bandwidth, measured on this GPU by bbc_measure_l2_read
        l2 = max(measure_l2_read_gbs(0) for _ in range(5))        # a peak: best of 5
        per["rerank"].update({"bound": "l2", "peak_GBs": l2,
                              "pipe": "L2 -> SM reads (rows shared by the queries of a list)",
                              "peak_source": "measured: bbc_measure_l2_read (48 MiB L2-resident, "
                                             "best of 4/8/16 loads in flight x 4/8 CTAs/SM, best of 5)"})
    for v in per.values():
        v["GBs"] = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 else None
        v["frac"] = v["GBs"] / v["peak_GBs"] if v["GBs"] else None
        if "hbm_view" in v and v["ms"] > 0:
            hv = v["hbm_view"]
            hv["GBs"] = hv["code_bytes"] / (v["ms"] / 1e3) / 1e9
            hv["frac"] = hv["GBs"] / peak
    if info.kind == 1 and getattr(info, "nbits", 8) == 4:
        # 4-bit PQ scan: lookups by byte permutes on the integer ALU pipe (64 lanes/clk/SM);
        # the kernel spends 16 ALU operations per 8 lookups (bbc_pq4.cuh), so the pipe's lookup
        # peak is 148 x 64 / 2 per clock at the measured max SM clock
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                mhz = float(json.load(f)["sm_max_mhz"])
        except Exception:
            mhz = 1965.0
        lk = main_objs * info.m
        pk = 148 * 32 * mhz * 1e6 / 1e9                      # G lookups / s
        per["scan"] = {"ms": scan_ms, "bound": "alu", "unit": "Glookup/s",
                       "pipe": "integer ALU: PRMT/LOP3/SHF, 16 ops per 8 lookups",
                       "lookups": lk, "peak_Glookups": pk,
                       "Glookups": lk / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else None,
                       "hbm_view": {"code_bytes": main_objs * info.m / 2, "peak_GBs": peak}}
        per["scan"]["frac"] = per["scan"]["Glookups"] / pk if per["scan"]["Glookups"] else None
        per["scan"]["GBs"] = None
    if info.kind != 1:
        # RaBitQ scan = list-major integer GEMM on the tensor cores (kind::i8): 2 ops per code bit
        # per (object, query) pair of the Push pass, against the int8 dense peak (measured bf16
        # TFLOP/s x the nominal int8/bf16 ratio 2, B200_PROFILING.md)
        ops = 2.0 * stats["probed"] * info.dpad
        tpk = tensor_peak_tops("i8")
        per["scan"] = {"ms": scan_ms, "bound": "tensor", "pipe": "tcgen05.mma kind::i8",
                       "ops": ops, "peak_TOPs": tpk,
                       "TOPs": ops / (scan_ms / 1e3) / 1e12 if scan_ms > 0 else None,
                       "hbm_view": {"code_bytes": main_objs * code_bytes, "peak_GBs": peak}}
        per["scan"]["frac"] = per["scan"]["TOPs"] / tpk if per["scan"]["TOPs"] else None
        per["scan"]["GBs"] = None
    dom = max(per, key=lambda n: per[n]["ms"])
    traffic = measured_traffic(cfg.name, nprobe, budget, dom)
    tens = per[dom]["bound"] == "tensor"
    lkp = "Glookups" in per[dom]
    roof = {"bound": per[dom]["bound"], "kernel": dom,
            "achieved": per[dom]["TOPs"] if tens else per[dom]["Glookups"] if lkp else per[dom]["GBs"],
            "peak": per[dom]["peak_TOPs"] if tens else per[dom]["peak_Glookups"] if lkp else per[dom]["peak_GBs"],
            "unit": "TOP/s" if tens else "Glookup/s" if lkp else "GB/s", "frac": per[dom]["frac"],
            "traffic": traffic,
            "peak_source": (f"{peak_src}: MEASURED_PEAKS.json hbm_gbs (copy)" if per[dom]["bound"] == "hbm" else
                            "measured: bbc_measure_l2_read (48 MiB L2-resident, best of 4/8/16 loads in flight x 4/8 CTAs/SM, best of 5)"
                            if per[dom]["bound"] == "l2" else
                            "measured bf16 TFLOP/s x 2 (int8/bf16 nominal ratio)" if tens else
                            "derived: 148 SMs x 64 ALU lanes/clk / 2 ops per lookup x sm_max_mhz (DESIGN.md 5)"),
            "per_kernel": per,
            "stage_ms_per_step": {k_: v / args.steps for k_, v in stage_ms.items()}}

    # ---------------- recall on sampled queries (fp64 brute-force ground truth)
    rq = min(args.recall_queries, nq)
    rec = None
    if rq > 0 and not args.profile_steps:
        X = database_in_id_order(path)
        gi, gd = groundtruth.cached_topk(f"{cfg.name}_{os.path.basename(path)}", Qh[:rq], X, k,
                                         datagen.cache_dir(), metric=cfg.metric)
        ids = out[0][:rq].cpu().numpy()
        ex = groundtruth.exact_of(Qh[:rq], X, ids, metric=cfg.metric)
        rec = {"recall": groundtruth.recall(ids, ex, gi, gd),
               "relative_error": (groundtruth.relative_error(out[1][:rq].cpu().numpy(), gd)
                                  if cfg.metric == "l2" else None),
               "metric": cfg.metric, "queries": rq}
    cpu = None
    if world == 1 and not args.no_cpu_baseline and not args.profile_steps:
        cpu = cpu_baseline(cfg, path, nprobe, budget, args.cpu_seconds, args.cpu_workers)

    line = {
        "metric": json.loads('"' + METRIC + '"'),
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if lists else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "N": cfg.N, "d": cfg.d, "quantizer": cfg.kind,
                   "M": cfg.M, "nlist": cfg.nlist, "nq_per_gpu": nq, "k": k, "nprobe": nprobe,
                   "budget": budget,
                   "parallelism": (f"list-sharded x{world} (NCCL)" if lists else f"query-sharded x{world}"),
                   "l2": "flushed (256 MB write) between timed steps",
                   **({} if args.bound_rerank is None else
                      {"rerank": f"Algorithm 3 (bound-aware, eps0 = {args.bound_rerank}, "
                                 f"{args.bound_rerank_gathers}-order gathers)"}),
                   **({"rerank": "Algorithm 4 (early re-ranking: exact distances below tau_pred straight after the scan pass)",
                       "early_objects_per_query": stats["early_objects"] / nq,
                       "early_candidates_per_query": stats["early_candidates"] / nq}
                      if args.early_rerank else {}),
                   "probed_per_query": stats["probed"] / nq,
                   "candidates_per_query": stats["candidates"] / nq,
                   "microbatches": stats["microbatches"],
                   **({} if rec is None else rec)},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": nq * cfg.d * 4,
                "d2h_bytes_per_step": nq * k * 12},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def bucket_sweep(cfg, path, g, nprobe, budget):
    """Exp-6 / Table 4 analog: the number of buckets (equal-width B, or m
    equal-depth buckets remapped from the 255 cells) against the candidate superset size, recall
    and device time, at the workload's operating point."""
    import torch
    X = database_in_id_order(path)
    Q = synth.generate_queries(cfg)
    q = torch.from_numpy(Q).cuda()
    rq = 100
    gi, gd = groundtruth.cached_topk(f"{cfg.name}_{os.path.basename(path)}", Q[:rq], X, cfg.k,
                                     datagen.cache_dir(), metric=cfg.metric)
    st = torch.cuda.current_stream()
    ws = g.workspace(len(Q), cfg.k, nprobe, budget)
    # equal-width B, then the paper's n_ew = 256 -> m equal-depth remap at its m values (56, 80,
    # 92, 120 for its datasets) and a few more
    runs = [(B, 0) for B in (1, 3, 7, 15, 31, 63, 127, 255)] + [(255, m) for m in (8, 16, 56, 80, 92, 120, 255)]
    for B, m in runs:
        g.set_buckets(B)
        g.set_remap(m)
        g.search(q, cfg.k, nprobe, budget, workspace=ws)
        torch.cuda.synchronize()
        ms = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            ids, _ = g.search(q, cfg.k, nprobe, budget, workspace=ws)
            b.record(st)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        idn = ids[:rq].cpu().numpy()
        r = groundtruth.recall(idn, groundtruth.exact_of(Q[:rq], X, idn, metric=cfg.metric), gi, gd)
        s = g.last_stats()
        print(json.dumps({"bucket_sweep": cfg.name, "B": B, "equal_depth_m": m, "nprobe": nprobe, "budget": budget,
                          "ms": float(np.median(ms)), "qps": len(Q) / (float(np.median(ms)) / 1e3),
                          "superset_over_budget": s["candidates"] / len(Q) / budget,
                          "recall": round(r, 4)}), flush=True)
    g.set_buckets(255)
    g.set_remap(0)


args_sweep_nprobe = None
args_sweep_budget = None


def sweep(cfg, path, g, rank):
    import torch
    X = database_in_id_order(path)
    Q = synth.generate_queries(cfg)
    q = torch.from_numpy(Q).cuda()
    rq = 100
    gi, gd = groundtruth.cached_topk(f"{cfg.name}_{os.path.basename(path)}", Q[:rq], X, cfg.k,
                                     datagen.cache_dir(), metric=cfg.metric)
    st = torch.cuda.current_stream()
    # nprobe in {1, 1.5, 2, 3, 4} x the config's (here also 1.25 and 1.75, and
    # 6 and 8 for the weakly clustered C2/C3), budget in {1, 1.5, 2, 3, 4} x k (and 1.25, 1.75)
    mults = args_sweep_nprobe or (1, 1.25, 1.5, 1.75, 2, 3, 4, 6, 8)
    for nprobe in sorted({int(round(m * cfg.nprobe)) for m in mults}):
        if nprobe > cfg.nlist or nprobe > 2048:
            continue
        for bm in (args_sweep_budget or (1.0, 1.25, 1.5, 1.75, 2.0, 3.0, 4.0)) + ((6.0, 8.0) if cfg.pq_bits == 4 else ()):
            budget = int(bm * cfg.k)
            ws = g.workspace(len(Q), cfg.k, nprobe, budget, max_bytes=60 << 30)
            g.search(q, cfg.k, nprobe, budget, workspace=ws)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            ids, d2 = g.search(q, cfg.k, nprobe, budget, workspace=ws)
            b.record(st)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            idn = ids[:rq].cpu().numpy()
            r = groundtruth.recall(idn, groundtruth.exact_of(Q[:rq], X, idn, metric=cfg.metric), gi, gd)
            s = g.last_stats()
            print(json.dumps({"sweep": cfg.name, "nprobe": nprobe, "budget": budget,
                              "recall": round(r, 4), "qps": len(Q) / (ms / 1e3), "ms": ms,
                              "probed_per_q": s["probed"] / len(Q),
                              "cand_per_q": s["candidates"] / len(Q)}), flush=True)


if __name__ == "__main__":
    main()
