#!/usr/bin/env python
"""Benchmark: IsoRank CFG-pair similarities/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "c2"): all-pairs ISO similarity over a
seeded synthetic corpus of 2,000 CFGs with 16-64 basic blocks, fp64 (the
reference's arithmetic), alpha 0.85, tol 1e-9, max_iter 1000.  A step is one
full all-pairs pass: K(K+1)/2 = 2,001,000 unique alignments (ISO is
symmetric; the K x K matrix is filled by mirroring), each run to convergence.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun, one rank per GPU): the upper triangle is split into N
cost-balanced unit ranges (no data-path collective while aligning), and the
per-rank score tiles are assembled with one NCCL all-gather (the path's only
exchange); value = all units / max-over-ranks device time ("strong").

--impl reference: the reference's CPU algorithm (the pinned C restatement in
oracle/, all host threads) on bounded samples of the same workload; rank 0
only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "CFG-pair similarities/sec (IsoRank, all-pairs, device-timed)"
UNIT = "pairs/s"
SEED = 2
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: 64 fp64 FMA/clk/SM at max clock
NOMINAL_SMEM_TBS = 148 * 128 * 1.965e9 / 1e12       # 37.2: 128 B/clk/SM


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64")
    ap.add_argument("--graphs", type=int, default=None, help="override corpus size (debug)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=6.0, help="wall budget of the CPU sample")
    return ap.parse_args()


def corpus(args):
    from paper_1707_02423_b200 import synth
    cfg = dict(synth.CONFIGS[args.config])
    if args.graphs:
        cfg["n_graphs"] = args.graphs
    mats = synth.random_corpus(cfg["n_graphs"], cfg["lo"], cfg["hi"], seed=SEED, weighting=cfg["weighting"])
    return cfg, mats


def workload_desc(cfg, args, k):
    return {"workload": f"{args.config}: all-pairs IsoRank over {k} synthetic CFGs, "
                        f"{cfg['lo']}-{cfg['hi']} basic blocks ({cfg['weighting']} edge weights)",
            "graphs": k, "unique_alignments": k * (k + 1) // 2, "alpha": 0.85, "tol": 1e-9,
            "max_iter": 1000, "l2": "flushed (256 MiB write) between timed steps",
            "parallelism": f"dp{args.gpus} (cost-balanced triangle ranges + NCCL all-gather)"}


# ----------------------------------------------------------------- CPU arm
def cpu_sample(mats, seconds, seed=0):
    """C restatement of the reference (oracle/, pthreads over all host cores) on
    a random sample of the workload's unordered pairs, grown until `seconds`."""
    from oracle import ffi
    from paper_1707_02423_b200.corpus import pack
    threads = os.cpu_count() or 1
    packed = pack(mats)
    k = len(mats)
    rng = np.random.default_rng(seed)
    done, t_total, batch = 0, 0.0, max(threads, 8)
    while t_total < seconds:
        ia = rng.integers(0, k, batch).astype(np.int32)
        ib = rng.integers(0, k, batch).astype(np.int32)
        t0 = time.perf_counter()
        ffi.iso_batch(packed, ia, ib, threads=threads)
        t_total += time.perf_counter() - t0
        done += batch
        batch = min(batch * 2, 4096)
    return done / t_total, threads, done, t_total


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, mats = corpus(args)
    threads = os.cpu_count() or 1
    per_step = max(2.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
    for w in range(args.warmup):
        cpu_sample(mats, per_step / 4, seed=100 + w)
    vals, pairs, secs = [], 0, 0.0
    for s in range(args.steps):
        v, thr, n, t = cpu_sample(mats, per_step, seed=s)
        vals.append(v)
        pairs += n
        secs += t
    value = pairs / secs
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded CFG corpus, reference edge-weighting rules)",
            "config": workload_desc(cfg, args, len(mats)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{pairs} random unordered pairs of the workload over {args.steps} steps "
                                       f"(~{per_step:.0f} s each); C restatement of sasscfg isorank "
                                       "(oracle/isorank_ref.c, pinned to reference golden vectors)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                clk, mxc = float(f[1]), float(f[2])
            except ValueError:
                continue
            mx = mxc
            sm.append(clk)
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [c for c in sm if c > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1707_02423_b200 as P
    from paper_1707_02423_b200 import _native as nat
    from paper_1707_02423_b200 import workload

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    cfg, mats = corpus(args)
    k = len(mats)
    prm = nat.params(0.85, 1e-9, 1000, args.precision)
    corpus_d = P.DeviceCorpus(mats, device=local)
    n_units = corpus_d.n_units()
    bounds = corpus_d.split(world)
    u0, u1 = int(bounds[rank]), int(bounds[rank + 1])
    chunk = int(max(bounds[1:] - bounds[:-1]))
    d_lin = torch.empty(chunk, dtype=torch.float64, device=dev)
    it_lin = torch.zeros(chunk, dtype=torch.int32, device=dev)
    gathered = torch.empty(world * chunk, dtype=torch.float64, device=dev) if world > 1 else None
    full = torch.empty(n_units, dtype=torch.float64, device=dev)
    scores = torch.empty((k, k), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    sp = st.cuda_stream

    def step(ev=None):
        if ev is not None:
            ev[0].record(st)
        nat.check(nat.lib.cfgsim_allpairs_range(corpus_d.handle, u0, u1, 0, nat.C.byref(prm), nat.ptr(d_lin),
                                                nat.ptr(it_lin), sp))
        if ev is not None:
            ev[1].record(st)
        if world > 1:
            dist.all_gather_into_tensor(gathered, d_lin)
            for r in range(world):  # drop the per-rank padding
                a, b = int(bounds[r]), int(bounds[r + 1])
                full[a:b].copy_(gathered[r * chunk:r * chunk + (b - a)])
            src = full
        else:
            src = d_lin
        nat.check(nat.lib.cfgsim_allpairs_scatter(corpus_d.handle, 0, nat.ptr(src), None, nat.ptr(scores), None, sp))
        if ev is not None:
            ev[2].record(st)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # algorithmic work of this rank's units (iteration counts from the run itself)
    iters_local = it_lin[: u1 - u0].cpu().numpy()
    perm, a_idx, b_idx = workload.triangle_units(corpus_d.n_nodes)
    ga, gb = perm[a_idx[u0:u1]], perm[b_idx[u0:u1]]
    n_nodes = corpus_d.n_nodes
    N = np.maximum(n_nodes[ga], n_nodes[gb])
    S, Z = workload.operator_stats(mats, int(n_nodes.max()))
    flops_rank = float(workload.pair_flops(N, S[ga, N], S[gb, N], Z[ga, N], Z[gb, N], iters_local).sum())
    smem_rank = float(workload.pair_smem_bytes(N, iters_local, 8 if args.precision == "fp64" else 4).sum())

    launches0 = nat.launch_count()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for s in range(args.steps):
            flush.fill_(s)  # write 256 MiB (> 126 MB L2) outside the timed events
            step(evs[s])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = nat.launch_count() - launches0
    t_step = sum(e[0].elapsed_time(e[2]) for e in evs) / 1e3
    t_kern = sum(e[0].elapsed_time(e[1]) for e in evs) / 1e3
    tt = torch.tensor([t_step, t_kern, flops_rank, smem_rank], dtype=torch.float64, device=dev)
    if world > 1:
        mx = tt[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tt[2:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        tt = torch.cat([mx, sm])
    t_step, t_kern, flops_all, smem_all = (float(x) for x in tt.cpu())
    value = n_units * args.steps / t_step
    kern_time_per_step = t_kern / args.steps
    achieved_tf = flops_all / kern_time_per_step / 1e12 / world  # per GPU
    achieved_smem = smem_all / kern_time_per_step / 1e12 / world

    # ---- e2e: the public API with host inputs (pack + H2D + compute + D2H)
    e2e = None
    if not args.no_e2e and world == 1:
        tms = [P.TransitionMatrix(f"k{i:05d}.synth.c2", m, tuple(range(len(m))), P.ROW_STOCHASTIC)
               for i, m in enumerate(mats)]
        P.pairwise(tms, P.MeasureId.ISO, device=local, precision=args.precision)  # warm
        times = []
        for s in range(args.steps):
            flush.fill_(s)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pm = P.pairwise(tms, P.MeasureId.ISO, device=local, precision=args.precision)
            times.append(time.perf_counter() - t0)
        e2e = {"value": n_units / statistics.mean(times), "unit": UNIT,
               "h2d_bytes_per_step": int(P.corpus.packed_bytes(P.pack(tms))),
               "d2h_bytes_per_step": int(pm.scores.nbytes), "api": "paper_1707_02423_b200.pairwise(..., ISO)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, thr, n, t = cpu_sample(mats, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": thr, "kind": "port",
               "sample": f"{n} random unordered pairs of this workload, {t:.1f} s wall on {thr} threads; "
                         "C restatement of sasscfg isorank (oracle/isorank_ref.c)"}

    traffic = None
    tf = REPO / "profiles" / "traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(f"{args.config}_{args.precision}")
        except (ValueError, OSError):
            traffic = None

    if rank == 0:
        peak = NOMINAL_FP64_TFLOPS if args.precision == "fp64" else 2 * NOMINAL_FP64_TFLOPS
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_step / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic (seeded CFG corpus following the reference's listing/edge-weighting rules)",
            "config": workload_desc(cfg, args, k),
            "roofline": {"bound": "fp64-pipe" if args.precision == "fp64" else "fp32-pipe",
                         "achieved": achieved_tf, "peak": peak, "unit": "TFLOP/s", "frac": achieved_tf / peak,
                         "traffic": traffic,
                         "peak_source": "nominal 148 SM x 64 fp64 FMA/clk x 2 x 1.965 GHz (MEASURED_PEAKS.json "
                                        "has no fp64/smem figure)",
                         "flops_per_step": flops_all, "kernel_ms_per_step": 1e3 * kern_time_per_step,
                         "smem": {"achieved": achieved_smem, "peak": NOMINAL_SMEM_TBS, "unit": "TB/s",
                                  "frac": achieved_smem / NOMINAL_SMEM_TBS}},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
