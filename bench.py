#!/usr/bin/env python
"""bench.py -- BC TEPS of the B200 hot path (one JSON line on rank 0).

Default workload = BASELINE.json config 4: R-MAT scale 20, EF 16
((a,b,c,d) = (.57,.19,.19,.05), seed 1, label permutation), 65,536 source
vertices sampled uniformly without replacement among non-isolated vertices
(sample seed 2).  A *step* is one pass of the whole hot path (forward sweep,
backward sweep, BC update -- every SURVEY §8(a) row -- plus the NCCL BC
all-reduce when N > 1) over `--sources-per-gpu` sources per GPU (weak
scaling: at N = 8 one step is the full 65,536-source job).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat20]
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...   # the CPU oracle, same metric/config

value = sources processed by all ranks x m / max-over-ranks device time, m =
unique undirected edges (Eq.7; reading R16 -- the paper's
own published TEPS count 2m, reported beside as "teps_paper_convention").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

_emit = None  # set by main(): writes one JSON line to the real stdout

METRIC = "BC TEPS (sources·m/s) at 1/2/4/8 B200; % HBM roofline; speedup vs CPU oracle"

CONFIGS = {
    # name: (generator, kwargs, total sources (None = all), sources per gpu per step, prune)
    "rmat20": ("rmat", dict(scale=20, ef=16), 65536, 8192, False),
    "rmat12": ("rmat", dict(scale=12, ef=16), None, 4096, False),
    "rmat16": ("rmat", dict(scale=16, ef=16), None, 65536, False),
    "rmat16p": ("rmat", dict(scale=16, ef=16), None, 65536, True),
    "grid": ("grid", dict(R=512, C=512), None, 8192, False),
    "rmat23": ("rmat", dict(scale=23, ef=16), 16384, 2048, False),
}


def make_graph(cfg):
    import graphgen as gg

    kind, kw, _, _, _ = CONFIGS[cfg]
    if kind == "rmat":
        return gg.rmat(kw["scale"], kw["ef"], seed=1, permute=True)
    return gg.grid(kw["R"], kw["C"])


def source_list(g, cfg):
    import graphgen as gg

    total = CONFIGS[cfg][2]
    if total is None:
        # "all sources": isolated vertices contribute 0 and are not counted in TEPS (R15, R21)
        return g.non_isolated()
    return gg.sample_sources(g, total, seed=2)


def workload_name(cfg):
    return {
        "rmat20": "rmat20_ef16_sampled65536",
        "rmat12": "rmat12_ef16_all_sources",
        "rmat16": "rmat16_ef16_all_sources_prune_off",
        "rmat16p": "rmat16_ef16_all_sources_prune_on",
        "grid": "grid512x512_all_sources",
        "rmat23": "rmat23_ef16_sampled16384",
    }[cfg]


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def clocks_sampler_start(idx):
    if os.environ.get("BC_BENCH_NO_CLOCKS"):  # diagnosis only: the line then carries no clocks
        return None, None, ""
    try:
        f = open(os.path.join(ROOT, "gpurun_out", f"clocks_rank{idx}.csv") if os.path.isdir(
            os.path.join(ROOT, "gpurun_out")) else os.devnull, "w")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        p = subprocess.Popen(["nvidia-smi", "-i", str(idx), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                              "-lms", "500"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        # wait for the first sample: nvidia-smi's start-up (NVML init, driver
        # locks) must not overlap the timed region -- it stalls CUDA launches
        first = p.stdout.readline()
        return p, f, first
    except Exception:
        return None, None, ""



def clocks_sampler_stop(h):
    p, f, first = h
    if p is None:
        return None
    p.terminate()
    try:
        out, _ = p.communicate(timeout=5)
    except Exception:
        p.kill()
        out = ""
    out = first + out
    if f:
        f.write(out)
        f.close()
    sm, mx, reasons = [], [], set()
    for line in out.strip().splitlines():
        parts = [x.strip() for x in line.split(",")]
        if len(parts) < 9:
            continue
        try:
            sm.append(float(parts[1]))
            mx.append(float(parts[2]))
        except ValueError:
            continue
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for nm, val in zip(names, parts[5:9]):
            if val.lower().startswith("active"):
                reasons.add(nm)
    if not sm:
        return None
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
            "samples": len(sm)}


def cpu_baseline(g, sources, budget_s=15.0):
    """The oracle as it stands, on this host's cores, on a bounded sample."""
    import oracle

    # every core this process may run on (torchrun sets OMP_NUM_THREADS=1 per
    # rank; the oracle leg runs on rank 0 alone and gets the whole host)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else oracle.num_threads()
    rng = np.random.default_rng(7)
    pool = rng.permutation(sources)
    first = pool[:cores]
    t0 = time.perf_counter()
    oracle.bc(g, first, threads=cores)
    t1 = time.perf_counter() - t0
    done, tot_t = len(first), t1
    rounds = int(max(0, budget_s - t1) / max(t1, 1e-3))
    if rounds > 0:
        more = pool[cores: cores * (1 + rounds)]
        t0 = time.perf_counter()
        oracle.bc(g, more, threads=cores)
        tot_t += time.perf_counter() - t0
        done += len(more)
    return {"value": done * g.m / tot_t, "unit": "TEPS", "cores": cores, "kind": "oracle",
            "sample": f"{done} of the workload's sources (uniform sample, seed 7), {tot_t:.1f} s"}


def run_reference(args, cfg):
    """--impl reference: the CPU oracle timed as it stands (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    g = make_graph(cfg)
    S = source_list(g, cfg)
    # every core this process may run on (torchrun sets OMP_NUM_THREADS=1 per
    # rank; the oracle leg runs on rank 0 alone and gets the whole host)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else oracle.num_threads()
    # bounded sample per step: one source per core (whole run stays within minutes)
    per_step = cores if cfg not in ("rmat12",) else min(len(S), 16 * cores)
    rng = np.random.default_rng(11)
    pool = rng.permutation(S)
    for i in range(args.warmup):
        oracle.bc(g, pool[:per_step], threads=cores)
    t0 = time.perf_counter()
    done = 0
    for i in range(args.steps):
        chunk = pool[(i * per_step) % len(pool):][:per_step]
        oracle.bc(g, chunk, threads=cores)
        done += len(chunk)
    t = time.perf_counter() - t0
    v = done * g.m / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TEPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_name(cfg), "n": g.n, "m": g.m,
                                            "sources_per_step": per_step},
            "cpu_baseline": {"value": v, "unit": "TEPS", "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} sources per step (one per core), uniform sample seed 11"},
            "e2e": {"value": v, "unit": "TEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    _emit(line)


def algorithmic_bytes(st, K):
    """Algorithmic bytes per kernel class for the roofline.
    A = sum of reached adjacency, D = DAG lane-edges, N = reached
    lane-vertices over the run; K lanes share each column read.

    "survey": SURVEY.md §8(d-iii) exactly, B_alg = A(8/k + 2 b_d) + 16 D + 24 n
      with b_d = 1/8 (one mask bit per lane), split per sweep as
        fwd  A(4/K + 1/8) + 8 D + 16 N   (sigma per DAG edge; depth 4 + sigma 8 + BC 4 per vertex)
        bwd  A(4/K + 1/8) + 8 D +  8 N   (coef per DAG edge; coef written once)
    "rows": what this build's rows actually move, sb = bytes per stored
      sigma value (2 for 16-bit rows, 4 for 32-bit, 8 for fp64):
        fwd  A(4/K + 1/8) + sb D + sb N
        bwd  A(4/K + 1/8) + 8 D + (sb + 16) N  (sigma and accumulator read, accumulator re-zeroed)"""
    A, D, N = st["adj_reached"], st["dag_edges"], st["reached"]
    nb, b = st["narrow_batches"], max(1, st["batches"])
    mid = st.get("mid_batches", 0)
    sb = (2.0 * nb + 4.0 * mid + 8.0 * max(0, b - nb - mid)) / b
    scan = A * (4.0 / K + 1.0 / 8.0)
    return {"survey": {"fwd": scan + 8.0 * D + 16.0 * N, "bwd": scan + 8.0 * D + 8.0 * N},
            "rows": {"fwd": scan + sb * D + sb * N, "bwd": scan + 8.0 * D + (sb + 16.0) * N}}


def slices_bytes(st):
    """Slices mode (one source per CTA, both sweeps in one kernel): SURVEY.md
    §8(d-iii) unbatched, k = 1 and an int32 depth (b_d = 4):
    B_alg = A (8 + 8) + 16 D + 24 n over the run."""
    A, D, N = st["adj_reached"], st["dag_edges"], st["reached"]
    return A * 16.0 + 16.0 * D + 24.0 * N


def main():
    # the one JSON line goes to the real stdout; everything else the process
    # prints there (NCCL's version banner, library chatter) goes to stderr
    json_fd = os.dup(1)
    os.dup2(2, 1)
    global _emit
    _emit = lambda line: os.write(json_fd, (json.dumps(line) + "\n").encode())  # noqa: E731
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="rmat20", choices=sorted(CONFIGS))
    ap.add_argument("--sources-per-gpu", type=int, default=0)
    ap.add_argument("--lane-words", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    cfg = args.config
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_1602_00963_b200 as bcb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _, _, total, per_gpu_default, prune = CONFIGS[cfg]
    per_gpu = args.sources_per_gpu or per_gpu_default

    g = make_graph(cfg)
    S = source_list(g, cfg)
    per_gpu = min(per_gpu, len(S))
    G = bcb.Graph.from_csr(g, device=local)
    if prune:
        G.prune_degree1()
        import graphgen as gg  # noqa: F401
        om, rm, _, _ = G.pruning()
        S = S[rm[S] == 0]
        per_gpu = min(per_gpu, len(S))
        # a pruned source s stands for s and its omega(s) removed children (R13):
        # count |S+| = sum (1 + omega(s)) sources of the equivalent unpruned job
        splus_factor = float((1 + om[S].astype(np.float64)).sum()) / len(S)
    else:
        splus_factor = 1.0
    if args.lane_words:
        G.set_option(bcb.OPT_LANE_WORDS, args.lane_words)
    stream = torch.cuda.current_stream()
    out = torch.empty(g.n, dtype=torch.float64, device=f"cuda:{local}")

    def step_sources(i):
        start = ((i * world + rank) * per_gpu) % len(S)
        idx = (start + np.arange(per_gpu)) % len(S)
        return S[idx]

    def one_step(i, profile=False):
        G.compute(step_sources(i), out=out, stream=stream)
        if world > 1:
            dist.all_reduce(out)

    for i in range(args.warmup):
        one_step(i)
    torch.cuda.synchronize()

    sampler = clocks_sampler_start(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    agg = {"fwd_ms": 0.0, "bwd_ms": 0.0, "bwd_push_ms": 0.0, "bwd_fin_ms": 0.0, "fwd_launches": 0,
           "bwd_launches": 0, "kernel_launches": 0, "reached": 0, "adj_reached": 0, "dag_edges": 0,
           "num_sources": 0, "levels_total": 0, "batches": 0, "narrow_batches": 0, "narrow_fallbacks": 0,
           "mid_batches": 0}
    kbytes = {"survey": {"fwd": 0.0, "bwd": 0.0}, "rows": {"fwd": 0.0, "bwd": 0.0}}
    sbytes = 0.0
    lanes = 0
    e0.record(stream)
    for i in range(args.steps):
        one_step(args.warmup + i)
        st = G.stats()
        lanes = st["lanes"]
        for k in ("kernel_launches", "reached", "adj_reached", "dag_edges", "num_sources", "levels_total",
                  "batches", "narrow_batches", "narrow_fallbacks", "mid_batches"):
            agg[k] += st[k]
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clocks_sampler_stop(sampler)
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    sources_all = per_gpu * world * args.steps * splus_factor
    value = sources_all * g.m / (ms_max / 1e3)

    # ---- end to end through the C ABI with HOST buffers (sources H2D, BC D2H inside the region)
    e2e = None
    if not args.no_e2e:
        host_out = np.empty(g.n, np.float64)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.steps):
            G.compute(step_sources(args.warmup + i), out=host_out)
            if world > 1:
                tt = torch.from_numpy(host_out).to(f"cuda:{local}")
                dist.all_reduce(tt)
                host_out = tt.cpu().numpy()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        e2e = {"value": sources_all * g.m / dt, "unit": "TEPS", "h2d_bytes_per_step": 4 * per_gpu * world
               + (8 * g.n * world if world > 1 else 0), "d2h_bytes_per_step": 8 * g.n * world}

    # ---- per-kernel roofline pass: the same steps again with one batch
    # pipeline (kernels serialised on one stream, so a launch's CUDA-event
    # duration is that kernel's own; inside the timed region the pipelines
    # overlap kernels) and the library's per-launch events (BC_OPT_PROFILE)
    G.set_option(bcb.OPT_STREAMS, 1)
    G.set_option(bcb.OPT_PROFILE, 1)
    prof_steps = min(args.steps, 4)
    prof_ms = 0.0
    for i in range(prof_steps):
        torch.cuda.synchronize()
        one_step(args.warmup + i)
        torch.cuda.synchronize()
        st = G.stats()
        prof_ms += st["total_ms"]
        for k in ("fwd_ms", "bwd_ms", "bwd_push_ms", "bwd_fin_ms", "fwd_launches", "bwd_launches"):
            agg[k] += st[k]
        for model, d in algorithmic_bytes(st, st["lanes"]).items():
            for kk, vb in d.items():
                kbytes[model][kk] += vb
        sbytes += slices_bytes(st)
    G.set_option(bcb.OPT_PROFILE, 0)
    G.set_option(bcb.OPT_STREAMS, 0)

    if rank == 0:
        pk, pk_kind = peaks()
        peak = pk["hbm_gbs"]
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(cfg, {})
        except Exception:
            tr = {}
        slices = agg["bwd_ms"] == 0.0 and agg["fwd_ms"] > 0.0
        if not slices:
            kms = {"fwd": agg["fwd_ms"], "bwd": agg["bwd_ms"]}
            names = {"fwd": "lanes_level_kernel<fwd> (pull; + hub finalize)",
                     "bwd": "lanes_push_kernel<bwd> (+ finalize kernels)"}
            dom = max(kms, key=lambda k: kms[k])
            dom_ms = kms[dom]
            gbs = lambda b, t: b / (t / 1e3) / 1e9 if t > 0 else 0.0  # noqa: E731
            achieved = gbs(kbytes["survey"][dom], dom_ms)
            rows_ach = gbs(kbytes["rows"][dom], dom_ms)
            timing = (f"CUDA events around every launch on its stream, {prof_steps} of the timed steps re-run with one "
                      "batch pipeline (serialised kernels; the timed region overlaps up to 8 pipelines)")
            model = ("SURVEY.md §8(d-iii): per batch A(4/K + 1/8) + 8 D + 8 N for the backward, "
                     "A(4/K + 1/8) + 8 D + 16 N for the forward (A reached adjacency, D DAG lane-edges, N reached "
                     "lane-vertices; bench stats)")
            kern = {k: {"ms": kms[k], "alg_gb": kbytes["survey"][k] / 1e9, "gbs": gbs(kbytes["survey"][k], kms[k]),
                        "rows_model_gb": kbytes["rows"][k] / 1e9, "rows_model_gbs": gbs(kbytes["rows"][k], kms[k])}
                    for k in kms}
            extra = {"rows_model": {"achieved": rows_ach, "frac": rows_ach / peak,
                                    "formula": "bytes this build's rows move (16-bit sigma rows): backward "
                                               "A(4/K + 1/8) + 8 D + (sb + 16) N, forward A(4/K + 1/8) + sb D + sb N"}}
            limiter = ("L2 atomic units for the fp64 reds, unevenly loaded across slices (backward); row-gather "
                       "latency (forward); DESIGN.md §5")
        else:
            dom, dom_ms = "slices", agg["fwd_ms"]
            names = {"slices": "slices_lowdeg_sm_kernel (2-bit shared-memory state; forward + backward sweeps of "
                               "one source per CTA)"}
            achieved = sbytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
            timing = (f"CUDA events around the one persistent slices launch of each step, {prof_steps} of the timed "
                      "steps re-run (the same launch as in the timed region)")
            model = "SURVEY.md §8(d-iii) unbatched, k = 1, int32 depth: A (8 + 8) + 16 D + 24 n per run"
            kern = {"slices": {"ms": dom_ms, "alg_gb": sbytes / 1e9, "gbs": achieved}}
            extra = {}
            limiter = ("latency: each level's dependent L2 load chain (queue -> row -> sigma) and the barrier that "
                       "ends it (DESIGN.md §4.3); DRAM traffic is below the algorithmic bytes")
        td = tr.get(dom, {})
        traffic = td.get("dram_bytes_per_launch")
        if traffic is not None and td.get("time_s"):
            extra["dram_frac_ncu"] = td["dram_bytes"] / td["time_s"] / 1e9 / peak
        sect = {k: td[k] for k in ("ld_sectors_per_request", "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
                                   "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_red.sum",
                                   "smsp__inst_executed_op_global_red.sum") if k in td}
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": names[dom], "model": model, "limiter": limiter,
                "peak_kind": pk_kind, "kernel_share_of_step": dom_ms / prof_ms if prof_ms > 0 else None,
                "timing": timing, "kernels": kern, "sector_efficiency": sect or None,
                "ncu_source": td and tr.get("source"), **extra}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(g, S)
        if slices:
            l2_note = ("no flush: per step 296 CTAs sweep 296 sources at a time, each writing 20 B per reached vertex "
                       "(sigma/coef slot, queue, BC) -- 5.2 MB per source, far beyond L2 across a step")
        else:
            l2_note = ("inputs exceed L2 (per step: CSR 4*2m B streamed per level, sigma rows 2*K*n B per level, "
                       "accumulators 8*K*n B); no flush")
        line = {
            "metric": METRIC, "value": value, "unit": "TEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "n": g.n, "m": g.m, "sources_total": len(S),
                       "sources_per_gpu_per_step": per_gpu, "lanes_per_batch": lanes, "pruning": prune,
                       "teps_sources": "|S+| (pruned: each source counts 1 + omega(s))" if prune else "|S|",
                       "parallelism": f"source-sharded x{world} + NCCL BC all-reduce" if world > 1 else "1 GPU",
                       "l2": l2_note},
            "teps_paper_convention": 2 * value,
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": agg["kernel_launches"],
            "stats": {k: agg[k] for k in ("levels_total", "batches", "narrow_batches", "narrow_fallbacks",
                                          "reached", "adj_reached", "dag_edges")},
        }
        _emit(line)
    if world > 1:
        dist.destroy_process_group()
    G.close()


if __name__ == "__main__":
    main()
