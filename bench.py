#!/usr/bin/env python3
"""Benchmark: uncompressed-equivalent words/s for word count + inverted index
(BASELINE.json metric) on the C2 corpus (configs[1]: 1 GB-equivalent, 16
large files, depth-24 rule DAG with heavy multi-parent sharing), composed
deterministically on every box (synthetic, seed 2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = word count + inverted index over the whole corpus (both tasks,
render-ordered compact results).  value = W / t_step with t_step the device
time of the step measured with CUDA events on the library's stream (DAG
resident in HBM, L2 flushed between steps); e2e = W / wall time of the
public C-ABI path from the pinned host GTDC buffer (gt_open: H2D + device
DAG build, both gt_runs, D2H of the results, gt_close).

--impl reference times the reference's algorithm on the host cores through
the CPU restatement in oracle/ (the reference itself is pure Python/numba and
does not travel to the GPU box), on the same corpus, metric and step.
Multi-GPU (torchrun, one process per GPU, NCCL): by default (--shard-mode
corpus, weak scaling) the collection is partitioned by files into N
C2-shaped 16-file partitions, one grammar per GPU (rank 0's partition is the
N=1 workload); the vocabulary count vectors are summed with an NCCL
all-reduce (exact integer sums) and rank 0 assembles the global word count,
per-file inverted-index outputs stay on their rank.  --shard-mode files
(strong scaling) shards ONE corpus by token-balanced file ranges with the
DAG replicated (gt_set_files).  Device time is the max over ranks.
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

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "uncompressed-equivalent words/sec for word count & inverted index, 1–8 B200"
UNIT = "words/s"
TASKS = ("wordcount", "invertedindex")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="one profiled step, print kernel table")
    ap.add_argument("--shard-mode", default="corpus", choices=["corpus", "files"],
                    help="N>1: each rank owns its own 16-file partition of the collection "
                         "(weak scaling, default) or a file range of one corpus (strong)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *exc):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            out, _ = self.p.communicate(timeout=10)
            self.rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
        else:
            self.rows = []

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for n, v in zip(names, r[4:8]):
                    if v.strip() == "Active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def composed(args):
    from paper_2106_06889_b200.corpus import compose, config_spec
    spec = config_spec(args.config, scale=args.scale)
    blob, stats = compose(spec)
    return blob, stats


def task_columns(task: str, files: int) -> int:
    """Weight-row width of a task's top-down pass (word.cu td_levels)."""
    if task in ("wordcount", "sort"):
        return 1
    if task == "invertedindex":
        return max(1, (files + 63) // 64)  # presence bitsets
    return max(1, files)  # per-file counts


FUSED_REDUCE_MAX = 4 << 20  # word.cu kFusedReduceMax: the C = 1 reduce runs inside the top-down launch


def alg_bytes(kernel: str, info: dict, files: int, tasks=TASKS) -> float | None:
    """Algorithmic (compulsory) bytes of one bench step for a kernel, summed
    over the step's tasks: every input element read once,
    every output element written once, at device widths (u32 ids/freqs, u64
    weights/counts).  k_td_level: the non-root parent edges (child, parent,
    freq: 12 B) + every rule row written once and read once (16·C B);
    k_reduce_words: the word-major own pairs (12 B) + every rule row read once
    + the dense (C x V) output written once.  For C = 1 (word count, inverted
    index of <= 64 files) on grammars with at most FUSED_REDUCE_MAX own pairs
    the reduce runs inside the top-down launch, so k_td_levels carries both
    terms."""
    R, Eo, V, Te = info["num_rules"], info["own_pairs"], info["num_words"], info["td_edges"]
    tot = 0
    for t in tasks:
        C = task_columns(t, files)
        if kernel in ("k_td_level", "k_td_levels"):
            tot += 12 * Te + 16 * C * (R - 1)
            if C == 1 and Eo <= FUSED_REDUCE_MAX:
                tot += 12 * Eo + 8 * R + 8 * V
        elif kernel == "k_reduce_words":
            tot += 12 * Eo + 8 * C * R + 8 * C * V
        else:
            return None
    return tot


def ncu_traffic(kernel: str, tasks=TASKS):
    """DRAM bytes per step of the dominant kernel from the newest committed
    ncu metrics capture (profiles/*metrics.csv, tools/profile_round.sh):
    mean dram__bytes_read.sum + dram__bytes_write.sum per launch of each
    task's pass, summed over the step's passes; None without a capture."""
    import csv
    caps = sorted((ROOT / "profiles").glob("*metrics.csv"))
    if not caps or kernel not in ("k_td_level", "k_td_levels"):
        return None, None
    rows = list(csv.reader(caps[-1].open()))
    try:
        i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    except StopIteration:
        return None, None
    hdr = rows[i]
    per = {}
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")
        if "TdRows" not in name or not d.get("Metric Name", "").startswith("dram__bytes_"):
            continue
        mode = "SumMode" if "SumMode" in name else "OrMode"
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(d["Metric Unit"], 1.0)
        per.setdefault(mode, {}).setdefault(d["ID"], 0.0)
        per[mode][d["ID"]] += float(d["Metric Value"].replace(",", "")) * scale
    if not per:
        return None, None
    mean = {m: sum(v.values()) / len(v) for m, v in per.items()}
    modes = ["SumMode" if t in ("wordcount", "sort") else "OrMode" for t in tasks]
    if not all(m in mean for m in modes):
        return None, None
    return sum(mean[m] for m in modes), caps[-1].name


def cpu_reference_steps(blob, steps, warmup, workers):
    """The reference algorithm on host cores (oracle/ restatement)."""
    from oracle.oracle import OracleDag
    import paper_2106_06889_b200 as gt
    t0 = time.perf_counter()
    dag = OracleDag(blob, workers=workers)
    init_s = time.perf_counter() - t0
    cfg = gt.TraversalConfig()
    times = []
    for i in range(warmup + steps):
        t = time.perf_counter()
        for task in TASKS:
            gt.run_compact(dag, task, cfg)
        if i >= warmup:
            times.append(time.perf_counter() - t)
    # e2e: deserialize + build_dag + both tasks from host bytes
    t = time.perf_counter()
    d2 = OracleDag(blob, workers=workers)
    for task in TASKS:
        gt.run_compact(d2, task, cfg)
    e2e_s = time.perf_counter() - t
    return dag.info, times, init_s, e2e_s


def run_reference(args, rank):
    if rank != 0:
        return
    blob, stats = composed(args)
    cores = os.cpu_count() or 1
    info, times, init_s, e2e_s = cpu_reference_steps(blob, args.steps, min(args.warmup, 1), cores)
    W = info["words"]
    t = statistics.mean(times)
    line = {
        "metric": METRIC, "value": W / t, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (composed Zipfian grammar, seed 2)",
        "config": {"workload": f"{args.config}: word count + inverted index per step", "scale": args.scale,
                   "R": info["num_rules"], "E": info["total_elements"], "W": W,
                   "F": info["num_files"], "V": info["num_words"], "depth": info["depth"],
                   "rho": W / max(1, info["total_elements"])},
        "cpu_baseline": {"value": W / t, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"whole {args.config} corpus, {args.steps} steps of wordcount+invertedindex"},
        "e2e": {"value": W / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "init_ms": init_s * 1e3,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import compose, config_spec
    from paper_2106_06889_b200.device import DeviceDag
    from paper_2106_06889_b200.shard import shard_ranges
    # GT_BENCH_BACKEND=gloo lets a 1-GPU box exercise the N>1 code path
    # (ranks share device local % device_count); real runs use NCCL
    backend = os.environ.get("GT_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    corpus_mode = world == 1 or args.shard_mode == "corpus"

    # rank r's input: its own 16-file partition of the collection (corpus
    # mode, weak scaling; rank 0's is the N=1 workload) or the whole corpus
    # with a token-balanced file range (files mode, strong scaling)
    base = config_spec(args.config, scale=args.scale)
    seed = base.seed + (rank if corpus_mode else 0)
    blob, stats = compose(config_spec(args.config, seed=seed, scale=args.scale))
    pinned = torch.empty(len(blob), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = np.frombuffer(blob, dtype=np.uint8)
    src = (pinned.data_ptr(), len(blob))

    dag = DeviceDag(src, device=local)
    info = dag.info
    V = info["num_words"]
    if corpus_mode:
        lo, hi = 0, info["num_files"]
        W_rank = info["words"]
    else:
        toks = dag.dag_array("segment_token_counts")
        lo, hi = shard_ranges(toks, world)[rank]
        dag.set_files(lo, hi)
        W_rank = int(toks[lo:hi].sum())
    W_total = W_rank
    if dist:
        t = torch.tensor([W_rank], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        W_total = int(t.item())
        if not corpus_mode:
            assert W_total == info["words"]

    def counts_view(d):
        ptr = d.device_word_counts_ptr()

        class _CAI:  # __cuda_array_interface__ view of the library's u64[V] counts
            __cuda_array_interface__ = {"shape": (V,), "typestr": "<i8", "data": (ptr, False),
                                        "version": 3}
        return torch.as_tensor(_CAI(), device="cuda")

    def step(d):
        """word count (+ all-reduce of the vocab counts + rank-0 assembly when
        N > 1) and inverted index; returns (device ms, launches, d2h bytes)."""
        dev_ms, launches, d2h = 0.0, 0, 0
        for task in TASKS:
            r, v = d.run_raw(gt._abi.TASK_IDS[task])
            dev_ms += v.device_ms
            launches += v.kernel_launches
            d2h += v.d2h_bytes
            d.free_raw(r)
            if task == "wordcount" and dist:
                t = counts_view(d)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dist.all_reduce(t)  # exact integer sums over NVLink
                e1.record()
                e1.synchronize()
                dev_ms += e0.elapsed_time(e1)
                if rank == 0:  # the global word-count result, render order
                    c = d.assemble_counts(t.data_ptr(), gt._abi.TASK_IDS["wordcount"])
                    dev_ms += c.timings["device_ms"]
                    launches += c.timings["kernel_launches"]
                    d2h += c.timings["d2h_bytes"]
        return dev_ms, launches, d2h

    if args.profile_only:
        dag.profile(True)
        step(dag)
        rep = dag.profile_report()
        dag.profile(False)
        for k, (n, ms) in sorted(rep.items(), key=lambda kv: -kv[1][1]):
            print(f"{k:40s} {n:6d} {ms:10.4f} ms")
        return

    for _ in range(args.warmup):
        step(dag)

    # ---- timed region: K steps, L2 flushed between steps (outside the events).
    # Per-kernel CUDA events cost host and device time (~25 % of a C2 step),
    # so the timed region runs without them; the SAME K steps are then run
    # again with per-launch events on the library stream (gt_profile) for the
    # kernel table and the roofline.
    step_ms, launches = [], 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            dag.flush_l2()
            dag.sync()
            ms, nl, _ = step(dag)
            step_ms.append(ms)
            launches += nl
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    dag.profile(True)
    dag.profile_report()
    prof_ms = []
    for _ in range(args.steps):
        dag.flush_l2()
        dag.sync()
        prof_ms.append(step(dag)[0])
    torch.cuda.synchronize()
    rep = dag.profile_report()
    dag.profile(False)
    tot_ms = sum(step_ms)
    if dist:
        t = torch.tensor([tot_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        dist.barrier()
    ms_per_step = tot_ms / args.steps
    value = W_total / (ms_per_step / 1e3)

    # ---- dominant kernel of the timed region + roofline
    K = args.steps
    Fo = hi - lo
    named = {k: v for k, v in rep.items() if alg_bytes(k, info, Fo) is not None}
    peak, peak_src = peaks()
    roof = None
    if named:
        k_dom = max(named, key=lambda k: named[k][1])
        n_l, ms_l = named[k_dom]
        b = alg_bytes(k_dom, info, Fo)  # per step
        ach = b * K / (ms_l / 1e3) / 1e9
        # the committed ncu capture is of the default workload only
        traffic, traffic_src = ncu_traffic(k_dom) if args.config == "c2" and args.scale == 1.0 else (None, None)
        roof = {"bound": "hbm", "kernel": k_dom,
                # phase label -> the CUDA symbol in the ncu launch list
                "cuda_symbol": {"k_td_levels": "k_segred1_levels"}.get(k_dom, k_dom),
                "launches_per_step": n_l / K,
                "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "traffic_unit": "bytes per step (ncu dram read+write)",
                "traffic_source": traffic_src, "alg_bytes_per_step": b, "kernel_ms_per_step": ms_l / K,
                "share_of_step": (ms_l / K) / (sum(prof_ms) / K), "profiled_step_ms": sum(prof_ms) / K,
                "peak_source": peak_src,
                "kernel_timing": "CUDA events per launch on the library stream over K profiled steps "
                                 "(same workload, run after the unprofiled timed region)",
                # the top-down pass is a chain of grid-barrier-separated levels:
                # its time per level against the measured per-level floor
                # (grid barrier + item load + L2 gather + RED, tools/barrier_probe.cu)
                "latency_model": {"levels_per_launch": info["td_levels"],
                                  "us_per_level_upper": (ms_l / n_l) * 1e3 / max(1, info["td_levels"]),
                                  "floor_us_per_level": [2.0, 2.7], "barrier_us": 1.26,
                                  "floor_source": "profiles/r1_barrier_probe.txt"}}
    kernel_table = {k: {"launches_per_step": n / K, "ms_per_step": round(ms / K, 5)} for k, (n, ms) in
                    sorted(rep.items(), key=lambda kv: -kv[1][1])[:12]}

    # ---- e2e through the public C-ABI from pinned host bytes: gt_open (H2D +
    # device DAG build) + the step (+ collective) + D2H of results + gt_close
    e2e_times, d2h_bytes, parts = [], 0, []
    for i in range(max(3, min(args.steps, 20)) + 1):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = DeviceDag(src, device=local)
        if not corpus_mode:
            d.set_files(lo, hi)
        t1 = time.perf_counter()
        _, _, nb = step(d)
        t2 = time.perf_counter()
        d.close()
        el = time.perf_counter() - t0
        if i:
            e2e_times.append(el)
            parts.append((t1 - t0, t2 - t1, el - (t2 - t0)))
            d2h_bytes = nb
    e2e_s = statistics.mean(e2e_times)
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = len(blob)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        _, times, _, _ = cpu_reference_steps(blob, 3, 1, cores)
        tc = statistics.mean(times)
        cpu = {"value": W_rank / tc, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"whole {args.config} corpus, 3 steps of wordcount+invertedindex (oracle/ C restatement)"}

    if rank == 0:
        par = (f"{world} corpus partitions x 1 GPU (weak)" if corpus_mode and world > 1 else
               f"file-range shards x{world}, DAG replicated (strong)" if world > 1 else "1 GPU")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if corpus_mode else "strong", "vs_baseline": None, "dtype": "u64",
            "data": f"synthetic (composed Zipfian grammar, seed {base.seed}{'+rank' if corpus_mode and world > 1 else ''}; "
                    "composer in paper_2106_06889_b200/corpus.py)",
            "config": {"workload": f"{args.config}: word count + inverted index per step",
                       "scale": args.scale, "l2": "flushed between steps (256 MiB memset)",
                       "R": info["num_rules"], "E": info["total_elements"],
                       "L0": info["root_len"], "E_sub": info["sub_pairs"],
                       "E_own": info["own_pairs"], "E_td": info["td_edges"], "W": W_total,
                       "W_rank0": W_rank, "F": info["num_files"], "V": V, "depth": info["depth"],
                       "rho": info["words"] / max(1, info["total_elements"]),
                       "parallelism": par},
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": W_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h_bytes, "ms_per_step": e2e_s * 1e3,
                    "breakdown_ms": {k: round(statistics.mean(p[j] for p in parts) * 1e3, 4)
                                     for j, k in enumerate(("gt_open", "tasks_incl_d2h", "gt_close"))}},
            "gpu_launches": launches, "clocks": clk.summary(), "wall_s_timed_region": wall,
            "init_ms": info["init_ms"], "kernels": kernel_table,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
