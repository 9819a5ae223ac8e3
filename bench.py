#!/usr/bin/env python3
"""Benchmark: uncompressed-equivalent words/s for word count + inverted index
(BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c3|c4|c5] [--shard-mode files|corpus]

One step = word count + inverted index over the corpus (both tasks, render-
ordered compact results), through the public gt_run_many call (on <= 64
owned files the two tasks share ONE device pass).  Corpora are composed
deterministically on every box (paper_2106_06889_b200/corpus.py, synthetic
Zipfian, seeded).

N = 1 (the driver's headline): config C2 = BASELINE configs[1] (1 GB-
equivalent, 16 large files, depth-24 rule DAG with heavy multi-parent
sharing).  value = W / t_step, t_step the device time of the step measured
with CUDA events on the library's stream (DAG resident in HBM, L2 flushed
with a 256 MiB memset between steps); e2e = W / wall time of the public
C-ABI path from the pinned host GTDC buffer (gt_open: H2D + device DAG
build, gt_run_many, D2H of the results, gt_close).

N > 1 (torchrun, one process per GPU, NCCL): by default config C3 =
BASELINE configs[2] (100k small files) sharded by token-balanced file ranges
of ONE corpus with the DAG replicated on every GPU (strong scaling, SURVEY
§8e); the vocabulary count vectors are summed with an NCCL all-reduce (exact
integer sums), rank 0 assembles the global word count, every rank copies its
own files' inverted-index records to pinned host memory.  Device time is the
max over ranks.  The matching single-GPU point is `bench.py --config c3`.
--shard-mode corpus (weak scaling, opt-in): every rank owns its own C2-shaped
16-file partition of a collection (rank 0's is the N = 1 workload).

--impl reference times the reference's algorithm on the host cores through
the CPU restatement in oracle/ (the reference itself is pure Python/numba and
does not travel to the GPU box; its relation to the restatement is measured
in profiles/r2_reference_numba.json), same corpus, config, step and warm-up.
"""

from __future__ import annotations

import argparse
import csv
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
L2_NOTE = "L2 flushed between steps (256 MiB memset on the GPU arm)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="default: c2 at N = 1, c3 (strong scaling) at N > 1")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="one profiled step, print kernel table")
    ap.add_argument("--shard-mode", default="files", choices=["files", "corpus"],
                    help="N>1: a token-balanced file range of ONE corpus per rank (strong, default) "
                         "or each rank its own 16-file partition of a collection (weak)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.config is None:
        a.config = "c2" if world == 1 or a.shard_mode == "corpus" else "c3"
    return a


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


def corpus(args, seed=None):
    from paper_2106_06889_b200.corpus import compose, config_spec
    return compose(config_spec(args.config, seed=seed, scale=args.scale))


def config_dict(args, info: dict, world: int, corpus_mode: bool, W_total: int) -> dict:
    """The workload description — identical in both arms (same_config)."""
    par = (f"{world} corpus partitions x 1 GPU (weak)" if corpus_mode and world > 1 else
           f"{world} file-range shards, DAG replicated (strong)" if world > 1 else "1 shard")
    return {"workload": f"{args.config}: word count + inverted index per step", "scale": args.scale,
            "l2": L2_NOTE, "R": info["num_rules"], "E": info["total_elements"], "L0": info["root_len"],
            "E_sub": info["sub_pairs"], "E_own": info["own_pairs"], "W": W_total, "F": info["num_files"],
            "V": info["num_words"], "depth": info["depth"],
            "rho": info["words"] / max(1, info["total_elements"]), "parallelism": par}


# ---------------------------------------------------------------------------
# roofline: SURVEY.md §8(d) algorithmic bytes
# ---------------------------------------------------------------------------

def alg_bytes_task(task: str, info: dict, O: int) -> int:
    """SURVEY.md §8(d) algorithmic bytes of ONE task over the whole DAG: the
    compressed grammar read once plus the outputs written once, at device
    widths (u32 ids/freqs, u64 weights/counts).  O = output records of the
    task (the inverted index's (word, file) pairs)."""
    R, Es, Eo, L0, V, F = (info[k] for k in ("num_rules", "sub_pairs", "own_pairs", "root_len", "num_words",
                                              "num_files"))
    dag = 8 * Es + 8 * Eo + 4 * L0
    if task in ("wordcount", "sort"):
        return dag + 16 * (R + 1) + 16 * R + 8 * V
    if task == "invertedindex":
        return dag + 16 * R + 4 * (F + 1) + 8 * O
    if task == "termvector":
        return dag + 16 * R + 4 * (F + 1) + 12 * O
    raise ValueError(task)


def alg_bytes_step(info: dict, O_ii: int) -> tuple[int, int]:
    """(fused, per-task sum) algorithmic bytes of one bench step.  The fused
    pass (gt_run_many) reads the DAG ONCE for both tasks, so its compulsory
    bytes are the DAG + offsets once, both rule rows (weight and presence,
    16 B each: written once, read once) and both outputs — the conservative
    figure `roofline.frac` uses.  The per-task sum is SURVEY §8(d) applied
    to each task separately (the DAG counted twice)."""
    R, Es, Eo, L0, V, F = (info[k] for k in ("num_rules", "sub_pairs", "own_pairs", "root_len", "num_words",
                                              "num_files"))
    fused = 8 * Es + 8 * Eo + 4 * L0 + 16 * (R + 1) + 16 * R + 16 * R + 8 * V + 4 * (F + 1) + 8 * O_ii
    per_task = alg_bytes_task("wordcount", info, 0) + alg_bytes_task("invertedindex", info, O_ii)
    return fused, per_task


def build_stamp() -> str | None:
    p = ROOT / "paper_2106_06889_b200" / "_build" / "stamp"
    return p.read_text().strip() if p.exists() else None


def ncu_evidence(symbol: str):
    """The dominant kernel's DRAM bytes per launch and ncu DRAM throughput
    (% of peak) from the newest committed metrics capture
    (profiles/*_metrics.csv, tools/profile_round.sh), and whether that
    capture was taken of the library built from these sources
    (profiles/<tag>_stamp.txt == the build stamp)."""
    caps = sorted((ROOT / "profiles").glob("*_metrics.csv"), key=lambda p: p.name)

    def same(cap):
        f = cap.with_name(cap.name.replace("_metrics.csv", "_stamp.txt"))
        return f.exists() and f.read_text().strip() == build_stamp()
    # a capture of this very build first, then the newest by name
    caps = [c for c in caps if not same(c)] + [c for c in caps if same(c)]
    for cap in reversed(caps):
        rows = list(csv.reader(cap.open()))
        try:
            i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
        except StopIteration:
            continue
        hdr = rows[i]
        per = {}
        for r in rows[i + 1:]:
            d = dict(zip(hdr, r))
            if symbol not in d.get("Kernel Name", ""):
                continue
            m = d.get("Metric Name", "")
            try:
                v = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(d["Metric Unit"], 1.0)
            e = per.setdefault(d["ID"], {})
            if m.startswith("dram__bytes_"):
                e["bytes"] = e.get("bytes", 0.0) + v * scale
            elif m == "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed":
                e["pct"] = v
        per = {k: v for k, v in per.items() if "bytes" in v}
        if not per:
            continue
        stamp_f = cap.with_name(cap.name.replace("_metrics.csv", "_stamp.txt"))
        same = stamp_f.exists() and stamp_f.read_text().strip() == build_stamp()
        return {"traffic": statistics.mean(e["bytes"] for e in per.values()),
                "dram_frac_ncu": statistics.mean(e.get("pct", 0.0) for e in per.values()) / 100.0,
                "source": cap.name, "same_build": same, "launches": len(per)}
    return None


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def cpu_reference_steps(blob, steps, warmup, workers):
    """The reference algorithm on host cores (oracle/ restatement): warm-up
    steps, then timed steps of word count + inverted index."""
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


def reference_numba_note():
    """The real reference (numba) vs the restatement, measured once per round
    in the build container (tools/reference_numba_probe.py)."""
    p = ROOT / "profiles" / "r2_reference_numba.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return {"source": f"profiles/{p.name}", "where": "build container, same composed corpus and step",
            "reference_numba_words_per_s": {k: v["words_per_s"] for k, v in d["reference_numba"].items()},
            "port_words_per_s_same_host": d["port"]["words_per_s"],
            "port_speedup_over_reference_numba": d["port_speedup_over_reference_numba"],
            "reference_build_dag_s": d["reference_build_dag_s"]}


def run_reference(args, rank, world):
    if rank != 0:
        return
    blob, stats = corpus(args)
    cores = os.cpu_count() or 1
    info, times, init_s, e2e_s = cpu_reference_steps(blob, args.steps, args.warmup, cores)
    W = info["words"]
    t = statistics.mean(times)
    corpus_mode = world > 1 and args.shard_mode == "corpus"
    line = {
        "metric": METRIC, "value": W / t, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak" if corpus_mode or world == 1 else "strong",
        "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (composed Zipfian grammar; composer in paper_2106_06889_b200/corpus.py)",
        "config": config_dict(args, info, world, corpus_mode, W),
        "cpu_baseline": {"value": W / t, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"whole {args.config} corpus, {args.steps} steps of wordcount+invertedindex "
                                   f"after {args.warmup} warm-up steps"},
        # the contract's reference-arm e2e: the line's own value and unit
        "e2e": {"value": W / t, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # (the reference algorithm end to end from the GTDC bytes: load +
        # build_dag + both tasks, once — the counterpart of our e2e)
        "e2e_incl_build": {"value": W / e2e_s, "unit": UNIT},
        "init_ms": init_s * 1e3,
        "reference_numba": reference_numba_note(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import config_spec
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
    corpus_mode = world > 1 and args.shard_mode == "corpus"

    # rank r's input: the whole corpus with a token-balanced file range
    # (strong scaling, replicated DAG) or its own 16-file partition of a
    # collection (corpus mode, weak scaling; rank 0's is the N=1 workload)
    base = config_spec(args.config, scale=args.scale)
    blob, stats = corpus(args, seed=base.seed + (rank if corpus_mode else 0))
    pinned = torch.empty(len(blob), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = np.frombuffer(blob, dtype=np.uint8)
    src = (pinned.data_ptr(), len(blob))

    dag = DeviceDag(src, device=local)
    info = dag.info
    V = info["num_words"]
    if world == 1 or corpus_mode:
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
        """word count + inverted index through gt_run_many (one shared device
        pass on <= 64 owned files), + the all-reduce of the vocab counts and
        rank-0 assembly when N > 1; returns (device ms, launches, d2h bytes,
        inverted-index records of this rank)."""
        dev_ms, launches, d2h, n_ii = 0.0, 0, 0, 0
        rs = d.run_many_raw([gt._abi.TASK_IDS[t] for t in TASKS])
        for (r, v), task in zip(rs, TASKS):
            dev_ms += v.device_ms
            launches += v.kernel_launches
            d2h += v.d2h_bytes
            if task == "invertedindex":
                n_ii = int(v.n)
            d.free_raw(r)
        if dist:
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
        return dev_ms, launches, d2h, n_ii

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
    # Per-kernel CUDA events cost host and device time, so the timed region
    # runs without them; the SAME K steps are then run again with per-launch
    # events on the library stream (gt_profile) for the kernel table and the
    # roofline.
    step_ms, launches, n_ii = [], 0, 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            dag.flush_l2()
            dag.sync()
            ms, nl, _, n_ii = step(dag)
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

    # ---- roofline: the dominant kernel of the step, SURVEY §8(d) bytes
    K = args.steps
    peak, peak_src = peaks()
    k_dom = max(rep, key=lambda k: rep[k][1]) if rep else None
    roof = None
    if k_dom:
        n_l, ms_l = rep[k_dom]
        kern_s = ms_l / K / 1e3
        fused_bytes, per_task_bytes = alg_bytes_step(info, n_ii)
        fused = k_dom == "k_td_levels" and n_l == K  # one shared pass per step (td_wc_ii_records)
        if fused:
            b, scope = fused_bytes, "kernel"
        else:  # the step's compulsory bytes over the step's device time
            b, scope, kern_s = per_task_bytes, "step", ms_per_step / 1e3
        ach = b / kern_s / 1e9
        ev = ncu_evidence("WcPresMode") if fused else None
        roof = {"bound": "hbm", "kernel": k_dom, "scope": scope,
                "cuda_symbol": "k_segred1_levels<1024, 1, gt::WcPresMode, ...>" if fused else None,
                "launches_per_step": n_l / K,
                "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "alg_bytes_per_step": b, "alg_bytes_source": "SURVEY.md §8(d); bench.py alg_bytes_step",
                "frac_survey_per_task_sum": per_task_bytes / kern_s / 1e9 / peak,
                "alg_bytes_per_task_sum": per_task_bytes,
                "traffic": ev["traffic"] if ev else None,
                "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                "dram_frac_ncu": ev["dram_frac_ncu"] if ev else None,
                "ncu_source": ev["source"] if ev else None,
                "ncu_same_build": ev["same_build"] if ev else None,
                "kernel_ms_per_step": kern_s * 1e3,
                "share_of_step": (ms_l / K) / (sum(prof_ms) / K), "profiled_step_ms": sum(prof_ms) / K,
                "peak_source": peak_src,
                "kernel_timing": "CUDA events per launch on the library stream over K profiled steps "
                                 "(same workload, run after the unprofiled timed region)"}
        # the single-parent contraction (contract.cu): built on the DAG's
        # second top-down run (a warm-up step), then every timed step runs
        # over the heads only — the §8(d) bytes above are the whole DAG's,
        # the lists the pass actually reads are these
        cs = [int(x) for x in dag.dag_array("cont_sizes")]
        levels = info["td_levels"]
        if cs:
            heads, cedges, levels = cs
            R, Eo, V, F = (info[k] for k in ("num_rules", "own_pairs", "num_words", "num_files"))
            moved = 12 * cedges + 12 * Eo + 32 * heads + 8 * V + 4 * (F + 1) + 8 * n_ii
            roof["contraction"] = {"heads": heads, "rules": R, "head_edges": cedges, "td_edges": info["td_edges"],
                                   "levels": levels, "td_levels": info["td_levels"],
                                   "list_bytes_per_step": moved,
                                   "frac_list_bytes": moved / kern_s / 1e9 / peak}
        if fused:
            # the top-down pass is a chain of grid-barrier-separated levels:
            # its time per level against the measured per-level floor
            # (grid barrier + item load + L2 gather + RED, tools/barrier_probe.cu)
            roof["latency_model"] = {"levels_per_launch": levels,
                                     "us_per_level_upper": (ms_l / n_l) * 1e3 / max(1, levels),
                                     "floor_us_per_level": [2.0, 2.7], "barrier_us": 1.26,
                                     "floor_source": "profiles/r1_barrier_probe.txt"}
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
        if world > 1 and not corpus_mode:
            d.set_files(lo, hi)
        t1 = time.perf_counter()
        _, _, nb, _ = step(d)
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
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if corpus_mode or world == 1 else "strong", "vs_baseline": None, "dtype": "u64",
            "data": f"synthetic (composed Zipfian grammar, seed {base.seed}{'+rank' if corpus_mode else ''}; "
                    "composer in paper_2106_06889_b200/corpus.py)",
            "config": config_dict(args, info, world, corpus_mode, W_total),
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": W_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h_bytes, "ms_per_step": e2e_s * 1e3,
                    "breakdown_ms": {k: round(statistics.mean(p[j] for p in parts) * 1e3, 4)
                                     for j, k in enumerate(("gt_open", "tasks_incl_d2h", "gt_close"))}},
            "gpu_launches": launches, "clocks": clk.summary(), "wall_s_timed_region": wall,
            # the single-parent contraction is a derived index of
            # the DAG, built once during the DAG's second run (a warm-up step):
            # every timed step computes both tasks from the root seeds over it;
            # every e2e repetition is a first run on a fresh DAG, without it
            "derived_index": {"contraction": roof.get("contraction") if roof else None,
                              "built_in": "warm-up step 2 (gt_run_many call 2 on the DAG)",
                              "e2e_uses_it": False},
            "init_ms": info["init_ms"], "W_rank0": W_rank, "kernels": kernel_table,
            "reference_numba": reference_numba_note(),
        }
        if world > 1 and not corpus_mode:
            line["scaling_note"] = f"single-GPU point of this workload: bench.py --config {args.config}"
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
