#!/usr/bin/env python
"""Benchmark: BFS GTEPS (harmonic mean over the 64 seeded roots) on the
RCM-reordered Kronecker graph of BASELINE.json configs[2] (scale 26,
edgefactor 16) -- the largest configuration that fits one B200.

A "step" is one sweep of the 64 seeded roots (reference bench.py:124-134),
each root one BFS (BfsEngine.run, engine.py:518-604) over the HBM-resident
RCM graph with the L2 flushed before it.  Per-root time = the mean of that
root's device traversal time over the K timed sweeps; the headline per-root
TEPS numerator is the raw input pairs in the root's component (reference
bench.py:186-189, 336-338; the paper's / north star's convention), the dedup
numerator (traversed edges, engine.py:599-600) is reported alongside; value =
harmonic mean over the 64 roots (bench.py:235-237).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--scale S] [--graph kronecker|chunglu]
                  [--impl ours|reference] [--replicas]

Rank 0 prints ONE JSON line.  ``--impl reference`` times the CPU reference
path (the oracle's C + OpenMP port of BfsEngine, modes hybrid_reduced -- the
paper's full method -- and hybrid, on all host cores) on the same config; it
never loads the CUDA library.  ``--gpus N`` (torchrun): the 1D vertex-block
partition (one traversal per root over all GPUs, strong scaling);
``--replicas`` instead shards the 64 roots over per-GPU graph replicas
(throughput mode, labelled as such).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BFS GTEPS (harmonic mean, 64 roots) on RCM-reordered Kronecker graphs"
UNIT = "GTEPS"
N_ROOTS = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5, help="timed sweeps of the 64 roots")
    ap.add_argument("--warmup", type=int, default=3, help="untimed sweeps (W >= 3)")
    ap.add_argument("--graph", default="kronecker", choices=["kronecker", "chunglu"],
                    help="kronecker (configs[0..3]) or chunglu (configs[4]: n=2^24, gamma 2.1, seed 7)")
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--seed", type=int, default=None, help="default: 1 (kronecker), 7 (chunglu)")
    ap.add_argument("--mode", default="hybrid")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-roots", type=int, default=0, help="only run N roots once (for ncu)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: shard the 64 independent roots over per-GPU graph replicas (throughput mode). "
                         "Default: ONE traversal per root over the 1D vertex-block partition of all GPUs")
    ap.add_argument("--dump-levels", default=None,
                    help="write every timed root's level records (direction, executed, n_f, m_f, scanned, byte-model "
                         "bytes, device seconds) to this JSON file: the data roofline.by_direction is computed from")
    ap.add_argument("--partitioned", action="store_true",
                    help="force the 1D-partition path (device-side exchange) also at one GPU (loopback check)")
    ap.add_argument("--validate-roots", type=int, default=N_ROOTS,
                    help="validate this many roots' trees on the GPU (outside the timed region)")
    a = ap.parse_args()
    if a.seed is None:
        a.seed = 7 if a.graph == "chunglu" else 1
    a.warmup = max(a.warmup, 0)
    a.steps = max(a.steps, 1)
    return a


def workload(args):
    """(config.workload name, data description) of the graph being measured."""
    if args.graph == "chunglu":
        return (f"chunglu-n2^{args.scale}-g2.1-d20-rcm-bfs",
                f"synthetic Chung-Lu power law (generator.py ChungLuParams recipe, seed {args.seed})")
    return (f"kronecker-s{args.scale}-ef{args.edgefactor}-rcm-bfs",
            f"synthetic Kronecker (reference generator, seed {args.seed})")


def hmean(x):
    x = np.asarray(x, dtype=np.float64)
    return float(x.size / np.sum(1.0 / x))


# ---------------------------------------------------------------------------
# byte model, per root, from the level records


def level_bytes(levels, n_dev: int, n_plus_dev: int):
    """SURVEY.md 8(d) byte model without its per-vertex level term (the engine,
    like the reference, keeps no level array unless asked to), per level:
    TD level: |F|*(4 queue + 16 offsets) + 4*E_TD + n_next*(4 parent + 4 queue)
    BU level: 3*(n_dev/8) + 8*U + 4*C + n_next*(4 parent).
    Returns [(executed direction, bytes, device seconds)] per level."""
    out = []
    reached = 0
    for i, r in enumerate(levels):
        reached += r.n_f
        n_next = levels[i + 1].n_f if i + 1 < len(levels) else 0
        d = getattr(r, "executed_direction", None) or r.direction  # the work actually done
        if d == "top_down":
            b = r.n_f * 20 + 4 * r.scanned_edges + n_next * 8
        else:
            U = max(n_plus_dev - reached, 0)
            b = 3 * (n_dev // 8) + 8 * U + 4 * r.scanned_edges + n_next * 4
        out.append((d, int(b), float(getattr(r, "wall_time", 0.0))))
    return out


def algorithmic_bytes(levels, n_dev: int, n_plus_dev: int) -> int:
    return int(sum(b for _, b, _ in level_bytes(levels, n_dev, n_plus_dev)))


def by_direction(per_root, peak):
    """Roofline per step kind (top-down / bottom-up levels of all timed roots):
    sum of algorithmic bytes / sum of level device time (%globaltimer spans,
    the grid barrier closing each level included)."""
    out = {}
    for d, key in (("top_down", "top_down"), ("bottom_up", "bottom_up")):
        B = sum(b for lv in per_root for (x, b, _) in lv if x == d)
        T = sum(t for lv in per_root for (x, _, t) in lv if x == d)
        n = sum(1 for lv in per_root for (x, _, _) in lv if x == d)
        out[key] = {"levels": n, "bytes": B, "seconds": T,
                    "achieved": (B / T / 1e9) if T > 0 else None,
                    "frac": (B / T / 1e9 / peak) if T > 0 else None}
    # the dominant level of each kind (largest byte volume): the kernel phases
    # the north star's 50% target is about
    for d in ("top_down", "bottom_up"):
        big = [max((y for y in lv if y[0] == d), key=lambda y: y[1], default=None) for lv in per_root]
        big = [y for y in big if y is not None]
        if big:
            B = sum(y[1] for y in big)
            T = sum(y[2] for y in big)
            out[d]["largest_level"] = {"bytes_mean": B / len(big), "achieved": B / T / 1e9,
                                       "frac": B / T / 1e9 / peak}
    return out


class ClockSampler:
    """SM clocks / throttle reasons during the timed region (NVML, else nvidia-smi)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self) -> bool:
        """NVML at 100 Hz (a short timed region still gets tens of samples);
        False if NVML is unusable, so the nvidia-smi loop takes over."""
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = ((0x8, 2), (0x40, 3), (0x20, 4), (0x4, 5))  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            return False
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                row = [str(sm), str(mx), "", "", "", ""]
                for bit, col in bits:
                    row[col] = "Active" if r & bit else "Not Active"
                self.samples.append(row)
            except Exception:
                pass
            self._stop.wait(0.01)
        return True

    def _run(self):
        if self._run_nvml():
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5,
                ).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(name: str):
    """ncu dram bytes per bfs_persistent launch for this workload (profiles/roofline_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            return json.load(f).get(name)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU reference arm (the oracle's C + OpenMP port of BfsEngine, all host cores)


def default_partition_factor(n: int) -> int:
    """engine.py:70-72 (the CPU engine's lambda)."""
    return 10 if n < (1 << 26) else 20


def cpu_graph(args):
    """The same workload built by the oracle on the host (C + OpenMP restatement
    of generator.py / graph.py / reorder.py): no CUDA library is loaded."""
    import oracle

    t0 = time.perf_counter()
    if args.graph == "chunglu":
        n, e = oracle.chunglu_generate(1 << args.scale, seed=args.seed)
    else:
        n, e = oracle.kronecker_generate(args.scale, args.edgefactor, seed=args.seed)
    t1 = time.perf_counter()
    g = oracle.build_csr(n, e)
    t2 = time.perf_counter()
    perm, n_plus, ranges = oracle.rcm(g)
    t3 = time.perf_counter()  # rcm and apply_permutation timed apart (reference bench.py:160-163)
    g2 = oracle.apply_permutation(g, perm)
    del g
    t4 = time.perf_counter()
    inv = oracle.inverse(perm)
    return dict(n=n, edges=e, g2=g2, perm=perm, inv=inv, n_plus=n_plus, ranges=ranges,
                timings={"generate_s": t1 - t0, "csr_build_s": t2 - t1, "rcm_s": t3 - t2,
                         "apply_permutation_s": t4 - t3})


def raw_pairs_for(ranges, inv, edges, roots):
    """Raw input pairs whose first endpoint lies in each root's component."""
    starts = np.array([a for a, _ in ranges], np.int64)
    lab_u = inv[edges[:, 0]].astype(np.int64)
    out, cache = [], {}
    for s in roots:
        ci = int(np.searchsorted(starts, s, side="right") - 1)
        if ci not in cache:
            a, b = ranges[ci]
            cache[ci] = int(np.count_nonzero((lab_u >= a) & (lab_u < b)))
        out.append(cache[ci])
    return np.array(out, np.int64)


def cpu_run(g2, gd, s, mode, threads):
    """One BfsEngine.run in the oracle port; returns its elapsed_time (the level
    loop, engine.py:534-598, reset excluded)."""
    import oracle

    lam = default_partition_factor(g2.n)
    _, _, _, el = oracle.bfs_run(g2, int(s), mode, threads=threads, partition_factor=lam,
                                 g_desc_dst=gd if mode == "hybrid_reduced" else None)
    return el


def cpu_sample(g2, gd, roots, raw, mode, threads, seconds, max_roots=N_ROOTS):
    """hmean GTEPS of the port over roots until `seconds` elapse (>= 1 root; one warm-up root first)."""
    cpu_run(g2, gd, roots[0], mode, threads)
    teps, t0 = [], time.perf_counter()
    for s, rp in zip(roots[:max_roots], raw[:max_roots]):
        teps.append(rp / cpu_run(g2, gd, s, mode, threads))
        if time.perf_counter() - t0 > seconds:
            break
    return hmean(teps) / 1e9, len(teps)


def run_reference(args):
    """bench.py --impl reference: the reference's CPU path on this box's host
    cores, same config / metric / unit as our arm.  Primary = hybrid_reduced
    (the paper's full method, Alg. 6 over the descending-degree adjacency) at
    all host threads: each step runs a bounded sample of ceil(64 / K) roots so
    the K steps cover all 64 seeded roots; value = hmean over the 64 roots.
    Also sampled: mode hybrid (all threads) and both modes at 1 thread."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    oracle.build()
    threads = os.cpu_count() or 1
    cg = cpu_graph(args)
    g2 = cg["g2"]
    t0 = time.perf_counter()
    gd = oracle.degree_sort_rows(g2, True)  # degree_sort_adjacency(g, "descending")
    t_desc = time.perf_counter() - t0
    roots = oracle.sample_sources(g2.degrees, N_ROOTS, 1)
    raw = raw_pairs_for(cg["ranges"], cg["inv"], cg["edges"], roots)
    del cg["edges"]
    primary = "hybrid_reduced"
    rps = -(-N_ROOTS // args.steps)  # roots per step
    for i in range(args.warmup):
        for j in range(rps):
            cpu_run(g2, gd, roots[(i * rps + j) % N_ROOTS], primary, threads)
    per_root = {}
    step_wall = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        for j in range(rps):
            k = (i * rps + j) % N_ROOTS
            el = cpu_run(g2, gd, roots[k], primary, threads)
            per_root.setdefault(k, []).append(el)
        step_wall.append(time.perf_counter() - t0)
    teps = [raw[k] / float(np.mean(v)) for k, v in sorted(per_root.items())]
    v = hmean(teps) / 1e9
    modes = {f"{primary}_t{threads}": {"gteps": v, "roots": len(teps)}}
    b, used = cpu_sample(g2, gd, roots, raw, "hybrid", threads, 20.0, 16)
    modes[f"hybrid_t{threads}"] = {"gteps": b, "roots": used}
    for m in (primary, "hybrid"):
        b, used = cpu_sample(g2, gd, roots, raw, m, 1, 8.0, 4)
        modes[f"{m}_t1"] = {"gteps": b, "roots": used}
    sample = (f"{len(teps)} seeded roots ({rps} per step) of the {workload(args)[0]} graph, oracle C port of "
              f"BfsEngine mode {primary} (td_striped + bu_reduced, lambda {default_partition_factor(g2.n)}), "
              f"OpenMP {threads} threads; graph built by the oracle on the host")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(step_wall)), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": workload(args)[1],
        "config": {"workload": workload(args)[0], "scale": args.scale, "edgefactor": args.edgefactor,
                   "roots": N_ROOTS, "mode": primary},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "modes": modes,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "preprocessing_s": dict(cg["timings"], degree_sort_desc_s=t_desc),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def build_graph(args, rb, torch):
    """Device preprocessing of the workload (timed separately, not part of the
    metric): generator -> build_csr -> rcm + apply_permutation.  Returns the RCM
    graph, its stats, the 64 roots, their raw-pair numerators and the timings."""
    # one tiny pass first so module loading is not billed to the timings
    _w = rb.build_csr(rb.kronecker_generate(rb.KroneckerParams(scale=10), device=True))
    _p, _ = rb.rcm(_w)
    rb.apply_permutation(_w, _p)
    if args.graph == "chunglu":
        rb.chunglu_generate(rb.ChungLuParams(n=1 << 10), device=True)
    torch.cuda.synchronize()
    del _w, _p
    t0 = time.perf_counter()
    if args.graph == "chunglu":
        el = rb.chunglu_generate(rb.ChungLuParams(n=1 << args.scale, seed=args.seed), device=True)
    else:
        el = rb.kronecker_generate(rb.KroneckerParams(scale=args.scale, edgefactor=args.edgefactor, seed=args.seed),
                                   device=True)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    g = rb.build_csr(el)
    torch.cuda.synchronize()
    t_csr = time.perf_counter() - t0
    t0 = time.perf_counter()
    perm, stats = rb.rcm(g)
    torch.cuda.synchronize()
    t_rcm = time.perf_counter() - t0
    t0 = time.perf_counter()
    g2 = rb.apply_permutation(g, perm)
    torch.cuda.synchronize()
    t_app = time.perf_counter() - t0
    del g
    deg2 = g2.device_arrays()[2]
    roots = rb.sample_sources(deg2.cpu().numpy(), N_ROOTS, 1)
    inv_t = perm.device_arrays()[1]
    lab = inv_t[el.edges[:, 0].long()].long()
    starts = np.array([a for a, _ in stats.component_ranges], np.int64)
    raw_cache, raw = {}, []
    for s in roots:
        ci = int(np.searchsorted(starts, s, side="right") - 1)
        if ci not in raw_cache:
            a, b = stats.component_ranges[ci]
            raw_cache[ci] = int(((lab >= a) & (lab < b)).sum().item())
        raw.append(raw_cache[ci])
    del lab, el
    torch.cuda.empty_cache()
    prep = {"generate": t_gen, "csr_build": t_csr, "rcm": t_rcm, "apply_permutation": t_app,
            "rcm_plus_relabel": t_rcm + t_app}
    return g2, stats, roots, np.array(raw, np.int64), prep


def run_ours(args):
    import torch

    import paper_2012_10026_b200 as rb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    one_gpu = os.environ.get("RB_BENCH_ONE_GPU") == "1"  # debug: all ranks share cuda:0, gloo collectives
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.partitioned:
        import torch.distributed as dist

        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    g2, stats, roots, raw, prep = build_graph(args, rb, torch)
    if (world > 1 and not args.replicas) or args.partitioned:
        return run_partitioned(args, rb, torch, dist, g2, stats, roots, raw, world, rank, prep)

    eng = rb.BfsEngine(g2, rb.BfsParams(mode=args.mode))
    n_dev = eng.n_dev
    n_plus_dev = stats.n_non_isolated
    # this rank's roots: all 64 on one GPU; replicas take every world-th root
    my = list(range(rank, N_ROOTS, world))
    if args.profile_roots:
        my = my[: args.profile_roots]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    sweeps = 1 if args.profile_roots else args.steps

    for _ in range(args.warmup if not args.profile_roots else 0):
        for j in my:
            flush.zero_()
            eng.run_device(int(roots[j]))
    if args.profile_roots:
        eng.run_device(int(roots[my[0]]))  # one warm-up root before the profiled one
    torch.cuda.synchronize()

    t_root = {j: [] for j in my}
    levels_of = {}
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev_a = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev_a.record()
        for _ in range(sweeps):
            for j in my:
                flush.zero_()
                el_s, levels = eng.run_device(int(roots[j]))
                t_root[j].append(el_s)
                levels_of[j] = levels
        ev_b.record()
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    wall_ms = ev_a.elapsed_time(ev_b)

    mean_t = {j: float(np.mean(v)) for j, v in t_root.items()}
    teps = {j: raw[j] / mean_t[j] for j in my}
    teps_dedup = {j: (sum(r.m_f for r in levels_of[j]) // 2) / mean_t[j] for j in my}
    per_root = [level_bytes(levels_of[j], n_dev, n_plus_dev) for j in my]
    bytes_alg = [sum(b for _, b, _ in lv) for lv in per_root]

    # ---- e2e through the public API: BfsEngine.run -> BfsResult with the host predecessor
    for j in my[:3]:  # warm the host path (pinned staging buffers, result-array pool)
        eng.run(int(roots[j]))
    e2e_t = {}
    for j in my:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = eng.run(int(roots[j]))
        e2e_t[j] = time.perf_counter() - t0
    d2h = 4 * n_dev + 64 * len(res.levels)

    # ---- tree validation on the GPU (validate.py rules), outside the timed region
    n_val, n_ok = 0, 0
    if args.validate_roots > 0:
        val = rb.Validator(g2)
        full = torch.full((g2.n,), -1, dtype=torch.int32, device="cuda")
        for j in my[: args.validate_roots]:
            eng.run_device(int(roots[j]))
            full[:n_dev] = eng.parent_device()
            bad, _, _ = val.validate_device(int(roots[j]), full)
            n_val += 1
            n_ok += int((bad < 0).all())
        del val, full

    # ---- one harmonic mean over all 64 roots (replicas: gathered from every rank)
    loc = np.zeros((N_ROOTS, 5), np.float64)
    for j in my:
        loc[j] = [1.0, teps[j], teps_dedup[j], raw[j] / e2e_t[j], mean_t[j]]
    if dist is not None:
        tt = torch.from_numpy(loc).to("cuda" if not one_gpu else "cpu")
        dist.all_reduce(tt)
        loc = tt.cpu().numpy()
        mx = torch.tensor([wall_ms], dtype=torch.float64, device=tt.device)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        wall_ms = float(mx.item())
    got = loc[:, 0] > 0
    value = hmean(loc[got, 1]) / 1e9
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    sweep_ms = 1e3 * float(loc[got, 4].sum()) / max(world, 1)  # device traversal time of one sweep (per GPU)
    peak, peak_kind = measured_peak()
    ach = float(np.sum(bytes_alg) / np.sum([mean_t[j] for j in my]) / 1e9)
    traffic = load_traffic(workload(args)[0])
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": sweeps, "warmup": args.warmup,
        "ms_per_step": sweep_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": workload(args)[1] + ", built on device",
        "config": {"workload": workload(args)[0], "scale": args.scale, "edgefactor": args.edgefactor,
                   "roots": int(got.sum()), "step": f"one sweep of the {N_ROOTS} seeded roots",
                   "mode": args.mode,
                   "parallelism": f"replicas x{world} (roots sharded; throughput mode)" if world > 1 else "single",
                   "l2": "flushed (256 MiB write) before every root", "n": int(g2.n), "n_plus": int(n_plus_dev),
                   "m_directed": int(g2.m_directed)},
        "gteps_dedup_hmean": hmean(loc[got, 2]) / 1e9,
        "gteps_min": float(loc[got, 1].min()) / 1e9, "gteps_max": float(loc[got, 1].max()) / 1e9,
        "ms_per_root_mean": 1e3 * float(loc[got, 4].mean()),
        "depth_median": float(np.median([len(levels_of[j]) for j in my])) - 1,
        "preprocessing_s": prep,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "frac_of_nominal_8tbs": ach / 8000.0,  # the north star's nominal HBM3e figure
                     "peak_kind": peak_kind, "kernel": "bfs_persistent",
                     "bytes_per_launch": float(np.mean(bytes_alg)),
                     "launch_ms": 1e3 * float(np.mean([mean_t[j] for j in my])),
                     "traffic": None if traffic is None else traffic.get("bytes_per_launch"),
                     "by_direction": by_direction(per_root, peak)},
        "e2e": {"value": hmean(loc[got, 3]) / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * N_ROOTS,
                "d2h_bytes_per_step": int(d2h) * N_ROOTS,
                "api": "BfsEngine.run(source) -> BfsResult with host predecessor, per root"},
        "validation": {"roots": n_val, "passed": n_ok,
                       "method": "GPU Validator: the 5 rules of validate.py (tree edges, levels, spans, coverage)"},
        "gpu_launches": int(sweeps * len(my) * 2),  # bfs_reset_all + bfs_persistent per root
        "clocks": clk.summary(),
        "timed_wall_ms_per_step": wall_ms / sweeps,
    }
    if world > 1:
        # roots are independent: total raw pairs of the sweep / per-GPU sweep time
        line["replica_throughput_gteps"] = float(raw[got].sum()) / (sweep_ms / 1e3) / 1e9
    if args.dump_levels:
        dump = {"workload": workload(args)[0], "peak_gbs": peak, "n_dev": int(n_dev), "n_plus": int(n_plus_dev),
                "byte_model": "TD: 20*n_f + 4*scanned + 8*n_next; BU: 3*n_dev/8 + 8*U + 4*scanned + 4*n_next "
                              "(SURVEY 8(d), bench.level_bytes)",
                "roots": [{"root": int(roots[j]), "mean_s": mean_t[j],
                           "levels": [{"label": r.direction, "executed": r.executed_direction, "n_f": r.n_f,
                                       "m_f": r.m_f, "scanned": r.scanned_edges, "bytes": b, "seconds": t}
                                      for r, (_, b, t) in zip(levels_of[j], level_bytes(levels_of[j], n_dev,
                                                                                          n_plus_dev))]}
                          for j in my]}
        with open(args.dump_levels, "w") as f:
            json.dump(dump, f)
    if not args.no_cpu_baseline and not args.profile_roots and world == 1:
        try:
            line["cpu_baseline"] = cpu_baseline_sample(g2, roots, raw, args.cpu_seconds)
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": repr(ex)}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def cpu_baseline_sample(g2, roots, raw, seconds):
    """The oracle port of BfsEngine (hybrid_reduced, the paper's best CPU mode,
    all host threads) on the host copy of the same RCM graph, bounded sample."""
    import oracle

    oracle.build()
    go = oracle.Csr(g2.n, g2.row_starts, g2.dst, g2.degrees)
    gd = oracle.degree_sort_rows(go, True)
    threads = os.cpu_count() or 1
    v, used = cpu_sample(go, gd, roots, raw, "hybrid_reduced", threads, seconds)
    return {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{used} seeded roots of the same RCM graph, oracle C port of BfsEngine hybrid_reduced "
                      f"(Alg. 6), OpenMP {threads} threads"}


def run_partitioned(args, rb, torch, dist, g2, stats, roots, raw, world, rank, prep):
    """--gpus N > 1: ONE traversal per root over the 1D vertex-block partition
    of all GPUs with the exchange on the device (distributed.DeviceExchangeBfs:
    one persistent launch per rank per root; next-frontier words and counters
    stored into every peer's buffers over NVLink, a system-scope barrier per
    level).  Per-root time = max over ranks of the device event time; value =
    harmonic mean over the 64 roots (strong scaling: same graph, same roots)."""
    from paper_2012_10026_b200.distributed import DeviceExchangeBfs, partition_bounds

    n_plus = stats.n_non_isolated
    deg_host = g2.degrees
    bounds = partition_bounds(g2.row_starts, n_plus, world)
    drv = DeviceExchangeBfs(g2, bounds, rank, world, hybrid=args.mode != "level_sync")
    my = list(range(N_ROOTS)) if not args.profile_roots else list(range(args.profile_roots))
    sweeps = 1 if args.profile_roots else args.steps
    for _ in range(args.warmup):
        for j in my:
            drv.run(int(roots[j]), int(deg_host[roots[j]]))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    t_root = {j: [] for j in my}
    recs_of = {}
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for _ in range(sweeps):
            for j in my:
                flush.zero_()
                recs_of[j] = drv.run(int(roots[j]), int(deg_host[roots[j]]))
                t_root[j].append(drv.elapsed())
    dist.barrier()
    loc = np.array([float(np.mean(t_root[j])) for j in my], np.float64)
    t = torch.from_numpy(loc).cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the root's time = its slowest rank
    times = t.cpu().numpy()
    teps = [raw[j] / times[i] for i, j in enumerate(my)]
    # e2e: the same traversal + every rank's parent block copied to its host
    e2e = []
    for j in my[: min(len(my), 16)]:
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        drv.run(int(roots[j]), int(deg_host[roots[j]]))
        _ = drv.local.parents().cpu().numpy()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e.append(raw[j] / float(tt.item()))
    if rank == 0:
        peak, peak_kind = measured_peak()
        alg = [algorithmic_bytes([type("R", (), dict(direction="top_down" if r.direction == 0 else "bottom_up",
                                                       n_f=r.n_f, scanned_edges=r.scanned))() for r in recs_of[j]],
                                 n_plus, n_plus) for j in my]
        ach = float(np.sum(alg) / np.sum(times) / 1e9) / world  # per GPU
        line = {
            "metric": METRIC, "value": hmean(teps) / 1e9, "unit": UNIT, "n_gpus": world, "steps": sweeps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.sum(times)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": workload(args)[1] + ", built on device",
            "config": {"workload": workload(args)[0], "scale": args.scale, "edgefactor": args.edgefactor,
                       "roots": len(my), "step": f"one sweep of the {len(my)} seeded roots", "mode": args.mode,
                       "parallelism": f"1d-partition x{world} (device-side exchange over NVLink peer memory)",
                       "partition_bounds": bounds, "l2": "flushed (256 MiB write) before every root"},
            "preprocessing_s": prep,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "peak_kind": peak_kind, "kernel": "bfs_dist (per GPU)", "traffic": None},
            "e2e": {"value": hmean(e2e) / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * N_ROOTS,
                    "d2h_bytes_per_step": int(4 * (bounds[1] - bounds[0])) * N_ROOTS},
            "gpu_launches": int(sweeps * len(my) * 3),  # reset + exchange reset + bfs_dist per root
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    drv.close()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
