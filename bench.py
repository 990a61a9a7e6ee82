"""Benchmark of the exit-measure hot path (BASELINE.json metric: walks/s and
walk-steps/s for A, % of the FP32 issue roofline).

One "step" = one pass of the hot path over the whole workload: every walk of
every pole run to the eps-shell and binned into the (n_poles, n0 + n1) int64
count rows (the reference's run_accumulate, S/backend.py:147-199, S/ =
/root/reference/pkg/src/exitmeasure/).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2]
                    [--precision fp32|ref64] [--chain max|woe]
    python bench.py --impl reference ...   # the reference's own CPU path

Workload at N=1: BASELINE configs[1] (cfg2, the unit square with
K=[[2,.8],[.8,1]], 256 poles x 1e5 walks, eps 1e-5, 512 edge bins).
Multi-GPU (one process per GPU, torchrun): by default "scaling": "weak" --
the walks are independent units, so every rank walks all poles x n walks on
its own replicate range [r n, (r+1) n) (walks keyed by their global replicate
index: the ranks' rows add up to the N*n-walk estimate exactly), no collective
inside the timed region, rows summed once afterwards.  `--scaling strong`
instead shards the fixed workload's rows cyclically over the ranks (pole i ->
rank i mod N, RNG keyed by the global pole id) and ends every step with the
NCCL all-gather of the count rows, inside the timed region --
north_star's strong-scaling target, which only the large configs can meet
(compute-side proxy in profiles/r01_shard_proxy.txt: cfg3 / cfg4 / cfg5 at 8
GPUs 0.97 / 0.97 / 0.99; cfg2's 0.53 ms job is launch/tail bound at 8 GPUs).
Timing: CUDA events on each rank, max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# Algorithmic FP32 lane-ops per walk step of the IMPLEMENTED chain, counted
# with SURVEY.md §8(d)'s convention: add/sub/mul/fma/min/max/compare = 1 on
# the path a step takes -- no selects, and exclusive branch arms weighted by
# how often a step takes them (cfg3: the centred disk on 17.7% of steps,
# cfg4: the centred ball on 25.4%, from the chains' float64 restatements);
# sqrt/rsqrt/rcp/sin/cos are XU ops, counted apart; RNG and per-walk
# bookkeeping excluded.  Term by term in DESIGN.md §3.3.
F_STEP = {
    (1, "woe"): (11, 3), (1, "max"): (11, 3),   # K = I: both chains are the sphere step
    (2, "woe"): (15, 2), (2, "max"): (14, 2),    # max: sheared box axes
    (2, "tangent"): (37, 3),                     # tangent balls in the whitened parallelogram
    (3, "woe"): (19, 4), (3, "max"): (29, 6),    # concentric hole: shared |v|^2, |Av|^2, one rcp
    (3, "tangent"): (49.1, 6.2),                 # one rolling / hole-tangent disk, else centred (difference form)
    (4, "woe"): (22, 4), (4, "max"): (31, 6),    # balls: frame rotated onto K's eigenbasis
    (4, "tangent"): (76.3, 8.0),                 # rolling balls, else the centred ball (difference form)
    (5, "woe"): (36, 4), (5, "max"): (41, 4),    # max: sheared box axes, world-unit notch
    (5, "tangent"): (87, 5),                     # tangent balls in 3D, notch planes as faces
}

# the reference chain's FP32 ops per step (same counting
# convention) and its measured steps per walk.  walks/s x F x steps is the
# FP32 work the REFERENCE algorithm would have to issue to match our walks/s
# (cfg5 has no reference path: the numpy WoE restatement's ~81 steps).
F_REF = {1: (23.2, 12.6), 2: (25.2, 45.3), 3: (28.2, 59.5), 4: (33.9, 72.4), 5: (42.9, 81.0)}


class ClockSampler:
    """NVML clocks + throttle reasons sampled on a thread during the timed
    region (the recipe's clocks line)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: int):
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            idx = device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[device])
                except ValueError:
                    idx = device
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self._nv = None
            self.error = str(e)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((mhz, reasons))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mhz = sorted(s[0] for s in self.samples)
        active = set()
        for _, r in self.samples:
            for name, bit in self.REASONS.items():
                if r & bit:
                    active.add(name)
        return {"sm_mhz": float(mhz[len(mhz) // 2]), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(active), "samples": len(self.samples)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference_walks_per_s(cfg, n_sample: int, threads: int):
    """The reference's own CPU path (oracle/_ref, the unmodified exitmeasure
    package with its compiled Cython kernel) on a bounded sample of the
    workload: all poles x n_sample walks.  Falls back to the C restatement
    (oracle/em_oracle.c) if oracle/_ref is absent."""
    ref = ROOT / "oracle" / "_ref"
    sub = cfg.subset(None, n_sample)
    if (ref / "exitmeasure").exists():
        sys.path.insert(0, str(ref))
        from exitmeasure import backend as rb
        from exitmeasure.geometry import Ball, Box, BoundaryPointSet, make_domain

        # the reference's OWN CPU path, never this library installed over it
        assert not hasattr(rb, "_em_b200_original"), "plugin installed over the reference"
        assert rb.BACKEND == "compiled", rb.BACKEND

        from paper_2409_03686_b200 import backend as B

        geom = B.pack_geometry(sub.dom)
        if sub.index in (1, 2, 4):
            outer = (Ball(np.zeros(sub.d), 1.0) if sub.index in (1, 4)
                     else Box(np.array([0.5, 0.5]), 0.5))
            dom = make_domain(outer, gamma0=())
            pts = np.ascontiguousarray(sub.fam1.points)
            s1 = rb.pack_side(BoundaryPointSet(pts, np.zeros(len(pts), int),
                                               np.arange(len(pts), dtype=float), ()),
                              sub.d, sub.eps)
            s0 = rb.pack_side(None, sub.d, sub.eps)
        elif sub.index == 3:
            from exitmeasure.geometry import catalog, side_points

            dom = catalog("annulus")
            s0 = rb.pack_side(side_points(dom, "gamma0", [512]), 2, sub.eps)
            s1 = rb.pack_side(side_points(dom, "gamma1", [512]), 2, sub.eps)
        else:
            dom = None
        if dom is not None:
            t0 = time.perf_counter()
            r = rb.run_accumulate(dom, sub.kt.k_sqrt, sub.poles, sub.seed, sub.eps, 10**6,
                                  n_sample, s0, s1, threads=threads)
            dt = time.perf_counter() - t0
            walks = sub.n_poles * n_sample
            return (walks / dt, float(r.steps_sum.sum()) / dt, "reference", dt,
                    float(r.steps_sum.sum()) / walks)
        del geom
    from oracle import oracle as O

    from paper_2409_03686_b200 import backend as B

    geom = B.pack_geometry(sub.dom)
    s0 = B.pack_side(sub.fam0, sub.d, sub.eps)
    s1 = B.pack_side(sub.fam1, sub.d, sub.eps)
    t0 = time.perf_counter()
    raw0, raw1, ss, *_ = O.run_accumulate_packed(
        geom.gi, geom.gf, geom.comp_side, sub.kt.k_sqrt, sub.poles, sub.seed, sub.eps, 10**6,
        n_sample, (s0.anchors, s0.blk, s0.blkf), (s1.anchors, s1.blk, s1.blkf), threads=threads)
    dt = time.perf_counter() - t0
    walks = sub.n_poles * n_sample
    return walks / dt, float(ss.sum()) / dt, "port", dt, float(ss.sum()) / walks


# walks per pole per step of the `--impl reference` arm (~0.2-1 s of CPU work
# per step on 16 host threads, so a K-step run ends in minutes) ...
REF_SAMPLE = {1: 10_000, 2: 16_384, 3: 1024, 4: 256, 5: 16}
# ... and of the in-bench `cpu_baseline` leg: about 10 s of CPU work on the
# GPU box's 16 host threads (cfg1: the whole 3.2e5-walk workload), see
# profiles/r01_cpu_baseline.json for threads=1 / all and linearity in N
CPU_SAMPLE = {1: 10_000, 2: 163_840, 3: 32_768, 4: 16_384, 5: 1024}


# committed ncu captures of the walk kernel per (config, chain): key metrics
# in "metric,value,unit" rows (tools/ncu_metrics.py from the raw page of one
# `ncu --set full` capture of `bench.py --config C`)
PROFILES = {(2, "tangent"): "profiles/r02_cfg2_walk_f32_ncu_metrics.csv",
            (3, "tangent"): "profiles/r02_cfg3_walk_f32_ncu_metrics.csv",
            (4, "tangent"): "profiles/r02_cfg4_walk_f32_ncu_metrics.csv",
            (5, "tangent"): "profiles/r02_cfg5_walk_f32_ncu_metrics.csv"}


def profiled_ncu(cfg_index: int, precision: str, chain: str):
    """DRAM bytes per launch and issue / pipe utilisation of the walk kernel
    from the committed capture of this configuration, or None."""
    import csv

    rel = PROFILES.get((cfg_index, chain)) if precision == "fp32" else None
    if rel is None or not (ROOT / rel).exists():
        return None
    vals = {}
    for row in csv.reader(open(ROOT / rel)):
        if len(row) == 3:
            vals[row[0]] = (row[1], row[2])
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {"source": rel}
    try:
        out["traffic"] = sum(float(vals[k][0]) * scale[vals[k][1]]
                             for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except (KeyError, ValueError):
        out["traffic"] = None
    keys = {"issue_active": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "pipe_fma": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "pipe_alu": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "pipe_xu": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "warps_active": "sm__warps_active.avg.pct_of_peak_sustained_active"}
    try:
        out["issue"] = {k: round(float(vals[v][0]) / 100.0, 4) for k, v in keys.items()}
        out["issue"]["source"] = rel + " (fractions of peak)"
    except (KeyError, ValueError):
        out["issue"] = None
    return out


def workload_name(cfg) -> str:
    """The workload string both arms put in config.workload."""
    bins = (len(cfg.fam0) if cfg.fam0 is not None else 0) + len(cfg.fam1)
    return (f"{cfg.name}: {cfg.n_poles} poles x {cfg.n_rep:.0e} walks, eps {cfg.eps:g}, "
            f"{bins} bins")


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    from paper_2409_03686_b200 import configs

    cfg = configs.get(args.config)
    threads = os.cpu_count() or 1
    n_sample = args.ref_sample or REF_SAMPLE[cfg.index]
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        v = cpu_reference_walks_per_s(cfg, n_sample, threads)
        if i >= args.warmup:
            vals.append(v)
        info = v
    wps = float(np.median([v[0] for v in vals]))
    sps = float(np.median([v[1] for v in vals]))
    ms = float(np.median([v[3] for v in vals])) * 1e3
    sample = (f"{cfg.name}: all {cfg.n_poles} poles x {n_sample} walks/pole "
              f"({cfg.n_poles * n_sample:.3g} walks) per step, threads={threads}")
    line = {
        "impl": "reference", "metric": "walks/s", "value": wps, "unit": "walks/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "steps_per_s": sps, "mean_steps_per_walk": info[4],
        "config": {"workload": workload_name(cfg), "precision": "fp64 (the reference chain)",
                   "sample_per_step": f"{cfg.n_poles} poles x {n_sample} walks",
                   "threads": threads},
        "cpu_baseline": {"value": wps, "unit": "walks/s", "cores": threads, "kind": info[2],
                         "sample": sample},
        "e2e": {"value": wps, "unit": "walks/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _nccl_lines():
    """The communicator-init lines NCCL wrote under NCCL_DEBUG=INFO (the
    NCCL_DEBUG_FILE this harness sets): rank / nranks per communicator."""
    import glob
    import re

    out = []
    for f in sorted(glob.glob(os.environ.get("EM_NCCL_LOG_GLOB", "/nonexistent"))):
        for line in open(f, errors="replace"):
            if re.search(r"nranks \d+", line, re.I) and re.search(r"init complete", line, re.I):
                out.append(line.strip())
    return out


def run_ours(args):
    import torch

    world, rank, local = _dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    dist = None
    if world > 1:
        import torch.distributed as dist

        # NCCL's communicator-init lines (rank / nranks) into per-rank files
        # rank 0 reads back (NCCL reads these at init; a launcher's own
        # settings win)
        logdir = Path(os.environ.get("TMPDIR", "/tmp")) / \
            f"em_nccl_{os.environ.get('TORCHELASTIC_RUN_ID', 'run')}_{os.environ.get('MASTER_PORT', 'x')}"
        logdir.mkdir(parents=True, exist_ok=True)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", str(logdir / "nccl.%h.%p.log"))
        os.environ.setdefault("EM_NCCL_LOG_GLOB", str(logdir / "nccl.*.log"))
        # EXITMEASURE_B200_DEVICE pins every rank to one device: the harness
        # self-test on a 1-GPU box (--dist-backend gloo; the ranks' kernels
        # are independent, the exchange runs on the host)
        if os.environ.get("EXITMEASURE_B200_DEVICE") is not None:
            local = int(os.environ["EXITMEASURE_B200_DEVICE"])
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    device = local if world > 1 else 0
    torch.cuda.set_device(device)
    coll_dev = "cuda" if args.dist_backend == "nccl" else "cpu"  # small collectives
    from paper_2409_03686_b200 import _native, backend, configs, distributed

    cfg = configs.get(args.config)
    if args.n_rep:
        cfg = cfg.subset(None, args.n_rep)
    weak = args.scaling == "weak"
    if weak:
        # weak scaling: every rank walks ALL poles on its own replicate range
        # [rank n, (rank + 1) n) (walks are keyed by their global replicate
        # index, so the ranks' counts add up to the N*n-walk estimate exactly);
        # no collective on the data path, one sum of the rows after timing
        ids = np.arange(cfg.n_poles)
        rep_start = rank * cfg.n_rep
    else:
        # strong scaling (default): cyclic row shard of the fixed workload,
        # then ONE NCCL all-gather of the count rows + step statistics and the
        # un-permute to pole order, all inside the timed region
        ids = distributed.shard_rows(cfg.n_poles, world, rank)
        rep_start = 0
    geom = backend.pack_geometry(cfg.dom)
    s0 = backend.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = backend.pack_side(cfg.fam1, cfg.d, cfg.eps)
    plan = backend.Plan(geom, cfg.kt.k_sqrt, cfg.poles[ids], cfg.eps, 10**6, s0, s1,
                        precision=args.precision, chain=args.chain, device=device,
                        pole_ids=ids, grid=args.grid,
                        flags={"auto": 0, "persistent": _native.EM_FLAG_PERSISTENT,
                               "pole-blocks": _native.EM_FLAG_POLE_BLOCKS}[args.sched]
                        | (_native.EM_FLAG_ONE_WALK_PER_LANE if args.lanes == "one" else 0))
    row = plan.n0 + plan.n1
    m_local = len(ids)
    m_pad = m_local if weak else -(-cfg.n_poles // world)
    # one flat block per rank: counts (m_pad, row) | stats (3, m_pad), so the
    # exchange is ONE all-gather
    blk_len = m_pad * row + 3 * m_pad
    buf = torch.zeros(blk_len, dtype=torch.int64, device="cuda")
    counts = buf[: m_pad * row].view(m_pad, row)
    stats = buf[m_pad * row:].view(3, m_pad)
    gathered = full = perm = None
    if world > 1 and not weak:
        gathered = torch.zeros((world, blk_len), dtype=torch.int64, device="cuda")
        perm = distributed.cyclic_gather_index(cfg.n_poles, world, m_pad, device="cuda")
        full = torch.zeros((cfg.n_poles, row), dtype=torch.int64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    kev = []  # CUDA events around the library's launches (zeroing + walk kernel)

    def one_step(timed=False):
        if timed:
            kev.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
            kev[-1][0].record(stream)
        plan.run_device(cfg.seed, cfg.n_rep, counts.data_ptr(), stats.data_ptr(),
                        stream.cuda_stream, rep_start)
        if timed:
            kev[-1][1].record(stream)
        if gathered is not None:
            distributed.exchange_rows(buf, gathered, perm, m_pad, row, full)

    for _ in range(args.warmup):
        flush.zero_()
        one_step()
    torch.cuda.synchronize()
    steps_per_run = int(stats[0, :m_local].sum().item())
    # every walk of every pole counted exactly once (this rank's rows; at N>1
    # strong also the gathered full matrix) -- checked on the device
    if not bool((counts[:m_local].sum(1) == cfg.n_rep).all().item()):
        raise RuntimeError("count rows do not sum to the walk count")
    if full is not None:
        assert bool((full.sum(1) == cfg.n_rep).all().item()), "gathered rows wrong"
    ffma_peak, _ = _native.fp32_peak(device)
    info = _native.device_info(device)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    with ClockSampler(device) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            one_step(timed=True)
            ev[i][1].record(stream)
            launches += plan.last_launches() + (2 if gathered is not None else 0)
        torch.cuda.synchronize()
    plan.check()  # budget errors of the (asynchronous) runs
    # the walk kernel's average launch duration over the timed steps: CUDA
    # events on its stream around the library call (the 7 us zeroing launch
    # before it included; profiles/r02_cfg3_launches.csv has the split)
    kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    combined_ok = None
    if dist and weak:
        # the one exchange, outside the timed region: sum the ranks' rows into
        # the N*n-walk estimate and check every row counts all of its walks
        if coll_dev == "cpu":
            c = counts.cpu()
            dist.all_reduce(c)
            counts.copy_(c)
        else:
            dist.all_reduce(counts)
        combined_ok = bool((counts.sum(dim=1) == world * cfg.n_rep).all().item())
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = float(sum(step_ms))
    if dist:
        t = torch.tensor([tot_ms, kernel_ms], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, kernel_ms = float(t[0].item()), float(t[1].item())
        st = torch.tensor([steps_per_run], device=coll_dev, dtype=torch.int64)
        dist.all_reduce(st)
        steps_total_run = int(st.item())
    else:
        steps_total_run = steps_per_run
    walks = cfg.total_walks * (world if weak else 1) * args.steps
    value = walks / (tot_ms * 1e-3)
    steps_per_s = steps_total_run * args.steps / (tot_ms * 1e-3)
    clocks = clk.summary()

    # roofline: FP32 issue bound of the walk kernel on this GPU.  The kernel's
    # own duration (CUDA events around the launch on its stream, averaged over
    # the timed runs' last launch) sets `achieved`; the step time also holds
    # the zeroing / fold launches and, at N > 1, the gather.
    fp32, xu = F_STEP[(cfg.index, plan.chain if plan.precision == "fp32" else "woe")]
    steps_per_gpu_run = steps_total_run / world
    achieved = fp32 * steps_per_gpu_run / (kernel_ms * 1e-3) / 1e12
    clk_mhz = clocks["sm_mhz"] or (info["clock_khz"] / 1e3)
    peak_nominal = info["sm_count"] * 128 * clk_mhz * 1e6 / 1e12
    peak_ffma = ffma_peak / 1e12

    # e2e through the public API, host numpy in / out, every step: plan
    # creation + upload of the inputs, the walk, the exchange, the D2H of the
    # rows.  N = 1: the REFERENCE's own entry point exitmeasure.backend.
    # run_accumulate with this backend installed by plugin.install() (when the
    # reference package is importable); N > 1: distributed.
    # run_accumulate_sharded on every rank, wall time max over ranks.
    e2e_vals, api, ref_be = [], None, None
    n_e2e = max(3, min(args.steps, 11))
    if world == 1:
        ref_be = _plugin_backend(plan.precision, plan.chain, device)
        if ref_be is not None:
            api = ("exitmeasure.backend.run_accumulate (the reference's entry point) with "
                   "paper_2409_03686_b200.plugin.install(cache=False) -- the reference's "
                   "AccumulateResult (float64 raw0/raw1) out")
            call = lambda: ref_be.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed,
                                                 cfg.eps, 10**6, cfg.n_rep, s0, s1)
        else:
            api = "paper_2409_03686_b200.backend.run_accumulate(cache=False)"
            call = lambda: backend.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed,
                                                  cfg.eps, 10**6, cfg.n_rep, s0, s1,
                                                  precision=plan.precision, chain=plan.chain,
                                                  device=device, cache=False)
    elif weak:
        api = "paper_2409_03686_b200.backend.run_accumulate(cache=False) per rank (own replicate range)"
        call = lambda: backend.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed,
                                              cfg.eps, 10**6, cfg.n_rep, s0, s1,
                                              precision=plan.precision, chain=plan.chain,
                                              device=device, cache=False)
    else:
        api = ("paper_2409_03686_b200.distributed.run_accumulate_sharded (row shard, NCCL "
               "all-gather, full rows on every rank)")
        call = lambda: distributed.run_accumulate_sharded(
            cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6, cfg.n_rep, s0, s1,
            precision=plan.precision, chain=plan.chain)
    for _ in range(n_e2e):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        r = call()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], device=coll_dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e_vals.append(dt)
    if world == 1 and ref_be is not None:
        from paper_2409_03686_b200 import plugin

        plugin.uninstall(ref_be)  # the cpu_baseline leg below times the reference itself
    e2e_walks = cfg.total_walks * (world if weak else 1)
    e2e_val = e2e_walks / float(np.median(e2e_vals[1:]))
    in_ids = ids if (weak or world == 1) else np.arange(cfg.n_poles)
    h2d = (cfg.poles.nbytes + s0.anchors.nbytes + s1.anchors.nbytes + geom.gi.nbytes
           + geom.gf.nbytes + cfg.kt.k_sqrt.nbytes)
    d2h = (len(in_ids) * row * 8 + 3 * 8 * len(in_ids)) if (weak or world == 1) else \
        (m_pad * row + 3 * m_pad) * 8
    grid_note = ("candidate-grid cache warm after the first call (the grid is a pure "
                 "function of the anchors; ~1 s host build)" if cfg.index in (4, 5)
                 else "no candidate grid on this config (closed-form binner)")

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            n_sample = CPU_SAMPLE[cfg.index]
            c = cpu_reference_walks_per_s(cfg, n_sample, os.cpu_count() or 1)
            cpu = {"value": c[0], "unit": "walks/s", "cores": os.cpu_count() or 1,
                   "kind": c[2],
                   "sample": f"{cfg.name}: all {cfg.n_poles} poles x {n_sample} walks/pole "
                             f"({c[3]:.1f} s), steps/s {c[1]:.3g}"}
        prof = profiled_ncu(cfg.index, plan.precision, plan.chain)
        line = {
            "metric": "walks/s", "value": value, "unit": "walks/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if weak else "strong",
            "vs_baseline": None,
            "dtype": "f32" if plan.precision == "fp32" else "f64", "data": "synthetic",
            "steps_per_s": steps_per_s,
            "mean_steps_per_walk": steps_total_run / (cfg.total_walks * (world if weak else 1)),
            "config": {"workload": workload_name(cfg),
                       "precision": plan.precision, "chain": plan.chain,
                       "parallelism": (f"{world} GPU(s), each all poles x {cfg.n_rep:.0e} walks on "
                                       "its own replicate range; rows summed once after timing"
                                       + ("" if combined_ok is None else
                                          f" (row sums {'ok' if combined_ok else 'WRONG'})")
                                       if weak else
                                       f"rows cyclic over {world} GPU(s) (pole i -> rank i mod "
                                       f"{world})" + (f", one {args.dist_backend.upper()} all-gather "
                                                      "of the count rows + step statistics and the "
                                                      "un-permute to pole order inside every timed "
                                                      "step" if world > 1 else "")),
                       "l2": "flushed between timed steps (256 MiB write)",
                       "counts": "int64 (n_poles, n0+n1) rows + step stats",
                       "scheduler": plan.last_scheduler(),
                       "walks_per_lane": plan.last_walks_per_lane(),
                       "build": _native.build_info()},
            "roofline": {"bound": "fp32_issue", "achieved": achieved, "peak": peak_nominal,
                         "unit": "Top/s", "frac": achieved / peak_nominal,
                         "kernel_ms": kernel_ms,
                         "kernel_ms_note": "average over the timed steps of the library's "
                                           "launches (walk kernel + its 7 us zeroing launch), "
                                           "CUDA events on the launching stream",
                         "traffic": prof["traffic"] if prof else None,
                         "traffic_note": ("DRAM bytes per launch of the walk kernel from the "
                                          f"committed ncu --set full capture ({prof['source']}); "
                                          "algorithmic: the int64 count rows") if prof else
                                         "no committed capture of this configuration",
                         "algorithmic_bytes": int(cfg.n_poles * row * 8),
                         "f_step": {"fp32": fp32, "xu": xu,
                                    "convention": "SURVEY 8(d): add/sub/mul/fma/min/max/compare "
                                                  "on the path a step takes (no selects, no "
                                                  "discarded branch arms); XU and RNG apart; "
                                                  "DESIGN.md 3.3"},
                         "peak_note": f"{info['sm_count']} SMs x 128 FP32 lanes x median SM "
                                      f"clock under load {clk_mhz:.0f} MHz (MEASURED_PEAKS.json "
                                      "has no FP32 figure)",
                         "peak_measured_ffma": peak_ffma,
                         "frac_of_measured_ffma": achieved / peak_ffma,
                         "frac_at_max_clock": achieved / (info["sm_count"] * 128 *
                                                          (clocks["sm_max_mhz"] or 1965) * 1e-6),
                         "ncu": prof["issue"] if prof else None,
                         "reference_chain_equivalent": {
                             "frac": (value / world) * F_REF[cfg.index][0] * F_REF[cfg.index][1]
                                     / (peak_nominal * 1e12),
                             "note": "walks/s x the reference chain's FP32 ops/step x its "
                                     "steps/walk (SURVEY 8d) / peak: the FP32 issue share the "
                                     "reference algorithm would need for the same walks/s (not "
                                     "a roofline fraction)"}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "walks/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "api": api,
                    "timing": ("wall clock per call, median of the calls after the first"
                               + (", max over ranks" if world > 1 else "")),
                    "caches": "plan cache off (plan creation + input upload in every call); "
                              + grid_note},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if world > 1:
            nl = _nccl_lines()
            line["config"]["nccl"] = {"init_lines": nl[:world], "n_lines": len(nl)}
        print(json.dumps(line), flush=True)
    plan.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _plugin_backend(precision, chain, device):
    """The reference's backend module with this library installed (oracle/_ref
    holds the unmodified reference package), or None when it is absent."""
    ref = ROOT / "oracle" / "_ref"
    if not (ref / "exitmeasure").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        from paper_2409_03686_b200 import plugin

        return plugin.install(precision=precision, chain=chain, device=device, cache=False)
    except Exception as e:  # pragma: no cover - reference import problems
        print(f"bench.py: plugin path unavailable ({e})", file=sys.stderr)
        return None


def run_harness_check(args):
    """The launch / rendezvous / max-over-ranks plumbing without a GPU
    (gloo): each rank reports itself, rank 0 prints one line with n_gpus."""
    import torch
    import torch.distributed as dist

    world, rank, _ = _dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    r = torch.tensor([rank], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ranks = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(ranks, r)
        seen = sorted(int(x.item()) for x in ranks)
    else:
        seen = [0]
    if rank == 0:
        print(json.dumps({"harness_check": True, "n_gpus": world, "ranks": seen,
                          "max_over_ranks": float(t.item())}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def self_launch(argv, n: int) -> int:
    """--gpus N without a torchrun environment: launch N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1 (each rank turns NCCL
    init logging on, run_ours)."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())]
    return subprocess.call(cmd + list(argv), env=env)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3,
                    help="BASELINE config (default 3: the annulus, the config BASELINE.json "
                         "shards over 1/2/4/8 GPUs)")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--chain", default=None)
    ap.add_argument("--n-rep", type=int, default=None, help="override walks per pole")
    ap.add_argument("--ref-sample", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--grid", type=int, default=0, help="persistent blocks (0 = auto)")
    ap.add_argument("--lanes", default="auto", choices=["auto", "one"],
                    help="one: force the one-walk-per-lane kernel where the packed "
                         "two-walks-per-lane kernel exists (A/B)")
    ap.add_argument("--sched", default="auto", choices=["auto", "persistent", "pole-blocks"],
                    help="auto: per-block shared-memory histograms where the rows exceed half "
                         "the L2, else pole-cycling persistent warps; pole-blocks / persistent "
                         "force one (A/B)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N>1: strong (default) = cyclic row shard of the fixed workload + "
                         "NCCL all-gather of the rows inside every timed step; weak = every "
                         "rank walks all poles on its own replicate range, no collective in "
                         "the timed region")
    ap.add_argument("--harness-check", action="store_true",
                    help="launch / rendezvous plumbing only (gloo, no GPU)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 exchange backend (gloo: the multi-rank harness self-test on one "
                         "GPU with EXITMEASURE_B200_DEVICE=0; not a measurement)")
    args = ap.parse_args(argv)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(argv, args.gpus)
    if args.harness_check:
        return run_harness_check(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
