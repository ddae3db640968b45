#!/usr/bin/env python
"""bench.py -- Power Foam rasterizer throughput on B200 (BASELINE.json metric).

Default workload: train8_1m (1M-cell Mip-NeRF-360-shaped foam, a batch of 8
views at 1920x1080, forward + backward, per-cell gradient all-reduce over NCCL
when N > 1).  One step = one pass of the whole hot path (K0 edge records, K1
projection/binning, K2 scan, K3 emit, K4 radix sort, K5 ranges, K6 forward
blend, K7 backward, K8 unpack, + all-reduce) over one batch of views.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

`--gpus N` without torchrun re-launches itself under torch.distributed.run with
N ranks (one per GPU).  Multi-GPU scaling follows SURVEY §8(e): the batch is
FIXED (train8_1m: 8 views, sweep64_3m: 64 views) and dealt round-robin over the
ranks (rank r renders views r, r+N, ...) -- "scaling": "strong"; `--scaling
weak` gives every rank its own full batch instead, and at N > 1 the strong run
also reports a weak-scaling figure as an extra field.  Rank 0 prints ONE JSON
line; `value` = frames (views) per second of the whole job.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "frames/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
SM_COUNT = 148
FP32_LANES_PER_SM = 128


# ----------------------------------------------------------------------------
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="train8_1m",
                    choices=["train8_1m", "mip360_1m", "nerfsynth200k", "sweep64_3m", "small360"])
    ap.add_argument("--views", type=int, default=None,
                    help="views per step: the whole batch (strong) or per GPU (weak); "
                         "default: the preset's batch")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (SURVEY 8(e)): the preset's batch dealt over the ranks; "
                         "weak: every rank renders a full batch of its own")
    ap.add_argument("--dipoles", action="store_true",
                    help="oriented-point dipole cells (NEXT-1) on the workload's foam")
    ap.add_argument("--detail", type=int, default=0, metavar="K",
                    help="K detail sites per dipole face (NEXT-2; implies --dipoles)")
    ap.add_argument("--fisheye", action="store_true",
                    help="equidistant fisheye cameras (NEXT-4), 200 deg image circle")
    ap.add_argument("--lists", default="cech", choices=["cech", "knn"],
                    help="neighbour lists: Čech-filtered (default) or unfiltered sym-16NN "
                         "(the paper's extraneous-edge comparison, P:236)")
    ap.add_argument("--trace", action="store_true",
                    help="render with the NEXT-4 adjacency-walk ray tracer (pf_trace_forward) "
                         "instead of the tile rasterizer (forward only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def orbit_cameras(name, total):
    """The workload's batch of `total` views (an orbit around the scene)."""
    import pf_synth
    if name in ("train8_1m", "mip360_1m", "sweep64_3m"):
        step = math.radians(5.625) if name == "sweep64_3m" else 2 * math.pi / total
        return pf_synth._cams_mip360(total, 1920, 1080, az_step=step,
                                     jitter=0.3 if name == "sweep64_3m" else 0.0, seed=3)
    if name == "nerfsynth200k":
        return pf_synth._cams_nerfsynth(total, 800, 800)
    return pf_synth.make_cameras(name, n=total)


def plan_views(name, views, scaling, world, rank):
    """The view deal of SURVEY §8(e).  Returns (total views of the job, indices of
    this rank's views in the job's orbit).  strong: the batch (`views`, default the
    preset's) is fixed and dealt round-robin -- rank r gets r, r+N, ...; weak: the
    orbit has views*N cameras, dealt the same way (views per rank fixed)."""
    per = views or default_views(name)
    total = per * world if scaling == "weak" else per
    if total < world:
        raise SystemExit(f"bench.py: {total} views cannot be dealt over {world} ranks "
                         f"(every rank needs at least one view)")
    if world < 1 or not (0 <= rank < world):
        raise SystemExit("bench.py: bad world size / rank")
    return total, list(range(total))[rank::world]


def workload_cameras(name, views, scaling, world, rank):
    total, idx = plan_views(name, views, scaling, world, rank)
    cams = orbit_cameras(name, total)
    return [cams[i] for i in idx], total


def aggregate_fps(n_local_views, ms_local, reduce_sum=None, reduce_max=None):
    """Whole-job frames/s: the views ALL ranks processed in one step divided by the
    slowest rank's step time (max over ranks).  reduce_* are the collectives
    (identity on one process)."""
    n = reduce_sum(n_local_views) if reduce_sum else n_local_views
    ms = reduce_max(ms_local) if reduce_max else ms_local
    return n / (ms / 1e3), n, ms


def default_views(name):
    return {"train8_1m": 8, "mip360_1m": 1, "nerfsynth200k": 8, "sweep64_3m": 64,
            "small360": 4}[name]


# ----------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
def flops_model(cnt, K=0):
    """Algorithmic FP32 work per view from the per-pixel counters:
    F_fwd = 8 X_s + 14 X_h + 16 X_p + 15 X_c;  F_bwd = F_fwd (replay) + 60 X_c
    + 30 * (active plane endpoints, <= 2 X_c).  With K detail sites (NEXT-2,
    DESIGN §13) each composited segment adds (40 + 86 K) forward (two chart points,
    two K-site soft-Voronoi evaluations at 16 K, the 8-axis SV blend at 54 K) and
    (558 + 46 K) more backward (the reverse chain, the outer product 24 K x 2)."""
    Xs, Xh, Xp, Xc = (float(v) for v in cnt)
    f_fwd = 8 * Xs + 14 * Xh + 16 * Xp + 15 * Xc
    f_bwd = f_fwd + 60 * Xc + 30 * 2 * Xc
    if K:
        f_fwd += (40 + 86 * K) * Xc
        f_bwd += (40 + 86 * K) * Xc + (558 + 46 * K) * Xc
    return f_fwd, f_bwd


def load_peaks():
    try:
        return json.load(open(PEAKS_PATH)), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def workload_tag(args):
    return (args.workload + ("+dipoles" if args.dipoles and not args.detail else "") +
            (f"+detail{args.detail}" if args.detail else "") +
            ("+fisheye" if args.fisheye else "") + ("+trace" if args.trace else "") +
            ("+knn_lists" if args.lists == "knn" else ""))


def is_train(args):
    """fwd+bwd training step, or a forward render (render-FPS workloads, --trace)."""
    return not args.trace and args.workload not in ("mip360_1m", "sweep64_3m")


def make_config(args, sc, W, H, total_views, ws):
    """The JSON line's `config` -- built identically by both arms."""
    train = is_train(args)
    return {"workload": workload_tag(args), "cells": sc.num_cells, "edges": sc.num_edges,
            "batch_views": total_views, "views_per_gpu": total_views / ws,
            "global_batch_views": total_views, "view_deal": "round-robin (rank r: r, r+N, ...)",
            "width": W, "height": H, "pass": "fwd+bwd" if train else "fwd",
            "parallelism": f"dp{ws} (views sharded, per-cell grad all-reduce)",
            "l2": "inputs larger than L2 (scene records+edges+grad_out > 126 MB)",
            "k0_policy": "edge records rebuilt every step (training)" if train
            else "static scene: edge records built once at creation"}


# ----------------------------------------------------------------------------
def run_reference(args):
    """The reference arm = the oracle (CPU, double, O3 tile lists, all host cores),
    as it stands, on the workload's own scene and views.  Every step (warm-up and
    timed) renders ONE WHOLE view of the batch (forward, + backward for training
    workloads) -- a bounded sample of the workload's step -- cycling through the
    batch; frames/s = views rendered / time, measured, not extrapolated.  Under
    torchrun only rank 0 works."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import pf_synth
    wl = args.workload
    sc = pf_synth.make_scene(wl, variant=args.lists, dipoles=args.dipoles, detail=args.detail)
    total, _ = plan_views(wl, args.views, args.scaling, ws, 0)
    cams = orbit_cameras(wl, total)
    if args.fisheye:
        cams = [pf_synth.fisheye(c, 200.0) for c in cams]
    train = is_train(args)
    H, W = cams[0].height, cams[0].width
    g = pf_synth.make_grad_out(1, H, W, seed=12)[0] if train else None

    def one_view(k):
        cam = cams[k % len(cams)]
        if args.trace:
            oracle.trace(sc, cam)
            return
        oracle.render(sc, cam, mode=oracle.O3)
        if train:
            oracle.backward(sc, cam, g, mode=oracle.O3)

    k = 0
    for _ in range(args.warmup):
        one_view(k)
        k += 1
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_view(k)
        k += 1
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    val = 1.0 / dt
    cores = oracle.num_threads()
    sample = (f"each step = one whole {W}x{H} view of the {total}-view batch (views cycled), "
              f"oracle {'tracer' if args.trace else 'O3'} "
              f"{'forward+backward' if train else 'forward'} in double on "
              f"{cores} host threads: {dt:.2f} s per view")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt,
            "step_views": 1, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": make_config(args, sc, W, H, total, ws),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "the oracle on rank 0's host cores; ms_per_step is one view (step_views)"}
    print(json.dumps(line), flush=True)


def cpu_baseline(sc, cam, seconds, train=True, calib=None, trace=False):
    """Times the oracle (O3 tile-list mode, double, OpenMP over all host cores) on
    a bounded sample of pixel rows of one view and extrapolates to frames/s.
    Each oracle call rebuilds its own fp32 binning (a fixed per-frame cost A), so
    two samples of different size give A and the per-pixel cost B:
    frame time = A + B * W * H  (forward + backward when train)."""
    import oracle
    import pf_synth
    H, W = cam.height, cam.width
    g = pf_synth.make_grad_out(1, H, W, seed=12)[0]

    def run(rows):
        y = (np.arange(rows) * max(H // max(rows, 1), 1))[:rows]
        y = y[y < H]
        pix = np.stack(np.meshgrid(np.arange(W), y), -1).reshape(-1, 2)
        t0 = time.perf_counter()
        if trace:
            oracle.trace(sc, cam, pixels=pix)
            return time.perf_counter() - t0, pix.shape[0]
        oracle.render(sc, cam, mode=oracle.O3, pixels=pix)
        if train:
            oracle.backward(sc, cam, g[pix[:, 1], pix[:, 0]], mode=oracle.O3, pixels=pix)
        return time.perf_counter() - t0, pix.shape[0]

    if calib is None:
        t1, n1 = run(2)
        t1b, n1b = run(8)
        B = max((t1b - t1) / max(n1b - n1, 1), 1e-9)
        A = max(t1 - B * n1, 0.0)
        calib = {"A": A, "B": B}
    A, B = calib["A"], calib["B"]
    rows = int(max(4, min(H, (seconds - A) / B / W)))
    t, n = run(rows)
    # refine the per-pixel cost with the big sample (A from the calibration)
    B2 = max((t - A) / n, 1e-12)
    frame = A + B2 * W * H
    return {"value": 1.0 / frame, "calib": {"A": A, "B": B2}, "cores": oracle.num_threads(),
            "sample": f"{n} pixels ({rows} rows) of one {W}x{H} view, oracle "
                      f"{'tracer' if trace else 'O3'} "
                      f"{'forward+backward' if train else 'forward'} in {t:.1f}s; "
                      f"per-frame fixed cost (own fp32 binning) {A:.2f}s + {B2 * 1e6:.2f}us/pixel "
                      f"-> {frame:.1f}s per frame"}


def load_traffic(kernel_tag, workload, full=False):
    """DRAM bytes per launch of a kernel from the newest committed ncu export of the
    SAME workload (full=True: the whole record, incl. the warp-instruction count).
    A capture of another workload is not this launch's traffic: None then."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        if kernel_tag in d and d[kernel_tag].get("workload") == workload:
            if full:
                return d[kernel_tag]
            return d[kernel_tag]["traffic_bytes"], d[kernel_tag]["source"]
    return None if full else (None, None)


# ----------------------------------------------------------------------------
def _free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def share_gpu():
    """Test-only knob (PF_BENCH_SHARE_GPU=1): every rank on cuda:0 with the gloo
    backend, so the N-rank path of this script (self-launch, view deal, all-reduce
    timing, whole-job FPS) can be exercised on a one-GPU box.  Never a bench number."""
    return os.environ.get("PF_BENCH_SHARE_GPU") == "1"


def self_launch(args):
    """`--gpus N` outside torchrun: re-exec under torch.distributed.run with N ranks
    (one per GPU, rendezvous on 127.0.0.1).  Fails loudly if fewer than N GPUs are
    visible, or if a torchrun world size disagrees with --gpus."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None:
        if int(ws_env) != args.gpus and not (args.gpus == 1 and args.impl == "reference"):
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
        return
    if args.gpus <= 1 or args.impl == "reference":
        return
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus and not share_gpu():
        raise SystemExit(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, "
                         f"found {n}")
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # keep the communicator INIT lines visible
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execvpe(sys.executable, cmd, env)


def main():
    args = parse()
    self_launch(args)
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2604_24994_b200 as pf
    import pf_synth

    ws, rank, local = dist_env()
    if share_gpu():
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if share_gpu():
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def red(x, op):
        if ws == 1:
            return x
        t = torch.tensor([float(x)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    red_sum = lambda x: red(x, dist.ReduceOp.SUM)
    red_max = lambda x: red(x, dist.ReduceOp.MAX)
    wl = args.workload
    t_gen = time.perf_counter()
    sc = pf_synth.make_scene(wl, variant=args.lists, dipoles=args.dipoles, detail=args.detail)
    cams, total = workload_cameras(wl, args.views, args.scaling, ws, rank)
    if args.fisheye:
        cams = [pf_synth.fisheye(c, 200.0) for c in cams]
    nv = len(cams)
    t_gen = time.perf_counter() - t_gen
    H, W = cams[0].height, cams[0].width
    train = is_train(args)
    # render-FPS workloads draw a fixed scene: its edge records (K0) are built once at
    # creation (PF_STATIC_SCENE); training workloads rebuild them every step
    r = pf.Renderer.from_scene(sc, dev, flags=0 if train else pf.PF_INFERENCE | pf.PF_STATIC_SCENE)
    # render-only handle for the training workloads' forward-only figure (no backward
    # state saved; edge records still rebuilt per call, as in training).  The render
    # workloads time `r` itself, so value, ms_per_step and k0_policy describe one run.
    r_inf = r.sibling(pf.PF_INFERENCE) if train else r
    N = sc.num_cells
    grad_out = torch.from_numpy(pf_synth.make_grad_out(nv, H, W, seed=12 + rank)).to(dev)
    flat = torch.zeros(r.grad_size, device=dev, dtype=torch.float32)
    out = torch.empty((nv, H, W, 4), device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()

    from paper_2604_24994_b200 import dist as pfd

    def render(rr, o):
        return rr.trace(cams, out=o) if args.trace else rr.forward(cams, out=o)

    def step():
        if train:
            pfd.train_step(r, cams, grad_out, flat, out=out)   # fwd, bwd, NCCL all-reduce
        else:
            render(r, out)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # ---------------- timed region (device events, max over ranks) ----------
    r.set_profiling(True)
    r.stage_times()
    l0 = r.launch_count()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.5)          # let the sampler take its first reading
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    time.sleep(0.25)
    clocks = clk.stop()
    launches = r.launch_count() - l0
    stages = r.stage_times()
    r.set_profiling(False)
    fps, n_all, ms_step = aggregate_fps(nv, e0.elapsed_time(e1) / args.steps, red_sum, red_max)

    # ---------------- forward-only throughput (extra) ------------------------
    for _ in range(2):
        render(r_inf, out)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        render(r_inf, out)
    f1.record(stream)
    barrier()
    fwd_fps, _, fwd_ms = aggregate_fps(nv, f0.elapsed_time(f1) / args.steps, red_sum, red_max)

    # ---------------- the all-reduce alone (N > 1): time and bus bandwidth ----
    allreduce = None
    if ws > 1 and train:
        for _ in range(3):
            dist.all_reduce(flat, op=dist.ReduceOp.SUM)
        barrier()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(args.steps):
            dist.all_reduce(flat, op=dist.ReduceOp.SUM)
        q1.record(stream)
        barrier()
        ar_ms = red_max(q0.elapsed_time(q1) / args.steps)
        nbytes = flat.numel() * 4
        allreduce = {"ms": ar_ms, "bytes": nbytes,
                     "busbw_gbs": 2 * (ws - 1) / ws * nbytes / (ar_ms / 1e3) / 1e9,
                     "algbw_gbs": nbytes / (ar_ms / 1e3) / 1e9,
                     "note": "one dist.all_reduce(SUM) of the flat f32 gradient buffer over "
                             "NCCL, max over ranks; busbw = 2(N-1)/N * bytes / t"}

    # ---------------- weak-scaling figure at N > 1 (extra) --------------------
    weak = None
    if ws > 1 and args.scaling == "strong" and train:
        wcams, wtotal = workload_cameras(wl, args.views, "weak", ws, rank)
        if args.fisheye:
            wcams = [pf_synth.fisheye(c, 200.0) for c in wcams]
        wnv = len(wcams)
        wg = torch.from_numpy(pf_synth.make_grad_out(wnv, H, W, seed=12 + rank)).to(dev)
        wout = torch.empty((wnv, H, W, 4), device=dev, dtype=torch.float32)
        for _ in range(2):
            pfd.train_step(r, wcams, wg, flat, out=wout)
        barrier()
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        for _ in range(args.steps):
            pfd.train_step(r, wcams, wg, flat, out=wout)
        w1.record(stream)
        barrier()
        wfps, wn, wms = aggregate_fps(wnv, w0.elapsed_time(w1) / args.steps, red_sum, red_max)
        weak = {"value": wfps, "unit": UNIT, "views_per_gpu": wnv, "global_batch_views": wn,
                "ms_per_step": wms, "note": "every rank renders its own full batch"}
        del wg, wout

    # ---------------- end to end: host buffers through the public API -------
    e2e = None
    if not args.no_e2e:
        g_host = grad_out.cpu().pin_memory() if train else None
        res_host = [(torch.empty(r.grad_size, dtype=torch.float32) if train
                     else torch.empty(out.shape, dtype=torch.float32)).pin_memory()
                    for _ in range(2)]
        # double-buffered device copies; H2D and D2H on their own streams (PCIe is
        # full duplex): the step's dL/dimage uploads while its forward runs (the
        # forward does not read it), its gradients download while the next
        # step's forward runs.  Every step still moves its own bytes both ways.
        g_dev = [torch.empty_like(grad_out) for _ in range(2)]
        flats = [flat, torch.zeros_like(flat)]
        outs = [out, torch.empty_like(out)]
        h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev = {k: [torch.cuda.Event(), torch.cuda.Event()] for k in ("h2d", "used", "d2h")}
        for b in range(2):
            for k in ev:
                ev[k][b].record(stream)
        step_no = [0]

        # the download of step k's result is enqueued during step k+1, once its forward
        # call has returned: the forward's own small readback (the pair counts, the
        # call's one host sync) then never waits behind a large D2H on the bus
        pending = [None]

        def enqueue_d2h(bp):
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev["used"][bp])
                res_host[bp].copy_(flats[bp] if train else outs[bp], non_blocking=True)
                ev["d2h"][bp].record(d2h)

        def e2e_step():
            b = step_no[0] & 1
            step_no[0] += 1
            prev = pending[0]
            if train:   # the step's dL/dimage arrives from the host, grads go back
                with torch.cuda.stream(h2d):
                    h2d.wait_event(ev["used"][b])        # step k-2's backward read g_dev[b]
                    g_dev[b].copy_(g_host, non_blocking=True)
                    ev["h2d"][b].record(h2d)
                stream.wait_event(ev["d2h"][b])          # step k-2's download of flats[b]

                def before_backward():
                    stream.wait_event(ev["h2d"][b])
                    if prev is not None:
                        enqueue_d2h(prev)                # step k-1's gradients go down

                pfd.train_step(r, cams, g_dev[b], flats[b], out=out,
                               before_backward=before_backward)
            else:       # forward-only: the rendered images go back to the host
                stream.wait_event(ev["d2h"][b])
                render(r, outs[b])
                if prev is not None:
                    enqueue_d2h(prev)                    # step k-1's images go down
            ev["used"][b].record(stream)
            pending[0] = b

        for _ in range(2):
            e2e_step()
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        enqueue_d2h(pending[0])                          # the last step's download, and
        for b in range(2):                               # every download is in the region
            stream.wait_event(ev["d2h"][b])
        a1.record(stream)
        barrier()
        e2e_fps, _, _ = aggregate_fps(nv, a0.elapsed_time(a1) / args.steps, red_sum, red_max)
        e2e = {"value": e2e_fps, "unit": UNIT,
               "h2d_bytes_per_step": int(g_host.numel() * 4) if train else 64 * nv,
               "d2h_bytes_per_step": int(res_host[0].numel() * 4),
               "note": ("H2D of the step's dL/dimage from pinned host (overlapping its "
                        "forward) + fwd + bwd (+ all-reduce) + D2H of the per-cell gradients "
                        "(enqueued during the next step, after its forward call), every step; "
                        "the last step's download inside the timed region") if train
               else ("fwd through the C-ABI (host cameras) + D2H of the rendered images "
                     "(enqueued during the next step, after its forward call), every step; "
                     "the last step's download inside the timed region")}

    trace = None
    if args.trace:
        # NEXT-4: one tracer launch per view, latency-bound pointer chasing; the
        # algorithmic bytes of a walk step are the cell's records (A, B, E: 40 B) and
        # its edge records (16 B x degree) plus the next cell's CSR index (4 B)
        _, tst = r.trace(cams[:1], stats=True)
        deg_mean = sc.num_edges / max(sc.num_cells, 1)
        b_launch = tst["visited"] * (44 + 16 * deg_mean) + 16 * W * H
        t_launch = fwd_ms / nv / 1e3
        peaks_t, _ = load_peaks()
        hbm_t = float(peaks_t.get("hbm_gbs", 6650.0))
        trace = {"stats_view0": tst, "cells_per_ray": tst["visited"] / max(tst["rays"], 1),
                 "locates_per_ray": tst["located"] / max(tst["rays"], 1),
                 "segments_per_ray": tst["segments"] / max(tst["rays"], 1),
                 "roofline": {"bound": "hbm", "kernel": "k9_trace",
                              "achieved": b_launch / t_launch / 1e9, "peak": hbm_t,
                              "unit": "GB/s", "frac": b_launch / t_launch / 1e9 / hbm_t,
                              "algorithmic_bytes_per_launch": b_launch,
                              "note": "walk-step records (cellA/B/E + edges + CSR index) "
                                      "per launch / launch time (step time / views)"}}

    # ---------------- counters -> algorithmic flops, roofline ----------------
    cnt = np.zeros(4)
    for c in cams[:2]:
        cnt += r.debug_counters(c).sum(dim=(0, 1)).double().cpu().numpy()
    cnt /= min(2, len(cams))
    f_fwd, f_bwd = flops_model(cnt, K=args.detail)
    peaks, peaks_kind = load_peaks()
    k6_ms, k6_n = stages["K6_forward"]
    k7_ms, k7_n = stages["K7_backward"]
    sm_max = clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = SM_COUNT * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    dom = "K7_backward" if (train and k7_ms >= k6_ms) else "K6_forward"
    d_ms, d_n = stages[dom]
    d_avg = d_ms / max(d_n, 1)
    # views per launch: one per launch for 1080p views, all views of the call for a
    # fused small-view launch (DESIGN 6, launch shape)
    views_per_launch = nv * args.steps / max(d_n, 1)
    d_flops = (f_bwd if dom == "K7_backward" else f_fwd) * views_per_launch
    achieved = d_flops / (d_avg / 1e3) / 1e12 if d_avg > 0 else 0.0
    ktag = ("k7_backward" if dom == "K7_backward" else "k6_forward") + ("_detail" if args.detail else "")
    if not train and not args.detail:
        ktag = "k6_forward_inference"                    # render workloads run the inference K6
    traffic, traffic_src = load_traffic(ktag, workload_tag(args))
    prof = load_traffic(ktag, workload_tag(args), full=True) or {}
    kname = dom
    if args.detail and dom == "K7_backward" and d_n > nv * args.steps:
        # split detail backward (DESIGN 13): the stage is the K7 replay + the K7D chain,
        # one launch of each per view (1080p); the captures are per-view launches too
        kname = "K7_backward (K7 replay + K7D chain)"
        parts = [load_traffic(t, workload_tag(args), full=True)
                 for t in ("k7_backward_detail", "k7d_detail_chain")]
        if all(parts):
            traffic = sum(p_["traffic_bytes"] for p_ in parts)
            traffic_src = " + ".join(p_["source"] for p_ in parts)
            prof = {"warp_inst": sum(p_.get("warp_inst", 0.0) for p_ in parts),
                    "issue_pct_of_peak": None}
        else:
            traffic, traffic_src, prof = None, None, {}
        per_view_ms = d_ms / (nv * args.steps)
        d_avg, views_per_launch = per_view_ms, 1.0       # per view: both kernels
        d_flops = f_bwd
        achieved = d_flops / (d_avg / 1e3) / 1e12 if d_avg > 0 else 0.0
    roofline = {"bound": "alu", "kernel": kname, "achieved": achieved, "peak": fp32_peak,
                "unit": "TFLOP/s", "frac": achieved / fp32_peak if fp32_peak else None,
                "traffic": traffic, "traffic_unit": "bytes/launch (dram read+write)",
                "traffic_source": traffic_src or ("no committed ncu capture of this kernel "
                                                  "on this workload"),
                "peak_note": f"FP32 = {SM_COUNT} SM x {FP32_LANES_PER_SM} lanes x 2 x "
                             f"{sm_max:.0f} MHz (guide unit counts; no tensor-core path)",
                "avg_launch_ms": d_avg, "views_per_launch": views_per_launch,
                "algorithmic_flops_per_launch": d_flops}
    if prof.get("warp_inst") and d_avg > 0:
        # the SM issue roofline: 4 schedulers x 148 SMs x clock warp-instructions/s
        issue_peak = 4 * SM_COUNT * sm_max * 1e6
        roofline["issue"] = {
            "warp_inst_per_launch": prof["warp_inst"],
            "achieved_ginst_s": prof["warp_inst"] / (d_avg / 1e3) / 1e9,
            "peak_ginst_s": issue_peak / 1e9,
            "frac": prof["warp_inst"] / (d_avg / 1e3) / issue_peak,
            "ncu_issue_pct": prof.get("issue_pct_of_peak"),
            "note": "instruction count of one launch from the committed ncu capture "
                    "(same kernel, same workload); the FP32 fraction is below this because "
                    "the path is not FMA-shaped (a plane clip is ~17 SASS instructions for "
                    "16 algorithmic flops) and the per-(warp, cell) lockstep work (sphere "
                    "test, warp plane cull, compositing, K6->K7 record) is overhead; the "
                    "algorithmic flops count every list plane (~11 per hit), the warp plane "
                    "cull leaves ~5.8 per (warp, hit cell) (profiles/r02_k6_experiments.md)"}
    sort_ms, sort_n = stages["K4_sort"]
    pairs = r.pair_counts(nv)
    P = float(np.mean(pairs))
    bcount = r.debug_binning(cams[0])["count"]
    n_vis = float((bcount > 0).sum().item())
    # depth-first binning (DESIGN 6, K4): per sort batch of <= 8 views, the visible
    # cells are radix-sorted by (view, depth key) over 32 + view bits, then the pairs by
    # (view, tile) over tile + view bits with 32-bit keys (9- and 8-bit digits);
    # algorithmic bytes per item and pass: cells 8 (histogram key read) + 12 read + 12
    # write, pairs 4 + 8 + 8
    vbits = math.ceil(math.log2(min(nv, 8))) if nv > 1 else 0
    tbits = math.ceil(math.log2((W + 15) // 16 * ((H + 15) // 16)))
    passes_cells = math.ceil((32 + vbits) / 9)          # 9-bit digits (PF_SORT_BITS_WIDE)
    passes_pairs = math.ceil((tbits + vbits) / 8)
    sort_bytes = 32.0 * n_vis * nv * passes_cells + 20.0 * P * nv * passes_pairs
    sort_ms_step = sort_ms / args.steps
    sort_gbs = sort_bytes / (sort_ms_step / 1e3) / 1e9 if sort_ms > 0 else None
    # the 48-bit pair sort this replaces: 6 passes over every pair
    legacy_bytes = 32.0 * P * nv * math.ceil((32 + tbits + vbits) / 8)
    hbm = float(peaks.get("hbm_gbs", 6650.0))

    # ---------------- whole-step rooflines (SURVEY §8(d) byte and flop models) -------
    deg_mean = sc.num_edges / max(N, 1)
    T_tiles = ((W + 15) // 16) * ((H + 15) // 16)
    pix = W * H
    b_view = (36 * N + 8 * N + 16 * n_vis + 12 * P + 8 * P + 8 * T_tiles
              + n_vis * (48 + 16 * deg_mean) + 4 * P + 24 * pix)
    if train:
        b_view += n_vis * (48 + 16 * deg_mean) + 4 * P + 24 * pix + 72 * n_vis + 16 * pix
    b_step = nv * b_view + sort_bytes
    f_step = nv * (f_bwd if train else f_fwd)
    step_s = ms_step / 1e3   # the slowest rank's step
    roofline_step = {
        "fp32_frac": f_step / step_s / (fp32_peak * 1e12),
        "hbm_frac": b_step / step_s / (hbm * 1e9),
        "flops_per_step": f_step, "bytes_per_step": b_step,
        "model": "SURVEY 8(d): B_K1..K6 (+ backward) per view + the measured sort passes; "
                 "F_fwd/F_bwd from the counters; N_vis from view 0's binning",
    }

    # ---------------- NEXT-3: GPU Čech graph build of this scene (extra) --------
    cech = None
    try:
        cb = pf.CechBuilder()
        st_, ra_ = r._tensors[0], r._tensors[2]
        off_, idx_ = cb.build(st_, ra_)
        ok = bool(torch.equal(off_, r._tensors[5]) and torch.equal(idx_, r._tensors[6]))
        ts_ = []
        for _ in range(5):
            c0_, c1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0_.record(stream)
            cb.build(st_, ra_)
            c1_.record(stream)
            torch.cuda.synchronize()
            ts_.append(c0_.elapsed_time(c1_))
        cech = {"build_ms": float(np.median(ts_)), "edges": int(idx_.numel()),
                "equals_input_lists": ok, "note": "pf_cech_build (LBVH), incl. its one sync"}
        cb.close()
    except Exception as ex:  # noqa
        cech = {"error": str(ex)}

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = cpu_baseline(sc, cams[0], args.cpu_seconds, train=train, trace=args.trace)
            cpu = {"value": cpu["value"], "unit": UNIT, "cores": cpu["cores"], "kind": "oracle",
                   "sample": cpu["sample"]}
        except Exception as ex:  # noqa
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle",
                   "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (pf_synth seeded generator, random-init foam)",
            "config": make_config(args, sc, W, H, total, ws),
            "views_this_rank": nv, "allreduce": allreduce, "weak_scaling": weak,
            **({"shared_gpu_test": "PF_BENCH_SHARE_GPU=1: all ranks on cuda:0 over gloo "
                                   "(path test, not a measurement)"} if share_gpu() else {}),
            "clocks": clocks, "gpu_launches": int(launches),
            "e2e": e2e, "roofline": trace["roofline"] if trace else roofline, "roofline_step": roofline_step, "cpu_baseline": cpu,
            "fwd_fps": fwd_fps, "fwdbwd_fps": fps if train else None,
            "mpix_s": fps * W * H / 1e6, "fwd_mpix_s": fwd_fps * W * H / 1e6,
            "stage_ms_per_step": {k: v[0] / args.steps for k, v in stages.items()},
            "stage_launches_per_step": {k: v[1] / args.steps for k, v in stages.items()},
            "pairs_per_view": P, "counters_per_view": {"X_s": cnt[0], "X_h": cnt[1],
                                                       "X_p": cnt[2], "X_c": cnt[3]},
            "sort": {"ms_per_step": sort_ms_step, "launches_per_step": sort_n / args.steps,
                     "pairs_per_step": P * nv, "visible_cells_per_step": n_vis * nv,
                     "passes_cells": passes_cells, "passes_pairs": passes_pairs,
                     "bytes_per_step": sort_bytes, "achieved_gbs": sort_gbs,
                     "hbm_frac": (sort_gbs / hbm) if sort_gbs else None,
                     "legacy_pair_sort_bytes": legacy_bytes,
                     "legacy_equivalent_gbs": legacy_bytes / (sort_ms_step / 1e3) / 1e9
                     if sort_ms > 0 else None,
                     "model": "depth-first binning: visible cells sorted by (view, depth), "
                              "pairs by (view, tile); legacy = one 48-bit sort of all pairs"},
            "peaks_source": peaks_kind, "scene_gen_s": t_gen, "cech_graph": cech,
            "trace": trace,
        }
        print(json.dumps(line), flush=True)
    r.close()
    if r_inf is not r:
        r_inf.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
