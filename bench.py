#!/usr/bin/env python
"""Benchmark: decomposed frames/sec at 1080p (BASELINE.json `metric`).

Workload (BASELINE.json configs[2]): synthetic 1920x1080 clip, K = 8 base
colors, streaming frames (segment + per-frame aux + 2 outer x 2 Gauss-Newton
steps x 16 PCG iterations, fixed iteration counts), warm-started frame to
frame.  A "step" is one streaming frame.  Frame 1 (refinement) runs before
the timed region.  Multi-GPU (--gpus N under torchrun): independent clips per
rank (configs[4]: clips shard across GPUs with no data-path collective),
weak scaling; time = max over ranks of the CUDA-event time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the reference algorithm on the host CPU: the
compiled fp64 restatement of the reference solver (oracle/ls_oracle.c,
pinned to the reference's own outputs by tests/test_oracle_c.py; the
reference package is pure Python/NumPy at ~390 s per 1080p frame and
cannot travel to the GPU box) on full-size frames of the same workload,
every host thread.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decomposed frames/sec at 1080p"
UNIT = "frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="1080p", choices=["1080p", "4k"],
                    help="1080p: BASELINE configs[2] (N>1: one clip per GPU, configs[4]); "
                         "4k: configs[3], 3840x2160 split into row bands, one band per GPU")
    ap.add_argument("--bands", type=int, default=0,
                    help="4k on one process: solve as this many row bands (0: whole frame)")
    ap.add_argument("--height", type=int, default=None)
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--K", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clip", action="store_true", help="skip the timed whole-clip run")
    ap.add_argument("--clip-frames", type=int, default=300)
    ap.add_argument("--profile-only", action="store_true",
                    help="run warmup + steps without the extra legs (for ncu)")
    return ap.parse_args()


def metric_for(args) -> str:
    return METRIC if args.workload == "1080p" else "decomposed frames/sec at 2160p"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_from_profiles(kernel: str):
    """dram bytes per launch from the committed ncu capture summary, if any."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(kernel)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU legs: the compiled restatement of the reference (oracle/ls_oracle.c,
# pinned to the reference's outputs by tests/test_oracle_c.py) on FULL-SIZE
# frames of the same synthetic workload, all host threads (OpenMP over rows)
# ---------------------------------------------------------------------------
def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class CpuClip:
    """Host frames of the bench clip (same generator and seed as the GPU
    leg) and the streaming loop of pipeline.py:136-166 run by the C oracle."""

    def __init__(self, H, W, K, n_frames, seed=0, threads=None):
        import torch
        from oracle import c_oracle as CO
        from paper_1908_01961_b200 import synth
        self.CO = CO
        torch.set_num_threads(max(1, host_cores()))
        clip = synth.make_clip(H, W, K, n_frames, seed=seed, device="cpu")
        self.frames = [f.double().numpy() for f in clip.frames]
        self.colors = clip.colors
        self.seed = seed
        self.threads = threads or host_cores()
        CO.set_threads(self.threads)
        ids = CO.segment(self.frames[0], self.colors)
        r, T = CO.initialize(self.frames[0], ids, self.colors)
        self.prev = _Prev(r, T)

    def frame(self, i):
        """Streaming frame i (segment + aux + 2 outer x 2 GN x 16 PCG), warm
        started from frame i-1's result.  Returns the seconds it took."""
        from dataclasses import replace
        from oracle import lumisplit_oracle as O
        cfg = replace(O.Config(tol_rel=0.0), refine=False, outer_iterations=2)
        t0 = time.perf_counter()
        st = self.CO.stream_frame(self.frames[i], self.colors, self.prev, self.frames[i - 1], O.Weights(),
                                  cfg, self.seed + i)
        dt = time.perf_counter() - t0
        self.prev = _Prev(st.r, st.T)
        return dt


class _Prev:
    def __init__(self, r, T):
        self.r, self.T = r, T


def run_reference(args):
    """The reference arm: the compiled restatement of the reference solver
    (oracle/ls_oracle.c; the reference package itself is pure Python/NumPy,
    ~390 s per 1080p streaming frame) on full-size frames of the
    same workload with every host thread: W warm-up + K timed streaming
    frames, each a whole frame (no strips, no extrapolation)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    H, W, K = args.height, args.width, args.K
    cores = host_cores()
    cc = CpuClip(H, W, K, 1 + args.warmup + args.steps, seed=0, threads=cores)
    for i in range(args.warmup):
        cc.frame(1 + i)
    times = [cc.frame(1 + args.warmup + i) for i in range(args.steps)]
    t = sum(times)
    value = args.steps / t
    sample = (f"{args.steps} full {W}x{H} K={K} streaming frames (segment + aux + 2x2 GN x 16 PCG, fp64) of "
              f"the compiled reference restatement (oracle/ls_oracle.c, OpenMP, {cores} threads), after "
              f"{args.warmup} warm-up frames; same synthetic clip as the GPU arm")
    line = {"metric": metric_for(args), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{W}x{H} K={K} streaming frames (BASELINE configs[2])",
                       "H": H, "W": W, "K": K, "gn_steps_per_frame": 4, "pcg_iterations": 16,
                       "frame_seconds": times},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample, "cpu": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    from paper_1908_01961_b200 import synth, _device, clips, bands as band_mod
    from paper_1908_01961_b200.energy import EnergyWeights
    from paper_1908_01961_b200.palette import BaseColorPalette
    from paper_1908_01961_b200.pipeline import StreamingDecomposer
    from paper_1908_01961_b200.solver import SolveConfig

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    H, W, K = args.height, args.width, args.K
    steps, warmup = args.steps, args.warmup
    e2e_on = not (args.no_e2e or args.profile_only)
    n_frames = 1 + warmup + 2 * steps + (steps if e2e_on else 0)
    four_k = args.workload == "4k"
    pal_seed = 0 if four_k else rank      # 4k: every rank holds a band of the same clip
    clip = synth.make_clip(H, W, K, n_frames, seed=pal_seed, device=dev)
    frames = clip.frames
    pal = BaseColorPalette(colors=clip.colors)
    cfg = SolveConfig(tol_rel=0.0)        # fixed iteration counts
    bands, nb_total, spec = 0, 1, None
    if four_k and world > 1:              # one row band per GPU
        specs = band_mod.plan_bands(H, world)
        spec = specs[rank]
        bands = band_mod.BandedSolver(dev, H, W, K, exchange=band_mod.DistExchange(specs))
        frames = [f[spec.ya:spec.yb].contiguous() for f in frames]
        nb_total = world
    elif four_k and args.bands > 1:       # all bands in this process
        bands, nb_total = args.bands, args.bands
    dec = StreamingDecomposer(pal, EnergyWeights(), cfg, seed=pal_seed, bands=bands)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = dec.first(frames[0])
    torch.cuda.synchronize()
    first_ms = (time.perf_counter() - t0) * 1e3
    n_first_records = len(st.records)
    for i in range(warmup):
        dec.step(frames[1 + i])
    torch.cuda.synchronize()

    if isinstance(bands, band_mod.BandedSolver):
        prof_solvers = [b.solver for b in bands.bands]
    elif bands:
        prof_solvers = [b.solver for b in band_mod.banded_solver(dev, H, W, K, bands).bands]
    else:
        prof_solvers = [_device.get_solver(dev, H, W, K)]
    for ps in prof_solvers:
        ps.profile(False)              # resets the launch counters; no per-kernel events
    clocks = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local])
                          if os.environ.get("CUDA_VISIBLE_DEVICES") else local)

    def timed(first_frame):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e_a.record()
        for i in range(steps):
            dec.step(frames[first_frame + i])
        e_b.record()
        torch.cuda.synchronize()
        return e_a.elapsed_time(e_b), (time.perf_counter() - w0) * 1e3

    # (1) the headline: K frames, nothing but the solve in the timed region
    clocks.start()
    t_ms, wall_ms = timed(1 + warmup)
    clk = clocks.stop()
    launches = sum(ps.profile_read()["launches"] for ps in prof_solvers)
    # (2) the next K frames again with CUDA events around every solver kernel
    #     (per-kernel durations for the roofline; the events cost ~5% of the
    #     frame time, so this pass is not the headline)
    for ps in prof_solvers:
        ps.profile(True)
    prof_t_ms, _ = timed(1 + warmup + steps)
    prof = None
    for ps in prof_solvers:
        pr = ps.profile_read()
        ps.profile(False)
        if prof is None:
            prof = pr
            continue
        for k, v in pr.items():
            if isinstance(v, dict):
                prof[k] = {"count": prof[k]["count"] + v["count"], "ms": prof[k]["ms"] + v["ms"]}
            else:
                prof[k] += v
    if four_k and world > 1:   # strong scaling: the same frames, time = max over ranks
        th = clips.aggregate(steps if rank == 0 else 0, t_ms / 1e3)
    else:
        th = clips.aggregate(steps, t_ms / 1e3)     # frames summed, time = max over ranks
    t_ms = th.seconds * 1e3
    value = th.fps

    # --- roofline of the dominant kernel (algorithmic bytes / event time) ---
    split = world if (four_k and world > 1) else 1     # GPUs sharing one frame
    # one launch covers one band's own rows (the whole frame without bands)
    N = H * W // nb_total
    U = K + 4
    ent_per_px = prof["adjacency_entries"] / N
    # k_pcg_apply: reads X, z, p_prev (3U), edge, row_ptr, entries; writes p, q (2U).
    # (With LS_X_DEFERRED=1 -- round 1's layout -- it also reads and writes x for
    # the deferred x-update: 7U.  By default every search direction is kept and
    # x = sum alpha_i p_i is formed once after the loop, k_pcg_combine.)
    x_deferred = os.environ.get("LS_X_DEFERRED") == "1"
    bytes_apply = N * (4 * ((7 if x_deferred else 5) * U + 2) + 2 * ent_per_px)
    # k_pcg_update: reads z, q, dinv (3U); writes z (U) -- only the preconditioned
    # residual is carried (r = z / dinv on the fly); the last of the 16 launches
    # writes nothing (3U): the per-launch average
    n_it = cfg.pcg_iterations
    bytes_update = N * 4 * U * (4 * (n_it - 1) + 3) / n_it
    kern = {
        "apply": (prof["apply"], bytes_apply),
        "update": (prof["update"], bytes_update),
    }
    kname = {"apply": "k_pcg_apply", "update": "k_pcg_update"}
    dom = max(kern, key=lambda k: kern[k][0]["ms"])
    pst, bpl = kern[dom]
    avg_ms = pst["ms"] / max(pst["count"], 1)
    peak, peak_src = peaks()
    achieved = bpl / (avg_ms / 1e3) / 1e9
    per_kernel = {k: {"launches": v[0]["count"], "avg_us": 1e3 * v[0]["ms"] / max(v[0]["count"], 1),
                      "share_of_step": v[0]["ms"] / prof_t_ms if world == 1 else None,
                      "algorithmic_bytes": v[1],
                      "achieved_gbs": v[1] / (v[0]["ms"] / max(v[0]["count"], 1) / 1e3) / 1e9
                      if v[0]["count"] else None}
                  for k, v in kern.items()}
    for k in ("energy_grad", "trial"):
        per_kernel[k] = {"launches": prof[k]["count"],
                         "avg_us": 1e3 * prof[k]["ms"] / max(prof[k]["count"], 1)}
    it_us = per_kernel["apply"]["avg_us"] + per_kernel["update"]["avg_us"]
    it_bytes = bytes_apply + bytes_update
    pcg_iter = {"bytes": it_bytes, "us": it_us,
                "achieved_gbs": it_bytes / (it_us / 1e6) / 1e9 if it_us else None,
                "frac": it_bytes / (it_us / 1e6) / 1e9 / peak if it_us else None}
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic_from_profiles(kname[dom]),
                "kernel": kname[dom], "peak_source": peak_src,
                "algorithmic_bytes_per_launch": bpl, "avg_launch_us": avg_ms * 1e3,
                "pcg_x_update": ("deferred into the operator (7U per launch)" if x_deferred else
                                 "directions stored, x = sum alpha_i p_i in one pass after the loop "
                                 "(operator 5U per launch)"),
                "per_kernel": per_kernel,
                # one PCG iteration as a unit: operator + update bytes over their
                # summed average launch times
                "pcg_iteration": pcg_iter,
                "timing": f"per-kernel CUDA events over a second timed pass of {steps} frames "
                          f"({prof_t_ms / steps:.2f} ms/frame with the events)",
                # SURVEY.md 8(d) compulsory-traffic model of a whole streaming
                # frame, B_frame = 4 N (860 U + 298) bytes, over the measured frame time
                "frame_model": {"bytes": 4 * H * W * (860 * U + 298),
                                "achieved_gbs": 4 * H * W * (860 * U + 298) / (t_ms / steps / 1e3) / 1e9 / split,
                                "frac": 4 * H * W * (860 * U + 298) / (t_ms / steps / 1e3) / 1e9 / split / peak,
                                "note": "per GPU"}}

    # --- frame 1 again with everything warm (refinement path, host-driven) ---
    # (twice: the first re-run still pays for switching the contexts back from
    # the streaming graphs; the warm figure is the faster of the two)
    first_warm_ms, first_rerun_ms = None, None
    if not args.profile_only:
        runs = []
        for _ in range(2):
            dec1 = StreamingDecomposer(pal, EnergyWeights(), cfg, seed=pal_seed, bands=bands)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dec1.first(frames[0])
            torch.cuda.synchronize()
            runs.append((time.perf_counter() - t0) * 1e3)
            del dec1
        first_rerun_ms, first_warm_ms = runs[0], min(runs)

    # --- e2e through the public API with host buffers ---
    e2e = None
    if e2e_on:
        host = [frames[1 + warmup + 2 * steps + i].cpu().pin_memory() for i in range(steps)]
        # the warm-up frames of the headline pass again, as pinned host frames
        host_warm = [frames[1 + i].cpu().pin_memory() for i in range(warmup)]
        # the step's result as the reference's arrays: r (H, W, 3) and T (H, W, K+1)
        # (energy.py:74-94), interleaved on the device by the unpack kernel, then D2H
        from paper_1908_01961_b200.energy import export_reference_layout
        Hl, Wl = int(st.layers.X.shape[1]), int(st.layers.X.shape[2])
        NB = 3      # read-back buffers in flight (absorbs host-link jitter)
        dev_r = [torch.empty((Hl, Wl, 3), dtype=torch.float32, device=dev) for _ in range(NB)]
        dev_T = [torch.empty((Hl, Wl, K + 1), dtype=torch.float32, device=dev) for _ in range(NB)]
        out_host = [(torch.empty((Hl, Wl, 3), dtype=torch.float32).pin_memory(),
                     torch.empty((Hl, Wl, K + 1), dtype=torch.float32).pin_memory()) for _ in range(NB)]
        side = torch.cuda.Stream(device=dev)
        main = torch.cuda.current_stream()
        up = torch.cuda.Stream(device=dev)

        def e2e_loop(hf):
            """len(hf) frames through dec.step from pinned host memory; returns the
            CUDA-event time of the whole loop (every H2D and D2H inside it)."""
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

            def upload(j):   # frame j's host -> device copy on the upload stream
                with torch.cuda.stream(up):
                    t = hf[j].to(dev, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(up)
                return t, ev

            n = len(hf)
            copied = [None] * NB
            e0.record()
            up.wait_stream(main)
            nxt = upload(0)
            for i in range(n):
                fdev, ev = nxt
                main.wait_event(ev)
                fdev.record_stream(main)
                if i + 1 < n and not os.environ.get("LS_E2E_SERIAL"):
                    nxt = upload(i + 1)          # the next frame's upload overlaps this solve
                elif i + 1 < n:
                    nxt = (hf[i + 1].to(dev, non_blocking=True), torch.cuda.Event())
                    nxt[1].record(main)
                s2 = dec.step(fdev)
                if copied[i % NB] is not None:      # frame i-NB's read-back of this buffer pair
                    main.wait_event(copied[i % NB])
                export_reference_layout(s2.layers, dev_r[i % NB], dev_T[i % NB])
                done = torch.cuda.Event()
                done.record()
                side.wait_event(done)
                with torch.cuda.stream(side):
                    out_host[i % NB][0].copy_(dev_r[i % NB], non_blocking=True)
                    out_host[i % NB][1].copy_(dev_T[i % NB], non_blocking=True)
                    copied[i % NB] = torch.cuda.Event()
                    copied[i % NB].record(side)
            main.wait_stream(side)
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1)

        # untimed warm-up of the same loop: the first pass pays for the upload
        # stream's allocator blocks and the copy-stream setup (~1 ms/frame
        # over 20 frames, tools/e2e_probe.py)
        e2e_loop(host_warm)
        e_ms = e2e_loop(host)
        eth = clips.aggregate(steps, e_ms / 1e3)
        if four_k and world > 1:
            eth = clips.aggregate(steps if rank == 0 else 0, e_ms / 1e3)
        e2e = {"value": eth.fps, "unit": UNIT,
               "h2d_bytes_per_step": int(host[0].numel() * 4),
               "d2h_bytes_per_step": int((out_host[0][0].numel() + out_host[0][1].numel()) * 4),
               "api": "pipeline.StreamingDecomposer.step (reference decompose_frames loop); the result "
                      "as the reference's r (H,W,3) and T (H,W,K+1) arrays (unpacked on the device); "
                      "frame i+1's H2D and frame i's D2H on copy streams beside frame i's / i+1's solve"}

    # --- a whole 300-frame clip through decompose_frames,
    #     frame 1 (refinement) included, timed end to end (N = 1 only) ---
    clip300 = None
    if rank == 0 and world == 1 and not four_k and not args.profile_only and not args.no_clip:
        from paper_1908_01961_b200.pipeline import decompose_frames
        n300 = args.clip_frames
        big = synth.make_clip(H, W, K, n300, seed=1, device=dev)
        pal300 = BaseColorPalette(colors=big.colors)
        kept = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = decompose_frames(big.frames, EnergyWeights(), cfg, seed=1, palette=pal300,
                               on_frame=lambda i, s: kept.append(s.status) if i < 0 else None)
        torch.cuda.synchronize()
        sec = time.perf_counter() - t0
        clip300 = {"frames": n300, "seconds": sec, "fps": n300 / sec,
                   "first_frame_ms": 1e3 * res.frame_seconds[0],
                   "streaming_ms_median": 1e3 * statistics.median(res.frame_seconds[1:]),
                   "api": "pipeline.decompose_frames (generator palette, frame 1 refined), device-resident frames, "
                          "host wall clock with a device synchronisation at both ends"}
        del big, res

    # --- CPU baseline (rank 0, N = 1 only): 3 full streaming frames of the
    #     compiled reference restatement on every host thread, the last 2 timed
    #     (a single timed frame showed host noise of +-20% between runs) ---
    cpu = None
    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.profile_only):
        cores = host_cores()
        cc = CpuClip(H, W, K, 4, seed=0, threads=cores)
        cc.frame(1)
        dt = cc.frame(2) + cc.frame(3)
        cpu = {"value": 2.0 / dt, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"2 full {W}x{H} K={K} streaming frames (segment + aux + 2x2 GN x 16 PCG, fp64) of the "
                         f"compiled reference restatement (oracle/ls_oracle.c, OpenMP over rows, {cores} "
                         f"threads), after 1 untimed frame",
               "cpu": cpu_model()}

    if rank == 0:
        line = {"metric": metric_for(args), "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
                "warmup": warmup, "ms_per_step": t_ms / steps, "higher_is_better": True,
                "scaling": "strong" if four_k else "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": {"workload": (f"{W}x{H} K={K} streaming frames as {nb_total} row band(s) "
                                        f"(BASELINE configs[3]; one band per GPU, halo + all-gather over "
                                        f"NCCL)" if four_k else
                                        f"{W}x{H} K={K} streaming frames (BASELINE configs[2]); "
                                        f"N>1: one independent clip per GPU (configs[4])"),
                           "bands": nb_total,
                           "H": H, "W": W, "K": K, "gn_steps_per_frame": 4, "pcg_iterations": 16,
                           "l2": "per-frame working set (~0.9 GB) exceeds the 126 MB L2; no flush",
                           "first_frame_ms": first_ms, "first_frame_warm_ms": first_warm_ms,
                           "first_frame_rerun_ms": first_rerun_ms,
                           "first_frame_records": n_first_records,
                           # whole-clip rate of a 300-frame clip including
                           # frame 1 (refinement), from the warm frame-1 time and the measured
                           # streaming frame time (extrapolated, not a timed 300-frame run)
                           "whole_clip_fps_300_est": (300.0 / ((first_warm_ms + 299 * t_ms / steps) / 1e3)
                                                      if first_warm_ms else None),
                           "whole_clip": clip300,
                           "wall_ms_per_step": wall_ms / steps},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.height is None:
        args.height = 2160 if args.workload == "4k" else 1080
    if args.width is None:
        args.width = 3840 if args.workload == "4k" else 1920
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
