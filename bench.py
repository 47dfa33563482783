#!/usr/bin/env python
"""Benchmark of the Snake-NeRF 2x2-window training hot path on B200.

Metric (BASELINE.json): training rays/s of the 2x2 window (ray generation +
segmentation + sampling, field fwd/bwd, compositing + loss + backward, fused
Adam, periodic occupancy update), whole job over N GPUs; plus render rays/s.

Workload: config 5 (6x6 grid of 128 m tiles, 16 synthetic views ~1650^2 px at
0.5 m, a 65,536-ray global batch, window at position (2,2)).  Ray-sharded data
parallelism (strong scaling, BASELINE config 5): rank r of N trains rays
[r*B/N, (r+1)*B/N) of the global counter-RNG stream, with an NCCL allreduce of
the 7.01 MB gradient; the loss is normalised by the global B.

`python bench.py [--gpus N --steps K --warmup W]`           (our arm)
`python bench.py --impl reference [...]`                     (CPU reference arm)

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N ranks (one process per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training rays/sec (2x2 window, fwd+bwd+Adam)"
UNIT = "rays/s"
B_GLOBAL = 65536          # BASELINE config 5: one global batch, sharded over the ranks
WINDOW = (2, 2)
FLOP_FWD = 17664          # per sample (density 4,096 + colour 13,568), SURVEY.md §8
FLOP_FWD_BWD = 52992      # per sample
FLOP_BWD = FLOP_FWD_BWD - FLOP_FWD  # 35,328: the backward's own work (its forward recompute is credited to field_fwd)
SCATTER_BYTES = 8 * 8 * 8  # per sample: 8 levels x 8 corners x float2 of reds
DTYPE = "bf16 MLP operands (tcgen05, fp32 accumulate); fp32 hash grid, compositing, Adam; fp64 rays"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line) via NVML in a 5 ms background thread; the
    timed region is ~0.1-0.3 s, shorter than nvidia-smi's sampling period."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    self.reasons |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    pass
                time.sleep(self.period)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._t.join()

    def summary(self):
        rs = sorted(n for n, b in self.REASONS.items() if self.reasons & b)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": rs, "samples": len(self.samples),
                "source": "NVML, 5 ms, during the timed region"}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def relaunch(n: int) -> int:
    """One process per GPU: re-executes this command under torch.distributed.run
    (rendezvous on 127.0.0.1) and returns its exit code."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator size / NVLS visible in the log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def cpu_baseline(scene, n_rays: int, steps: int, warmup: int):
    """The CPU oracle trainer (oracle/, the reference's algorithm restated; the
    absent trainer/field bodies have no other CPU implementation) on all host
    cores, on a bounded sample of the same workload (same scene, window,
    seeds; n_rays per iteration instead of 65,536)."""
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.abi import FieldConfig, TrainConfig

    cores = os.cpu_count() or 1
    ses = Session(Oracle(), scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=n_rays, seed=2),
                  workers=cores)
    ses.set_window(*WINDOW)
    t0 = time.perf_counter()
    n_acc = ses.build_accept().size
    t_accept = time.perf_counter() - t0
    for i in range(warmup):
        ses.train_step(i, 0, n_rays)
    t0 = time.perf_counter()
    for i in range(steps):
        ses.train_step(warmup + i, 0, n_rays)
    dt = time.perf_counter() - t0
    return {"value": n_rays * steps / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"oracle trainer on cfg5 window {WINDOW}: {steps} timed iterations x {n_rays} rays "
                      f"(after {warmup} warm-up; accepted-ray list of {n_acc} built once in {t_accept:.1f} s, untimed)"}


def cpu_render_baseline(scene, fc, R: int, W: int, n: int = 8192):
    """The oracle's render path (sample_pixels -> field forward -> composite)
    on the host cores for a bounded sample of the render view's pixels: the
    central half of the image, which the centre 2x2 window covers (the oracle
    holds one 2x2 window; the GPU render holds all 16 tiles)."""
    import numpy as np

    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.abi import TrainConfig

    cores = os.cpu_count() or 1
    ses = Session(Oracle(), scene, fc, TrainConfig.defaults(batch_rays=n), workers=cores)
    ses.set_window(1, 1)
    rng = np.random.default_rng(0)
    px = np.stack([np.zeros(n, np.int64), rng.integers(R // 4, 3 * R // 4, n), rng.integers(W // 4, 3 * W // 4, n)],
                  axis=1).astype(np.int32)
    ses.sample_pixels(px[:512])  # warm-up
    ses.forward()
    ses.composite()
    t0 = time.perf_counter()
    ses.sample_pixels(px)
    ses.forward()
    ses.composite()
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "rays/s", "cores": cores, "kind": "port",
            "sample": f"oracle render of {n} pixels of the config-4 view's central half (window (1, 1)), "
                      "sample + field forward + composite"}


def run_reference(args):
    """The reference arm: the CPU oracle trainer (restated reference algorithm,
    primitives pinned bit-for-bit to the reference sources) on all host cores,
    exactly --steps timed iterations after --warmup, each a bounded 2048-ray
    sample of the same workload.  Under torchrun only rank 0 runs."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2507_01631_b200 import synth

    scene = synth.config_scene(5, seed=0)
    n = 4096
    cb = cpu_baseline(scene, n, args.steps, args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (fp64 rays)", "data": "synthetic",
            "config": {"workload": "cfg5 6x6 grid, 2x2 window at (2,2), 16 views ~1650^2 px, bounded ray sample",
                       "rays_per_step": n},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


KERNEL_UNITS = {
    # phase: (bound, per-sample, per-ray, unit) algorithmic work
    "field_bwd": ("tensor", FLOP_BWD, 0, "flop"),
    "field_fwd": ("tensor", FLOP_FWD, 0, "flop"),
    "composite": ("hbm", 40, 36, "byte"),
    "sampler": ("hbm", 22, 79, "byte"),
    "adam": ("hbm", 0, 0, "byte"),
}


def red_peak():
    """Measured red.global.add throughput of this GPU model (tools/red_peak.cu
    on a B200, committed as profiles/red_peak.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "red_peak.json")) as f:
            r = json.load(f)
        width = {"red.global.add.f32": 4, "red.global.add.v2.f32": 8, "red.global.add.v4.f32": 16}
        # every width sustains the same lane-request rate (~214 G/s on B200):
        # the scatter is bound by red requests, not bytes
        lanes = max(v["GBps"] * 1e9 / width[v["op"]] for v in r["variants"] if v["op"] in width)
        return {"GBps": float(r["best_GBps"]), "lanes_per_s": lanes, "source": r.get("source", "profiles/red_peak.json")}
    except Exception:
        return None


def red_lanes():
    """Dynamic red requests per sample of the backward's scatter, counted by
    ncu on a profiled launch (tools/summarize_profiles.py ->
    profiles/red_lanes.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "red_lanes.json")) as f:
            return json.load(f)
    except Exception:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2507_01631_b200 import synth
    from paper_2507_01631_b200.abi import FieldConfig, TrainConfig
    from paper_2507_01631_b200.tilefield import Context, snake_path, tile_init

    rank, world, local = dist_env()
    if "RANK" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    BG = args.global_batch  # BASELINE config 5: 65,536 (the default; other values for scaling studies only)
    if BG % world:
        raise SystemExit(f"bench.py: the {BG}-ray batch does not split over {world} ranks")
    B = BG // world  # strong scaling: this rank's shard of the global batch
    scene = synth.config_scene(5, seed=0)
    fc = FieldConfig.defaults()
    tc = TrainConfig.defaults(batch_rays=BG, seed=2)
    stream = torch.cuda.current_stream(dev)
    ctx = Context(scene, fc, tc, device=local, max_rays=B, stream=stream.cuda_stream)
    ctx.set_window(*WINDOW)
    grads = ctx.grad_tensor()
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(it, ev=None):
        if ev:
            ev[0].record(stream)
        ctx.forward_backward(it, rank * B, B)
        if world > 1:
            dist.all_reduce(grads)
        ctx.optimizer_step(it)
        if ev:
            ev[1].record(stream)
        l2.zero_()  # flush L2 between timed iterations (outside the step's events)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    _, n_samples = ctx.last_batch()
    # the timed region runs without per-phase events (they cost ~1%); the
    # per-kernel breakdown comes from a second, instrumented pass below
    l0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i, evs[i])
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the K steps, each between its own pair of events: the L2 flush between
    # iterations is not part of a step (the whole bracket is reported too)
    ms = sum(a.elapsed_time(b) for a, b in evs)
    ms_bracket = ev0.elapsed_time(ev1)
    launches = ctx.launches() - l0
    ctx.profile_enable(True)
    for i in range(args.steps):
        step(args.warmup + args.steps + i)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    t = torch.tensor([ms, ms_bracket], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, ms_bracket_max = float(t[0].item()), float(t[1].item())
    value = BG * args.steps / (ms_max / 1e3)

    hbm, tf_burst, tf_sust, peak_src = peaks()
    K = args.steps
    kern = {}
    for ph, (ph_ms, nl) in prof.items():
        if ph_ms <= 0:
            continue
        kern[ph] = {"ms_per_step": ph_ms / K, "share": ph_ms / ms, "launches": nl}
        if ph in KERNEL_UNITS:
            bound, ps, pr, u = KERNEL_UNITS[ph]
            if ph == "adam":
                work = 28 * 1752595 * K
            else:
                work = (ps * n_samples + pr * B) * K
            sec = ph_ms / 1e3
            if bound == "tensor":
                kern[ph].update(bound="tensor", achieved=work / sec / 1e12, unit="TFLOP/s")
            else:
                kern[ph].update(bound="hbm", achieved=work / sec / 1e9, unit="GB/s")
    dom = max((p for p in kern if p in KERNEL_UNITS), key=lambda p: kern[p]["ms_per_step"])
    d = kern[dom]
    peak = (tf_sust if d["bound"] == "tensor" else hbm)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(dom)
        except Exception:
            traffic = None
    roofline = {"kernel": dom, "bound": d["bound"], "achieved": d["achieved"], "peak": peak,
                "unit": d["unit"], "frac": d["achieved"] / peak, "traffic": traffic,
                "peak_source": f"{peak_src} ({'bf16 sustained' if d['bound'] == 'tensor' else 'HBM copy'})",
                "per_launch_work": KERNEL_UNITS[dom][1] * n_samples,
                "per_launch_work_unit": KERNEL_UNITS[dom][3],
                "per_unit": f"{KERNEL_UNITS[dom][1]} {KERNEL_UNITS[dom][3]}/sample x {n_samples} samples/launch"}
    red = red_peak()
    if dom == "field_bwd" and red:
        # The backward is bound by its hash-gradient scatter (8 levels x 8
        # corners x float2 of global reds per sample), not the tensor cores:
        # reported against the measured red.global throughput of this GPU
        # (tools/red_peak.cu, profiles/red_peak.json) beside the tensor peak.
        bwd_ms = d["ms_per_step"]
        ach = SCATTER_BYTES * n_samples / (bwd_ms / 1e3) / 1e9
        roofline["limiter"] = {
            "resource": "global fp32 reds of the hash-table gradients (random indices into the 7 MB window tables)",
            "red_bytes_per_sample": SCATTER_BYTES, "achieved": ach, "unit": "GB/s of red payload",
            "peak": red["GBps"], "frac": ach / red["GBps"], "peak_source": red["source"]}
        rl = red_lanes()
        if rl:
            # the same bound in the unit the hardware limits: red requests
            # (one per lane per red instruction, any width); the count per
            # sample is ncu's dynamic count on a profiled launch (the
            # butterfly merges and v4 pairing make it data dependent)
            lps = rl["lane_reds_per_sample"] * n_samples / (bwd_ms / 1e3)
            roofline["limiter"].update({
                "red_requests_per_sample": rl["lane_reds_per_sample"],
                "achieved_requests_per_s": lps, "peak_requests_per_s": red["lanes_per_s"],
                "frac_requests": lps / red["lanes_per_s"],
                "requests_source": rl["source"]})

    # ---- end to end through the public API with host buffers: window slides
    # (pinned host <-> HBM tile state + crops), accepted-list rebuilds, loss
    # readback every step; the window moves every `move_every` iterations
    # along the snake (default 16 = the occupancy interval; the paper trains
    # hundreds of iterations per position, so this over-weights the slide).
    # Steady state of the snake: training starts at a position whose successor
    # is already being staged; every move inside the timed region is a regular
    # prefetched move (the one-off initial load of a run is not timed, like
    # the device metric's).
    path = snake_path(scene.grid_rows, scene.grid_cols)
    ctx.set_window(*path[0])
    ctx.prefetch_window(*path[1])
    h0, d0 = ctx.copy_bytes()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_steps = args.steps
    for i in range(e2e_steps):
        if i % args.move_every == 0 and i > 0:
            k = i // args.move_every
            ctx.set_window(*path[k % len(path)])
            ctx.prefetch_window(*path[(k + 1) % len(path)])  # staged on the side stream
        ctx.forward_backward(10_000 + i, rank * B, B)
        if world > 1:
            dist.all_reduce(grads)
        ctx.optimizer_step(10_000 + i)
        # every step's loss/status reaches the host: requested now, read after
        # the next step is enqueued (pipelined, the stream never drains)
        ctx.request_loss()
        if i > 0:
            ctx.poll_loss()
    ctx.poll_loss()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    h1, d1 = ctx.copy_bytes()
    te = torch.tensor([e2e_s], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": BG * e2e_steps / float(te.item()), "unit": UNIT,
           "h2d_bytes_per_step": (h1 - h0) // e2e_steps, "d2h_bytes_per_step": (d1 - d0) // e2e_steps,
           "window_move_every": args.move_every, "window_moves": (e2e_steps - 1) // args.move_every,
           "what": "public API, host images/tile records: every move stages crops + tile state "
                   "(pinned H2D/D2H) and rebuilds the accepted list (new pixels Newton-solved, the "
                   "previous position's pixels copied from its memo); every step's loss/status copied to the "
                   "host and read (pipelined one step behind)"}

    # ---- render (config 4: 4x4-tile ROI, random-init weights, occupancy all on)
    render = None
    if not args.no_render:
        render = bench_render(args, rank, world, dev)

    out = None
    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu:
            cb = cpu_baseline(scene, 16384, 6, 1)
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
               "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
               "config": {"workload": "cfg5: 6x6 grid of 128 m tiles, 2x2 window at (2,2), 16 synthetic views "
                                      "~1650^2 px at 0.5 m, random-init fields",
                          "rays_per_gpu_per_step": B, "global_batch": BG,
                          "samples_per_step_per_gpu": n_samples,
                          "samples_per_ray": n_samples / B, "parallelism": f"ray-sharded dp{world}",
                          "l2": "flushed between timed iterations (256 MB write)",
                          "timing": "sum of the K steps' own CUDA-event pairs (the flush between them excluded)",
                          "ms_per_step_incl_flush": ms_bracket_max / K},
               "roofline": roofline, "kernels": kern, "cpu_baseline": cb, "e2e": e2e,
               "gpu_launches": launches, "clocks": clk.summary(), "render": render}
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def bench_render(args, rank=0, world=1, dev=None):
    """Config 4: the full 4096^2-class novel view of a 4x4-tile ROI from
    random-init tiles (render_view: every pixel, chunks of 2^20 rays).  With N
    ranks the view's rows are split across the GPUs (no collective); time is
    the max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2507_01631_b200.abi import FieldConfig, Roi, TrainConfig
    from paper_2507_01631_b200.synth import Scene, make_camera
    from paper_2507_01631_b200.tilefield import Context, tile_init

    roi = Roi(0.0, 512.0, 0.0, 512.0, 0.0, 40.0)
    cam = make_camera(roi, 0.125, 12.0, 40.0)
    img = np.zeros((cam.image_rows, cam.image_cols, 3), np.uint8)
    scene = Scene(roi, 4, 4, [cam], [img], 0.125)
    fc = FieldConfig.defaults()
    chunk = 1 << 20
    ctx = Context(scene, fc, TrainConfig.defaults(batch_rays=chunk), max_rays=chunk)
    tiles = [(r, c) for r in range(4) for c in range(4)]
    states = [tile_init(fc, 1, r, c) for r, c in tiles]
    color = ctx.color()[0]
    ctx.render_setup(tiles, states, color)
    # this rank's share of the view: a contiguous band of rows
    R, W = cam.image_rows, cam.image_cols
    r0, r1 = R * rank // world, R * (rank + 1) // world
    rr, cc = np.meshgrid(np.arange(r0, r1), np.arange(W), indexing="ij")
    px = np.stack([rr.ravel(), cc.ravel()], axis=1).astype(np.int32)
    n = px.shape[0]
    ctx.render_pixels(cam, px[:chunk])  # warm-up
    # the caller's output buffers, allocated (and faulted in) before timing,
    # like the training e2e's pinned inputs
    outs = (np.zeros(3 * n, np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32))
    for o in outs:
        o.fill(1.0)
    ctx.profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rgb, dep, op = ctx.render_pixels(cam, px, out=outs)
    wall = time.perf_counter() - t0
    prof = ctx.profile_read()
    dev_ms = sum(prof[p][0] for p in ("sampler", "field_fwd", "composite"))
    ctx.close()
    t = torch.tensor([dev_ms, wall], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, wall = float(t[0]), float(t[1])
    total = R * W
    cpu = None
    if rank == 0 and world == 1 and not getattr(args, "no_cpu", False):
        cpu = cpu_render_baseline(scene, fc, R, W)
    return {"value": total / (dev_ms / 1e3), "unit": "rays/s", "cpu_baseline": cpu,
            "e2e": {"value": total / wall, "unit": "rays/s", "h2d_bytes_per_step": total * 8,
                    "d2h_bytes_per_step": total * 20},
            "config": f"cfg4: 4x4-tile ROI (512 m), full {R}x{W} novel view at 0.125 m over {world} GPU(s) "
                      "(row bands, no collective), random-init weights, occupancy all on, midpoint samples",
            "rays": total,
            "phases_ms": {p: prof[p][0] for p in ("sampler", "field_fwd", "composite")}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--move-every", type=int, default=16, help="e2e: iterations per window position")
    ap.add_argument("--global-batch", type=int, default=B_GLOBAL,
                    help="rays per step over all ranks (default: BASELINE config 5's 65,536; other values are "
                         "for scaling studies, not the headline)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
