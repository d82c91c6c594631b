"""Benchmark of the frequency-bucketed hybrid ocean step (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

One "step" = one frame of the hybrid step over the configured scene
(SURVEY 8(d)): FFT background (rotation + IFFT2 + normals), boundary
injection, advect + cull + compaction + splat, per-bucket smoothing, gain-sum
+ normals + smoothstep blend at the patch nodes.  Default workload: C3
(1024^2 FFT / 4000 m, lambda 1.2, one 256 m patch on a 1024^2 grid, 16 log
buckets 0.3-6 rad/s, n_theta 2), warmed to steady state (~0.86M live
particles) by running the step itself at dt = 0.1 for 200 s of simulated
time, then timed at dt = 1/60.  Synthetic seeded inputs (no dataset exists).

metric: particles splatted per second (live particles x frames/s, whole job);
fps and ms/frame are reported beside it.  L2 is flushed (256 MiB written,
then read back)
between timed steps; steps are timed with CUDA events on the launching
stream, max over ranks.

--impl reference times the CPU oracle port of the reference algorithm
(oracle/, numpy, the reference's own single-threaded numpy path) on the host
cores, on the same config, as a bounded sample.

Multi-GPU (torchrun, one process per GPU): weak scaling -- every rank owns
one C3-geometry patch (seeded layout in the shared 4000 m tile, own Philox
stream), runs the replicated background, and every frame the composite is
exchanged at FFT resolution: each rank resamples its patch boxes of the
stitched grid, one NCCL all-gather moves them, every rank pastes them over the
background (sharding.CompositeGather).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WARM_DT = 0.1
WARM_SECONDS = 200.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--warm-seconds", type=float, default=WARM_SECONDS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--stage-frames", type=int, default=30)
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--patches", type=int, default=None, help="use the first N patches of a multi-patch scene")
    ap.add_argument("--deterministic", action="store_true", help="device.deterministic (fixed-point sums)")
    ap.add_argument("--exchange", action="store_true",
                    help="run the multi-GPU composite exchange even at N=1 (a 1-rank NCCL group): checks "
                         "and times that path on one GPU")
    return ap.parse_args()


def scene_config(name: str, rank: int, world: int, patches: int | None = None):
    """(config of this rank, Philox keys or None, scaling).  Single-patch
    scenes (C3, PR1) scale weakly: rank r owns patch r of a seeded layout of
    `world` same-size patches.  Multi-patch scenes (C2, C4, C5) scale
    strongly: the scene's patches are split into contiguous blocks
    (sharding.shard_config), each patch keeping its global Philox key."""
    from dataclasses import replace
    from paper_2511_02852_b200 import scenes
    from paper_2511_02852_b200.sharding import shard_config
    cfg = scenes.PRESETS[name]()
    if patches is not None and patches < len(cfg.patches):
        cfg = replace(cfg, patches=cfg.patches[:patches]).validate()
        tracked = {pc.track_source for pc in cfg.patches}
        if any(pc.track_source >= 0 for pc in cfg.patches):
            cfg = replace(cfg, sources=cfg.sources[:max(tracked) + 1]).validate()
    if len(cfg.patches) == 1:
        if world > 1:
            p0 = cfg.patches[0]
            org = scenes.seeded_layout(world, p0.size[0], cfg.fft_domain, seed=cfg.seed + 100)
            # one coherent scene: every rank keeps cfg.seed (the replicated
            # background is identical everywhere) and its patch draws its own
            # Philox stream, key (seed, rank) -- the patch's global id
            cfg = replace(cfg, patches=(replace(p0, origin=org[rank]),)).validate()
            return cfg, [(cfg.seed, rank)], "weak"
        return cfg, None, "weak"
    local, _, keys = shard_config(cfg, rank, world)
    return local.validate(), keys, "strong"


# ------------------------------------------------------------ clocks ----
class ClockSampler:
    def __init__(self, index: int = 0):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=10)
        self.fh.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------- reference ---
def cpu_scene_from(sim, cfg):
    """Build the CPU oracle scene in the GPU simulation's current state
    (pools in bucket-segment order, ledgers, Philox stream positions)."""
    from oracle import particles_ref, scene_ref
    sc = scene_ref.OracleScene(cfg.scene_dict(), h0=sim.fft_state.h0 if sim.fft_state is not None else None)
    sc.frame = sim.frame
    led = sim.ledger_host()
    rng_words = sim.rng.cpu().numpy().view(np.uint64)
    for k in range(sim.n_patches):
        ps = sim.pool(k)
        pos, d, a = ps.positions, ps.directions, ps.amplitudes
        sc.pools[k] = particles_ref.Pool(pos, d, a, ps.buckets.astype(np.int32), np.zeros(len(a)))
        sc.ledgers[k].acc = led["acc"][k].copy()
        sc.ledgers[k].groups = led["groups"][k].copy()
        sc.ledgers[k].e_in = led["e_in"][k].copy()
        sc.ledgers[k].e_out = led["e_out"][k].copy()
        w = rng_words[8 * k: 8 * k + 8]
        c0 = sum(int(w[2 + i]) << (64 * i) for i in range(4))
        d_idx = int(w[6])
        gen = np.random.Generator(np.random.Philox(key=[int(w[0]), int(w[1])], counter=(c0 + d_idx // 4) % (1 << 256)))
        gen.bit_generator.random_raw(d_idx % 4)
        sc.rngs[k] = gen
    return sc


def time_cpu_frames(sc, seconds: float, min_frames: int = 2, max_frames: int | None = None):
    n, t0 = 0, time.perf_counter()
    live = []
    while True:
        sc.step()
        if sc.background is not None and sc.patches:
            sc.composite()                          # the FFT-resolution composite, as the GPU step
        n += 1
        live.append(sum(len(p) for p in sc.pools))
        el = time.perf_counter() - t0
        if (el >= seconds and n >= min_frames) or (max_frames is not None and n >= max_frames):
            break
    return el / n, float(np.mean(live)), n


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import scene_ref
    cfg, _, _ = scene_config(args.config, 0, 1, args.patches)
    sc = scene_ref.OracleScene(cfg.scene_dict())
    t_warm = time.perf_counter()
    n_warm = int(round(args.warm_seconds / WARM_DT))
    for _ in range(n_warm):                       # same warm-up as the GPU arm, no synthesis
        sc.step(dt=WARM_DT, synth=False, fft=False)
    warm_s = time.perf_counter() - t_warm
    n_w = min(max(3, args.warmup), 20)            # W >= 3 untimed full frames (~1 s each at C3: capped at 20)
    for _ in range(n_w):
        sc.step()
    budget = 90.0
    frame_s, live, n = time_cpu_frames(sc, seconds=budget, min_frames=1, max_frames=max(1, args.steps))
    pps = live / frame_s
    line = {"impl": "reference", "metric": "particles splatted/s (hybrid step)", "value": pps,
            "unit": "particles/s", "n_gpus": args.gpus, "steps": n, "warmup": n_w,
            "ms_per_step": frame_s * 1e3, "fps": 1.0 / frame_s, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, steady state via the step itself)",
            "config": {"workload": f"{args.config} hybrid step", "live_particles": live, "fft_n": cfg.fft_n,
                       "patch_res": cfg.patches[0].res, "n_omega": cfg.n_omega, "n_theta": cfg.n_theta},
            "cpu_baseline": {"value": pps, "unit": "particles/s", "cores": 1, "kind": "port",
                             "sample": f"{n} full {args.config} frames after {n_warm} warm-up frames "
                                       f"(warm-up {warm_s:.1f}s); numpy single-threaded"},
            "e2e": {"value": pps, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- ours ---
def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.exchange:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    from paper_2511_02852_b200 import Simulation
    from paper_2511_02852_b200 import _native as N
    from paper_2511_02852_b200.sharding import CompositeGather

    cfg, keys, scaling = scene_config(args.config, rank, world, args.patches)
    if args.deterministic:
        from dataclasses import replace
        cfg = replace(cfg, deterministic=True).validate()
    sim = Simulation(cfg, device=dev, rng_seed_keys=keys)
    gather = None
    if world > 1 or args.exchange:
        # the composite exchange at FFT resolution: every rank's
        # patch boxes of the stitched grid, all-gathered and pasted on every rank
        gather = CompositeGather(sim.box_np.reshape(-1, 4), cfg.fft_n, world, device=dev)

    def exchange_ops():
        gather.pack(sim.composite_frame)            # this rank's patch boxes of its frame composite
        gather.gather()
        gather.paste_others(sim.composite_frame)    # the other ranks' boxes into this frame composite

    if gather is not None:
        # the frame's composite (stitched_heights, part of the step) goes through
        # the exchange: pack + NCCL all-gather + paste at the end of every frame
        # graph (one graph launch per step, no host work in between)
        exchange_ops()                              # NCCL communicator set up outside capture
        torch.cuda.synchronize()
        sim.post_frame = exchange_ops

    # steady state: the step itself at dt = 0.1
    n_warm = int(round(args.warm_seconds / WARM_DT))
    sim.run_frames(n_warm, dt=WARM_DT)
    torch.cuda.synchronize()
    sim.check()
    sim.prepare_graphs()
    for _ in range(max(3, args.warmup)):
        sim.step(stats=False)
    torch.cuda.synchronize()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_sum = torch.empty((), dtype=torch.int64, device=dev)

    def flush_l2():
        # write a 256 MiB buffer (> 126 MB L2), then read it back: the read
        # evicts the flush's own dirty lines too, so their write-back happens
        # here and not inside the next timed step
        flush.zero_()
        torch.sum(flush.view(torch.int64), dim=0, out=flush_sum)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    live_before = sim.live_particles()
    clocks = ClockSampler(local)
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for k in range(args.steps):
        flush_l2()                                 # L2 flush between timed steps (outside the events)
        starts[k].record()
        sim.step(stats=False)
        ends[k].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(np.sum(step_ms))
    step_pct = {"p50": float(np.percentile(step_ms, 50)), "p90": float(np.percentile(step_ms, 90)),
                "max": float(np.max(step_ms))}
    live_after = sim.live_particles()
    sim.check()
    if gather is not None:                         # the assembled composite of the last frame
        assert bool(torch.isfinite(sim.composite_frame).all())
    live = 0.5 * (live_before + live_after)
    if world > 1:
        t = torch.tensor([total_ms, live], dtype=torch.float64, device=dev)
        tm = t.clone()
        dist.all_reduce(tm[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        total_ms, live_all = float(tm[0]), float(t[1])
    else:
        live_all = live
    ms_per_step = total_ms / args.steps
    fps = 1e3 / ms_per_step
    value = live_all * fps

    # per-stage device times (eager frames, flushed, events on the launching stream)
    stage = {}
    for _ in range(args.stage_frames):
        flush_l2()
        for kname, v in sim.timed_frame().items():
            stage[kname] = stage.get(kname, 0.0) + v
    stage = {k: v / args.stage_frames for k, v in stage.items()}

    # e2e through the public API with host buffers, every step: H2D of the
    # frame index from pinned memory, the graph step, D2H of every blended
    # patch tile + the live counts into pinned memory.  HostFramePipe overlaps
    # frame k's host copy with frame k+1's compute (the timed region ends
    # when the last copy has landed).
    from paper_2511_02852_b200.harness import HostFramePipe
    pipe = HostFramePipe(sim)
    for _ in range(3):
        pipe.step()
    # one pinned source per step: the loop runs ahead of the device, so a
    # reused buffer could be rewritten before its H2D copy executes
    host_frames = torch.arange(sim.frame, sim.frame + args.e2e_steps, dtype=torch.int64).pin_memory()
    torch.cuda.synchronize()
    e2e_start, e2e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_start.record()
    last = 0
    for k in range(args.e2e_steps):
        sim.frame_dev.copy_(host_frames[k:k + 1], non_blocking=True)
        last = pipe.step()
    with torch.cuda.stream(pipe.copy):
        e2e_end.record(pipe.copy)
    tiles, counts = pipe.result(last)
    torch.cuda.synchronize()
    assert int(counts.sum()) == sim.live_particles() and bool(torch.isfinite(tiles).all())
    e2e_ms = e2e_start.elapsed_time(e2e_end) / args.e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    e2e_value = live_all * 1e3 / e2e_ms
    e2e_bytes = pipe.bytes_per_frame

    # roofline of the dominant particle kernel, hs_advect_resident (in-place
    # advect + cull + splat): per live particle it must read x, y, ux, uy (f64)
    # and amp (f32) = 36 B and write the new x, y = 16 B
    adv_bytes = 52.0 * live
    adv_ms = stage.get("advect", float("nan"))
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = adv_bytes / (adv_ms * 1e-3) / 1e9 if adv_ms == adv_ms and adv_ms > 0 else None
    # DRAM bytes per hs_advect_resident launch from the committed ncu launch list
    # of this workload (tools/ncu_launches.sh -> tools/traffic_json.py)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tp):
        try:
            ks = json.load(open(tp))["kernels"]
            k = next(k for k in ks if k.startswith("advect_resident_kernel"))
            traffic = ks[k]["dram_read_bytes"] + ks[k]["dram_write_bytes"]
        except (OSError, KeyError, ValueError, StopIteration):
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sc = cpu_scene_from(sim, cfg)
        frame_s, cpu_live, n_cpu = time_cpu_frames(sc, seconds=args.cpu_seconds)
        cpu = {"value": cpu_live / frame_s, "unit": "particles/s", "cores": 1, "kind": "port",
               "sample": f"{n_cpu} full {args.config} frames of the numpy oracle (reference algorithm) from the "
                         f"GPU's steady state ({cpu_live:.0f} live particles), single thread"}

    if rank == 0:
        line = {
            "metric": "particles splatted/s (hybrid step)", "value": value, "unit": "particles/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "fps": fps, "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64+f32",
            "data": "synthetic (seeded h0 + Philox streams; steady state reached by the step itself)",
            "config": {"workload": f"{args.config} hybrid step"
                                   + (" (1 patch per GPU)" if scaling == "weak" else
                                      f" ({len(cfg.patches)} of its patches on rank 0)"),
                       "live_particles": live_all,
                       "fft_n": cfg.fft_n, "fft_domain_m": cfg.fft_domain, "patch_res": cfg.patches[0].res,
                       "n_patches": len(cfg.patches) * (world if scaling == "weak" else 1),
                       "fft_cascades": list(cfg.fft_cascades), "n_sources": len(cfg.sources),
                       "n_omega": cfg.n_omega, "n_theta": cfg.n_theta, "dt": cfg.dt,
                       "warm_start": f"{n_warm} frames at dt={WARM_DT}", "l2": "flushed between timed steps (256 MiB written, then read back)",
                       "parallelism": (f"patch-sharded x{world}" if world > 1 else "single GPU"),
                       "deterministic": bool(cfg.deterministic),
                       "step": "FFT background + boundary injection + resident advect/cull/splat + per-bucket "
                               "smoothing + upsample-sum/normals/blend at the patch nodes + FFT-resolution "
                               "composite (one CUDA graph); pool compaction every %d frames" % sim.compact_period},
            "step_ms_percentiles": step_pct,
            "gpu_launches": (sim.kernel_launches_per_frame() + (1 if gather else 0)) * args.steps,
            "stages_ms": stage,
            "roofline": {"bound": "hbm", "kernel": "hs_advect_resident (in-place advect+cull+splat)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "algorithmic_bytes": adv_bytes, "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
            "e2e": {"value": e2e_value, "unit": "particles/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 8, "d2h_bytes_per_step": e2e_bytes,
                    "note": "host copy of frame k overlaps frame k+1 (HostFramePipe, pinned, depth 2)"},
            "clocks": clk,
            "wall_s_timed": wall,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
