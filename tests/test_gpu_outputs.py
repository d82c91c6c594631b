"""Headless run outputs and the energy ledger on the B200:
stats.csv / timings.csv / frame_*.raw + .meta as the reference's `run`
(harness.py:274-329), the ledger balance of test_harness.py:113-136 with
kinematic emitters booking through the same ledger, and rerun determinism of
every integer / serially-accumulated statistic."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _small_cfg(**kw):
    from dataclasses import replace
    from paper_2511_02852_b200 import PatchConfig, SimConfig, SourceConfig
    cfg = SimConfig(fft_n=64, fft_domain=500.0, dt=0.05, frames=6, n_omega=8, n_theta=8, seed=7,
                    patches=(PatchConfig(origin=(200.0, 200.0), size=(100.0, 100.0), res=65, margin=10.0),),
                    sources=(SourceConfig(position=(250.0, 250.0), velocity=(2.0, 1.0, 0.3), hull_extent=1.5,
                                          volume_rate=0.01, submersion=0.5),),
                    write_frames=True, output_stride=2)
    return replace(cfg, **kw).validate()


def test_run_writes_reference_layout(cuda, tmp_path):
    from paper_2511_02852_b200 import run, stats_header
    cfg = _small_cfg()
    stats = run(cfg, str(tmp_path))
    assert len(stats) == cfg.frames
    lines = (tmp_path / "stats.csv").read_text().splitlines()
    assert lines[0] == stats_header(cfg)
    assert len(lines) == cfg.frames + 1
    for k, (line, s) in enumerate(zip(lines[1:], stats)):
        f = line.split(",")
        assert int(f[0]) == k and float(f[1]) == s.t
        assert int(f[2]) == int(s.particle_counts.sum())
        assert [int(x) for x in f[3:3 + 8]] == [int(c) for c in s.particle_counts]
    frames = sorted(tmp_path.glob("frame_*.raw"))
    assert [p.name for p in frames] == [f"frame_{k:06d}.raw" for k in range(0, cfg.frames, 2)]
    for p in frames:
        assert p.stat().st_size == cfg.fft_n * cfg.fft_n * 4
        meta = p.with_suffix(".meta").read_text()
        assert meta.startswith(f"res={cfg.fft_n}x{cfg.fft_n} spacing={cfg.fft_domain / cfg.fft_n!r} origin=0.0,0.0 t=")
        assert np.isfinite(np.fromfile(p, dtype="<f4")).all()
    t = (tmp_path / "timings.csv").read_text().splitlines()
    assert len(t) == cfg.frames + 1 and t[0].endswith(",total_ms")
    assert (tmp_path / "config.echo").exists()


def test_energy_ledger_balances_with_emitters(cuda):
    """injected - despawned == resident crest energy per bucket, emissions
    included (test_harness.py:113-136; 250 frames at dt = 0.1)."""
    from paper_2511_02852_b200 import Simulation, particle_energy
    cfg = _small_cfg(dt=0.1, frames=0, write_frames=False)
    sim = Simulation(cfg, device=cuda)
    for _ in range(250):
        sim.step(stats=False)
    sim.check()
    ps = sim.pool(0)
    led = sim.ledger_host()
    resident = np.zeros(8)
    for b in range(8):
        amp = ps.segment(b)["amp"]
        crest = amp > 0
        resident[b] = np.sum(particle_energy(cfg.rho, cfg.g, amp[crest], sim.table.buckets[b].radius))
    inj, des = led["e_in"][0], led["e_out"][0]
    drift = inj - des - resident
    assert inj.sum() > 0 and des.sum() > 0
    assert np.all(np.abs(drift) <= 0.05 * np.maximum(inj, 1e-12)), drift / np.maximum(inj, 1e-12)


def test_rerun_is_deterministic_where_serial(cuda):
    """Two runs of one config: per-bucket counts, the injection ledger and
    every pool position are bit-identical (integer and fixed-order fp64
    work); heights agree to fp32 atomic-order noise (splat reductions)."""
    from paper_2511_02852_b200 import Simulation
    cfg = _small_cfg(write_frames=False)
    sims = [Simulation(cfg, device=cuda) for _ in range(2)]
    for s in sims:
        for _ in range(40):
            s.step(stats=False)
    a, b = sims
    np.testing.assert_array_equal(a.counts_host(), b.counts_host())
    np.testing.assert_array_equal(a.ledger_host()["e_in"], b.ledger_host()["e_in"])
    pa, pb = a.pool(0), b.pool(0)
    for k in range(8):
        np.testing.assert_array_equal(pa.segment(k)["pos"], pb.segment(k)["pos"])
    ha, hb = a.patch_heights(0).cpu().numpy(), b.patch_heights(0).cpu().numpy()
    assert np.abs(ha - hb).max() <= 1e-6 * max(1e-6, np.abs(ha).max())


@pytest.mark.parametrize("scene", ["c2", "c4"])
def test_frame_composite_equals_stitched_heights(cuda, scene):
    """Every frame ends with the FFT-resolution composite (the background copy
    on the FFT branch, the patch nodes blended in by hs_compose from its staged
    tiles): it equals the on-demand stitched_heights (hs_composite,
    harness.py:219-241) to fp32 rounding."""
    from paper_2511_02852_b200 import Simulation, scenes
    cfg = getattr(scenes, scene)(frames=6)
    sim = Simulation(cfg, device=cuda)
    for _ in range(cfg.frames):
        sim.step(stats=False)
    got = sim.composite_frame.clone().cpu().numpy()
    want = sim.stitched_heights().cpu().numpy()
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-6 * scale
    assert np.mean(got == want) > 0.999


def test_host_frame_pipe_delivers_every_frame(cuda):
    """HostFramePipe (bench.py's e2e path): the host copy of each frame's
    blended tiles and live counts, taken from the frame's own per-parity
    buffers while the next frame runs, equals what a fully synchronised run
    of the same deterministic scene holds after that frame (both length
    parities, nine frames)."""
    import torch
    from paper_2511_02852_b200 import PatchConfig, Simulation, SimConfig
    from paper_2511_02852_b200.harness import HostFramePipe
    cfg = SimConfig(fft_n=128, dt=0.05, frames=10, n_omega=8, n_theta=8,
                    patches=(PatchConfig(origin=(200.0, 200.0), size=(100.0, 100.0), res=129, margin=10.0),),
                    write_frames=False, deterministic=True).validate()
    ref = Simulation(cfg, device=cuda)
    want = []
    for _ in range(9):
        ref.step(stats=False)
        torch.cuda.synchronize()
        want.append((ref.blend_h.cpu().clone(), ref.live.cpu().clone()))
    sim = Simulation(cfg, device=cuda)
    pipe = HostFramePipe(sim)
    got, slots = [], []
    for k in range(9):
        slots.append(pipe.step())
        if k >= 1:                                   # read frame k - 1 while frame k runs
            tiles, counts = pipe.result(slots[k - 1])
            got.append((tiles[: pipe.n].clone(), counts.clone()))
    tiles, counts = pipe.result(slots[-1])
    got.append((tiles[: pipe.n].clone(), counts.clone()))
    assert len(got) == len(want)
    for k, ((gt, gc), (wt, wc)) in enumerate(zip(got, want)):
        assert torch.equal(gc, wc), f"frame {k}: live counts differ"
        assert torch.equal(gt, wt[: pipe.n]), f"frame {k}: blended tiles differ"
