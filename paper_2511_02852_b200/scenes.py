"""BASELINE.json scene presets expressed in the (extended) config schema.

SURVEY.md section 8 legend; knob mapping in SURVEY App. A.  Inputs are
synthetic and seeded: h0 from numpy default_rng(seed) (as the reference's
init_fft), per-patch Philox streams key=(seed, patch), seeded non-overlapping
patch layouts.

  PR1  256^2 / 1000 m, U10 10, F 100 km, gamma 3.3, s 8; one 64 m patch on a
       256 grid; 8 log buckets 0.5-4 rad/s; n_theta 16; dt 1/60, 120 frames
  C2   512^2 / 2000 m, U10 15, s 10; 4 x 128 m patches on 512 grids (seeded
       layout); 12 equal-energy buckets; n_theta 8 (~62k live at steady
       state, BASELINE's ~65k); 300 frames; one point wake
       source per patch moving straight at 8 m/s on a seeded heading, 256
       particles per frame (128-direction Kelvin fan + troughs)
  C3   1024^2 / 4000 m, lambda 1.2; one 256 m patch on a 1024 grid; 16 log
       buckets 0.3-6 rad/s; n_theta 2 (~0.86M live at steady state)
  C4   3 summed 512^2 cascades over 4000 / 1000 / 250 m with disjoint |k|
       bands (FFT band widened to 6 rad/s), U10 20, gamma 5, s 4; 8 x 128 m
       patches on 512 grids; 16 log buckets 0.3-6 rad/s (the range is
       unspecified; C3's), n_theta 5 (~4.3M live, BASELINE's ~4M)
  C5   2048^2 / 8000 m; 64 x 192 m patches on 768 grids; 16 buckets;
       n_theta 16; one ship per patch on a seeded heading at 5-15 m/s, 1024
       Kelvin-wedge particles per frame, the patch tracking its ship
"""
from __future__ import annotations

from dataclasses import replace

import numpy as np

from .config import PatchConfig, SimConfig, SourceConfig  # noqa: F401  (re-exported for presets)


def seeded_layout(n: int, size: float, domain: float, seed: int, margin: float = 0.0) -> list:
    """`n` non-overlapping square patch origins uniform in the tile
    (rejection sampling; overlap rule of coupling.py:85-92)."""
    rng = np.random.default_rng(seed)
    out: list = []
    tries = 0
    while len(out) < n:
        tries += 1
        if tries > 100000:
            raise RuntimeError("could not place patches without overlap")
        o = rng.uniform(margin, domain - size - margin, size=2)
        if all(abs(o[0] - p[0]) >= size or abs(o[1] - p[1]) >= size for p in out):
            out.append((float(o[0]), float(o[1])))
    return out


def pr1(**kw) -> SimConfig:
    cfg = SimConfig(u10=10.0, fetch=100000.0, g=9.81, gamma=3.3, spread_s=8.0, n_omega=8, n_theta=16,
                    bucket_spacing="log", omega_lo=0.5, omega_hi=4.0, dt=1.0 / 60.0, frames=120, seed=0,
                    fft_n=256, fft_domain=1000.0, fft_choppiness=1.0,
                    patches=(PatchConfig(origin=(468.0, 468.0), size=(64.0, 64.0), res=256, margin=8.0),),
                    write_frames=False)
    return replace(cfg, **kw).validate()


def wake_sources(origins, size: float, speeds, count: int, hull: float, seed: int, start_back: float):
    """One kinematic wake source per patch on a seeded heading, starting
    `start_back` metres behind the patch centre so it crosses the middle."""
    rng = np.random.default_rng(seed)
    out = []
    for o, v in zip(origins, speeds):
        th = float(rng.uniform(0.0, 2.0 * np.pi))
        c = (o[0] + 0.5 * size, o[1] + 0.5 * size)
        p = (c[0] - start_back * np.cos(th), c[1] - start_back * np.sin(th))
        out.append(SourceConfig(position=p, velocity=(v * np.cos(th), v * np.sin(th), 0.0), hull_extent=hull,
                                volume_rate=0.05, submersion=0.5, wake_count=count))
    return tuple(out)


def c2(**kw) -> SimConfig:
    org = seeded_layout(4, 128.0, 2000.0, seed=2)
    src = wake_sources(org, 128.0, [8.0] * 4, count=128, hull=1.0, seed=22, start_back=20.0)
    cfg = SimConfig(u10=15.0, fetch=100000.0, spread_s=10.0, n_omega=12, n_theta=8, dt=1.0 / 60.0, frames=300,
                    seed=2, fft_n=512, fft_domain=2000.0, fft_choppiness=1.0,
                    patches=tuple(PatchConfig(origin=o, size=(128.0, 128.0), res=512, margin=10.0) for o in org),
                    sources=src, write_frames=False)
    return replace(cfg, **kw).validate()


def c3(**kw) -> SimConfig:
    cfg = SimConfig(u10=10.0, fetch=100000.0, n_omega=16, n_theta=2, bucket_spacing="log", omega_lo=0.3,
                    omega_hi=6.0, dt=1.0 / 60.0, frames=600, seed=3, fft_n=1024, fft_domain=4000.0,
                    fft_choppiness=1.2,
                    patches=(PatchConfig(origin=(1872.0, 1872.0), size=(256.0, 256.0), res=1024, margin=10.0),),
                    write_frames=False)
    return replace(cfg, **kw).validate()


def c4(**kw) -> SimConfig:
    """3 summed cascades 4000 / 1000 / 250 m (disjoint |k| bands, config.cascade_bands)
    over a band widened to 6 rad/s so every tile carries energy."""
    org = seeded_layout(8, 128.0, 4000.0, seed=4)
    cfg = SimConfig(u10=20.0, fetch=100000.0, gamma=5.0, spread_s=4.0, n_omega=16, n_theta=5,
                    bucket_spacing="log", omega_lo=0.3, omega_hi=6.0, dt=1.0 / 60.0, frames=600, seed=4, fft_n=512, fft_domain=4000.0, fft_choppiness=1.0,
                    fft_cascades=(4000.0, 1000.0, 250.0), fft_band_hi=6.0,
                    patches=tuple(PatchConfig(origin=o, size=(128.0, 128.0), res=512, margin=10.0) for o in org),
                    write_frames=False)
    return replace(cfg, **kw).validate()


def c5(n_patches: int = 64, **kw) -> SimConfig:
    """`n_patches` < 64 builds the first ships of the fleet (one GPU's share)."""
    org = seeded_layout(64, 192.0, 8000.0, seed=5)[:n_patches]
    speeds = np.random.default_rng(55).uniform(5.0, 15.0, size=64)[:n_patches]
    src = wake_sources(org, 192.0, speeds, count=512, hull=10.0, seed=56, start_back=0.0)
    cfg = SimConfig(u10=10.0, fetch=100000.0, n_omega=16, n_theta=16, dt=1.0 / 60.0, frames=600, seed=5,
                    fft_n=2048, fft_domain=8000.0, fft_choppiness=1.0,
                    patches=tuple(PatchConfig(origin=o, size=(192.0, 192.0), res=768, margin=10.0, track_source=k)
                                  for k, o in enumerate(org)),
                    sources=src, write_frames=False)
    return replace(cfg, **kw).validate()


PRESETS = {"PR1": pr1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}
