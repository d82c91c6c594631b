"""Clone a running B200 `Simulation` into an `OracleScene` -- TEST
INFRASTRUCTURE ONLY (used by tests/ and bench.py's CPU leg, never by the
product).

The scene-level parity tests warm a BASELINE scene to steady state on the
GPU (the pipeline itself, dt = 0.1), copy its whole state
into the CPU oracle and then step both: per-bucket pools (bucket-segment
order is the reference's stable order restricted to each bucket,
particles.py:167-178), injection ledgers (particles.py:187-202), each patch's
Philox stream position, kinematic source positions and the patches'
current (retracked) rectangles (harness.py:115-123).  The GPU state is read
through the Simulation's public accessors only.

Cloned particles get birth time CLONED (-1) in the oracle, so a test can
tell them (advected identically, bit for bit) from the ones injected or
emitted after the clone.
"""
from __future__ import annotations

import numpy as np

from . import particles_ref, scene_ref

CLONED = -1.0


def philox_generator(words: np.ndarray) -> np.random.Generator:
    """numpy Generator(Philox) positioned at a device stream state
    [key0, key1, counter0 (4 words), draw index, pad] (HsInjectArgs.rng)."""
    w = np.asarray(words).view(np.uint64)
    c0 = sum(int(w[2 + i]) << (64 * i) for i in range(4))
    d_idx = int(w[6])
    gen = np.random.Generator(np.random.Philox(key=[int(w[0]), int(w[1])],
                                               counter=(c0 + d_idx // 4) % (1 << 256)))
    gen.bit_generator.random_raw(d_idx % 4)
    return gen


def oracle_from_sim(sim, cfg) -> scene_ref.OracleScene:
    """An OracleScene in `sim`'s current state (after its last full frame).

    The oracle uses the GPU's background h0 (identical inputs, as north_star
    allows) so no second 2048^2 host init is needed."""
    h0 = None
    if sim.fft_state is not None and not cfg.fft_cascades:
        h0 = sim.fft_state.h0
        h0 = h0.cpu().numpy() if hasattr(h0, "cpu") else np.asarray(h0)
    sc = scene_ref.OracleScene(cfg.scene_dict(), h0=h0)
    sc.frame = sim.frame
    led = sim.ledger_host()
    rng_words = sim.rng.cpu().numpy().view(np.uint64)
    regions = sim.current_regions()
    for k in range(sim.n_patches):
        ps = sim.pool(k)
        a = ps.amplitudes
        sc.pools[k] = particles_ref.Pool(ps.positions, ps.directions, a, ps.buckets.astype(np.int32),
                                         np.full(len(a), CLONED))
        sc.ledgers[k].acc = led["acc"][k].copy()
        sc.ledgers[k].groups = led["groups"][k].copy()
        sc.ledgers[k].e_in = led["e_in"][k].copy()
        sc.ledgers[k].e_out = led["e_out"][k].copy()
        sc.rngs[k] = philox_generator(rng_words[8 * k: 8 * k + 8])
        r = regions[k]
        sc.patches[k] = particles_ref.Patch(float(r.origin[0]), float(r.origin[1]), r.l1, r.l2, r.margin)
    if sc.sources:
        pos = sim.source_positions()
        nb_body = sim.n_bodies
        for j, src in enumerate(sc.sources):
            src.position = pos[nb_body + j].copy()
    return sc


__all__ = ["CLONED", "oracle_from_sim", "philox_generator"]
