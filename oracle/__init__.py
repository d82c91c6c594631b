"""CPU oracle for the hybrid ocean step -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference `hybridsea` algorithm
for the per-frame hybrid step (arXiv 2511.02852, reference package under
`pkg/src/hybridsea/`).  Each function cites the reference file:line it
follows.  It exists so the CUDA product path can be checked against it.

Rules (enforced by review):
  * only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its
    `cpu_baseline` leg and `--impl reference` arm) may import this package;
  * the product package `paper_2511_02852_b200` never imports it, and fails
    loudly when its CUDA library is missing instead of falling back here.

Pinning: the oracle is pinned against golden vectors produced by running the
reference package itself (`tests/golden/make_golden.py`, committed together
with its `.npz` outputs) plus the reference's own frozen known-answer
constants (`pkg/tests/test_spectrum.py:32-36,60-64`, `test_particles.py:76-84,
222-231`).  See `tests/test_oracle_golden.py`.
"""
from . import philox_ref, spectrum_ref, ocean_ref, particles_ref, synth_ref, blend_ref, scene_ref  # noqa: F401
