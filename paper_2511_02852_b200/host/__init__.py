"""numpy-in / numpy-out face of the package: the reference `hybridsea` API
(`pkg/src/hybridsea/__init__.py:8-59`) with the reference's return types.

The device API (`paper_2511_02852_b200`) hands back fp32 torch tensors on the
GPU so a caller can chain steps without host copies.  A user switching from
the reference imports this instead:

    import paper_2511_02852_b200.host as hybridsea

Every call still runs on the B200 (the same kernels); this layer only moves
inputs to the device and results back to numpy (HeightField arrays, sampler
and synthesis outputs, stitched grids).  Submodules mirror the reference's:
`host.fft_background`, `host.patch_synthesis`, `host.coupling`,
`host.harness`; spectrum, particles, config, errors and interaction are the
package's own modules (their results are host values already).
"""
from ..config import BodyConfig, PatchConfig, SimConfig, load_config, parse_config  # noqa: F401
from ..errors import CapacityError, ConfigError, NumericError  # noqa: F401
from ..particles import (InjectionLedger, ParticleSet, PatchRegion, WaveParticle, advect,  # noqa: F401
                         groups_per_step, inject)
from ..spectrum import (BucketTable, DirectionalSpectrum, FrequencyBucket, SpectrumParams,  # noqa: F401
                        band_energy, build_buckets, derive_params, evaluate_1d, evaluate_2d, evaluate_dir)
from .coupling import BlendMask, PatchSurface, SurfaceSampler, build_mask, query_surface  # noqa: F401
from .fft_background import FftState, HeightField, evolve_and_synthesize, init_fft  # noqa: F401
from .harness import FrameStats, Simulation, bench_table, benchmark, run, trend_matrix  # noqa: F401
from .patch_synthesis import (LayerStack, SmoothingKernel, accumulate, build_kernels,  # noqa: F401
                              finish_field, plan_layers, smooth_and_sum, synthesize)

from .. import config, errors, interaction, particles, spectrum  # noqa: F401,E402  (hybridsea.<module>)
from . import coupling, fft_background, harness, patch_synthesis  # noqa: F401,E402

__version__ = "0.1.0"
