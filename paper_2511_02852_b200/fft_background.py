"""Global periodic FFT height field on the B200.

Mirror of `hybridsea.fft_background` (`pkg/src/hybridsea/fft_background.py`).
`init_fft` forms h0 on the GPU (`hs_init_h0`, csrc/init.cu) from the same
PCG64 stream numpy's default_rng(seed) draws, so h0 matches the reference's
to ~1e-14 relative (host numpy formation with `on_device=False`); every
per-frame operation -- `evolve_and_synthesize`, `sample_periodic` -- is a CUDA kernel
from libhybridsea_b200 (csrc/fft.cu, csrc/synth.cu).  Outputs are fp32
device tensors.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _native as N
from ._layout import stream_ptr
from .errors import ConfigError, NumericError
from .normal_draws import pcg64_seed_state, ziggurat_r, ziggurat_tables
from .spectrum import DirectionalSpectrum, directional_density


def _device(device) -> torch.device:
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True, eq=False)
class FftState:
    """Spectral state of the background tile (fft_background.py:30-47).

    `h0` is kept on the host in complex128 (reference semantics) and on the
    device as interleaved complex64 (`h0_dev`).  conj(h0(-k)) is gathered by
    the kernel itself, so `h0_mirror_conj` is derived, not stored.
    """
    n: int
    domain_size: float
    g: float
    rng_seed: int
    choppiness: float
    h0: np.ndarray
    device: torch.device = field(default=None)
    h0_dev: torch.Tensor = field(default=None, repr=False)
    kf_dev: torch.Tensor = field(default=None, repr=False)
    twiddle_dev: torch.Tensor = field(default=None, repr=False)
    omega_dev: torch.Tensor = field(default=None, repr=False)

    @property
    def spacing(self) -> float:
        return self.domain_size / self.n

    @property
    def kf(self) -> np.ndarray:
        return 2.0 * math.pi * np.fft.fftfreq(self.n, d=self.domain_size / self.n)

    @property
    def kx(self) -> np.ndarray:
        return np.meshgrid(self.kf, self.kf, indexing="ij")[0]

    @property
    def ky(self) -> np.ndarray:
        return np.meshgrid(self.kf, self.kf, indexing="ij")[1]

    @property
    def omega(self) -> np.ndarray:
        return np.sqrt(self.g * np.hypot(self.kx, self.ky))



def _h0_get(self) -> np.ndarray:
    """Host complex128 h0; a device-initialised state downloads it on first use."""
    h = self.__dict__.get("_h0")
    if h is None and self.__dict__.get("_h0_dev64") is not None:
        h = self.__dict__["_h0_dev64"].cpu().numpy().view(np.complex128)[..., 0]
        self.__dict__["_h0"] = h
        self.__dict__["_h0_dev64"] = None
    return h


def _h0_set(self, value) -> None:
    self.__dict__["_h0"] = value
    if value is not None and self.__dict__.get("h0_dev") is not None:
        # an h0 injected into an uploaded state (the reference tests'
        # object.__setattr__ precedent, test_fft_background.py:121-127) reaches the device
        h = np.asarray(value)
        dev = np.stack([h.real, h.imag], axis=-1).astype(np.float32)
        self.__dict__["h0_dev"].copy_(torch.from_numpy(np.ascontiguousarray(dev)))


def _mirror_get(self) -> np.ndarray:
    idx = (-np.arange(self.n)) % self.n
    return np.conj(self.h0[np.ix_(idx, idx)])


def _mirror_set(self, value) -> None:
    """The kernels gather conj(h0(-k)) from h0 itself: an explicit mirror must
    be that array (it is, whenever it was formed from the same h0)."""
    if not np.array_equal(np.asarray(value), _mirror_get(self)):
        raise ValueError("h0_mirror_conj must equal conj(h0[-k]) of the state's h0 (derived on the device)")


FftState.h0 = property(_h0_get, _h0_set)   # the dataclass __init__ / replace() go through the setter
FftState.h0_mirror_conj = property(_mirror_get, _mirror_set)


def _upload(state: FftState, device, h0_dev=None, kf_dev=None) -> FftState:
    dev = _device(device)
    n = state.n
    if h0_dev is None:
        h0 = np.stack([state.h0.real, state.h0.imag], axis=-1).astype(np.float32)
        h0_dev = torch.from_numpy(np.ascontiguousarray(h0)).to(dev)
    k = np.arange(n)
    tw = np.stack([np.cos(2.0 * math.pi * k / n), np.sin(2.0 * math.pi * k / n)], -1).astype(np.float32)
    object.__setattr__(state, "device", dev)
    object.__setattr__(state, "h0_dev", h0_dev)
    object.__setattr__(state, "kf_dev", kf_dev if kf_dev is not None else torch.from_numpy(state.kf.copy()).to(dev))
    object.__setattr__(state, "twiddle_dev", torch.from_numpy(np.ascontiguousarray(tw)).to(dev))
    # dispersion on the (|i|, |j|) quarter grid, the reference's own expression
    # (fft_background.py:40-47); the kernel mirrors it over the four quadrants
    kq = state.kf[: n // 2 + 1]
    om = np.sqrt(state.g * np.hypot(kq[:, None], kq[None, :]))
    object.__setattr__(state, "omega_dev", torch.from_numpy(np.ascontiguousarray(om)).to(dev))
    return state


@dataclass(eq=False)
class HeightField:
    """Elevation, horizontal displacement and unit normals on a grid
    (fft_background.py:50-74).  Arrays are torch tensors (fp32, on the GPU
    for fields produced here); index [i, j] sits at origin + (i, j) spacing."""
    resolution: int
    origin: np.ndarray
    spacing: float
    height: torch.Tensor
    displacement: torch.Tensor
    normal: torch.Tensor
    periodic: bool = False

    def validate(self) -> None:
        """Finite values and unit normals (fft_background.py:63-74); device or numpy arrays."""
        arrs = [torch.as_tensor(a) for a in (self.height, self.displacement, self.normal)]
        if not all(bool(torch.isfinite(a).all()) for a in arrs):
            raise ValueError("height field contains non-finite values")
        norms = torch.linalg.vector_norm(arrs[2].double(), dim=-1)
        if not bool(torch.allclose(norms, torch.ones_like(norms), atol=1e-6)):
            raise ValueError("normals are not unit length")

    def to_numpy(self) -> dict:
        return {"height": self.height.double().cpu().numpy(),
                "displacement": self.displacement.double().cpu().numpy(),
                "normal": self.normal.double().cpu().numpy()}


def resolved_band(spectrum: DirectionalSpectrum, n: int, domain_size: float,
                  band: tuple | None = None) -> tuple[float, float]:
    """Sampled band clipped to the fundamental and the inscribed Nyquist
    circle (fft_background.py:90-99); `band` overrides [0.5, 2.5] omega_p."""
    g = spectrum.params.g
    lo, hi = spectrum.params.band
    if band is not None:
        lo = band[0] if band[0] is not None else lo
        hi = band[1] if band[1] is not None else hi
    w_min = math.sqrt(g * 2.0 * math.pi / domain_size)
    w_max = math.sqrt(g * math.pi * n / domain_size)
    return max(lo, w_min), min(hi, w_max)


def init_fft(spectrum: DirectionalSpectrum, n: int, domain_size: float, seed: int,
             choppiness: float = 1.0, *, band: tuple | None = None, kband: tuple | None = None,
             device=None, on_device: bool | None = None) -> FftState:
    """Initial complex amplitudes, variance-matched to the directional
    spectrum (fft_background.py:102-146).  `kband` = (k_lo, k_hi) keeps
    k_lo <= |k| < k_hi only (one tile of a summed-cascade background,
    config.cascade_bands).

    On a CUDA device (the default there) `hs_init_h0` forms h0 on the GPU from
    default_rng(seed)'s own PCG64 stream (normal_draws.py): the draws equal
    the reference's to ~1e-14 relative.  `on_device=False` keeps the host
    fp64 numpy formation (the reference's exact arithmetic)."""
    if n < 2 or (n & (n - 1)) != 0:
        raise ConfigError(f"fft grid size must be a power of two >= 2, got {n}")
    if domain_size <= 0:
        raise ConfigError(f"fft domain_size must be positive, got {domain_size}")
    if n < 4:
        raise ConfigError("the B200 FFT path needs fft.n >= 4")
    p = spectrum.params
    g = p.g
    dev = _device(device)
    if on_device is None:
        on_device = dev.type == "cuda"
    w_lo, w_hi = resolved_band(spectrum, n, domain_size, band)
    k_lo, k_hi = w_lo ** 2 / g * (1.0 - 1e-12), w_hi ** 2 / g * (1.0 + 1e-12)
    if on_device:
        return _init_on_device(spectrum, n, domain_size, seed, choppiness, k_lo, k_hi, kband, dev)
    kf = 2.0 * math.pi * np.fft.fftfreq(n, d=domain_size / n)
    kx, ky = np.meshgrid(kf, kf, indexing="ij")
    kmag = np.hypot(kx, ky)
    dk = 2.0 * math.pi / domain_size
    live = (kmag >= k_lo) & (kmag <= k_hi)
    live[0, 0] = False
    if kband is not None:
        live &= (kmag >= kband[0]) & (kmag < kband[1])
    kl = kmag[live]
    om = np.sqrt(g * kl)
    theta = np.arctan2(ky[live], kx[live]) - spectrum.mean_direction
    var = np.zeros((n, n))
    var[live] = directional_density(p, om, theta) * (g / (2.0 * om)) / kl * dk * dk / 2.0
    xi = np.random.default_rng(seed).standard_normal((n, n, 2))
    h0 = np.sqrt(var / 2.0) * (xi[..., 0] + 1j * xi[..., 1])
    h0[~live] = 0.0
    st = FftState(n=n, domain_size=domain_size, g=g, rng_seed=seed, choppiness=choppiness, h0=h0)
    return _upload(st, dev)


_ZIG_DEV: dict = {}


def _zig_tables(dev: torch.device):
    key = str(dev)
    if key not in _ZIG_DEV:
        k, w, f = ziggurat_tables()
        _ZIG_DEV[key] = (torch.from_numpy(k.view(np.int64).copy()).to(dev), torch.from_numpy(w.copy()).to(dev),
                         torch.from_numpy(f.copy()).to(dev))
    return _ZIG_DEV[key]


def _init_on_device(spectrum, n, domain_size, seed, choppiness, k_lo, k_hi, kband, dev,
                    xi_out: torch.Tensor | None = None) -> FftState:
    """hs_init_h0: draws, band mask and variance on the GPU (fp64); the host
    keeps a complex128 mirror of the result for the reference API.
    `xi_out` (float64, n*n*2, test hook) receives the Gaussian draws."""
    p = spectrum.params
    st = FftState(n=n, domain_size=domain_size, g=p.g, rng_seed=seed, choppiness=choppiness, h0=None)
    kf = torch.from_numpy(st.kf.copy()).to(dev)
    zk, zw, zf = _zig_tables(dev)
    L = N.lib()
    work = torch.empty(int(L.hs_init_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    h0 = torch.empty((n, n, 2), dtype=torch.float64, device=dev)
    h0_f32 = torch.empty((n, n, 2), dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    s, inc = pcg64_seed_state(seed)
    m64 = (1 << 64) - 1
    a = N.HsInitArgs(n=n, spread_const=int(p.spread_s is not None), g=p.g, dk=2.0 * math.pi / domain_size,
                     kf=N.ptr(kf), alpha=p.alpha, omega_p=p.omega_p, gamma=p.gamma, sigma_low=p.sigma_low,
                     sigma_high=p.sigma_high, spread_s=float(p.spread_s or 0.0),
                     mean_direction=float(spectrum.mean_direction), k_lo=k_lo, k_hi=k_hi,
                     kb_lo=float(kband[0]) if kband is not None else 0.0,
                     kb_hi=float(kband[1]) if kband is not None else 0.0,
                     zig_k=N.ptr(zk), zig_w=N.ptr(zw), zig_f=N.ptr(zf), zig_r=ziggurat_r(), work=N.ptr(work),
                     xi=N.ptr(xi_out), h0=N.ptr(h0), h0_f32=N.ptr(h0_f32), status=N.ptr(status))
    a.pcg_state[0], a.pcg_state[1] = s >> 64, s & m64
    a.pcg_inc[0], a.pcg_inc[1] = inc >> 64, inc & m64
    with torch.cuda.device(dev):
        N.call("hs_init_h0", a, torch.cuda.current_stream(dev).cuda_stream)
        code = int(status.item())
    if code:
        raise NumericError(f"hs_init_h0: status {code} (1: ziggurat run past the chunk window, "
                           "2: raw stream shorter than 2 n^2 draws)")
    st.__dict__["_h0_dev64"] = h0                # host mirror formed lazily (FftState.h0)
    return _upload(st, dev, h0_dev=h0_f32.view(n * n * 2).view(n, n, 2), kf_dev=kf)


def device_draws(spectrum: DirectionalSpectrum, n: int, domain_size: float, seed: int, device=None) -> torch.Tensor:
    """The (n, n, 2) Gaussian draws `hs_init_h0` forms for `seed` (test hook:
    equals default_rng(seed).standard_normal((n, n, 2)) to ~1e-14)."""
    dev = _device(device)
    xi = torch.empty((n, n, 2), dtype=torch.float64, device=dev)
    w_lo, w_hi = resolved_band(spectrum, n, domain_size)
    _init_on_device(spectrum, n, domain_size, seed, 1.0, w_lo ** 2 / spectrum.params.g * (1.0 - 1e-12),
                    w_hi ** 2 / spectrum.params.g * (1.0 + 1e-12), None, dev, xi_out=xi)
    return xi


def with_h0(state: FftState, h0: np.ndarray) -> FftState:
    """Copy of the state with custom amplitudes (test hook; the reference
    tests set h0 directly, test_fft_background.py:121-127)."""
    st = replace(state, h0=np.asarray(h0, dtype=complex))
    return _upload(st, state.device)


def zeroed(state: FftState) -> FftState:
    return with_h0(state, np.zeros_like(state.h0))


def spectral_at(state: FftState, t: float) -> np.ndarray:
    """Evolved Hermitian spectrum at time t (fft_background.py:155-159):
    h0 e^{-i w t} + conj(h0(-k)) e^{+i w t}, in fp64 on the device (hs_spectral_at;
    inside the frame this rotation is fused into the row transform)."""
    dev = state.device or _device(None)
    h0 = torch.from_numpy(np.ascontiguousarray(np.asarray(state.h0, dtype=np.complex128)).view(np.float64)).to(dev)
    om = state.omega_dev if state.omega_dev is not None else torch.from_numpy(
        np.ascontiguousarray(state.omega[: state.n // 2 + 1, : state.n // 2 + 1])).to(dev)
    out = torch.empty_like(h0)
    N.call_raw("hs_spectral_at", N.vp(N.ptr(h0)), N.vp(N.ptr(om)), N.i32(state.n), N.dbl(float(t)),
               N.vp(N.ptr(out)), N.vp(stream_ptr()))
    return out.cpu().numpy().view(np.complex128).reshape(state.n, state.n)


class FftWorkspace:
    """Scratch + outputs for one background transform (reused across calls)."""

    def __init__(self, n: int, device, normals: bool = True):
        self.n = n
        self.work_a = torch.empty((n, n, 2), dtype=torch.float32, device=device)
        self.work_b = torch.empty((n // 2 + 1, n, 2), dtype=torch.float32, device=device)
        self.height = torch.empty((n, n), dtype=torch.float32, device=device)
        self.disp = torch.empty((2, n, n), dtype=torch.float32, device=device)
        self.normal = torch.empty((n, n, 3), dtype=torch.float32, device=device) if normals else None
        self.sumsq = torch.zeros(1, dtype=torch.float64, device=device)

    def field(self, state: FftState) -> HeightField:
        nrm = self.normal
        return HeightField(resolution=state.n, origin=np.zeros(2), spacing=state.spacing, height=self.height,
                           displacement=self.disp.permute(1, 2, 0), normal=nrm, periodic=True)


def fft_args(state: FftState, ws: FftWorkspace, t: float = 0.0, frame_ptr=None, dt: float = 0.0) -> N.HsFftArgs:
    return N.HsFftArgs(n=state.n, emit_normals=int(ws.normal is not None), g=state.g, t=float(t),
                       choppiness=float(state.choppiness), frame_ptr=N.ptr(frame_ptr), dt=float(dt),
                       spacing=state.spacing, kf=N.ptr(state.kf_dev), h0=N.ptr(state.h0_dev),
                       twiddle=N.ptr(state.twiddle_dev), work_a=N.ptr(ws.work_a), work_b=N.ptr(ws.work_b),
                       height=N.ptr(ws.height), dx=N.ptr(ws.disp[0]), dy=N.ptr(ws.disp[1]),
                       normal=N.ptr(ws.normal), sumsq=N.ptr(ws.sumsq), omega=N.ptr(state.omega_dev))


def evolve_and_synthesize(state: FftState, t: float, *, normals: bool = True,
                          workspace: FftWorkspace | None = None) -> HeightField:
    """Height field of the background tile at time t (fft_background.py:181-208).

    One CUDA call: dispersion rotation e^{-i w t} with the mirrored
    conjugate, inverse 2-D FFT to height + choppy displacement, periodic
    central-difference normals.  Returns fresh fp32 device tensors unless a
    workspace is given (then its buffers are overwritten)."""
    ws = workspace if workspace is not None else FftWorkspace(state.n, state.device, normals)
    N.call("hs_fft_evolve", fft_args(state, ws, t=t), stream_ptr())
    return ws.field(state)


def sample_periodic(field: HeightField, points) -> tuple[torch.Tensor, torch.Tensor]:
    """Bilinear height and renormalised normal at world points with
    wrap-around (fft_background.py:222-249); points (..., 2)."""
    dev = field.height.device
    pts = torch.as_tensor(np.asarray(points, dtype=np.float64) if not torch.is_tensor(points) else points,
                          dtype=torch.float64, device=dev)
    shape = pts.shape[:-1]
    flat = pts.reshape(-1, 2).contiguous()
    out_h = torch.empty(flat.shape[0], dtype=torch.float32, device=dev)
    out_n = torch.empty((flat.shape[0], 3), dtype=torch.float32, device=dev)
    nrm = field.normal.contiguous() if field.normal is not None else None
    args = N.HsSampleArgs(n_points=flat.shape[0], points=N.ptr(flat), bg_height=N.ptr(field.height.contiguous()),
                          bg_normal=N.ptr(nrm), bg_n=field.resolution, bg_spacing=field.spacing,
                          bg_x0=float(field.origin[0]), bg_y0=float(field.origin[1]), n_patches=0, patches=0,
                          patch_height=0, patch_normal=0, out_height=N.ptr(out_h), out_normal=N.ptr(out_n),
                          clamped_only=0)
    N.call("hs_sample", args, stream_ptr())
    return out_h.reshape(shape), out_n.reshape(shape + (3,))


def max_imag_residue(state: FftState, t: float) -> float:
    """Reference diagnostic (fft_background.py:223-231); the B200 transform
    produces real outputs by construction, so report the Hermitian defect of
    the rotated spectrum instead (host fp64)."""
    phase = state.omega * t
    rot = np.cos(phase) - 1j * np.sin(phase)
    hh = state.h0 * rot + state.h0_mirror_conj * np.conj(rot)
    idx = (-np.arange(state.n)) % state.n
    defect = np.abs(hh - np.conj(hh[np.ix_(idx, idx)])).max()
    peak = np.abs(hh).max()
    return 0.0 if peak == 0 else float(defect / peak)
