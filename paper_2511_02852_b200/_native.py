"""ctypes binding of the C ABI in include/hybridsea_b200.h.

The library is built in-tree (`build_lib.py`, `__graft_entry__.build()`).
There is no fallback: if the library is missing or a call fails, this module
raises.  Struct layouts mirror the header field by field; `_check_layout`
asserts the sizes the CUDA side was compiled with.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# HS_LIB selects an experiment build (tools/, build_lib.build(out=...)); default: the product library
LIB_PATH = os.environ.get("HS_LIB") or os.path.join(_PKG, "_lib", "libhybridsea_b200.so")

HS_STATUS_POOL_OVERFLOW = 1
HS_STATUS_STAGE_OVERFLOW = 2
HS_STATUS_BOX_OVERFLOW = 8
HS_MAX_BUCKETS = 32
HS_MAX_PATCHES = 256
HS_MAX_SOURCES = 1024
HS_SMOOTH_FUSED_MAX_H = 40

vp = C.c_void_p
dbl = C.c_double
i32 = C.c_int
i64 = C.c_longlong


class HsBucket(C.Structure):
    _fields_ = [("omega", dbl), ("width", dbl), ("radius", dbl), ("speed", dbl), ("s1d", dbl),
                ("spread_s", dbl), ("spread_c", dbl), ("pad", dbl)]


class HsPatch(C.Structure):
    _fields_ = [("x0", dbl), ("y0", dbl), ("x1", dbl), ("y1", dbl), ("l1", dbl), ("l2", dbl),
                ("margin", dbl), ("texel", dbl), ("pool_base", i64), ("stage_base", i64),
                ("grid_base", i64), ("pool_capacity", i32), ("stage_capacity", i32), ("res", i32),
                ("ny", i32), ("layer_base", i32), ("track", i32), ("sx0", dbl), ("sy0", dbl)]


class HsLayer(C.Structure):
    _fields_ = [("raw_off", i64), ("sm_off", i64), ("f", i32), ("H", i32), ("pad", i32), ("ncx", i32),
                ("ncy", i32), ("wx", i32), ("wy", i32), ("taps_off", i32), ("gain", C.c_float),
                ("mid_off", i32), ("raw_pitch", i32), ("group", i32), ("ticket", i32),
                ("pad2", i32)]


class HsPool(C.Structure):
    _fields_ = [("x", vp), ("y", vp), ("ux", vp), ("uy", vp), ("amp", vp), ("birth", vp)]


HS_FIXED_SPLAT_BITS = 32
HS_FIXED_ENERGY_BITS = 24
HS_FIXED_SUMSQ_BITS = 32
HS_MAX_CASCADES = 4


class HsBgTile(C.Structure):
    _fields_ = [("height", vp), ("n", i32), ("pad", i32), ("spacing", dbl)]


class HsFftArgs(C.Structure):
    _fields_ = [("n", i32), ("emit_normals", i32), ("g", dbl), ("t", dbl), ("choppiness", dbl),
                ("frame_ptr", vp), ("dt", dbl), ("spacing", dbl), ("kf", vp), ("h0", vp),
                ("twiddle", vp), ("work_a", vp), ("work_b", vp), ("height", vp), ("dx", vp),
                ("dy", vp), ("normal", vp), ("sumsq", vp), ("frame_advance", vp),
                ("omega", vp), ("fixed_point", i32)]


class HsResidentArgs(C.Structure):
    _fields_ = [("n_patches", i32), ("nb", i32), ("buckets", vp), ("patches", vp), ("dt", dbl),
                ("rho", dbl), ("g", dbl), ("pool", HsPool), ("seg_base", vp), ("seg_cap", vp),
                ("tile_map", vp), ("max_tiles", i32), ("len_in", vp), ("len_out", vp), ("live", vp),
                ("stage", HsPool), ("stage_count", vp), ("e_out", vp), ("raw_layers", vp), ("layers", vp),
                ("clamped", vp), ("status", vp), ("fixed_point", i32)]


class HsInjectArgs(C.Structure):
    _fields_ = [("n_patches", i32), ("nb", i32), ("n_theta", i32), ("buckets", vp), ("patches", vp),
                ("half_rate", vp), ("mean_dir", dbl), ("beta", dbl), ("rho", dbl), ("g", dbl),
                ("acc", vp), ("groups", vp), ("e_in", vp), ("rng", vp), ("stage", HsPool),
                ("stage_count", vp), ("scratch", vp), ("member_capacity", i32), ("status", vp),
                ("zero_words", vp), ("n_zero_words", i32), ("append", i32), ("res", HsResidentArgs),
                ("birth_t", dbl), ("birth_frame", vp), ("birth_dt", dbl)]


class HsAdvectArgs(C.Structure):
    _fields_ = [("n_patches", i32), ("nb", i32), ("buckets", vp), ("patches", vp), ("dt", dbl),
                ("rho", dbl), ("g", dbl), ("in_", HsPool), ("in_count", vp), ("stage", HsPool),
                ("stage_count", vp), ("out", HsPool), ("out_count", vp), ("dropped", HsPool),
                ("dropped_count", vp), ("e_out", vp), ("splat", i32), ("raw_layers", vp),
                ("raw_layers_len", i64), ("layers", vp), ("clamped", vp), ("tile_state", vp),
                ("max_tiles", i32), ("tile_counter", vp), ("status", vp), ("keep_words", vp),
                ("in_seg_base", vp), ("out_slack_prefix", vp), ("raw_is_clear", i32), ("fixed_point", i32)]


class HsSource(C.Structure):
    _fields_ = [("vx", dbl), ("vy", dbl), ("hull_extent", dbl), ("e_ring", dbl), ("e_wake", dbl),
                ("amp_ring", dbl), ("amp_wake", dbl), ("n_ring", i32), ("n_wake", i32), ("ring_bucket", i32),
                ("wake_bucket", i32), ("dir_off", i32), ("body", i32)]


HS_MAX_PROBES = 8


class HsBody(C.Structure):
    _fields_ = [("pos", dbl * 3), ("vel", dbl * 3), ("yaw", dbl), ("yaw_rate", dbl), ("submerged", dbl),
                ("prev_submerged", dbl), ("mean_submersion", dbl), ("mass", dbl), ("hull_extent", dbl),
                ("draft", dbl), ("drag_linear", dbl), ("drag_yaw", dbl), ("thrust_force", dbl),
                ("yaw_torque", dbl), ("displaced", dbl), ("probe_off", (dbl * 3) * HS_MAX_PROBES),
                ("probe_vol", dbl * HS_MAX_PROBES), ("n_probes", i32), ("pad", i32)]


class HsBodyArgs(C.Structure):
    _fields_ = [("n_bodies", i32), ("bodies", vp), ("dt", dbl), ("rho", dbl), ("g", dbl), ("flat", i32),
                ("bg_height", vp), ("bg_n", i32), ("bg_spacing", dbl), ("n_extra_bg", i32),
                ("extra_bg", HsBgTile * (HS_MAX_CASCADES - 1)), ("n_patches", i32), ("patches", vp),
                ("patch_height", vp), ("frame", vp)]


class HsEmitArgs(C.Structure):
    _fields_ = [("n_sources", i32), ("n_patches", i32), ("nb", i32), ("sources", vp), ("dirs", vp),
                ("pos_in", vp), ("pos_out", vp), ("patches", vp), ("buckets", vp), ("dt", dbl), ("beta", dbl),
                ("rho", dbl), ("g", dbl), ("pool", HsPool), ("seg_base", vp), ("seg_cap", vp), ("len", vp),
                ("live", vp), ("e_in", vp), ("raw_layers", vp), ("layers", vp), ("clamped", vp), ("status", vp),
                ("bodies", vp), ("n_theta", i32), ("fixed_point", i32)]


class HsLayoutArgs(C.Structure):
    _fields_ = [("n_patches", i32), ("nb", i32), ("patches", vp), ("count", vp), ("slack", vp),
                ("slack_prefix", vp), ("seg_base", vp), ("seg_cap", vp), ("len", vp), ("live", vp),
                ("tile_map", vp), ("max_tiles", i32), ("status", vp)]


class HsSplatArgs(C.Structure):
    _fields_ = [("n_patches", i32), ("nb", i32), ("patches", vp), ("pool", HsPool), ("count", vp),
                ("raw_layers", vp), ("raw_layers_len", i64), ("layers", vp), ("clamped", vp),
                ("max_count", i32)]


class HsSmoothArgs(C.Structure):
    _fields_ = [("n_layers", i32), ("layers", vp), ("taps", vp), ("raw_layers", vp),
                ("smooth_layers", vp), ("tile_info", vp), ("total_tiles", i32), ("max_H", i32),
                ("mid", vp), ("xtile_prefix", vp), ("total_xtiles", i32), ("ytile_prefix", vp),
                ("total_ytiles", i32), ("max_H_wide", i32), ("tickets", vp)]


class HsComposeArgs(C.Structure):
    _fields_ = [("n_patches", i32), ("nb", i32), ("patches", vp), ("layers", vp),
                ("smooth_layers", vp), ("tile_info", vp), ("total_tiles", i32),
                ("bg_height", vp), ("bg_normal", vp), ("bg_n", i32), ("bg_spacing", dbl),
                ("patch_height", vp), ("patch_normal", vp), ("blend_height", vp),
                ("blend_normal", vp), ("blend_mode", i32), ("interior_sumsq", vp),
                ("interior_count", vp), ("frame_advance", vp), ("n_extra_bg", i32),
                ("extra_bg", HsBgTile * (HS_MAX_CASCADES - 1)), ("fixed_point", i32), ("composite", vp)]


class HsBoxArgs(C.Structure):
    _fields_ = [("n", i32), ("spacing", dbl), ("composite", vp), ("n_local", i32), ("patches", vp), ("bw", i32),
                ("bh", i32), ("payload", vp), ("slots", i32), ("world", i32), ("rank", i32), ("status", vp)]


class HsSampleArgs(C.Structure):
    _fields_ = [("n_points", i32), ("points", vp), ("bg_height", vp), ("bg_normal", vp), ("bg_n", i32),
                ("bg_spacing", dbl), ("bg_x0", dbl), ("bg_y0", dbl), ("n_patches", i32),
                ("patches", vp), ("patch_height", vp), ("patch_normal", vp), ("out_height", vp),
                ("out_normal", vp), ("clamped_only", i32), ("n_extra_bg", i32),
                ("extra_bg", HsBgTile * (HS_MAX_CASCADES - 1)), ("from_heights", i32)]


class HsCompositeArgs(C.Structure):
    _fields_ = [("n", i32), ("spacing", dbl), ("bg_height", vp), ("bg_normal", vp), ("n_patches", i32),
                ("patches", vp), ("patch_height", vp), ("patch_normal", vp), ("box", vp),
                ("box_prefix", vp), ("total_box", i32), ("out", vp), ("n_extra_bg", i32),
                ("extra_bg", HsBgTile * (HS_MAX_CASCADES - 1))]


class HsFinishArgs(C.Structure):
    _fields_ = [("nx", i32), ("ny", i32), ("spacing", dbl), ("chop_scale", dbl), ("height", vp),
                ("normal", vp), ("disp", vp)]


class HsInitArgs(C.Structure):
    _fields_ = [("n", i32), ("spread_const", i32), ("g", dbl), ("dk", dbl), ("kf", vp), ("alpha", dbl),
                ("omega_p", dbl), ("gamma", dbl), ("sigma_low", dbl), ("sigma_high", dbl), ("spread_s", dbl),
                ("mean_direction", dbl), ("k_lo", dbl), ("k_hi", dbl), ("kb_lo", dbl), ("kb_hi", dbl),
                ("pcg_state", C.c_uint64 * 2), ("pcg_inc", C.c_uint64 * 2), ("zig_k", vp), ("zig_w", vp),
                ("zig_f", vp), ("zig_r", dbl), ("work", vp), ("xi", vp), ("h0", vp), ("h0_f32", vp),
                ("status", vp)]


ABI_STRUCTS = [HsBucket, HsPatch, HsLayer, HsPool, HsFftArgs, HsInjectArgs, HsAdvectArgs, HsSplatArgs,
               HsSmoothArgs, HsComposeArgs, HsSampleArgs, HsCompositeArgs, HsFinishArgs, HsResidentArgs,
               HsLayoutArgs, HsSource, HsEmitArgs, HsBody, HsBodyArgs, HsInitArgs, HsBoxArgs]

EXPECTED_SIZES = {HsBucket: 64, HsPatch: 128, HsLayer: 72, HsPool: 48, HsSource: 80}

# every symbol include/hybridsea_b200.h declares
EXPORTS = ["hs_abi_version", "hs_last_error", "hs_struct_size", "hs_configure_device", "hs_stream_create",
           "hs_stream_destroy", "hs_fft_evolve", "hs_inject", "hs_advect", "hs_splat",
           "hs_smooth", "hs_compose", "hs_sample", "hs_composite", "hs_finish", "hs_sumsq",
           "hs_advance_frame", "hs_periodic_normals", "hs_advect_resident", "hs_append_resident",
           "hs_resident_layout", "hs_track", "hs_emit", "hs_bodies", "hs_init_h0",
           "hs_init_workspace_bytes", "hs_fixed_to_float", "hs_clear", "hs_box_pack", "hs_box_paste",
           "hs_spectral_at", "hs_conv1d_zero"]

_lib = None


def _check_layout() -> None:
    for st, size in EXPECTED_SIZES.items():
        if C.sizeof(st) != size:
            raise RuntimeError(f"{st.__name__} is {C.sizeof(st)} bytes, C ABI expects {size}")


def lib() -> C.CDLL:
    """Load the CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"hybridsea_b200 CUDA library not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    _check_layout()
    L = C.CDLL(LIB_PATH)
    L.hs_last_error.restype = C.c_char_p
    L.hs_abi_version.restype = C.c_int
    for name in EXPORTS[3:]:
        getattr(L, name).restype = C.c_int
    L.hs_struct_size.restype = C.c_int
    L.hs_struct_size.argtypes = [C.c_int]
    for k, st in enumerate(ABI_STRUCTS):
        if L.hs_struct_size(k) != C.sizeof(st):
            raise RuntimeError(f"{st.__name__}: ctypes {C.sizeof(st)} bytes != C {L.hs_struct_size(k)}")
    L.hs_sumsq.argtypes = [vp, i64, vp, vp]
    L.hs_advance_frame.argtypes = [vp, vp]
    L.hs_periodic_normals.argtypes = [vp, vp, i32, dbl, vp]
    L.hs_fixed_to_float.argtypes = [vp, vp, i64, i32, vp]
    L.hs_clear.argtypes = [vp, i64, vp]
    L.hs_spectral_at.argtypes = [vp, vp, i32, dbl, vp, vp]
    L.hs_conv1d_zero.argtypes = [vp, vp, i64, i32, i64, vp, i32, vp]
    L.hs_stream_create.argtypes = [C.POINTER(vp), C.c_int]
    L.hs_stream_destroy.argtypes = [vp]
    L.hs_init_workspace_bytes.restype = i64
    L.hs_init_workspace_bytes.argtypes = [C.c_int]
    if L.hs_abi_version() != 1:
        raise RuntimeError("hybridsea_b200 ABI version mismatch")
    _lib = L
    return L


_configured: set = set()


def configure_device(device) -> None:
    """hs_configure_device once per device (kernel attributes and occupancy):
    must run before the first graph capture, since attribute calls inside a
    capture invalidate it."""
    import torch
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx in _configured:
        return
    with torch.cuda.device(idx):
        L = lib()
        if L.hs_configure_device() != 0:
            raise RuntimeError(f"hs_configure_device failed: {L.hs_last_error().decode(errors='replace')}")
    _configured.add(idx)


class OwnedStream:
    """A CUDA stream created by the library (hs_stream_create), exposed to
    torch as an ExternalStream and destroyed with this object."""

    def __init__(self, device, priority: int = 0):
        import torch
        dev = torch.device(device)
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        ptr = vp()
        with torch.cuda.device(idx):
            L = lib()
            if L.hs_stream_create(C.byref(ptr), int(priority)) != 0:
                raise RuntimeError(f"hs_stream_create failed: {L.hs_last_error().decode(errors='replace')}")
        self.ptr = ptr.value
        self.stream = torch.cuda.ExternalStream(self.ptr, device=torch.device("cuda", idx))

    def __del__(self):
        try:
            if self.ptr and _lib is not None:
                _lib.hs_stream_destroy(vp(self.ptr))
        except Exception:
            pass


def call(name: str, args, stream) -> None:
    """Invoke `name(&args, stream)`; raise with the library's message on error."""
    L = lib()
    rc = getattr(L, name)(C.byref(args), vp(stream))
    if rc != 0:
        raise RuntimeError(f"{name} failed ({rc}): {L.hs_last_error().decode(errors='replace')}")


def call_raw(name: str, *args) -> None:
    L = lib()
    rc = getattr(L, name)(*args)
    if rc != 0:
        raise RuntimeError(f"{name} failed ({rc}): {L.hs_last_error().decode(errors='replace')}")


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def struct_array_bytes(items) -> np.ndarray:
    """Pack a list of ctypes structs into a uint8 numpy array (for upload)."""
    if not items:
        return np.zeros(0, dtype=np.uint8)
    size = C.sizeof(items[0])
    buf = bytearray(size * len(items))
    for k, it in enumerate(items):
        buf[k * size:(k + 1) * size] = bytes(it)
    return np.frombuffer(bytes(buf), dtype=np.uint8).copy()


def pool_struct(x=None, y=None, ux=None, uy=None, amp=None, birth=None) -> HsPool:
    return HsPool(ptr(x), ptr(y), ptr(ux), ptr(uy), ptr(amp), ptr(birth))
