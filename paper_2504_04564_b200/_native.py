"""ctypes binding of libsvdbgpu.so (include/svdbgpu.h). Fails loudly when the library is missing:
there is no CPU fallback anywhere in the product path."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsvdbgpu.so")


class TF(C.Structure):
    _fields_ = [("domain_lo", C.c_double), ("domain_hi", C.c_double), ("density_scale", C.c_double),
                ("n_entries", C.c_int32), ("rgba", C.POINTER(C.c_float))]


class Camera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("look_at", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_y_deg", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


class Settings(C.Structure):
    _fields_ = [("spp", C.c_int32), ("max_bounces", C.c_int32), ("rr_start_bounce", C.c_int32),
                ("seed", C.c_uint64), ("mode", C.c_int32), ("iso_value", C.c_double),
                ("ambient", C.c_float * 3), ("background", C.c_float * 3), ("ea_step", C.c_double),
                ("ea_min_transmittance", C.c_double), ("tile_rank", C.c_int32),
                ("tile_nranks", C.c_int32), ("kernel", C.c_int32), ("majorant_cell", C.c_int32),
                ("precision", C.c_int32), ("hdda", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("paths", C.c_uint64), ("samples", C.c_uint64), ("lookups", C.c_uint64),
                ("render_ms", C.c_double), ("macrocell_ms", C.c_double), ("launches", C.c_uint32),
                ("reserved", C.c_uint32)]


class GridInfo(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("background", C.c_float), ("voxel_type", C.c_int32),
                ("codec", C.c_int32), ("value_domain", C.c_float * 2), ("n_upper", C.c_uint64),
                ("n_lower", C.c_uint64), ("n_leaf", C.c_uint64), ("n_root", C.c_uint64),
                ("svdb_bytes", C.c_uint64), ("device_bytes", C.c_uint64),
                ("leaf_payload_bytes", C.c_uint64), ("device", C.c_int32), ("reserved", C.c_int32)]


class CompressReport(C.Structure):
    _fields_ = [("background", C.c_float), ("num_bricks", C.c_uint64), ("bricks_activated", C.c_uint64),
                ("voxels_activated", C.c_uint64), ("frozen_bytes", C.c_uint64),
                ("dense_bytes", C.c_uint64), ("achieved_ratio", C.c_double)]


# exported symbol -> (restype, argtypes); tests check this list against include/svdbgpu.h
P = C.c_void_p
SLAB_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_float))
SIGNATURES = {
    "svdbgpu_abi_version": (C.c_int, []),
    "svdbgpu_last_error": (C.c_char_p, []),
    "svdbgpu_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "svdbgpu_free": (None, [P]),
    "svdbgpu_grid_create": (C.c_int, [P, C.c_size_t, C.c_int32, C.c_int32, C.POINTER(P)]),
    "svdbgpu_grid_destroy": (C.c_int, [P]),
    "svdbgpu_grid_info_get": (C.c_int, [P, C.POINTER(GridInfo)]),
    "svdbgpu_grid_leaf_codes": (C.c_int, [P, C.c_uint64, C.c_uint64, P, P]),
    "svdbgpu_read_voxels": (C.c_int, [P, P, C.c_size_t, P]),
    "svdbgpu_sample": (C.c_int, [P, P, C.c_size_t, C.c_int32, P]),
    "svdbgpu_gradient": (C.c_int, [P, P, C.c_size_t, P]),
    "svdbgpu_read_voxels_device": (C.c_int, [P, P, C.c_size_t, P, P]),
    "svdbgpu_sample_device": (C.c_int, [P, P, C.c_size_t, C.c_int32, P, P]),
    "svdbgpu_macrocells": (C.c_int, [P, C.POINTER(TF), C.POINTER(C.c_int32), P, P, P, P, C.c_size_t]),
    "svdbgpu_render": (C.c_int, [P, C.POINTER(TF), C.POINTER(Camera), C.POINTER(Settings), P,
                                 C.POINTER(Stats)]),
    "svdbgpu_render_device": (C.c_int, [P, C.POINTER(TF), C.POINTER(Camera), C.POINTER(Settings), P,
                                        C.c_int32, P, C.POINTER(Stats)]),
    "svdbgpu_render_multi": (C.c_int, [P, C.c_int32, C.POINTER(TF), C.POINTER(Camera), C.POINTER(Settings), P,
                                       C.POINTER(Stats), C.POINTER(C.c_double)]),
    "svdbgpu_nccl_version": (C.c_int, [C.POINTER(C.c_int32)]),
    "svdbgpu_tiles_for_rank": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "svdbgpu_unpack_tiles_device": (C.c_int, [P, C.c_int32, C.c_int64, C.c_int32, C.c_int32, P, P]),
    "svdbgpu_compress": (C.c_int, [P, C.POINTER(C.c_int32), C.c_int32, C.c_double, C.c_int32,
                                   C.c_int32, C.POINTER(P), C.POINTER(C.c_size_t),
                                   C.POINTER(CompressReport)]),
    "svdbgpu_synth": (C.c_int, [C.c_int32, C.POINTER(C.c_int32), C.c_uint64, C.c_int32, P]),
    "svdbgpu_compress_stream": (C.c_int, [SLAB_FN, P, C.POINTER(C.c_int32), C.c_int32, C.c_double, C.c_int32,
                                          C.c_int32, C.POINTER(P), C.POINTER(C.c_size_t),
                                          C.POINTER(CompressReport), C.POINTER(C.c_double)]),
    "svdbgpu_synth_compress": (C.c_int, [C.c_int32, C.POINTER(C.c_int32), C.c_uint64, C.c_double, C.c_int32,
                                         C.c_int32, C.POINTER(P), C.POINTER(C.c_size_t), C.POINTER(CompressReport),
                                         C.POINTER(C.c_double)]),
    "svdbgpu_quantise": (C.c_int, [P, C.c_size_t, C.c_int32, C.c_int32, C.POINTER(P), C.POINTER(C.c_size_t)]),
}

_lib = None


def lib():
    """Load libsvdbgpu.so once. Raises (never falls back) if it has not been built."""
    global _lib
    if _lib is None:
        path = os.environ.get("SVDBGPU_LIB", LIB_PATH)  # A/B builds (csrc/Makefile `variants`)
        if not os.path.exists(path):
            raise ImportError(f"{path} not built: run `make -C paper_2504_04564_b200/csrc` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
