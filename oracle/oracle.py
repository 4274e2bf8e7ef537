"""ctypes face of the CPU oracles — TEST INFRASTRUCTURE ONLY.

Two checkers live here:

* ``Oracle``  — ``oracle/liboracle.so``: our plain-C restatement (svdb_oracle.c) of the
  reference hot path plus the north-star additions (leaf codec, EA march, ratio tracking).
* ``Reference`` — ``oracle/_ref/libsvdbref.so``: the UNMODIFIED reference headers
  (/root/reference/proj/include) compiled in place behind ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` / ``--impl reference``
legs may import this module, and only as the checker / baseline — never as the product path.
Scene objects are duck-typed (anything with the attribute names of the product's
TransferFunction / Camera / RenderSettings works).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsvdbref.so")

MODES = {"pathtrace": 0, "iso": 1, "ea": 2, "ratio": 3}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class _TF(C.Structure):
    _fields_ = [("domain_lo", C.c_double), ("domain_hi", C.c_double),
                ("density_scale", C.c_double), ("n_entries", C.c_int),
                ("rgba", C.POINTER(C.c_float))]


class _Cam(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("look_at", C.c_double * 3),
                ("up", C.c_double * 3), ("fov_y_deg", C.c_double),
                ("width", C.c_int), ("height", C.c_int)]


class _Settings(C.Structure):
    _fields_ = [("spp", C.c_int), ("max_bounces", C.c_int), ("rr_start_bounce", C.c_int),
                ("seed", C.c_uint64), ("mode", C.c_int), ("iso_value", C.c_double),
                ("ambient", C.c_float * 3), ("background", C.c_float * 3),
                ("ea_step", C.c_double), ("ea_min_transmittance", C.c_double),
                ("tile_rank", C.c_int), ("tile_nranks", C.c_int), ("threads", C.c_int),
                ("majorant_cell", C.c_int), ("hdda", C.c_int)]


def _take_bytes(ptr, n: int) -> bytes:
    # ctypes.string_at takes a C int size: copy > 2 GiB buffers through memmove instead
    buf = bytearray(n)
    if n:
        C.memmove((C.c_char * n).from_buffer(buf), ptr, n)
    return bytes(buf)


def _f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _f64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _mode_of(settings) -> int:
    m = getattr(settings, "mode", "pathtrace")
    if isinstance(m, int):
        return m
    return MODES[getattr(m, "name", m)]


def tf_entries(tf) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(tf.entries, dtype=np.float32).reshape(-1, 4))


def _cam9(cam):
    return (C.c_double * 9)(*cam.position, *cam.look_at, *cam.up)


class Oracle:
    """Plain-C restatement (liboracle.so)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.so_open.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.so_close.argtypes = [C.c_void_p]
        L.so_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_float), C.POINTER(C.c_uint64)]
        L.so_read_voxels.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int]
        L.so_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
        L.so_macrocells.argtypes = [C.c_void_p, C.POINTER(_TF), C.POINTER(C.c_int), C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
        L.so_render.argtypes = [C.c_void_p, C.POINTER(_TF), C.POINTER(_Cam), C.POINTER(_Settings),
                                C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.so_quantize.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_size_t), C.c_void_p, C.c_void_p]
        L.so_decode.argtypes = [C.c_int, C.c_int, C.c_float, C.c_float]
        L.so_decode.restype = C.c_float
        L.so_mix64.argtypes = [C.c_uint64]
        L.so_mix64.restype = C.c_uint64
        L.so_rng_uniforms.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_size_t, C.c_void_p]
        L.so_free.argtypes = [C.c_void_p]
        L.so_synth.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
        L.so_sparse_threshold.argtypes = [C.c_int]
        L.so_sparse_threshold.restype = C.c_double

    def open(self, svdb: bytes) -> "OracleGrid":
        return OracleGrid(self, svdb)

    SYNTH_KINDS = {"marschner_lobb": 0, "fbm_smoke": 1, "turbulence": 2, "sparse": 3}

    def synth(self, kind, dims, seed: int = 0, threads: int = 0) -> np.ndarray:
        """Restated synthetic volume [z, y, x] float32 (synth_oracle.c), bit-identical to the
        product's svdbgpu_synth, so baselines can build inputs without the product library."""
        k = self.SYNTH_KINDS[kind] if isinstance(kind, str) else int(kind)
        dx, dy, dz = (int(d) for d in dims)
        out = np.empty((dz, dy, dx), dtype=np.float32)
        rc = self.lib.so_synth(k, (C.c_int32 * 3)(dx, dy, dz), seed, threads, out.ctypes.data)
        if rc:
            raise OracleError(rc, "synth")
        return out

    def sparse_threshold(self, dim_max: int) -> float:
        return self.lib.so_sparse_threshold(dim_max)

    def quantize(self, svdb: bytes, codec: int):
        """-> (dequantised svdb bytes, codes[n_leaf,512] u8, params[n_leaf,2] f32)."""
        buf = np.frombuffer(svdb, dtype=np.uint8)
        n_leaf = int(np.frombuffer(svdb[52:60], dtype=np.uint64)[0])
        codes = np.zeros((max(n_leaf, 1), 512), dtype=np.uint8)
        params = np.zeros((max(n_leaf, 1), 2), dtype=np.float32)
        out = C.c_void_p()
        n_out = C.c_size_t()
        rc = self.lib.so_quantize(buf.ctypes.data, len(svdb), codec, C.byref(out), C.byref(n_out),
                                  codes.ctypes.data, params.ctypes.data)
        if rc:
            raise OracleError(rc, "quantize")
        data = _take_bytes(out, n_out.value)
        self.lib.so_free(out)
        return data, codes[:n_leaf], params[:n_leaf]

    def rng_uniforms(self, seed, px, py, s, n):
        out = np.zeros(n, dtype=np.float64)
        self.lib.so_rng_uniforms(seed, px, py, s, n, out.ctypes.data)
        return out


class OracleGrid:
    def __init__(self, orc: Oracle, svdb: bytes):
        self.o = orc
        self._buf = np.frombuffer(svdb, dtype=np.uint8)
        h = C.c_void_p()
        rc = orc.lib.so_open(self._buf.ctypes.data, len(svdb), C.byref(h))
        if rc:
            raise OracleError(rc, "so_open")
        self.h = h
        dims = (C.c_int * 3)()
        bg = C.c_float()
        counts = (C.c_uint64 * 4)()
        orc.lib.so_info(h, dims, C.byref(bg), counts)
        self.dims = tuple(dims)
        self.background = bg.value
        self.counts = tuple(counts)

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.so_close(self.h)
            self.h = None

    def read_voxels(self, ijk, cached=False):
        ijk = np.ascontiguousarray(ijk, dtype=np.int32).reshape(-1, 3)
        out = np.zeros(len(ijk), dtype=np.float32)
        self.o.lib.so_read_voxels(self.h, ijk.ctypes.data, len(ijk), out.ctypes.data, int(cached))
        return out

    def sample(self, xyz, mode=1):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(len(xyz), dtype=np.float32)
        self.o.lib.so_sample(self.h, xyz.ctypes.data, len(xyz), mode, out.ctypes.data)
        return out

    def macrocells(self, tf):
        ent = tf_entries(tf)
        t = _TF(tf.domain_lo, tf.domain_hi, tf.density_scale, len(ent), _f32p(ent))
        cells = (C.c_int * 3)()
        self.o.lib.so_macrocells(self.h, C.byref(t), cells, None, None, None, None, 0)
        n = cells[0] * cells[1] * cells[2]
        cmin = np.zeros(n, np.float32); cmax = np.zeros(n, np.float32)
        maj = np.zeros(n, np.float32); empty = np.zeros(n, np.uint8)
        self.o.lib.so_macrocells(self.h, C.byref(t), cells, cmin.ctypes.data, cmax.ctypes.data,
                                 maj.ctypes.data, empty.ctypes.data, n)
        return tuple(cells), cmin, cmax, maj, empty

    def render(self, tf, cam, settings, tile_rank=0, tile_nranks=1, threads=0, rgb=None):
        """-> (rgb[H,W,3] float32, lookups, paths)."""
        ent = tf_entries(tf)
        t = _TF(tf.domain_lo, tf.domain_hi, tf.density_scale, len(ent), _f32p(ent))
        c = _Cam((C.c_double * 3)(*cam.position), (C.c_double * 3)(*cam.look_at),
                 (C.c_double * 3)(*cam.up), cam.fov_y_deg, cam.width, cam.height)
        s = _Settings(settings.spp, settings.max_bounces, settings.rr_start_bounce,
                      settings.seed, _mode_of(settings), settings.iso_value,
                      (C.c_float * 3)(*settings.ambient_radiance),
                      (C.c_float * 3)(*settings.background_color),
                      getattr(settings, "ea_step", 0.5),
                      getattr(settings, "ea_min_transmittance", 1e-4),
                      tile_rank, tile_nranks, threads, getattr(settings, "majorant_cell", 0),
                      int(getattr(settings, "hdda", 0)))
        if rgb is None:
            rgb = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
        lk = C.c_uint64()
        pa = C.c_uint64()
        rc = self.o.lib.so_render(self.h, C.byref(t), C.byref(c), C.byref(s), rgb.ctypes.data,
                                  C.byref(lk), C.byref(pa))
        if rc:
            raise OracleError(rc, "so_render")
        return rgb, lk.value, pa.value


class Reference:
    """The unmodified reference (oracle/_ref/libsvdbref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_compress.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                   C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_void_p]
        L.ref_build_ops.argtypes = [C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_size_t)]
        L.ref_grid_open.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.ref_grid_close.argtypes = [C.c_void_p]
        L.ref_read_voxels.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int]
        L.ref_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
        L.ref_gradient.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.ref_macrocells.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_int,
                                     C.c_double, C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_double)]
        L.ref_dda.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_void_p,
                              C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_render.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_int, C.c_double,
                                 C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.c_uint64, C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_int,
                                 C.c_void_p]
        L.ref_render_tiles.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_int,
                                       C.c_double, C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_int, C.c_int,
                                       C.c_int, C.c_void_p, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.c_int]
        L.ref_woodcock.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_int,
                                   C.c_double, C.c_double, C.c_void_p, C.c_double, C.c_double,
                                   C.c_uint64, C.c_size_t, C.c_void_p, C.POINTER(C.c_uint64)]
        L.ref_rng_uniforms.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_size_t, C.c_void_p]
        L.ref_hardware_threads.restype = C.c_int

    def _check(self, rc, what):
        if rc:
            raise OracleError(rc, f"{what}: {self.lib.ref_last_error().decode()}")

    def _take(self, p, n):
        data = _take_bytes(p, n.value)
        self.lib.ref_free(p)
        return data

    def compress(self, data: np.ndarray, voxel_type: int = 1, quality: float = 1.0, metric: int = 2):
        """data[z,y,x] float32 -> (svdb bytes, report dict). voxel_type 0 = u8 source."""
        data = np.ascontiguousarray(data, dtype=np.float32)
        dz, dy, dx = data.shape
        out = C.c_void_p(); n = C.c_size_t()
        rep = np.zeros(7, dtype=np.uint64)
        self._check(self.lib.ref_compress(data.ctypes.data, dx, dy, dz, voxel_type, quality, metric,
                                          C.byref(out), C.byref(n), rep.ctypes.data), "compress")
        report = dict(background=float(rep[0:1].view(np.float32)[0]), num_bricks=int(rep[1]),
                      bricks_activated=int(rep[2]), voxels_activated=int(rep[3]),
                      frozen_bytes=int(rep[4]), dense_bytes=int(rep[5]),
                      achieved_ratio=float(rep[6:7].view(np.float64)[0]))
        return self._take(out, n), report

    def build_ops(self, dims, background, ops, prune=False) -> bytes:
        """ops: list of (kind, (x,y,z), value); kind 0 voxel, 1 lower tile, 2 upper tile."""
        kinds = np.array([o[0] for o in ops] or [0], dtype=np.int32)
        xyz = np.array([o[1] for o in ops] or [(0, 0, 0)], dtype=np.int32).reshape(-1, 3)
        vals = np.array([o[2] for o in ops] or [0], dtype=np.float32)
        out = C.c_void_p(); n = C.c_size_t()
        self._check(self.lib.ref_build_ops(dims[0], dims[1], dims[2], background, kinds.ctypes.data,
                                           xyz.ctypes.data, vals.ctypes.data, len(ops), int(prune),
                                           C.byref(out), C.byref(n)), "build_ops")
        return self._take(out, n)

    def open(self, svdb: bytes) -> "RefGrid":
        return RefGrid(self, svdb)

    def hardware_threads(self) -> int:
        return self.lib.ref_hardware_threads()

    def rng_uniforms(self, seed, px, py, s, n):
        out = np.zeros(n, dtype=np.float64)
        self.lib.ref_rng_uniforms(seed, px, py, s, n, out.ctypes.data)
        return out


class RefGrid:
    def __init__(self, ref: Reference, svdb: bytes):
        self.r = ref
        self._buf = np.frombuffer(svdb, dtype=np.uint8)
        h = C.c_void_p()
        ref._check(ref.lib.ref_grid_open(self._buf.ctypes.data, len(svdb), C.byref(h)), "open")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_grid_close(self.h)
            self.h = None

    def read_voxels(self, ijk, cached=False):
        ijk = np.ascontiguousarray(ijk, dtype=np.int32).reshape(-1, 3)
        out = np.zeros(len(ijk), dtype=np.float32)
        self.r._check(self.r.lib.ref_read_voxels(self.h, ijk.ctypes.data, len(ijk), out.ctypes.data,
                                                 int(cached)), "read_voxels")
        return out

    def sample(self, xyz, mode=1):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(len(xyz), dtype=np.float32)
        self.r._check(self.r.lib.ref_sample(self.h, xyz.ctypes.data, len(xyz), mode, out.ctypes.data),
                      "sample")
        return out

    def gradient(self, xyz):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        out = np.zeros_like(xyz)
        self.r._check(self.r.lib.ref_gradient(self.h, xyz.ctypes.data, len(xyz), out.ctypes.data),
                      "gradient")
        return out

    def macrocells(self, tf):
        ent = tf_entries(tf)
        cells = (C.c_int * 3)()
        secs = C.c_double()
        self.r._check(self.r.lib.ref_macrocells(self.h, tf.domain_lo, tf.domain_hi, ent.ctypes.data,
                                                len(ent), tf.density_scale, cells, None, None, None,
                                                None, 0, C.byref(secs)), "macrocells")
        n = cells[0] * cells[1] * cells[2]
        cmin = np.zeros(n, np.float32); cmax = np.zeros(n, np.float32)
        maj = np.zeros(n, np.float32); empty = np.zeros(n, np.uint8)
        self.r._check(self.r.lib.ref_macrocells(self.h, tf.domain_lo, tf.domain_hi, ent.ctypes.data,
                                                len(ent), tf.density_scale, cells, cmin.ctypes.data,
                                                cmax.ctypes.data, maj.ctypes.data, empty.ctypes.data,
                                                n, C.byref(secs)), "macrocells")
        self.macrocell_seconds = secs.value
        return tuple(cells), cmin, cmax, maj, empty

    def dda(self, origin, direction, t0=0.0, t1=float("inf"), cap=4096):
        ray = (C.c_double * 6)(*origin, *direction)
        cells = np.zeros((cap, 3), np.int32)
        ts = np.zeros((cap, 2), np.float64)
        n = C.c_size_t()
        self.r._check(self.r.lib.ref_dda(self.h, ray, t0, t1, cells.ctypes.data, ts.ctypes.data, cap,
                                         C.byref(n)), "dda")
        k = min(n.value, cap)
        return cells[:k], ts[:k]

    def render(self, tf, cam, settings, threads=0):
        ent = tf_entries(tf)
        rgb = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
        mode = _mode_of(settings)
        if mode not in (0, 1):
            raise ValueError("the reference renders pathtrace and iso only")
        self.r._check(self.r.lib.ref_render(
            self.h, tf.domain_lo, tf.domain_hi, ent.ctypes.data, len(ent), tf.density_scale,
            _cam9(cam), cam.fov_y_deg, cam.width, cam.height, settings.spp, settings.max_bounces,
            settings.rr_start_bounce, settings.seed, mode, settings.iso_value,
            (C.c_float * 3)(*settings.ambient_radiance), (C.c_float * 3)(*settings.background_color),
            threads, rgb.ctypes.data), "render")
        return rgb

    def render_tiles(self, tf, cam, settings, tile_stride=1, tile_phase=0, threads=0, rgb=None,
                     count=True):
        """Reference per-pixel body over a tile subset (needs macrocells(tf) first).
        -> (rgb, lookups, paths, seconds). count=False traces through the stock GridField (no
        per-lookup counter in the timed loop) and returns lookups = 0."""
        ent = tf_entries(tf)
        if rgb is None:
            rgb = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
        lk = C.c_uint64(); pa = C.c_uint64(); sec = C.c_double()
        self.r._check(self.r.lib.ref_render_tiles(
            self.h, tf.domain_lo, tf.domain_hi, ent.ctypes.data, len(ent), tf.density_scale,
            _cam9(cam), cam.fov_y_deg, cam.width, cam.height, settings.spp, settings.max_bounces,
            settings.rr_start_bounce, settings.seed, (C.c_float * 3)(*settings.ambient_radiance),
            threads, tile_stride, tile_phase, rgb.ctypes.data, C.byref(lk), C.byref(pa),
            C.byref(sec), int(bool(count))), "render_tiles")
        return rgb, lk.value, pa.value, sec.value

    def woodcock(self, tf, sigma_maj, origin, direction, t0, t1, seed, n):
        ent = tf_entries(tf)
        ray = (C.c_double * 6)(*origin, *direction)
        out = np.zeros(n, np.float64)
        nxt = C.c_uint64()
        self.r._check(self.r.lib.ref_woodcock(self.h, tf.domain_lo, tf.domain_hi, ent.ctypes.data,
                                              len(ent), tf.density_scale, sigma_maj, ray, t0, t1,
                                              seed, n, out.ctypes.data, C.byref(nxt)), "woodcock")
        return out, nxt.value


def have_reference() -> bool:
    return os.path.exists(REF_SO)
