"""Host-side mirror of the reference svdb API for the hot path, over the C-ABI (libsvdbgpu.so).

Names, argument meaning and error behaviour follow /root/reference/proj/include/svdb:

* ``TransferFunction``  transfer.hpp:23-35 (same validation, same ``Error(Errc.size_mismatch)``)
* ``Camera`` / ``RenderSettings`` / ``RenderMode`` / ``Image``  render.hpp:25-58
* ``compress`` / ``CompressionParams`` / ``CompressionReport``  compress.hpp:68-95, 221-283
* ``DeviceGrid``  the FrozenGrid of frozen.hpp:70-131, resident on one B200
  (``read_voxel`` frozen.hpp:82, ``sample`` sample.hpp:97, ``gradient`` sample.hpp:102)
* ``render``  render.hpp:319-325
* ``build_macrocells`` / ``update_majorants``  macrocell.hpp:74-116

Every compute call runs on the GPU through the C-ABI; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N


class Errc(enum.IntEnum):
    """errors.hpp:11-23"""
    io_error = 0
    size_mismatch = 1
    non_finite_voxel = 2
    out_of_bounds = 3
    misaligned = 4
    empty_box = 5
    invalid_quality = 6
    bad_magic = 7
    version_mismatch = 8
    corrupt_index = 9
    dims_mismatch = 10


class Error(RuntimeError):
    """svdb::Error (errors.hpp:43-54) for codes 1..11; ``code`` is the Errc, or the raw ABI
    status (SVDBGPU_E_*) for device-side failures."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = Errc(status - 1) if 1 <= status <= 11 else status
        super().__init__(message)


E_CUDA, E_INVALID_ARG, E_NO_DEVICE, E_OOM, E_UNSUPPORTED, E_NCCL = 64, 65, 66, 67, 68, 69


def _take_bytes(ptr, n: int) -> bytes:
    # ctypes.string_at takes a C int size: copy > 2 GiB buffers through memmove instead
    buf = bytearray(n)
    if n:
        C.memmove((C.c_char * n).from_buffer(buf), ptr, n)
    return bytes(buf)


def _check(rc: int):
    if rc:
        msg = N.lib().svdbgpu_last_error()
        raise Error(rc, msg.decode() if msg else f"status {rc}")


class VoxelType(enum.IntEnum):
    u8 = 0
    f32 = 1


class Metric(enum.IntEnum):
    closest = 0
    farthest = 1
    median = 2


class Codec(enum.IntEnum):
    """Device leaf codecs (include/svdbgpu.h)."""
    f32 = 0
    unorm8 = 1
    affine8 = 2
    affine4 = 3
    auto8 = 4


class RenderMode(enum.IntEnum):
    pathtrace = 0
    iso = 1
    ea = 2
    ratio = 3


@dataclass
class CompressionParams:
    quality: float = 1.0
    metric: Metric = Metric.median


@dataclass
class CompressionReport:
    background: float
    num_bricks: int
    bricks_activated: int
    voxels_activated: int
    frozen_bytes: int
    dense_bytes: int
    achieved_ratio: float


def compress(volume: np.ndarray, params: CompressionParams = CompressionParams(),
             voxel_type: VoxelType = VoxelType.f32, threads: int = 0):
    """Fixed-rate encoder (compress.hpp:221-283) on the host, native and multi-threaded.
    ``volume`` is indexed [z, y, x] (x fastest, volume.hpp:32-33). u8 sources must already
    hold byte/255.0f values (DenseVolume::load_raw, volume.hpp:91-97).
    Returns (SVDB v1 bytes, CompressionReport); the bytes equal the reference's
    serialize_frozen(compress(...).first)."""
    vol = np.ascontiguousarray(volume, dtype=np.float32)
    if vol.ndim != 3:
        raise Error(Errc.size_mismatch + 1, "volume must be 3-D [z, y, x]")
    dims = (C.c_int32 * 3)(vol.shape[2], vol.shape[1], vol.shape[0])
    out = C.c_void_p()
    n = C.c_size_t()
    rep = N.CompressReport()
    L = N.lib()
    _check(L.svdbgpu_compress(vol.ctypes.data, dims, int(voxel_type), float(params.quality),
                              int(params.metric), threads, C.byref(out), C.byref(n), C.byref(rep)))
    data = _take_bytes(out, n.value)
    L.svdbgpu_free(out)
    return data, CompressionReport(rep.background, rep.num_bricks, rep.bricks_activated,
                                   rep.voxels_activated, rep.frozen_bytes, rep.dense_bytes,
                                   rep.achieved_ratio)


class OwnedBuffer(np.ndarray):
    """A uint8 array over a buffer the library malloc'd (freed with svdbgpu_free when the array and
    every view of it are gone): large containers reach Python without a copy."""

    @staticmethod
    def take(ptr, n: int) -> "OwnedBuffer":
        import weakref
        if n == 0:
            N.lib().svdbgpu_free(ptr)
            return np.zeros(0, np.uint8).view(OwnedBuffer)
        raw = (C.c_uint8 * n).from_address(ptr.value)
        arr = np.ctypeslib.as_array(raw).view(OwnedBuffer)
        weakref.finalize(raw, N.lib().svdbgpu_free, C.c_void_p(ptr.value))
        arr._raw = raw  # keeps the ctypes object (and so the finalizer) alive with the array
        return arr


def _report(rep) -> "CompressionReport":
    return CompressionReport(rep.background, rep.num_bricks, rep.bricks_activated, rep.voxels_activated,
                             rep.frozen_bytes, rep.dense_bytes, rep.achieved_ratio)


def synth_compress(kind: str, dims: Sequence[int], seed: int = 0, params: CompressionParams = CompressionParams(),
                   device: int = 0):
    """The synth(kind, dims, seed) volume compressed on the GPU without a dense host array (streaming
    device encoder, svdbgpu_synth_compress): the same bytes as compress(synth(...)). Returns
    (SVDB v1 buffer, CompressionReport, encode seconds); kinds fbm_smoke / turbulence / sparse."""
    dx, dy, dz = (int(d) for d in dims)
    out = C.c_void_p()
    n = C.c_size_t()
    rep = N.CompressReport()
    sec = C.c_double()
    _check(N.lib().svdbgpu_synth_compress(SYNTH_KINDS[kind], (C.c_int32 * 3)(dx, dy, dz), seed, float(params.quality),
                                          int(params.metric), device, C.byref(out), C.byref(n), C.byref(rep),
                                          C.byref(sec)))
    return OwnedBuffer.take(out, n.value), _report(rep), sec.value


def compress_stream(slab_fn, dims: Sequence[int], params: CompressionParams = CompressionParams(),
                    voxel_type: VoxelType = VoxelType.f32, device: int = 0):
    """The fixed-rate encoder over a volume streamed through the GPU in 32-slice z-slabs
    (svdbgpu_compress_stream): ``slab_fn(z0, nz)`` returns slices [z0, z0 + nz) as float32 [nz, y, x]
    (called five times per slab, same values each time). Same bytes as compress() on the dense
    volume. Returns (SVDB v1 buffer, CompressionReport, encode seconds)."""
    dx, dy, dz = (int(d) for d in dims)
    err = []

    def cb(user, z0, nz, dst):
        try:
            a = np.ascontiguousarray(slab_fn(int(z0), int(nz)), dtype=np.float32)
            if a.size != dx * dy * nz:
                raise ValueError(f"slab_fn({z0}, {nz}) returned {a.size} values, want {dx * dy * nz}")
            C.memmove(dst, a.ctypes.data, a.nbytes)
            return 0
        except Exception as exc:  # reported through the library as IoError
            err.append(exc)
            return 1

    fn = N.SLAB_FN(cb)
    out = C.c_void_p()
    n = C.c_size_t()
    rep = N.CompressReport()
    sec = C.c_double()
    rc = N.lib().svdbgpu_compress_stream(fn, None, (C.c_int32 * 3)(dx, dy, dz), int(voxel_type), float(params.quality),
                                         int(params.metric), device, C.byref(out), C.byref(n), C.byref(rep),
                                         C.byref(sec))
    if rc and err:
        raise err[0]
    _check(rc)
    return OwnedBuffer.take(out, n.value), _report(rep), sec.value


def quantise(svdb: bytes, codec: "Codec" = None, device: int = 0) -> bytes:
    """SVDB v1 -> quantised SVDB v2 (leaves as N-bit codes + per-leaf lo/scale, encoded on the GPU
    with the device codec; include/svdbgpu.h ``svdbgpu_quantise``). ``DeviceGrid`` loads the result
    to exactly the grid it builds from the v1 bytes with that codec."""
    codec = Codec.auto8 if codec is None else codec
    buf = np.frombuffer(svdb, dtype=np.uint8) if len(svdb) else np.zeros(1, np.uint8)
    out = C.c_void_p()
    n = C.c_size_t()
    L = N.lib()
    _check(L.svdbgpu_quantise(buf.ctypes.data, len(svdb), int(codec), device, C.byref(out), C.byref(n)))
    data = _take_bytes(out, n.value)
    L.svdbgpu_free(out)
    return data


SYNTH_KINDS = {"marschner_lobb": 0, "fbm_smoke": 1, "turbulence": 2, "sparse": 3}


def synth(kind: str, dims: Sequence[int], seed: int = 0, threads: int = 0) -> np.ndarray:
    """Deterministic synthetic volume [z, y, x] float32 (BASELINE.json configs)."""
    dx, dy, dz = (int(d) for d in dims)
    out = np.empty((dz, dy, dx), dtype=np.float32)
    _check(N.lib().svdbgpu_synth(SYNTH_KINDS[kind], (C.c_int32 * 3)(dx, dy, dz), seed, threads,
                                 out.ctypes.data))
    return out


class TransferFunction:
    """Piecewise-linear RGBA over evenly spaced entries (transfer.hpp:23-96)."""

    def __init__(self, domain_lo: float, domain_hi: float, entries, density_scale: float = 1.0):
        ent = np.ascontiguousarray(np.asarray(entries, dtype=np.float32).reshape(-1, 4))
        if not domain_hi > domain_lo:
            raise Error(Errc.size_mismatch + 1, "transfer function domain must have hi > lo")
        if len(ent) < 2:
            raise Error(Errc.size_mismatch + 1, "transfer function needs at least 2 entries")
        if not (density_scale > 0.0) or not np.isfinite(density_scale):
            raise Error(Errc.size_mismatch + 1, "density_scale must be positive")
        if not np.all((ent[:, 3] >= 0.0) & (ent[:, 3] <= 1.0)):
            raise Error(Errc.size_mismatch + 1, "transfer function alpha must be in [0,1]")
        self.domain_lo = float(domain_lo)
        self.domain_hi = float(domain_hi)
        self.density_scale = float(density_scale)
        self.entries = ent

    def _c(self) -> N.TF:
        return N.TF(self.domain_lo, self.domain_hi, self.density_scale, len(self.entries),
                    self.entries.ctypes.data_as(C.POINTER(C.c_float)))


@dataclass
class Camera:
    """render.hpp:25-32"""
    position: tuple = (0.0, 0.0, 0.0)
    look_at: tuple = (0.0, 0.0, 1.0)
    up: tuple = (0.0, 1.0, 0.0)
    fov_y_deg: float = 45.0
    width: int = 512
    height: int = 512

    def _c(self) -> N.Camera:
        return N.Camera((C.c_double * 3)(*self.position), (C.c_double * 3)(*self.look_at),
                        (C.c_double * 3)(*self.up), self.fov_y_deg, self.width, self.height)


def frame_camera(dims, width=512, height=512, fov_y_deg=45.0) -> Camera:
    """The CLI's auto-framing (tools/svdb.cpp:267-274): look at the centre from -z at
    2.2 x the largest extent."""
    ext = [float(d - 1) for d in dims]
    c = [e * 0.5 for e in ext]
    return Camera(position=(c[0], c[1], c[2] - 2.2 * max(1.0, max(ext))), look_at=tuple(c),
                  fov_y_deg=fov_y_deg, width=width, height=height)


@dataclass
class RenderSettings:
    """render.hpp:39-49 (+ EA step / termination; ``threads`` is accepted and ignored: the
    device decides its own parallelism and results never depend on it)."""
    spp: int = 16
    max_bounces: int = 64
    rr_start_bounce: int = 3
    seed: int = 0
    mode: RenderMode = RenderMode.pathtrace
    iso_value: float = 0.5
    ambient_radiance: tuple = (1.0, 1.0, 1.0)
    background_color: tuple = (0.0, 0.0, 0.0)
    threads: int = 0
    ea_step: float = 0.5
    ea_min_transmittance: float = 1e-4
    kernel: int = 0  # 0 auto (path-regenerating tracer), 1 per-pixel (A/B); images identical
    # majorant grid cell edge: 0 = the reference's 32^3 macrocells (bit parity); 128 / 8 =
    # lower-node / leaf-node majorants (node-majorant tracking, statistically equal)
    majorant_cell: int = 0
    # tracking arithmetic (pathtrace / ratio): 0 = FP64 reference-exact (bit parity); 2 = mixed
    # (FP64 ray / DDA / distances, FP32 step log, sampler, TF, throughput) and 1 = all FP32, both
    # matching the FP64 image within a tolerance at matched streams
    precision: int = 0
    # 1: hierarchical empty-space skipping over the node tree (lower-node level, then the majorant
    # grid); statistically equal to the flat DDA, different streams
    hdda: int = 0

    def _c(self, tile_rank: int = 0, tile_nranks: int = 1) -> N.Settings:
        return N.Settings(self.spp, self.max_bounces, self.rr_start_bounce, self.seed, int(self.mode),
                          self.iso_value, (C.c_float * 3)(*self.ambient_radiance),
                          (C.c_float * 3)(*self.background_color), self.ea_step,
                          self.ea_min_transmittance, tile_rank, tile_nranks, self.kernel,
                          self.majorant_cell, self.precision, int(self.hdda))


@dataclass
class Image:
    """Linear-light image (render.hpp:51-58): pixels[y, x] = (r, g, b), row 0 at the top."""
    width: int
    height: int
    pixels: np.ndarray
    stats: dict = field(default_factory=dict)

    def at(self, x: int, y: int):
        return self.pixels[y, x]


def _stats_dict(s: N.Stats) -> dict:
    return dict(paths=s.paths, samples=s.samples, lookups=s.lookups, render_ms=s.render_ms,
                macrocell_ms=s.macrocell_ms, launches=s.launches)


class DeviceGrid:
    """A frozen grid resident on one GPU (FrozenGrid, frozen.hpp:70-131)."""

    def __init__(self, svdb: bytes, codec: Codec = Codec.auto8, device: int = 0):
        self._h = None
        buf = np.frombuffer(svdb, dtype=np.uint8)
        h = C.c_void_p()
        _check(N.lib().svdbgpu_grid_create(buf.ctypes.data, len(svdb), int(codec), device, C.byref(h)))
        self._h = h
        info = N.GridInfo()
        _check(N.lib().svdbgpu_grid_info_get(h, C.byref(info)))
        self.dims = tuple(info.dims)
        self.background = info.background
        self.voxel_type = VoxelType(info.voxel_type)
        self.codec = Codec(info.codec)
        self.value_domain = tuple(info.value_domain)
        self.counts = dict(upper=info.n_upper, lower=info.n_lower, leaf=info.n_leaf, root=info.n_root)
        self.svdb_bytes = info.svdb_bytes
        self.device_bytes = info.device_bytes
        self.leaf_payload_bytes = info.leaf_payload_bytes
        self.device = info.device

    @classmethod
    def from_svdb(cls, svdb: bytes, codec: Codec = Codec.auto8, device: int = 0) -> "DeviceGrid":
        return cls(svdb, codec, device)

    def close(self):
        if self._h:
            N.lib().svdbgpu_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def read_voxels(self, ijk) -> np.ndarray:
        ijk = np.ascontiguousarray(ijk, dtype=np.int32).reshape(-1, 3)
        out = np.empty(len(ijk), dtype=np.float32)
        _check(N.lib().svdbgpu_read_voxels(self._h, ijk.ctypes.data, len(ijk), out.ctypes.data))
        return out

    def read_voxel(self, ijk) -> float:
        return float(self.read_voxels([ijk])[0])

    def sample(self, xyz, mode: int = 1) -> np.ndarray:
        """mode 0 = nearest, 1 = trilinear (SampleMode, sample.hpp:16-19)."""
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(xyz), dtype=np.float32)
        _check(N.lib().svdbgpu_sample(self._h, xyz.ctypes.data, len(xyz), int(mode), out.ctypes.data))
        return out

    def gradient(self, xyz) -> np.ndarray:
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        out = np.empty_like(xyz)
        _check(N.lib().svdbgpu_gradient(self._h, xyz.ctypes.data, len(xyz), out.ctypes.data))
        return out

    def macrocells(self, tf: TransferFunction | None = None):
        """-> (cells, cell_min, cell_max, majorant, empty) like build_macrocells +
        update_majorants (macrocell.hpp:74-116)."""
        L = N.lib()
        cells = (C.c_int32 * 3)()
        ctf = tf._c() if tf is not None else None
        _check(L.svdbgpu_macrocells(self._h, C.byref(ctf) if ctf else None, cells, None, None, None,
                                    None, 0))
        n = cells[0] * cells[1] * cells[2]
        cmin = np.empty(n, np.float32); cmax = np.empty(n, np.float32)
        maj = np.zeros(n, np.float32); empty = np.ones(n, np.uint8)
        _check(L.svdbgpu_macrocells(self._h, C.byref(ctf) if ctf else None, cells, cmin.ctypes.data,
                                    cmax.ctypes.data, maj.ctypes.data if tf else None,
                                    empty.ctypes.data if tf else None, n))
        return tuple(cells), cmin, cmax, maj, empty

    def leaf_codes(self, first: int = 0, count: int | None = None):
        """Stored leaf payload (codes as laid out on the device) and per-leaf (lo, scale)."""
        n = self.counts["leaf"] - first if count is None else count
        stride = {Codec.f32: 2048, Codec.affine4: 256}.get(self.codec, 512)
        codes = np.empty((n, stride), np.uint8)
        params = np.zeros((n, 2), np.float32)
        _check(N.lib().svdbgpu_grid_leaf_codes(self._h, first, n, codes.ctypes.data, params.ctypes.data))
        return codes, params


def render(grid: DeviceGrid, tf: TransferFunction, cam: Camera, settings: RenderSettings,
           tile_rank: int = 0, tile_nranks: int = 1, out: np.ndarray | None = None) -> Image:
    """svdb::render (render.hpp:319-325) on the GPU: macrocell ranges (cached per grid),
    majorants for ``tf``, one path-tracing launch, image copied back to the host. ``out`` (optional,
    float32 [H, W, 3], C-contiguous; e.g. a pinned buffer for a full-speed device-to-host copy)
    receives the image instead of a new array."""
    if out is None:
        rgb = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
    else:
        if out.dtype != np.float32 or out.shape != (cam.height, cam.width, 3) or not out.flags.c_contiguous:
            raise Error(E_INVALID_ARG, "out must be a C-contiguous float32 [height, width, 3] array")
        rgb = out
    st = N.Stats()
    ctf, ccam, cst = tf._c(), cam._c(), settings._c(tile_rank, tile_nranks)
    _check(N.lib().svdbgpu_render(grid.handle, C.byref(ctf), C.byref(ccam), C.byref(cst),
                                  rgb.ctypes.data, C.byref(st)))
    return Image(cam.width, cam.height, rgb, _stats_dict(st))


def render_multi(grids: Sequence[DeviceGrid], tf: TransferFunction, cam: Camera, settings: RenderSettings) -> Image:
    """render() over several GPUs of this process (svdbgpu_render_multi): grids[k] is the same SVDB
    on a distinct device; interleaved 16x16 tiles per device, one NCCL gather to grids[0]'s device.
    The frame is bit-identical to render() on one device. stats gain ``gather_ms``."""
    rgb = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
    st = N.Stats()
    g_ms = C.c_double()
    hs = (C.c_void_p * len(grids))(*[g.handle for g in grids])
    ctf, ccam, cst = tf._c(), cam._c(), settings._c()
    _check(N.lib().svdbgpu_render_multi(hs, len(grids), C.byref(ctf), C.byref(ccam), C.byref(cst),
                                        rgb.ctypes.data, C.byref(st), C.byref(g_ms)))
    d = _stats_dict(st)
    d["gather_ms"] = g_ms.value
    return Image(cam.width, cam.height, rgb, d)


def nccl_version() -> int:
    """NCCL version code used by render_multi (0 and an Error if NCCL cannot be loaded)."""
    v = C.c_int32()
    _check(N.lib().svdbgpu_nccl_version(C.byref(v)))
    return v.value


def render_device(grid: DeviceGrid, tf: TransferFunction, cam: Camera, settings: RenderSettings,
                  out_ptr: int, stream_ptr: int = 0, packed: bool = False, tile_rank: int = 0,
                  tile_nranks: int = 1) -> dict:
    """Device-buffer render into ``out_ptr`` (e.g. a torch CUDA tensor's data_ptr())."""
    st = N.Stats()
    ctf, ccam, cst = tf._c(), cam._c(), settings._c(tile_rank, tile_nranks)
    _check(N.lib().svdbgpu_render_device(grid.handle, C.byref(ctf), C.byref(ccam), C.byref(cst),
                                         C.c_void_p(out_ptr), int(packed), C.c_void_p(stream_ptr),
                                         C.byref(st)))
    return _stats_dict(st)


def sample_device(grid: DeviceGrid, xyz_ptr: int, n: int, mode: int, out_ptr: int, stream_ptr: int = 0):
    """K2 on device buffers: n positions (3 x f64 each) -> n floats (mode 0 nearest, 1 trilinear)."""
    _check(N.lib().svdbgpu_sample_device(grid.handle, C.c_void_p(xyz_ptr), n, mode, C.c_void_p(out_ptr),
                                         C.c_void_p(stream_ptr)))


def tiles_for_rank(width: int, height: int, rank: int, nranks: int) -> int:
    return int(N.lib().svdbgpu_tiles_for_rank(width, height, rank, nranks))


def unpack_tiles_device(packed_ptr: int, nranks: int, max_tiles: int, width: int, height: int,
                        rgb_ptr: int, stream_ptr: int = 0):
    _check(N.lib().svdbgpu_unpack_tiles_device(C.c_void_p(packed_ptr), nranks, max_tiles, width,
                                               height, C.c_void_p(rgb_ptr), C.c_void_p(stream_ptr)))


def device_count() -> int:
    n = C.c_int32()
    rc = N.lib().svdbgpu_device_count(C.byref(n))
    return n.value if rc == 0 else 0
