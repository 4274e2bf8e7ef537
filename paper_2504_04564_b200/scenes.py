"""The BASELINE.json workloads, as reusable scene definitions.

C1  64^3 Marschner-Lobb, u8 -> UNORM8, 512x512 emission-absorption, 1 spp, seed 1
C2  256^3 fBm smoke, u8 -> UNORM8, 1024x1024 delta tracking, single scattering, 16 spp, seed 2
C3  1024^3 ridged turbulence f32 -> AFFINE8 / AFFINE4, 1920x1080 multi-bounce, 64 spp, seed 3
C4  2048^3 sparse (~35% leaves) -> AFFINE8, 3840x2160 multi-scatter ratio tracking, 16 spp
C5  the C3 volume with F32 leaves (the reference's layout) vs AFFINE8

``scaled(name, f)`` shrinks a config by an integer factor for tests and bounded CPU samples while
keeping its transfer function, camera framing and integrator.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

from .api import Camera, Codec, RenderMode, RenderSettings, TransferFunction, VoxelType, frame_camera


@dataclass(frozen=True)
class Scene:
    name: str
    volume: str          # synth kind
    dims: tuple
    voxel_type: VoxelType
    volume_seed: int
    codec: Codec
    width: int
    height: int
    settings: RenderSettings
    tf: TransferFunction
    fov_y_deg: float = 45.0
    # camera = centre + distance * max_extent * normalize(view); (0,0,-1) at 2.2 is the CLI's
    # auto-framing (tools/svdb.cpp:267-274); the large configs move in so the volume fills the frame
    distance: float = 2.2
    view: tuple = (0.0, 0.0, -1.0)

    def camera(self) -> Camera:
        if self.distance == 2.2 and self.view == (0.0, 0.0, -1.0):
            return frame_camera(self.dims, self.width, self.height, self.fov_y_deg)
        ext = [float(d - 1) for d in self.dims]
        c = [e * 0.5 for e in ext]
        n = sum(v * v for v in self.view) ** 0.5
        r = self.distance * max(1.0, max(ext))
        pos = tuple(c[a] + r * self.view[a] / n for a in range(3))
        return Camera(position=pos, look_at=tuple(c), fov_y_deg=self.fov_y_deg, width=self.width,
                      height=self.height)


def _tf_ml():
    return TransferFunction(0.0, 1.0, [[0.0, 0.0, 0.0, 0.0], [0.1, 0.3, 0.9, 0.02],
                                       [0.2, 0.8, 0.6, 0.15], [0.9, 0.8, 0.2, 0.45],
                                       [1.0, 0.3, 0.1, 0.9]], density_scale=0.25)


def _tf_smoke(n):
    # alpha ramp 0 -> 1; mean free path ~0.1 N at the median density
    return TransferFunction(0.0, 1.0, [[0.85, 0.85, 0.9, 0.0], [0.9, 0.88, 0.85, 0.5],
                                       [0.95, 0.9, 0.8, 1.0]], density_scale=40.0 / n)


def _tf_turbulence(n):
    return TransferFunction(0.0, 1.0, [[0.8, 0.85, 0.95, 0.0], [0.8, 0.85, 0.95, 0.0],
                                       [0.9, 0.88, 0.85, 0.35], [0.95, 0.9, 0.8, 0.8],
                                       [1.0, 0.95, 0.9, 1.0]], density_scale=24.0 / n)


def _tf_sparse(n):
    return TransferFunction(0.0, 1.0, [[0.9, 0.9, 0.9, 0.0], [0.9, 0.85, 0.8, 0.6],
                                       [0.95, 0.9, 0.85, 1.0]], density_scale=48.0 / n)


_NEAR = dict(distance=1.3, view=(0.25, 0.2, -1.0))

SCENES = {
    "C1": Scene("C1", "marschner_lobb", (64, 64, 64), VoxelType.u8, 0, Codec.unorm8, 512, 512,
                RenderSettings(spp=1, seed=1, mode=RenderMode.ea, ea_step=0.5), _tf_ml(),
                distance=1.8, view=(0.3, 0.4, -1.0)),
    "C2": Scene("C2", "fbm_smoke", (256, 256, 256), VoxelType.u8, 2, Codec.unorm8, 1024, 1024,
                RenderSettings(spp=16, max_bounces=1, rr_start_bounce=3, seed=2), _tf_smoke(256),
                distance=1.6, view=(0.2, 0.3, -1.0)),
    "C3": Scene("C3", "turbulence", (1024, 1024, 1024), VoxelType.f32, 3, Codec.affine8, 1920, 1080,
                RenderSettings(spp=64, max_bounces=64, rr_start_bounce=3, seed=3), _tf_turbulence(1024),
                **_NEAR),
    "C3_4bit": Scene("C3_4bit", "turbulence", (1024, 1024, 1024), VoxelType.f32, 3, Codec.affine4,
                     1920, 1080, RenderSettings(spp=64, max_bounces=64, rr_start_bounce=3, seed=3),
                     _tf_turbulence(1024), **_NEAR),
    "C4": Scene("C4", "sparse", (2048, 2048, 2048), VoxelType.f32, 4, Codec.affine8, 3840, 2160,
                RenderSettings(spp=16, max_bounces=64, rr_start_bounce=3, seed=4, mode=RenderMode.ratio),
                _tf_sparse(2048), **_NEAR),
    "C5": Scene("C5", "turbulence", (1024, 1024, 1024), VoxelType.f32, 3, Codec.f32, 1920, 1080,
                RenderSettings(spp=64, max_bounces=64, rr_start_bounce=3, seed=3), _tf_turbulence(1024),
                **_NEAR),
}

_TF_BY_VOLUME = {"fbm_smoke": _tf_smoke, "turbulence": _tf_turbulence, "sparse": _tf_sparse}


def scaled(name: str, factor: int = 1, spp: int | None = None, image_factor: int | None = None,
           mode: RenderMode | None = None) -> Scene:
    """Config ``name`` with the volume shrunk by ``factor`` per axis (optical depth kept: the
    TF density scale follows the size) and the image by ``image_factor`` (default factor)."""
    s = SCENES[name]
    f = max(1, int(factor))
    fi = f if image_factor is None else max(1, int(image_factor))
    dims = tuple(max(8, d // f) for d in s.dims)
    tf = _TF_BY_VOLUME[s.volume](dims[0]) if s.volume in _TF_BY_VOLUME else s.tf
    st = replace(s.settings, spp=spp if spp is not None else s.settings.spp,
                 mode=mode if mode is not None else s.settings.mode)
    return replace(s, dims=dims, width=max(16, s.width // fi), height=max(16, s.height // fi),
                   settings=st, tf=tf)
