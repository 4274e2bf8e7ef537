"""Randomised parity sweep: small random grids (voxels, leaf tiles, upper-level tiles, random
background), random transfer functions, cameras (outside, inside, grazing) and settings, rendered
on the B200 and by the unmodified reference (pathtrace / iso) or the C restatement (ea / ratio),
plus random sample positions through the sampler. Seeds are fixed, so failures reproduce."""
import os

import numpy as np
import pytest

import paper_2504_04564_b200 as P
from helpers import MIN_IDENTICAL, SplitMix, bits, image_parity

pytestmark = pytest.mark.gpu

MODES = [P.RenderMode.pathtrace, P.RenderMode.iso, P.RenderMode.ea, P.RenderMode.ratio]


def _random_case(ref, seed):
    r = SplitMix(seed)
    dims = tuple(8 + int(r.uniform() * 90) for _ in range(3))
    background = float(np.float32(r.uniform() * 0.4)) if r.uniform() < 0.5 else 0.0
    ops = []
    for _ in range(200 + int(r.uniform() * 4000)):
        c = tuple(int(r.uniform() * d) for d in dims)
        ops.append((0, c, float(np.float32(r.uniform()))))
    for _ in range(int(r.uniform() * 30)):
        o = tuple(8 * int(r.uniform() * max(1, d // 8)) for d in dims)
        ops.append((1, o, float(np.float32(r.uniform()))))
    svdb = ref.build_ops(dims, background, ops)
    n = 2 + int(r.uniform() * 6)
    ent = [[float(np.float32(r.uniform())) for _ in range(3)] + [float(np.float32(r.uniform()))] for _ in range(n)]
    tf = P.TransferFunction(0.0, float(np.float32(0.5 + r.uniform())), ent, 0.01 + r.uniform() * 0.2)
    centre = tuple((d - 1) / 2 for d in dims)
    kind = r.uniform()
    if kind < 0.6:   # outside
        pos = tuple(c + (r.uniform() - 0.5) * 4 * max(dims) for c in centre)
    elif kind < 0.8:  # inside
        pos = tuple(c + (r.uniform() - 0.5) * 0.8 * d for c, d in zip(centre, dims))
    else:            # grazing: along a face
        pos = (centre[0], -0.5 * dims[1], centre[2] + (r.uniform() - 0.5))
    look = tuple(c + (r.uniform() - 0.5) * d for c, d in zip(centre, dims))
    cam = P.Camera(position=pos, look_at=look, fov_y_deg=20 + r.uniform() * 60,
                   width=8 + int(r.uniform() * 40), height=8 + int(r.uniform() * 40))
    mode = MODES[int(r.uniform() * 4)]
    st = P.RenderSettings(spp=1 + int(r.uniform() * 8), seed=int(r.uniform() * 1e9), mode=mode,
                          max_bounces=int(r.uniform() * 8), rr_start_bounce=int(r.uniform() * 4),
                          iso_value=r.uniform() * 0.8, ambient_radiance=(0.6, 0.8, 1.0),
                          background_color=(0.1, 0.2, 0.3))
    return svdb, tf, cam, st


@pytest.mark.parametrize("seed", range(int(os.environ.get("SVDB_RANDOM_SEEDS", "24"))))  # wider sweeps: env
def test_random_scene_parity(gpu, ref, orc, seed):
    svdb, tf, cam, st = _random_case(ref, 1000 + seed)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    img = P.render(g, tf, cam, st).pixels
    if st.mode in (P.RenderMode.pathtrace, P.RenderMode.iso):
        want = ref.open(svdb).render(tf, cam, st)
    else:
        want, _, _ = orc.open(svdb).render(tf, cam, st)
    same, rmse = image_parity(img, want)
    print(f"seed {seed} {st.mode.name} {cam.width}x{cam.height} spp {st.spp}: identical {same:.4f} rmse {rmse:.2e}")
    assert rmse <= 1e-3 and same >= MIN_IDENTICAL


@pytest.mark.parametrize("seed", range(6))
def test_random_samples_bit_exact(gpu, ref, seed):
    svdb, _, _, _ = _random_case(ref, 5000 + seed)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    rng = np.random.default_rng(seed)
    dims = np.array(g.dims, np.float64)
    xyz = rng.uniform(-2.0, dims + 2.0, (20000, 3))  # inside, on and beyond the box faces
    got = g.sample(xyz)
    want = ref.open(svdb).sample(xyz)
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("seed", range(int(os.environ.get("SVDB_RANDOM_QSEEDS", "8"))))
def test_random_quantised_scene_parity(gpu, ref, orc, seed):
    # N-bit leaves: the oracle image is the reference on the dequantised SVDB
    svdb, tf, cam, st = _random_case(ref, 3000 + seed)
    codec = P.Codec.affine8 if seed % 2 == 0 else P.Codec.affine4
    g = P.DeviceGrid(svdb, codec)
    deq, _, _ = orc.quantize(svdb, int(codec))
    img = P.render(g, tf, cam, st).pixels
    if st.mode in (P.RenderMode.pathtrace, P.RenderMode.iso):
        want = ref.open(deq).render(tf, cam, st)
    else:
        want, _, _ = orc.open(deq).render(tf, cam, st)
    same, rmse = image_parity(img, want)
    print(f"seed {seed} {codec.name} {st.mode.name}: identical {same:.4f} rmse {rmse:.2e}")
    assert rmse <= 1e-3 and same >= MIN_IDENTICAL
