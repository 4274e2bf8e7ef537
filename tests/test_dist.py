"""CPU multi-process (gloo, world_size 2 and 3) coverage of the multi-GPU image split:
interleaved 16x16 tiles, packed per-rank buffers, ONE gather to rank 0, un-interleave.
The per-rank renderer here is the CPU oracle (a stand-in with identical per-pixel semantics);
on the B200 box the same layout is produced by k_trace/k_render with packed output and
un-interleaved by k_unpack (tests/test_gpu_render.py::test_tile_split_is_bit_identical)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import dist as D
from paper_2504_04564_b200 import scenes as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, svdb, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = S.scaled("C2", 8, spp=2, image_factor=10)
    cam = sc.camera()
    img, _, _ = Oracle().open(svdb).render(sc.tf, cam, sc.settings, tile_rank=rank, tile_nranks=world, threads=2)
    n_max = D.max_tiles(cam.width, cam.height, world)
    packed = torch.from_numpy(D.pack_tiles(img, rank, world, pad_to=n_max))
    allp = D.gather_packed(packed, world, rank)
    if rank == 0:
        frame = D.unpack_tiles(allp.numpy(), world, n_max, cam.width, cam.height)
        np.save(out_path, frame)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_tile_split_gather_is_bit_identical(tmp_path, orc, world):
    sc = S.scaled("C2", 8, spp=2, image_factor=10)
    vol = P.synth(sc.volume, sc.dims, sc.volume_seed)
    svdb, _ = P.compress(vol, voxel_type=sc.voxel_type)
    out = str(tmp_path / "frame.npy")
    mp.start_processes(_worker, args=(world, _free_port(), svdb, out), nprocs=world, join=True,
                       start_method="spawn")
    frame = np.load(out)
    full, _, _ = orc.open(svdb).render(sc.tf, sc.camera(), sc.settings)
    assert np.array_equal(frame.view(np.uint32), full.view(np.uint32))


def test_tile_layout_matches_native_partition():
    for (w, h, n) in [(1920, 1080, 8), (100, 37, 3), (16, 16, 2)]:
        assert sum(len(D.tile_ids(w, h, r, n)) for r in range(n)) == D.tiles_x(w) * ((h + 15) // 16)
        for r in range(n):
            assert len(D.tile_ids(w, h, r, n)) == P.tiles_for_rank(w, h, r, n)
    rgb = np.random.default_rng(0).random((37, 100, 3)).astype(np.float32)
    n = 3
    m = D.max_tiles(100, 37, n)
    allp = np.concatenate([D.pack_tiles(rgb, r, n, pad_to=m) for r in range(n)])
    assert np.array_equal(D.unpack_tiles(allp, n, m, 100, 37), rgb)


def _bench(*argv, env=None):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *argv], capture_output=True, text=True,
                       env=e, timeout=600)
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    return p.returncode, (json.loads(lines[-1]) if lines else None), p.stderr


@pytest.mark.parametrize("n", [2, 3])
def test_bench_gpus_flag_spawns_ranks(n):
    # `bench.py --gpus N` without a launcher re-runs itself under torch.distributed.run with N ranks;
    # the CPU check drives the same rank wiring, encode-once sharing and product gather over gloo
    rc, line, err = _bench("--gpus", str(n), "--cpu-check")
    assert rc == 0, err[-2000:]
    assert line["world"] == n and line["n_gpus"] == n and line["backend"] == "gloo"
    assert line["bit_identical"]


def test_bench_rejects_gpus_world_mismatch():
    rc, line, err = _bench("--gpus", "2", "--cpu-check", env={"WORLD_SIZE": "1", "RANK": "0"})
    assert rc == 2 and line is None and "WORLD_SIZE" in err


def test_reference_arm_never_loads_the_product_library():
    # --impl reference builds its input with the oracle's synth + the reference's compress and times
    # the stock render body: libsvdbgpu.so must not be mapped (perf anchor voided)
    from oracle.oracle import have_reference
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    rc, line, err = _bench("--impl", "reference", "--config", "C2", "--scale", "4", "--width", "64",
                           "--height", "48", "--steps", "1", "--warmup", "0")
    assert rc == 0, err[-2000:]
    assert line["impl"] == "reference" and line["value"] > 0
    assert not any("libsvdbgpu" in p for p in line["native_so_loaded"])
    assert any("libsvdbref" in p for p in line["native_so_loaded"])
