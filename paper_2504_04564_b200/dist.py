"""Multi-GPU image split: the volume is replicated on every rank, the frame is
split into interleaved 16x16 tiles (tile t = ty * tiles_x + tx belongs to rank t % nranks), each
rank renders its tiles into a packed buffer (tile k of the rank at k * 768 floats, pixels
row-major inside the tile) and ONE gather brings the packed buffers to rank 0, which
un-interleaves them. Paths are independent and keyed per (pixel, sample), so the assembled frame
is bit-identical for any rank count.

The device un-interleave is ``svdbgpu_unpack_tiles_device`` (render.cu k_unpack); the numpy
``pack_tiles`` / ``unpack_tiles`` here state the same layout for host-side use and tests.
"""
from __future__ import annotations

import numpy as np

TILE = 16


def tiles_x(width: int) -> int:
    return (width + TILE - 1) // TILE


def tile_ids(width: int, height: int, rank: int, nranks: int) -> np.ndarray:
    total = tiles_x(width) * ((height + TILE - 1) // TILE)
    return np.arange(rank, total, nranks, dtype=np.int64)


def max_tiles(width: int, height: int, nranks: int) -> int:
    return len(tile_ids(width, height, 0, nranks))


def pack_tiles(rgb: np.ndarray, rank: int, nranks: int, pad_to: int | None = None) -> np.ndarray:
    """rgb[H, W, 3] -> this rank's packed tiles [(pad_to or n_tiles) * 256 * 3]."""
    h, w, _ = rgb.shape
    ids = tile_ids(w, h, rank, nranks)
    n = len(ids) if pad_to is None else pad_to
    out = np.zeros((n, TILE, TILE, 3), np.float32)
    tx = tiles_x(w)
    for k, t in enumerate(ids):
        y0, x0 = (t // tx) * TILE, (t % tx) * TILE
        blk = rgb[y0:y0 + TILE, x0:x0 + TILE]
        out[k, :blk.shape[0], :blk.shape[1]] = blk
    return out.reshape(-1)


def unpack_tiles(packed_all: np.ndarray, nranks: int, n_max: int, width: int, height: int) -> np.ndarray:
    """Concatenated packed buffers of ranks 0..n-1 (each n_max tiles) -> rgb[H, W, 3]."""
    p = np.asarray(packed_all, np.float32).reshape(nranks, n_max, TILE, TILE, 3)
    out = np.zeros((height, width, 3), np.float32)
    tx = tiles_x(width)
    total = tx * ((height + TILE - 1) // TILE)
    for t in range(total):
        r, k = t % nranks, t // nranks
        y0, x0 = (t // tx) * TILE, (t % tx) * TILE
        hh, ww = min(TILE, height - y0), min(TILE, width - x0)
        out[y0:y0 + hh, x0:x0 + ww] = p[r, k, :hh, :ww]
    return out


def gather_packed(packed, world: int, rank: int):
    """The single collective: gather every rank's packed tile buffer (torch tensor, equal sizes)
    to rank 0. NCCL over NVLink on CUDA tensors, gloo on CPU tensors. Returns the concatenated
    buffer on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return packed
    if rank == 0:
        bufs = [torch.empty_like(packed) for _ in range(world)]
        dist.gather(packed, gather_list=bufs, dst=0)
        return torch.cat(bufs)
    dist.gather(packed, dst=0)
    return None
