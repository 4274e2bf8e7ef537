"""B200-native compressed-VDB volume path tracer (arXiv 2504.04564 hot path).

The product is libsvdbgpu.so (hand-written sm_100a CUDA + C++ host, C-ABI in include/svdbgpu.h);
this package is its host-side Python mirror of the reference svdb API.
"""
from .api import (  # noqa: F401
    Camera, Codec, CompressionParams, CompressionReport, DeviceGrid, Errc, Error, Image, Metric,
    RenderMode, RenderSettings, TransferFunction, VoxelType, compress, device_count, frame_camera,
    compress_stream, nccl_version, quantise, render, render_device, render_multi, sample_device, synth,
    synth_compress, tiles_for_rank, unpack_tiles_device,
)
