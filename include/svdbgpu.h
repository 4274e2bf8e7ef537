/* svdbgpu.h — C-ABI of the B200-native compressed-VDB path tracer (libsvdbgpu.so).
 *
 * Drop-in boundary for the reference's hot path (svdb, /root/reference/proj/include/svdb).
 * The reference boundary is a C++ Field concept + entry points; a GPU cannot sit behind a
 * per-lookup host functor, so this ABI replaces the ENTRY POINTS:
 *
 *   svdbgpu_grid_create     <- parse_frozen()            io.hpp:183-256  (+ device upload / codec)
 *   svdbgpu_read_voxels     <- FrozenGrid::read_voxel    frozen.hpp:82-99 / Accessor::read 234-246
 *   svdbgpu_sample          <- sample(Accessor,p,mode)   sample.hpp:97-100 (nearest/trilinear 39-72)
 *   svdbgpu_gradient        <- gradient(Accessor,p)      sample.hpp:81-95, 102-105
 *   svdbgpu_macrocells      <- build_macrocells()+update_majorants() macrocell.hpp:74-116
 *   svdbgpu_render          <- render(grid,tf,cam,rs)    render.hpp:319-325 (render_field 276-315)
 *   svdbgpu_render_multi    <- render() with render_field's tile parallel_for (render.hpp:289-313)
 *                              spread over devices, one NCCL gather (SURVEY.md §8b ndev/devs, §8e)
 *   svdbgpu_compress        <- compress(volume,params)   compress.hpp:221-283 (host encoder)
 *   svdbgpu_quantise        <- serialize_frozen()        io.hpp:121-175 (+ quantised leaf section, new)
 *
 * Conventions: plain pointers and sizes only; every function returns 0 on success, svdb::Errc+1
 * (errors.hpp:11-23: 1 IoError .. 11 DimsMismatch) for the reference's own error classes, or one
 * of the SVDBGPU_E_* codes below. svdbgpu_last_error() gives the message (thread-local).
 * Host-buffer entry points copy to/from the device inside the call; *_device variants take
 * device pointers and a cudaStream_t passed as void*. Grids are immutable after creation and
 * may be shared by threads; every call is synchronous with respect to its outputs.
 */
#ifndef SVDBGPU_H
#define SVDBGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVDBGPU_ABI_VERSION 1

enum {
    SVDBGPU_OK = 0,
    /* 1..11 = svdb::Errc + 1 (io_error .. dims_mismatch) */
    SVDBGPU_E_CUDA = 64,        /* CUDA runtime failure (message has the cudaError string) */
    SVDBGPU_E_INVALID_ARG = 65, /* null pointer / bad enum / size */
    SVDBGPU_E_NO_DEVICE = 66,   /* no CUDA device visible: there is NO CPU fallback */
    SVDBGPU_E_OOM = 67,         /* device allocation failed */
    SVDBGPU_E_UNSUPPORTED = 68,
    SVDBGPU_E_NCCL = 69         /* NCCL missing or a collective failed (multi-device render) */
};

/* Leaf codecs of the device layout. */
enum {
    SVDBGPU_CODEC_F32 = 0,     /* 512 x f32 per leaf, the reference's values verbatim */
    SVDBGPU_CODEC_UNORM8 = 1,  /* 512 x u8, value = code/255.0f (exact for u8 sources) */
    SVDBGPU_CODEC_AFFINE8 = 2, /* 512 x u8, value = fmaf(code, scale, lo), per-leaf lo/scale */
    SVDBGPU_CODEC_AFFINE4 = 3, /* 512 x u4, value = fmaf(code, scale, lo), per-leaf lo/scale */
    SVDBGPU_CODEC_AUTO8 = 4    /* UNORM8 if every leaf is byte/255-exact, else AFFINE8 */
};

/* Render modes: the reference's two (render.hpp:34-37) + the north-star integrators. */
enum {
    SVDBGPU_MODE_PATHTRACE = 0, /* delta (Woodcock) tracking, reference draw order */
    SVDBGPU_MODE_ISO = 1,       /* interval iso-surface march (render.hpp:193-255) */
    SVDBGPU_MODE_EA = 2,        /* emission-absorption ray-march with the TF */
    SVDBGPU_MODE_RATIO = 3      /* multi-scatter path, ratio-tracked escape transmittance */
};

/* Tracking arithmetic. FP64 reproduces the reference bit for bit (render.hpp is FP64). The other
   two keep the reference's algorithm and per-pixel draw order: FP32 runs everything in single
   precision; MIXED keeps ray origins/directions, distances and the DDA in FP64 and runs the step
   log, uniforms, transfer function, trilinear weights and throughput in FP32. Both match the
   reference images within a tolerance instead of bit for bit. */
enum { SVDBGPU_PRECISION_FP64 = 0, SVDBGPU_PRECISION_FP32 = 1, SVDBGPU_PRECISION_MIXED = 2 };

/* Kernel variants for A/B measurement; both produce bit-identical images. */
enum { SVDBGPU_KERNEL_AUTO = 0, SVDBGPU_KERNEL_PER_PIXEL = 1 };

typedef struct svdbgpu_grid svdbgpu_grid;

/* TransferFunction (transfer.hpp:23-35): evenly spaced RGBA entries over [domain_lo, domain_hi]. */
typedef struct {
    double domain_lo, domain_hi, density_scale;
    int32_t n_entries;
    const float* rgba; /* n_entries x 4, host memory */
} svdbgpu_tf;

/* Camera (render.hpp:25-32) */
typedef struct {
    double position[3], look_at[3], up[3];
    double fov_y_deg;
    int32_t width, height;
} svdbgpu_camera;

/* RenderSettings (render.hpp:39-49) + north-star extensions. */
typedef struct {
    int32_t spp, max_bounces, rr_start_bounce;
    uint64_t seed;
    int32_t mode;            /* SVDBGPU_MODE_* */
    double iso_value;
    float ambient[3];        /* ambient_radiance */
    float background[3];     /* background_color */
    double ea_step;          /* EA: march step in voxels (default 0.5) */
    double ea_min_transmittance; /* EA: early-out threshold (default 1e-4) */
    int32_t tile_rank, tile_nranks; /* image split: 16x16 tiles t with t % nranks == rank */
    int32_t kernel;          /* SVDBGPU_KERNEL_*: 0 auto (path-regenerating tracer), 1 per-pixel */
    int32_t majorant_cell;   /* majorant grid cell edge: 0/32 = the reference's 32^3 macrocells
                                (bit-parity mode); 128 = lower-node, 8 = leaf-node majorants
                                (node-majorant tracking; statistically equal, different streams) */
    int32_t precision;       /* SVDBGPU_PRECISION_*: tracking arithmetic (pathtrace / ratio) */
    int32_t hdda;            /* 1: hierarchical DDA — empty 128^3 lower-node regions are skipped in one
                                coarse step, the majorant grid is walked inside non-empty ones
                                (pathtrace / ratio, FP64; statistically equal, different streams) */
} svdbgpu_settings;

typedef struct {
    uint64_t paths;      /* camera paths traced (pixels x spp of this rank) */
    uint64_t samples;    /* trilinear reconstructions performed */
    uint64_t lookups;    /* lattice taps delivered = 8 x samples (sample.hpp:56-63) */
    double render_ms;    /* render kernel time, CUDA events on the launch stream */
    double macrocell_ms; /* macrocell range build (0 when cached) + majorant update */
    uint32_t launches;   /* kernels launched by the call */
    uint32_t reserved;
} svdbgpu_stats;

typedef struct {
    int32_t dims[3];
    float background;
    int32_t voxel_type; /* 0 u8, 1 f32 (header field, io.hpp:27) */
    int32_t codec;      /* resolved SVDBGPU_CODEC_* */
    float value_domain[2];
    uint64_t n_upper, n_lower, n_leaf, n_root;
    uint64_t svdb_bytes;   /* FrozenLayout::total_bytes (frozen.hpp:62-67) */
    uint64_t device_bytes; /* resident device footprint of the tree */
    uint64_t leaf_payload_bytes;
    int32_t device;
    int32_t reserved;
} svdbgpu_grid_info;

typedef struct {
    float background;
    uint64_t num_bricks, bricks_activated, voxels_activated, frozen_bytes, dense_bytes;
    double achieved_ratio;
} svdbgpu_compress_report; /* CompressionReport (compress.hpp:87-95) */

/* ---- library ---- */
int svdbgpu_abi_version(void);
const char* svdbgpu_last_error(void);
int svdbgpu_device_count(int32_t* out);
void svdbgpu_free(void* p); /* frees buffers returned by svdbgpu_compress */

/* ---- grid ---- */
int svdbgpu_grid_create(const uint8_t* svdb, size_t n, int32_t codec, int32_t device,
                        svdbgpu_grid** out);
int svdbgpu_grid_destroy(svdbgpu_grid* g);
int svdbgpu_grid_info_get(const svdbgpu_grid* g, svdbgpu_grid_info* out);
/* Decoded leaf payload of one leaf (codes as stored, lo/scale) for codec parity checks. */
int svdbgpu_grid_leaf_codes(const svdbgpu_grid* g, uint64_t first, uint64_t count, uint8_t* codes,
                            float* params);

/* ---- lookups (host buffers) ---- */
int svdbgpu_read_voxels(const svdbgpu_grid* g, const int32_t* ijk, size_t n, float* out);
int svdbgpu_sample(const svdbgpu_grid* g, const double* xyz, size_t n, int32_t mode /*0 nearest,1 trilinear*/,
                   float* out);
int svdbgpu_gradient(const svdbgpu_grid* g, const double* xyz, size_t n, double* out);
/* ---- lookups (device buffers) ---- */
int svdbgpu_read_voxels_device(const svdbgpu_grid* g, const int32_t* d_ijk, size_t n, float* d_out,
                               void* stream);
int svdbgpu_sample_device(const svdbgpu_grid* g, const double* d_xyz, size_t n, int32_t mode,
                          float* d_out, void* stream);

/* ---- macrocells: exact closed-box ranges (cached per grid) + majorants for tf ---- */
int svdbgpu_macrocells(svdbgpu_grid* g, const svdbgpu_tf* tf, int32_t* cells3, float* cmin,
                       float* cmax, float* majorant, uint8_t* empty, size_t cap);

/* ---- render ----
 * svdbgpu_render: rgb_out is the host image W*H*3 float, row-major from the top row, linear
 * light (render.hpp:51-58). With tile_nranks > 1 only this rank's tiles are written.
 * svdbgpu_render_device: d_out is a device buffer; packed != 0 writes this rank's tiles
 * contiguously (tile k of the rank at d_out + k*16*16*3, pixels row-major inside the tile). */
int svdbgpu_render(svdbgpu_grid* g, const svdbgpu_tf* tf, const svdbgpu_camera* cam,
                   const svdbgpu_settings* s, float* rgb_out, svdbgpu_stats* stats);
int svdbgpu_render_device(svdbgpu_grid* g, const svdbgpu_tf* tf, const svdbgpu_camera* cam,
                          const svdbgpu_settings* s, float* d_out, int32_t packed, void* stream,
                          svdbgpu_stats* stats);
/* Multi-device render from one process: grids[k] holds the same SVDB on a
 * distinct device (svdbgpu_grid_create with that device id). Device k renders the interleaved
 * 16x16 tiles t with t % ndev == k into a packed buffer; ONE NCCL gather (grouped ncclSend/ncclRecv
 * over NVLink/NVSwitch) brings them to grids[0]'s device, which un-interleaves them; rgb_out is the
 * full host image W*H*3 as svdbgpu_render writes it, bit-identical for any ndev. settings->tile_*
 * must be 0/1 (the call does the split). stats: summed paths / samples / lookups / launches, max
 * render_ms and macrocell_ms over devices; *gather_ms (optional) = the gather's device time. NCCL
 * (libnccl.so.2) is loaded at first use; ndev > 1 without it fails with SVDBGPU_E_NCCL. */
int svdbgpu_render_multi(svdbgpu_grid* const* grids, int32_t ndev, const svdbgpu_tf* tf,
                         const svdbgpu_camera* cam, const svdbgpu_settings* s, float* rgb_out,
                         svdbgpu_stats* stats, double* gather_ms);
/* Version of the NCCL the multi-device render uses (ncclGetVersion code, e.g. 22803). */
int svdbgpu_nccl_version(int32_t* out);
/* Tiles owned by rank r of n for a W x H image. */
int64_t svdbgpu_tiles_for_rank(int32_t width, int32_t height, int32_t rank, int32_t nranks);
/* Un-interleave nranks packed buffers (each max_tiles*768 floats, back to back) into d_rgb. */
int svdbgpu_unpack_tiles_device(const float* d_packed, int32_t nranks, int64_t max_tiles,
                                int32_t width, int32_t height, float* d_rgb, void* stream);

/* ---- host encoder (compress.hpp:221-283), byte-identical SVDB v1 output ---- */
int svdbgpu_compress(const float* data, const int32_t dims[3], int32_t voxel_type, double quality,
                     int32_t metric /*0 closest,1 farthest,2 median*/, int32_t threads,
                     uint8_t** svdb_out, size_t* n_out, svdbgpu_compress_report* report);

/* ---- streaming device encoder: the same SVDB v1 bytes as svdbgpu_compress on
 * the dense volume, without a dense host array. The volume is streamed through `device` in z-slabs of
 * 32 slices (five passes: range + brick scan, histogram, exact background, block decisions, leaf
 * records); host memory holds only the output container and 5 B per 8^3 block.
 * svdbgpu_compress_stream: fn(user, z0, nz, out) fills slices [z0, z0+nz) (x fastest, dims[0]*dims[1]*nz
 * floats) and returns 0; it is called five times per slab, in slab order, and must return the same
 * values each time. svdbgpu_synth_compress: the svdbgpu_synth volumes of kind 1-3 generated on the
 * device (bit-identical to svdbgpu_synth). *seconds (optional) = encode wall time. *svdb_out is freed
 * with svdbgpu_free. */
typedef int (*svdbgpu_slab_fn)(void* user, int32_t z0, int32_t nz, float* out);
int svdbgpu_compress_stream(svdbgpu_slab_fn fn, void* user, const int32_t dims[3], int32_t voxel_type,
                            double quality, int32_t metric, int32_t device, uint8_t** svdb_out, size_t* n_out,
                            svdbgpu_compress_report* report, double* seconds);
int svdbgpu_synth_compress(int32_t kind, const int32_t dims[3], uint64_t seed, double quality, int32_t metric,
                           int32_t device, uint8_t** svdb_out, size_t* n_out, svdbgpu_compress_report* report,
                           double* seconds);

/* ---- quantised container: SVDB v1 -> "SVDB v2" with N-bit leaves ----
 * Same header / root / upper / lower sections as v1 (io.hpp:22-43) with version 2 and the codec in
 * the header's padding word (offset 68); each leaf record is {origin 3 x i32, pad, active mask 512
 * bits, lo f32, scale f32, codes (512 B UNORM8/AFFINE8, 256 B AFFINE4)} — 600 / 344 B instead of
 * 2128 B. The codes are the device codec's (a v2 file loads to exactly the grid svdbgpu_grid_create
 * builds from the v1 file with that codec). svdbgpu_grid_create accepts v2 with codec AUTO8 or the
 * stored codec. *out is freed with svdbgpu_free. */
int svdbgpu_quantise(const uint8_t* svdb, size_t n, int32_t codec, int32_t device, uint8_t** out, size_t* n_out);

/* ---- synthetic volumes (host, deterministic; x fastest) ----
 * kind 0 Marschner-Lobb (u8-quantised, values k/255), 1 fBm smoke (u8-quantised),
 * 2 ridged turbulence f32 in [0,1], 3 sparse thresholded fBm f32 (~35% leaves). */
int svdbgpu_synth(int32_t kind, const int32_t dims[3], uint64_t seed, int32_t threads, float* out);

#ifdef __cplusplus
}
#endif
#endif /* SVDBGPU_H */
