/* oracle/svdb_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference hot path (svdb, /root/reference/proj/include/svdb)
 * plus the north-star additions the reference lacks (N-bit leaf codec, emission-absorption
 * ray-march, ratio tracking). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the CHECKER. The product never links it.
 *
 * Parity pins:
 *   - reference-path functions are validated bit-exactly against the unmodified reference
 *     compiled in place (oracle/_ref/libsvdbref.so, see tests/test_oracle.py) and against the
 *     committed golden vectors in tests/golden/ (generated from that build by
 *     tests/golden/make_golden.py);
 *   - the codec / EA / ratio definitions have no reference implementation: "parity unpinned"
 *     by reference tests; they are pinned by analytic known-answer tests (Beer-Lambert,
 *     homogeneous-cube MC, delta-vs-ratio agreement) in tests/test_oracle.py.
 */
#ifndef SVDB_ORACLE_H
#define SVDB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct so_grid so_grid;

typedef struct {
    double domain_lo, domain_hi, density_scale;
    int n_entries;
    const float* rgba; /* n_entries x 4 */
} so_tf;

typedef struct {
    double position[3], look_at[3], up[3];
    double fov_y_deg;
    int width, height;
} so_camera;

enum { SO_PATHTRACE = 0, SO_ISO = 1, SO_EA = 2, SO_RATIO = 3 };

typedef struct {
    int spp, max_bounces, rr_start_bounce;
    uint64_t seed;
    int mode;
    double iso_value;
    float ambient[3];
    float background[3];
    double ea_step;              /* EA march step in voxels */
    double ea_min_transmittance; /* EA early termination threshold */
    int tile_rank, tile_nranks;  /* interleaved 16x16 tiles: t % nranks == rank */
    int threads;                 /* 0 = all cores */
    int majorant_cell;           /* 0/32 reference macrocells; 8 / 128 node-majorant grids */
    int hdda;                    /* 1: hierarchical DDA (128^3 lower-node regions, then the majorant grid) */
} so_settings;

/* SVDB v1 container (io.hpp:22-43); returns 0 or Errc+1 (errors.hpp:11-23). */
int so_open(const uint8_t* bytes, size_t n, so_grid** out);
void so_close(so_grid* g);
void so_info(const so_grid* g, int* dims3, float* background, uint64_t* counts4);

int so_read_voxels(const so_grid* g, const int32_t* ijk, size_t n, float* out, int cached);
int so_sample(const so_grid* g, const double* xyz, size_t n, int mode, float* out);

int so_macrocells(const so_grid* g, const so_tf* tf, int* cells3, float* cmin, float* cmax,
                  float* maj, uint8_t* empty, size_t cap);

/* Renders the tiles selected by settings->tile_rank/tile_nranks into rgb (W*H*3). */
int so_render(const so_grid* g, const so_tf* tf, const so_camera* cam, const so_settings* s,
              float* rgb, uint64_t* lookups, uint64_t* paths);

/* N-bit leaf codec (new; no reference function). codec: 0 = f32 identity, 1 = unorm8
 * (byte/255.0f, exact for u8 sources), 2 = affine8, 3 = affine4. Writes a dequantised SVDB
 * (same topology, leaf values = decoded) into *out (malloc'd), codes (n_leaf*512 bytes,
 * one code per byte) and params (n_leaf*2 floats: lo, scale) if non-null. */
int so_quantize(const uint8_t* bytes, size_t n, int codec, uint8_t** out, size_t* n_out,
                uint8_t* codes, float* params);
float so_decode(int codec, int code, float lo, float scale);

/* RNG (rng.hpp:12-67). */
uint64_t so_mix64(uint64_t x);
void so_rng_uniforms(uint64_t seed, int px, int py, int s, size_t n, double* out);

/* Synthetic volumes (synth_oracle.c), bit-identical to svdbgpu_synth: dense f32, x fastest. */
int so_synth(int kind, const int32_t dims[3], uint64_t seed, int threads, float* out);
/* Sparse field (kind 3) size calibration: per-8^3-block max of the pre-threshold density, and the
 * threshold used at a given max dimension. */
int so_sparse_block_max(const int32_t dims[3], uint64_t seed, int threads, double* block_max);
double so_sparse_threshold(int dim_max);

void so_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
