/* oracle/svdb_oracle.c — TEST INFRASTRUCTURE ONLY (see svdb_oracle.h).
 *
 * CPU restatement, in plain C, of the reference svdb hot path. Every function cites the
 * reference file:line it restates (paths under /root/reference/proj/include/svdb/).
 * Compiled with -ffp-contract=off so double expressions round exactly like the reference's
 * x86-64 Release build (no FMA contraction, SSE2 doubles).
 */
#define _GNU_SOURCE
#include "svdb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ---- layout constants: tree.hpp:25-41, frozen.hpp:52-60, io.hpp:22-43 ---- */
#define UPPER_SLOTS 32768
#define LOWER_SLOTS 4096
#define LEAF_VOXELS 512
#define HDR_BYTES 72ull
#define ROOT_BYTES 16ull
#define UPPER_BYTES (16ull + 4ull * UPPER_SLOTS + 2ull * (UPPER_SLOTS / 8))
#define LOWER_BYTES (16ull + 4ull * LOWER_SLOTS + 2ull * (LOWER_SLOTS / 8))
#define LEAF_BYTES (16ull + LEAF_VOXELS / 8 + 4ull * LEAF_VOXELS)

/* Errc (errors.hpp:11-23) + 1 */
enum { E_IO = 1, E_SIZE, E_NONFINITE, E_OOB, E_MISALIGNED, E_EMPTYBOX, E_QUALITY, E_MAGIC,
       E_VERSION, E_CORRUPT, E_DIMS };

struct so_grid {
    const uint8_t* base; /* owned copy */
    size_t size;
    int dims[3];
    float background;
    uint64_t n_upper, n_lower, n_leaf, n_root;
    const uint8_t *root, *upper, *lower, *leaf;
};

static inline uint32_t rd_u32(const uint8_t* p) { uint32_t v; memcpy(&v, p, 4); return v; }
static inline int32_t rd_i32(const uint8_t* p) { int32_t v; memcpy(&v, p, 4); return v; }
static inline uint64_t rd_u64(const uint8_t* p) { uint64_t v; memcpy(&v, p, 8); return v; }
static inline float rd_f32(const uint8_t* p) { float v; memcpy(&v, p, 4); return v; }

/* BitMask::test (tree.hpp:94): LSB-first u64 words */
static inline int mask_test(const uint8_t* words, int i) { return (int)((rd_u64(words + 8 * (i >> 6)) >> (i & 63)) & 1u); }

/* node record accessors (io.hpp:33-39) */
static inline const uint8_t* upper_rec(const so_grid* g, uint64_t i) { return g->upper + i * UPPER_BYTES; }
static inline const uint8_t* lower_rec(const so_grid* g, uint64_t i) { return g->lower + i * LOWER_BYTES; }
static inline const uint8_t* leaf_rec(const so_grid* g, uint64_t i) { return g->leaf + i * LEAF_BYTES; }
#define REC_PAYLOAD 16
#define UPPER_CHILD (16 + 4 * UPPER_SLOTS)
#define UPPER_TILE (UPPER_CHILD + UPPER_SLOTS / 8)
#define LOWER_CHILD (16 + 4 * LOWER_SLOTS)
#define LOWER_TILE (LOWER_CHILD + LOWER_SLOTS / 8)
#define LEAF_VALUES (16 + LEAF_VOXELS / 8)

/* parse_frozen (io.hpp:183-256) */
int so_open(const uint8_t* bytes, size_t n, so_grid** out)
{
    *out = NULL;
    if (n < 4) return E_CORRUPT;
    if (memcmp(bytes, "SVDB", 4) != 0) return E_MAGIC;
    if (n < HDR_BYTES) return E_CORRUPT;
    if (rd_u32(bytes + 4) != 1) return E_VERSION;
    if (rd_u32(bytes + 8) > 1) return E_CORRUPT;
    int d[3] = {(int)rd_u32(bytes + 12), (int)rd_u32(bytes + 16), (int)rd_u32(bytes + 20)};
    if (d[0] < 1 || d[1] < 1 || d[2] < 1) return E_CORRUPT;
    uint64_t nu = rd_u64(bytes + 36), nl = rd_u64(bytes + 44), nf = rd_u64(bytes + 52), nr = rd_u64(bytes + 60);
    const uint64_t lim = 1ull << 32;
    if (nu > lim || nl > lim || nf > lim || nr > lim) return E_CORRUPT;
    if (HDR_BYTES + ROOT_BYTES * nr + UPPER_BYTES * nu + LOWER_BYTES * nl + LEAF_BYTES * nf != n) return E_CORRUPT;
    so_grid* g = (so_grid*)calloc(1, sizeof(so_grid));
    uint8_t* copy = (uint8_t*)malloc(n);
    memcpy(copy, bytes, n);
    g->base = copy;
    g->size = n;
    memcpy(g->dims, d, sizeof d);
    g->background = rd_f32(bytes + 24);
    g->n_upper = nu; g->n_lower = nl; g->n_leaf = nf; g->n_root = nr;
    g->root = copy + HDR_BYTES;
    g->upper = g->root + ROOT_BYTES * nr;
    g->lower = g->upper + UPPER_BYTES * nu;
    g->leaf = g->lower + LOWER_BYTES * nl;
    for (uint64_t i = 0; i < nr; ++i)
        if (rd_u32(g->root + 16 * i + 12) >= nu) { so_close(g); return E_CORRUPT; }
    for (uint64_t i = 0; i < nu; ++i) {
        const uint8_t* r = upper_rec(g, i);
        for (int s = 0; s < UPPER_SLOTS; ++s)
            if (mask_test(r + UPPER_CHILD, s) && rd_u32(r + REC_PAYLOAD + 4 * s) >= nl) { so_close(g); return E_CORRUPT; }
    }
    for (uint64_t i = 0; i < nl; ++i) {
        const uint8_t* r = lower_rec(g, i);
        for (int s = 0; s < LOWER_SLOTS; ++s)
            if (mask_test(r + LOWER_CHILD, s) && rd_u32(r + REC_PAYLOAD + 4 * s) >= nf) { so_close(g); return E_CORRUPT; }
    }
    *out = g;
    return 0;
}

void so_close(so_grid* g)
{
    if (!g) return;
    free((void*)g->base);
    free(g);
}

void so_info(const so_grid* g, int* dims3, float* background, uint64_t* counts4)
{
    memcpy(dims3, g->dims, 12);
    *background = g->background;
    counts4[0] = g->n_upper; counts4[1] = g->n_lower; counts4[2] = g->n_leaf; counts4[3] = g->n_root;
}

/* TreeConfig slot math (tree.hpp:43-71) */
static inline int upper_slot(int x, int y, int z) { return ((x >> 7) & 31) + 32 * (((y >> 7) & 31) + 32 * ((z >> 7) & 31)); }
static inline int lower_slot(int x, int y, int z) { return ((x >> 3) & 15) + 16 * (((y >> 3) & 15) + 16 * ((z >> 3) & 15)); }
static inline int leaf_voxel(int x, int y, int z) { return (x & 7) + 8 * ((y & 7) + 8 * (z & 7)); }

/* CoordZyxLess (vec.hpp:140-149) */
static inline int zyx_less(int ax, int ay, int az, int bx, int by, int bz)
{
    if (az != bz) return az < bz;
    if (ay != by) return ay < by;
    return ax < bx;
}

/* FrozenGrid::find_upper (frozen.hpp:101-110): lower_bound over the zyx-sorted root */
static const uint8_t* find_upper(const so_grid* g, int ox, int oy, int oz)
{
    /* std::lower_bound probe order (libstdc++), so unsorted roots resolve identically */
    uint64_t lo = 0, len = g->n_root;
    while (len > 0) {
        uint64_t half = len >> 1;
        const uint8_t* e = g->root + 16 * (lo + half);
        if (zyx_less(rd_i32(e), rd_i32(e + 4), rd_i32(e + 8), ox, oy, oz)) { lo = lo + half + 1; len = len - half - 1; }
        else len = half;
    }
    if (lo == g->n_root) return NULL;
    const uint8_t* e = g->root + 16 * lo;
    if (rd_i32(e) != ox || rd_i32(e + 4) != oy || rd_i32(e + 8) != oz) return NULL;
    return upper_rec(g, rd_u32(e + 12));
}

static inline float bits_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* read from a lower record (frozen.hpp:94-98 / 262-271): tile bit before child bit */
static inline float read_lower(const so_grid* g, const uint8_t* lr, int x, int y, int z, const uint8_t** leaf_out)
{
    int ls = lower_slot(x, y, z);
    if (mask_test(lr + LOWER_TILE, ls)) return bits_f32(rd_u32(lr + REC_PAYLOAD + 4 * ls));
    if (!mask_test(lr + LOWER_CHILD, ls)) return g->background;
    const uint8_t* lf = leaf_rec(g, rd_u32(lr + REC_PAYLOAD + 4 * ls));
    if (leaf_out) *leaf_out = lf;
    return rd_f32(lf + LEAF_VALUES + 4 * leaf_voxel(x, y, z));
}

static inline float read_upper(const so_grid* g, const uint8_t* ur, int x, int y, int z,
                               const uint8_t** lower_out, const uint8_t** leaf_out)
{
    int us = upper_slot(x, y, z);
    if (mask_test(ur + UPPER_TILE, us)) return bits_f32(rd_u32(ur + REC_PAYLOAD + 4 * us));
    if (!mask_test(ur + UPPER_CHILD, us)) return g->background;
    const uint8_t* lr = lower_rec(g, rd_u32(ur + REC_PAYLOAD + 4 * us));
    if (lower_out) *lower_out = lr;
    return read_lower(g, lr, x, y, z, leaf_out);
}

/* FrozenGrid::read_voxel (frozen.hpp:82-99) */
static float read_voxel(const so_grid* g, int x, int y, int z)
{
    const uint8_t* ur = find_upper(g, x & ~4095, y & ~4095, z & ~4095);
    if (!ur) return g->background;
    return read_upper(g, ur, x, y, z, NULL, NULL);
}

/* Accessor (frozen.hpp:228-277): node caches keyed on origin equality */
typedef struct {
    const so_grid* g;
    const uint8_t *upper, *lower, *leaf;
    uint64_t reads;
} acc_t;

static inline int rec_origin_is(const uint8_t* rec, int x, int y, int z)
{
    return rd_i32(rec) == x && rd_i32(rec + 4) == y && rd_i32(rec + 8) == z;
}

static float acc_read(acc_t* a, int x, int y, int z)
{
    a->reads++;
    if (a->leaf && rec_origin_is(a->leaf, x & ~7, y & ~7, z & ~7))
        return rd_f32(a->leaf + LEAF_VALUES + 4 * leaf_voxel(x, y, z));
    if (a->lower && rec_origin_is(a->lower, x & ~127, y & ~127, z & ~127))
        return read_lower(a->g, a->lower, x, y, z, &a->leaf);
    if (a->upper && rec_origin_is(a->upper, x & ~4095, y & ~4095, z & ~4095))
        return read_upper(a->g, a->upper, x, y, z, &a->lower, &a->leaf);
    a->upper = find_upper(a->g, x & ~4095, y & ~4095, z & ~4095);
    if (!a->upper) return a->g->background;
    return read_upper(a->g, a->upper, x, y, z, &a->lower, &a->leaf);
}

int so_read_voxels(const so_grid* g, const int32_t* ijk, size_t n, float* out, int cached)
{
    acc_t a = {g, NULL, NULL, NULL, 0};
    for (size_t i = 0; i < n; ++i)
        out[i] = cached ? acc_read(&a, ijk[3 * i], ijk[3 * i + 1], ijk[3 * i + 2])
                        : read_voxel(g, ijk[3 * i], ijk[3 * i + 1], ijk[3 * i + 2]);
    return 0;
}

/* ---- sampler: sample.hpp:24-72 ---- */
static inline int lattice_coord(double v)
{
    double f = floor(v);
    if (f < -1.0e9) return -1000000000;
    if (f > 1.0e9) return 1000000000;
    return (int)f;
}

static float sample_trilinear(acc_t* a, double px, double py, double pz)
{
    int x0 = lattice_coord(px), y0 = lattice_coord(py), z0 = lattice_coord(pz);
    double wx = px - floor(px), wy = py - floor(py), wz = pz - floor(pz);
    double v000 = acc_read(a, x0, y0, z0);
    double v100 = acc_read(a, x0 + 1, y0, z0);
    double v010 = acc_read(a, x0, y0 + 1, z0);
    double v110 = acc_read(a, x0 + 1, y0 + 1, z0);
    double v001 = acc_read(a, x0, y0, z0 + 1);
    double v101 = acc_read(a, x0 + 1, y0, z0 + 1);
    double v011 = acc_read(a, x0, y0 + 1, z0 + 1);
    double v111 = acc_read(a, x0 + 1, y0 + 1, z0 + 1);
    double v00 = v000 * (1.0 - wx) + v100 * wx;
    double v10 = v010 * (1.0 - wx) + v110 * wx;
    double v01 = v001 * (1.0 - wx) + v101 * wx;
    double v11 = v011 * (1.0 - wx) + v111 * wx;
    double v0 = v00 * (1.0 - wy) + v10 * wy;
    double v1 = v01 * (1.0 - wy) + v11 * wy;
    return (float)(v0 * (1.0 - wz) + v1 * wz);
}

static float sample_nearest(acc_t* a, double px, double py, double pz)
{
    return acc_read(a, lattice_coord(px + 0.5), lattice_coord(py + 0.5), lattice_coord(pz + 0.5));
}

int so_sample(const so_grid* g, const double* xyz, size_t n, int mode, float* out)
{
    acc_t a = {g, NULL, NULL, NULL, 0};
    for (size_t i = 0; i < n; ++i)
        out[i] = mode == 0 ? sample_nearest(&a, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2])
                           : sample_trilinear(&a, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    return 0;
}

/* ---- transfer function: transfer.hpp:47-91 ---- */
static inline double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
static inline double dmax(double a, double b) { return a < b ? b : a; }
static inline double dmin(double a, double b) { return b < a ? b : a; }

static inline double tf_normalized(const so_tf* tf, double v)
{
    return dclamp((v - tf->domain_lo) / (tf->domain_hi - tf->domain_lo), 0.0, 1.0);
}

static void tf_lookup(const so_tf* tf, double v, double out[4])
{
    size_t n = (size_t)tf->n_entries;
    double u = tf_normalized(tf, v) * (double)(n - 1);
    size_t i0 = (size_t)u;
    if (n - 2 < i0) i0 = n - 2;
    double t = u - (double)i0;
    const float* a = tf->rgba + 4 * i0;
    const float* b = a + 4;
    for (int c = 0; c < 4; ++c) out[c] = (1.0 - t) * (double)a[c] + t * (double)b[c];
}

static inline double tf_alpha(const so_tf* tf, double v) { double c[4]; tf_lookup(tf, v, c); return c[3]; }
static inline double tf_extinction(const so_tf* tf, double v) { return tf->density_scale * tf_alpha(tf, v); }

static double tf_max_alpha_in_range(const so_tf* tf, double vlo, double vhi)
{
    if (vhi < vlo) { double t = vlo; vlo = vhi; vhi = t; }
    double m = dmax(tf_alpha(tf, vlo), tf_alpha(tf, vhi));
    double ulo = tf_normalized(tf, vlo), uhi = tf_normalized(tf, vhi);
    size_t n = (size_t)tf->n_entries;
    for (size_t i = 0; i < n; ++i) {
        double u = (double)i / (double)(n - 1);
        if (u > ulo && u < uhi) m = dmax(m, (double)tf->rgba[4 * i + 3]);
    }
    return m;
}

/* ---- macrocells: macrocell.hpp:29-116 ---- */
typedef struct {
    int cells[3];
    int dims[3];
    int cell; /* edge in voxels: 32 = the reference's kMacrocellSize (macrocell.hpp:29); 8/128 =
                 leaf/lower-node majorant grids (north-star node-majorant mode) */
    float *cmin, *cmax, *maj;
    uint8_t* empty;
    /* hierarchical DDA (NEW, north-star "empty-space skipping is a hierarchical DDA over the node
       tree"): coarse cells = 128^3 lower-node regions, cdraw[c] = some majorant-grid cell inside has
       a positive float majorant; NULL when the flat DDA is used */
    int ccells[3];
    uint8_t* cdraw;
} mc_t;

static inline int cell_count_axis(int d, int cd) { int n = (d - 1 + cd - 1) / cd; return n < 1 ? 1 : n; }

typedef struct {
    const so_grid* g;
    const so_tf* tf;
    mc_t* mc;
    atomic_long next;
} mc_job_t;

static void mc_cell(const so_grid* g, const so_tf* tf, mc_t* mc, size_t i)
{
    const int cd = mc->cell;
    int cx = (int)(i % mc->cells[0]), cy = (int)((i / mc->cells[0]) % mc->cells[1]),
        cz = (int)(i / ((size_t)mc->cells[0] * mc->cells[1]));
    int lo[3] = {cx * cd, cy * cd, cz * cd};
    int c3[3] = {cx, cy, cz}, hi[3];
    for (int a = 0; a < 3; ++a) { int h = (c3[a] + 1) * cd; hi[a] = h < g->dims[a] - 1 ? h : g->dims[a] - 1; }
    acc_t acc = {g, NULL, NULL, NULL, 0};
    float mn = INFINITY, mx = -INFINITY;
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x) {
                float v = acc_read(&acc, x, y, z);
                mn = v < mn ? v : mn;
                mx = mx < v ? v : mx;
            }
    mc->cmin[i] = mn; mc->cmax[i] = mx;
    if (tf) {
        double m = tf->density_scale * tf_max_alpha_in_range(tf, mn, mx);
        mc->maj[i] = (float)m;
        mc->empty[i] = m == 0.0 ? 1 : 0;
    } else {
        mc->maj[i] = 0.0f; mc->empty[i] = 1;
    }
}

static void* mc_worker(void* arg)
{
    mc_job_t* J = (mc_job_t*)arg;
    size_t nc = (size_t)J->mc->cells[0] * J->mc->cells[1] * J->mc->cells[2];
    for (;;) {
        long i = atomic_fetch_add(&J->next, 1);
        if ((size_t)i >= nc) break;
        mc_cell(J->g, J->tf, J->mc, (size_t)i);
    }
    return NULL;
}

/* build_macrocells + update_majorants (macrocell.hpp:74-116), cells in parallel (independent) */
static void mc_build(const so_grid* g, const so_tf* tf, int cd, mc_t* mc)
{
    mc->cell = cd;
    for (int a = 0; a < 3; ++a) { mc->dims[a] = g->dims[a]; mc->cells[a] = cell_count_axis(g->dims[a], cd); }
    size_t nc = (size_t)mc->cells[0] * mc->cells[1] * mc->cells[2];
    mc->cmin = (float*)malloc(nc * 4); mc->cmax = (float*)malloc(nc * 4);
    mc->maj = (float*)malloc(nc * 4); mc->empty = (uint8_t*)malloc(nc);
    mc_job_t J;
    J.g = g; J.tf = tf; J.mc = mc;
    atomic_init(&J.next, 0);
    int nt = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if ((size_t)nt > nc) nt = (int)nc;
    if (nt > 256) nt = 256;
    pthread_t th[256];
    for (int i = 1; i < nt; ++i) pthread_create(&th[i], NULL, mc_worker, &J);
    mc_worker(&J);
    for (int i = 1; i < nt; ++i) pthread_join(th[i], NULL);
}

static void mc_free(mc_t* mc) { free(mc->cmin); free(mc->cmax); free(mc->maj); free(mc->empty); free(mc->cdraw); }

#define COARSE_CELL 128
/* coarse flags of the hierarchical DDA over the majorant grid (cell must divide 128) */
static void mc_build_coarse(mc_t* mc)
{
    const int R = COARSE_CELL / mc->cell;
    for (int a = 0; a < 3; ++a) mc->ccells[a] = cell_count_axis(mc->dims[a], COARSE_CELL);
    size_t nc = (size_t)mc->ccells[0] * mc->ccells[1] * mc->ccells[2];
    mc->cdraw = (uint8_t*)calloc(nc ? nc : 1, 1);
    for (int z = 0; z < mc->cells[2]; ++z)
        for (int y = 0; y < mc->cells[1]; ++y)
            for (int x = 0; x < mc->cells[0]; ++x) {
                size_t i = (size_t)x + (size_t)mc->cells[0] * ((size_t)y + (size_t)mc->cells[1] * (size_t)z);
                if (mc->maj[i] > 0.0f)
                    mc->cdraw[(size_t)(x / R) + (size_t)mc->ccells[0] * ((size_t)(y / R) + (size_t)mc->ccells[1] * (size_t)(z / R))] = 1;
            }
}

static inline size_t mc_index(const mc_t* mc, const int c[3])
{
    return (size_t)c[0] + (size_t)mc->cells[0] * ((size_t)c[1] + (size_t)mc->cells[1] * (size_t)c[2]);
}

int so_macrocells(const so_grid* g, const so_tf* tf, int* cells3, float* cmin, float* cmax,
                  float* maj, uint8_t* empty, size_t cap)
{
    mc_t mc;
    mc_build(g, tf, 32, &mc);
    mc.cdraw = NULL;
    memcpy(cells3, mc.cells, 12);
    size_t nc = (size_t)mc.cells[0] * mc.cells[1] * mc.cells[2];
    if (cmin && nc <= cap) {
        memcpy(cmin, mc.cmin, nc * 4); memcpy(cmax, mc.cmax, nc * 4);
        memcpy(maj, mc.maj, nc * 4); memcpy(empty, mc.empty, nc);
    }
    mc_free(&mc);
    return 0;
}

/* ---- rng: rng.hpp:12-67 ---- */
uint64_t so_mix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

typedef struct { uint64_t state; } rng_t;

static inline rng_t rng_for_pixel_sample(uint64_t seed, int px, int py, int s)
{
    uint64_t h = so_mix64(seed);
    h = so_mix64(h ^ (((uint64_t)(uint32_t)px << 32) | (uint32_t)py));
    h = so_mix64(h ^ (uint64_t)(uint32_t)s);
    rng_t r = {so_mix64(h)}; /* Rng(h): state = mix64(h) (rng.hpp:42) */
    return r;
}

static inline double rng_uniform(rng_t* r)
{
    r->state += 0x9E3779B97F4A7C15ull;
    uint64_t x = r->state;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return (double)(x >> 11) * 0x1.0p-53;
}

void so_rng_uniforms(uint64_t seed, int px, int py, int s, size_t n, double* out)
{
    rng_t r = rng_for_pixel_sample(seed, px, py, s);
    for (size_t i = 0; i < n; ++i) out[i] = rng_uniform(&r);
}

/* ---- rays / DDA: dda.hpp:15-109 ---- */
typedef struct { double o[3], d[3]; } ray_t;

static inline void ray_at(const ray_t* r, double t, double p[3])
{
    for (int a = 0; a < 3; ++a) p[a] = r->o[a] + r->d[a] * t;
}

static int clip_ray_box(const ray_t* r, const double lo[3], const double hi[3], double* t0, double* t1)
{
    for (int a = 0; a < 3; ++a) {
        double o = r->o[a], d = r->d[a];
        if (d == 0.0) {
            if (o < lo[a] || o > hi[a]) return 0;
            continue;
        }
        double inv = 1.0 / d;
        double ta = (lo[a] - o) * inv, tb = (hi[a] - o) * inv;
        if (ta > tb) { double t = ta; ta = tb; tb = t; }
        *t0 = dmax(*t0, ta);
        *t1 = dmin(*t1, tb);
        if (*t0 > *t1) return 0;
    }
    return 1;
}

/* Incremental Amanatides-Woo state; dda_next returns 0 when traversal ends. */
typedef struct {
    int c[3], step[3];
    double t_next[3], t_delta[3], t_cur, t1;
    int done;
    int last_axis; /* axis stepped after the last visit (-1: the traversal ended there) */
    int lo[3], hi[3]; /* cell index range walked: the grid, or one HDDA region of it */
} dda_t;

static int dda_init_forced(const int dims[3], const int cells[3], int cell, const ray_t* r, double t0, double t1,
                           int force_axis, int force_cell, const int* clo, const int* chi, dda_t* s);
static int dda_init_cells(const int dims[3], const int cells[3], int cell, const ray_t* r, double t0, double t1,
                          dda_t* s)
{
    return dda_init_forced(dims, cells, cell, r, t0, t1, -1, 0, NULL, NULL, s);
}

/* dda_init over the cell range [clo, chi] (NULL: the whole grid) with the start cell on force_axis
   given (the hierarchical DDA's region entry face); the walk ends when it leaves the range */
static int dda_init_forced(const int dims[3], const int cells[3], int cell, const ray_t* r, double t0, double t1,
                           int force_axis, int force_cell, const int* clo, const int* chi, dda_t* s)
{
    for (int a = 0; a < 3; ++a) {
        s->lo[a] = clo ? clo[a] : 0;
        s->hi[a] = chi ? chi[a] : cells[a] - 1;
    }
    double lo[3] = {0, 0, 0};
    double hi[3] = {(double)(dims[0] - 1), (double)(dims[1] - 1), (double)(dims[2] - 1)};
    if (!clip_ray_box(r, lo, hi, &t0, &t1)) return 0;
    if (!(t0 <= t1)) return 0;
    double e[3], cs = (double)cell;
    ray_at(r, t0, e);
    for (int a = 0; a < 3; ++a) {
        s->c[a] = a == force_axis ? force_cell : (int)dclamp(floor(e[a] / cs), (double)s->lo[a], (double)s->hi[a]);
        s->step[a] = 0;
        s->t_next[a] = INFINITY;
        s->t_delta[a] = INFINITY;
        double d = r->d[a];
        if (d > 0.0) {
            s->step[a] = 1;
            s->t_next[a] = ((double)(s->c[a] + 1) * cs - r->o[a]) / d;
            s->t_delta[a] = cs / d;
        } else if (d < 0.0) {
            s->step[a] = -1;
            s->t_next[a] = ((double)s->c[a] * cs - r->o[a]) / d;
            s->t_delta[a] = -cs / d;
        }
    }
    s->t_cur = t0;
    s->t1 = t1;
    s->done = 0;
    s->last_axis = -1;
    return 1;
}

static int dda_init(const mc_t* mc, const ray_t* r, double t0, double t1, dda_t* s)
{
    return dda_init_cells(mc->dims, mc->cells, mc->cell, r, t0, t1, s);
}

/* Produces the next visit (cell, ta, tb) over a grid of `cells`; "continue" is implicit. */
static int dda_next_cells(const int cells[3], dda_t* s, int cell[3], double* ta, double* tb)
{
    if (s->done) return 0;
    int axis = 0;
    if (s->t_next[1] < s->t_next[axis]) axis = 1;
    if (s->t_next[2] < s->t_next[axis]) axis = 2;
    double t_exit = dmin(s->t_next[axis], s->t1);
    t_exit = dmax(t_exit, s->t_cur);
    memcpy(cell, s->c, 12);
    *ta = s->t_cur;
    *tb = t_exit;
    s->last_axis = -1;
    if (t_exit >= s->t1) { s->done = 1; return 1; }
    s->t_cur = t_exit;
    s->c[axis] += s->step[axis];
    if (s->c[axis] < s->lo[axis] || s->c[axis] > s->hi[axis]) { s->done = 1; return 1; }
    (void)cells;
    s->t_next[axis] += s->t_delta[axis];
    s->last_axis = axis;
    return 1;
}

static int dda_next(const mc_t* mc, dda_t* s, int cell[3], double* ta, double* tb)
{
    return dda_next_cells(mc->cells, s, cell, ta, tb);
}

/* One flight's majorant-cell visits. Flat: the reference's DDA (dda.hpp:52-109) over the majorant
 * grid. Hierarchical (mc->cdraw): a DDA over 128^3 lower-node regions skips regions without draws
 * in one step; inside a region with draws the majorant-grid DDA restarts at the region entry
 * (dda_init on [ta_c, tb_c]) and its visits are produced in order. */
typedef struct {
    const mc_t* mc;
    const ray_t* ray;
    dda_t coarse, fine;
    int in_fine;
    int entry_axis; /* face through which the next region is entered (-1: the flight's first region) */
} flight_t;

static __thread int g_trace;
#include <stdio.h>
static int flight_init(const mc_t* mc, const ray_t* r, flight_t* f)
{
    if (g_trace)
        fprintf(stderr, "[oracle] ray %a %a %a %a %a %a\n", r->o[0], r->o[1], r->o[2], r->d[0], r->d[1], r->d[2]);
    f->mc = mc;
    f->ray = r;
    f->in_fine = 0;
    f->entry_axis = -1;
    if (!mc->cdraw) {
        f->in_fine = 1;
        return dda_init(mc, r, 0.0, INFINITY, &f->fine);
    }
    return dda_init_cells(mc->dims, mc->ccells, COARSE_CELL, r, 0.0, INFINITY, &f->coarse);
}

/* debug tracing of one (pixel, sample): SO_TRACE="x,y,s" */

static int flight_next_impl(flight_t* f, int cell[3], double* ta, double* tb);
static int flight_next(flight_t* f, int cell[3], double* ta, double* tb)
{
    if (g_trace) {
        int r = flight_next_impl(f, cell, ta, tb);
        if (r) fprintf(stderr, "[oracle] visit %d %d %d %a %a\n", cell[0], cell[1], cell[2], *ta, *tb);
        else fprintf(stderr, "[oracle] flight end\n");
        return r;
    }
    return flight_next_impl(f, cell, ta, tb);
}

static int flight_next_impl(flight_t* f, int cell[3], double* ta, double* tb)
{
    const mc_t* mc = f->mc;
    if (!mc->cdraw)
        return dda_next(mc, &f->fine, cell, ta, tb);
    for (;;) {
        if (f->in_fine) {
            if (dda_next(mc, &f->fine, cell, ta, tb)) return 1;
            f->in_fine = 0;
        }
        int cc[3];
        double a, b;
        if (!dda_next_cells(mc->ccells, &f->coarse, cc, &a, &b)) return 0;
        if (g_trace) fprintf(stderr, "[oracle] region %d %d %d %a %a\n", cc[0], cc[1], cc[2], a, b);
        const int ax = f->entry_axis;
        f->entry_axis = f->coarse.last_axis;
        if (!mc->cdraw[(size_t)cc[0] + (size_t)mc->ccells[0] * ((size_t)cc[1] + (size_t)mc->ccells[1] * (size_t)cc[2])])
            continue;
        /* the entry face fixes the first majorant cell on its axis (floor of a coordinate lying on
           the face would decide it by the last ulp of the ray) */
        /* the region's own cells bound the majorant-grid walk (a t_next recomputed at the restart
           may differ from the region's exit time by an ulp; stepping past the face would visit a
           sliver of the next region's cell) */
        const int R = COARSE_CELL / mc->cell;
        int rlo[3], rhi[3];
        for (int k = 0; k < 3; ++k) {
            rlo[k] = cc[k] * R;
            rhi[k] = (cc[k] + 1) * R < mc->cells[k] ? (cc[k] + 1) * R - 1 : mc->cells[k] - 1;
        }
        int fc = 0;
        if (ax >= 0)
            fc = f->coarse.step[ax] > 0 ? rlo[ax] : rhi[ax];
        if (dda_init_forced(mc->dims, mc->cells, mc->cell, f->ray, a, b, ax, fc, rlo, rhi, &f->fine)) f->in_fine = 1;
    }
}

/* ---- integrators: render.hpp:100-187 ---- */
typedef struct {
    const so_grid* g;
    const so_tf* tf;
    const mc_t* mc;
    const so_settings* s;
    acc_t acc;
} ctx_t;

/* woodcock_track (render.hpp:106-124) */
static int woodcock(ctx_t* cx, double sigma_maj, const ray_t* r, double t0, double t1, rng_t* rng,
                    double* t_ev, float* v_ev)
{
    if (!(sigma_maj > 0.0)) return 0;
    double inv = 1.0 / sigma_maj;
    double t = t0;
    for (;;) {
        t -= log(1.0 - rng_uniform(rng)) * inv;
        if (t >= t1) return 0;
        double p[3];
        ray_at(r, t, p);
        float v = sample_trilinear(&cx->acc, p[0], p[1], p[2]);
        double st = tf_extinction(cx->tf, v);
        if (rng_uniform(rng) < st * inv) { *t_ev = t; *v_ev = v; return 1; }
    }
}

/* next_event (render.hpp:137-151) */
static int next_event(ctx_t* cx, const ray_t* r, rng_t* rng, double* t_ev, float* v_ev)
{
    flight_t d;
    if (!flight_init(cx->mc, r, &d)) return 0;
    int c[3];
    double ta, tb;
    while (flight_next(&d, c, &ta, &tb)) {
        size_t ci = mc_index(cx->mc, c);
        if (cx->mc->empty[ci]) continue;
        if (woodcock(cx, (double)cx->mc->maj[ci], r, ta, tb, rng, t_ev, v_ev)) return 1;
    }
    return 0;
}

/* sample_isotropic (render.hpp:128-134) */
static void sample_isotropic(rng_t* rng, double d[3])
{
    double z = 1.0 - 2.0 * rng_uniform(rng);
    double phi = 2.0 * 3.14159265358979323846 * rng_uniform(rng);
    double r = sqrt(dmax(0.0, 1.0 - z * z));
    d[0] = r * cos(phi); d[1] = r * sin(phi); d[2] = z;
}

static inline double max3(const double v[3]) { return dmax(v[0], dmax(v[1], v[2])); }

/* trace_path (render.hpp:160-187) */
static void trace_path(ctx_t* cx, ray_t ray, rng_t* rng, float out[3])
{
    double tp[3] = {1.0, 1.0, 1.0};
    int bounces = 0;
    for (;;) {
        double t;
        float v;
        if (!next_event(cx, &ray, rng, &t, &v)) {
            for (int c = 0; c < 3; ++c) out[c] = (float)(tp[c] * (double)cx->s->ambient[c]);
            return;
        }
        if (++bounces > cx->s->max_bounces) { out[0] = out[1] = out[2] = 0.0f; return; }
        double rgba[4];
        tf_lookup(cx->tf, v, rgba);
        for (int c = 0; c < 3; ++c) tp[c] *= (double)(float)rgba[c]; /* tf.rgb() -> Vec3f */
        double p[3];
        ray_at(&ray, t, p);
        memcpy(ray.o, p, sizeof p);
        sample_isotropic(rng, ray.d);
        if (bounces >= cx->s->rr_start_bounce) {
            double survive = dclamp(max3(tp), 0.05, 0.95);
            if (rng_uniform(rng) >= survive) { out[0] = out[1] = out[2] = 0.0f; return; }
            for (int c = 0; c < 3; ++c) tp[c] /= survive;
        }
    }
}

/* NEW (no reference function): multi-scatter path with ratio-tracked escape.
 * Along each flight segment the tentative collisions of delta tracking (same majorants,
 * same per-cell restart) also drive a ratio-tracking transmittance estimate
 * Tr = prod(1 - sigma_t/sigma_maj); the segment contributes throughput*Tr*ambient.
 * The first tentative collision accepted by the delta-tracking test (one extra draw per
 * tentative collision while no event is pending) is the scattering vertex; tracking
 * continues past it to the box exit for Tr only. Bounce cutoff and Russian roulette
 * follow trace_path (render.hpp:173-185). */
static void trace_ratio(ctx_t* cx, ray_t ray, rng_t* rng, float out[3])
{
    double tp[3] = {1.0, 1.0, 1.0};
    double L[3] = {0.0, 0.0, 0.0};
    int bounces = 0;
    for (;;) {
        double Tr = 1.0;
        int have = 0;
        double t_ev = 0.0;
        float v_ev = 0.0f;
        flight_t d;
        if (flight_init(cx->mc, &ray, &d)) {
            int c[3];
            double ta, tb;
            while (Tr > 0.0 && flight_next(&d, c, &ta, &tb)) {
                size_t ci = mc_index(cx->mc, c);
                if (cx->mc->empty[ci]) continue;
                double sm = (double)cx->mc->maj[ci];
                if (!(sm > 0.0)) continue;
                double inv = 1.0 / sm;
                double t = ta;
                for (;;) {
                    t -= log(1.0 - rng_uniform(rng)) * inv;
                    if (t >= tb) break;
                    double p[3];
                    ray_at(&ray, t, p);
                    float v = sample_trilinear(&cx->acc, p[0], p[1], p[2]);
                    double r = tf_extinction(cx->tf, v) * inv;
                    if (!have && rng_uniform(rng) < r) { have = 1; t_ev = t; v_ev = v; }
                    Tr *= 1.0 - r;
                    if (!(Tr > 0.0)) break;
                }
            }
        }
        for (int k = 0; k < 3; ++k) L[k] += tp[k] * Tr * (double)cx->s->ambient[k];
        if (!have) break;
        if (++bounces > cx->s->max_bounces) break;
        double rgba[4];
        tf_lookup(cx->tf, v_ev, rgba);
        for (int k = 0; k < 3; ++k) tp[k] *= (double)(float)rgba[k];
        double p[3];
        ray_at(&ray, t_ev, p);
        memcpy(ray.o, p, sizeof p);
        sample_isotropic(rng, ray.d);
        if (bounces >= cx->s->rr_start_bounce) {
            double survive = dclamp(max3(tp), 0.05, 0.95);
            if (rng_uniform(rng) >= survive) break;
            for (int k = 0; k < 3; ++k) tp[k] /= survive;
        }
    }
    for (int k = 0; k < 3; ++k) out[k] = (float)L[k];
}

/* NEW (no reference function): front-to-back emission-absorption march.
 * Samples at t_k = t0 + (k + j)*dt over the clipped box segment [t0, t1], j = third draw of
 * the pixel-sample stream; per sample: rgba = TF(v) (FP64 lerp as transfer.hpp:47-56),
 * a = 1 - exp(-density_scale*alpha*dt), C += T*a*rgb, T *= 1 - a; stop when
 * T < ea_min_transmittance. Result C + T*background. Samples inside empty macrocells
 * contribute exactly nothing (alpha == 0 there), which is what lets the GPU skip them. */
static void trace_ea(ctx_t* cx, const ray_t* ray, rng_t* rng, float out[3])
{
    double j = rng_uniform(rng);
    double C[3] = {0.0, 0.0, 0.0}, T = 1.0;
    double lo[3] = {0, 0, 0};
    double hi[3] = {(double)(cx->g->dims[0] - 1), (double)(cx->g->dims[1] - 1), (double)(cx->g->dims[2] - 1)};
    double t0 = 0.0, t1 = INFINITY;
    double dt = cx->s->ea_step;
    if (clip_ray_box(ray, lo, hi, &t0, &t1) && t0 <= t1) {
        for (long k = 0;; ++k) {
            double t = t0 + ((double)k + j) * dt;
            if (!(t < t1)) break;
            double p[3];
            ray_at(ray, t, p);
            float v = sample_trilinear(&cx->acc, p[0], p[1], p[2]);
            double rgba[4];
            tf_lookup(cx->tf, v, rgba);
            double a = 1.0 - exp(-(cx->tf->density_scale * rgba[3]) * dt);
            for (int c = 0; c < 3; ++c) C[c] += T * a * rgba[c];
            T *= 1.0 - a;
            if (T < cx->s->ea_min_transmittance) break;
        }
    }
    for (int c = 0; c < 3; ++c) out[c] = (float)(C[c] + T * (double)cx->s->background[c]);
}

/* ISO (render.hpp:193-255) */
static float sample_tri_ctx(ctx_t* cx, const ray_t* r, double t)
{
    double p[3];
    ray_at(r, t, p);
    return sample_trilinear(&cx->acc, p[0], p[1], p[2]);
}

static void trace_iso(ctx_t* cx, const ray_t* ray, float out[3])
{
    const double step = 0.25, iso = cx->s->iso_value;
    int hit = 0;
    double hit_t = 0.0;
    dda_t d;
    if (dda_init(cx->mc, ray, 0.0, INFINITY, &d)) {
        int c[3];
        double ta, tb;
        while (!hit && dda_next(cx->mc, &d, c, &ta, &tb)) {
            size_t ci = mc_index(cx->mc, c);
            if (iso < cx->mc->cmin[ci] || iso > cx->mc->cmax[ci]) continue;
            double t_prev = ta;
            double f_prev = (double)sample_tri_ctx(cx, ray, t_prev) - iso;
            if (f_prev == 0.0) { hit = 1; hit_t = t_prev; break; }
            for (double t = ta + step;; t += step) {
                t = dmin(t, tb);
                double f = (double)sample_tri_ctx(cx, ray, t) - iso;
                if (f == 0.0 || (f_prev < 0.0) != (f < 0.0)) {
                    double a = t_prev, b = t;
                    for (int i = 0; i < 16; ++i) {
                        double m = 0.5 * (a + b);
                        double fm = (double)sample_tri_ctx(cx, ray, m) - iso;
                        if (fm == 0.0) { a = b = m; break; }
                        if ((f_prev < 0.0) == (fm < 0.0)) a = m; else b = m;
                    }
                    hit = 1;
                    hit_t = 0.5 * (a + b);
                    break;
                }
                t_prev = t;
                f_prev = f;
                if (t >= tb) break;
            }
        }
    }
    if (!hit) { memcpy(out, cx->s->background, 12); return; }
    double p[3];
    ray_at(ray, hit_t, p);
    /* sample_gradient (sample.hpp:81-95), h = 0.5 */
    const double h = 0.5;
    double gx = (double)(sample_trilinear(&cx->acc, p[0] + h, p[1], p[2]) - sample_trilinear(&cx->acc, p[0] - h, p[1], p[2])) / (2.0 * h);
    double gy = (double)(sample_trilinear(&cx->acc, p[0], p[1] + h, p[2]) - sample_trilinear(&cx->acc, p[0], p[1] - h, p[2])) / (2.0 * h);
    double gz = (double)(sample_trilinear(&cx->acc, p[0], p[1], p[2] + h) - sample_trilinear(&cx->acc, p[0], p[1], p[2] - h)) / (2.0 * h);
    double len = sqrt(gx * gx + gy * gy + gz * gz);
    if (len == 0.0) { out[0] = out[1] = out[2] = 0.0f; return; }
    gx /= len; gy /= len; gz /= len;
    out[0] = (float)fabs(gx); out[1] = (float)fabs(gy); out[2] = (float)fabs(gz);
}

/* camera_ray (render.hpp:259-269) */
static void normalize3(double v[3])
{
    double len = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    v[0] /= len; v[1] /= len; v[2] /= len;
}

static void cross3(const double a[3], const double b[3], double o[3])
{
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

static ray_t camera_ray(const so_camera* cam, double px, double py)
{
    double fwd[3], right[3], up[3];
    for (int a = 0; a < 3; ++a) fwd[a] = cam->look_at[a] - cam->position[a];
    normalize3(fwd);
    cross3(fwd, cam->up, right);
    normalize3(right);
    cross3(right, fwd, up);
    double tan_half = tan(cam->fov_y_deg * 3.14159265358979323846 / 360.0);
    double aspect = (double)cam->width / (double)cam->height;
    double ndc_x = (2.0 * px / (double)cam->width - 1.0) * tan_half * aspect;
    double ndc_y = (1.0 - 2.0 * py / (double)cam->height) * tan_half;
    ray_t r;
    for (int a = 0; a < 3; ++a) {
        r.o[a] = cam->position[a];
        r.d[a] = fwd[a] + right[a] * ndc_x + up[a] * ndc_y;
    }
    normalize3(r.d);
    return r;
}

/* ---- render_field (render.hpp:276-315), threaded over 16x16 tiles ---- */
typedef struct {
    const so_grid* g;
    const so_tf* tf;
    const mc_t* mc;
    const so_camera* cam;
    const so_settings* s;
    float* rgb;
    long* tiles;
    long n_tiles;
    atomic_long next;
    atomic_ullong lookups, paths;
} job_t;

static void* render_worker(void* arg)
{
    job_t* jb = (job_t*)arg;
    const so_camera* cam = jb->cam;
    const so_settings* s = jb->s;
    int tiles_x = (cam->width + 15) / 16;
    uint64_t reads = 0, paths = 0;
    for (;;) {
        long k = atomic_fetch_add(&jb->next, 1);
        if (k >= jb->n_tiles) break;
        long t = jb->tiles[k];
        ctx_t cx = {jb->g, jb->tf, jb->mc, s, {jb->g, NULL, NULL, NULL, 0}};
        int tx = (int)(t % tiles_x) * 16, ty = (int)(t / tiles_x) * 16;
        for (int y = ty; y < ty + 16 && y < cam->height; ++y)
            for (int x = tx; x < tx + 16 && x < cam->width; ++x) {
                double acc3[3] = {0, 0, 0};
                for (int sm = 0; sm < s->spp; ++sm) {
                    rng_t rng = rng_for_pixel_sample(s->seed, x, y, sm);
                    {
                        const char* tr = getenv("SO_TRACE");
                        int tx = -1, ty = -1, ts = -1;
                        if (tr) sscanf(tr, "%d,%d,%d", &tx, &ty, &ts);
                        g_trace = x == tx && y == ty && sm == ts;
                    }
                    double jx = rng_uniform(&rng);
                    double jy = rng_uniform(&rng);
                    ray_t ray = camera_ray(cam, (double)x + jx, (double)y + jy);
                    float c[3];
                    switch (s->mode) {
                    case SO_ISO: trace_iso(&cx, &ray, c); break;
                    case SO_EA: trace_ea(&cx, &ray, &rng, c); break;
                    case SO_RATIO: trace_ratio(&cx, ray, &rng, c); break;
                    default: trace_path(&cx, ray, &rng, c); break;
                    }
                    for (int ch = 0; ch < 3; ++ch) acc3[ch] += (double)c[ch];
                    ++paths;
                }
                for (int ch = 0; ch < 3; ++ch) acc3[ch] /= (double)s->spp;
                size_t o = ((size_t)y * (size_t)cam->width + (size_t)x) * 3;
                for (int ch = 0; ch < 3; ++ch) jb->rgb[o + ch] = (float)acc3[ch];
            }
        reads += cx.acc.reads;
    }
    atomic_fetch_add(&jb->lookups, reads);
    atomic_fetch_add(&jb->paths, paths);
    return NULL;
}

int so_render(const so_grid* g, const so_tf* tf, const so_camera* cam, const so_settings* s,
              float* rgb, uint64_t* lookups, uint64_t* paths)
{
    if (tf->n_entries < 2 || !(tf->domain_hi > tf->domain_lo)) return E_SIZE;
    if (s->spp < 1 || cam->width < 1 || cam->height < 1) return E_SIZE;
    int cd = s->majorant_cell;
    if (cd == 0) cd = 32;
    if (cd != 8 && cd != 32 && cd != 128) return E_SIZE;
    if (s->hdda && cd >= COARSE_CELL) return E_SIZE;
    mc_t mc;
    mc_build(g, tf, cd, &mc);
    mc.cdraw = NULL;
    if (s->hdda && (s->mode == SO_PATHTRACE || s->mode == SO_RATIO))
        mc_build_coarse(&mc);
    int tiles_x = (cam->width + 15) / 16, tiles_y = (cam->height + 15) / 16;
    long total = (long)tiles_x * tiles_y;
    int nr = s->tile_nranks > 0 ? s->tile_nranks : 1;
    job_t jb;
    memset(&jb, 0, sizeof jb);
    jb.g = g; jb.tf = tf; jb.mc = &mc; jb.cam = cam; jb.s = s; jb.rgb = rgb;
    jb.tiles = (long*)malloc(sizeof(long) * (size_t)(total + 1));
    for (long t = 0; t < total; ++t)
        if (t % nr == s->tile_rank) jb.tiles[jb.n_tiles++] = t;
    atomic_init(&jb.next, 0);
    atomic_init(&jb.lookups, 0);
    atomic_init(&jb.paths, 0);
    int nt = s->threads > 0 ? s->threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if (nt > 256) nt = 256;
    pthread_t th[256];
    for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, render_worker, &jb);
    for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
    if (lookups) *lookups = atomic_load(&jb.lookups);
    if (paths) *paths = atomic_load(&jb.paths);
    free(jb.tiles);
    mc_free(&mc);
    return 0;
}

/* ---- N-bit leaf codec (NEW) ---- */
float so_decode(int codec, int code, float lo, float scale)
{
    switch (codec) {
    case 1: return (float)code / 255.0f;
    case 2:
    case 3: return fmaf((float)code, scale, lo);
    default: return lo;
    }
}

static int encode_leaf(int codec, const float* vals, uint8_t* codes, float* lo_out, float* sc_out)
{
    if (codec == 1) {
        for (int i = 0; i < LEAF_VOXELS; ++i) {
            float v = vals[i];
            if (!(v >= 0.0f && v <= 1.0f)) return E_SIZE;
            long c = lrintf(v * 255.0f);
            if ((float)c / 255.0f != v) return E_SIZE; /* not a byte/255 value */
            codes[i] = (uint8_t)c;
        }
        *lo_out = 0.0f;
        *sc_out = 0.0f;
        return 0;
    }
    int levels = codec == 2 ? 255 : 15;
    float lo = vals[0], hi = vals[0];
    for (int i = 1; i < LEAF_VOXELS; ++i) {
        lo = vals[i] < lo ? vals[i] : lo;
        hi = hi < vals[i] ? vals[i] : hi;
    }
    if (lo == 0.0f) lo = 0.0f; /* canonical +0 (the device encoder does the same) */
    if (hi == 0.0f) hi = 0.0f;
    float scale = hi > lo ? (hi - lo) / (float)levels : 0.0f;
    for (int i = 0; i < LEAF_VOXELS; ++i) {
        int c = 0;
        if (scale > 0.0f) {
            float q = floorf((vals[i] - lo) / scale + 0.5f);
            c = q < 0.0f ? 0 : (q > (float)levels ? levels : (int)q);
        }
        codes[i] = (uint8_t)c;
    }
    *lo_out = lo;
    *sc_out = scale;
    return 0;
}

int so_quantize(const uint8_t* bytes, size_t n, int codec, uint8_t** out, size_t* n_out,
                uint8_t* codes, float* params)
{
    so_grid* g;
    int rc = so_open(bytes, n, &g);
    if (rc) return rc;
    uint8_t* o = (uint8_t*)malloc(n);
    memcpy(o, bytes, n);
    uint8_t* leaves = o + (g->leaf - g->base);
    uint8_t tmp[LEAF_VOXELS];
    for (uint64_t i = 0; i < g->n_leaf; ++i) {
        uint8_t* rec = leaves + i * LEAF_BYTES;
        float vals[LEAF_VOXELS];
        memcpy(vals, rec + LEAF_VALUES, sizeof vals);
        if (codec == 0) continue;
        float lo, sc;
        uint8_t* cd = codes ? codes + i * LEAF_VOXELS : tmp;
        rc = encode_leaf(codec, vals, cd, &lo, &sc);
        if (rc) { free(o); so_close(g); return rc; }
        if (params) { params[2 * i] = lo; params[2 * i + 1] = sc; }
        for (int v = 0; v < LEAF_VOXELS; ++v) vals[v] = so_decode(codec, cd[v], lo, sc);
        memcpy(rec + LEAF_VALUES, vals, sizeof vals);
    }
    so_close(g);
    *out = o;
    *n_out = n;
    return 0;
}

void so_free(void* p) { free(p); }
