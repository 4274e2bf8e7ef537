/* oracle/synth_oracle.c — TEST INFRASTRUCTURE ONLY (see svdb_oracle.h).
 *
 * Plain-C restatement of the BASELINE.json synthetic volumes, so the reference
 * arm of bench.py and the CPU tests can build the same inputs without loading the product library
 * (libsvdbgpu.so). Must be bit-identical to svdbgpu_synth (tests/test_oracle.py pins it). The
 * lattice hashing follows svdb::hash_counter (rng.hpp:21-24) semantics: mix64(mix64(seed) ^ c).
 *
 *   kind 0  Marschner-Lobb (f_M = 6, alpha = 0.25) on [-1,1]^3, u8-quantised (load_raw, volume.hpp:91-97)
 *   kind 1  5-octave value-noise fBm smoke with a radial falloff, u8-quantised, background exactly 0
 *   kind 2  6-octave ridged turbulence, dense f32 in [0,1]
 *   kind 3  5-octave thresholded fBm, f32, background exactly 0; the threshold is calibrated per
 *           volume size so 35% of the 8^3 leaf blocks hold non-background voxels (C4)
 *
 * Compiled with -ffp-contract=off like the rest of the oracle; the product's host encoder is built
 * for baseline x86-64 (no FMA), so both round every double op identically.
 */
#define _GNU_SOURCE
#include "svdb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static uint64_t mix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static uint64_t hash_counter(uint64_t seed, uint64_t c) { return mix64(mix64(seed) ^ c); }
static double smooth(double f) { return f * f * (3.0 - 2.0 * f); }
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
static int mini(int a, int b) { return a < b ? a : b; }

/* One value-noise octave: a (cells+2)^3 lattice of values in [-1,1], smoothstep-interpolated. */
typedef struct {
    int cells, n;
    double scale; /* lattice units per voxel */
    float* lat;
} octave_t;

static void octave_init(octave_t* o, int cells, int dim_max, uint64_t seed)
{
    o->cells = cells;
    o->n = cells + 2;
    o->scale = (double)cells / (double)(dim_max - 1 > 1 ? dim_max - 1 : 1);
    size_t m = (size_t)o->n * o->n * o->n;
    o->lat = (float*)malloc(m * sizeof(float));
    for (size_t i = 0; i < m; ++i)
        o->lat[i] = (float)((double)(hash_counter(seed, i) >> 11) * 0x1.0p-53 * 2.0 - 1.0);
}

/* lattice blended at (y, z) for every lattice x index */
static void octave_row(const octave_t* o, int y, int z, double* out)
{
    double v = y * o->scale, w = z * o->scale;
    int j = mini((int)v, o->cells), k = mini((int)w, o->cells);
    double fv = smooth(v - j), fw = smooth(w - k);
    const float* p00 = &o->lat[(size_t)o->n * ((size_t)j + (size_t)o->n * (size_t)k)];
    const float* p10 = p00 + o->n;
    const float* p01 = p00 + (size_t)o->n * o->n;
    const float* p11 = p01 + o->n;
    for (int i = 0; i < o->n; ++i) {
        double a = p00[i] + (p10[i] - (double)p00[i]) * fv;
        double b = p01[i] + (p11[i] - (double)p01[i]) * fv;
        out[i] = a + (b - a) * fw;
    }
}

static double octave_at_x(const octave_t* o, const double* r, int x)
{
    double u = x * o->scale;
    int i = mini((int)u, o->cells);
    return r[i] + (r[i + 1] - r[i]) * smooth(u - i);
}

static float quantise_u8(double v)
{
    double c = clampd(v, 0.0, 1.0);
    int b = (int)lround(c * 255.0);
    return (float)b / 255.0f; /* load_raw's u8 mapping (volume.hpp:97) */
}

/* Sparse-field threshold on d = 0.5 + 0.5 fBm, per volume size (max dimension), so the share of
 * 8^3 blocks with a voxel above it is 35% (calibrated by tools/calibrate_sparse.py from the exact
 * per-block maxima of d: the 65th percentile; log2-linear between the calibrated sizes). */
double so_sparse_threshold(int dim_max)
{
    static const int sz[] = {64, 128, 256, 512, 1024, 2048, 4096};
    static const double th[] = {0.7263, 0.6573, 0.6089, 0.5796, 0.5630, 0.5540, 0.5494};
    const int n = (int)(sizeof(sz) / sizeof(sz[0]));
    if (dim_max <= sz[0])
        return th[0];
    for (int i = 1; i < n; ++i)
        if (dim_max == sz[i])
            return th[i];
        else if (dim_max < sz[i]) {
            double a = log2((double)sz[i - 1]), b = log2((double)sz[i]), x = log2((double)dim_max);
            return th[i - 1] + (th[i] - th[i - 1]) * ((x - a) / (b - a));
        }
    return th[n - 1];
}

typedef struct {
    int kind, dims[3], octaves;
    octave_t* oct;
    float* out;         /* dense volume, or NULL */
    double* block_max;  /* per-8^3-block max of the pre-threshold density d (kind 3), or NULL */
    double threshold;
    int64_t next_row;   /* work counter: rows of 8^3 blocks */
    pthread_mutex_t mu;
} synth_job;

static double voxel(const synth_job* J, const double* const* rp, int x, int y, int z, double* d_out)
{
    const int* dims = J->dims;
    if (J->kind == 0) {
        /* Marschner-Lobb (f_M = 6, alpha = 0.25) on [-1,1]^3 */
        const double pi = 3.14159265358979323846;
        double px = dims[0] > 1 ? -1.0 + 2.0 * (double)x / (double)(dims[0] - 1) : 0.0;
        double py = dims[1] > 1 ? -1.0 + 2.0 * (double)y / (double)(dims[1] - 1) : 0.0;
        double pz = dims[2] > 1 ? -1.0 + 2.0 * (double)z / (double)(dims[2] - 1) : 0.0;
        const double fm = 6.0, a = 0.25;
        double rr = sqrt(px * px + py * py);
        double rho_r = cos(2.0 * pi * fm * cos(pi * rr / 2.0));
        double val = (1.0 - sin(pi * pz / 2.0) + a * (1.0 + rho_r)) / (2.0 * (1.0 + a));
        return quantise_u8(val);
    }
    double f = 0.0, amp = 1.0, norm = 0.0;
    for (int o = 0; o < J->octaves; ++o) {
        double nv = octave_at_x(&J->oct[o], rp[o], x);
        f += amp * (J->kind == 2 ? fabs(nv) : nv);
        norm += amp;
        amp *= 0.5;
    }
    f /= norm;
    if (J->kind == 1) {
        double cx = 0.5 * (dims[0] - 1), cy = 0.5 * (dims[1] - 1), cz = 0.5 * (dims[2] - 1);
        double dx = (x - cx) / (0.5 * dims[0]), dy = (y - cy) / (0.5 * dims[1]), dz = (z - cz) / (0.5 * dims[2]);
        double fall = clampd(1.0 - sqrt(dx * dx + dy * dy + dz * dz), 0.0, 1.0);
        double d = (0.5 + 0.5 * f) * (0.35 + 0.65 * fall) - 0.25;
        return quantise_u8(d * 3.0);
    }
    if (J->kind == 2) {
        double t = 1.0 - f;
        return (float)clampd(t * t * t, 0.0, 1.0);
    }
    double d = 0.5 + 0.5 * f;
    if (d_out)
        *d_out = d;
    return (float)clampd((d - J->threshold) * 4.0, 0.0, 1.0);
}

static void* synth_worker(void* arg)
{
    synth_job* J = (synth_job*)arg;
    const int* dims = J->dims;
    size_t lsize = 0;
    for (int o = 0; o < J->octaves; ++o)
        lsize += (size_t)J->oct[o].n;
    double* lrow = (double*)malloc((lsize ? lsize : 1) * sizeof(double));
    const double* rp[8];
    const int bx = (dims[0] + 7) / 8, by = (dims[1] + 7) / 8, bz = (dims[2] + 7) / 8;
    /* work item = one (y, z) row of 8^3 blocks: 8 x 8 voxel rows, disjoint block_max entries */
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t item = J->next_row++;
        pthread_mutex_unlock(&J->mu);
        if (item >= (int64_t)by * bz)
            break;
        const int iy = (int)(item % by), iz = (int)(item / by);
        double* bm = J->block_max ? J->block_max + ((size_t)iz * by + (size_t)iy) * bx : NULL;
        for (int z = 8 * iz; z < mini(8 * iz + 8, dims[2]); ++z)
            for (int y = 8 * iy; y < mini(8 * iy + 8, dims[1]); ++y) {
                size_t off = 0;
                for (int o = 0; o < J->octaves; ++o) {
                    octave_row(&J->oct[o], y, z, lrow + off);
                    rp[o] = lrow + off;
                    off += (size_t)J->oct[o].n;
                }
                float* row = J->out ? J->out + ((size_t)z * dims[1] + (size_t)y) * (size_t)dims[0] : NULL;
                for (int x = 0; x < dims[0]; ++x) {
                    double d = 0.0;
                    float v = (float)voxel(J, rp, x, y, z, bm ? &d : NULL);
                    if (row)
                        row[x] = v;
                    if (bm && d > bm[x / 8])
                        bm[x / 8] = d;
                }
            }
    }
    free(lrow);
    return NULL;
}

static int run_synth(int kind, const int32_t dims[3], uint64_t seed, int threads, float* out, double* block_max)
{
    if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1 || kind < 0 || kind > 3)
        return 2; /* Errc::size_mismatch + 1 */
    if (block_max && kind != 3)
        return 2;
    synth_job J;
    memset(&J, 0, sizeof J);
    J.kind = kind;
    memcpy(J.dims, dims, sizeof J.dims);
    int dmax = dims[0] > dims[1] ? dims[0] : dims[1];
    dmax = dmax > dims[2] ? dmax : dims[2];
    J.octaves = kind == 0 ? 0 : (kind == 2 ? 6 : 5);
    int base_cells = kind == 2 ? 4 : 6;
    J.oct = (octave_t*)calloc((size_t)(J.octaves ? J.octaves : 1), sizeof(octave_t));
    for (int o = 0; o < J.octaves; ++o)
        octave_init(&J.oct[o], base_cells << o, dmax, seed * 1315423911ull + (uint64_t)o + 1);
    J.out = out;
    J.block_max = block_max;
    J.threshold = so_sparse_threshold(dmax);
    if (block_max) {
        size_t nb = (size_t)((dims[0] + 7) / 8) * (size_t)((dims[1] + 7) / 8) * (size_t)((dims[2] + 7) / 8);
        for (size_t i = 0; i < nb; ++i)
            block_max[i] = -1.0e300;
    }
    pthread_mutex_init(&J.mu, NULL);
    int nt = threads > 0 ? threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1)
        nt = 1;
    if (nt > 256)
        nt = 256;
    pthread_t th[256];
    for (int i = 1; i < nt; ++i)
        pthread_create(&th[i], NULL, synth_worker, &J);
    synth_worker(&J);
    for (int i = 1; i < nt; ++i)
        pthread_join(th[i], NULL);
    pthread_mutex_destroy(&J.mu);
    for (int o = 0; o < J.octaves; ++o)
        free(J.oct[o].lat);
    free(J.oct);
    return 0;
}

int so_synth(int kind, const int32_t dims[3], uint64_t seed, int threads, float* out)
{
    return run_synth(kind, dims, seed, threads, out, NULL);
}

int so_sparse_block_max(const int32_t dims[3], uint64_t seed, int threads, double* block_max)
{
    return run_synth(3, dims, seed, threads, NULL, block_max);
}
