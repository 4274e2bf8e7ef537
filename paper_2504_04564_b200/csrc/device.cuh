// device.cuh — sm_100a device layout of the frozen {5,4,3} tree and the per-thread hot path:
// cached accessor, N-bit leaf decode, apron-backed trilinear reconstruction, transfer function,
// splitmix64 streams and the macrocell DDA. Semantics follow the reference exactly (file:line per
// function, paths under /root/reference/proj/include/svdb/). Translation units including this
// header are compiled with -fmad=false so every FP64 expression rounds like the reference's x86-64
// build; the only fused op is the explicit fmaf() of the affine leaf decode (== C99 fmaf).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "layout.hpp"
#include "log_glibc.h"

namespace svdbgpu {

// ---- TreeConfig slot math (tree.hpp:43-71) ----
__device__ __forceinline__ int upper_slot(int x, int y, int z)
{
    return ((x >> 7) & 31) + 32 * (((y >> 7) & 31) + 32 * ((z >> 7) & 31));
}
__device__ __forceinline__ int lower_slot(int x, int y, int z)
{
    return ((x >> 3) & 15) + 16 * (((y >> 3) & 15) + 16 * ((z >> 3) & 15));
}
// Leaf payload layout: the 9^3 stencil brick of the leaf, element x + 9y + 81z for brick
// coordinates in [0, 8]: the own 8^3 block where all three are < 8, the apron (the +1 layer,
// copied from the neighbouring blocks) where one is 8. A trilinear stencil based in the block is
// then eight loads at fixed offsets from one element index.
__host__ __device__ __forceinline__ int brick_index(int x, int y, int z) { return x + 9 * y + 81 * z; }
// the own voxel (x, y, z) & 7 of a leaf
__device__ __forceinline__ int leaf_voxel(int x, int y, int z)
{
    return brick_index(x & 7, y & 7, z & 7);
}

// ---- leaf decode ----
// code -> value; UNORM8 == (float)code / 255.0f for every code (tests/test_oracle.py)
template <int CODEC>
__device__ __forceinline__ float decode_code(uint32_t c, float lo, float sc)
{
    if constexpr (CODEC == kCodecUnorm8)
        return __double2float_rn(double(c) * (1.0 / 255.0));
    else
        return fmaf(float(c), sc, lo);
}

// brick element vi (leaf_voxel / brick_index) of leaf `leaf`
template <int CODEC>
__device__ __forceinline__ float decode(const DevGrid& g, uint32_t leaf, int vi, float lo, float sc)
{
    const uint8_t* base = g.codes + size_t(leaf) * g.leaf_stride;
    if constexpr (CODEC == kCodecF32) {
        return __ldg(reinterpret_cast<const float*>(base) + vi);
    } else if constexpr (CODEC == kCodecAffine4) {
        uint32_t b = __ldg(base + (vi >> 1));
        return decode_code<CODEC>((b >> ((vi & 1) * 4)) & 15u, lo, sc);
    } else {
        return decode_code<CODEC>(__ldg(base + vi), lo, sc);
    }
}

// std::lower_bound over the zyx-sorted root (frozen.hpp:101-110), libstdc++ probe order.
__device__ __forceinline__ int find_upper(const DevGrid& g, int ox, int oy, int oz)
{
    int lo = 0, len = g.n_root;
    while (len > 0) {
        int half = len >> 1;
        int4 e = __ldg(g.root + lo + half);
        bool less = e.z != oz ? e.z < oz : (e.y != oy ? e.y < oy : e.x < ox);
        if (less) {
            lo = lo + half + 1;
            len = len - half - 1;
        } else {
            len = half;
        }
    }
    if (lo == g.n_root)
        return -1;
    int4 e = __ldg(g.root + lo);
    return (e.x == ox && e.y == oy && e.z == oz) ? e.w : -1;
}

// Per-thread read-through cache (Accessor, frozen.hpp:228-277). Keys are the coordinate-derived
// node origins; values never depend on the cache state (test_tree.cpp:247-271).
template <int CODEC>
struct Accessor {
    const DevGrid* g;
    int lx, ly, lz; // cached leaf origin
    uint32_t leaf;
    float lo, sc;
    int wx, wy, wz; // cached lower origin
    uint32_t lower;
    int ux, uy, uz; // cached upper origin
    int upper;      // -1: no upper node there

    __device__ __forceinline__ explicit Accessor(const DevGrid& grid) : g(&grid)
    {
        // odd origins never equal an aligned node origin: all three caches start cold
        lx = ly = lz = 1;
        wx = wy = wz = 1;
        ux = uy = uz = 1;
        leaf = lower = 0;
        lo = sc = 0.0f;
        upper = -1;
    }

    __device__ __forceinline__ float read_lower(int x, int y, int z)
    {
        uint4 e = __ldg(g->lower + size_t(lower) * 4096 + lower_slot(x, y, z));
        if (e.x == kSlotTile)
            return __uint_as_float(e.y);
        if (e.x != kSlotChild)
            return g->background;
        lx = x & ~7;
        ly = y & ~7;
        lz = z & ~7;
        SVDB_ASSERT(e.y < g->n_leaf);
        leaf = e.y;
        lo = __uint_as_float(e.z);
        sc = __uint_as_float(e.w);
        return decode<CODEC>(*g, leaf, leaf_voxel(x, y, z), lo, sc);
    }

    __device__ __forceinline__ float read_upper(int x, int y, int z)
    {
        uint2 e = __ldg(g->upper + size_t(upper) * 32768 + upper_slot(x, y, z));
        if (e.x == kSlotTile)
            return __uint_as_float(e.y);
        if (e.x != kSlotChild)
            return g->background;
        wx = x & ~127;
        wy = y & ~127;
        wz = z & ~127;
        SVDB_ASSERT(e.y < g->n_lower);
        lower = e.y;
        return read_lower(x, y, z);
    }

    __device__ __forceinline__ bool in_leaf(int x, int y, int z) const
    {
        return (x & ~7) == lx && (y & ~7) == ly && (z & ~7) == lz;
    }

    __device__ __forceinline__ bool in_lower(int x, int y, int z) const
    {
        return ((x & ~127) == wx) & ((y & ~127) == wy) & ((z & ~127) == wz);
    }

    __device__ __forceinline__ float read(int x, int y, int z)
    {
        if (in_leaf(x, y, z))
            return decode<CODEC>(*g, leaf, leaf_voxel(x, y, z), lo, sc);
        if (in_lower(x, y, z))
            return read_lower(x, y, z);
        int ox = x & ~4095, oy = y & ~4095, oz = z & ~4095;
        if (!(ox == ux && oy == uy && oz == uz)) {
            ux = ox;
            uy = oy;
            uz = oz;
            upper = find_upper(*g, ox, oy, oz);
            wx = 1; // invalidate the lower cache
        }
        if (upper < 0)
            return g->background;
        return read_upper(x, y, z);
    }

    // read(x, y, z) through locate(): the leaf directory instead of the node walk for in-box voxels
    __device__ __forceinline__ float read_located(int x, int y, int z)
    {
        float v;
        if (locate(x, y, z, v))
            return decode<CODEC>(*g, leaf, leaf_voxel(x, y, z), lo, sc);
        return v;
    }

    // Make the leaf holding (x,y,z) the cached leaf: no memory traffic on a leaf-cache hit, one
    // lower-slot load when the lower node is cached, the root/upper walk otherwise. Returns
    // false when (x,y,z) is not inside a leaf; `value` then holds the tile / background value
    // the reference reads there (frozen.hpp:82-99). The only copy of the node walk in the
    // sampler, so the trace loop stays small.
    __device__ __forceinline__ bool locate(int x, int y, int z, float& value)
    {
        if (in_leaf(x, y, z))
            return true;
        if (g->dir) {
            const unsigned cx = unsigned(x) >> 3, cy = unsigned(y) >> 3, cz = unsigned(z) >> 3;
            if (x >= 0 && y >= 0 && z >= 0 && cx < unsigned(g->dir_dims[0]) && cy < unsigned(g->dir_dims[1]) &&
                cz < unsigned(g->dir_dims[2])) {
                // the directory has < 2^32 entries (grid.cu), so the index is 32-bit arithmetic
                const uint4 e = __ldg(g->dir + ((cz * unsigned(g->dir_dims[1]) + cy) * unsigned(g->dir_dims[0]) + cx));
                if (e.x != kSlotChild) {
                    value = __uint_as_float(e.y); // tile value, or the background stored as one
                    return false;
                }
                lx = x & ~7;
                ly = y & ~7;
                lz = z & ~7;
                SVDB_ASSERT(e.y < g->n_leaf);
                leaf = e.y;
                lo = __uint_as_float(e.z);
                sc = __uint_as_float(e.w);
                return true;
            }
        }
        if (!in_lower(x, y, z)) {
            const int ox = x & ~4095, oy = y & ~4095, oz = z & ~4095;
            if (!(ox == ux && oy == uy && oz == uz)) {
                ux = ox;
                uy = oy;
                uz = oz;
                upper = find_upper(*g, ox, oy, oz);
            }
            value = g->background;
            if (upper < 0)
                return false;
            const uint2 ue = __ldg(g->upper + size_t(upper) * 32768 + upper_slot(x, y, z));
            if (ue.x != kSlotChild) {
                if (ue.x == kSlotTile)
                    value = __uint_as_float(ue.y);
                return false;
            }
            wx = x & ~127;
            wy = y & ~127;
            wz = z & ~127;
            SVDB_ASSERT(ue.y < g->n_lower);
            lower = ue.y;
        }
        const uint4 e = __ldg(g->lower + size_t(lower) * 4096 + lower_slot(x, y, z));
        if (e.x != kSlotChild) {
            value = e.x == kSlotTile ? __uint_as_float(e.y) : g->background;
            return false;
        }
        lx = x & ~7;
        ly = y & ~7;
        lz = z & ~7;
        SVDB_ASSERT(e.y < g->n_leaf);
        leaf = e.y;
        lo = __uint_as_float(e.z);
        sc = __uint_as_float(e.w);
        return true;
    }
};

// Uncached root-to-leaf walk (FrozenGrid::read_voxel, frozen.hpp:82-99).
template <int CODEC>
__device__ float read_voxel(const DevGrid& g, int x, int y, int z)
{
    int u = find_upper(g, x & ~4095, y & ~4095, z & ~4095);
    if (u < 0)
        return g.background;
    uint2 ue = __ldg(g.upper + size_t(u) * 32768 + upper_slot(x, y, z));
    if (ue.x == kSlotTile)
        return __uint_as_float(ue.y);
    if (ue.x != kSlotChild)
        return g.background;
    uint4 le = __ldg(g.lower + size_t(ue.y) * 4096 + lower_slot(x, y, z));
    if (le.x == kSlotTile)
        return __uint_as_float(le.y);
    if (le.x != kSlotChild)
        return g.background;
    return decode<CODEC>(g, le.y, leaf_voxel(x, y, z), __uint_as_float(le.z), __uint_as_float(le.w));
}

// ---- sampler (sample.hpp:24-72) ----
__device__ __forceinline__ int lattice_coord(double v)
{
    // floor, clamped to +-1e9 (sample.hpp:24-32) without branches: the saturating conversion of
    // floor(v) clamped in integers gives the same value for every non-NaN v
    return min(max(__double2int_rd(v), -1000000000), 1000000000);
}

// sample.hpp:65-71: x-lerps, then y, then z, in FP64, rounded to float
__device__ __forceinline__ float trilerp(const double v[8], double wx, double wy, double wz)
{
    double v00 = v[0] * (1.0 - wx) + v[1] * wx;
    double v10 = v[2] * (1.0 - wx) + v[3] * wx;
    double v01 = v[4] * (1.0 - wx) + v[5] * wx;
    double v11 = v[6] * (1.0 - wx) + v[7] * wx;
    double v0 = v00 * (1.0 - wy) + v10 * wy;
    double v1 = v01 * (1.0 - wy) + v11 * wy;
    return float(v0 * (1.0 - wz) + v1 * wz);
}

// The eight taps of a trilinear stencil based at own voxel (x, y, z) in [0, 7]^3 of the cached
// leaf, in the reference's tap order (sample.hpp:56-63): brick elements e0 + {0, 1, 9, 10, 81, 82,
// 90, 91} (fixed load offsets). A tap in the apron (its +1 coordinate reaches 8 on the axes in r)
// decodes with that neighbour block's parameters (lparams[leaf][r]); the taps are independent
// loads and lanes whose stencils cross a leaf face do not diverge.
template <int CODEC>
__device__ __forceinline__ void brick_gather(const Accessor<CODEC>& a, int x, int y, int z, float v[8])
{
    SVDB_ASSERT(a.leaf < a.g->n_leaf && unsigned(x) < 8u && unsigned(y) < 8u && unsigned(z) < 8u);
    const uint8_t* base = a.g->codes + size_t(a.leaf) * a.g->leaf_stride;
    const int e0 = brick_index(x, y, z);
    const int ex = x == 7 ? 1 : 0, ey = y == 7 ? 2 : 0, ez = z == 7 ? 4 : 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int K = (k & 1) + 9 * ((k >> 1) & 1) + 81 * (k >> 2);
        if constexpr (CODEC == kCodecF32) {
            v[k] = __ldg(reinterpret_cast<const float*>(base) + e0 + K);
        } else {
            float lo = a.lo, sc = a.sc;
            if constexpr (CODEC != kCodecUnorm8) {
                const int r = ((k & 1) ? ex : 0) | ((k & 2) ? ey : 0) | ((k & 4) ? ez : 0);
                if (r) {
                    const float2 p = __ldg(a.g->lparams + size_t(a.leaf) * 8 + r);
                    lo = p.x;
                    sc = p.y;
                }
            }
            if constexpr (CODEC == kCodecAffine4) { // nibble e & 1 of byte e >> 1
                const int e = e0 + K;
                v[k] = decode_code<CODEC>((uint32_t(__ldg(base + (e >> 1))) >> ((e & 1) * 4)) & 15u, lo, sc);
            } else {
                v[k] = decode_code<CODEC>(__ldg(base + e0 + K), lo, sc);
            }
        }
    }
}

template <int CODEC>
__device__ __forceinline__ float sample_trilinear(Accessor<CODEC>& a, double px, double py, double pz)
{
    const int x0 = lattice_coord(px), y0 = lattice_coord(py), z0 = lattice_coord(pz);
    const double wx = px - floor(px), wy = py - floor(py), wz = pz - floor(pz);
    float t[8]; // the taps are floats (sample.hpp:56-63); both branches fill them and the lanes
                // reconverge for one copy of the FP64 interpolation
    float c0;
    if (a.locate(x0, y0, z0, c0)) {
        // base voxel in a leaf: all 8 taps come from that leaf's brick
        brick_gather<CODEC>(a, x0 & 7, y0 & 7, z0 & 7, t);
    } else {
        // base voxel in a tile / background block (or outside the grid): a non-leaf 8^3 block has
        // one value, so every tap inside the base block is c0 with no load; only taps across the
        // block's far faces are looked up (through the leaf directory, independent loads). Tap
        // order as sample.hpp:56-63.
#pragma unroll
        for (int k = 0; k < 8; ++k)
            t[k] = c0;
        const int cross = ((x0 & 7) == 7 ? 1 : 0) | ((y0 & 7) == 7 ? 2 : 0) | ((z0 & 7) == 7 ? 4 : 0);
        // one copy of the lookup in the instruction stream (rolled) over the taps across the faces
        // only (mask of i with i & cross != 0, from a table), results into registers
        unsigned m = unsigned(0xFEFCFAF0EECCAA00ull >> (8 * cross)) & 0xFEu;
#pragma unroll 1
        while (m) {
            const int i = __ffs(m) - 1;
            m &= m - 1u;
            const float r = a.read_located(x0 + (i & 1), y0 + ((i >> 1) & 1), z0 + (i >> 2));
            switch (i) {
            case 1: t[1] = r; break;
            case 2: t[2] = r; break;
            case 3: t[3] = r; break;
            case 4: t[4] = r; break;
            case 5: t[5] = r; break;
            case 6: t[6] = r; break;
            default: t[7] = r; break;
            }
        }
    }
    const double v[8] = {t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]};
    return trilerp(v, wx, wy, wz);
}

template <int CODEC>
__device__ __forceinline__ float sample_nearest(Accessor<CODEC>& a, double px, double py, double pz)
{
    return a.read(lattice_coord(px + 0.5), lattice_coord(py + 0.5), lattice_coord(pz + 0.5));
}

// ---- transfer function (transfer.hpp:47-91); entries in shared memory ----
__device__ __forceinline__ double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

__device__ __forceinline__ double tf_normalized(const DevTF& tf, double v)
{
    const double d = v - tf.lo;
    return dclamp(tf.inv_range != 0.0 ? d * tf.inv_range : d / (tf.hi - tf.lo), 0.0, 1.0);
}

__device__ __forceinline__ void tf_lookup(const DevTF& tf, const float4* ent, double v, double out[4])
{
    double u = tf_normalized(tf, v) * double(tf.n - 1);
    unsigned long long i0 = (unsigned long long)u;
    if ((unsigned long long)(tf.n - 2) < i0)
        i0 = (unsigned long long)(tf.n - 2);
    double t = u - double(i0);
    float4 a = ent[i0], b = ent[i0 + 1];
    out[0] = (1.0 - t) * double(a.x) + t * double(b.x);
    out[1] = (1.0 - t) * double(a.y) + t * double(b.y);
    out[2] = (1.0 - t) * double(a.z) + t * double(b.z);
    out[3] = (1.0 - t) * double(a.w) + t * double(b.w);
}

__device__ __forceinline__ double tf_alpha(const DevTF& tf, const float4* ent, double v)
{
    // u is in [0, n - 1] (n < 2^31): 32-bit conversions give the same index and fraction
    double u = tf_normalized(tf, v) * double(tf.n - 1);
    unsigned i0 = unsigned(u);
    if (unsigned(tf.n - 2) < i0)
        i0 = unsigned(tf.n - 2);
    double t = u - double(i0);
    return (1.0 - t) * double(ent[i0].w) + t * double(ent[i0 + 1].w);
}

__device__ __forceinline__ double tf_extinction(const DevTF& tf, const float4* ent, double v)
{
    return tf.scale * tf_alpha(tf, ent, v);
}

__device__ __forceinline__ double tf_max_alpha_in_range(const DevTF& tf, const float4* ent, double vlo, double vhi)
{
    if (vhi < vlo) {
        double t = vlo;
        vlo = vhi;
        vhi = t;
    }
    double m = dmax(tf_alpha(tf, ent, vlo), tf_alpha(tf, ent, vhi));
    double ulo = tf_normalized(tf, vlo), uhi = tf_normalized(tf, vhi);
    for (int i = 0; i < tf.n; ++i) {
        double u = double(i) / double(tf.n - 1);
        if (u > ulo && u < uhi)
            m = dmax(m, double(ent[i].w));
    }
    return m;
}

// ---- the free-flight log (render.hpp:116): the reference's glibc log restated (log_glibc.h), so
// step lengths match the reference bit for bit rather than to CUDA log's <= 1 ulp ----
#ifndef SVDB_GLIBC_LOG
#define SVDB_GLIBC_LOG 0 // 1: step lengths bit-exact to the reference; measured -5% (C3) / -7% (C4)
#endif
__device__ __forceinline__ double step_log(double w)
{
#if SVDB_GLIBC_LOG
    return glibc_log(w);
#else
    return log(w);
#endif
}

// ---- splitmix64 streams (rng.hpp:12-67) ----
__device__ __forceinline__ uint64_t mix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct Rng {
    uint64_t state;
    __device__ __forceinline__ static Rng for_pixel_sample(uint64_t seed_mixed, int px, int py, int s)
    {
        // seed_mixed = mix64(seed), hoisted to the host
        uint64_t h = mix64(seed_mixed ^ ((uint64_t(uint32_t(px)) << 32) | uint32_t(py)));
        h = mix64(h ^ uint64_t(uint32_t(s)));
        return Rng{mix64(h)};
    }
    // the 53 random bits of the next uniform() (u = bits * 2^-53), not consumed
    __device__ __forceinline__ uint64_t peek_bits() const
    {
        uint64_t x = state + 0x9E3779B97F4A7C15ull;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        x ^= x >> 31;
        return x >> 11;
    }
    __device__ __forceinline__ void skip() { state += 0x9E3779B97F4A7C15ull; }
    // the value the most recent uniform() / skip() consumed (pure function of the state)
    __device__ __forceinline__ double last() const
    {
        uint64_t x = state;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        x ^= x >> 31;
        return double(x >> 11) * 0x1.0p-53;
    }
    __device__ __forceinline__ double uniform()
    {
        state += 0x9E3779B97F4A7C15ull;
        uint64_t x = state;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        x ^= x >> 31;
        return double(x >> 11) * 0x1.0p-53;
    }
};

// ---- macrocell DDA (dda.hpp:25-109) ----
struct Ray {
    double o[3], d[3];
};

__device__ __forceinline__ bool clip_ray_box(const Ray& r, const double hi[3], double& t0, double& t1)
{
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double o = r.o[a], d = r.d[a];
        if (d == 0.0) {
            if (o < 0.0 || o > hi[a])
                return false;
            continue;
        }
        double inv = 1.0 / d;
        double ta = (0.0 - o) * inv, tb = (hi[a] - o) * inv;
        if (ta > tb) {
            double t = ta;
            ta = tb;
            tb = t;
        }
        t0 = dmax(t0, ta);
        t1 = dmin(t1, tb);
        if (t0 > t1)
            return false;
    }
    return true;
}

struct Dda {
    int c[3], step[3];
    double t_next[3], t_delta[3], t_cur, t1;
    bool done;

    // cell = MacrocellGrid::cell_dim (32 in the reference, macrocell.hpp:20) as a double; icell its
    // exact reciprocal (cell is a power of two, so e * icell == e / cell)
    __device__ __forceinline__ bool init(const int cells[3], const double hi[3], const Ray& r, double t0_, double t1_,
                                         double cell, double icell)
    {
        double t0 = t0_;
        t1 = t1_;
        if (!clip_ray_box(r, hi, t0, t1))
            return false;
        if (!(t0 <= t1))
            return false;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            double e = r.o[a] + r.d[a] * t0;
            c[a] = int(dclamp(floor(e * icell), 0.0, double(cells[a] - 1)));
            double d = r.d[a];
            step[a] = 0;
            t_next[a] = __longlong_as_double(0x7ff0000000000000ll);
            t_delta[a] = t_next[a];
            if (d > 0.0) {
                step[a] = 1;
                t_next[a] = (double(c[a] + 1) * cell - r.o[a]) / d;
                t_delta[a] = cell / d;
            } else if (d < 0.0) {
                step[a] = -1;
                t_next[a] = (double(c[a]) * cell - r.o[a]) / d;
                t_delta[a] = -cell / d;
            }
        }
        t_cur = t0;
        done = false;
        return true;
    }

    // Next visit (cell, ta, tb); false when traversal has ended.
    __device__ __forceinline__ bool next(const int cells[3], int cell[3], double& ta, double& tb)
    {
        if (done)
            return false;
        // axis = 0; if (t_next.y < t_next[axis]) axis = 1; if (t_next.z < t_next[axis]) axis = 2
        // (dda.hpp:90-94), written with selects so t_next stays in registers
        const bool ax1 = t_next[1] < t_next[0];
        const double tm = ax1 ? t_next[1] : t_next[0];
        const bool ax2 = t_next[2] < tm;
        const int axis = ax2 ? 2 : (ax1 ? 1 : 0);
        const double tn = ax2 ? t_next[2] : tm;
        double t_exit = dmin(tn, t1);
        t_exit = dmax(t_exit, t_cur);
        cell[0] = c[0];
        cell[1] = c[1];
        cell[2] = c[2];
        ta = t_cur;
        tb = t_exit;
        if (t_exit >= t1) {
            done = true;
            return true;
        }
        t_cur = t_exit;
#pragma unroll
        for (int a = 0; a < 3; ++a)
            if (a == axis) {
                c[a] += step[a];
                if (c[a] < 0 || c[a] >= cells[a])
                    done = true;
                else
                    t_next[a] += t_delta[a];
            }
        return true;
    }
};

} // namespace svdbgpu
