// grid.cu — device layout build (K0), lattice lookups (K1/K2) and macrocell ranges/majorants (K3).
//
//   K0 grid_create      <- parse_frozen (io.hpp:183-256) + device relayout / leaf codec
//   K1 k_read_voxels    <- FrozenGrid::read_voxel (frozen.hpp:82-99)
//   K2 k_sample         <- sample(Accessor, p, mode) (sample.hpp:97-100), gradient (sample.hpp:81-95)
//   K3 k_cell_ranges    <- build_macrocells (macrocell.hpp:74-103)
//      k_majorants      <- update_majorants (macrocell.hpp:108-116)
#include "device.cuh"
#include "grid_impl.hpp"

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>

namespace svdbgpu {

namespace {

constexpr uint64_t kHdr = 72, kRootRec = 16;
constexpr uint64_t kUpperRec = 16 + 4ull * 32768 + 2ull * 4096;
constexpr uint64_t kLowerRec = 16 + 4ull * 4096 + 2ull * 512;
constexpr uint64_t kLeafRec = 16 + 64 + 4ull * 512;

inline uint32_t rd_u32(const uint8_t* p) { uint32_t v; std::memcpy(&v, p, 4); return v; }
inline int32_t rd_i32(const uint8_t* p) { int32_t v; std::memcpy(&v, p, 4); return v; }
inline uint64_t rd_u64(const uint8_t* p) { uint64_t v; std::memcpy(&v, p, 8); return v; }
inline float rd_f32(const uint8_t* p) { float v; std::memcpy(&v, p, 4); return v; }
inline bool bit(const uint8_t* words, int i) { return (rd_u64(words + 8 * (i >> 6)) >> (i & 63)) & 1u; }

// ---- K0: leaf codec, one warp per leaf, 128-bit coalesced loads of the staged records ----
// Own voxel vi (reference order x + 8y + 64z) -> its element of the 9^3 brick (device.cuh)
__device__ __forceinline__ int brick_of_voxel(int vi) { return brick_index(vi & 7, (vi >> 3) & 7, vi >> 6); }
constexpr int kBrickA4Bytes = (729 + 1) / 2; // 4-bit brick: 729 nibbles

// 4-bit: write the brick bytes of one leaf from its 512 codes (one per byte, reference order, in
// shared memory): own nibbles from the codes, apron nibbles 0 (k_build_apron ORs them in)
__device__ __forceinline__ void write_brick_a4(const uint8_t* s_codes, uint8_t* dst, int lane)
{
    for (int i = lane; i < kBrickA4Bytes; i += 32) {
        uint32_t b = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = 2 * i + h, x = e % 9, y = (e / 9) % 9, z = e / 81;
            if (e < 729 && x < 8 && y < 8 && z < 8)
                b |= uint32_t(s_codes[x + 8 * (y + 8 * z)]) << (4 * h);
        }
        dst[i] = uint8_t(b);
    }
}

template <int CODEC>
__global__ void __launch_bounds__(256) k_leaf_encode(const uint8_t* __restrict__ staging, uint64_t n_leaf,
                                                     uint8_t* __restrict__ codes_base, uint32_t stride,
                                                     float2* __restrict__ params, int* __restrict__ bad)
{
    const int lane = threadIdx.x & 31;
    const uint64_t leaf = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (leaf >= n_leaf)
        return;
    uint8_t* codes = codes_base + leaf * stride; // this leaf's 9^3 brick (own voxels written here)
    const float4* vals = reinterpret_cast<const float4*>(staging + leaf * kLeafRec + 80);
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        v[j] = __ldg(vals + j * 32 + lane); // floats [4(32j+lane), +4): 512 B per warp step
    if constexpr (CODEC == kCodecF32) {
        float* dst = reinterpret_cast<float*>(codes);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int vi = 4 * (j * 32 + lane);
            dst[brick_of_voxel(vi)] = v[j].x;
            dst[brick_of_voxel(vi + 1)] = v[j].y;
            dst[brick_of_voxel(vi + 2)] = v[j].z;
            dst[brick_of_voxel(vi + 3)] = v[j].w;
        }
        if (lane == 0)
            params[leaf] = make_float2(0.0f, 0.0f);
        return;
    } else if constexpr (CODEC == kCodecUnorm8) {
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float f[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int c = __float2int_rn(__fmul_rn(f[k], 255.0f));
                ok &= f[k] >= 0.0f && f[k] <= 1.0f && c >= 0 && c <= 255 &&
                      __double2float_rn(double(c) * (1.0 / 255.0)) == f[k];
                codes[brick_of_voxel(4 * (j * 32 + lane) + k)] = uint8_t(c & 255);
            }
        }
        if (!ok)
            atomicExch(bad, 1);
        if (lane == 0)
            params[leaf] = make_float2(0.0f, 0.0f);
        return;
    } else {
        constexpr int levels = CODEC == kCodecAffine8 ? 255 : 15;
        float lo = v[0].x, hi = v[0].x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            lo = fminf(lo, fminf(fminf(v[j].x, v[j].y), fminf(v[j].z, v[j].w)));
            hi = fmaxf(hi, fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)));
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
        }
        if (lo == 0.0f)
            lo = 0.0f; // canonical +0 (the oracle does the same)
        if (hi == 0.0f)
            hi = 0.0f;
        const float scale = hi > lo ? __fdiv_rn(__fsub_rn(hi, lo), float(levels)) : 0.0f;
        auto q = [&](float x) -> uint32_t {
            if (!(scale > 0.0f))
                return 0u;
            float r = floorf(__fadd_rn(__fdiv_rn(__fsub_rn(x, lo), scale), 0.5f));
            return r < 0.0f ? 0u : (r > float(levels) ? uint32_t(levels) : uint32_t(r));
        };
        __shared__ uint8_t s_codes[CODEC == kCodecAffine4 ? 8 : 1][512]; // 4-bit: staged per leaf
        const int w = threadIdx.x >> 5;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t c[4] = {q(v[j].x), q(v[j].y), q(v[j].z), q(v[j].w)};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int vi = 4 * (j * 32 + lane) + k;
                if constexpr (CODEC == kCodecAffine8)
                    codes[brick_of_voxel(vi)] = uint8_t(c[k]);
                else
                    s_codes[w][vi] = uint8_t(c[k]);
            }
        }
        if constexpr (CODEC == kCodecAffine4) {
            __syncwarp();
            write_brick_a4(s_codes[w], codes, lane);
        }
        if (lane == 0)
            params[leaf] = make_float2(lo, scale);
    }
}

// SVDB v2 (quantised leaves, `svdbgpu_quantise`): the records already hold the codes (reference
// voxel order) and the per-leaf (lo, scale); place the codes in the leaf's 9^3 brick.
// Record: origin/pad 16 B | active mask 64 B | lo, scale 8 B | codes main_bytes.
template <int CODEC>
__global__ void __launch_bounds__(256) k_leaf_load(const uint8_t* __restrict__ staging, uint64_t n_leaf,
                                                   uint32_t rec, uint8_t* __restrict__ codes_base, uint32_t stride,
                                                   float2* __restrict__ params)
{
    __shared__ uint8_t s_codes[8][512];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t leaf = uint64_t(blockIdx.x) * 8 + w;
    if (leaf >= n_leaf)
        return;
    const uint8_t* r = staging + leaf * rec + 88;
    uint8_t* dst = codes_base + leaf * stride;
    if constexpr (CODEC == kCodecAffine4) {
        for (int vi = lane; vi < 512; vi += 32)
            s_codes[w][vi] = uint8_t((__ldg(r + (vi >> 1)) >> ((vi & 1) * 4)) & 15u);
        __syncwarp();
        write_brick_a4(s_codes[w], dst, lane);
    } else {
        for (int vi = lane; vi < 512; vi += 32)
            dst[brick_of_voxel(vi)] = __ldg(r + vi);
    }
    if (lane == 0)
        params[leaf] = *reinterpret_cast<const float2*>(staging + leaf * rec + 80);
}

// The own codes of leaves [first, first + count) in the reference voxel order (main_bytes per
// leaf; the inverse of the brick placement), for the v2 container
template <int CODEC>
__global__ void k_leaf_unbrick(DevGrid g, uint64_t first, uint64_t count, uint8_t* __restrict__ out)
{
    const uint64_t n = count * 512;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t l = i >> 9;
        const int vi = int(i & 511), e = brick_of_voxel(vi);
        const uint8_t* src = g.codes + (first + l) * g.leaf_stride;
        if constexpr (CODEC == kCodecF32) {
            reinterpret_cast<float*>(out)[i] = reinterpret_cast<const float*>(src)[e];
        } else if constexpr (CODEC == kCodecAffine4) {
            if (vi & 1)
                continue;
            const uint32_t c0 = (src[e >> 1] >> ((e & 1) * 4)) & 15u, e1 = brick_of_voxel(vi + 1);
            const uint32_t c1 = (src[e1 >> 1] >> ((e1 & 1) * 4)) & 15u;
            out[l * 256 + (vi >> 1)] = uint8_t(c0 | (c1 << 4));
        } else {
            out[i] = src[e];
        }
    }
}

// Lower slot table with the child leaf's decode parameters folded in (one 16-B load per miss).
__global__ void k_expand_lower(const uint2* __restrict__ staged, uint64_t n_slots,
                               const float2* __restrict__ params, uint4* __restrict__ lower)
{
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_slots;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint2 e = staged[i];
        uint4 o = make_uint4(e.x, e.y, 0u, 0u);
        if (e.x == kSlotChild) {
            float2 p = params[e.y];
            o.z = __float_as_uint(p.x);
            o.w = __float_as_uint(p.y);
        }
        lower[i] = o;
    }
}

// Apron build: leaf L (origin o) also stores the +1 layer of its 9^3 stencil brick — the 217
// voxels with coordinate 8 on some axis — copied as the neighbour's own codes, plus the
// neighbour's decode parameters per region (a tile/background neighbour is stored as code 0
// with (lo = value, scale = 0), so fmaf(0, 0, value) == value). Region r (bits: x, y, z at 8)
// lies entirely in the neighbour block at o + 8*(r&1, r>>1&1, r>>2&1). Decoding an apron tap
// therefore reproduces exactly what the reference reads at that voxel (frozen.hpp:82-99).
__device__ __forceinline__ void apron_entry(int e, int& r, int& x, int& y, int& z)
{
    x = y = z = 0;
    if (e < 64) { r = 1; y = e & 7; z = e >> 3; }
    else if (e < 128) { r = 2; x = (e - 64) & 7; z = (e - 64) >> 3; }
    else if (e < 192) { r = 4; x = (e - 128) & 7; y = (e - 128) >> 3; }
    else if (e < 200) { r = 3; z = e - 192; }
    else if (e < 208) { r = 5; y = e - 200; }
    else if (e < 216) { r = 6; x = e - 208; }
    else { r = 7; }
}

// Resolve the block at origin (x,y,z): {kind, payload, lo, scale} of the lower slot, or a
// tile/background value in payload with kind tile.
__device__ uint4 resolve_block(const DevGrid& g, int x, int y, int z)
{
    const uint4 bg = make_uint4(kSlotTile, __float_as_uint(g.background), 0, 0);
    int u = find_upper(g, x & ~4095, y & ~4095, z & ~4095);
    if (u < 0)
        return bg;
    uint2 ue = __ldg(g.upper + size_t(u) * 32768 + upper_slot(x, y, z));
    if (ue.x == kSlotTile)
        return make_uint4(kSlotTile, ue.y, 0, 0);
    if (ue.x != kSlotChild)
        return bg;
    uint4 le = __ldg(g.lower + size_t(ue.y) * 4096 + lower_slot(x, y, z));
    if (le.x == kSlotChild || le.x == kSlotTile)
        return le;
    return bg;
}

// Leaf directory build: one thread per 8^3 block, the same resolution as the apron build
__global__ void k_build_dir(DevGrid g, int3 dd, uint4* __restrict__ dir)
{
    const uint64_t n = uint64_t(dd.x) * dd.y * dd.z;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const int cx = int(i % uint64_t(dd.x)), cy = int((i / uint64_t(dd.x)) % uint64_t(dd.y)),
                  cz = int(i / (uint64_t(dd.x) * dd.y));
        dir[i] = resolve_block(g, 8 * cx, 8 * cy, 8 * cz);
    }
}

template <int CODEC>
__global__ void __launch_bounds__(256) k_build_apron(DevGrid g, const int4* __restrict__ lorg, uint64_t n_leaf,
                                                     const float2* __restrict__ own, int* __restrict__ bad)
{
    __shared__ uint4 s_info[8][8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t leaf = uint64_t(blockIdx.x) * 8 + w;
    const bool live = leaf < n_leaf;
    if (live && lane >= 1 && lane < 8) {
        const int4 o = lorg[leaf];
        uint4 info = resolve_block(g, o.x + 8 * (lane & 1), o.y + 8 * ((lane >> 1) & 1), o.z + 8 * (lane >> 2));
        s_info[w][lane] = info;
        float2 p = info.x == kSlotChild ? make_float2(__uint_as_float(info.z), __uint_as_float(info.w))
                                        : make_float2(__uint_as_float(info.y), 0.0f);
        g.lparams[leaf * 8 + lane] = p;
    }
    if (live && lane == 0)
        g.lparams[leaf * 8] = own[leaf];
    __syncwarp();
    if (!live)
        return;
    uint8_t* dst = const_cast<uint8_t*>(g.codes) + leaf * g.leaf_stride;
    bool ok = true;
    for (int a = lane; a < 217; a += 32) {
        int r, x, y, z;
        apron_entry(a, r, x, y, z); // (x, y, z): the voxel in the neighbour block r
        const uint4 info = s_info[w][r];
        const int vi = brick_index(x, y, z); // its element in the neighbour's brick
        const int e = brick_index(r & 1 ? 8 : x, r & 2 ? 8 : y, r & 4 ? 8 : z); // and in this one
        const uint8_t* nb = g.codes + size_t(info.y) * g.leaf_stride;
        const float cval = __uint_as_float(info.y);
        if constexpr (CODEC == kCodecF32) {
            reinterpret_cast<float*>(dst)[e] = info.x == kSlotChild ? reinterpret_cast<const float*>(nb)[vi] : cval;
        } else {
            uint32_t c = 0;
            if (info.x == kSlotChild) {
                c = CODEC == kCodecAffine4 ? (nb[vi >> 1] >> ((vi & 1) * 4)) & 15u : nb[vi];
            } else if (CODEC == kCodecUnorm8) {
                int q = __float2int_rn(__fmul_rn(cval, 255.0f));
                ok &= q >= 0 && q <= 255 && __double2float_rn(double(q) * (1.0 / 255.0)) == cval;
                c = uint32_t(q & 255);
            }
            if constexpr (CODEC == kCodecAffine4) // nibble e & 1 of byte e >> 1: OR into its word
                atomicOr(reinterpret_cast<unsigned*>(dst) + (e >> 3), c << (((e >> 1) & 3) * 8 + (e & 1) * 4));
            else
                dst[e] = uint8_t(c);
        }
    }
    if (!ok)
        atomicExch(bad, 1);
}

// ---- K1 ----
template <int CODEC>
__global__ void k_read_voxels(DevGrid g, const int32_t* __restrict__ ijk, size_t n, float* __restrict__ out)
{
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        out[i] = read_voxel<CODEC>(g, ijk[3 * i], ijk[3 * i + 1], ijk[3 * i + 2]);
}

// ---- K2 ----
template <int CODEC>
__global__ void k_sample(DevGrid g, const double* __restrict__ xyz, size_t n, int mode, float* __restrict__ out)
{
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        Accessor<CODEC> a(g);
        double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        out[i] = mode == 0 ? sample_nearest<CODEC>(a, x, y, z) : sample_trilinear<CODEC>(a, x, y, z);
    }
}

template <int CODEC>
__global__ void k_gradient(DevGrid g, const double* __restrict__ xyz, size_t n, double* __restrict__ out)
{
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        Accessor<CODEC> a(g);
        double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        const double h = 0.5;
        out[3 * i] = double(sample_trilinear<CODEC>(a, x + h, y, z) - sample_trilinear<CODEC>(a, x - h, y, z)) / (2.0 * h);
        out[3 * i + 1] = double(sample_trilinear<CODEC>(a, x, y + h, z) - sample_trilinear<CODEC>(a, x, y - h, z)) / (2.0 * h);
        out[3 * i + 2] = double(sample_trilinear<CODEC>(a, x, y, z + h) - sample_trilinear<CODEC>(a, x, y, z - h)) / (2.0 * h);
    }
}

// ---- K3: exact closed-box ranges, one CTA per 32^3 cell (33^3 voxels incl. shared layer) ----
template <int CODEC>
__global__ void __launch_bounds__(256) k_cell_ranges(DevGrid g, int cx_n, int cy_n, int cd, float* __restrict__ cmin,
                                                     float* __restrict__ cmax)
{
    const int cell = blockIdx.x;
    const int cx = cell % cx_n, cy = (cell / cx_n) % cy_n, cz = cell / (cx_n * cy_n);
    const int x0 = cx * cd, y0 = cy * cd, z0 = cz * cd;
    const int ex = min(x0 + cd, g.dims[0] - 1) - x0 + 1;
    const int ey = min(y0 + cd, g.dims[1] - 1) - y0 + 1;
    const int ez = min(z0 + cd, g.dims[2] - 1) - z0 + 1;
    Accessor<CODEC> a(g);
    float mn = __int_as_float(0x7f800000), mx = -mn;
    const int total = ex * ey * ez;
    // thread t walks x-rows so consecutive reads stay in the cached leaf
    for (int r = threadIdx.x; r < ey * ez; r += blockDim.x) {
        int y = y0 + r % ey, z = z0 + r / ey;
        for (int x = x0; x < x0 + ex; ++x) {
            float v = a.read(x, y, z);
            mn = v < mn ? v : mn;
            mx = mx < v ? v : mx;
        }
    }
    (void)total;
    __shared__ float smn[8], smx[8];
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        float o = __shfl_xor_sync(0xffffffffu, mn, off);
        mn = o < mn ? o : mn;
        o = __shfl_xor_sync(0xffffffffu, mx, off);
        mx = mx < o ? o : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        smn[threadIdx.x >> 5] = mn;
        smx[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) {
            mn = smn[w] < mn ? smn[w] : mn;
            mx = mx < smx[w] ? smx[w] : mx;
        }
        cmin[cell] = mn;
        cmax[cell] = mx;
    }
}

__global__ void k_majorants(DevTF tf, const float4* __restrict__ ent_g, const float* __restrict__ cmin,
                            const float* __restrict__ cmax, int n, float* __restrict__ maj,
                            double* __restrict__ inv_maj, float* __restrict__ inv_maj_f,
                            uint8_t* __restrict__ empty)
{
    extern __shared__ float4 s_tf[];
    const float4* ent = s_tf;
    if (tf.n > kTfSmemMax) {
        ent = ent_g;
    } else {
        for (int i = threadIdx.x; i < tf.n; i += blockDim.x)
            s_tf[i] = ent_g[i];
        __syncthreads();
    }
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    double m = tf.scale * tf_max_alpha_in_range(tf, ent, double(cmin[i]), double(cmax[i]));
    maj[i] = float(m);
    // woodcock_track's inv_maj = 1.0 / sigma_maj with sigma_maj = double(float majorant)
    // (render.hpp:113, 147); 0 marks "no draws here" (empty or zero float majorant)
    inv_maj[i] = float(m) > 0.0f ? 1.0 / double(float(m)) : 0.0;
    inv_maj_f[i] = float(inv_maj[i]);
    if (empty)
        empty[i] = m == 0.0 ? 1 : 0;
}

int grid_blocks(size_t n, int threads = 256)
{
    size_t b = (n + threads - 1) / threads;
    return int(b < 148 * 64 ? (b ? b : 1) : 148 * 64);
}

} // namespace

int cuda_fail(cudaError_t e, const char* what)
{
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
        return fail_code(SVDBGPU_E_NO_DEVICE, std::string("no CUDA device (no CPU fallback): ") + cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation)
        return fail_code(SVDBGPU_E_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    return fail_code(SVDBGPU_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

GridImpl::~GridImpl()
{
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaFree(d_root);
    cudaFree(d_upper);
    cudaFree(d_lower);
    cudaFree(d_codes);
    cudaFree(d_lparams);
    cudaFree(d_cmin);
    cudaFree(d_cmax);
    cudaFree(d_maj);
    cudaFree(d_inv_maj);
    cudaFree(d_inv_maj_f);
    cudaFree(d_dir);
    cudaFree(d_tf);
    cudaFree(d_img);
    cudaFree(d_gather);
    cudaFree(d_cdraw);
    cudaFree(d_camtab);
    cudaFree(d_sbuf);
    cudaFree(d_counters);
    cudaFree(d_scratch);
    if (ev0)
        cudaEventDestroy(ev0);
    if (ev1)
        cudaEventDestroy(ev1);
    if (stream)
        cudaStreamDestroy(stream);
    cudaSetDevice(prev);
}

int validate_tf(const svdbgpu_tf* tf)
{
    // TransferFunction ctor (transfer.hpp:23-35)
    if (!tf || !tf->rgba)
        return fail_code(SVDBGPU_E_INVALID_ARG, "transfer function is null");
    if (!(tf->domain_hi > tf->domain_lo))
        return fail(Errc::size_mismatch, "transfer function domain must have hi > lo");
    if (tf->n_entries < 2)
        return fail(Errc::size_mismatch, "transfer function needs at least 2 entries");
    if (!(tf->density_scale > 0.0) || !std::isfinite(tf->density_scale))
        return fail(Errc::size_mismatch, "density_scale must be positive");
    for (int i = 0; i < tf->n_entries; ++i) {
        float a = tf->rgba[4 * i + 3];
        if (!(a >= 0.0f && a <= 1.0f))
            return fail(Errc::size_mismatch, "transfer function alpha must be in [0,1]");
    }
    return 0;
}

int GridImpl::upload_tf(const svdbgpu_tf* tf, cudaStream_t s, DevTF* out)
{
    if (int rc = validate_tf(tf))
        return rc;
    if (tf->n_entries > tf_cap) {
        cudaFree(d_tf);
        d_tf = nullptr;
        SVDB_CUDA(cudaMalloc(&d_tf, sizeof(float4) * size_t(tf->n_entries)));
        tf_cap = tf->n_entries;
    }
    SVDB_CUDA(cudaMemcpyAsync(d_tf, tf->rgba, sizeof(float4) * size_t(tf->n_entries), cudaMemcpyHostToDevice, s));
    *out = DevTF{tf->domain_lo, tf->domain_hi, tf->density_scale, tf->n_entries, 0.0};
    {
        const double range = tf->domain_hi - tf->domain_lo;
        int e = 0;
        if (std::isfinite(range) && range > 0.0 && std::frexp(range, &e) == 0.5 && e > -1000 && e < 1000)
            out->inv_range = std::ldexp(1.0, 1 - e); // exact reciprocal of the power of two
    }
    return 0;
}

#define SVDB_CODEC_DISPATCH(codec, F)                                                         \
    switch (codec) {                                                                           \
    case kCodecF32: F(kCodecF32); break;                                                       \
    case kCodecUnorm8: F(kCodecUnorm8); break;                                                 \
    case kCodecAffine8: F(kCodecAffine8); break;                                               \
    default: F(kCodecAffine4); break;                                                          \
    }

int GridImpl::ensure_ranges(cudaStream_t s, float* ms, int cd)
{
    if (ranges_valid && cd == cell_dim) {
        if (ms)
            *ms = 0.0f;
        return 0;
    }
    if (cd != 8 && cd != 32 && cd != 128)
        return fail_code(SVDBGPU_E_INVALID_ARG, "majorant cell size must be 8, 32 or 128 voxels");
    cudaFree(d_cmin);
    cudaFree(d_cmax);
    cudaFree(d_maj);
    cudaFree(d_inv_maj);
    cudaFree(d_inv_maj_f);
    d_cmin = d_cmax = d_maj = nullptr;
    d_inv_maj = nullptr;
    d_inv_maj_f = nullptr;
    ranges_valid = false;
    cell_dim = cd;
    for (int a = 0; a < 3; ++a) // cell_counts_for (macrocell.hpp:66-70) with cell_dim cd
        cells[a] = std::max(1, (dg.dims[a] - 1 + cd - 1) / cd);
    size_t nc = size_t(cells[0]) * cells[1] * cells[2];
    SVDB_CUDA(cudaMalloc(&d_cmin, nc * 4));
    SVDB_CUDA(cudaMalloc(&d_cmax, nc * 4));
    SVDB_CUDA(cudaMalloc(&d_maj, nc * 4));
    SVDB_CUDA(cudaMalloc(&d_inv_maj, nc * 8));
    SVDB_CUDA(cudaMalloc(&d_inv_maj_f, nc * 4));
    SVDB_CUDA(cudaEventRecord(ev0, s));
#define LAUNCH_RANGES(C) k_cell_ranges<C><<<unsigned(nc), 256, 0, s>>>(dg, cells[0], cells[1], cd, d_cmin, d_cmax)
    SVDB_CODEC_DISPATCH(codec, LAUNCH_RANGES)
#undef LAUNCH_RANGES
    SVDB_CUDA(cudaGetLastError());
    SVDB_CUDA(cudaEventRecord(ev1, s));
    SVDB_CUDA(cudaEventSynchronize(ev1));
    float t = 0.0f;
    cudaEventElapsedTime(&t, ev0, ev1);
    if (ms)
        *ms = t;
    ranges_valid = true;
    return 0;
}

int majorants(GridImpl* g, const DevTF& tf, cudaStream_t s, uint8_t* d_empty)
{
    int nc = g->cells[0] * g->cells[1] * g->cells[2];
    k_majorants<<<(nc + 255) / 256, 256, tf_smem_bytes(tf.n), s>>>(tf, g->d_tf, g->d_cmin, g->d_cmax, nc,
                                                                            g->d_maj, g->d_inv_maj, g->d_inv_maj_f, d_empty);
    SVDB_CUDA(cudaGetLastError());
    return 0;
}

// Hierarchical DDA (render settings.hdda): one flag per 128^3 lower-node region over the majorant
// grid of g->cell_dim (which divides 128): set when some majorant cell inside has a positive float
// majorant, i.e. tracking would draw there (oracle/svdb_oracle.c mc_build_coarse).
__global__ void k_coarse_flags(const float* __restrict__ maj, int3 cells, int R, int3 cc, uint8_t* __restrict__ draw)
{
    const int n = cc.x * cc.y * cc.z;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int x0 = (i % cc.x) * R, y0 = ((i / cc.x) % cc.y) * R, z0 = (i / (cc.x * cc.y)) * R;
        uint8_t any = 0;
        for (int z = z0; z < min(z0 + R, cells.z) && !any; ++z)
            for (int y = y0; y < min(y0 + R, cells.y) && !any; ++y)
                for (int x = x0; x < min(x0 + R, cells.x); ++x)
                    if (maj[x + cells.x * (y + cells.y * z)] > 0.0f) {
                        any = 1;
                        break;
                    }
        draw[i] = any;
    }
}

int coarse_flags(GridImpl* g, const int ccells[3], cudaStream_t s)
{
    const size_t n = size_t(ccells[0]) * size_t(ccells[1]) * size_t(ccells[2]);
    if (n > g->cdraw_cap || !g->d_cdraw) {
        cudaFree(g->d_cdraw);
        g->d_cdraw = nullptr;
        g->cdraw_cap = 0;
        SVDB_CUDA(cudaMalloc(&g->d_cdraw, n));
        g->cdraw_cap = n;
    }
    k_coarse_flags<<<unsigned(std::min<size_t>((n + 255) / 256, 148 * 8)), 256, 0, s>>>(
        g->d_maj, make_int3(g->cells[0], g->cells[1], g->cells[2]), 128 / g->cell_dim,
        make_int3(ccells[0], ccells[1], ccells[2]), g->d_cdraw);
    SVDB_CUDA(cudaGetLastError());
    return 0;
}

int grid_create(const uint8_t* b, size_t n, int codec, int device, GridImpl** out)
{
    NvtxRange nvtx("svdbgpu grid_create (validate, upload, leaf codec, apron, directory)");
    *out = nullptr;
    if (!b && n)
        return fail_code(SVDBGPU_E_INVALID_ARG, "svdb bytes are null");
    if (codec < 0 || codec > SVDBGPU_CODEC_AUTO8)
        return fail_code(SVDBGPU_E_INVALID_ARG, "unknown codec");
    // ---- parse_frozen validation (io.hpp:183-256) ----
    if (n < 4)
        return fail(Errc::corrupt_index, "unexpected end of SVDB data");
    if (std::memcmp(b, "SVDB", 4) != 0)
        return fail(Errc::bad_magic, "not an SVDB file");
    if (n < 8)
        return fail(Errc::corrupt_index, "unexpected end of SVDB data");
    uint32_t version = rd_u32(b + 4);
    if (version != 1 && version != 2)
        return fail(Errc::version_mismatch, "unsupported SVDB version " + std::to_string(version));
    if (n < kHdr)
        return fail(Errc::corrupt_index, "unexpected end of SVDB data");
    uint32_t vt = rd_u32(b + 8);
    if (vt > 1)
        return fail(Errc::corrupt_index, "invalid voxel type");
    int dims[3] = {int(rd_u32(b + 12)), int(rd_u32(b + 16)), int(rd_u32(b + 20))};
    if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
        return fail(Errc::corrupt_index, "invalid dims");
    uint64_t nu = rd_u64(b + 36), nl = rd_u64(b + 44), nf = rd_u64(b + 52), nr = rd_u64(b + 60);
    const uint64_t lim = 1ull << 32;
    if (nu > lim || nl > lim || nf > lim || nr > lim)
        return fail(Errc::corrupt_index, "implausible section counts");
    // v2 (this repo's quantised-leaf container, svdbgpu_quantise): the v1 layout with the codec in
    // the header's padding word and leaf records {origin/pad, active mask, lo/scale, codes}
    int stored = -1;
    uint64_t leaf_rec = kLeafRec;
    if (version == 2) {
        stored = int(rd_u32(b + 68));
        if (stored != kCodecUnorm8 && stored != kCodecAffine8 && stored != kCodecAffine4)
            return fail(Errc::corrupt_index, "invalid quantised leaf codec");
        if (codec != SVDBGPU_CODEC_AUTO8 && codec != stored)
            return fail_code(SVDBGPU_E_UNSUPPORTED, "a quantised SVDB is loaded with its stored codec (or AUTO8)");
        leaf_rec = 88 + (stored == kCodecAffine4 ? 256 : 512);
    }
    if (kHdr + kRootRec * nr + kUpperRec * nu + kLowerRec * nl + leaf_rec * nf != n)
        return fail(Errc::corrupt_index, "section counts do not match data size");
    const uint8_t* root = b + kHdr;
    const uint8_t* up = root + kRootRec * nr;
    const uint8_t* low = up + kUpperRec * nu;
    const uint8_t* leaf = low + kLowerRec * nl;
    std::vector<int4> h_root(size_t(nr ? nr : 1));
    for (uint64_t i = 0; i < nr; ++i) {
        const uint8_t* e = root + 16 * i;
        h_root[i] = make_int4(rd_i32(e), rd_i32(e + 4), rd_i32(e + 8), int(rd_u32(e + 12)));
        if (rd_u32(e + 12) >= nu)
            return fail(Errc::corrupt_index, "root entry references missing upper node");
    }
    std::vector<uint2> h_upper(size_t(nu) * 32768);
    for (uint64_t i = 0; i < nu; ++i) {
        const uint8_t* r = up + kUpperRec * i;
        const uint8_t* child = r + 16 + 4 * 32768;
        const uint8_t* tile = child + 4096;
        for (int s = 0; s < 32768; ++s) {
            uint32_t p = rd_u32(r + 16 + 4 * s);
            bool c = bit(child, s);
            if (c && p >= nl)
                return fail(Errc::corrupt_index, "upper node child index out of range");
            h_upper[i * 32768 + s] = bit(tile, s) ? make_uint2(kSlotTile, p) : (c ? make_uint2(kSlotChild, p) : make_uint2(0, 0));
        }
    }
    std::vector<uint2> h_lower(size_t(nl) * 4096);
    for (uint64_t i = 0; i < nl; ++i) {
        const uint8_t* r = low + kLowerRec * i;
        const uint8_t* child = r + 16 + 4 * 4096;
        const uint8_t* tile = child + 512;
        for (int s = 0; s < 4096; ++s) {
            uint32_t p = rd_u32(r + 16 + 4 * s);
            bool c = bit(child, s);
            if (c && p >= nf)
                return fail(Errc::corrupt_index, "lower node child index out of range");
            h_lower[i * 4096 + s] = bit(tile, s) ? make_uint2(kSlotTile, p) : (c ? make_uint2(kSlotChild, p) : make_uint2(0, 0));
        }
    }

    int ndev = 0;
    SVDB_CUDA(cudaGetDeviceCount(&ndev));
    if (ndev < 1)
        return fail_code(SVDBGPU_E_NO_DEVICE, "no CUDA device (no CPU fallback)");
    if (device < 0 || device >= ndev)
        return fail_code(SVDBGPU_E_INVALID_ARG, "device ordinal out of range");
    SVDB_CUDA(cudaSetDevice(device));

    auto g = std::make_unique<GridImpl>();
    g->device = device;
    g->voxel_type = int(vt);
    g->value_domain[0] = rd_f32(b + 28);
    g->value_domain[1] = rd_f32(b + 32);
    g->n_upper = nu;
    g->n_lower = nl;
    g->n_leaf = nf;
    g->n_root = nr;
    g->svdb_bytes = n;
    SVDB_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    SVDB_CUDA(cudaEventCreate(&g->ev0));
    SVDB_CUDA(cudaEventCreate(&g->ev1));
    SVDB_CUDA(cudaMalloc(&g->d_counters, 128)); // [0] samples [1] work queue [2..15] stats
    cudaStream_t s = g->stream;

    SVDB_CUDA(cudaMalloc(&g->d_root, sizeof(int4) * h_root.size()));
    SVDB_CUDA(cudaMemcpyAsync(g->d_root, h_root.data(), sizeof(int4) * h_root.size(), cudaMemcpyHostToDevice, s));
    SVDB_CUDA(cudaMalloc(&g->d_upper, sizeof(uint2) * (h_upper.size() ? h_upper.size() : 1)));
    if (!h_upper.empty())
        SVDB_CUDA(cudaMemcpyAsync(g->d_upper, h_upper.data(), sizeof(uint2) * h_upper.size(), cudaMemcpyHostToDevice, s));
    SVDB_CUDA(cudaMalloc(&g->d_lower, sizeof(uint4) * (h_lower.size() ? h_lower.size() : 1)));

    // leaf origins from the node path (lower origin + slot offset), for the apron build
    std::vector<int4> h_lorg(size_t(nf ? nf : 1), make_int4(0, 0, 0, 0));
    for (uint64_t i = 0; i < nl; ++i) {
        const uint8_t* r = low + kLowerRec * i;
        const int ox = rd_i32(r), oy = rd_i32(r + 4), oz = rd_i32(r + 8);
        for (int s2 = 0; s2 < 4096; ++s2) {
            const uint2 e = h_lower[i * 4096 + s2];
            if (e.x == kSlotChild)
                h_lorg[e.y] = make_int4(ox + 8 * (s2 & 15), oy + 8 * ((s2 >> 4) & 15), oz + 8 * (s2 >> 8), 0);
        }
    }

    // ---- leaves: stage records in chunks, encode with the codec, then build the aprons ----
    int resolved = stored >= 0 ? stored : codec;
    if (resolved == SVDBGPU_CODEC_AUTO8)
        resolved = vt == 0 ? kCodecUnorm8 : kCodecAffine8;
    const uint32_t main_bytes = resolved == kCodecF32 ? 2048u : (resolved == kCodecAffine4 ? 256u : 512u);
    // the 9^3 brick (729 elements) per leaf, padded to a multiple of 128 B
    const uint32_t stride = resolved == kCodecF32 ? 2944u : (resolved == kCodecAffine4 ? 384u : 768u);
    float2* d_params = nullptr;
    uint2* d_lstage = nullptr;
    uint8_t* d_stage = nullptr;
    int4* d_lorg = nullptr;
    int* d_bad = nullptr;
    const uint64_t chunk = std::min<uint64_t>(nf ? nf : 1, 1ull << 18); // 256 Ki leaves <= 558 MB staging
    SVDB_CUDA(cudaMalloc(&d_params, sizeof(float2) * (nf ? nf : 1)));
    SVDB_CUDA(cudaMalloc(&d_bad, sizeof(int)));
    SVDB_CUDA(cudaMalloc(&g->d_codes, size_t(stride) * (nf ? nf : 1)));
    SVDB_CUDA(cudaMalloc(&g->d_lparams, sizeof(float2) * 8 * (nf ? nf : 1)));
    SVDB_CUDA(cudaMalloc(&d_lorg, sizeof(int4) * h_lorg.size()));
    SVDB_CUDA(cudaMemcpyAsync(d_lorg, h_lorg.data(), sizeof(int4) * h_lorg.size(), cudaMemcpyHostToDevice, s));
    if (nl) {
        SVDB_CUDA(cudaMalloc(&d_lstage, sizeof(uint2) * h_lower.size()));
        SVDB_CUDA(cudaMemcpyAsync(d_lstage, h_lower.data(), sizeof(uint2) * h_lower.size(), cudaMemcpyHostToDevice, s));
    }
    if (nf)
        SVDB_CUDA(cudaMalloc(&d_stage, size_t(leaf_rec * chunk)));
    g->dg.dims[0] = dims[0];
    g->dg.dims[1] = dims[1];
    g->dg.dims[2] = dims[2];
    g->dg.background = rd_f32(b + 24);
    g->dg.n_root = int(nr);
    g->dg.root = g->d_root;
    g->dg.upper = g->d_upper;
    g->dg.lower = g->d_lower;
    g->dg.codes = g->d_codes;
    g->dg.lparams = g->d_lparams;
    g->dg.leaf_stride = stride;
    g->dg.main_bytes = main_bytes;
    g->dg.n_leaf = uint32_t(nf);
    g->dg.n_lower = uint32_t(nl);
    for (int attempt = 0; attempt < 2; ++attempt) {
        SVDB_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
        for (uint64_t first = 0; first < nf; first += chunk) {
            uint64_t cnt = std::min(chunk, nf - first);
            SVDB_CUDA(cudaMemcpyAsync(d_stage, leaf + leaf_rec * first, size_t(leaf_rec * cnt), cudaMemcpyHostToDevice, s));
            unsigned blocks = unsigned((cnt + 7) / 8);
            uint8_t* dst = g->d_codes + size_t(stride) * first;
            float2* par = d_params + first;
            if (stored >= 0) {
                if (stored == kCodecAffine4)
                    k_leaf_load<kCodecAffine4><<<blocks, 256, 0, s>>>(d_stage, cnt, uint32_t(leaf_rec), dst, stride, par);
                else
                    k_leaf_load<kCodecAffine8><<<blocks, 256, 0, s>>>(d_stage, cnt, uint32_t(leaf_rec), dst, stride, par);
            } else {
#define LAUNCH_ENCODE(C) k_leaf_encode<C><<<blocks, 256, 0, s>>>(d_stage, cnt, dst, stride, par, d_bad)
                SVDB_CODEC_DISPATCH(resolved, LAUNCH_ENCODE)
#undef LAUNCH_ENCODE
            }
            SVDB_CUDA(cudaGetLastError());
        }
        if (nl) {
            k_expand_lower<<<grid_blocks(h_lower.size()), 256, 0, s>>>(d_lstage, h_lower.size(), d_params, g->d_lower);
            SVDB_CUDA(cudaGetLastError());
        }
        if (nf) {
            unsigned blocks = unsigned((nf + 7) / 8);
#define LAUNCH_APRON(C) k_build_apron<C><<<blocks, 256, 0, s>>>(g->dg, d_lorg, nf, d_params, d_bad)
            SVDB_CODEC_DISPATCH(resolved, LAUNCH_APRON)
#undef LAUNCH_APRON
            SVDB_CUDA(cudaGetLastError());
        }
        int bad = 0;
        SVDB_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
        SVDB_CUDA(cudaStreamSynchronize(s));
        if (!bad)
            break;
        if (codec == SVDBGPU_CODEC_AUTO8 && resolved == kCodecUnorm8 && stored < 0) {
            resolved = kCodecAffine8; // same layout
            continue;
        }
        cudaFree(d_stage);
        cudaFree(d_params);
        cudaFree(d_bad);
        cudaFree(d_lorg);
        cudaFree(d_lstage);
        return fail(Errc::size_mismatch, "UNORM8 codec needs every leaf value (and tile/background value "
                                         "adjacent to a leaf) to be byte/255 exact");
    }
    cudaFree(d_stage);
    cudaFree(d_bad);
    cudaFree(d_lorg);
    cudaFree(d_lstage);
    cudaFree(d_params);

    g->codec = resolved;
    g->leaf_payload_bytes = uint64_t(stride) * nf + 64 * nf;
    g->device_bytes = sizeof(int4) * h_root.size() + sizeof(uint2) * h_upper.size() + sizeof(uint4) * h_lower.size() +
                      uint64_t(stride) * nf + 64 * nf;
    // leaf directory over the grid's box, when it costs at most 1 GiB or no more than the lower table
    // (and has < 2^32 entries: the device indexes it with 32-bit arithmetic)
    {
        const int3 dd = make_int3((dims[0] + 7) / 8, (dims[1] + 7) / 8, (dims[2] + 7) / 8);
        const uint64_t nd = uint64_t(dd.x) * dd.y * dd.z, bytes = nd * sizeof(uint4);
        const char* off = std::getenv("SVDBGPU_NO_LEAF_DIR"); // diagnostics: force the node walk
        if (nd && nd < (1ull << 32) && !(off && off[0] == '1') &&
            (bytes <= (1ull << 30) || bytes <= sizeof(uint4) * h_lower.size()) &&
            cudaMalloc(&g->d_dir, bytes) == cudaSuccess) {
            k_build_dir<<<grid_blocks(nd), 256, 0, s>>>(g->dg, dd, g->d_dir);
            SVDB_CUDA(cudaGetLastError());
            SVDB_CUDA(cudaStreamSynchronize(s));
            g->dg.dir = g->d_dir;
            g->dg.dir_dims[0] = dd.x;
            g->dg.dir_dims[1] = dd.y;
            g->dg.dir_dims[2] = dd.z;
            g->device_bytes += bytes;
        } else {
            cudaGetLastError(); // an over-budget or failed allocation just means no directory
        }
    }
    *out = g.release();
    return 0;
}

int grid_leaf_codes(const GridImpl* g, uint64_t first, uint64_t count, uint8_t* codes, float* params)
{
    if (first + count > g->n_leaf)
        return fail_code(SVDBGPU_E_INVALID_ARG, "leaf range out of bounds");
    SVDB_CUDA(cudaSetDevice(g->device));
    if (codes && count) { // the leaves' own 8^3 blocks out of their bricks (the apron is derived data)
        const uint64_t step = std::min<uint64_t>(count, 1ull << 18);
        uint8_t* d_out = nullptr;
        SVDB_CUDA(cudaMalloc(&d_out, size_t(step) * g->dg.main_bytes));
        for (uint64_t f = 0; f < count; f += step) {
            const uint64_t c = std::min(step, count - f);
#define LAUNCH_UNBRICK(C) k_leaf_unbrick<C><<<grid_blocks(c * 512), 256>>>(g->dg, first + f, c, d_out)
            SVDB_CODEC_DISPATCH(g->codec, LAUNCH_UNBRICK)
#undef LAUNCH_UNBRICK
            const cudaError_t e = cudaMemcpy(codes + size_t(f) * g->dg.main_bytes, d_out, size_t(c) * g->dg.main_bytes,
                                             cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                cudaFree(d_out);
                SVDB_CUDA(e);
            }
        }
        cudaFree(d_out);
    }
    if (params && count) {
        // params live folded in the lower table; recover them by scanning it on the host
        std::vector<uint4> low(size_t(g->n_lower) * 4096);
        SVDB_CUDA(cudaMemcpy(low.data(), g->d_lower, sizeof(uint4) * low.size(), cudaMemcpyDeviceToHost));
        for (auto& e : low)
            if (e.x == kSlotChild && e.y >= first && e.y < first + count) {
                std::memcpy(&params[2 * (e.y - first)], &e.z, 4);
                std::memcpy(&params[2 * (e.y - first) + 1], &e.w, 4);
            }
    }
    return 0;
}

int read_voxels_device(const GridImpl* g, const int32_t* d_ijk, size_t n, float* d_out, cudaStream_t s)
{
    if (!n)
        return 0;
#define LAUNCH_RV(C) k_read_voxels<C><<<grid_blocks(n), 256, 0, s>>>(g->dg, d_ijk, n, d_out)
    SVDB_CODEC_DISPATCH(g->codec, LAUNCH_RV)
#undef LAUNCH_RV
    SVDB_CUDA(cudaGetLastError());
    return 0;
}

int sample_device(const GridImpl* g, const double* d_xyz, size_t n, int mode, float* d_out, cudaStream_t s)
{
    if (!n)
        return 0;
#define LAUNCH_S(C) k_sample<C><<<grid_blocks(n), 256, 0, s>>>(g->dg, d_xyz, n, mode, d_out)
    SVDB_CODEC_DISPATCH(g->codec, LAUNCH_S)
#undef LAUNCH_S
    SVDB_CUDA(cudaGetLastError());
    return 0;
}

int gradient_device(const GridImpl* g, const double* d_xyz, size_t n, double* d_out, cudaStream_t s)
{
    if (!n)
        return 0;
#define LAUNCH_G(C) k_gradient<C><<<grid_blocks(n), 256, 0, s>>>(g->dg, d_xyz, n, d_out)
    SVDB_CODEC_DISPATCH(g->codec, LAUNCH_G)
#undef LAUNCH_G
    SVDB_CUDA(cudaGetLastError());
    return 0;
}


// svdbgpu_quantise: SVDB v1 -> v2 with the leaves encoded on the GPU by the device codec (the
// k_leaf_encode arithmetic). Header, root, upper and lower sections are kept byte for byte (version
// 2, codec in the padding word); each leaf record keeps its origin and active mask and carries
// (lo, scale) + codes instead of 512 floats: 600 B (8-bit) / 344 B (4-bit) vs 2128 B.
int quantise_svdb(const uint8_t* b, size_t n, int codec, int device, std::vector<uint8_t>& out)
{
    if (codec != kCodecUnorm8 && codec != kCodecAffine8 && codec != kCodecAffine4 && codec != SVDBGPU_CODEC_AUTO8)
        return fail_code(SVDBGPU_E_INVALID_ARG, "quantise needs UNORM8, AFFINE8, AFFINE4 or AUTO8");
    if (n >= 8 && std::memcmp(b, "SVDB", 4) == 0 && rd_u32(b + 4) != 1)
        return fail(Errc::version_mismatch, "quantise reads SVDB version 1");
    GridImpl* gp = nullptr;
    if (int rc = grid_create(b, n, codec, device, &gp))
        return rc;
    std::unique_ptr<GridImpl> g(gp);
    const uint64_t nf = g->n_leaf, nl = g->n_lower, nu = g->n_upper, nr = g->n_root;
    const uint32_t mb = g->dg.main_bytes;
    const uint64_t head = kHdr + kRootRec * nr + kUpperRec * nu + kLowerRec * nl;
    const uint64_t rec = 88 + mb;
    std::vector<uint8_t> codes(size_t(mb) * (nf ? nf : 1));
    std::vector<float> params(2 * size_t(nf ? nf : 1));
    if (nf)
        if (int rc = grid_leaf_codes(g.get(), 0, nf, codes.data(), params.data()))
            return rc;
    out.resize(size_t(head + rec * nf));
    std::memcpy(out.data(), b, size_t(head));
    const uint32_t v2 = 2, cv = uint32_t(g->codec);
    std::memcpy(out.data() + 4, &v2, 4);
    std::memcpy(out.data() + 68, &cv, 4);
    const uint8_t* leaf = b + head;
    for (uint64_t i = 0; i < nf; ++i) {
        uint8_t* d = out.data() + head + rec * i;
        std::memcpy(d, leaf + kLeafRec * i, 80); // origin, pad, active mask
        std::memcpy(d + 80, &params[2 * i], 8);
        std::memcpy(d + 88, codes.data() + size_t(mb) * i, mb);
    }
    return 0;
}

} // namespace svdbgpu
