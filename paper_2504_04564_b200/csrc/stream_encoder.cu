// stream_encoder.cu — the fixed-rate encoder over a volume streamed through the GPU in z-slabs
// ("histogram / background / brick ranges are HBM-bound scans; streaming leaf
// build for >= 2048^3"). Output: the SVDB v1 container BYTE-IDENTICAL to svdbgpu_compress on the
// dense volume (= the reference's serialize_frozen(compress(v, params).first), compress.hpp:221-283),
// without ever holding the dense volume on the host. Peak host memory = the container itself plus
// per-8^3-block state (5 B per block).
//
// A slab is 32 z-slices (one brick layer, four leaf-block layers). The volume is produced five times
// (on the device by the synthetic generators, or copied from a host callback), once per pass:
//   1. min / max / finite check + per-brick ranges   (from_data volume.hpp:39-63; compress.hpp:97-145)
//   2. histogram over [min, max]                     (compute_histogram volume.hpp:177-206)
//   3. exact counts of the values in the modal bin   (detect_background volume.hpp:208-222): sort + RLE
//   host: brick order + budget (choose_bricks), shared with the dense encoder
//   4. per-8^3-block decision: absent / leaf / uniform tile / corner leaf (compress.hpp:171-215, 253-268)
//   host: lower-node prune, z,y,x indices, header / root / upper / lower (write_tree)
//   5. leaf records (origin, active mask, 512 values) written on the device, copied into place
// Every value passes through from_data's -0 -> +0 normalisation, as in the dense encoder.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>

#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <unordered_map>
#include <vector>

#include "grid_impl.hpp"
#include "svdbgpu_internal.hpp"

namespace svdbgpu {
namespace {

constexpr int kSlab = 32;
constexpr uint64_t kLeafRecBytes = 16 + 64 + 4ull * 512;

__device__ __forceinline__ float nzf(float v) { return v == 0.0f ? 0.0f : v; }
// monotone float <-> int mapping for atomicMin / atomicMax
__device__ __forceinline__ int ford(float f)
{
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
inline float ford_inv(int i)
{
    const int j = i >= 0 ? i : i ^ 0x7fffffff;
    float f;
    std::memcpy(&f, &j, 4);
    return f;
}

// ---- device synthetic generators: svdbgpu_synth's arithmetic (host_encoder.cpp), op for op ----
struct OctaveDev {
    int cells, n;
    double scale;
    const float* lat;
};
struct SynthArgs {
    int kind, octaves;
    int dims[3];
    double threshold; // sparse field
    OctaveDev oct[6];
};

__device__ __forceinline__ double smooth_d(double f) { return f * f * (3.0 - 2.0 * f); }
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

__device__ float synth_voxel(const SynthArgs& S, int x, int y, int z)
{
    double f = 0.0, amp = 1.0, norm = 0.0;
    for (int o = 0; o < S.octaves; ++o) {
        const OctaveDev& O = S.oct[o];
        // Octave::row (the lattice blended at (y, z)) at lattice columns i, i + 1, then Octave::at_x
        const double v = y * O.scale, w = z * O.scale;
        const int j = min(int(v), O.cells), k = min(int(w), O.cells);
        const double fv = smooth_d(v - j), fw = smooth_d(w - k);
        const float* p00 = O.lat + size_t(O.n) * (size_t(j) + size_t(O.n) * size_t(k));
        const float* p10 = p00 + O.n;
        const float* p01 = p00 + size_t(O.n) * O.n;
        const float* p11 = p01 + O.n;
        const double u = x * O.scale;
        const int i = min(int(u), O.cells);
        double r[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const double a = __ldg(p00 + i + q) + (__ldg(p10 + i + q) - double(__ldg(p00 + i + q))) * fv;
            const double b = __ldg(p01 + i + q) + (__ldg(p11 + i + q) - double(__ldg(p01 + i + q))) * fv;
            r[q] = a + (b - a) * fw;
        }
        const double nv = r[0] + (r[1] - r[0]) * smooth_d(u - i);
        f += amp * (S.kind == 2 ? fabs(nv) : nv);
        norm += amp;
        amp *= 0.5;
    }
    f /= norm;
    if (S.kind == 1) { // fBm smoke, u8-quantised (load_raw's mapping, volume.hpp:97)
        const double cx = 0.5 * (S.dims[0] - 1), cy = 0.5 * (S.dims[1] - 1), cz = 0.5 * (S.dims[2] - 1);
        const double dx = (x - cx) / (0.5 * S.dims[0]), dy = (y - cy) / (0.5 * S.dims[1]),
                     dz = (z - cz) / (0.5 * S.dims[2]);
        const double fall = clampd(1.0 - sqrt(dx * dx + dy * dy + dz * dz), 0.0, 1.0);
        const double d = (0.5 + 0.5 * f) * (0.35 + 0.65 * fall) - 0.25;
        const double c = clampd(d * 3.0, 0.0, 1.0);
        const int b = int(lround(c * 255.0));
        return float(b) / 255.0f;
    }
    if (S.kind == 2) {
        const double t = 1.0 - f;
        return float(clampd(t * t * t, 0.0, 1.0));
    }
    const double d = 0.5 + 0.5 * f;
    return float(clampd((d - S.threshold) * 4.0, 0.0, 1.0));
}

__global__ void k_synth_slab(const __grid_constant__ SynthArgs S, int z0, int nz, float* __restrict__ out)
{
    const long long n = (long long)S.dims[0] * S.dims[1] * nz;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int x = int(i % S.dims[0]);
        const long long r = i / S.dims[0];
        const int y = int(r % S.dims[1]), z = z0 + int(r / S.dims[1]);
        out[i] = synth_voxel(S, x, y, z);
    }
}

// ---- pass 1: min / max / finite + brick ranges ----
__global__ void k_stats(const float* __restrict__ v, long long n, int* __restrict__ mn, int* __restrict__ mx,
                        int* __restrict__ nonfinite)
{
    float lo = INFINITY, hi = -INFINITY;
    bool bad = false;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float s = nzf(v[i]);
        bad |= !isfinite(s);
        lo = fminf(lo, s);
        hi = fmaxf(hi, s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mn, ford(lo));
        atomicMax(mx, ford(hi));
        if (bad)
            atomicOr(nonfinite, 1);
    }
}

// one CTA per brick of the slab's brick layer (bz fixed)
__global__ void __launch_bounds__(256) k_brick_ranges(const float* __restrict__ v, int dx, int dy, int dz, int z0,
                                                      int nbx, int nby, float* __restrict__ blo, float* __restrict__ bhi)
{
    const int bx = blockIdx.x % nbx, by = blockIdx.x / nbx, bz = z0 / kEncBrick;
    const int x0 = bx * kEncBrick, y0 = by * kEncBrick;
    const int wx = min(kEncBrick, dx - x0), wy = min(kEncBrick, dy - y0), wz = min(kEncBrick, dz - z0);
    float lo = INFINITY, hi = -INFINITY;
    for (int e = threadIdx.x; e < kEncBrick * kEncBrick * kEncBrick; e += blockDim.x) {
        const int x = e & 31, y = (e >> 5) & 31, z = e >> 10;
        if (x < wx && y < wy && z < wz) {
            const float s = nzf(v[size_t(x0 + x) + size_t(dx) * (size_t(y0 + y) + size_t(dy) * size_t(z))]);
            lo = fminf(lo, s);
            hi = fmaxf(hi, s);
        }
    }
    __shared__ float slo[8], shi[8];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        slo[threadIdx.x >> 5] = lo;
        shi[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) {
            lo = fminf(lo, slo[w]);
            hi = fmaxf(hi, shi[w]);
        }
        const size_t b = size_t(bx) + size_t(nbx) * (size_t(by) + size_t(nby) * size_t(bz));
        blo[b] = lo;
        bhi[b] = hi;
    }
}

// ---- pass 2 / 3: histogram bin (compute_histogram) and the modal bin's values ----
__device__ __forceinline__ int bin_of(double s, double hlo, double hhi, int bins)
{
    if (hhi <= hlo)
        return 0;
    const int b = int(floor((s - hlo) / (hhi - hlo) * double(bins)));
    return b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
}

__global__ void __launch_bounds__(256) k_hist(const float* __restrict__ v, long long n, double hlo, double hhi, int bins,
                                              unsigned long long* __restrict__ hist)
{
    __shared__ unsigned h[1024];
    for (int i = threadIdx.x; i < bins; i += blockDim.x)
        h[i] = 0;
    __syncthreads();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        atomicAdd(&h[bin_of(double(nzf(v[i])), hlo, hhi, bins)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < bins; i += blockDim.x)
        if (h[i])
            atomicAdd(hist + i, (unsigned long long)h[i]);
}

__global__ void k_select_bin(const float* __restrict__ v, long long n, double hlo, double hhi, int bins, int best,
                             float* __restrict__ out, unsigned long long* __restrict__ count)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x < n;
         i += (long long)gridDim.x * blockDim.x) {
        float s = 0.0f;
        bool take = false;
        if (i < n) {
            s = nzf(v[i]);
            take = bin_of(double(s), hlo, hhi, bins) == best;
        }
        const unsigned m = __ballot_sync(0xffffffffu, take);
        unsigned long long base = 0;
        if ((threadIdx.x & 31) == 0 && m)
            base = atomicAdd(count, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take)
            out[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = s;
    }
}

// ---- pass 4: per-8^3-block decision, one warp per block of the slab ----
__global__ void k_block_state(const float* __restrict__ v, int dx, int dy, int dz, int z0, int nz,
                              const uint8_t* __restrict__ chosen, int nbx, int nby, float bg,
                              uint8_t* __restrict__ state, float* __restrict__ tile_val)
{
    const int lx = (dx + 7) / 8, ly = (dy + 7) / 8, lzs = (nz + 7) / 8;
    const long long nblk = (long long)lx * ly * lzs;
    const int lane = threadIdx.x & 31;
    const int cx1 = dx - 1, cy1 = dy - 1, cz1 = dz - 1;
    for (long long wb = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wb < nblk;
         wb += ((long long)gridDim.x * blockDim.x) >> 5) {
        const int bx = int(wb % lx), by = int((wb / lx) % ly), bz = z0 / 8 + int(wb / ((long long)lx * ly));
        const int x0 = bx * 8, y0 = by * 8, zz0 = bz * 8;
        const bool corner = (bx == 0 && by == 0 && bz == 0) || (bx == cx1 / 8 && by == cy1 / 8 && bz == cz1 / 8);
        uint8_t st = kBlkAbsent;
        float tv = 0.0f;
        const size_t brick = size_t(x0 / kEncBrick) + size_t(nbx) * (size_t(y0 / kEncBrick) + size_t(nby) * size_t(zz0 / kEncBrick));
        if (chosen[brick]) {
            const bool full = x0 + 8 <= dx && y0 + 8 <= dy && zz0 + 8 <= dz;
            if (!full) {
                st = kBlkLeaf; // set_voxel path: partially active, never collapses
            } else {
                auto at = [&](int x, int y, int z) {
                    return nzf(v[size_t(x) + size_t(dx) * (size_t(y) + size_t(dy) * size_t(z - z0))]);
                };
                const float v0 = at(x0, y0, zz0);
                bool all_bg = true, uniform = true;
#pragma unroll 4
                for (int k = 0; k < 16; ++k) {
                    const int vi = lane + 32 * k;
                    const float s = at(x0 + (vi & 7), y0 + ((vi >> 3) & 7), zz0 + (vi >> 6));
                    all_bg &= !(s != bg);
                    uniform &= !(s != v0);
                }
                all_bg = __all_sync(0xffffffffu, all_bg);
                uniform = __all_sync(0xffffffffu, uniform);
                if (!all_bg) {
                    if (uniform) {
                        st = kBlkTile; // fully active uniform leaf -> lower tile (v0 != B)
                        tv = v0;
                    } else {
                        st = kBlkLeaf;
                    }
                }
            }
        }
        if (corner && st == kBlkAbsent)
            st = kBlkCornerLeaf; // corner set_voxel creates a background leaf, partially active
        if (lane == 0) {
            const size_t b = size_t(bx) + size_t(lx) * (size_t(by) + size_t(ly) * size_t(bz));
            state[b] = st;
            tile_val[b] = tv;
        }
    }
}

// ---- pass 5: leaf records {origin, pad, mask 512 bits, 512 f32}, one warp per block of the slab ----
__global__ void k_leaf_records(const float* __restrict__ v, int dx, int dy, int dz, int z0, int nz,
                               const uint8_t* __restrict__ state, const uint32_t* __restrict__ leaf_index,
                               uint64_t first_leaf, float bg, uint8_t* __restrict__ recs)
{
    const int lx = (dx + 7) / 8, ly = (dy + 7) / 8, lzs = (nz + 7) / 8;
    const long long nblk = (long long)lx * ly * lzs;
    const int lane = threadIdx.x & 31;
    const int cx1 = dx - 1, cy1 = dy - 1, cz1 = dz - 1;
    for (long long wb = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wb < nblk;
         wb += ((long long)gridDim.x * blockDim.x) >> 5) {
        const int bx = int(wb % lx), by = int((wb / lx) % ly), bz = z0 / 8 + int(wb / ((long long)lx * ly));
        const size_t b = size_t(bx) + size_t(lx) * (size_t(by) + size_t(ly) * size_t(bz));
        const uint8_t st = state[b];
        if (st != kBlkLeaf && st != kBlkCornerLeaf)
            continue;
        const int x0 = bx * 8, y0 = by * 8, zz0 = bz * 8;
        uint8_t* r = recs + (uint64_t(leaf_index[b]) - first_leaf) * kLeafRecBytes;
        const bool brick = st == kBlkLeaf;
        const bool c0 = bx == 0 && by == 0 && bz == 0;
        const bool c1 = bx == cx1 / 8 && by == cy1 / 8 && bz == cz1 / 8;
        const int vc1 = (cx1 & 7) + 8 * ((cy1 & 7) + 8 * (cz1 & 7));
        float* vals = reinterpret_cast<float*>(r + 80);
        uint32_t* mask = reinterpret_cast<uint32_t*>(r + 16);
#pragma unroll 4
        for (int k = 0; k < 16; ++k) {
            const int vi = lane + 32 * k;
            const int gx = x0 + (vi & 7), gy = y0 + ((vi >> 3) & 7), gz = zz0 + (vi >> 6);
            const bool inside = gx < dx && gy < dy && gz < dz;
            float val = bg;
            bool on = false;
            const bool corner_voxel = (c0 && vi == 0) || (c1 && vi == vc1);
            if ((brick && inside) || corner_voxel) {
                val = nzf(v[size_t(gx) + size_t(dx) * (size_t(gy) + size_t(dy) * size_t(gz - z0))]);
                on = true;
            }
            vals[vi] = val;
            const unsigned m = __ballot_sync(0xffffffffu, on);
            if (lane == 0)
                mask[k] = m;
        }
        if (lane < 4) // origin x, y, z and the zero pad
            reinterpret_cast<int32_t*>(r)[lane] = lane == 0 ? x0 : (lane == 1 ? y0 : (lane == 2 ? zz0 : 0));
    }
}

// ---- slab sources ----
struct SlabSource {
    virtual ~SlabSource() = default;
    virtual int produce(int z0, int nz, float* d_slab, cudaStream_t s) = 0;
};

struct SynthSource : SlabSource {
    SynthArgs S{};
    std::vector<float*> d_lat;
    ~SynthSource() override
    {
        for (float* p : d_lat)
            cudaFree(p);
    }
    int init(int kind, const int32_t dims[3], uint64_t seed)
    {
        std::vector<SynthOctave> oct;
        synth_lattices(kind, dims, seed, oct);
        S.kind = kind;
        S.octaves = int(oct.size());
        for (int a = 0; a < 3; ++a)
            S.dims[a] = dims[a];
        S.threshold = sparse_threshold(std::max(dims[0], std::max(dims[1], dims[2])));
        for (size_t o = 0; o < oct.size(); ++o) {
            float* p = nullptr;
            SVDB_CUDA(cudaMalloc(&p, oct[o].lat.size() * sizeof(float)));
            d_lat.push_back(p);
            SVDB_CUDA(cudaMemcpy(p, oct[o].lat.data(), oct[o].lat.size() * sizeof(float), cudaMemcpyHostToDevice));
            S.oct[o] = OctaveDev{oct[o].cells, oct[o].n, oct[o].scale, p};
        }
        return 0;
    }
    int produce(int z0, int nz, float* d_slab, cudaStream_t s) override
    {
        const long long n = (long long)S.dims[0] * S.dims[1] * nz;
        k_synth_slab<<<unsigned(std::min<long long>((n + 255) / 256, 148LL * 64)), 256, 0, s>>>(S, z0, nz, d_slab);
        SVDB_CUDA(cudaGetLastError());
        return 0;
    }
};

struct CallbackSource : SlabSource {
    SlabFn fn = nullptr;
    void* user = nullptr;
    int dims[3] = {0, 0, 0};
    float* pinned = nullptr;
    ~CallbackSource() override { cudaFreeHost(pinned); }
    int produce(int z0, int nz, float* d_slab, cudaStream_t s) override
    {
        const size_t bytes = size_t(dims[0]) * size_t(dims[1]) * size_t(nz) * sizeof(float);
        if (!pinned)
            SVDB_CUDA(cudaMallocHost(&pinned, size_t(dims[0]) * size_t(dims[1]) * kSlab * sizeof(float)));
        SVDB_CUDA(cudaStreamSynchronize(s)); // the previous slab's copy has left the pinned buffer
        if (int rc = fn(user, z0, nz, pinned))
            return fail(Errc::io_error, "slab callback returned " + std::to_string(rc));
        SVDB_CUDA(cudaMemcpyAsync(d_slab, pinned, bytes, cudaMemcpyHostToDevice, s));
        return 0;
    }
};

template <typename T>
struct DevArr {
    T* p = nullptr;
    ~DevArr() { cudaFree(p); }
    int alloc(size_t n)
    {
        SVDB_CUDA(cudaMalloc(&p, (n ? n : 1) * sizeof(T)));
        return 0;
    }
};

int grid_for(long long n, int threads = 256) { return int(std::min<long long>((n + threads - 1) / threads, 148LL * 32)); }

int encode(SlabSource& src, const int32_t dims[3], int voxel_type, double quality, int metric, HostBuf& out,
           svdbgpu_compress_report* rep)
{
    NvtxRange nvtx("svdbgpu streaming encoder");
    const int dx = dims[0], dy = dims[1], dz = dims[2];
    const long long slab_vox = (long long)dx * dy * kSlab;
    const int nslabs = (dz + kSlab - 1) / kSlab;
    const int nbx = (dx + kEncBrick - 1) / kEncBrick, nby = (dy + kEncBrick - 1) / kEncBrick,
              nbz = (dz + kEncBrick - 1) / kEncBrick;
    const size_t nbricks = size_t(nbx) * nby * nbz;
    const int lx = (dx + 7) / 8, ly = (dy + 7) / 8, lz = (dz + 7) / 8;
    const size_t nblk = size_t(lx) * ly * lz;
    cudaStream_t s = nullptr;
    SVDB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    DevArr<float> slab, blo, bhi, sel, sel_alt, uniq;
    DevArr<int> d_mm;
    DevArr<unsigned long long> hist, cnt, counts;
    DevArr<int> nruns;
    int arc = 0;
    if ((arc = slab.alloc(size_t(slab_vox))) || (arc = blo.alloc(nbricks)) || (arc = bhi.alloc(nbricks)) ||
        (arc = d_mm.alloc(3)) || (arc = hist.alloc(1024)) || (arc = cnt.alloc(1)))
        return arc;
    auto for_slabs = [&](auto&& body) -> int {
        for (int k = 0; k < nslabs; ++k) {
            const int z0 = k * kSlab, nz = std::min(kSlab, dz - z0);
            if (int rc = src.produce(z0, nz, slab.p, s))
                return rc;
            if (int rc = body(z0, nz))
                return rc;
        }
        return 0;
    };

    // 1. min / max / finite + brick ranges
    {
        const int init[3] = {0x7fffffff, int(0x80000000), 0};
        SVDB_CUDA(cudaMemcpyAsync(d_mm.p, init, sizeof init, cudaMemcpyHostToDevice, s));
        if (int rc = for_slabs([&](int z0, int nz) {
                const long long n = (long long)dx * dy * nz;
                k_stats<<<grid_for(n), 256, 0, s>>>(slab.p, n, d_mm.p, d_mm.p + 1, d_mm.p + 2);
                k_brick_ranges<<<unsigned(nbx * nby), 256, 0, s>>>(slab.p, dx, dy, dz, z0, nbx, nby, blo.p, bhi.p);
                SVDB_CUDA(cudaGetLastError());
                return 0;
            }))
            return rc;
    }
    int mm[3];
    SVDB_CUDA(cudaMemcpyAsync(mm, d_mm.p, sizeof mm, cudaMemcpyDeviceToHost, s));
    SVDB_CUDA(cudaStreamSynchronize(s));
    if (mm[2])
        return fail(Errc::non_finite_voxel, "volume contains NaN or Inf");
    const float vmin = ford_inv(mm[0]), vmax = ford_inv(mm[1]);

    // 2. histogram + modal bin (volume.hpp:177-206)
    const int bins = voxel_type == 0 ? 256 : 1024;
    const double hlo = vmin, hhi = vmax;
    SVDB_CUDA(cudaMemsetAsync(hist.p, 0, 1024 * sizeof(unsigned long long), s));
    if (int rc = for_slabs([&](int, int nz) {
            const long long n = (long long)dx * dy * nz;
            k_hist<<<grid_for(n), 256, 0, s>>>(slab.p, n, hlo, hhi, bins, hist.p);
            SVDB_CUDA(cudaGetLastError());
            return 0;
        }))
        return rc;
    std::vector<unsigned long long> h(static_cast<size_t>(bins));
    SVDB_CUDA(cudaMemcpyAsync(h.data(), hist.p, size_t(bins) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    SVDB_CUDA(cudaStreamSynchronize(s));
    int best_bin = 0;
    for (int i = 1; i < bins; ++i)
        if (h[size_t(i)] > h[size_t(best_bin)])
            best_bin = i;

    // 3. exact counts within the modal bin (detect_background, volume.hpp:208-222): the bin's values
    //    of each slab are gathered, sorted and run-length encoded on the device
    std::unordered_map<float, uint64_t> exact;
    {
        if ((arc = sel.alloc(size_t(slab_vox))) || (arc = sel_alt.alloc(size_t(slab_vox))) ||
            (arc = uniq.alloc(size_t(slab_vox))) || (arc = counts.alloc(size_t(slab_vox))) || (arc = nruns.alloc(1)))
            return arc;
        size_t sort_tmp = 0, rle_tmp = 0;
        cub::DoubleBuffer<float> keys(sel.p, sel_alt.p);
        cub::DeviceRadixSort::SortKeys(nullptr, sort_tmp, keys, int(slab_vox));
        cub::DeviceRunLengthEncode::Encode(nullptr, rle_tmp, sel.p, uniq.p, counts.p, nruns.p, int(slab_vox));
        DevArr<uint8_t> tmp;
        if (int rc = tmp.alloc(std::max(sort_tmp, rle_tmp)))
            return rc;
        std::vector<float> hu;
        std::vector<unsigned long long> hc;
        if (int rc = for_slabs([&](int, int nz) {
                const long long n = (long long)dx * dy * nz;
                SVDB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), s));
                k_select_bin<<<grid_for(n), 256, 0, s>>>(slab.p, n, hlo, hhi, bins, best_bin, sel.p, cnt.p);
                unsigned long long m = 0;
                SVDB_CUDA(cudaMemcpyAsync(&m, cnt.p, sizeof m, cudaMemcpyDeviceToHost, s));
                SVDB_CUDA(cudaStreamSynchronize(s));
                if (!m)
                    return 0;
                cub::DoubleBuffer<float> kb(sel.p, sel_alt.p);
                size_t t1 = sort_tmp;
                SVDB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, t1, kb, int(m), 0, 32, s));
                size_t t2 = rle_tmp;
                SVDB_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, t2, kb.Current(), uniq.p, counts.p, nruns.p, int(m), s));
                int r = 0;
                SVDB_CUDA(cudaMemcpyAsync(&r, nruns.p, sizeof r, cudaMemcpyDeviceToHost, s));
                SVDB_CUDA(cudaStreamSynchronize(s));
                hu.resize(size_t(r));
                hc.resize(size_t(r));
                SVDB_CUDA(cudaMemcpyAsync(hu.data(), uniq.p, size_t(r) * sizeof(float), cudaMemcpyDeviceToHost, s));
                SVDB_CUDA(cudaMemcpyAsync(hc.data(), counts.p, size_t(r) * sizeof(unsigned long long),
                                          cudaMemcpyDeviceToHost, s));
                SVDB_CUDA(cudaStreamSynchronize(s));
                for (int i = 0; i < r; ++i)
                    exact[hu[size_t(i)]] += hc[size_t(i)];
                return 0;
            }))
            return rc;
        cudaFree(sel_alt.p);
        sel_alt.p = nullptr;
        cudaFree(uniq.p);
        uniq.p = nullptr;
        cudaFree(counts.p);
        counts.p = nullptr;
    }
    bool have = false;
    float bg = 0.0f;
    uint64_t best_count = 0;
    for (auto& [val, c] : exact)
        if (!have || c > best_count || (c == best_count && val < bg)) {
            have = true;
            bg = val;
            best_count = c;
        }

    // host: brick order + budget (compress.hpp:97-145, 237-251)
    std::vector<float> hlo_b(nbricks), hhi_b(nbricks);
    SVDB_CUDA(cudaMemcpyAsync(hlo_b.data(), blo.p, nbricks * sizeof(float), cudaMemcpyDeviceToHost, s));
    SVDB_CUDA(cudaMemcpyAsync(hhi_b.data(), bhi.p, nbricks * sizeof(float), cudaMemcpyDeviceToHost, s));
    SVDB_CUDA(cudaStreamSynchronize(s));
    std::vector<uint8_t> chosen;
    uint64_t budget = 0, voxels_activated = 0;
    choose_bricks(dims, hlo_b.data(), hhi_b.data(), bg, metric, quality, chosen, budget, voxels_activated);

    // 4. per-block decision on the device
    DevArr<uint8_t> d_chosen, d_state;
    DevArr<float> d_tile;
    if ((arc = d_chosen.alloc(nbricks)) || (arc = d_state.alloc(nblk)) || (arc = d_tile.alloc(nblk)))
        return arc;
    SVDB_CUDA(cudaMemcpyAsync(d_chosen.p, chosen.data(), nbricks, cudaMemcpyHostToDevice, s));
    if (int rc = for_slabs([&](int z0, int nz) {
            const long long nb = (long long)lx * ly * ((nz + 7) / 8);
            k_block_state<<<grid_for(nb * 32), 256, 0, s>>>(slab.p, dx, dy, dz, z0, nz, d_chosen.p, nbx, nby, bg,
                                                             d_state.p, d_tile.p);
            SVDB_CUDA(cudaGetLastError());
            return 0;
        }))
        return rc;
    std::vector<uint8_t> state(nblk);
    std::vector<float> tile_val(nblk);
    SVDB_CUDA(cudaMemcpyAsync(state.data(), d_state.p, nblk, cudaMemcpyDeviceToHost, s));
    SVDB_CUDA(cudaMemcpyAsync(tile_val.data(), d_tile.p, nblk * sizeof(float), cudaMemcpyDeviceToHost, s));
    SVDB_CUDA(cudaStreamSynchronize(s));

    // host: prune, indices, header / root / upper / lower records (write_tree, shared with compress)
    std::vector<uint32_t> leaf_index;
    uint64_t n_leaf = 0, leaf_offset = 0;
    write_tree(dims, voxel_type, bg, vmin, vmax, state, tile_val, 0, out, leaf_index, n_leaf, leaf_offset);

    // 5. leaf records, slab by slab, copied into place (leaf order = block order = slab order)
    if (n_leaf) {
        DevArr<uint32_t> d_index;
        DevArr<uint8_t> recs;
        const size_t slab_blocks = size_t(lx) * ly * (kSlab / 8);
        if ((arc = d_index.alloc(nblk)) || (arc = recs.alloc(slab_blocks * kLeafRecBytes)))
            return arc;
        SVDB_CUDA(cudaMemcpyAsync(d_index.p, leaf_index.data(), nblk * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        uint64_t next = 0; // first leaf index of the current slab
        if (int rc = for_slabs([&](int z0, int nz) {
                size_t b0 = size_t(lx) * ly * size_t(z0 / 8), b1 = size_t(lx) * ly * size_t(std::min(lz, (z0 + nz + 7) / 8));
                uint64_t cnt_leaf = 0;
                for (size_t b = b0; b < b1; ++b)
                    cnt_leaf += state[b] == kBlkLeaf || state[b] == kBlkCornerLeaf;
                if (!cnt_leaf)
                    return 0;
                const long long nb = (long long)lx * ly * ((nz + 7) / 8);
                k_leaf_records<<<grid_for(nb * 32), 256, 0, s>>>(slab.p, dx, dy, dz, z0, nz, d_state.p, d_index.p, next,
                                                                  bg, recs.p);
                SVDB_CUDA(cudaGetLastError());
                SVDB_CUDA(cudaMemcpyAsync(out.p + leaf_offset + next * kLeafRecBytes, recs.p, cnt_leaf * kLeafRecBytes,
                                          cudaMemcpyDeviceToHost, s));
                SVDB_CUDA(cudaStreamSynchronize(s));
                next += cnt_leaf;
                return 0;
            }))
            return rc;
    }
    if (rep) {
        rep->background = bg;
        rep->num_bricks = uint64_t(nbricks);
        rep->bricks_activated = budget;
        rep->voxels_activated = voxels_activated;
        rep->frozen_bytes = out.n;
        rep->dense_bytes = uint64_t(dx) * uint64_t(dy) * uint64_t(dz) * 4;
        rep->achieved_ratio = double(out.n) / double(rep->dense_bytes);
    }
    return 0;
}

int check_args(const int32_t dims[3], int voxel_type, double quality, int metric, int device)
{
    if (!(quality >= 0.0 && quality <= 1.0))
        return fail(Errc::invalid_quality, "quality must be in [0,1]");
    if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
        return fail(Errc::size_mismatch, "volume dims must be positive");
    if (voxel_type != 0 && voxel_type != 1)
        return fail(Errc::size_mismatch, "voxel_type must be 0 (u8) or 1 (f32)");
    if (metric < 0 || metric > 2)
        return fail_code(SVDBGPU_E_INVALID_ARG, "metric must be 0..2");
    int ndev = 0;
    SVDB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail_code(SVDBGPU_E_INVALID_ARG, "device out of range");
    SVDB_CUDA(cudaSetDevice(device));
    return 0;
}

} // namespace

int stream_compress_synth(int kind, const int32_t dims[3], uint64_t seed, double quality, int metric, int device,
                          HostBuf& out, svdbgpu_compress_report* rep, double* seconds)
{
    if (kind < 1 || kind > 3)
        return fail_code(SVDBGPU_E_UNSUPPORTED, "streaming synthesis covers the fBm-based volumes (kinds 1-3); "
                                                "Marschner-Lobb needs the host libm (use svdbgpu_synth + svdbgpu_compress)");
    const int voxel_type = kind == 1 ? 0 : 1;
    if (int rc = check_args(dims, voxel_type, quality, metric, device))
        return rc;
    const auto t0 = std::chrono::steady_clock::now();
    SynthSource src;
    if (int rc = src.init(kind, dims, seed))
        return rc;
    int rc = encode(src, dims, voxel_type, quality, metric, out, rep);
    if (seconds)
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

int stream_compress_callback(SlabFn fn, void* user, const int32_t dims[3], int voxel_type, double quality, int metric,
                             int device, HostBuf& out, svdbgpu_compress_report* rep, double* seconds)
{
    if (!fn)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null slab callback");
    if (int rc = check_args(dims, voxel_type, quality, metric, device))
        return rc;
    const auto t0 = std::chrono::steady_clock::now();
    CallbackSource src;
    src.fn = fn;
    src.user = user;
    for (int a = 0; a < 3; ++a)
        src.dims[a] = dims[a];
    int rc = encode(src, dims, voxel_type, quality, metric, out, rep);
    if (seconds)
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

} // namespace svdbgpu
