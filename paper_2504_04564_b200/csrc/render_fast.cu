// render_fast.cu — k_trace_f: the persistent path-regenerating tracer of render.cu with the
// tracking arithmetic in FP32 (SVDBGPU_PRECISION_FP32).
//
// Same algorithm, state machine and per-(pixel, sample) draw order as the FP64 kernel — which
// follows render.hpp:100-187 (woodcock_track, next_event, trace_path) and dda.hpp:52-109 — but
// ray, DDA, step lengths, trilinear weights, transfer function and throughput in single
// precision: uniforms are the top 24 bits of the same splitmix64 outputs (rng.hpp:54-63), the
// step uses the hardware log2. Decoded voxel values are unchanged (same device.cuh decode). A
// sample-position or step length differing in the last float bits can flip a rare accept or
// cell-exit decision, after which that one path follows other draws, so the image matches the
// FP64 / reference image within the north-star tolerance (relative RMSE <= 1e-3 at matched
// streams and spp, tests/test_gpu_fast.py) instead of bit for bit. Per-pixel accumulation stays in
// FP64 in sample order (render.hpp:297-310).
//
// Why: the FP64 kernel is bound by the latency of its FP64 dependency chains and by register /
// shared-memory capacity (24 warps per SM); here the per-lane state halves (204 B of shared memory
// per lane), 32 warps per SM fit, and the step / DDA / sampler chains run on the FP32 pipes.
// This TU is compiled with FMA contraction on (the FP64 TUs use -fmad=false).
#include "device.cuh"
#include "render_args.hpp"
#include "svdbgpu.h"

#include <algorithm>

namespace svdbgpu {

namespace {

constexpr int kT = 64;          // threads per CTA
constexpr int kMinBlocks = 16;  // 32 warps per SM
constexpr int kAdvIters = 3;    // advance steps per advance-phase invocation
constexpr unsigned kFull = 0xffffffffu;

enum : int { kNeedPixel = 0, kNeedPath = 1, kNeedSegment = 2, kNeedCell = 3, kInCell = 4, kPoint = 5, kScatter = 6 };

struct RayF {
    float o[3], d[3];
};

// splitmix64 uniform (rng.hpp:54-63) truncated to 24 bits: the float just below the double draw
__device__ __forceinline__ float u24(uint64_t x)
{
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return float(uint32_t(x >> 40)) * 0x1.0p-24f;
}

struct RngF {
    uint64_t state;
    __device__ __forceinline__ float uniform()
    {
        state += 0x9E3779B97F4A7C15ull;
        return u24(state);
    }
    __device__ __forceinline__ float peek() const { return u24(state + 0x9E3779B97F4A7C15ull); }
    __device__ __forceinline__ void skip() { state += 0x9E3779B97F4A7C15ull; }
};

__device__ __forceinline__ float kInfF() { return __int_as_float(0x7f800000); }

// transfer.hpp:47-67 in float; lo / 1/(hi-lo) / scale converted once per launch
struct TfF {
    float lo, inv_range, scale;
    int n;
    const float4* ent;
    __device__ __forceinline__ float u_of(float v) const
    {
        return fminf(fmaxf((v - lo) * inv_range, 0.0f), 1.0f) * float(n - 1);
    }
    __device__ __forceinline__ float extinction(float v) const
    {
        const float u = u_of(v);
        const int i0 = min(int(u), n - 2);
        const float t = u - float(i0);
        return scale * ((1.0f - t) * ent[i0].w + t * ent[i0 + 1].w);
    }
    __device__ __forceinline__ void rgb(float v, float out[3]) const
    {
        const float u = u_of(v);
        const int i0 = min(int(u), n - 2);
        const float t = u - float(i0);
        const float4 a = ent[i0], b = ent[i0 + 1];
        out[0] = (1.0f - t) * a.x + t * b.x;
        out[1] = (1.0f - t) * a.y + t * b.y;
        out[2] = (1.0f - t) * a.z + t * b.z;
    }
};

__device__ __forceinline__ int lattice_coord_f(float v)
{
    const float f = floorf(v);
    return f < -1.0e9f ? -1000000000 : (f > 1.0e9f ? 1000000000 : int(f));
}

// sample_trilinear (sample.hpp:46-72) with float weights; taps through the apron brick as in the
// FP64 sampler (device.cuh), per-tap accessor reads when the base voxel is not in a leaf
template <int CODEC>
__device__ __forceinline__ float sample_f(Accessor<CODEC>& a, float px, float py, float pz)
{
    const int x0 = lattice_coord_f(px), y0 = lattice_coord_f(py), z0 = lattice_coord_f(pz);
    const float wx = px - floorf(px), wy = py - floorf(py), wz = pz - floorf(pz);
    float v[8];
    float c0;
    if (a.locate(x0, y0, z0, c0)) {
        const int x = x0 & 7, y = y0 & 7, z = z0 & 7;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            v[k] = brick_tap_f<CODEC>(a, x + (k & 1), y + ((k >> 1) & 1), z + (k >> 2));
    } else {
        v[0] = c0;
#pragma unroll 1
        for (int i = 1; i < 8; ++i)
            v[i] = a.read(x0 + (i & 1), y0 + ((i >> 1) & 1), z0 + (i >> 2));
    }
    const float v00 = v[0] * (1.0f - wx) + v[1] * wx, v10 = v[2] * (1.0f - wx) + v[3] * wx;
    const float v01 = v[4] * (1.0f - wx) + v[5] * wx, v11 = v[6] * (1.0f - wx) + v[7] * wx;
    const float v0 = v00 * (1.0f - wy) + v10 * wy, v1 = v01 * (1.0f - wy) + v11 * wy;
    return v0 * (1.0f - wz) + v1 * wz;
}

// camera_ray (render.hpp:259-269) from the host-exact basis
__device__ __forceinline__ RayF camera_ray_f(const CamArgs& c, float px, float py)
{
    const float ndc_x = (2.0f * px / float(c.w) - 1.0f) * float(c.tan_half * c.aspect);
    const float ndc_y = (1.0f - 2.0f * py / float(c.h)) * float(c.tan_half);
    RayF r;
    float d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.o[a] = float(c.pos[a]);
        d[a] = float(c.fwd[a]) + float(c.right[a]) * ndc_x + float(c.up[a]) * ndc_y;
    }
    const float il = rsqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a)
        r.d[a] = d[a] * il;
    return r;
}

// Macrocell DDA (dda.hpp:25-109) in float, per-lane state in shared memory (SoA)
struct SharedDdaF {
    volatile int* si;   // [7][kT]: c0..2, step0..2, done
    volatile float* sf; // [8][kT]: t_next0..2, t_delta0..2, t_cur, t1
    int tid;
    __device__ __forceinline__ volatile int& ci(int k) { return si[k * kT + tid]; }
    __device__ __forceinline__ volatile float& cf(int k) { return sf[k * kT + tid]; }
    __device__ __forceinline__ bool done() { return ci(6) != 0; }
    __device__ __forceinline__ int index(const int cells[3]) { return ci(0) + cells[0] * (ci(1) + cells[1] * ci(2)); }

    __device__ __forceinline__ bool init(const int cells[3], const float hi[3], const RayF& r, float cell, float icell)
    {
        float t0 = 0.0f, t1 = kInfF();
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float o = r.o[a], d = r.d[a];
            if (d == 0.0f) {
                if (o < 0.0f || o > hi[a])
                    return false;
                continue;
            }
            const float inv = 1.0f / d;
            float ta = (0.0f - o) * inv, tb = (hi[a] - o) * inv;
            if (ta > tb) {
                const float tt = ta;
                ta = tb;
                tb = tt;
            }
            t0 = fmaxf(t0, ta);
            t1 = fminf(t1, tb);
            if (t0 > t1)
                return false;
        }
        if (!(t0 <= t1))
            return false;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float o = r.o[a], d = r.d[a];
            const int c = int(fminf(fmaxf(floorf((o + d * t0) * icell), 0.0f), float(cells[a] - 1)));
            int step = 0;
            float tn = kInfF(), td = kInfF();
            if (d != 0.0f) {
                step = d > 0.0f ? 1 : -1;
                tn = (float(d > 0.0f ? c + 1 : c) * cell - o) / d;
                td = (d > 0.0f ? cell : -cell) / d;
            }
            ci(a) = c;
            ci(3 + a) = step;
            cf(a) = tn;
            cf(3 + a) = td;
        }
        cf(6) = t0;
        cf(7) = t1;
        ci(6) = 0;
        return true;
    }

    __device__ __forceinline__ bool next(const int cells[3], float& ta, float& tb)
    {
        if (ci(6))
            return false;
        const float n0 = cf(0), n1 = cf(1), n2 = cf(2), t_cur = cf(6), t1 = cf(7);
        const bool ax1 = n1 < n0;
        const float tm = ax1 ? n1 : n0;
        const bool ax2 = n2 < tm;
        const int axis = ax2 ? 2 : (ax1 ? 1 : 0);
        const float t_exit = fmaxf(fminf(ax2 ? n2 : tm, t1), t_cur);
        ta = t_cur;
        tb = t_exit;
        if (t_exit >= t1) {
            ci(6) = 1;
            return true;
        }
        cf(6) = t_exit;
        const int c = ci(axis) + ci(3 + axis);
        ci(axis) = c;
        if (c < 0 || c >= cells[axis])
            ci(6) = 1;
        else
            cf(axis) = (axis == 0 ? n0 : (axis == 1 ? n1 : n2)) + cf(3 + axis);
        return true;
    }
};

template <int CODEC, int MODE>
__global__ void __launch_bounds__(kT, kMinBlocks) k_trace_f(const __grid_constant__ RenderArgs A, long long n_units)
{
    extern __shared__ float4 s_ent[];
    for (int i = threadIdx.x; i < A.tf.n; i += blockDim.x)
        s_ent[i] = A.tf_ent[i];
    __syncthreads();
    constexpr bool RATIO = MODE == SVDBGPU_MODE_RATIO;
    const int lane = threadIdx.x & 31;
    const int tid = threadIdx.x;
    unsigned long long* work = A.counters + 1;
    const TfF tf{float(A.tf.lo), float(1.0 / (A.tf.hi - A.tf.lo)), float(A.tf.scale), A.tf.n, s_ent};
    const float hi[3] = {float(A.hi[0]), float(A.hi[1]), float(A.hi[2])};
    const float cell = float(A.cell), icell = float(A.icell);

    // ---- per-lane state: registers for the step loop, shared memory (SoA) for the rest ----
    __shared__ int s_dda_i[7][kT];
    __shared__ float s_dda_f[8][kT];
    SharedDdaF dda{&s_dda_i[0][0], &s_dda_f[0][0], tid};
    __shared__ float s_ray[6][kT];
    __shared__ int s_acc[14][kT];
    __shared__ double s_sum[3][kT];                    // per-pixel FP64 accumulation
    __shared__ float s_cold[RATIO ? 9 : 5][kT];        // tp0..2, t_ev, v_ev (+ L0..2, Tr)
    __shared__ int s_ci[RATIO ? 6 : 5][kT];            // px, py, s, bounces, out_off (+ have)
    volatile float* cold = &s_cold[0][tid];
    volatile int* ci = &s_ci[0][tid];
    volatile double* sum = &s_sum[0][tid];
    auto tp = [&](int k) -> volatile float& { return cold[k * kT]; };
    volatile float& t_ev = cold[3 * kT];
    volatile float& v_ev = cold[4 * kT];
    auto Lr = [&](int k) -> volatile float& { return cold[(5 + k) * kT]; }; // ratio only
    volatile float& Tr = cold[(RATIO ? 8 : 0) * kT];                          // ratio only
    volatile int &px = ci[0], &py = ci[kT], &s = ci[2 * kT], &bounces = ci[3 * kT], &out_off = ci[4 * kT];
    volatile int& have = ci[(RATIO ? 5 : 0) * kT]; // ratio only

    Accessor<CODEC> acc(A.g);
    auto acc_io = [&](bool store) {
        volatile int* p = &s_acc[0][tid];
        int* f[14] = {&acc.lx, &acc.ly, &acc.lz, reinterpret_cast<int*>(&acc.leaf), reinterpret_cast<int*>(&acc.lo),
                      reinterpret_cast<int*>(&acc.sc), &acc.wx, &acc.wy, &acc.wz, reinterpret_cast<int*>(&acc.lower),
                      &acc.ux, &acc.uy, &acc.uz, &acc.upper};
#pragma unroll
        for (int k = 0; k < 14; ++k) {
            if (store)
                p[k * kT] = *f[k];
            else
                *f[k] = p[k * kT];
        }
    };
    acc_io(true);
    auto ray_load = [&]() {
        RayF r;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            r.o[k] = reinterpret_cast<volatile float*>(s_ray[k])[tid];
            r.d[k] = reinterpret_cast<volatile float*>(s_ray[3 + k])[tid];
        }
        return r;
    };
    auto ray_store = [&](const RayF& r) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            reinterpret_cast<volatile float*>(s_ray[k])[tid] = r.o[k];
            reinterpret_cast<volatile float*>(s_ray[3 + k])[tid] = r.d[k];
        }
    };

    RngF rng{0};
    float t = 0.0f, tb = 0.0f, inv = 0.0f, inv_ahead = 0.0f;
    uint32_t samples = 0;
    int state = kNeedPixel;
    bool done = false;
    long long unit = 0;
    int fill = 32;

    auto finish_path = [&](float r0, float r1, float r2) {
        sum[0] += double(r0);
        sum[kT] += double(r1);
        sum[2 * kT] += double(r2);
        s = s + 1;
        state = kNeedPath;
    };
    auto finish_ratio = [&]() { finish_path(Lr(0), Lr(1), Lr(2)); };
    // scattering vertex (render.hpp:173-185)
    auto bounce = [&](float te, float ve) {
        bounces = bounces + 1;
        if (bounces > A.max_bounces) {
            if constexpr (RATIO)
                finish_ratio();
            else
                finish_path(0.0f, 0.0f, 0.0f);
            return;
        }
        float alb[3];
        tf.rgb(ve, alb);
        float tpv[3] = {tp(0) * alb[0], tp(1) * alb[1], tp(2) * alb[2]};
        {
            RayF ray = ray_load();
            ray.o[0] += ray.d[0] * te;
            ray.o[1] += ray.d[1] * te;
            ray.o[2] += ray.d[2] * te;
            const float u0 = rng.uniform(), u1 = rng.uniform();
            const float z = 1.0f - 2.0f * u0;
            const float r = sqrtf(fmaxf(0.0f, 1.0f - z * z));
            float sp, cp;
            sincospif(2.0f * u1, &sp, &cp);
            ray.d[0] = r * cp;
            ray.d[1] = r * sp;
            ray.d[2] = z;
            ray_store(ray);
        }
        if (bounces >= A.rr_start) {
            const float survive = fminf(fmaxf(fmaxf(tpv[0], fmaxf(tpv[1], tpv[2])), 0.05f), 0.95f);
            if (rng.uniform() >= survive) {
                if constexpr (RATIO)
                    finish_ratio();
                else
                    finish_path(0.0f, 0.0f, 0.0f);
                return;
            }
            const float is = 1.0f / survive;
            tpv[0] *= is;
            tpv[1] *= is;
            tpv[2] *= is;
        }
        tp(0) = tpv[0];
        tp(1) = tpv[1];
        tp(2) = tpv[2];
        state = kNeedSegment;
    };
    auto end_segment = [&]() {
        if constexpr (RATIO) {
            const float tr = Tr;
            Lr(0) = Lr(0) + tp(0) * tr * A.ambient[0];
            Lr(1) = Lr(1) + tp(1) * tr * A.ambient[1];
            Lr(2) = Lr(2) + tp(2) * tr * A.ambient[2];
            if (!have)
                finish_ratio();
            else
                state = kScatter;
        } else {
            finish_path(tp(0) * A.ambient[0], tp(1) * A.ambient[1], tp(2) * A.ambient[2]);
        }
    };
    auto do_start = [&]() {
        if (state == kScatter) {
            bounce(t_ev, v_ev);
            if (state == kNeedSegment)
                goto segment;
        }
        if (state == kNeedPath) {
            if (s == A.spp) {
                const double inv_spp = 1.0 / double(A.spp);
                A.out[out_off] = float(sum[0] * inv_spp);
                A.out[out_off + 1] = float(sum[kT] * inv_spp);
                A.out[out_off + 2] = float(sum[2 * kT] * inv_spp);
                state = kNeedPixel;
                return;
            }
            {
                const Rng r0 = Rng::for_pixel_sample(A.seed_mixed, px, py, s);
                rng.state = r0.state;
            }
            const float jx = rng.uniform(), jy = rng.uniform();
            ray_store(camera_ray_f(A.cam, float(px) + jx, float(py) + jy));
            tp(0) = tp(1) = tp(2) = 1.0f;
            bounces = 0;
            if constexpr (RATIO)
                Lr(0) = Lr(1) = Lr(2) = 0.0f;
            state = kNeedSegment;
        }
    segment:
        if constexpr (RATIO) {
            Tr = 1.0f;
            have = 0;
        }
        if (!dda.init(A.cells, hi, ray_load(), cell, icell)) {
            end_segment();
            return;
        }
        inv_ahead = __ldg(A.inv_maj_f + dda.index(A.cells));
        state = kNeedCell;
    };
    // kNeedCell -> next macrocell (empty cells draw nothing); kInCell -> one tentative step
    auto do_advance = [&]() {
        const float lg = __log2f(1.0f - rng.peek()); // step draw, consumed only where it is used
        if (state == kNeedCell) {
            float ta, tbb;
            if ((RATIO && !(Tr > 0.0f)) || !dda.next(A.cells, ta, tbb)) {
                end_segment();
                return;
            }
            inv = inv_ahead;
            if (!dda.done())
                inv_ahead = __ldg(A.inv_maj_f + dda.index(A.cells));
            if (!(inv > 0.0f))
                return;
            t = ta;
            tb = tbb;
        }
        rng.skip();
        t -= lg * 0.693147182f * inv;
        state = t >= tb ? kNeedCell : kPoint;
    };
    auto accept = [&](float v) {
        const float st = tf.extinction(v);
        if constexpr (RATIO) {
            const float r = st * inv;
            if (!have && rng.uniform() < r) {
                have = 1;
                t_ev = t;
                v_ev = v;
            }
            const float tr = Tr * (1.0f - r);
            Tr = tr;
            if (!(tr > 0.0f))
                end_segment();
            else
                state = kInCell;
        } else {
            if (rng.uniform() < st * inv) {
                t_ev = t;
                v_ev = v;
                state = kScatter;
            } else {
                state = kInCell;
            }
        }
    };
    auto do_sample = [&]() {
        acc_io(false);
        const RayF r = ray_load();
        ++samples;
        const float v = sample_f<CODEC>(acc, r.o[0] + r.d[0] * t, r.o[1] + r.d[1] * t, r.o[2] + r.d[2] * t);
        acc_io(true);
        accept(v);
    };

    for (;;) {
        // ---- hand out pixels: 8x4 blocks per warp from the global counter ----
        unsigned need = __ballot_sync(kFull, state == kNeedPixel && !done);
        while (need) {
            if (fill >= 32) {
                unsigned long long u = 0;
                if (lane == 0)
                    u = atomicAdd(work, 1ull);
                unit = (long long)__shfl_sync(kFull, u, 0);
                fill = 0;
                if (unit >= n_units) {
                    if ((need >> lane) & 1u)
                        done = true;
                    break;
                }
            }
            const int below = __popc(need & ((1u << lane) - 1u));
            const int avail = 32 - fill;
            if (((need >> lane) & 1u) && below < avail) {
                const int p = fill + below;
                const long long k = unit >> 3;
                const int w = int(unit & 7);
                const int lx = (w & 1) * 8 + (p & 7), ly = (w >> 1) * 4 + (p >> 3);
                const long long tt = k * A.nranks + A.rank;
                const int qx = int(tt % A.tiles_x) * 16 + lx, qy = int(tt / A.tiles_x) * 16 + ly;
                if (qx < A.cam.w && qy < A.cam.h) {
                    px = qx;
                    py = qy;
                    out_off = int(A.packed ? (k * 256 + ly * 16 + lx) * 3 : ((long long)qy * A.cam.w + qx) * 3);
                    s = 0;
                    sum[0] = sum[kT] = sum[2 * kT] = 0.0;
                    state = kNeedPath;
                }
            }
            const int take = min(__popc(need), avail);
            fill += take;
            for (int i = 0; i < take; ++i)
                need &= need - 1u;
        }
        const unsigned live = __ballot_sync(kFull, !done);
        if (live == 0)
            break;
        if (done)
            continue;
        // ---- run the phase most lanes are waiting in ----
        const int nS = __popc(__ballot_sync(live, state == kPoint));
        const int nA = __popc(__ballot_sync(live, state == kNeedCell || state == kInCell));
        const int nT = __popc(__ballot_sync(live, state == kNeedPath || state == kNeedSegment || state == kScatter));
        if (nS >= nA && nS >= nT) {
            if (state == kPoint)
                do_sample();
        } else if (nA >= nT) {
#pragma unroll 1
            for (int k = 0; k < kAdvIters && (state == kNeedCell || state == kInCell); ++k)
                do_advance();
        } else if (state == kNeedPath || state == kNeedSegment || state == kScatter) {
            do_start();
        }
    }
    unsigned long long s64 = samples;
#pragma unroll
    for (int off = 16; off; off >>= 1)
        s64 += __shfl_xor_sync(kFull, s64, off);
    if (lane == 0 && s64)
        atomicAdd(A.counters, s64);
}

template <int CODEC, int MODE>
int launch(const RenderArgs& A, long long n_units, size_t smem, cudaStream_t s)
{
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trace_f<CODEC, MODE>, kT, smem);
    const long long blocks = std::min<long long>((long long)std::max(per_sm, 1) * sms, (n_units * 32 + kT - 1) / kT);
    k_trace_f<CODEC, MODE><<<unsigned(blocks), kT, smem, s>>>(A, n_units);
    return 0;
}

} // namespace

int launch_trace_fast(const RenderArgs& A, int codec, int mode, long long n_units, size_t smem, cudaStream_t s)
{
    const bool ratio = mode == SVDBGPU_MODE_RATIO;
    switch (codec) {
    case kCodecF32: return ratio ? launch<kCodecF32, SVDBGPU_MODE_RATIO>(A, n_units, smem, s)
                                 : launch<kCodecF32, SVDBGPU_MODE_PATHTRACE>(A, n_units, smem, s);
    case kCodecUnorm8: return ratio ? launch<kCodecUnorm8, SVDBGPU_MODE_RATIO>(A, n_units, smem, s)
                                    : launch<kCodecUnorm8, SVDBGPU_MODE_PATHTRACE>(A, n_units, smem, s);
    case kCodecAffine8: return ratio ? launch<kCodecAffine8, SVDBGPU_MODE_RATIO>(A, n_units, smem, s)
                                     : launch<kCodecAffine8, SVDBGPU_MODE_PATHTRACE>(A, n_units, smem, s);
    default: return ratio ? launch<kCodecAffine4, SVDBGPU_MODE_RATIO>(A, n_units, smem, s)
                          : launch<kCodecAffine4, SVDBGPU_MODE_PATHTRACE>(A, n_units, smem, s);
    }
}

} // namespace svdbgpu
