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
#include <type_traits>


namespace svdbgpu {

namespace {

constexpr int kT = 64;          // threads per CTA
constexpr int kMinBlocks = 16;                           // 32 warps per SM (pure FP32)
constexpr int kMinBlocksMixed = 14; // FP64 geometry: 212 B of shared state per lane
constexpr int kAdvIters = 3;       // advance steps per advance-phase invocation
constexpr unsigned kFull = 0xffffffffu;

enum : int { kNeedPixel = 0, kNeedPath = 1, kNeedSegment = 2, kNeedCell = 3, kInCell = 4, kPoint = 5, kScatter = 6,
             kEscape = 7 }; // flight over: result written in the start phase (as render.cu's k_trace)

// geometry type G: float (pure FP32) or double (FP64 ray / DDA / t, FP32 everything else)
template <typename G>
struct RayG {
    G o[3], d[3];
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
    __device__ __forceinline__ double uniform53() // the reference's draw (rng.hpp:54-63)
    {
        state += 0x9E3779B97F4A7C15ull;
        uint64_t x = state;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        x ^= x >> 31;
        return double(x >> 11) * 0x1.0p-53;
    }
    __device__ __forceinline__ void skip() { state += 0x9E3779B97F4A7C15ull; }
};

template <typename G>
__device__ __forceinline__ G kInfG() { return G(__int_as_float(0x7f800000)); }
template <typename G>
__device__ __forceinline__ G gmin(G a, G b) { return b < a ? b : a; }
template <typename G>
__device__ __forceinline__ G gmax(G a, G b) { return a < b ? b : a; }

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

template <typename G>
__device__ __forceinline__ int lattice_coord_g(G f) // f = floor(v)
{
    return f < G(-1.0e9) ? -1000000000 : (f > G(1.0e9) ? 1000000000 : int(f));
}

// sample_trilinear (sample.hpp:46-72) with float weights; taps through the apron brick as in the
// FP64 sampler (device.cuh), per-tap accessor reads when the base voxel is not in a leaf
template <int CODEC, typename G>
__device__ __forceinline__ float sample_f(Accessor<CODEC>& a, G px, G py, G pz)
{
    const G fx = floor(px), fy = floor(py), fz = floor(pz);
    const int x0 = lattice_coord_g(fx), y0 = lattice_coord_g(fy), z0 = lattice_coord_g(fz);
    const float wx = float(px - fx), wy = float(py - fy), wz = float(pz - fz);
    float v[8];
    float c0;
    if (a.locate(x0, y0, z0, c0)) {
        brick_gather<CODEC>(a, x0 & 7, y0 & 7, z0 & 7, v);
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
template <typename G>
__device__ __forceinline__ RayG<G> camera_ray_g(const CamArgs& c, G px, G py)
{
    const G ndc_x = (G(2) * px / G(c.w) - G(1)) * G(c.tan_half) * G(c.aspect);
    const G ndc_y = (G(1) - G(2) * py / G(c.h)) * G(c.tan_half);
    RayG<G> r;
    G d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.o[a] = G(c.pos[a]);
        d[a] = G(c.fwd[a]) + G(c.right[a]) * ndc_x + G(c.up[a]) * ndc_y;
    }
    const G len = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a)
        r.d[a] = d[a] / len;
    return r;
}

// Macrocell DDA (dda.hpp:25-109) in float, per-lane state in shared memory (SoA)
template <typename G>
struct SharedDdaG {
    volatile int* si; // [7][kT]: c0..2, step0..2, (unused)
    volatile G* sf;   // [8][kT]: t_next0..2, t_delta0..2, t_cur, t1
    int tid;
    __device__ __forceinline__ volatile int& ci(int k) { return si[k * kT + tid]; }
    __device__ __forceinline__ volatile G& cf(int k) { return sf[k * kT + tid]; }
    __device__ __forceinline__ int index(const int cells[3]) { return ci(0) + cells[0] * (ci(1) + cells[1] * ci(2)); }

    __device__ __forceinline__ bool init(const int cells[3], const G hi[3], const RayG<G>& r, G cell, G icell)
    {
        G t0 = G(0), t1 = kInfG<G>();
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const G o = r.o[a], d = r.d[a];
            if (d == G(0)) {
                if (o < G(0) || o > hi[a])
                    return false;
                continue;
            }
            const G inv = G(1) / d;
            G ta = (G(0) - o) * inv, tb = (hi[a] - o) * inv;
            if (ta > tb) {
                const G tt = ta;
                ta = tb;
                tb = tt;
            }
            t0 = gmax(t0, ta);
            t1 = gmin(t1, tb);
            if (t0 > t1)
                return false;
        }
        if (!(t0 <= t1))
            return false;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const G o = r.o[a], d = r.d[a];
            const int c = int(gmin(gmax(G(floor((o + d * t0) * icell)), G(0)), G(cells[a] - 1)));
            int step = 0;
            G tn = kInfG<G>(), td = kInfG<G>();
            if (d != G(0)) {
                step = d > G(0) ? 1 : -1;
                tn = (G(d > G(0) ? c + 1 : c) * cell - o) / d;
                td = (d > G(0) ? cell : -cell) / d;
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

    // One cell visit of a walk known not to be over (the caller's lookahead register says so),
    // walk position in the caller's tb register; reports whether the walk is over after this
    // visit, else the next cell's linear index (as k_trace's SharedDda::next_ahead).
    __device__ __forceinline__ void next_ahead(const int cells[3], G& ta, G& tb, bool& over, int& ahead)
    {
        const G n0 = cf(0), n1 = cf(1), n2 = cf(2), t_cur = tb, t1 = cf(7);
        const bool ax1 = n1 < n0;
        const G tm = ax1 ? n1 : n0;
        const bool ax2 = n2 < tm;
        const int axis = ax2 ? 2 : (ax1 ? 1 : 0);
        const G tn = ax2 ? n2 : tm;
        const G t_exit = gmax(gmin(tn, t1), t_cur);
        int c0 = ci(0), c1 = ci(1), c2 = ci(2);
        ta = t_cur;
        tb = t_exit;
        over = true;
        ahead = 0;
        if (t_exit >= t1)
            return;
        const int c = (ax2 ? c2 : (ax1 ? c1 : c0)) + ci(3 + axis);
        ci(axis) = c;
        if (c < 0 || c >= cells[axis])
            return;
        cf(axis) = tn + cf(3 + axis);
        c0 = axis == 0 ? c : c0;
        c1 = axis == 1 ? c : c1;
        c2 = axis == 2 ? c : c2;
        over = false;
        ahead = c0 + cells[0] * (c1 + cells[1] * c2);
    }
};

template <int CODEC, int MODE, typename G, bool CHUNK>
__global__ void __launch_bounds__(kT, sizeof(G) == 4 ? kMinBlocks : kMinBlocksMixed)
    k_trace_f(const __grid_constant__ RenderArgs A, long long n_units)
{
    extern __shared__ float4 s_tf[];
    const float4* s_ent = s_tf;
    if (A.tf.n > kTfSmemMax) { // large tables are read in place (L1-cached)
        s_ent = A.tf_ent;
    } else {
        for (int i = threadIdx.x; i < A.tf.n; i += blockDim.x)
            s_tf[i] = A.tf_ent[i];
        __syncthreads();
    }
    constexpr bool RATIO = MODE == SVDBGPU_MODE_RATIO;
    const int lane = threadIdx.x & 31;
    const int tid = threadIdx.x;
    unsigned long long* work = A.counters + 1;
    const TfF tf{float(A.tf.lo), float(1.0 / (A.tf.hi - A.tf.lo)), float(A.tf.scale), A.tf.n, s_ent};
    const G hi[3] = {G(A.hi[0]), G(A.hi[1]), G(A.hi[2])};
    const G cell = G(A.cell), icell = G(A.icell);
    using Ray = RayG<G>;

    // ---- per-lane state: registers for the step loop, shared memory (SoA) for the rest ----
    __shared__ int s_dda_i[7][kT];
    __shared__ G s_dda_f[8][kT];
    SharedDdaG<G> dda{&s_dda_i[0][0], &s_dda_f[0][0], tid};
    __shared__ G s_ray[6][kT];
    __shared__ G s_tev[kT];
    // no accessor state between gathers (cold locate = one directory load): its per-lane state
    // would otherwise cost CTAs per SM
    __shared__ double s_sum[3][kT];                    // per-pixel FP64 accumulation
    __shared__ float s_cold[RATIO ? 8 : 5][kT];        // tp0..2, (unused), v_ev (+ L0..2)
    // ratio transmittance stays FP64: a float product underflows to 0 (ending the flight) long
    // before the reference's double does, which would change the draws that follow
    __shared__ double s_tr[RATIO ? kT : 1];
    __shared__ int s_ci[5 + (RATIO ? 1 : 0) + (CHUNK ? 1 : 0)][kT]; // px, py, s, bounces, out_off (+ have, s_end)
    volatile float* cold = &s_cold[0][tid];
    volatile int* ci = &s_ci[0][tid];
    volatile double* sum = &s_sum[0][tid];
    auto tp = [&](int k) -> volatile float& { return cold[k * kT]; };
    volatile G& t_ev = reinterpret_cast<volatile G*>(s_tev)[tid];
    volatile float& v_ev = cold[4 * kT];
    auto Lr = [&](int k) -> volatile float& { return cold[(5 + k) * kT]; }; // ratio only
    volatile double& Tr = reinterpret_cast<volatile double*>(s_tr)[RATIO ? tid : 0]; // ratio only
    volatile int &px = ci[0], &py = ci[kT], &s = ci[2 * kT], &bounces = ci[3 * kT], &out_off = ci[4 * kT];
    volatile int& have = ci[(RATIO ? 5 : 0) * kT]; // ratio only
    volatile int& s_end = ci[(CHUNK ? (RATIO ? 6 : 5) : 0) * kT]; // chunked: end of the lane's samples

    Accessor<CODEC> acc(A.g);
    auto ray_load = [&]() {
        Ray r;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            r.o[k] = reinterpret_cast<volatile G*>(s_ray[k])[tid];
            r.d[k] = reinterpret_cast<volatile G*>(s_ray[3 + k])[tid];
        }
        return r;
    };
    auto ray_store = [&](const Ray& r) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            reinterpret_cast<volatile G*>(s_ray[k])[tid] = r.o[k];
            reinterpret_cast<volatile G*>(s_ray[3 + k])[tid] = r.d[k];
        }
    };

    RngF rng{0};
    constexpr bool MIXED = sizeof(G) == 8;
    using I = float;
    const I* inv_tab = A.inv_maj_f;
    G t = G(0), tb = G(0);
    I inv = I(0), inv_ahead = I(0);
    uint32_t samples = 0;
    int state = kNeedPixel;
    bool done = false;
    long long unit = 0;
    int fill = 32;

    auto finish_path = [&](float r0, float r1, float r2) {
        if constexpr (CHUNK) { // the sample's result, summed in order by k_reduce (render.cu)
            float* o = A.sbuf + (size_t(out_off / 3) * size_t(A.spp) + size_t(s)) * 3;
            o[0] = r0;
            o[1] = r1;
            o[2] = r2;
        } else {
            sum[0] += double(r0);
            sum[kT] += double(r1);
            sum[2 * kT] += double(r2);
        }
        s = s + 1;
        state = kNeedPath;
    };
    auto finish_ratio = [&]() { finish_path(Lr(0), Lr(1), Lr(2)); };
    // scattering vertex (render.hpp:173-185)
    auto bounce = [&](G te, float ve) {
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
            Ray ray = ray_load();
            ray.o[0] += ray.d[0] * te;
            ray.o[1] += ray.d[1] * te;
            ray.o[2] += ray.d[2] * te;
            if constexpr (MIXED) { // sample_isotropic (render.hpp:128-134) in FP64: a float
                // direction would move every later point of the path by ~1e-7 of its length
                const double u0 = rng.uniform53(), u1 = rng.uniform53();
                const double z = 1.0 - 2.0 * u0;
                const double r = sqrt(fmax(0.0, 1.0 - z * z));
                double sp, cp;
                sincos(2.0 * 3.14159265358979323846 * u1, &sp, &cp);
                ray.d[0] = G(r * cp);
                ray.d[1] = G(r * sp);
                ray.d[2] = G(z);
            } else {
                const float u0 = rng.uniform(), u1 = rng.uniform();
                const float z = 1.0f - 2.0f * u0;
                const float r = sqrtf(fmaxf(0.0f, 1.0f - z * z));
                float sp, cp;
                sincospif(2.0f * u1, &sp, &cp);
                ray.d[0] = G(r * cp);
                ray.d[1] = G(r * sp);
                ray.d[2] = G(z);
            }
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
            const float tr = float(Tr);
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
    auto flight_over = [&]() { state = kEscape; };
    auto do_start = [&]() {
        if (state == kEscape)
            end_segment();
        if (state == kScatter) {
            bounce(t_ev, v_ev);
            if (state == kNeedSegment)
                goto segment;
        }
        if (state == kNeedPath) {
            if constexpr (CHUNK) {
                if (s == s_end) {
                    state = kNeedPixel;
                    return;
                }
            }
            if (s == A.spp) {
                const double inv_spp = 1.0 / double(A.spp);
                A.out[out_off] = float(sum[0] * inv_spp);
                A.out[out_off + 1] = float(sum[kT] * inv_spp);
                A.out[out_off + 2] = float(sum[2 * kT] * inv_spp);
                state = kNeedPixel;
                return;
            }
            bool from_table = false;
            if constexpr (CHUNK) {
                if (A.camtab) { // FP64 camera ray + post-jitter stream from k_camera_rays (render.cu)
                    const double2* rec = A.camtab + 2 * (size_t(out_off / 3) * size_t(A.spp) + size_t(s));
                    const double2 a = __ldg(rec), b = __ldg(rec + 1);
                    rng.state = uint64_t(__double_as_longlong(b.y));
                    Ray r;
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        r.o[k] = G(A.cam.pos[k]);
                    r.d[0] = G(a.x);
                    r.d[1] = G(a.y);
                    r.d[2] = G(b.x);
                    ray_store(r);
                    from_table = true;
                }
            }
            if (!from_table) {
                {
                    const Rng r0 = Rng::for_pixel_sample(A.seed_mixed, px, py, s);
                    rng.state = r0.state;
                }
                G jx, jy;
                if constexpr (MIXED) {
                    jx = rng.uniform53();
                    jy = rng.uniform53();
                } else {
                    jx = rng.uniform();
                    jy = rng.uniform();
                }
                ray_store(camera_ray_g<G>(A.cam, G(px) + jx, G(py) + jy));
            }
            tp(0) = tp(1) = tp(2) = 1.0f;
            bounces = 0;
            if constexpr (RATIO)
                Lr(0) = Lr(1) = Lr(2) = 0.0f;
            state = kNeedSegment;
        }
    segment:
        if constexpr (RATIO) {
            Tr = 1.0;
            have = 0;
        }
        if (!dda.init(A.cells, hi, ray_load(), cell, icell)) {
            end_segment();
            return;
        }
        tb = dda.cf(6); // the walk position (next_ahead)
        inv_ahead = __ldg(inv_tab + dda.index(A.cells));
        state = kNeedCell;
    };
    // kNeedCell -> next macrocell (empty cells draw nothing); kInCell -> one tentative step
    auto do_advance = [&]() {
        const float lg = __log2f(1.0f - rng.peek()); // step draw, consumed only where it is used
        if (state == kNeedCell) {
            if (inv_ahead < I(0)) { // the walk ended with the previous visit (ratio: Tr > 0 here)
                flight_over();
                return;
            }
            bool over;
            int ahead;
            dda.next_ahead(A.cells, t, tb, over, ahead); // t of an empty cell is never read
            inv = inv_ahead;
            inv_ahead = over ? I(-1) : __ldg(inv_tab + ahead);
            if (!(inv > I(0)))
                return;
        }
        rng.skip();
        t -= G(lg * 0.693147182f) * G(inv);
        state = t >= tb ? kNeedCell : kPoint;
    };
    auto accept = [&](float v) {
        const float st = tf.extinction(v);
        if constexpr (RATIO) {
            const float r = float(st * inv);
            if (!have && rng.uniform() < r) {
                have = 1;
                t_ev = t;
                v_ev = v;
            }
            const double tr = Tr * (1.0 - double(r));
            Tr = tr;
            if (!(tr > 0.0f))
                flight_over();
            else
                state = kInCell;
        } else {
            if (rng.uniform() < float(st * inv)) {
                t_ev = t;
                v_ev = v;
                state = kScatter;
            } else {
                state = kInCell;
            }
        }
    };
    auto do_sample = [&]() {
        acc = Accessor<CODEC>(A.g); // no accessor state between gathers (cold locate = one directory load)
        const Ray r = ray_load();
        ++samples;
        accept(sample_f<CODEC, G>(acc, r.o[0] + r.d[0] * t, r.o[1] + r.d[1] * t, r.o[2] + r.d[2] * t));
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
                long long blk = unit;
                int j = 0;
                if constexpr (CHUNK) { // unit = block * nchunks + chunk (fits 32 bits)
                    blk = (long long)(unsigned(unit) / unsigned(A.nchunks));
                    j = int(unsigned(unit) - unsigned(blk) * unsigned(A.nchunks));
                }
                const long long k = blk >> 3;
                const int w = int(blk & 7);
                const int lx = (w & 1) * 8 + (p & 7), ly = (w >> 1) * 4 + (p >> 3);
                const long long tt = k * A.nranks + A.rank;
                const int qx = int(tt % A.tiles_x) * 16 + lx, qy = int(tt / A.tiles_x) * 16 + ly;
                if (qx < A.cam.w && qy < A.cam.h) {
                    px = qx;
                    py = qy;
                    out_off = int(A.packed ? (k * 256 + ly * 16 + lx) * 3 : ((long long)qy * A.cam.w + qx) * 3);
                    if constexpr (CHUNK) {
                        s = j * A.chunk;
                        s_end = min(A.spp, (j + 1) * A.chunk);
                    } else {
                        s = 0;
                        sum[0] = sum[kT] = sum[2 * kT] = 0.0;
                    }
                    state = kNeedPath;
                }
            }
            fill += min(__popc(need), avail);
            need &= ~__ballot_sync(kFull, ((need >> lane) & 1u) && below < avail); // served lanes
        }
        // ---- run the phase most lanes are waiting in (finished lanes sit in kNeedPixel) ----
        const int nS = __popc(__ballot_sync(kFull, state == kPoint));
        const int nA = __popc(__ballot_sync(kFull, state == kNeedCell || state == kInCell));
        const int nT = __popc(__ballot_sync(kFull, state == kNeedPath || state == kNeedSegment || state == kScatter ||
                                                       state == kEscape));
        if (nS + nA + nT == 0) {
            if (__all_sync(kFull, done))
                break;
            continue;
        }
        if (nS >= nA && nS >= nT) {
            if (state == kPoint)
                do_sample();
        } else if (nA >= nT) {
#pragma unroll 1
            for (int k = 0; k < kAdvIters && (state == kNeedCell || state == kInCell); ++k)
                do_advance();
        } else if (state == kNeedPath || state == kNeedSegment || state == kScatter || state == kEscape) {
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

template <int CODEC, int MODE, typename G>
int launch(const RenderArgs& A, long long n_units, size_t smem, cudaStream_t s)
{
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto kern = A.chunk ? k_trace_f<CODEC, MODE, G, true> : k_trace_f<CODEC, MODE, G, false>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kT, smem);
    const long long blocks = std::min<long long>((long long)std::max(per_sm, 1) * sms, (n_units * 32 + kT - 1) / kT);
    kern<<<unsigned(blocks), kT, smem, s>>>(A, n_units);
    return 0;
}

template <int CODEC, typename G>
int launch_mode(const RenderArgs& A, int mode, long long n_units, size_t smem, cudaStream_t s)
{
    return mode == SVDBGPU_MODE_RATIO ? launch<CODEC, SVDBGPU_MODE_RATIO, G>(A, n_units, smem, s)
                                      : launch<CODEC, SVDBGPU_MODE_PATHTRACE, G>(A, n_units, smem, s);
}

template <typename G>
int launch_codec(const RenderArgs& A, int codec, int mode, long long n_units, size_t smem, cudaStream_t s)
{
    switch (codec) {
    case kCodecF32: return launch_mode<kCodecF32, G>(A, mode, n_units, smem, s);
    case kCodecUnorm8: return launch_mode<kCodecUnorm8, G>(A, mode, n_units, smem, s);
    case kCodecAffine8: return launch_mode<kCodecAffine8, G>(A, mode, n_units, smem, s);
    default: return launch_mode<kCodecAffine4, G>(A, mode, n_units, smem, s);
    }
}

} // namespace

int launch_trace_fast(const RenderArgs& A, int codec, int mode, int precision, long long n_units, size_t smem,
                      cudaStream_t s)
{
    return precision == SVDBGPU_PRECISION_FP32 ? launch_codec<float>(A, codec, mode, n_units, smem, s)
                                               : launch_codec<double>(A, codec, mode, n_units, smem, s);
}

} // namespace svdbgpu
