// render.cu — the reference-exact (FP64) render kernels and the render() entry point.
//
//   k_trace  (pathtrace K4, ratio K6): persistent, path-regenerating tracer. Every lane is a small
//            state machine over its own pixels; each loop iteration runs the phase (start /
//            advance / gather) most lanes of the warp are waiting in. Per-lane state lives in
//            shared memory between phases; 71 registers, 28 warps per SM.
//   k_render (EA K5, ISO, and the per-pixel A/B baseline): one thread per pixel, a CTA per 16x16
//            image tile (the reference's tile, render.hpp:285-313), each warp an 8x4 pixel block.
//   render() sets up majorants, launches one of them (or render_fast.cu's FP32-arithmetic tracer)
//            and reports stats.
// Samples of a pixel run in index order and accumulate in FP64 (render.hpp:297-310) in both
// kernels, so the image is independent of the launch shape and of how tiles are split over GPUs.
//
//   render_field  render.hpp:276-315   -> k_trace / k_render
//   camera_ray    render.hpp:259-269   -> host basis (exact) + camera_ray
//   trace_path    render.hpp:160-187   -> k_trace state machine (Tracer::trace_path in k_render)
//   next_event    render.hpp:137-151   -> SharedDda + do_advance (Tracer::next_event)
//   woodcock_track render.hpp:106-124  -> do_advance + accept (Tracer::woodcock)
//   trace_iso     render.hpp:193-255   -> Tracer::trace_iso
#include "device.cuh"
#include "grid_impl.hpp"
#include "render_args.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>


namespace svdbgpu {

namespace {

// TF entries to shared memory when they fit (kTfSmemMax), else read in place from global memory
__device__ __forceinline__ const float4* stage_tf(const RenderArgs& A, float4* smem)
{
    if (A.tf.n > kTfSmemMax)
        return A.tf_ent;
    for (int i = threadIdx.x; i < A.tf.n; i += blockDim.x)
        smem[i] = A.tf_ent[i];
    __syncthreads();
    return smem;
}

constexpr double kPi = 3.14159265358979323846;

__device__ __forceinline__ double kInf() { return __longlong_as_double(0x7ff0000000000000ll); }

// a / b from y = RN(1 / b): q = RN(a y) corrected once with the exact residual fma(-q, b, a) gives
// RN(a / b) (Markstein's correction; bit-identical to the IEEE division, checked on 5e8 operand pairs
// including worst-case divisor significands, tools/check_div.c). Tiny divisors take the division.
__device__ __forceinline__ double div_by_rcp(double a, double b, double y)
{
    if (!(fabs(b) > 0x1p-900))
        return a / b;
    const double q = a * y;
    return fma(fma(-q, b, a), y, q);
}

template <int CODEC>
struct Tracer {
    const RenderArgs& A;
    const float4* ent; // shared-memory TF entries
    Accessor<CODEC> acc;
    uint32_t samples;

    __device__ __forceinline__ Tracer(const RenderArgs& a, const float4* e) : A(a), ent(e), acc(a.g), samples(0) {}

    __device__ __forceinline__ float sample_at(const Ray& r, double t)
    {
        ++samples;
        return sample_trilinear<CODEC>(acc, r.o[0] + r.d[0] * t, r.o[1] + r.d[1] * t, r.o[2] + r.d[2] * t);
    }

    __device__ __forceinline__ int cell_index(const int c[3]) const
    {
        return c[0] + A.cells[0] * (c[1] + A.cells[1] * c[2]);
    }

    // woodcock_track (render.hpp:106-124)
    __device__ __forceinline__ bool woodcock(double sigma_maj, const Ray& r, double t0, double t1, Rng& rng,
                                             double& t_ev, float& v_ev)
    {
        if (!(sigma_maj > 0.0))
            return false;
        double inv = 1.0 / sigma_maj;
        double t = t0;
        for (;;) {
            t -= step_log(1.0 - rng.uniform()) * inv;
            if (t >= t1)
                return false;
            float v = sample_at(r, t);
            double st = tf_extinction(A.tf, ent, double(v));
            if (rng.uniform() < st * inv) {
                t_ev = t;
                v_ev = v;
                return true;
            }
        }
    }

    // next_event (render.hpp:137-151): DDA over 32^3 macrocells, empty cells draw nothing
    __device__ __forceinline__ bool next_event(const Ray& r, Rng& rng, double& t_ev, float& v_ev)
    {
        Dda d;
        if (!d.init(A.cells, A.hi, r, 0.0, kInf(), A.cell, A.icell))
            return false;
        int c[3];
        double ta, tb;
        while (d.next(A.cells, c, ta, tb)) {
            float m = __ldg(A.maj + cell_index(c));
            if (m == 0.0f)
                continue; // empty (maj == 0); a zero float majorant also draws nothing
            if (woodcock(double(m), r, ta, tb, rng, t_ev, v_ev))
                return true;
        }
        return false;
    }

    __device__ __forceinline__ void isotropic(Rng& rng, double d[3])
    {
        double u0 = 0.0, u1 = 0.0;
#pragma unroll 1
        for (int k = 0; k < 2; ++k) { // two draws, one copy of the generator in the code
            const double u = rng.uniform();
            if (k == 0)
                u0 = u;
            else
                u1 = u;
        }
        double z = 1.0 - 2.0 * u0;
        double phi = 2.0 * kPi * u1;
        double r = sqrt(dmax(0.0, 1.0 - z * z));
        double sp, cp;
        sincos(phi, &sp, &cp); // same values as sin()/cos(), one argument reduction
        d[0] = r * cp;
        d[1] = r * sp;
        d[2] = z;
    }

    __device__ __forceinline__ void scatter_albedo(float v, double tp[3])
    {
        double rgba[4];
        tf_lookup(A.tf, ent, double(v), rgba);
        tp[0] *= double(float(rgba[0])); // tf.rgb() returns Vec3f (transfer.hpp:58-62)
        tp[1] *= double(float(rgba[1]));
        tp[2] *= double(float(rgba[2]));
    }

    // trace_path (render.hpp:160-187)
    __device__ void trace_path(Ray ray, Rng& rng, float out[3])
    {
        double tp[3] = {1.0, 1.0, 1.0};
        int bounces = 0;
        for (;;) {
            double t;
            float v;
            if (!next_event(ray, rng, t, v)) {
                out[0] = float(tp[0] * double(A.ambient[0]));
                out[1] = float(tp[1] * double(A.ambient[1]));
                out[2] = float(tp[2] * double(A.ambient[2]));
                return;
            }
            if (++bounces > A.max_bounces) {
                out[0] = out[1] = out[2] = 0.0f;
                return;
            }
            scatter_albedo(v, tp);
            ray.o[0] = ray.o[0] + ray.d[0] * t;
            ray.o[1] = ray.o[1] + ray.d[1] * t;
            ray.o[2] = ray.o[2] + ray.d[2] * t;
            isotropic(rng, ray.d);
            if (bounces >= A.rr_start) {
                double survive = dclamp(dmax(tp[0], dmax(tp[1], tp[2])), 0.05, 0.95);
                if (rng.uniform() >= survive) {
                    out[0] = out[1] = out[2] = 0.0f;
                    return;
                }
                tp[0] /= survive;
                tp[1] /= survive;
                tp[2] /= survive;
            }
        }
    }

    // Ratio-tracked escape + delta-tracked scattering (oracle/svdb_oracle.c trace_ratio).
    __device__ void trace_ratio(Ray ray, Rng& rng, float out[3])
    {
        double tp[3] = {1.0, 1.0, 1.0};
        double L[3] = {0.0, 0.0, 0.0};
        int bounces = 0;
        for (;;) {
            double Tr = 1.0;
            bool have = false;
            double t_ev = 0.0;
            float v_ev = 0.0f;
            Dda d;
            if (d.init(A.cells, A.hi, ray, 0.0, kInf(), A.cell, A.icell)) {
                int c[3];
                double ta, tb;
                while (Tr > 0.0 && d.next(A.cells, c, ta, tb)) {
                    float m = __ldg(A.maj + cell_index(c));
                    if (m == 0.0f)
                        continue;
                    double inv = 1.0 / double(m);
                    double t = ta;
                    for (;;) {
                        t -= step_log(1.0 - rng.uniform()) * inv;
                        if (t >= tb)
                            break;
                        float v = sample_at(ray, t);
                        double r = tf_extinction(A.tf, ent, double(v)) * inv;
                        if (!have && rng.uniform() < r) {
                            have = true;
                            t_ev = t;
                            v_ev = v;
                        }
                        Tr *= 1.0 - r;
                        if (!(Tr > 0.0))
                            break;
                    }
                }
            }
            L[0] += tp[0] * Tr * double(A.ambient[0]);
            L[1] += tp[1] * Tr * double(A.ambient[1]);
            L[2] += tp[2] * Tr * double(A.ambient[2]);
            if (!have)
                break;
            if (++bounces > A.max_bounces)
                break;
            scatter_albedo(v_ev, tp);
            ray.o[0] = ray.o[0] + ray.d[0] * t_ev;
            ray.o[1] = ray.o[1] + ray.d[1] * t_ev;
            ray.o[2] = ray.o[2] + ray.d[2] * t_ev;
            isotropic(rng, ray.d);
            if (bounces >= A.rr_start) {
                double survive = dclamp(dmax(tp[0], dmax(tp[1], tp[2])), 0.05, 0.95);
                if (rng.uniform() >= survive)
                    break;
                tp[0] /= survive;
                tp[1] /= survive;
                tp[2] /= survive;
            }
        }
        out[0] = float(L[0]);
        out[1] = float(L[1]);
        out[2] = float(L[2]);
    }

    // Emission-absorption march (oracle/svdb_oracle.c trace_ea). Samples falling in an empty
    // macrocell (majorant 0 => alpha 0 on its whole closed box) contribute exactly nothing, so
    // the march jumps over runs of empty cells without changing a single sample position.
    __device__ void trace_ea(const Ray& ray, Rng& rng, float out[3])
    {
        double j = rng.uniform();
        double C[3] = {0.0, 0.0, 0.0}, T = 1.0;
        double t0 = 0.0, t1 = kInf();
        const double dt = A.ea_step;
        if (clip_ray_box(ray, A.hi, t0, t1) && t0 <= t1) {
            for (long long k = 0;; ++k) {
                double t = t0 + (double(k) + j) * dt;
                if (!(t < t1))
                    break;
                double p[3] = {ray.o[0] + ray.d[0] * t, ray.o[1] + ray.d[1] * t, ray.o[2] + ray.d[2] * t};
                int c[3];
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    c[a] = int(dclamp(floor(p[a] * A.icell), 0.0, double(A.cells[a] - 1)));
                if (__ldg(A.maj + cell_index(c)) == 0.0f) {
                    // exact skip: find this empty cell's exit along the ray and resume at the
                    // last sample index before it (the per-sample test handles the rest)
                    double te = t1;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        if (ray.d[a] > 0.0)
                            te = dmin(te, (double(c[a] + 1) * A.cell - ray.o[a]) / ray.d[a]);
                        else if (ray.d[a] < 0.0)
                            te = dmin(te, (double(c[a]) * A.cell - ray.o[a]) / ray.d[a]);
                    }
                    double kk = floor((te - t0) / dt - j) - 1.0;
                    if (kk > double(k))
                        k = (long long)kk;
                    continue;
                }
                ++samples;
                float v = sample_trilinear<CODEC>(acc, p[0], p[1], p[2]);
                double rgba[4];
                tf_lookup(A.tf, ent, double(v), rgba);
                double a = 1.0 - exp(-(A.tf.scale * rgba[3]) * dt);
                C[0] += T * a * rgba[0];
                C[1] += T * a * rgba[1];
                C[2] += T * a * rgba[2];
                T *= 1.0 - a;
                if (T < A.ea_min_t)
                    break;
            }
        }
        out[0] = float(C[0] + T * double(A.background[0]));
        out[1] = float(C[1] + T * double(A.background[1]));
        out[2] = float(C[2] + T * double(A.background[2]));
    }

    // trace_iso_hit + trace_iso (render.hpp:193-255)
    __device__ void trace_iso(const Ray& ray, float out[3])
    {
        const double step = 0.25, iso = A.iso;
        bool hit = false;
        double hit_t = 0.0;
        Dda d;
        if (d.init(A.cells, A.hi, ray, 0.0, kInf(), A.cell, A.icell)) {
            int c[3];
            double ta, tb;
            while (!hit && d.next(A.cells, c, ta, tb)) {
                int ci = cell_index(c);
                if (iso < double(__ldg(A.cmin + ci)) || iso > double(__ldg(A.cmax + ci)))
                    continue;
                double t_prev = ta;
                double f_prev = double(sample_at(ray, t_prev)) - iso;
                if (f_prev == 0.0) {
                    hit = true;
                    hit_t = t_prev;
                    break;
                }
                for (double t = ta + step;; t += step) {
                    t = dmin(t, tb);
                    double f = double(sample_at(ray, t)) - iso;
                    if (f == 0.0 || (f_prev < 0.0) != (f < 0.0)) {
                        double a = t_prev, b = t;
                        for (int i = 0; i < 16; ++i) {
                            double m = 0.5 * (a + b);
                            double fm = double(sample_at(ray, m)) - iso;
                            if (fm == 0.0) {
                                a = b = m;
                                break;
                            }
                            if ((f_prev < 0.0) == (fm < 0.0))
                                a = m;
                            else
                                b = m;
                        }
                        hit = true;
                        hit_t = 0.5 * (a + b);
                        break;
                    }
                    t_prev = t;
                    f_prev = f;
                    if (t >= tb)
                        break;
                }
            }
        }
        if (!hit) {
            out[0] = A.background[0];
            out[1] = A.background[1];
            out[2] = A.background[2];
            return;
        }
        double p[3] = {ray.o[0] + ray.d[0] * hit_t, ray.o[1] + ray.d[1] * hit_t, ray.o[2] + ray.d[2] * hit_t};
        const double h = 0.5;
        samples += 6;
        double gx = double(sample_trilinear<CODEC>(acc, p[0] + h, p[1], p[2]) - sample_trilinear<CODEC>(acc, p[0] - h, p[1], p[2])) / (2.0 * h);
        double gy = double(sample_trilinear<CODEC>(acc, p[0], p[1] + h, p[2]) - sample_trilinear<CODEC>(acc, p[0], p[1] - h, p[2])) / (2.0 * h);
        double gz = double(sample_trilinear<CODEC>(acc, p[0], p[1], p[2] + h) - sample_trilinear<CODEC>(acc, p[0], p[1], p[2] - h)) / (2.0 * h);
        double len = sqrt(gx * gx + gy * gy + gz * gz);
        if (len == 0.0) {
            out[0] = out[1] = out[2] = 0.0f;
            return;
        }
        gx /= len;
        gy /= len;
        gz /= len;
        out[0] = float(fabs(gx));
        out[1] = float(fabs(gy));
        out[2] = float(fabs(gz));
    }
};

// camera_ray (render.hpp:259-269); the basis and tan_half come exact from the host
__device__ __forceinline__ Ray camera_ray(const CamArgs& c, double px, double py)
{
    // rolled loops keep one copy of each FP64 division (same operations as render.hpp:266-268)
    double qx = 0.0, qy = 0.0;
#pragma unroll 1
    for (int k = 0; k < 2; ++k) {
        const double q = 2.0 * (k == 0 ? px : py) / double(k == 0 ? c.w : c.h);
        if (k == 0)
            qx = q;
        else
            qy = q;
    }
    double ndc_x = (qx - 1.0) * c.tan_half * c.aspect;
    double ndc_y = (1.0 - qy) * c.tan_half;
    Ray r;
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.o[a] = c.pos[a];
        d[a] = c.fwd[a] + c.right[a] * ndc_x + c.up[a] * ndc_y;
    }
    double len = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
        const double q = (k == 0 ? d[0] : (k == 1 ? d[1] : d[2])) / len;
        if (k == 0)
            r.d[0] = q;
        else if (k == 1)
            r.d[1] = q;
        else
            r.d[2] = q;
    }
    return r;
}

template <int CODEC, int MODE>
__global__ void __launch_bounds__(256) k_render(const __grid_constant__ RenderArgs A)
{
    extern __shared__ float4 s_tf[];
    const float4* s_ent = stage_tf(A, s_tf);

    const long long k = blockIdx.x; // k-th tile of this rank
    const long long t = k * A.nranks + A.rank;
    const int tx = int(t % A.tiles_x) * 16, ty = int(t / A.tiles_x) * 16;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (w & 1) * 8 + (lane & 7), ly = (w >> 1) * 4 + (lane >> 3);
    const int px = tx + lx, py = ty + ly;
    uint32_t samples = 0;
    if (px < A.cam.w && py < A.cam.h) {
        Tracer<CODEC> tr(A, s_ent);
        double acc[3] = {0.0, 0.0, 0.0};
        for (int s = 0; s < A.spp; ++s) {
            Rng rng = Rng::for_pixel_sample(A.seed_mixed, px, py, s);
            double jx = rng.uniform();
            double jy = rng.uniform();
            Ray ray = camera_ray(A.cam, double(px) + jx, double(py) + jy);
            float c[3];
            if constexpr (MODE == SVDBGPU_MODE_PATHTRACE)
                tr.trace_path(ray, rng, c);
            else if constexpr (MODE == SVDBGPU_MODE_RATIO)
                tr.trace_ratio(ray, rng, c);
            else if constexpr (MODE == SVDBGPU_MODE_EA)
                tr.trace_ea(ray, rng, c);
            else
                tr.trace_iso(ray, c);
            acc[0] += double(c[0]);
            acc[1] += double(c[1]);
            acc[2] += double(c[2]);
        }
        acc[0] /= double(A.spp);
        acc[1] /= double(A.spp);
        acc[2] /= double(A.spp);
        size_t o = A.packed ? (size_t(k) * 256 + size_t(ly) * 16 + size_t(lx)) * 3
                            : (size_t(py) * size_t(A.cam.w) + size_t(px)) * 3;
        A.out[o] = float(acc[0]);
        A.out[o + 1] = float(acc[1]);
        A.out[o + 2] = float(acc[2]);
        samples = tr.samples;
    }
    // per-warp reduction of the sample counter (stats only)
    unsigned long long s64 = samples;
#pragma unroll
    for (int off = 16; off; off >>= 1)
        s64 += __shfl_xor_sync(0xffffffffu, s64, off);
    if (lane == 0 && s64)
        atomicAdd(A.counters, s64);
}

// ---------------------------------------------------------------------------------------------
// k_trace: persistent, path-regenerating delta/ratio tracker (K4 / K6 production kernel).
//
// k_render runs "for each sample: trace the whole path" per lane, so a warp waits for its
// longest path every sample (ncu: 2.2 active lanes per warp). Here every lane is a small state
// machine and one loop iteration = one tentative collision: phase A (divergent but ALU-only)
// advances the lane to its next tentative collision point — starting a new sample or a new
// pixel, re-entering the DDA after a scatter, skipping empty or exhausted cells — and phase B
// (re-converged) does the trilinear gather + accept test. Each lane still owns whole pixels and
// walks their samples in index order with the reference's FP64 arithmetic and draw order, so
// the image is bit-identical to k_render and to the CPU oracles. Pixels are handed out in 8x4
// blocks per warp from a global counter (lanes refill individually, so no lane idles at a pixel
// boundary); the grid is sized to the resident CTA count.
// state >> 2 is the lane's phase group: 0 idle (needs a work item), 1 start, 2 advance, 3 gather
enum : int { kNeedPixel = 0,
             kNeedPath = 4, kNeedSegment = 5, kScatter = 6,
             kEscape = 7, // flight over (left the grid / Tr = 0): result written in the start phase
             kNeedCell = 8, kInCell = 9,
             kNeedRegion = 10, // hierarchical DDA: next 128^3 lower-node region
             kPoint = 12,
             kNeedLog = 13 }; // tentative step whose cell-exit decision needs the exact FP64 log   // flight over (left the grid / Tr = 0): result written in the start phase

// The macrocell DDA of device.cuh (dda.hpp:52-109), same arithmetic, with its 23 words of
// per-lane state in shared memory (SoA, conflict-free) instead of registers: it is touched once
// per cell visit, and the registers it frees buy resident warps for latency hiding.
template <int T>
struct SharedDda {
    volatile int* si;    // [7][T]: c0..2, step0..2, done
    volatile double* sd; // [8][T]: t_next0..2, t_delta0..2, t_cur, t1
    int tid;
    __device__ __forceinline__ volatile int& ci(int k) { return si[k * T + tid]; }
    __device__ __forceinline__ volatile double& cd(int k) { return sd[k * T + tid]; }
    __device__ __forceinline__ int cx() { return ci(0); }
    __device__ __forceinline__ int cy() { return ci(1); }
    __device__ __forceinline__ int cz() { return ci(2); }
    __device__ __forceinline__ bool done() { return ci(6) != 0; }
    __device__ __forceinline__ int stepv(int axis) { return ci(3 + axis); }
    __device__ __forceinline__ void set_done() { ci(6) = 1; }
    __device__ __forceinline__ int index(const int cells[3])
    {
        SVDB_ASSERT(unsigned(ci(0)) < unsigned(cells[0]) && unsigned(ci(1)) < unsigned(cells[1]) &&
                    unsigned(ci(2)) < unsigned(cells[2]));
        return ci(0) + cells[0] * (ci(1) + cells[1] * ci(2));
    }

    // clip_ray_box + dda_traverse setup (dda.hpp:25-86), the operations and their order per axis
    // exactly the reference's. The axes are unrolled so their independent FP64 chains (reciprocal,
    // slab products, the t_next divisions) interleave (measured +3.8% C3 over a rolled loop).
    __device__ __forceinline__ bool init(const int cells[3], const double hi[3], const Ray& r, double t0, double t1,
                                         double cell, double icell, int force_axis = -1, int force_cell = 0,
                                         const int* clo = nullptr, const int* chi = nullptr)
    {
        double inv[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double o = r.o[a], d = r.d[a], h = hi[a];
            inv[a] = 0.0;
            if (d == 0.0) {
                if (o < 0.0 || o > h)
                    return false;
                continue;
            }
            inv[a] = 1.0 / d;
            double ta = (0.0 - o) * inv[a], tb = (h - o) * inv[a];
            if (ta > tb) {
                const double tt = ta;
                ta = tb;
                tb = tt;
            }
            t0 = dmax(t0, ta);
            t1 = dmin(t1, tb);
            if (t0 > t1)
                return false;
        }
        if (!(t0 <= t1))
            return false;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double o = r.o[a], d = r.d[a];
            const double e = o + d * t0;
            // force_axis: the hierarchical DDA's region entry face fixes the start cell on that axis
            const int c = a == force_axis ? force_cell
                                          : int(dclamp(floor(e * icell), clo ? double(clo[a]) : 0.0,
                                                       chi ? double(chi[a]) : double(cells[a] - 1)));
            int step = 0;
            double tn = __longlong_as_double(0x7ff0000000000000ll), td = tn;
            if (d != 0.0) {
                step = d > 0.0 ? 1 : -1;
                // (c' cell - o) / d from the slab reciprocal RN(1/d) with one exact correction
                // (div_by_rcp: the IEEE quotient, one reciprocal per axis instead of two divisions)
                tn = (double(d > 0.0 ? c + 1 : c) * cell - o) / d;
                // cell is a power of two, so +-cell * RN(1/d) == RN(+-cell / d) exactly (dda.hpp:80, 84)
                td = (d > 0.0 ? cell : -cell) * inv[a];
            }
            ci(a) = c;
            ci(3 + a) = step;
            cd(a) = tn;
            cd(3 + a) = td;
        }
        cd(6) = t0;
        cd(7) = t1;
        ci(6) = 0;
        return true;
    }

    __device__ __forceinline__ bool next(const int cells[3], int cell[3], double& ta, double& tb)
    {
        if (done())
            return false;
        const double n0 = cd(0), n1 = cd(1), n2 = cd(2), t_cur = cd(6), t1 = cd(7);
        const bool ax1 = n1 < n0;
        const double tm = ax1 ? n1 : n0;
        const bool ax2 = n2 < tm;
        const int axis = ax2 ? 2 : (ax1 ? 1 : 0);
        const double tn = ax2 ? n2 : tm;
        double t_exit = dmin(tn, t1);
        t_exit = dmax(t_exit, t_cur);
        cell[0] = ci(0);
        cell[1] = ci(1);
        cell[2] = ci(2);
        ta = t_cur;
        tb = t_exit;
        if (t_exit >= t1) {
            set_done();
            return true;
        }
        cd(6) = t_exit;
        const int c = (axis == 0 ? cell[0] : (axis == 1 ? cell[1] : cell[2])) + stepv(axis);
        ci(axis) = c;
        if (c < 0 || c >= cells[axis])
            set_done();
        else
            cd(axis) = (axis == 0 ? n0 : (axis == 1 ? n1 : n2)) + cd(3 + axis);
        return true;
    }

    // next() that also reports the axis the traversal steps across after this visit (-1: it ended)
    __device__ __forceinline__ bool next_axis(const int cells[3], int cell[3], double& ta, double& tb, int& stepped)
    {
        stepped = -1;
        if (done())
            return false;
        const double n0 = cd(0), n1 = cd(1), n2 = cd(2), t_cur = cd(6), t1 = cd(7);
        const bool ax1 = n1 < n0;
        const double tm = ax1 ? n1 : n0;
        const bool ax2 = n2 < tm;
        const int axis = ax2 ? 2 : (ax1 ? 1 : 0);
        const double tn = ax2 ? n2 : tm;
        double t_exit = dmin(tn, t1);
        t_exit = dmax(t_exit, t_cur);
        cell[0] = ci(0);
        cell[1] = ci(1);
        cell[2] = ci(2);
        ta = t_cur;
        tb = t_exit;
        if (t_exit >= t1) {
            set_done();
            return true;
        }
        cd(6) = t_exit;
        const int c = (axis == 0 ? cell[0] : (axis == 1 ? cell[1] : cell[2])) + stepv(axis);
        ci(axis) = c;
        if (c < 0 || c >= cells[axis]) {
            set_done();
            return true;
        }
        cd(axis) = (axis == 0 ? n0 : (axis == 1 ? n1 : n2)) + cd(3 + axis);
        stepped = axis;
        return true;
    }

    // next() for a walk that is known not to be over (the caller keeps that in a register: the
    // traversal has a visit left unless the previous call reported `over`), reporting whether the
    // traversal is over after this visit and else the linear index of the following cell (for the
    // majorant load one visit ahead); no done flag in shared memory. The walk position t_cur is the
    // caller's register tb (the previous visit's exit, or the entry after init), not the t_cur row.
    // RANGED: the walk is confined to the cell range [lo, hi] (an HDDA region), else to the grid
    template <bool RANGED>
    __device__ __forceinline__ void next_ahead(const int cells[3], const int lo[3], const int hi[3], double& ta,
                                               double& tb, bool& over, int& ahead)
    {
        const double n0 = cd(0), n1 = cd(1), n2 = cd(2), t_cur = tb, t1 = cd(7);
        const bool ax1 = n1 < n0;
        const double tm = ax1 ? n1 : n0;
        const bool ax2 = n2 < tm;
        const int axis = ax2 ? 2 : (ax1 ? 1 : 0);
        const double tn = ax2 ? n2 : tm;
        double t_exit = dmin(tn, t1);
        t_exit = dmax(t_exit, t_cur);
        int c0 = ci(0), c1 = ci(1), c2 = ci(2);
        ta = t_cur;
        tb = t_exit;
        over = true;
        ahead = 0;
        if (t_exit >= t1)
            return;
        // the stepped axis' values by selects on the two comparisons (tn is already t_next[axis])
        const int c = (ax2 ? c2 : (ax1 ? c1 : c0)) + stepv(axis);
        ci(axis) = c;
        if constexpr (RANGED) {
            const int lo_a = ax2 ? lo[2] : (ax1 ? lo[1] : lo[0]), hi_a = ax2 ? hi[2] : (ax1 ? hi[1] : hi[0]);
            if (c < lo_a || c > hi_a)
                return;
        } else if (unsigned(c) >= unsigned(ax2 ? cells[2] : (ax1 ? cells[1] : cells[0]))) { // selects, not an indexed constant load
            return;
        }
        cd(axis) = tn + cd(3 + axis);
        c0 = axis == 0 ? c : c0;
        c1 = axis == 1 ? c : c1;
        c2 = axis == 2 ? c : c2;
        over = false;
        ahead = c0 + cells[0] * (c1 + cells[1] * c2);
    }
};

constexpr int kTraceThreads = 64;   // 2 warps per CTA
constexpr int kTraceMinBlocks = 14; // <= 72 registers, <= 15 KB shared: 28 resident warps per SM (16 measured slower)
constexpr int kAdvIters = 3;        // advance steps per advance-phase invocation
constexpr int kChunkMinSpp = 16;    // one GPU: whole-pixel work items below this many samples per pixel
constexpr int kSplitChunk = 4;      // max samples per work item when the frame is split over ranks
constexpr int kSampleChunk = 16;    // max samples per work item on one GPU (8 / 32 measured -1%)

template <int CODEC, int MODE, bool CHUNK, bool HDDA>
__global__ void __launch_bounds__(kTraceThreads, kTraceMinBlocks) k_trace(const __grid_constant__ RenderArgs A, long long n_units)
{
    extern __shared__ float4 s_tf[];
    const float4* s_ent = stage_tf(A, s_tf);
    constexpr unsigned FULL = 0xffffffffu;
    constexpr bool RATIO = MODE == SVDBGPU_MODE_RATIO;
    constexpr int T = kTraceThreads;
    const int lane = threadIdx.x & 31;
    const int tid = threadIdx.x;
    unsigned long long* work = A.counters + 1;

    Tracer<CODEC> tr(A, s_ent);
    Rng rng{0};
    // The flight's ray is read only by the gather and written only at path start / scatter: kept
    // in shared memory (SoA) so the advance loop does not hold its 12 registers.
    __shared__ double s_ray[6][T];
    auto ray_load = [&]() {
        Ray r;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            r.o[k] = reinterpret_cast<volatile double*>(s_ray[k])[tid];
            r.d[k] = reinterpret_cast<volatile double*>(s_ray[3 + k])[tid];
        }
        return r;
    };
    auto ray_store = [&](const Ray& r) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            reinterpret_cast<volatile double*>(s_ray[k])[tid] = r.o[k];
            reinterpret_cast<volatile double*>(s_ray[3 + k])[tid] = r.d[k];
        }
    };
    // macrocell DDA state (23 words per lane) in shared memory, touched once per cell visit
    __shared__ int s_dda_i[7][T];
    __shared__ double s_dda_d[8][T];
    SharedDda<T> dda{&s_dda_i[0][0], &s_dda_d[0][0], tid};
    // hierarchical DDA: the lower-node-region DDA of the flight (oracle flight_init / flight_next)
    __shared__ int s_rdda_i[HDDA ? 7 : 1][T];
    __shared__ double s_rdda_d[HDDA ? 8 : 1][T];
    SharedDda<T> rdda{&s_rdda_i[0][0], &s_rdda_d[0][0], tid};
    __shared__ int s_rentry[T]; // HDDA: face through which the next region is entered (-1: first region)
    volatile int& r_entry = s_rentry[tid];
    __shared__ int s_rrange[HDDA ? 6 : 1][T]; // HDDA: majorant-cell range of the current region
    // The step loop's live values stay in registers: t, the cell's far end tb, 1/majorant of this
    // cell and of the next one (loaded one visit ahead), the RNG state.
    double t = 0.0, tb = 0.0, inv = 0.0, inv_ahead = 0.0;
#ifdef SVDB_PHASE_STATS
    unsigned st_empty = 0, st_full = 0;
#endif
    // Per-lane state touched only at sample start/end, scatter and pixel output lives in shared
    // memory (SoA, conflict-free). rows: acc0..2 (whole-pixel items only; chunked items write each
    // sample to sbuf), tp0..2, t_ev; ratio tracking adds L0..2, Tr. Names without a row of their own
    // alias the t_ev row and are written only by the initialisation below, before t_ev.
    constexpr int kA = CHUNK ? 0 : 3;
    __shared__ double s_cold_d[kA + 4 + (RATIO ? 4 : 0)][T];
    __shared__ int s_cold_i[6 + (RATIO ? 1 : 0) + (CHUNK ? 1 : 0)][T];
    constexpr int kAcc = CHUNK ? kA + 3 : 0;
    volatile double &acc0 = s_cold_d[kAcc][tid], &acc1 = s_cold_d[kAcc + (CHUNK ? 0 : 1)][tid],
                    &acc2 = s_cold_d[kAcc + (CHUNK ? 0 : 2)][tid];
    volatile double &tp0 = s_cold_d[kA][tid], &tp1 = s_cold_d[kA + 1][tid], &tp2 = s_cold_d[kA + 2][tid];
    volatile double& t_ev = s_cold_d[kA + 3][tid];
    constexpr int kR0 = RATIO ? kA + 4 : kA + 3, kR = RATIO ? 1 : 0;
    volatile double &L0 = s_cold_d[kR0][tid], &L1 = s_cold_d[kR0 + kR][tid], &L2 = s_cold_d[kR0 + 2 * kR][tid];
    volatile double& Tr = s_cold_d[kR0 + 3 * kR][tid];
    volatile int& have_d = s_cold_i[RATIO ? 6 : 0][tid];              // ratio: event pending (0/1)
    volatile int& s_end = s_cold_i[CHUNK ? (RATIO ? 7 : 6) : 0][tid]; // chunked: end of the lane's samples
    volatile int &px = s_cold_i[0][tid], &py = s_cold_i[1][tid], &s = s_cold_i[2][tid];
    volatile int &bounces = s_cold_i[3][tid], &out_off = s_cold_i[4][tid]; // see the work hand-out
    volatile float& v_ev = reinterpret_cast<volatile float&>(s_cold_i[5][tid]);
    struct HaveRef {
        volatile int& d;
        __device__ operator bool() const { return d != 0; }
        __device__ HaveRef& operator=(bool b) { d = b ? 1 : 0; return *this; }
    } have{have_d};
    acc0 = acc1 = acc2 = 0.0;
    tp0 = tp1 = tp2 = 1.0;
    L0 = L1 = L2 = 0.0;
    Tr = 1.0;
    t_ev = 0.0;
    have = false;
    px = py = s = bounces = out_off = 0;
    if constexpr (CHUNK)
        s_end = 0;
    v_ev = 0.0f;
    int state = kNeedPixel;
    bool done = false;
    long long unit = 0;
    int fill = 32;

    // path finished with float result r (render.hpp:306: accum += Vec3d(c))
    auto finish_path = [&](float r0, float r1, float r2) {
        if constexpr (CHUNK) { // the sample's result, summed in order by k_reduce
            SVDB_ASSERT(out_off / A.spp < A.npix && s < A.spp);
            float* o = A.sbuf + (size_t(out_off) + size_t(s)) * 3; // out_off = pixel * spp (chunked)
            o[0] = r0;
            o[1] = r1;
            o[2] = r2;
        } else {
            acc0 += double(r0);
            acc1 += double(r1);
            acc2 += double(r2);
        }
        ++s;
        state = kNeedPath;
    };
    // scattering vertex (render.hpp:173-185); returns 0 when the path continues (state
    // kNeedSegment), else how it ended: 2 absorbed (max bounces / Russian roulette), ratio 3
    auto bounce = [&](double te, float ve) -> int {
        if (++bounces > A.max_bounces)
            return RATIO ? 3 : 2;
        double tpv[3] = {tp0, tp1, tp2};
        tr.scatter_albedo(ve, tpv);
        tp0 = tpv[0];
        tp1 = tpv[1];
        tp2 = tpv[2];
        {
            Ray ray = ray_load();
            ray.o[0] = ray.o[0] + ray.d[0] * te;
            ray.o[1] = ray.o[1] + ray.d[1] * te;
            ray.o[2] = ray.o[2] + ray.d[2] * te;
            tr.isotropic(rng, ray.d);
            ray_store(ray);
        }
        if (bounces >= A.rr_start) {
            double survive = dclamp(dmax(tp0, dmax(tp1, tp2)), 0.05, 0.95);
            if (rng.uniform() >= survive)
                return RATIO ? 3 : 2;
            const double ys = 1.0 / survive; // render.hpp:184, tp /= survive per channel, exactly
#pragma unroll
            for (int k = 0; k < 3; ++k)
                s_cold_d[kA + k][tid] = div_by_rcp(s_cold_d[kA + k][tid], survive, ys);
        }
        state = kNeedSegment;
        return 0;
    };
    // a flight that ran out of cells (or of transmittance) ends in the start phase, batched with
    // the other lanes writing results and starting paths, instead of inside the advance / gather
    // iteration where it ran with a lane or two
    auto flight_over = [&]() { state = kEscape; };
    // kEscape / kScatter / kNeedPath / kNeedSegment: finish a flight, scatter, write a finished pixel,
    // start the next sample (render.hpp:298-302), or enter the macrocell DDA with a new flight
    // (render.hpp:142)
    auto do_start = [&]() {
        // how the flight / path ended: 1 escaped (result tp * ambient), 2 absorbed (0), 3 ratio (L)
        int fin = 0;
        if (state == kEscape) { // the flight left the grid (or Tr hit 0): escape / ratio segment end
            if constexpr (RATIO) {
                L0 += tp0 * Tr * double(A.ambient[0]);
                L1 += tp1 * Tr * double(A.ambient[1]);
                L2 += tp2 * Tr * double(A.ambient[2]);
                if (have)
                    state = kScatter;
                else
                    fin = 3;
            } else {
                fin = 1;
            }
        }
        if (state == kScatter) // the only copy of the scattering code in the loop
            fin = bounce(t_ev, v_ev);
        if (fin) { // the one result write (render.hpp:306)
            float r0 = 0.0f, r1 = 0.0f, r2 = 0.0f;
            if constexpr (RATIO) {
                r0 = float(L0);
                r1 = float(L1);
                r2 = float(L2);
            } else if (fin == 1) {
                r0 = float(tp0 * double(A.ambient[0]));
                r1 = float(tp1 * double(A.ambient[1]));
                r2 = float(tp2 * double(A.ambient[2]));
            }
            finish_path(r0, r1, r2);
        }
        if (state == kNeedSegment)
            goto segment;
        if (state == kNeedPath) {
            if constexpr (CHUNK) {
                if (s == s_end) { // sample range done; k_reduce writes the pixel
                    state = kNeedPixel;
                    return;
                }
            }
            if (s == A.spp) {
#pragma unroll 1
                for (int k = 0; k < 3; ++k) // render.hpp:308-310, one division site
                    A.out[out_off + k] = float(s_cold_d[CHUNK ? kAcc : k][tid] / double(A.spp));
                state = kNeedPixel;
                return;
            }
            bool from_table = false;
            if constexpr (CHUNK) {
                if (A.camtab) { // ray and post-jitter stream from k_camera_rays (same arithmetic)
                    SVDB_ASSERT(out_off / A.spp < A.npix && s < A.spp);
                    const double2* rec = A.camtab + 2 * (size_t(out_off) + size_t(s));
                    const double2 a = __ldg(rec), b = __ldg(rec + 1);
                    rng.state = uint64_t(__double_as_longlong(b.y));
                    Ray r;
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        r.o[k] = A.cam.pos[k];
                    r.d[0] = a.x;
                    r.d[1] = a.y;
                    r.d[2] = b.x;
                    ray_store(r);
                    from_table = true;
                }
            }
            if (!from_table) {
                rng = Rng::for_pixel_sample(A.seed_mixed, px, py, s);
                double jx = 0.0, jy = 0.0;
#pragma unroll 1
                for (int k = 0; k < 2; ++k) { // jitter draws (render.hpp:300-301), one generator copy
                    const double u = rng.uniform();
                    if (k == 0)
                        jx = u;
                    else
                        jy = u;
                }
                ray_store(camera_ray(A.cam, double(px) + jx, double(py) + jy));
            }
            tp0 = tp1 = tp2 = 1.0;
            bounces = 0;
            if constexpr (RATIO)
                L0 = L1 = L2 = 0.0;
            state = kNeedSegment;
        }
    segment:
        if constexpr (RATIO) {
            Tr = 1.0;
            have = false;
        }
#ifdef SVDB_TRACE_PIXEL
        if (px == SVDB_TRACE_X && py == SVDB_TRACE_Y && s == SVDB_TRACE_S) {
            const Ray rr = ray_load();
            printf("[gpu] ray %a %a %a %a %a %a\n", rr.o[0], rr.o[1], rr.o[2], rr.d[0], rr.d[1], rr.d[2]);
        }
#endif
        if constexpr (HDDA) {
            if (!rdda.init(A.ccells, A.hi, ray_load(), 0.0, kInf(), 128.0, 1.0 / 128.0)) {
                flight_over(); // missed the grid: the segment ends (next start phase)
                return;
            }
            r_entry = -1;
            state = kNeedRegion;
            return;
        }
        if (!dda.init(A.cells, A.hi, ray_load(), 0.0, kInf(), A.cell, A.icell)) {
            flight_over(); // missed the grid: the segment ends (next start phase)
            return;
        }
        tb = dda.cd(6); // the walk position (next_ahead)
        inv_ahead = __ldg(A.inv_maj + dda.index(A.cells));
        state = kNeedCell;
    };
    // kNeedCell -> next macrocell (empty cells draw nothing, render.hpp:145-146);
    // kInCell -> one tentative step t -= ln(1-u)/sigma_maj (render.hpp:116-118)
    auto do_advance = [&]() {
        // the step draw does not depend on the DDA: its bound is computed from the next uniform
        // before the cell lookup (independent chains interleave); the draw is consumed only if the
        // cell has draws, so the stream is unchanged
        // a float lower bound of the step length -ln(1 - u) from the next uniform (MUFU lg2:
        // |error| <= 4e-7 (1 + y); bound taken 10x wider), computed before the cell lookup
        // float(1 - u) from the integer draw: 1 - u = (2^53 - bits) * 2^-53 exactly, and rounding
        // the integer to float then scaling by a power of two is the same RN(1 - u) (no FP64 ops)
        float one_minus_u = __ull2float_rn((1ull << 53) - rng.peek_bits()) * 0x1p-53f, lg;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(one_minus_u)); // normal argument (>= 2^-53)
        // lower bound of y = -ln(1 - u), margins 4e-6 absolute and 4e-6 relative, pre-scaled by
        // 0.999998 (the decision's 1e-6 relative margins on each side) so the test below is one
        // product: y_lb = lg * (-ln 2 (1 - 4e-6) 0.999998, rounded towards 0) - 4e-6, in one FMA
        const float y_lb = __fmaf_rn(lg, -0x1.62e3a4p-1f, -4e-6f);
        if constexpr (HDDA) {
            if (state == kNeedRegion) { // next lower-node region; one without draws is skipped whole
                int rc[3];
                double ra, rb;
                int stepped;
                if (!rdda.next_axis(A.ccells, rc, ra, rb, stepped)) {
#ifdef SVDB_TRACE_PIXEL
                    if (px == SVDB_TRACE_X && py == SVDB_TRACE_Y && s == SVDB_TRACE_S)
                        printf("[gpu] flight end\n");
#endif
                    flight_over();
                    return;
                }
#ifdef SVDB_TRACE_PIXEL
                if (px == SVDB_TRACE_X && py == SVDB_TRACE_Y && s == SVDB_TRACE_S)
                    printf("[gpu] region %d %d %d %a %a\n", rc[0], rc[1], rc[2], ra, rb);
#endif
                const int entry = r_entry;
                r_entry = stepped;
                if (!__ldg(A.cdraw + (rc[0] + A.ccells[0] * (rc[1] + A.ccells[1] * rc[2]))))
                    return;
                // the region's cells bound the majorant-grid walk, and its entry face fixes the first
                // cell on that axis (oracle flight_next)
                const int R = 128 / int(A.cell);
                int rlo[3], rhi[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    rlo[k] = rc[k] * R;
                    rhi[k] = min(rlo[k] + R, A.cells[k]) - 1;
                    s_rrange[k][tid] = rlo[k];
                    s_rrange[3 + k][tid] = rhi[k];
                }
                int fc = 0;
                if (entry >= 0)
                    fc = rdda.stepv(entry) > 0 ? (entry == 0 ? rlo[0] : (entry == 1 ? rlo[1] : rlo[2]))
                                               : (entry == 0 ? rhi[0] : (entry == 1 ? rhi[1] : rhi[2]));
                if (!dda.init(A.cells, A.hi, ray_load(), ra, rb, A.cell, A.icell, entry, fc, rlo, rhi))
                    return;
                tb = dda.cd(6);
                inv_ahead = __ldg(A.inv_maj + dda.index(A.cells));
                state = kNeedCell;
                return;
            }
        }
        if (state == kNeedCell) {
            // (ratio: Tr > 0 here — accept() ends the flight as soon as it reaches 0)
            bool over;
            int ahead;
            int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
            if constexpr (HDDA) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    lo[k] = s_rrange[k][tid];
                    hi[k] = s_rrange[3 + k][tid];
                }
            }
            if (inv_ahead < 0.0) { // the walk ended with the previous visit
                if constexpr (HDDA)
                    state = kNeedRegion; // the region's majorant cells are done
                else
                    flight_over();
                return;
            }
            // the visit's range goes straight into the step registers: t of an empty cell is never
            // read (the next non-empty visit overwrites it), tb carries the walk position
            dda.template next_ahead<HDDA>(A.cells, lo, hi, t, tb, over, ahead);
#ifdef SVDB_TRACE_PIXEL
            if (px == SVDB_TRACE_X && py == SVDB_TRACE_Y && s == SVDB_TRACE_S)
                printf("[gpu] visit %a %a\n", t, tb);
#endif
            // 1.0 / double(majorant) precomputed per cell with the same IEEE division
            // (render.hpp:113), 0 marks an empty cell. This cell's was loaded one visit ahead;
            // issue the next cell's now so the load overlaps a whole iteration.
            inv = inv_ahead;
            inv_ahead = over ? -1.0 : __ldg(A.inv_maj + ahead); // -1: no cell after this one
#ifdef SVDB_PHASE_STATS
            ++(inv > 0.0 ? st_full : st_empty);
#endif
            if (!(inv > 0.0))
                return;
        }
        rng.skip();
        // The step leaves the cell when t - ln(1-u) * inv >= tb, and then only that decision is
        // used, never the new t (the next non-empty cell restarts at its entry, render.hpp:113-118).
        // When the float bound already clears the gap with margin (>= 1e-6 relative, far above every
        // rounding error) the decision is certain: no FP64 log. Otherwise the exact step is taken in
        // the gather phase (kNeedLog), batched with the collisions it mostly leads to.
        if (y_lb * float(inv) > float(tb - t)) {
            state = kNeedCell;
            return;
        }
        state = kNeedLog;
    };
    // kNeedLog: the exact step with the reference's FP64 log of the draw just consumed (render.hpp:116)
    auto do_exact_step = [&]() {
        t -= step_log(1.0 - rng.last()) * inv;
        state = t >= tb ? kNeedCell : kPoint;
    };
    // accept test on the gathered value (render.hpp:119-122) / ratio update
    auto accept = [&](float v) {
        double st = tf_extinction(A.tf, tr.ent, double(v));
        if constexpr (RATIO) {
            double r = st * inv;
            if (!have && rng.uniform() < r) {
                have = true;
                t_ev = t;
                v_ev = v;
            }
            Tr *= 1.0 - r;
            if (!(Tr > 0.0))
                flight_over();
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
    // kPoint: trilinear gather at the tentative collision + accept test (render.hpp:119-122). No
    // accessor state is kept between gathers: with the leaf directory a cold locate is one load.
    auto do_sample = [&]() {
        tr.acc = Accessor<CODEC>(A.g);
        accept(tr.sample_at(ray_load(), t));
    };

    for (;;) {
        // ---- hand out work items (warp-uniform point) ----
        unsigned need = __ballot_sync(FULL, state == kNeedPixel && !done);
        while (need) {
            if (fill >= 32) {
                unsigned long long u = 0;
                if (lane == 0)
                    u = atomicAdd(work, 1ull);
                unit = (long long)__shfl_sync(FULL, u, 0);
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
                px = int(tt % A.tiles_x) * 16 + lx;
                py = int(tt / A.tiles_x) * 16 + ly;
                if (px < A.cam.w && py < A.cam.h) {
                    const long long pix = A.packed ? k * 256 + ly * 16 + lx : (long long)py * A.cam.w + px;
                    // whole-pixel items: the pixel's first float in the image; chunked items: the
                    // pixel's first per-sample slot (pixel * spp < 2^31: the per-sample buffer is capped)
                    out_off = int(CHUNK ? pix * A.spp : pix * 3);
                    if constexpr (CHUNK) {
                        s = j * A.chunk;
                        s_end = min(A.spp, (j + 1) * A.chunk);
                    } else {
                        s = 0;
                    }
                    if constexpr (!CHUNK)
                        acc0 = acc1 = acc2 = 0.0;
                    state = kNeedPath;
                }
            }
            fill += min(__popc(need), avail);
            need &= ~__ballot_sync(FULL, ((need >> lane) & 1u) && below < avail); // served lanes
        }
        // ---- phase selection: run the one phase most lanes are waiting in; ties go to the
        // gather so its memory latency is paid by as many lanes as possible at once. Finished
        // lanes stay in kNeedPixel, which is in no phase ----
        const int group = state >> 2;
        const int nS = __popc(__ballot_sync(FULL, group == 3));
        const int nA = __popc(__ballot_sync(FULL, group == 2));
        const int nT = __popc(__ballot_sync(FULL, group == 1));
        if (nS + nA + nT == 0) { // every lane waits for a work item (none left: the warp is done)
            if (__all_sync(FULL, done))
                break;
            continue;
        }
        // argmax with ties to the gather, then the advance (same choice as "gather if it has the most
        // lanes, else advance unless the start phase has more")
        int phase = 2, best = nS;
        if (nA > best) {
            phase = 1;
            best = nA;
        }
        if (nT > best)
            phase = 0;
#ifdef SVDB_PHASE_STATS
        if (lane == 0) { // per phase: invocations and participating lanes
            const int n = phase == 0 ? nT : (phase == 1 ? nA : nS);
            atomicAdd(A.counters + 2 + 2 * phase, 1ull);
            atomicAdd(A.counters + 3 + 2 * phase, (unsigned long long)n);
        }
#endif
        if (phase == 0) {
            if (group == 1)
                do_start();
        } else if (phase == 1) {
#pragma unroll 1
            for (int k = 0; k < kAdvIters && (state >> 2) == 2; ++k)
                do_advance();
        } else {
            if (state == kNeedLog)
                do_exact_step();
            if (state == kPoint)
                do_sample();
        }
    }
    unsigned long long s64 = tr.samples;
#pragma unroll
    for (int off = 16; off; off >>= 1)
        s64 += __shfl_xor_sync(FULL, s64, off);
    if (lane == 0 && s64)
        atomicAdd(A.counters, s64);
#ifdef SVDB_PHASE_STATS
    atomicAdd(A.counters + 12, (unsigned long long)st_empty); // macrocell visits: empty / non-empty
    atomicAdd(A.counters + 13, (unsigned long long)st_full);
#endif
}

// Camera rays of a sample-chunked render, precomputed at full SIMD width (in k_trace a new path's
// camera ray ran with ~3 of 32 lanes active): per (pixel, sample) of this rank's tiles, the
// reference's per-sample prologue (render.hpp:298-302: Rng::for_pixel_sample, jitter jx, jy,
// camera_ray) with the same arithmetic as k_trace's in-kernel path. Record = ray direction and the
// RNG state after the two jitter draws; the origin is the camera position.
__global__ void k_camera_rays(const __grid_constant__ RenderArgs A, long long ntiles, double2* __restrict__ tab)
{
    const long long n = ntiles * 256 * A.spp;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long slot = i / A.spp;
        const int s = int(i - slot * A.spp);
        const long long k = slot >> 8;
        const int lx = int(slot & 15), ly = int((slot >> 4) & 15);
        const long long t = k * A.nranks + A.rank;
        const int px = int(t % A.tiles_x) * 16 + lx, py = int(t / A.tiles_x) * 16 + ly;
        if (px >= A.cam.w || py >= A.cam.h)
            continue;
        const size_t pix = A.packed ? size_t(slot) : size_t(py) * size_t(A.cam.w) + size_t(px);
        Rng rng = Rng::for_pixel_sample(A.seed_mixed, px, py, s);
        const double jx = rng.uniform();
        const double jy = rng.uniform();
        const Ray r = camera_ray(A.cam, double(px) + jx, double(py) + jy);
        double2* o = tab + 2 * (pix * size_t(A.spp) + size_t(s));
        o[0] = make_double2(r.d[0], r.d[1]);
        o[1] = make_double2(r.d[2], __longlong_as_double((long long)rng.state));
    }
}

__global__ void k_unpack(const float* __restrict__ packed, int nranks, long long max_tiles, int w, int h, int tiles_x,
                         float* __restrict__ rgb)
{
    long long n = (long long)w * h;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int x = int(i % w), y = int(i / w);
        long long t = (long long)(y >> 4) * tiles_x + (x >> 4);
        long long r = t % nranks, k = t / nranks;
        const float* src = packed + ((r * max_tiles + k) * 256 + (y & 15) * 16 + (x & 15)) * 3;
        rgb[i * 3] = src[0];
        rgb[i * 3 + 1] = src[1];
        rgb[i * 3 + 2] = src[2];
    }
}

// Sample-chunked renders: each pixel's per-sample results summed in sample order in FP64 and
// divided by spp, exactly render_field's accumulation (render.hpp:297-310). One thread per pixel
// slot of this rank's tiles; slots outside the image are skipped.
__global__ void k_reduce(const float* __restrict__ sbuf, float* __restrict__ out, long long ntiles, int nranks,
                         int rank, int tiles_x, int w, int h, int spp, int packed)
{
    const long long n = ntiles * 256;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long k = i >> 8;
        const int lx = int(i & 15), ly = int((i >> 4) & 15);
        const long long t = k * nranks + rank;
        const int px = int(t % tiles_x) * 16 + lx, py = int(t / tiles_x) * 16 + ly;
        if (px >= w || py >= h)
            continue;
        const size_t pix = packed ? size_t(k * 256 + ly * 16 + lx) : size_t(py) * size_t(w) + size_t(px);
        const float* src = sbuf + pix * size_t(spp) * 3;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if ((spp & 3) == 0) { // 16-B aligned rows: 4 samples (12 floats) per 3 vector loads
            const float4* v = reinterpret_cast<const float4*>(src);
            for (int q = 0; q < spp / 4; ++q) {
                const float4 x = __ldg(v + 3 * q), y = __ldg(v + 3 * q + 1), z = __ldg(v + 3 * q + 2);
                a0 += double(x.x); a1 += double(x.y); a2 += double(x.z);
                a0 += double(x.w); a1 += double(y.x); a2 += double(y.y);
                a0 += double(y.z); a1 += double(y.w); a2 += double(z.x);
                a0 += double(z.y); a1 += double(z.z); a2 += double(z.w);
            }
        } else {
            for (int s = 0; s < spp; ++s) {
                a0 += double(src[3 * s]);
                a1 += double(src[3 * s + 1]);
                a2 += double(src[3 * s + 2]);
            }
        }
        out[pix * 3] = float(a0 / double(spp));
        out[pix * 3 + 1] = float(a1 / double(spp));
        out[pix * 3 + 2] = float(a2 / double(spp));
    }
}

// Host camera basis with the reference's exact expression order (render.hpp:259-265, vec.hpp).
void host_camera(const svdbgpu_camera* c, CamArgs* o)
{
    auto normalize = [](double v[3]) {
        double len = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        v[0] /= len;
        v[1] /= len;
        v[2] /= len;
    };
    auto cross = [](const double a[3], const double b[3], double r[3]) {
        r[0] = a[1] * b[2] - a[2] * b[1];
        r[1] = a[2] * b[0] - a[0] * b[2];
        r[2] = a[0] * b[1] - a[1] * b[0];
    };
    double f[3] = {c->look_at[0] - c->position[0], c->look_at[1] - c->position[1], c->look_at[2] - c->position[2]};
    normalize(f);
    double r[3], u[3];
    cross(f, c->up, r);
    normalize(r);
    cross(r, f, u);
    for (int a = 0; a < 3; ++a) {
        o->pos[a] = c->position[a];
        o->fwd[a] = f[a];
        o->right[a] = r[a];
        o->up[a] = u[a];
    }
    volatile double fov = c->fov_y_deg; // keep (fov * pi) / 360 as two roundings
    o->tan_half = std::tan(fov * 3.14159265358979323846 / 360.0);
    o->aspect = double(c->width) / double(c->height);
    o->w = c->width;
    o->h = c->height;
}

uint64_t host_mix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

} // namespace

int64_t tiles_for_rank(int w, int h, int rank, int nranks)
{
    if (w < 1 || h < 1 || nranks < 1 || rank < 0 || rank >= nranks)
        return 0;
    int64_t total = int64_t((w + 15) / 16) * ((h + 15) / 16);
    return total > rank ? (total - rank + nranks - 1) / nranks : 0;
}

int render(GridImpl* g, const svdbgpu_tf* tf, const svdbgpu_camera* cam, const svdbgpu_settings* st, float* d_out,
           int packed, cudaStream_t s, svdbgpu_stats* stats)
{
    if (!cam || !st || !d_out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null camera/settings/output");
    if (cam->width < 1 || cam->height < 1)
        return fail(Errc::size_mismatch, "image size must be positive");
    if (st->spp < 1)
        return fail_code(SVDBGPU_E_INVALID_ARG, "spp must be >= 1");
    if (st->mode < 0 || st->mode > SVDBGPU_MODE_RATIO)
        return fail_code(SVDBGPU_E_INVALID_ARG, "unknown render mode");
    int nranks = st->tile_nranks > 0 ? st->tile_nranks : 1;
    int rank = st->tile_nranks > 0 ? st->tile_rank : 0;
    if (rank < 0 || rank >= nranks)
        return fail_code(SVDBGPU_E_INVALID_ARG, "tile_rank out of range");
    if (st->mode == SVDBGPU_MODE_EA && !(st->ea_step > 0.0))
        return fail_code(SVDBGPU_E_INVALID_ARG, "ea_step must be positive");
    if (st->precision < SVDBGPU_PRECISION_FP64 || st->precision > SVDBGPU_PRECISION_MIXED)
        return fail_code(SVDBGPU_E_INVALID_ARG, "unknown precision");
    const bool hdda = st->hdda != 0;
    if (hdda && (st->precision != SVDBGPU_PRECISION_FP64 || st->kernel == SVDBGPU_KERNEL_PER_PIXEL ||
                 (st->mode != SVDBGPU_MODE_PATHTRACE && st->mode != SVDBGPU_MODE_RATIO)))
        return fail_code(SVDBGPU_E_UNSUPPORTED, "the hierarchical DDA is implemented for FP64 pathtrace / ratio "
                                                "tracking in the path-regenerating kernel");
    if (hdda && st->majorant_cell >= 128)
        return fail_code(SVDBGPU_E_INVALID_ARG, "hierarchical DDA: the majorant grid must be finer than the "
                                                "128^3 lower-node regions (majorant_cell 8 or 32)");
    const bool fp32 = st->precision != SVDBGPU_PRECISION_FP64;
    if (fp32 && (st->kernel == SVDBGPU_KERNEL_PER_PIXEL ||
                 (st->mode != SVDBGPU_MODE_PATHTRACE && st->mode != SVDBGPU_MODE_RATIO)))
        return fail_code(SVDBGPU_E_UNSUPPORTED, "FP32 tracking is implemented for the pathtrace and ratio "
                                                "integrators of the path-regenerating kernel");
    SVDB_CUDA(cudaSetDevice(g->device));
    NvtxRange nvtx("svdbgpu render");
    RenderArgs A{};
    if (int rc = g->upload_tf(tf, s, &A.tf))
        return rc;
    float range_ms = 0.0f;
    if (int rc = g->ensure_ranges(s, &range_ms, st->majorant_cell > 0 ? st->majorant_cell : 32))
        return rc;
    SVDB_CUDA(cudaEventRecord(g->ev0, s));
    if (int rc = majorants(g, A.tf, s))
        return rc;
    A.cdraw = nullptr;
    if (hdda) {
        for (int a = 0; a < 3; ++a)
            A.ccells[a] = std::max(1, (g->dg.dims[a] - 1 + 127) / 128); // cell_counts_for at 128
        if (int rc = coarse_flags(g, A.ccells, s))
            return rc;
        A.cdraw = g->d_cdraw;
    }
    SVDB_CUDA(cudaEventRecord(g->ev1, s));
    SVDB_CUDA(cudaMemsetAsync(g->d_counters, 0, 128, s));

    A.g = g->dg;
    A.tf_ent = g->d_tf;
    A.maj = g->d_maj;
    A.inv_maj = g->d_inv_maj;
    A.inv_maj_f = g->d_inv_maj_f;
    A.cmin = g->d_cmin;
    A.cmax = g->d_cmax;
    for (int a = 0; a < 3; ++a) {
        A.cells[a] = g->cells[a];
        A.cell = double(g->cell_dim);
        A.icell = 1.0 / A.cell;
        A.hi[a] = double(g->dg.dims[a] - 1); // world box [0, dims-1] (macrocell.hpp:50-54)
    }
    host_camera(cam, &A.cam);
    A.spp = st->spp;
    A.max_bounces = st->max_bounces;
    A.rr_start = st->rr_start_bounce;
    A.seed_mixed = host_mix64(st->seed);
    A.iso = st->iso_value;
    for (int c = 0; c < 3; ++c) {
        A.ambient[c] = st->ambient[c];
        A.background[c] = st->background[c];
    }
    A.ea_step = st->ea_step;
    A.ea_min_t = st->ea_min_transmittance;
    A.rank = rank;
    A.nranks = nranks;
    A.tiles_x = (cam->width + 15) / 16;
    A.out = d_out;
    A.packed = packed;
    A.counters = g->d_counters;
    const int64_t ntiles = tiles_for_rank(cam->width, cam->height, rank, nranks);
    A.npix = packed ? ntiles * 256 : int64_t(cam->width) * cam->height;
    const size_t smem = tf_smem_bytes(tf->n_entries);
    cudaEvent_t e2 = nullptr, e3 = nullptr;
    SVDB_CUDA(cudaEventCreate(&e2));
    SVDB_CUDA(cudaEventCreate(&e3));
    SVDB_CUDA(cudaEventRecord(e2, s));
    const bool wave = st->kernel != SVDBGPU_KERNEL_PER_PIXEL &&
                      (st->mode == SVDBGPU_MODE_PATHTRACE || st->mode == SVDBGPU_MODE_RATIO);
    // sample-chunked work items for the path-regenerating tracers: a lane renders `chunk` samples
    // of a pixel, not all spp, so the last items of a frame are short (the frame's tail shrinks
    // from ~spp to ~chunk path lengths); per-sample results go through sbuf to k_reduce
    A.sbuf = nullptr;
    A.camtab = nullptr;
    A.chunk = 0;
    A.nchunks = 1;
    if (wave && ntiles > 0) {
        // one GPU: items of up to 16 samples, at least 2 per pixel, from 16 spp up (C3: 4 per pixel,
        // C2 / C4: 2); fewer spp keep whole pixels, whose tail is already short. Split frames
        // (N ranks, 1/N of the work each) use 4 so the tail stays small against the shorter frame
        const int chunk = nranks > 1 ? std::min(kSplitChunk, std::max(1, st->spp / 2))
                                     : (st->spp >= kChunkMinSpp ? std::min(kSampleChunk, st->spp / 2) : 0);
        const size_t npix = packed ? size_t(ntiles) * 256 : size_t(cam->width) * size_t(cam->height);
        const size_t bytes = npix * size_t(st->spp) * 3 * sizeof(float);
        if (chunk > 0 && chunk < st->spp && bytes <= (size_t(8) << 30)) {
            if (bytes > g->sbuf_cap) {
                cudaFree(g->d_sbuf);
                g->d_sbuf = nullptr;
                g->sbuf_cap = 0;
                SVDB_CUDA(cudaMalloc(&g->d_sbuf, bytes));
                g->sbuf_cap = bytes;
            }
            A.sbuf = g->d_sbuf;
            A.chunk = chunk;
            A.nchunks = (st->spp + chunk - 1) / chunk;
            const size_t tab = npix * size_t(st->spp) * 32;
            if (tab <= (size_t(16) << 30)) {
                if (tab > g->camtab_cap || !g->d_camtab) {
                    cudaFree(g->d_camtab);
                    g->d_camtab = nullptr;
                    g->camtab_cap = 0;
                    SVDB_CUDA(cudaMalloc(&g->d_camtab, tab));
                    g->camtab_cap = tab;
                }
                A.camtab = g->d_camtab;
            }
        }
    }
    if (ntiles > 0) {
        int sms = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const long long n_units = ntiles * 8 * A.nchunks;
#define LAUNCH_T(C, M)                                                                         \
    {                                                                                          \
        int per_sm = 1;                                                                        \
        auto kern = hdda ? (A.chunk ? k_trace<C, M, true, true> : k_trace<C, M, false, true>)    \
                         : (A.chunk ? k_trace<C, M, true, false> : k_trace<C, M, false, false>); \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTraceThreads, smem);       \
        long long blocks = std::min<long long>((long long)std::max(per_sm, 1) * sms, (n_units * 32 + kTraceThreads - 1) / kTraceThreads); \
        kern<<<unsigned(blocks), kTraceThreads, smem, s>>>(A, n_units);                          \
    }
#define LAUNCH_R(C, M) k_render<C, M><<<unsigned(ntiles), 256, smem, s>>>(A)
#define BY_MODE(C)                                                                             \
    switch (st->mode) {                                                                        \
    case SVDBGPU_MODE_PATHTRACE:                                                               \
        if (wave) LAUNCH_T(C, SVDBGPU_MODE_PATHTRACE) else LAUNCH_R(C, SVDBGPU_MODE_PATHTRACE); \
        break;                                                                                 \
    case SVDBGPU_MODE_ISO: LAUNCH_R(C, SVDBGPU_MODE_ISO); break;                                \
    case SVDBGPU_MODE_EA: LAUNCH_R(C, SVDBGPU_MODE_EA); break;                                  \
    default:                                                                                   \
        if (wave) LAUNCH_T(C, SVDBGPU_MODE_RATIO) else LAUNCH_R(C, SVDBGPU_MODE_RATIO);         \
        break;                                                                                 \
    }
        if (A.camtab) {
            const long long n = ntiles * 256 * st->spp;
            k_camera_rays<<<unsigned(std::min<long long>((n + 255) / 256, 148LL * 32)), 256, 0, s>>>(
                A, ntiles, g->d_camtab);
        }
        if (fp32)
            launch_trace_fast(A, g->codec, st->mode, st->precision, n_units, smem, s);
        else switch (g->codec) {
        case kCodecF32: BY_MODE(kCodecF32) break;
        case kCodecUnorm8: BY_MODE(kCodecUnorm8) break;
        case kCodecAffine8: BY_MODE(kCodecAffine8) break;
        default: BY_MODE(kCodecAffine4) break;
        }
#undef BY_MODE
#undef LAUNCH_R
        if (A.chunk) {
            const long long nslots = ntiles * 256;
            k_reduce<<<unsigned(std::min<long long>((nslots + 255) / 256, 148LL * 64)), 256, 0, s>>>(
                A.sbuf, d_out, ntiles, nranks, rank, A.tiles_x, cam->width, cam->height, st->spp, packed);
        }
        cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) {
            cudaEventDestroy(e2);
            cudaEventDestroy(e3);
            return cuda_fail(le, "k_render launch");
        }
    }
    SVDB_CUDA(cudaEventRecord(e3, s));
    unsigned long long samples = 0;
    SVDB_CUDA(cudaMemcpyAsync(&samples, g->d_counters, 8, cudaMemcpyDeviceToHost, s));
    SVDB_CUDA(cudaStreamSynchronize(s));
#ifdef SVDB_PHASE_STATS
    {
        unsigned long long c[16];
        cudaMemcpy(c, g->d_counters, 128, cudaMemcpyDeviceToHost);
        const char* names[3] = {"start", "advance", "gather"};
        fprintf(stderr, "[phase-stats] macrocell visits: empty %llu non-empty %llu\n", c[12], c[13]);
        fprintf(stderr, "[phase-stats] gathers %llu\n", samples);
        for (int p = 0; p < 3; ++p)
            fprintf(stderr, "[phase-stats] %-8s invocations %llu lanes/invocation %.2f\n", names[p], c[2 + 2 * p],
                    c[2 + 2 * p] ? double(c[3 + 2 * p]) / double(c[2 + 2 * p]) : 0.0);
    }
#endif
    float rms = 0.0f, mms = 0.0f;
    cudaEventElapsedTime(&rms, e2, e3);
    cudaEventElapsedTime(&mms, g->ev0, g->ev1);
    cudaEventDestroy(e2);
    cudaEventDestroy(e3);
    if (stats) {
        int64_t w = cam->width, h = cam->height;
        int tiles_x = (cam->width + 15) / 16;
        uint64_t pix = 0;
        for (int64_t kk = 0; kk < ntiles; ++kk) {
            int64_t t = kk * nranks + rank;
            int64_t x0 = (t % tiles_x) * 16, y0 = (t / tiles_x) * 16;
            pix += uint64_t(std::min<int64_t>(16, w - x0)) * uint64_t(std::min<int64_t>(16, h - y0));
        }
        stats->paths = pix * uint64_t(st->spp);
        stats->samples = samples;
        stats->lookups = samples * 8;
        stats->render_ms = rms;
        stats->macrocell_ms = double(range_ms) + double(mms);
        stats->launches = (range_ms > 0.0f ? 1u : 0u) + 1u + (hdda ? 1u : 0u) + (ntiles > 0 ? 1u : 0u) + (A.chunk ? 1u : 0u) +
                          (A.camtab ? 1u : 0u);
    }
    return 0;
}

int unpack_tiles(const float* d_packed, int nranks, int64_t max_tiles, int w, int h, float* d_rgb, cudaStream_t s)
{
    if (nranks < 1 || w < 1 || h < 1)
        return fail_code(SVDBGPU_E_INVALID_ARG, "bad unpack geometry");
    long long n = (long long)w * h;
    int blocks = int(std::min<long long>((n + 255) / 256, 148 * 32));
    k_unpack<<<blocks, 256, 0, s>>>(d_packed, nranks, max_tiles, w, h, (w + 15) / 16, d_rgb);
    SVDB_CUDA(cudaGetLastError());
    return 0;
}

} // namespace svdbgpu
