// K1 -- range-image conversion: IMU/pose transform + spherical binning with the
// reference's nearest-point collision rule, then the payload-ready validity
// bitmap.
//
// Replaces RigidTransform.apply (/root/reference/pkg/src/stpc/motion.py:70-72)
// fused with project_kernel (/root/reference/pkg/src/stpc/_kernels.py:311-355)
// and the valid-mask/packbits steps of project() / serialize()
// (/root/reference/pkg/src/stpc/range_image.py:198-200;
//  /root/reference/pkg/src/stpc/bitstream.py:219-220).
//
// Collision rule: the reference keeps `r < best[f]` scanning points in input
// order, i.e. the minimum range, ties going to the lowest index.  Positive f64
// values order like their u64 bit patterns, so a 64-bit atomicMin on the bits
// computes the same minimum independent of thread order; the optional second
// pass resolves the winning index with an atomicMin over indices whose range
// equals the minimum (identical to "first index wins").
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"
#include "dd.cuh"

namespace stpc {

static constexpr unsigned long long INF_BITS = 0x7ff0000000000000ull;

static bool getenv_flag(const char* name)
{
    const char* v = std::getenv(name);
    return v && *v && *v != '0';
}

__global__ void fill_u64_kernel(unsigned long long* p, unsigned long long v, long long n)
{
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (; i < n; i += stride) p[i] = v;
}

// Zeroing by kernel rather than cudaMemsetAsync: memsets may be executed by a
// copy engine and would queue behind a large concurrent H2D (the pipelined
// host encode overlaps exactly such copies with compute).
__global__ void zero_bytes_kernel(uint8_t* p, long long n)
{
    long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 16;
    const long long stride = (long long)gridDim.x * blockDim.x * 16;
    for (; i < n; i += stride) {
        if (i + 16 <= n && (((uintptr_t)(p + i)) & 15) == 0) {
            *reinterpret_cast<uint4*>(p + i) = make_uint4(0, 0, 0, 0);
        } else {
            for (long long j = i; j < min(i + 16, n); ++j) p[j] = 0;
        }
    }
}

void launch_zero(void* p, long long bytes, cudaStream_t s)
{
    if (bytes <= 0) return;
    int blocks = (int)std::min<long long>((bytes / 16 + 255) / 256 + 1, 148 * 16);
    STPC_LAUNCH();
    zero_bytes_kernel<<<blocks, 256, 0, s>>>((uint8_t*)p, bytes);
}

void launch_fill_u64(unsigned long long* p, unsigned long long v, long long n, cudaStream_t s)
{
    if (n <= 0) return;
    int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
    STPC_LAUNCH();
    fill_u64_kernel<<<blocks, 256, 0, s>>>(p, v, n);
}

// Within 1e-9 (relative) of an integer: the epsilon band of SURVEY.md A.6,
// orders of magnitude wider than the 2-ulp trig discrepancy it guards.
__device__ __forceinline__ bool near_edge(double q)
{
    return fabs(q - rint(q)) <= 1e-9 * fmax(1.0, fabs(q));
}

struct Binned {
    int status;  // 0 rejected, 1 dropped, 2 kept
    long long pix;
    double r;
    bool eps;
};

// One point: f32 -> f64 transform, then project_kernel's per-point body.
__device__ __forceinline__ Binned bin_point(double px, double py, double pz, const double* R,
                                            const double* T, const Geometry& g)
{
    Binned o{0, 0, 0.0, false};
    // ((x*r0 + y*r1) + z*r2) + t, no contraction (-fmad=false)
    double x = xform_coord(px, py, pz, R[0], R[1], R[2], T[0]);
    double y = xform_coord(px, py, pz, R[3], R[4], R[5], T[1]);
    double z = xform_coord(px, py, pz, R[6], R[7], R[8], T[2]);
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) return o;
    double r = sqrt((x * x + y * y) + z * z);
    if (r <= 0.0) return o;
    // Bin decisions: CUDA trig first; within 1e-9 of a bin edge the angle is
    // recomputed correctly rounded (dd.cuh) so the bin matches glibc's.
    double theta = atan2(x, y);
    double th_w = theta < 0.0 ? theta + 2.0 * 3.141592653589793 : theta;
    double qu = th_w / g.theta_r;
    bool eps = near_edge(qu);
    if (eps) {
        theta = dd::atan2_cr(x, y);
        th_w = theta < 0.0 ? theta + 2.0 * 3.141592653589793 : theta;
        qu = th_w / g.theta_r;
    }
    long long u = (long long)floor(qu) % (long long)g.w;
    if (u < 0) u += g.w;
    double cz = z / r;
    if (cz > 1.0) cz = 1.0;
    else if (cz < -1.0) cz = -1.0;
    double qv = (acos(cz) - g.phi_offset) / g.phi_r;
    if (near_edge(qv)) {
        eps = true;
        qv = (dd::acos_cr(cz) - g.phi_offset) / g.phi_r;
    }
    long long v = (long long)floor(qv);
    o.eps = eps;
    if (v < 0 || v >= g.h) { o.status = 1; return o; }
    o.status = 2;
    o.pix = v * (long long)g.w + u;
    o.r = r;
    return o;
}

__device__ __forceinline__ void warp_add_stats(long long* fs, int rej, int drop, int kept, int eps)
{
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        rej += __shfl_xor_sync(STPC_FULL, rej, off);
        drop += __shfl_xor_sync(STPC_FULL, drop, off);
        kept += __shfl_xor_sync(STPC_FULL, kept, off);
        eps += __shfl_xor_sync(STPC_FULL, eps, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (rej) atomicAdd((unsigned long long*)&fs[FS_REJECTED], (unsigned long long)rej);
        if (drop) atomicAdd((unsigned long long*)&fs[FS_DROPPED], (unsigned long long)drop);
        if (kept) atomicAdd((unsigned long long*)&fs[FS_KEPT], (unsigned long long)kept);
        if (eps) atomicAdd((unsigned long long*)&fs[FS_EPS_BAND], (unsigned long long)eps);
    }
}

// Fast bin decision in fp32 (SURVEY.md §7 "K1 convert").  The fp32 angles are
// within 2.6e-6 rad of the true ones (the budget below); whenever both angles
// lie more than FAST_MARGIN = 5e-6 rad from a bin edge the floor is therefore
// the same as the reference's fp64 (glibc) floor and the point is binned
// here.  The ~0.5% of points inside the margin (and any point with coordinates outside
// [1e-15, 1e15]) go to the exact fp64 path.
constexpr double FAST_MARGIN = 5e-6;

// 1/x and sqrt(x) on the MUFU with no IEEE fix-up sequence: both are within
// 2 ulp (2^-22 relative) of the rounded result for the normal, finite
// arguments the fast path feeds them (max >= 1e-15, x^2 + y^2 in [1e-30, 2e30]).
__device__ __forceinline__ float rcp_approx(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_approx(float x)
{
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// atan2 for the fast path, entirely in fp32: odd minimax-style polynomial of
// degree 13 in t = min/max (max error 3.2e-7 rad in float32 FMA evaluation,
// measured on 2M points; t carries <= 2^-21 relative error from the approximate
// reciprocal and product, i.e. <= 4.8e-7 rad) and float reflections (pi/2, pi
// rounded to float: <= 9e-8 rad each, plus half-ulp roundings <= 1.2e-7 rad per
// step).  The denominator is >= 1e-15 (normal); a subnormal numerator flushes
// to t = 0, an angle error below 1e-23 rad.
__device__ __forceinline__ float fast_atan2f(float y, float x)
{
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float t = mn * rcp_approx(mx);
    const float s2 = t * t;
    float p = 0.006811790633946657f;
    p = __fmaf_rn(p, s2, -0.0336042121052742f);
    p = __fmaf_rn(p, s2, 0.07962366193532944f);
    p = __fmaf_rn(p, s2, -0.1323334127664566f);
    p = __fmaf_rn(p, s2, 0.19807815551757812f);
    p = __fmaf_rn(p, s2, -0.3331736922264099f);
    p = __fmaf_rn(p, s2, 0.9999961256980896f);
    float r = p * t;
    r = ay > ax ? 1.57079637f - r : r;
    r = x < 0.0f ? 3.14159274f - r : r;
    return y < 0.0f ? -r : r;
}

// floor(q) for |q| < 2^22 on the FMA pipe: the round-down sum with 1.5 * 2^23
// holds floor(q) in its low mantissa bits (no FRND / F2I on the XU).
__device__ __forceinline__ float floor_bias(float q) { return __fadd_rd(q, 12582912.0f); }
__device__ __forceinline__ int bias_int(float biased) { return __float_as_int(biased) - 0x4B400000; }

// Error budget of the fp32 decision, in radians (a bin is theta_r or phi_r;
// fractions of a bin scale by 1/theta_r, 1/phi_r):
//   input rounding of x, y, z to float (|d atan2| <= relative perturbation)   0.6e-7
//   t = min/max by rcp.approx + product (<= 2^-22 + 2^-24 relative)            3.0e-7
//   polynomial + FFMA2 evaluation, every float t in [0, 1]
//     (tools/fast_atan_bound.py: 3.2e-7, + 0.6e-7 for its fp64 emulation)     3.8e-7
//   reflections: pi/2 and pi constants and roundings, the + 2 pi wrap          7.3e-7
//   q = angle * (1/bin): float 1/bin and the product, |angle| <= 2 pi          7.5e-7
// azimuth total 2.2e-6; the elevation replaces the wrap with
//   sqrt.approx of the fma'd x^2 + y^2 (<= 2^-22 + 2^-23 relative)            3.6e-7
//   phi_offset rounded to float and the subtraction, |phi_offset| <= 3.2       4.3e-7
// elevation total 2.6e-6 rad, against a margin of FAST_MARGIN = 5e-6 rad on
// both sides of every bin edge: 1.9x headroom at any resolution (the launch
// takes the exact path for every point when the margin exceeds half a bin or
// |phi_offset| > 3.2).  The margin test |frac - 1/2| < 1/2 - mu rounds frac -
// 1/2 by at most 3e-8 bins (exact for frac >= 1/4).
__device__ __forceinline__ bool fast_bin(float xf, float yf, float zf, bool guard, const ConvertArgs& a, int& u,
                                         int& v)
{
    // azimuth atan2(x, y) and elevation atan2(sqrt(x^2 + y^2), z) side by side
    // in packed fp32 (FFMA2 / FMUL2 / FADD2: the same IEEE roundings as
    // fast_atan2f, two lanes per instruction)
    const float rxy = sqrt_approx(__fmaf_rn(xf, xf, yf * yf));
    const float ax = fabsf(yf), ay = fabsf(xf), bx = fabsf(zf);
    const float2 mx = make_float2(fmaxf(ax, ay), fmaxf(bx, rxy));
    const float2 mn = make_float2(fminf(ax, ay), fminf(bx, rxy));
    const float2 t = __fmul2_rn(mn, make_float2(rcp_approx(mx.x), rcp_approx(mx.y)));
    const float2 s2 = __fmul2_rn(t, t);
    float2 p = make_float2(0.006811790633946657f, 0.006811790633946657f);
    p = __ffma2_rn(p, s2, make_float2(-0.0336042121052742f, -0.0336042121052742f));
    p = __ffma2_rn(p, s2, make_float2(0.07962366193532944f, 0.07962366193532944f));
    p = __ffma2_rn(p, s2, make_float2(-0.1323334127664566f, -0.1323334127664566f));
    p = __ffma2_rn(p, s2, make_float2(0.19807815551757812f, 0.19807815551757812f));
    p = __ffma2_rn(p, s2, make_float2(-0.3331736922264099f, -0.3331736922264099f));
    p = __ffma2_rn(p, s2, make_float2(0.9999961256980896f, 0.9999961256980896f));
    float2 r = __fmul2_rn(p, t);
    r.x = ay > ax ? 1.57079637f - r.x : r.x;
    r.x = yf < 0.0f ? 3.14159274f - r.x : r.x;
    r.x = xf < 0.0f ? -r.x : r.x;
    r.x = r.x < 0.0f ? r.x + 6.28318548f : r.x;
    r.y = rxy > bx ? 1.57079637f - r.y : r.y;
    r.y = zf < 0.0f ? 3.14159274f - r.y : r.y;
    // (qu, qv) = (theta / theta_r, (phi - phi_offset) / phi_r)
    const float2 q = __fmul2_rn(__fadd2_rn(r, make_float2(0.0f, -a.phi_off)), make_float2(a.inv_tr, a.inv_pr));
    const float bu = floor_bias(q.x), bv = floor_bias(q.y);
    const float2 fl = __fadd2_rn(make_float2(bu, bv), make_float2(-12582912.0f, -12582912.0f));  // exact
    const float2 d = __fadd2_rn(__fadd2_rn(q, make_float2(-fl.x, -fl.y)), make_float2(-0.5f, -0.5f));
    if (!(guard && fabsf(d.x) < a.hu && fabsf(d.y) < a.hv)) return false;
    // 0 <= qu <= 2 pi / theta_r, which CodecConfig does not tie to w: the
    // reference's floor(theta / theta_r) % w needs a true modulo whenever the
    // sensor's w bins cover less than the full circle.  (A point is only
    // accepted with mu < 0.5, i.e. 1/theta_r < 5e4, so |qu|, |qv| < 1e6 fit
    // the biased floor; see launch_convert.)
    const int uq = bias_int(bu);
    u = uq >= a.g.w ? uq % a.g.w : uq;
    v = bias_int(bv);
    return true;
}

// The classification every convert pass agrees on (the main kernels, the
// queue's overflow re-pass): PT_DROP / PT_KEEP (pix, r) decided here,
// PT_QUEUE for the exact fp64 path (bin_point), which also rejects the
// non-finite and zero-range points.  The fast decision needs 1e-15 <
// max(|x|, |y|), max |coord| < 1e15 and s < 1e30 (false for NaN and
// infinities), so coordinates are finite and r = sqrt(s) finite and
// positive wherever it is taken.
enum { PT_DROP = 1, PT_KEEP = 2, PT_QUEUE = 3 };
__device__ __forceinline__ int fast_point(double x, double y, double z, const ConvertArgs& a, int& pix, double& r)
{
    const double s = (x * x + y * y) + z * z;
    const float xf = (float)x, yf = (float)y, zf = (float)z;
    const float mxy = fmaxf(fabsf(xf), fabsf(yf));
    const float mall = fmaxf(mxy, fabsf(zf));
    const bool guard = s < 1e30 && mxy > 1e-15f && mall < 1e15f;
    int u, v;
    if (!fast_bin(xf, yf, zf, guard, a, u, v)) return PT_QUEUE;
    if (v < 0 || v >= a.g.h) return PT_DROP;
    r = sqrt(s);
    pix = v * a.g.w + u;
    return PT_KEEP;
}

// Points per thread: loads for all of them are issued before any binning.
template <class T> struct PPT { static constexpr int value = 8; };
template <> struct PPT<double> { static constexpr int value = 4; };

// Register-staged variant for inputs that are not 16-byte aligned (the TMA
// path below needs 16-byte source addresses).
// grid: (x = chunks of 256*PPT points of a frame, y = frame)
template <class T>
#ifndef STPC_CONVERT_MINB
#define STPC_CONVERT_MINB 4
#endif
__global__ void __launch_bounds__(256, STPC_CONVERT_MINB) convert_kernel(ConvertArgs a, const T* pts)
{
    constexpr int K = PPT<T>::value;
    constexpr int CH = 256 * K;
    __shared__ double xf[12];
    __shared__ int q_local[CH];
    __shared__ int q_n;
    __shared__ unsigned long long q_base;
    __shared__ int stat[4];
    const int f = blockIdx.y;
    const long long b = a.pt_off[f], e = a.pt_off[f + 1];
    const long long cb = b + (long long)blockIdx.x * CH;
    if (cb >= e) return;
    if (threadIdx.x < 12) xf[threadIdx.x] = a.xf[12 * f + threadIdx.x];
    if (threadIdx.x < 4) stat[threadIdx.x] = 0;
    if (threadIdx.x == 0) q_n = 0;
    // issue every load of this thread's points first
    T px[K], py[K], pz[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        long long i = cb + k * 256 + threadIdx.x;
        if (i < e) {
            const T* p = pts + 3 * i;
            px[k] = __ldg(p);
            py[k] = __ldg(p + 1);
            pz[k] = __ldg(p + 2);
        }
    }
    __syncthreads();
    unsigned long long* best = a.best + (long long)f * a.g.P;
    int rej = 0, drop = 0, kept = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        long long i = cb + k * 256 + threadIdx.x;
        if (i >= e) continue;
        double qx = (double)px[k], qy = (double)py[k], qz = (double)pz[k];
        double x = xform_coord(qx, qy, qz, xf[0], xf[1], xf[2], xf[9]);
        double y = xform_coord(qx, qy, qz, xf[3], xf[4], xf[5], xf[10]);
        double z = xform_coord(qx, qy, qz, xf[6], xf[7], xf[8], xf[11]);
        int pix;
        double r;
        const int st = fast_point(x, y, z, a, pix, r);
        if (st == PT_KEEP) {
            kept += 1;
            atomicMin(best + pix, (unsigned long long)__double_as_longlong(r));
        } else if (st == PT_QUEUE) {  // undecided: block-local queue
            int slot = atomicAdd(&q_n, 1);
            q_local[slot] = (int)(i - cb);
        } else {
            drop += 1;
        }
    }
    // block-level stats and one global reservation for the queued points
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        rej += __shfl_xor_sync(STPC_FULL, rej, o);
        drop += __shfl_xor_sync(STPC_FULL, drop, o);
        kept += __shfl_xor_sync(STPC_FULL, kept, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (rej) atomicAdd(&stat[0], rej);
        if (drop) atomicAdd(&stat[1], drop);
        if (kept) atomicAdd(&stat[2], kept);
    }
    __syncthreads();
    const int nq = q_n;
    if (threadIdx.x == 0) {
        long long* fs = a.fstats + (long long)f * FS_COUNT;
        if (stat[0]) atomicAdd((unsigned long long*)&fs[FS_REJECTED], (unsigned long long)stat[0]);
        if (stat[1]) atomicAdd((unsigned long long*)&fs[FS_DROPPED], (unsigned long long)stat[1]);
        if (stat[2]) atomicAdd((unsigned long long*)&fs[FS_KEPT], (unsigned long long)stat[2]);
        if (nq) q_base = atomicAdd(a.q_count, (unsigned long long)nq);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nq; j += 256) {
        unsigned long long qi = q_base + j;
        if (qi < (unsigned long long)a.q_cap) {  // else: overflow re-pass handles it
            a.q_idx[qi] = cb + q_local[j];
            a.q_frame[qi] = f;
        }
    }
}

// ---------------------------------------------------------------------------
// TMA-staged persistent convert (the product path for 16-byte aligned inputs).
//
// Work unit = CH = 256 consecutive points of one frame (unit u: frame u / mc,
// chunk u % mc, mc = chunks of the largest frame).  Every warp runs its own
// S-stage pipeline in shared memory over units gw, gw + GW, ... (gw = global
// warp index, GW = warps in the grid): lane 0 streams a unit's points and
// its frame's 12 transform coefficients in with cp.async.bulk, completing on
// the stage's mbarrier, and refills the stage with the unit S steps ahead as
// soon as the warp has read it.  No warp ever waits on another warp, and the
// loads of the next S - 1 units are in flight while a unit is binned (one
// unit is ~8 points x ~150 instructions per lane, several microseconds at
// the SM's shared issue rate: two stages hide the copy latency).
//
// Undecided points go into this CTA's private segment of the exact-path queue
// (a shared-memory slot counter, no global atomics); the per-CTA counts land
// in q_bcount and their total in q_count (a segment overflow forces the
// re-pass by pushing q_count past q_cap).  Frame statistics are warp-reduced
// per unit and added with one global atomic per nonzero counter.
__device__ __forceinline__ unsigned smem_u32(const void* p)
{
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity)
{
    unsigned done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

#ifndef STPC_CONVERT_STAGES
#define STPC_CONVERT_STAGES 2
#endif
// A staged unit as its consumers see it (stage header).
struct UnitHdr {
    long long cb;  // first point of the unit
    int f;         // frame
    int n;         // points in the unit (0: past its frame's end)
    int n_staged;  // the first n_staged points are wholly in the stage
    int lead;      // byte offset of point cb within the staged bytes
};

template <class T> struct Staged {
    static constexpr int CH = 256;  // points per warp unit
    static constexpr int S = STPC_CONVERT_STAGES;
    static constexpr int WARPS = 8;
    static constexpr int HDR_BYTES = 32;  // UnitHdr, written by lane 0 before the copy
    static_assert(sizeof(UnitHdr) <= HDR_BYTES, "stage header");
    static constexpr int XF_BYTES = 96;
    static constexpr int PT_BYTES = 3 * CH * (int)sizeof(T) + 32;
    static constexpr int STAGE = HDR_BYTES + XF_BYTES + PT_BYTES;  // 16-byte multiple
    static constexpr int SMEM = WARPS * S * STAGE + WARPS * S * 8;
    static constexpr int PPL = CH / 32;  // points per lane and unit
};

// Lane 0 of a warp: describe unit (f, c) in the stage header and stream its
// points and its frame's transform in (an empty unit completes the phase with
// a transaction-free arrive).  The header's generic stores are ordered before
// the consumers' reads by the mbarrier's release (arrive) / acquire (wait).
template <class T>
__device__ __forceinline__ void issue_unit(const ConvertArgs& a, const T* pts, uint8_t* stage,
                                           unsigned long long* full, int f, int c, long long pt_end_bytes)
{
    constexpr long long PB = 3 * (long long)sizeof(T);
    const long long b = __ldg(a.pt_off + f), e = __ldg(a.pt_off + f + 1);
    const long long cb = b + (long long)c * Staged<T>::CH;
    const int n = (int)max(0ll, min((long long)Staged<T>::CH, e - cb));
    UnitHdr* h = reinterpret_cast<UnitHdr*>(stage);
    if (n == 0) {
        h->n = 0;
        mbar_arrive_tx(full, 0u);
        return;
    }
    const long long lo = cb * PB, hi = (cb + n) * PB;
    const long long a0 = lo & ~15ll;
    long long a1 = (hi + 15) & ~15ll;
    if (a1 > pt_end_bytes) a1 = hi & ~15ll;  // never read past the last point: the tail loads directly
    const unsigned bytes = (unsigned)max(0ll, a1 - a0);
    h->cb = cb;
    h->f = f;
    h->n = n;
    h->lead = (int)(lo - a0);
    h->n_staged = a1 > lo ? min(n, (int)(a1 - lo) / (int)PB) : 0;
    mbar_arrive_tx(full, 96u + bytes);
    bulk_load(stage + Staged<T>::HDR_BYTES, a.xf + 12ll * f, 96u, full);
    if (bytes) bulk_load(stage + Staged<T>::HDR_BYTES + Staged<T>::XF_BYTES, (const uint8_t*)pts + a0, bytes, full);
}

#ifndef STPC_CONVERT_UNROLL
#define STPC_CONVERT_UNROLL 1
#endif
constexpr int CONVERT_UNROLL = STPC_CONVERT_UNROLL;

#ifndef STPC_CONVERT_STAGED_MINB
#define STPC_CONVERT_STAGED_MINB 4
#endif
// IDX32: the batch's grids hold fewer than 2^32 pixels, so a pixel's element
// index is one 32-bit add from the frame's base (a single register held per
// unit) instead of a 64-bit frame * P product rematerialised per point.
template <class T, bool IDX32>
__global__ void __launch_bounds__(256, STPC_CONVERT_STAGED_MINB)
    convert_staged_kernel(ConvertArgs a, const T* pts, int n_units, int mc, int seg)
{
    using SC = Staged<T>;
    constexpr int PB = 3 * (int)sizeof(T);
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ int q_n;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint8_t* ring = smem + w * SC::S * SC::STAGE;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + SC::WARPS * SC::S * SC::STAGE) + w * SC::S;
    const long long pt_end_bytes = __ldg(a.pt_off + a.n_frames) * (long long)PB;
    const int GW = gridDim.x * SC::WARPS;
    const int gw = blockIdx.x * SC::WARPS + w;
    // lane 0's issue cursor (frame fi, chunk ci), advanced by GW units per step
    const int step_f = GW / mc, step_c = GW - (GW / mc) * mc;
    int fi = gw / mc, ci = gw - (gw / mc) * mc;
    if (tid == 0) q_n = 0;
    if (lane == 0) {
        for (int s = 0; s < SC::S; ++s) mbar_init(full + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < SC::S && fi < a.n_frames; ++s) {
            issue_unit<T>(a, pts, ring + s * SC::STAGE, full + s, fi, ci, pt_end_bytes);
            fi += step_f;
            ci += step_c;
            if (ci >= mc) ci -= mc, fi += 1;
        }
    }
    __syncthreads();  // q_n
    long long* qi_seg = a.q_idx + (long long)blockIdx.x * seg;
    int* qf_seg = a.q_frame + (long long)blockIdx.x * seg;
    int k = 0;
    for (int u = gw; u < n_units; u += GW, ++k) {
        const int st = k % SC::S;
        const unsigned par = (unsigned)(k / SC::S) & 1u;
        uint8_t* stage = ring + st * SC::STAGE;
        mbar_wait(full + st, par);
        const UnitHdr h = *reinterpret_cast<const UnitHdr*>(stage);
        int drop = 0, nq = 0;  // kept = n - drop - nq (the exact path counts the queued points)
        if (h.n > 0) {
            const double* xfs = reinterpret_cast<const double*>(stage + SC::HDR_BYTES);
            double c[12];
#pragma unroll
            for (int t = 0; t < 12; ++t) c[t] = xfs[t];
            const uint8_t* sp = stage + SC::HDR_BYTES + SC::XF_BYTES + h.lead;
            unsigned long long* best = a.best + (IDX32 ? 0ll : (long long)h.f * a.g.P);
            const unsigned fb = IDX32 ? (unsigned)h.f * (unsigned)a.g.P : 0u;
            auto bin = [&](int j, T px, T py, T pz) {
                const double qx = (double)px, qy = (double)py, qz = (double)pz;
                const double x = xform_coord(qx, qy, qz, c[0], c[1], c[2], c[9]);
                const double y = xform_coord(qx, qy, qz, c[3], c[4], c[5], c[10]);
                const double z = xform_coord(qx, qy, qz, c[6], c[7], c[8], c[11]);
                int pix;
                double rr;
                const int cls = fast_point(x, y, z, a, pix, rr);
                if (cls == PT_KEEP) {
#if defined(STPC_CONVERT_EXP) && STPC_CONVERT_EXP == 1
                    if (rr == 1.2345) atomicMin(best + pix, (unsigned long long)__double_as_longlong(rr));
#elif defined(STPC_CONVERT_EXP) && STPC_CONVERT_EXP == 2
                    atomicMin(best + (pix & 0x3fff), (unsigned long long)__double_as_longlong(rr));
#else
                    if (IDX32)
                        atomicMin(best + (fb + (unsigned)pix), (unsigned long long)__double_as_longlong(rr));
                    else
                        atomicMin(best + pix, (unsigned long long)__double_as_longlong(rr));
#endif
                } else if (cls == PT_QUEUE) {
                    nq += 1;
                    const int slot = atomicAdd(&q_n, 1);
                    if (slot < seg) {
                        qi_seg[slot] = h.cb + j;
                        qf_seg[slot] = h.f;
                    }
                } else {
                    drop += 1;
                }
            };
            // the staged points from shared memory ...
#pragma unroll CONVERT_UNROLL
            for (int jj = 0; jj < SC::PPL; ++jj) {
                const int j = jj * 32 + lane;
                if (j < h.n_staged) {
                    const T* q = reinterpret_cast<const T*>(sp + PB * j);
                    bin(j, q[0], q[1], q[2]);
                }
            }
            // ... and the array's last point(s) past the 16-byte-aligned stage
            if (h.n_staged < h.n) {
                const int j = h.n_staged + lane;
                if (j < h.n) {
                    const T* q = pts + 3 * (h.cb + j);
                    bin(j, __ldg(q), __ldg(q + 1), __ldg(q + 2));
                }
            }
        }
        __syncwarp();  // every lane is done with the stage
        if (lane == 0 && fi < a.n_frames) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_unit<T>(a, pts, stage, full + st, fi, ci, pt_end_bytes);
            fi += step_f;
            ci += step_c;
            if (ci >= mc) ci -= mc, fi += 1;
        }
        if (h.n > 0) {
            drop = __reduce_add_sync(STPC_FULL, drop);
            nq = __reduce_add_sync(STPC_FULL, nq);
            if (lane == 0) {
                long long* fs = a.fstats + (long long)h.f * FS_COUNT;
                const int kept = h.n - drop - nq;
                if (drop) atomicAdd((unsigned long long*)&fs[FS_DROPPED], (unsigned long long)drop);
                if (kept) atomicAdd((unsigned long long*)&fs[FS_KEPT], (unsigned long long)kept);
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        const int nq = q_n;
        a.q_bcount[blockIdx.x] = min(nq, seg);
        unsigned long long add = (unsigned long long)nq;
        if (nq > seg) add += (unsigned long long)a.q_cap + 1;  // segment overflow: force the re-pass
        if (add) atomicAdd(a.q_count, add);
    }
}

__device__ __forceinline__ void exact_point(const ConvertArgs& a, double px, double py, double pz, int f)
{
    const double* xf = a.xf + 12 * f;
    Binned o = bin_point(px, py, pz, xf, xf + 9, a.g);
    long long* fs = a.fstats + (long long)f * FS_COUNT;
    atomicAdd((unsigned long long*)&fs[o.status == 0 ? FS_REJECTED : o.status == 1 ? FS_DROPPED : FS_KEPT], 1ull);
    if (o.eps) atomicAdd((unsigned long long*)&fs[FS_EPS_BAND], 1ull);
    if (o.status == 2)
        atomicMin(a.best + (long long)f * a.g.P + o.pix, (unsigned long long)__double_as_longlong(o.r));
}

// Queue overflow (more than q_cap undecided points): the queue is discarded and
// every undecided point (fast_point's PT_QUEUE, the same classification every
// main kernel applies) is re-derived here.  grid (1, frames): the usual
// no-overflow case costs one early exit per block.
template <class T>
__global__ void __launch_bounds__(256) convert_overflow_kernel(ConvertArgs a, const T* pts)
{
    if (*a.q_count <= (unsigned long long)a.q_cap) return;
    const int f = blockIdx.y;
    const long long b = a.pt_off[f], e = a.pt_off[f + 1];
    const double* xf = a.xf + 12 * f;
    for (long long i = b + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < e; i += (long long)gridDim.x * blockDim.x) {
        const T* p = pts + 3 * i;
        double px = (double)p[0], py = (double)p[1], pz = (double)p[2];
        double x = xform_coord(px, py, pz, xf[0], xf[1], xf[2], xf[9]);
        double y = xform_coord(px, py, pz, xf[3], xf[4], xf[5], xf[10]);
        double z = xform_coord(px, py, pz, xf[6], xf[7], xf[8], xf[11]);
        int pix;
        double r;
        if (fast_point(x, y, z, a, pix, r) == PT_QUEUE) exact_point(a, px, py, pz, f);
    }
}

// exact_point for one queued point per lane, the whole warp calling (`active`
// lanes hold a point): the frame statistics are added once per distinct
// (frame, counter) of the warp -- consecutive queue entries mostly share a
// frame, and per-point atomics on its few counters serialised.
__device__ __forceinline__ void exact_point_warp(const ConvertArgs& a, bool active, double px, double py, double pz,
                                                 int f)
{
    Binned o{0, 0, 0.0, false};
    if (active) {
        const double* xf = a.xf + 12 * f;
        o = bin_point(px, py, pz, xf, xf + 9, a.g);
        if (o.status == 2)
            atomicMin(a.best + (long long)f * a.g.P + o.pix, (unsigned long long)__double_as_longlong(o.r));
    }
    const int lane = threadIdx.x & 31;
    const int slot = o.status == 0 ? FS_REJECTED : o.status == 1 ? FS_DROPPED : FS_KEPT;
    const unsigned peers = __match_any_sync(STPC_FULL, active ? f * 8 + slot : -1);
    if (active && __ffs(peers) - 1 == lane)
        atomicAdd((unsigned long long*)&a.fstats[(long long)f * FS_COUNT + slot], (unsigned long long)__popc(peers));
    const unsigned ep = __match_any_sync(STPC_FULL, active && o.eps ? f : -1);
    if (active && o.eps && __ffs(ep) - 1 == lane)
        atomicAdd((unsigned long long*)&a.fstats[(long long)f * FS_COUNT + FS_EPS_BAND], (unsigned long long)__popc(ep));
}

// Exact fp64 path (CUDA atan2/acos + correctly rounded refinement in the eps
// band) for the queued points.
template <class T>
__global__ void __launch_bounds__(256) convert_exact_kernel(ConvertArgs a, const T* pts)
{
    const unsigned long long qn = *a.q_count;
    if (qn > (unsigned long long)a.q_cap) return;  // overflow re-pass handles them
    const long long n = (long long)qn;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += stride) {
        const long long q = base + threadIdx.x;
        const bool act = q < n;
        double px = 0.0, py = 0.0, pz = 0.0;
        int f = 0;
        if (act) {
            const T* p = pts + 3 * a.q_idx[q];
            px = (double)p[0], py = (double)p[1], pz = (double)p[2];
            f = a.q_frame[q];
        }
        exact_point_warp(a, act, px, py, pz, f);
    }
}

// The staged kernel's queue: CTA b's undecided points are q_idx[b * seg, +
// q_bcount[b]), spread over gridDim.y blocks per segment.
template <class T>
__global__ void __launch_bounds__(256) convert_exact_seg_kernel(ConvertArgs a, const T* pts, int seg)
{
    if (*a.q_count > (unsigned long long)a.q_cap) return;  // overflow re-pass handles them
    const int n = a.q_bcount[blockIdx.x];
    const long long off = (long long)blockIdx.x * seg;
    for (int base = blockIdx.y * blockDim.x; base < n; base += gridDim.y * blockDim.x) {
        const int q = base + threadIdx.x;
        const bool act = q < n;
        double px = 0.0, py = 0.0, pz = 0.0;
        int f = 0;
        if (act) {
            const T* p = pts + 3 * a.q_idx[off + q];
            px = (double)p[0], py = (double)p[1], pz = (double)p[2];
            f = a.q_frame[off + q];
        }
        exact_point_warp(a, act, px, py, pz, f);
    }
}

template <class T>
__global__ void __launch_bounds__(256) convert_win_kernel(ConvertArgs a, const T* pts)
{
    const int f = blockIdx.y;
    const long long b = a.pt_off[f], e = a.pt_off[f + 1];
    __shared__ double xf[12];
    if (threadIdx.x < 12) xf[threadIdx.x] = a.xf[12 * f + threadIdx.x];
    __syncthreads();
    const unsigned long long* best = a.best + (long long)f * a.g.P;
    long long* win = a.win + (long long)f * a.g.P;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = b + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < e; i += stride) {
        const T* p = pts + 3 * i;
        Binned o = bin_point((double)__ldg(p), (double)__ldg(p + 1), (double)__ldg(p + 2), xf, xf + 9, a.g);
        if (o.status == 2 && isfinite(o.r) &&
            (unsigned long long)__double_as_longlong(o.r) == best[o.pix])
            atomicMin((unsigned long long*)(win + o.pix), (unsigned long long)(i - b));
    }
}

__global__ void win_finalize_kernel(long long* win, const unsigned long long* best, long long n)
{
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (; i < n; i += stride)
        if (best[i] == INF_BITS) win[i] = -1;
}

static dim3 convert_grid(int max_pts, int n_frames)
{
    int bx = (max_pts + 255) / 256;
    if (bx < 1) bx = 1;
    if (bx > 1024) bx = 1024;
    return dim3(bx, n_frames);
}

template <class T>
static dim3 chunk_grid(int max_pts, int n_frames)
{
    int ch = 256 * PPT<T>::value;
    int bx = (max_pts + ch - 1) / ch;
    return dim3(bx < 1 ? 1 : bx, n_frames);
}

template <class T>
static void launch_regs(const ConvertArgs& a, int max_pts, cudaStream_t s)
{
    STPC_LAUNCH();
    convert_kernel<T><<<chunk_grid<T>(max_pts, a.n_frames), 256, 0, s>>>(a, (const T*)a.pts);
    STPC_LAUNCH();
    convert_exact_kernel<T><<<148 * 4, 256, 0, s>>>(a, (const T*)a.pts);
    STPC_LAUNCH();
    convert_overflow_kernel<T><<<dim3(1, a.n_frames), 256, 0, s>>>(a, (const T*)a.pts);
}

#ifndef STPC_EXACT_SPLIT
#define STPC_EXACT_SPLIT 4
#endif
constexpr int EXACT_SPLIT = STPC_EXACT_SPLIT;  // blocks per queue segment

template <class T>
static void launch_staged(const ConvertArgs& a, int max_pts, cudaStream_t s)
{
    using SC = Staged<T>;
    // CTAs resident per device (persistent grid); the dynamic shared-memory
    // opt-in is a per-device function attribute
    constexpr int MAX_DEV = 64;
    static int grid_max_dev[MAX_DEV] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& grid_max = grid_max_dev[dev < MAX_DEV ? dev : MAX_DEV - 1];
    if (!grid_max) {
        cudaFuncSetAttribute(convert_staged_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SC::SMEM);
        cudaFuncSetAttribute(convert_staged_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SC::SMEM);
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, convert_staged_kernel<T, true>, 32 * SC::WARPS, SC::SMEM);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        grid_max = std::max(1, std::min(per_sm * sms, CONVERT_MAX_GRID));
    }
    const int mc = std::max(1, (max_pts + SC::CH - 1) / SC::CH);
    const long long n_units = (long long)mc * a.n_frames;
    if (n_units >= (1ll << 31)) return launch_regs<T>(a, max_pts, s);
    const int grid = (int)std::min<long long>(grid_max, (n_units + SC::WARPS - 1) / SC::WARPS);
    const int seg = (int)std::max<long long>(1, a.q_cap / grid);
    STPC_LAUNCH();
    if ((long long)a.n_frames * a.g.P < (1ll << 32))
        convert_staged_kernel<T, true><<<grid, 32 * SC::WARPS, SC::SMEM, s>>>(a, (const T*)a.pts, (int)n_units, mc, seg);
    else
        convert_staged_kernel<T, false><<<grid, 32 * SC::WARPS, SC::SMEM, s>>>(a, (const T*)a.pts, (int)n_units, mc, seg);
    STPC_LAUNCH();
    convert_exact_seg_kernel<T><<<dim3(grid, EXACT_SPLIT), 256, 0, s>>>(a, (const T*)a.pts, seg);
    STPC_LAUNCH();
    convert_overflow_kernel<T><<<dim3(1, a.n_frames), 256, 0, s>>>(a, (const T*)a.pts);
}

void launch_convert(const ConvertArgs& a0, int max_pts, cudaStream_t s)
{
    if (a0.n_frames <= 0) return;
    ConvertArgs a = a0;
    a.inv_tr = (float)(1.0 / a.g.theta_r);
    a.inv_pr = (float)(1.0 / a.g.phi_r);
    a.phi_off = (float)a.g.phi_offset;
    float mu = (float)FAST_MARGIN * a.inv_tr;
    float mv = (float)FAST_MARGIN * a.inv_pr;
    // The fp32 decision is only sound where the margin is below half a bin
    // and phi_offset survives the float rounding within the error budget
    // (|phi_offset| <= 3.2, the error budget above): otherwise every point
    // takes the exact path (a negative half-width rejects every fraction).
    if (!(mu < 0.5f && mv < 0.5f && fabs(a.g.phi_offset) <= 3.2)) mu = mv = 1.0f;
    a.hu = 0.5f - mu;
    a.hv = 0.5f - mv;
    a.q_bcount = reinterpret_cast<int*>(a.q_count + 1);
    launch_zero(a.q_count, sizeof(unsigned long long), s);
    const bool aligned = (reinterpret_cast<uintptr_t>(a.pts) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(a.xf) & 15) == 0 && !getenv_flag("STPC_CONVERT_REGS");
    if (aligned) {
        if (a.pts_f64) launch_staged<double>(a, max_pts, s);
        else launch_staged<float>(a, max_pts, s);
        return;
    }
    if (a.pts_f64) launch_regs<double>(a, max_pts, s);
    else launch_regs<float>(a, max_pts, s);
}

void launch_convert_win(const ConvertArgs& a, int max_pts, cudaStream_t s)
{
    if (a.n_frames <= 0) return;
    long long n = (long long)a.n_frames * a.g.P;
    launch_fill_u64((unsigned long long*)a.win, 0x7fffffffffffffffull, n, s);
    STPC_LAUNCH();
    if (a.pts_f64)
        convert_win_kernel<double><<<convert_grid(max_pts, a.n_frames), 256, 0, s>>>(a, (const double*)a.pts);
    else
        convert_win_kernel<float><<<convert_grid(max_pts, a.n_frames), 256, 0, s>>>(a, (const float*)a.pts);
    int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
    STPC_LAUNCH();
    win_finalize_kernel<<<blocks, 256, 0, s>>>(a.win, a.best, n);
}

// Escape test without a division: rint(r / q) outside [1, 0xFFFF)
// (bitstream.py:176-182) <=> fl(r / q) <= 0.5 or fl(r / q) > 65534.5 (round
// half to even: rint(0.5) = 0, rint(65534.5) = 65534).  fl(r / q) is
// monotonic in r for q > 0, so both sets are half-lines in r, bounded by the
// largest doubles t_lo / t_hi with fl(t / q) <= 0.5 / <= 65534.5, found once
// on the host by bisection over the bit patterns with IEEE division.
static double largest_r_with_quot_le(double q, double x)
{
    unsigned long long lo = 0, hi = 0x7ff0000000000000ull;  // [+0, +inf]
    while (hi - lo > 1) {
        const unsigned long long mid = lo + (hi - lo) / 2;
        double r;
        std::memcpy(&r, &mid, 8);
        if (r / q <= x) lo = mid;
        else hi = mid;
    }
    double r;
    std::memcpy(&r, &lo, 8);
    return r;
}

void escape_thresholds(double range_quant, double& t_lo, double& t_hi)
{
    t_lo = largest_r_with_quot_le(range_quant, 0.5);
    t_hi = largest_r_with_quot_le(range_quant, 65534.5);
}

// One warp per 32 bitmap words (1024 pixels) of one frame: ballot the
// validity / escape predicates and store packbits-ordered words.
__global__ void __launch_bounds__(256) bitmap_kernel(const double* __restrict__ best, Geometry g,
                                                     double t_lo, double t_hi, uint8_t* vbits, uint8_t* ebits,
                                                     long long* fstats)
{
    const int f = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const long long words = (long long)g.pbs / 4;
    const long long wbase = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
    if (wbase >= words) return;
    const double* img = best + (long long)f * g.P;
    uint32_t my_v = 0, my_e = 0;
    int nvalid = 0;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
        const long long pix = (wbase + i) * 32 + lane;
        const double r = pix < g.P ? __ldg(img + pix) : __longlong_as_double(0x7ff0000000000000ll);
        const bool valid = isfinite(r);
        const bool esc = valid && (r <= t_lo || r > t_hi);
        const uint32_t mv = __ballot_sync(STPC_FULL, valid);
        const uint32_t me = __ballot_sync(STPC_FULL, esc);
        if (lane == i) {
            my_v = mv;
            my_e = me;
        }
        nvalid += __popc(mv);
    }
    if (wbase + lane < words) {
        reinterpret_cast<uint32_t*>(vbits + (long long)f * g.pbs)[wbase + lane] = natural_bits(my_v);
        reinterpret_cast<uint32_t*>(ebits + (long long)f * g.pbs)[wbase + lane] = natural_bits(my_e);
    }
    if (lane == 0 && nvalid)
        atomicAdd((unsigned long long*)&fstats[(long long)f * FS_COUNT + FS_VALID], (unsigned long long)nvalid);
}

void launch_bitmaps(const double* best, int n_frames, const Geometry& g, double range_quant,
                    uint8_t* vbits, uint8_t* ebits, long long* fstats, cudaStream_t s)
{
    if (n_frames <= 0) return;
    double t_lo, t_hi;
    escape_thresholds(range_quant, t_lo, t_hi);
    long long words = g.pbs / 4;
    long long warps = (words + 31) / 32;
    dim3 grid((unsigned)((warps + 7) / 8), n_frames);
    STPC_LAUNCH();
    bitmap_kernel<<<grid, 256, 0, s>>>(best, g, t_lo, t_hi, vbits, ebits, fstats);
}

}  // namespace stpc
