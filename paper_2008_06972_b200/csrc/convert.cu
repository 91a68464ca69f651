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
#include <cstring>

#include "kernels.cuh"
#include "dd.cuh"

namespace stpc {

static constexpr unsigned long long INF_BITS = 0x7ff0000000000000ull;

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
// within ~1.3e-6 rad of the true ones (input rounding 2^-24 relative plus the
// polynomial atan below); whenever both angles lie more than
// FAST_MARGIN = 1e-5 rad from a bin edge the floor is therefore the same as
// the reference's fp64 (glibc) floor and the point is binned here.  The ~1%
// of points inside the margin (and any point with coordinates outside
// [1e-15, 1e15]) go to the exact fp64 path.  Returns false when undecided.
constexpr double FAST_MARGIN = 1e-5;

// atan2 for the fast path, entirely in fp32: odd minimax-style polynomial of
// degree 13 in t = min/max (max error 3.2e-7 rad in float32 FMA evaluation,
// measured on 2M points) and float reflections (pi/2, pi rounded to float:
// <= 9e-8 rad each, plus half-ulp roundings <= 1.2e-7 rad per step).
__device__ __forceinline__ float fast_atan2f(float y, float x)
{
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float t = __fdividef(mn, mx);
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

// Error budget of the fp32 decision (in bins of the azimuth; elevation is
// analogous and smaller): angle error <= 3.2e-7 (polynomial) + 1.2e-7 (input
// rounding of x, y, z to float) + 5e-7 (reflections, + 2 pi wrap) rad, and
// qu = th * inv_tr in float adds a relative 1.2e-7, i.e. <= 2 pi * 1.2e-7 *
// inv_tr bins.  Total < 2.75e-6 * inv_tr bins against a margin of
// FAST_MARGIN * inv_tr = 1e-5 * inv_tr bins: 3.6x headroom at any resolution.
__device__ __forceinline__ bool fast_bin(double x, double y, double z, const Geometry& g, float inv_tr,
                                         float inv_pr, float phi_off, float mu, float mv, int& u, int& v)
{
    const float xf = (float)x, yf = (float)y, zf = (float)z;
    const float mxy = fmaxf(fabsf(xf), fabsf(yf));
    const float mall = fmaxf(mxy, fabsf(zf));
    // keep squares and ratios in float range (coordinates outside [1e-15,
    // 1e15] go exact: below 1e-15 x^2 + y^2 could underflow); degenerate
    // directions go exact
    if (!(mall < 1e15f && mxy > 1e-15f)) return false;
    float th = fast_atan2f(xf, yf);
    th = th < 0.0f ? th + 6.28318548f : th;
    const float qu = th * inv_tr;
    const float ph = fast_atan2f(sqrtf(xf * xf + yf * yf), zf);
    const float qv = (ph - phi_off) * inv_pr;
    const float flu = floorf(qu), flv = floorf(qv);
    const float fu = qu - flu, fv = qv - flv;
    if (fu < mu || fu > 1.0f - mu || fv < mv || fv > 1.0f - mv) return false;
    // 0 <= qu <= 2 pi / theta_r, which CodecConfig does not tie to w: the
    // reference's floor(theta / theta_r) % w needs a true modulo whenever the
    // sensor's w bins cover less than the full circle.  (A point is only
    // accepted with mu < 0.5, i.e. 1/theta_r < 5e4, so qu < 3.2e5 fits an int;
    // see launch_convert.)
    const int uq = (int)flu;
    u = uq >= g.w ? uq % g.w : uq;
    v = (int)flv;
    return true;
}

// Points per thread: loads for all of them are issued before any binning.
template <class T> struct PPT { static constexpr int value = 8; };
template <> struct PPT<double> { static constexpr int value = 4; };

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
        if (!(isfinite(x) && isfinite(y) && isfinite(z))) {
            rej += 1;
            continue;
        }
        double r = sqrt((x * x + y * y) + z * z);
        int u, v;
        if (r <= 0.0) {
            rej += 1;
        } else if (isfinite(r) && fast_bin(x, y, z, a.g, a.inv_tr, a.inv_pr, a.phi_off, a.mu, a.mv, u, v)) {
            if (v < 0 || v >= a.g.h) {
                drop += 1;
            } else {
                kept += 1;
                atomicMin(best + (v * a.g.w + u), (unsigned long long)__double_as_longlong(r));
            }
        } else {  // undecided: block-local queue
            int slot = atomicAdd(&q_n, 1);
            q_local[slot] = (int)(i - cb);
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
// every undecided point is re-derived here.  grid (1, frames): the usual
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
        if (!(isfinite(x) && isfinite(y) && isfinite(z))) continue;
        double r = sqrt((x * x + y * y) + z * z);
        int u, v;
        if (r <= 0.0 || (isfinite(r) && fast_bin(x, y, z, a.g, a.inv_tr, a.inv_pr, a.phi_off, a.mu, a.mv, u, v)))
            continue;
        exact_point(a, px, py, pz, f);
    }
}

// Exact fp64 path (CUDA atan2/acos + correctly rounded refinement in the eps
// band) for the queued points.
template <class T>
__global__ void __launch_bounds__(256) convert_exact_kernel(ConvertArgs a, const T* pts)
{
    const unsigned long long qn = *a.q_count;
    if (qn > (unsigned long long)a.q_cap) return;  // overflow re-pass handles them
    const long long n = (long long)qn;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        const long long i = a.q_idx[q];
        const T* p = pts + 3 * i;
        exact_point(a, (double)p[0], (double)p[1], (double)p[2], a.q_frame[q]);
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

void launch_convert(const ConvertArgs& a0, int max_pts, cudaStream_t s)
{
    if (a0.n_frames <= 0) return;
    ConvertArgs a = a0;
    a.inv_tr = (float)(1.0 / a.g.theta_r);
    a.inv_pr = (float)(1.0 / a.g.phi_r);
    a.phi_off = (float)a.g.phi_offset;
    a.mu = (float)FAST_MARGIN * a.inv_tr;
    a.mv = (float)FAST_MARGIN * a.inv_pr;
    // The fp32 decision is only sound where the margin is below half a bin
    // and phi_offset survives the float rounding within the error budget
    // (2^-24 |phi_offset| << FAST_MARGIN): otherwise every point takes the
    // exact path (mu = 1 rejects every fraction).
    if (!(a.mu < 0.5f && a.mv < 0.5f && fabs(a.g.phi_offset) < 16.0)) a.mu = a.mv = 1.0f;
    launch_zero(a.q_count, sizeof(unsigned long long), s);
    STPC_LAUNCH();
    if (a.pts_f64)
        convert_kernel<double><<<chunk_grid<double>(max_pts, a.n_frames), 256, 0, s>>>(a, (const double*)a.pts);
    else
        convert_kernel<float><<<chunk_grid<float>(max_pts, a.n_frames), 256, 0, s>>>(a, (const float*)a.pts);
    STPC_LAUNCH();
    if (a.pts_f64)
        convert_exact_kernel<double><<<148 * 4, 256, 0, s>>>(a, (const double*)a.pts);
    else
        convert_exact_kernel<float><<<148 * 4, 256, 0, s>>>(a, (const float*)a.pts);
    STPC_LAUNCH();
    if (a.pts_f64)
        convert_overflow_kernel<double><<<dim3(1, a.n_frames), 256, 0, s>>>(a, (const double*)a.pts);
    else
        convert_overflow_kernel<float><<<dim3(1, a.n_frames), 256, 0, s>>>(a, (const float*)a.pts);
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
