// K2 / K3b -- greedy plane-run growth per tile-row, and K3a -- temporal offset
// refit of key-frame runs.
//
// fit_rows replaces encode_tile_row + _add_tile + plane_from_sums + _span_ok
// (/root/reference/pkg/src/stpc/_kernels.py:23-76, 108-228) as called by
// encode_stream pass 1 and pass 2 (/root/reference/pkg/src/stpc/temporal.py:
// 127-154, 174-201).  refit replaces refit_spans (_kernels.py:231-279).
//
// One warp owns one (frame, tile-row) chain; the chain is inherently
// sequential (each decision changes the next union), so parallelism comes
// from the many chains of a batch and from the lanes inside each step:
//   * moments: lanes compute the 9 products of up to 32 pixels at once and
//     transpose them through shared memory; lane k then folds sum k over the
//     pixels in raster order -- the reference's rounding sequence, not a tree
//     (a shuffle tree flips run decisions).  Invalid
//     pixels contribute +0.0, which is exact: a running sum that starts at
//     +0.0 can never become -0.0 under round-to-nearest, and s + 0.0 == s;
//   * union re-test: order-independent AND over pixels, 32 lanes at a time
//     with an early-out vote (the reference's early return gives the same
//     verdict);
//   * the 3x3 solve runs redundantly in every lane (warp-uniform branches).
// Pass 2's `remaining` mask (valid & ~temporally covered) is realised by the
// refit kernel overwriting covered P-frame pixels with +inf (= invalid), so
// the fit needs no per-pixel exclusion test.
#include "kernels.cuh"
#include <cstdlib>

namespace stpc {

constexpr int FIT_WARPS = 4;  // warps per block

// q, r = p / d, p % d for 0 <= p < 2^24 without an integer divide: float
// reciprocal estimate, then an exact +-1 correction.
__device__ __forceinline__ void divmod_small(int p, int d, float rcp, int& q, int& r)
{
    q = __float2int_rz(((float)p + 0.5f) * rcp);
    r = p - q * d;
    if (r < 0) { q -= 1; r += d; }
    else if (r >= d) { q += 1; r -= d; }
}

struct Chain {
    const double* img;    // frame's best grid (covered pixels already +inf in pass 2)
    const uint8_t* crow;  // tile classes of this tile-row
    float4* cert;         // per-tile test certificates of this chain (CERT_F4 float4 per tile)
    bool skip1;           // pass 2: tiles of class 1 are fully masked
    int v0, rows;
};

// Fold the valid pixels of tile t onto the lane-owned running sums (lane k<9
// owns sum k; lanes >= 9 shadow sum 8).  Returns the valid count (uniform).
// The first 32 pixels of tile t+1 are loaded into `pf` while this step's
// solve and test run, hiding the L2/HBM latency of the next fold.
struct Prefetch {
    int t = -1;
    double r;
};

__device__ __forceinline__ double load_px(const Chain& ch, const Geometry& g, int t, int p, int& v, int& u)
{
    const int u0 = t * g.tw;
    const int cols = min(g.tw, g.w - u0);
    int dv, du;
    divmod_small(p, cols, __frcp_rn((float)cols), dv, du);
    v = ch.v0 + dv;
    u = u0 + du;
    return ch.img[(long long)v * g.w + u];
}

__device__ __forceinline__ int fold_tile(const Chain& ch, const Geometry& g, const Trig& tg, int t,
                                         double* sm, double& acc, Prefetch& pf)
{
    const int lane = threadIdx.x & 31;
    const bool hit = pf.t == t;
    const double pr = pf.r;
    // prefetch chunk 0 of the next tile (consumed by the next fold call)
    if (t + 1 < g.tx) {
        const int ncols = min(g.tw, g.w - (t + 1) * g.tw);
        double r = __longlong_as_double(0x7ff0000000000000ll);
        if (lane < ch.rows * ncols) {
            int v, u;
            r = load_px(ch, g, t + 1, lane, v, u);
        }
        pf.r = r;
        pf.t = t + 1;
    }
    if (ch.skip1 && ch.crow[t] == 1) return 0;
    const int kk = lane < 9 ? lane : 8;
    const int u0 = t * g.tw;
    const int cols = min(g.tw, g.w - u0);
    const int npx = ch.rows * cols;
    const float rc = __frcp_rn((float)cols);
    int cnt = 0;
    for (int base = 0; base < npx; base += 32) {
        int p = base + lane;
        double x = 0.0, y = 0.0, z = 0.0, one = 0.0;
        if (p < npx) {
            int dv, du;
            divmod_small(p, cols, rc, dv, du);
            int v = ch.v0 + dv, u = u0 + du;
            double r = (hit && base == 0) ? pr : ch.img[(long long)v * g.w + u];
            if (isfinite(r)) {
                double dx, dy, dz;
                ray_dir(tg, v, u, dx, dy, dz);
                x = r * dx;
                y = r * dy;
                z = r * dz;
                one = 1.0;
            }
        }
        cnt += __popc(__ballot_sync(STPC_FULL, one != 0.0));
        double* row = sm + lane * 9;
        row[0] = y * y;
        row[1] = y * z;
        row[2] = z * z;
        row[3] = y;
        row[4] = z;
        row[5] = x * y;
        row[6] = x * z;
        row[7] = x;
        row[8] = one;
        __syncwarp();
        const int nj = min(32, npx - base);
        if (nj == 16) {  // 4x4 tiles: fully unrolled ordered fold
#pragma unroll
            for (int j = 0; j < 16; ++j) acc += sm[j * 9 + kk];  // +0.0 for invalid: exact
        } else {
#pragma unroll 4
            for (int j = 0; j < nj; ++j) acc += sm[j * 9 + kk];
        }
        __syncwarp();
    }
    return cnt;
}

// ---------------------------------------------------------------------------
// Union re-test with per-tile certificates.
//
// The reference re-tests every pixel of the union [s, e] after each growth
// step (_span_ok, O(L^2) pixel tests per run; ~17 tests per pixel on a
// 64-beam frame).  Here a tile that passed a full test under plane
// P = (a, b, c) records a certificate over its valid pixels: the margin
// m = tau - max|r - r_hat| (>= 0), dmin = min|den|, rmin/rmax = min/max r_hat
// and the box [ymin, ymax] x [zmin, zmax] of the reconstructed points
// y^ = r_hat dy, z^ = r_hat dz.  For a new plane P' = P + (da, db, dc):
//     den'  = den + da dy + db dz,           |den'| >= dmin - |da| - |db|
//     r_hat' - r_hat = (dc den - c (da dy + db dz)) / (den den')
//                    = (dc - da y^ - db z^) / den'.
// The numerator is affine in (y^, z^), so its largest magnitude over the box
// is at a corner:  B = max_corners |dc - da y - db z| / (dmin - |da| - |db|).
// If B (inflated by a relative 1e-6 and 1e-9 m, far above fp64 rounding) is
// below m, rmin - B > 0, rmax + B < r_max and dmin - |da| - |db| > 1e-12,
// every pixel of the tile provably passes under P', exactly as the
// reference's per-pixel test decides, and the tile is not re-tested;
// otherwise it is tested pixel by pixel (and re-certified).  Verdicts are
// identical; only the work changes.
//
// Layout (CERT_F4 = 2 float4): c0 = (a, b, c, X), c1 = (dmin, yc, zc, radii).
// X is the slack min over the pixels of min(tau - |r - r_hat|, r_hat,
// r_max - r_hat), so the three conditions B < m, B < rmin, B < r_max - rmax
// are the single B < X.  The box is stored as centre (yc, zc) and radii
// (two bf16 values rounded up, packed in one word): the largest |n| over a
// box is |n(centre)| + |da| ry + |db| rz, one evaluation instead of four
// corners.  The check (cert_holds_f) is division-free and runs in fp32 with
// every rounding covered: max|n| (1 + 3e-6) < (X - 1e-9) (dmin - |da| - |db|).
// ---------------------------------------------------------------------------

// Order-preserving map of a float to unsigned (for REDUX min/max of signed values).
__device__ __forceinline__ unsigned f2key(float f)
{
    unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(unsigned k)
{
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

constexpr float CERT_EMPTY = 3.4e38f;  // m of a tile with no valid pixels

// The certificate of a tile that passed under plane (a, b, c), from its
// outward-rounded statistics: slack X, min |den| and the box of the
// reconstructed points.  The box is kept as centre and radii (the largest
// magnitude of an affine function over a box is its centre value plus the
// radius terms), the radii rounded up to 16 significant bits and packed.
__device__ __forceinline__ unsigned radius_bits(float r)  // r >= 0, rounded up to bf16 precision
{
    return (__float_as_uint(r) + 0xffffu) & 0xffff0000u;
}
__device__ __forceinline__ void cert_store(float4* ce, float a, float b, float c, float X, float dmin, float ylo,
                                           float yhi, float zlo, float zhi)
{
    const float yc = 0.5f * (ylo + yhi), zc = 0.5f * (zlo + zhi);
    const float ry = fmaxf(__fsub_ru(yhi, yc), __fsub_ru(yc, ylo));
    const float rz = fmaxf(__fsub_ru(zhi, zc), __fsub_ru(zc, zlo));
    ce[0] = make_float4(a, b, c, X);
    ce[1] = make_float4(dmin, yc, zc, __uint_as_float(radius_bits(ry) | (radius_bits(rz) >> 16)));
}

// Full pixel test of tile t under (a, b, c); on pass, lane 0 stores the
// tile's certificate.  Returns the verdict (warp-uniform).
__device__ bool test_tile(const Chain& ch, const Geometry& g, const Trig& tg, int t, double a, double b,
                          double c, double tau, double r_max)
{
    const int lane = threadIdx.x & 31;
    const int u0 = t * g.tw;
    const int cols = min(g.tw, g.w - u0);
    const int npx = ch.rows * cols;  // callers never test masked (class-1) tiles
    const float rc = __frcp_rn((float)cols);
    double X = 1e300, dmin = 1e300;  // slack min(tau - |r - r_hat|, r_hat, r_max - r_hat), as test_tile_pair
    double ylo = 1e300, yhi = -1e300, zlo = 1e300, zhi = -1e300;
    for (int base = 0; base < npx; base += 32) {
        int p = base + lane;
        bool bad = false;
        if (p < npx) {
            int dv, du;
            divmod_small(p, cols, rc, dv, du);
            int v = ch.v0 + dv, u = u0 + du;
            double r = ch.img[(long long)v * g.w + u];
            if (isfinite(r)) {
                double dx, dy, dz;
                ray_dir(tg, v, u, dx, dy, dz);
                double den = (dx + a * dy) + b * dz;
                double ad = fabs(den);
                if (ad < STPC_PARALLEL_EPS) {
                    bad = true;
                } else {
                    double r_hat = c / den;
                    if (r_hat <= 0.0 || r_hat > r_max || fabs(r - r_hat) > tau) {
                        bad = true;
                    } else {
                        X = fmin(X, fmin(fmin(tau - fabs(r - r_hat), r_hat), r_max - r_hat));
                        dmin = fmin(dmin, ad);
                        const double yh = r_hat * dy, zh = r_hat * dz;
                        ylo = fmin(ylo, yh);
                        yhi = fmax(yhi, yh);
                        zlo = fmin(zlo, zh);
                        zhi = fmax(zhi, zh);
                    }
                }
            }
        }
        if (__any_sync(STPC_FULL, bad)) return false;
    }
    // X, dmin are >= 0: their float bit patterns order like their values; the
    // signed box uses an order-preserving key.  One REDUX each, every value
    // rounded outward first.
    const unsigned ux = __reduce_min_sync(STPC_FULL, __float_as_uint(__double2float_rd(fmin(X, 3.0e38))));
    const unsigned ud = __reduce_min_sync(STPC_FULL, __float_as_uint(__double2float_rd(fmin(dmin, 3.0e38))));
    const unsigned ky0 = __reduce_min_sync(STPC_FULL, f2key(__double2float_rd(fmax(fmin(ylo, 3.0e38), -3.0e38))));
    const unsigned ky1 = __reduce_max_sync(STPC_FULL, f2key(__double2float_ru(fmin(fmax(yhi, -3.0e38), 3.0e38))));
    const unsigned kz0 = __reduce_min_sync(STPC_FULL, f2key(__double2float_rd(fmax(fmin(zlo, 3.0e38), -3.0e38))));
    const unsigned kz1 = __reduce_max_sync(STPC_FULL, f2key(__double2float_ru(fmin(fmax(zhi, -3.0e38), 3.0e38))));
    if (lane == 0)
        cert_store(ch.cert + CERT_F4 * t, (float)a, (float)b, (float)c, __uint_as_float(ux), __uint_as_float(ud),
                   key2f(ky0), key2f(ky1), key2f(kz0), key2f(kz1));  // a/b/c are f32-exact
    return true;
}

// Does tile j's certificate prove it passes under (a, b, c)?  Evaluated in
// fp32 (a, b, c and the certificate's plane are f32-exact) with every
// rounding covered: u = 2^-24 per operation, so the centre value n carries
// at most ~4u (|dc| + |da yc| + |db zc|) of error (E below takes 8u), the
// sums and products of lhs at most 4u relative (it takes 4e-6), dlo errs low
// by its 1e-6 factors and X high by 2e-6; the result implies the exact
//     (max_box |dc - da y - db z| / (dmin - |da| - |db|)) (1 + 1e-6) + 1e-9 < X.
// Branch-free: both loads issue at once; a NaN field fails the comparison;
// stale fields of an empty tile are ignored.
__device__ __forceinline__ bool cert_holds_f(const float4* cert, int j, float a, float b, float c)
{
    const float4 c0 = cert[CERT_F4 * j], c1 = cert[CERT_F4 * j + 1];
    const float da = a - c0.x, db = b - c0.y, dc = c - c0.z;
    const float ada = fabsf(da), adb = fabsf(db);
    const float dlo = __fmaf_rn(-(1.0f + 1e-6f), ada + adb, c1.x * (1.0f - 1e-6f));
    const float ry = __uint_as_float(__float_as_uint(c1.w) & 0xffff0000u);
    const float rz = __uint_as_float(__float_as_uint(c1.w) << 16);
    const float t1 = da * c1.y, t2 = db * c1.z;
    const float n = (dc - t1) - t2;
    const float E = 5e-7f * ((fabsf(dc) + fabsf(t1)) + fabsf(t2));
    const float T = __fmaf_rn(adb, rz, ada * ry);
    const float lhs = ((fabsf(n) + E) + T) * (1.0f + 4e-6f);
    const float rhs = __fmaf_rn(c0.w, 1.0f - 2e-6f, -1e-9f) * dlo;
    const bool proven = dlo > 1e-6f && lhs < rhs;
    return c0.w >= CERT_EMPTY || proven;
}

// Union [s, e] under (a, b, c): new tile e in full, older tiles by
// certificate, falling back to a full test where the certificate is too weak.
__device__ bool union_fits(const Chain& ch, const Geometry& g, const Trig& tg, int s, int e, double a,
                           double b, double c, double tau, double r_max)
{
    const int lane = threadIdx.x & 31;
    if (!test_tile(ch, g, tg, e, a, b, c, tau, r_max)) return false;
    const float af = (float)a, bf = (float)b, cf = (float)c;  // f32-exact
    for (int base = s; base < e; base += 32) {
        const int j = base + lane;
        bool weak = j < e && !cert_holds_f(ch.cert, j, af, bf, cf);
        uint32_t wm = __ballot_sync(STPC_FULL, weak);
        while (wm) {
            const int jj = base + __ffs(wm) - 1;
            wm &= wm - 1;
            if (!test_tile(ch, g, tg, jj, a, b, c, tau, r_max)) return false;
        }
    }
    return true;
}

// ---------------------------------------------------------------------------
// Start verdicts in parallel.  A START step folds its tile from zero, so its
// outcome (sums >= 3 pixels, solve ok, f32-rounded plane passes the tile)
// depends on that tile alone, not on the chain.  One thread per tile
// evaluates it with the identical sequential raster fold, and on a pass
// stores the tile's certificate (whose plane is the start plane).  The
// chains then skip residual tiles with a byte lookup.
// ---------------------------------------------------------------------------
// TW x TH > 0: compile-time tile shape (all pixel loads issued up front);
// 0 x 0: runtime shape.
// Start verdicts, staged: a block of START_TPB threads owns START_TPB
// consecutive tiles of one tile-row.  Thread-per-tile pixel reads would put
// every lane in a different 32-byte sector (the kernel measured L1-wavefront
// bound), so the block first copies its slab -- rows [v0, v1) x the tiles'
// columns -- and the column trig factors into shared memory with coalesced
// loads, tile-major with one double of padding per tile (conflict-free
// per-thread reads), then each thread folds, solves and tests its own tile.
constexpr int START_TPB = 128;
constexpr int START_MAXPX = 16;  // staged path: tiles of up to 16 pixels

template <int TW>
#ifndef STPC_STAGED_MINB
#define STPC_STAGED_MINB 8  // measured (start_p): 1 -> 5.92 ms, 6 -> 5.62, 8 -> 5.43
#endif
__global__ void __launch_bounds__(START_TPB, STPC_STAGED_MINB) start_tiles_staged_kernel(FitArgs A)
{
    constexpr int STRIDE = START_MAXPX + 1;
    __shared__ double s_r[START_TPB * STRIDE];
    __shared__ double s_st[START_TPB * (TW + 1)], s_ct[START_TPB * (TW + 1)];  // padded: conflict-free
    const Geometry& g = A.g;
    const int th = g.th;
    const int bpc = (g.tx + START_TPB - 1) / START_TPB;  // blocks per chain
    const long long cj = blockIdx.x / bpc;                // chain within this pass
    const int t0 = (int)(blockIdx.x % bpc) * START_TPB;
    const int job = (int)(cj / g.ty);
    const int tr = (int)(cj % g.ty);
    int frame;
    if (A.mode == 0) {
        frame = job * A.n_frames_group + A.k;
    } else {
        int np = A.n_frames_group - 1;
        int grp = job / np, i = job % np;
        frame = grp * A.n_frames_group + (i < A.k ? i : i + 1);
    }
    const long long slot = (long long)frame * g.ty + tr;
    const double* img = A.best + (long long)frame * g.P;
    const int v0 = tr * th, rows = min(th, g.h - v0);
    const int U0 = t0 * TW;
    const int ncol = min(START_TPB * TW, g.w - U0);
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    // coalesced staging: row by row, consecutive threads -> consecutive columns
    for (int dv = 0; dv < th; ++dv)
#pragma unroll
        for (int k = 0; k < TW; ++k) {
            const int c = k * START_TPB + threadIdx.x;
            const int tl = c / TW, du = c % TW;
            double r = INF;
            if (dv < rows && c < ncol) r = __ldg(img + (long long)(v0 + dv) * g.w + U0 + c);
            s_r[tl * STRIDE + dv * TW + du] = r;
        }
#pragma unroll
    for (int k = 0; k < TW; ++k) {
        const int c = k * START_TPB + threadIdx.x;
        const bool in = c < ncol;
        const int o = (c / TW) * (TW + 1) + c % TW;
        s_st[o] = in ? __ldg(A.tg.sin_t + U0 + c) : 0.0;
        s_ct[o] = in ? __ldg(A.tg.cos_t + U0 + c) : 0.0;
    }
    __syncthreads();
    const int t = t0 + threadIdx.x;
    if (t >= g.tx) return;
    uint8_t* sok = A.start_ok + slot * g.tx + t;
    if (A.mode != 0 && A.cls[slot * g.tx + t] == 1) {
        *sok = 0;
        return;
    }
    const double* rr = s_r + threadIdx.x * STRIDE;
    const double* st = s_st + threadIdx.x * (TW + 1);
    const double* ct = s_ct + threadIdx.x * (TW + 1);
    const int cols = min(TW, g.w - t * TW);
    // Branch-free ordered fold: an invalid pixel (or a column past the image
    // edge) contributes +0.0 to every sum, which is exact -- a running sum
    // that starts at +0.0 never becomes -0.0 -- so the lanes of a warp stay
    // converged through data-dependent validity.
    double sm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int dv = 0; dv < rows; ++dv) {
        const double sp = __ldg(A.tg.sin_p + v0 + dv), cp = __ldg(A.tg.cos_p + v0 + dv);
#pragma unroll
        for (int du = 0; du < TW; ++du) {
            const double rv = rr[dv * TW + du];
            const bool valid = du < cols && isfinite(rv);
            // an invalid pixel folds as r = 0: its products are +-0.0, and
            // adding either zero to a sum that started at +0.0 is exact
            const double r = valid ? rv : 0.0;
            const double dx = sp * st[du], dy = sp * ct[du], dz = cp;
            const double x = r * dx, y = r * dy, z = r * dz;
            sm[0] += y * y; sm[1] += y * z; sm[2] += z * z;
            sm[3] += y;     sm[4] += z;     sm[5] += x * y;
            sm[6] += x * z; sm[7] += x;     sm[8] += valid ? 1.0 : 0.0;
        }
    }
    // the chain's start step takes these sums instead of re-folding the tile
    // (stored for every tile with enough points; read only where the verdict passes)
    if (A.start_sums && sm[8] >= 3.0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) A.start_sums[k * A.sums_stride + slot * g.tx + t] = sm[k];
    }
    const bool empty = sm[8] == 0.0;  // no valid pixel: 2, which the chains skip over in bulk
    double a, b, c;
    bool ok = sm[8] >= 3.0 && plane_from_sums(sm, A.cond_limit, a, b, c);
    // certificate statistics in fp32, each rounded outward on conversion
    // (half the registers and selects of fp64 min/max)
    float X = 3.4e38f, dmin = 3.4e38f;
    float ylo = 3.4e38f, yhi = -3.4e38f, zlo = 3.4e38f, zhi = -3.4e38f;
    if (ok) {
        a = f32_round(a);
        b = f32_round(b);
        c = f32_round(c);
        // verdict and certificate statistics in one branch-free pass: the
        // verdict is the AND over valid pixels (the reference's early return
        // gives the same answer); masked pixels leave every statistic alone
        for (int dv = 0; dv < rows; ++dv) {
            const double sp = __ldg(A.tg.sin_p + v0 + dv), cp = __ldg(A.tg.cos_p + v0 + dv);
#pragma unroll
            for (int du = 0; du < TW; ++du) {
                const double r = rr[dv * TW + du];
                const bool valid = du < cols && isfinite(r);
                const double dy = sp * ct[du];
                const double den = (sp * st[du] + a * dy) + b * cp;
                const double ad = fabs(den);
                const bool par = ad < STPC_PARALLEL_EPS;
                const double r_hat = c / (par ? 1.0 : den);
                const double err = fabs(r - r_hat);
                const bool bad = par || r_hat <= 0.0 || r_hat > A.r_max || err > A.tau;
                ok = ok && !(valid && bad);
                const bool use = valid && !bad;
                const double yh = r_hat * dy, zh = r_hat * cp;
                // the pixel's slack: B < tau - err, B < r_hat, B < r_max - r_hat in one field
                const float xs = __double2float_rd(fmin(fmin(A.tau - err, r_hat), A.r_max - r_hat));
                X = use ? fminf(X, xs) : X;
                dmin = use ? fminf(dmin, __double2float_rd(ad)) : dmin;
                ylo = use ? fminf(ylo, __double2float_rd(yh)) : ylo;
                yhi = use ? fmaxf(yhi, __double2float_ru(yh)) : yhi;
                zlo = use ? fminf(zlo, __double2float_rd(zh)) : zlo;
                zhi = use ? fmaxf(zhi, __double2float_ru(zh)) : zhi;
            }
        }
    }
    *sok = ok ? 1 : (empty ? 2 : 0);
    if (!ok) return;
    cert_store(A.cert + (slot * g.tx + t) * CERT_F4, (float)a, (float)b, (float)c, X, dmin, ylo, yhi, zlo, zhi);
}

#ifndef STPC_START_MINB
#define STPC_START_MINB 2
#endif
template <int TW, int TH>
__global__ void __launch_bounds__(256, STPC_START_MINB) start_tiles_kernel(FitArgs A)
{
    const Geometry& g = A.g;
    const int tw = TW > 0 ? TW : g.tw;
    const int th = TH > 0 ? TH : g.th;
    const long long n_tiles = (long long)A.n_jobs * g.ty * g.tx;
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n_tiles) return;
    const int t = (int)(id % g.tx);
    const long long cj = id / g.tx;  // chain within this pass
    const int job = (int)(cj / g.ty);
    const int tr = (int)(cj % g.ty);
    int frame;
    if (A.mode == 0) {
        frame = job * A.n_frames_group + A.k;
    } else {
        int np = A.n_frames_group - 1;
        int grp = job / np, i = job % np;
        frame = grp * A.n_frames_group + (i < A.k ? i : i + 1);
    }
    const long long slot = (long long)frame * g.ty + tr;
    uint8_t* sok = A.start_ok + slot * g.tx + t;
    if (A.mode != 0 && A.cls[slot * g.tx + t] == 1) {
        *sok = 0;
        return;
    }
    const double* img = A.best + (long long)frame * g.P;
    const int v0 = tr * th, v1 = min(v0 + th, g.h);
    const int u0 = t * tw, u1 = min(u0 + tw, g.w);
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    constexpr int NP = TW * TH;
    double rr[NP > 0 ? NP : 1];
    if constexpr (NP > 0) {
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const int v = v0 + i / TW, u = u0 + i % TW;
            rr[i] = (v < v1 && u < u1) ? __ldg(img + (long long)v * g.w + u) : INF;
        }
    }
    auto pix = [&](int i, int& v, int& u) {
        if constexpr (NP > 0) {
            v = v0 + i / TW;
            u = u0 + i % TW;
        } else {
            v = v0 + i / (u1 - u0);
            u = u0 + i % (u1 - u0);
        }
    };
    const int npx = NP > 0 ? NP : (v1 - v0) * (u1 - u0);
    double sm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < (NP > 0 ? NP : 1); ++i) {
        for (int ii = i; ii < (NP > 0 ? i + 1 : npx); ++ii) {
            int v, u;
            pix(ii, v, u);
            const double r = NP > 0 ? rr[ii] : ((v < v1 && u < u1) ? img[(long long)v * g.w + u] : INF);
            if (!isfinite(r)) continue;
            double dx, dy, dz;
            ray_dir(A.tg, v, u, dx, dy, dz);
            const double x = r * dx, y = r * dy, z = r * dz;
            sm[0] += y * y; sm[1] += y * z; sm[2] += z * z;
            sm[3] += y;     sm[4] += z;     sm[5] += x * y;
            sm[6] += x * z; sm[7] += x;     sm[8] += 1.0;
        }
    }
    // the chain's start step takes these sums instead of re-folding the tile
    // (stored for every tile with enough points; read only where the verdict passes)
    if (A.start_sums && sm[8] >= 3.0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) A.start_sums[k * A.sums_stride + slot * g.tx + t] = sm[k];
    }
    const bool empty = sm[8] == 0.0;  // no valid pixel: 2, which the chains skip over in bulk
    double a, b, c;
    bool ok = sm[8] >= 3.0 && plane_from_sums(sm, A.cond_limit, a, b, c);
    if (ok) {
        a = f32_round(a);
        b = f32_round(b);
        c = f32_round(c);
        // verdict first (cheap, early exit); certificate statistics only on a pass
#pragma unroll
        for (int i = 0; i < (NP > 0 ? NP : 1); ++i) {
            for (int ii = i; ii < (NP > 0 ? i + 1 : npx) && ok; ++ii) {
                int v, u;
                pix(ii, v, u);
                const double r = NP > 0 ? rr[ii] : ((v < v1 && u < u1) ? img[(long long)v * g.w + u] : INF);
                if (!isfinite(r)) continue;
                double dx, dy, dz;
                ray_dir(A.tg, v, u, dx, dy, dz);
                if (!pixel_fits(r, dx, dy, dz, a, b, c, A.tau, A.r_max)) ok = false;
            }
        }
    }
    *sok = ok ? 1 : (empty ? 2 : 0);
    if (!ok) return;
    double m = 1e300, dmin = 1e300, rmin = 1e300, rmax = 0.0;
    double ylo = 1e300, yhi = -1e300, zlo = 1e300, zhi = -1e300;
#pragma unroll
    for (int i = 0; i < (NP > 0 ? NP : 1); ++i) {
        for (int ii = i; ii < (NP > 0 ? i + 1 : npx); ++ii) {
            int v, u;
            pix(ii, v, u);
            const double r = NP > 0 ? rr[ii] : ((v < v1 && u < u1) ? img[(long long)v * g.w + u] : INF);
            if (!isfinite(r)) continue;
            double dx, dy, dz;
            ray_dir(A.tg, v, u, dx, dy, dz);
            const double den = (dx + a * dy) + b * dz;
            const double r_hat = c / den;
            m = fmin(m, A.tau - fabs(r - r_hat));
            dmin = fmin(dmin, fabs(den));
            rmin = fmin(rmin, r_hat);
            rmax = fmax(rmax, r_hat);
            const double yh = r_hat * dy, zh = r_hat * dz;
            ylo = fmin(ylo, yh);
            yhi = fmax(yhi, yh);
            zlo = fmin(zlo, zh);
            zhi = fmax(zhi, zh);
        }
    }
    float4* ce = A.cert + (slot * g.tx + t) * CERT_F4;
    // one slack field: B < m, B < rmin and B < r_max - rmax are B < min of the three
    cert_store(ce, (float)a, (float)b, (float)c,
               __double2float_rd(fmin(fmin(fmin(m, rmin), A.r_max - rmax), 3.0e38)),
               __double2float_rd(fmin(dmin, 3.0e38)), __double2float_rd(ylo), __double2float_ru(yhi),
               __double2float_rd(zlo), __double2float_ru(zhi));
}

// plane_from_sums (common.cuh; _kernels.py:23-76) for the lanes b0.. that hold
// the running sums (lane b0 + k owns sum k; gl = lane - b0): the six divides
// of the inverse run in parallel, cofactor k in lane b0 + k, and are
// exchanged by shuffles.  Every operation, operand and order is that of
// plane_from_sums, so the bits are identical; all lanes of the warp must call
// it.
__device__ __forceinline__ bool plane_from_sums_lanes(double acc, int b0, int gl, double cond_limit, double& a,
                                                      double& b, double& c)
{
    const double s0 = shfl_d(acc, b0), s1 = shfl_d(acc, b0 + 1), s2 = shfl_d(acc, b0 + 2);
    const double s3 = shfl_d(acc, b0 + 3), s4 = shfl_d(acc, b0 + 4), s5 = shfl_d(acc, b0 + 5);
    const double s6 = shfl_d(acc, b0 + 6), s7 = shfl_d(acc, b0 + 7), s8 = shfl_d(acc, b0 + 8);
    const double m00 = s0, m01 = s1, m02 = -s3, m11 = s2, m12 = -s4, m22 = s8;
    const double r0 = -s5, r1 = -s6, r2 = s7;
    const double c00 = m11 * m22 - m12 * m12;
    const double c01 = m02 * m12 - m01 * m22;
    const double c02 = m01 * m12 - m02 * m11;
    const double det = (m00 * c00 + m01 * c01) + m02 * c02;
    double num;
    if (gl == 0) num = c00;
    else if (gl == 1) num = c01;
    else if (gl == 2) num = c02;
    else if (gl == 3) num = m00 * m22 - m02 * m02;  // c11
    else if (gl == 4) num = m01 * m02 - m00 * m12;  // c12
    else num = m00 * m11 - m01 * m01;               // c22
    const double q = num / det;
    const double i00 = shfl_d(q, b0), i01 = shfl_d(q, b0 + 1), i02 = shfl_d(q, b0 + 2);
    const double i11 = shfl_d(q, b0 + 3), i12 = shfl_d(q, b0 + 4), i22 = shfl_d(q, b0 + 5);
    a = b = c = 0.0;
    if (det == 0.0 || !isfinite(det)) return false;
    const double norm_m = pymax3((fabs(m00) + fabs(m01)) + fabs(m02), (fabs(m01) + fabs(m11)) + fabs(m12),
                                 (fabs(m02) + fabs(m12)) + fabs(m22));
    const double norm_i = pymax3((fabs(i00) + fabs(i01)) + fabs(i02), (fabs(i01) + fabs(i11)) + fabs(i12),
                                 (fabs(i02) + fabs(i12)) + fabs(i22));
    const double cond = norm_m * norm_i;
    if (!isfinite(cond) || cond > cond_limit) return false;
    const double pa = (i00 * r0 + i01 * r1) + i02 * r2;
    const double pb = (i01 * r0 + i11 * r1) + i12 * r2;
    const double pc = (i02 * r0 + i12 * r1) + i22 * r2;
    if (!(isfinite(pa) && isfinite(pb) && isfinite(pc))) return false;
    a = pa;
    b = pb;
    c = pc;
    return true;
}

__device__ __forceinline__ bool solve_round(double acc, double cond_limit, double& a, double& b, double& c)
{
    if (!plane_from_sums_lanes(acc, 0, threadIdx.x & 31, cond_limit, a, b, c)) return false;
    a = f32_round(a);
    b = f32_round(b);
    c = f32_round(c);
    return true;
}

__global__ void __launch_bounds__(FIT_WARPS * 32, 5) fit_rows_kernel(FitArgs A)
{
    __shared__ double smem[FIT_WARPS][32 * 9];
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const long long wid = (long long)blockIdx.x * FIT_WARPS + wib;
    if (wid >= (long long)A.n_jobs * g.ty) return;
    const int job = (int)(wid / g.ty);
    const int tr = (int)(wid % g.ty);
    int frame;
    if (A.mode == 0) {
        frame = job * A.n_frames_group + A.k;
    } else {
        int np = A.n_frames_group - 1;
        int grp = job / np, i = job % np;
        frame = grp * A.n_frames_group + (i < A.k ? i : i + 1);
    }
    const long long slot = (long long)frame * g.ty + tr;
    Chain ch;
    ch.img = A.best + (long long)frame * g.P;
    uint8_t* crow = A.cls + slot * g.tx;
    ch.crow = crow;
    ch.cert = A.cert + slot * g.tx * CERT_F4;
    ch.skip1 = A.mode != 0;
    ch.v0 = tr * g.th;
    ch.rows = min(g.th, g.h - ch.v0);
    const uint8_t run_cls = A.mode == 0 ? 1 : 2;
    double* sm = smem[wib];

    uint16_t* rs = A.run_s + slot * g.tx;
    uint16_t* rl = A.run_len + slot * g.tx;
    float* rabc = A.run_abc + slot * g.tx * 3;
    int n_runs = 0;
    int t = 0;
    Prefetch pf;
    const uint8_t* sok = A.start_ok + slot * g.tx;
    while (t < g.tx) {
        if (sok[t] != 1 || (ch.skip1 && crow[t] == 1)) {
            // residual start tiles (class 0 stays; covered tiles keep class 1):
            // jump to the next start tile with a 32-wide ballot
            int nt = g.tx;
            for (int base = t + 1; base < g.tx; base += 32) {
                const int j = base + lane;
                const uint32_t m = __ballot_sync(STPC_FULL, j < g.tx && sok[j] == 1 && !(ch.skip1 && crow[j] == 1));
                if (m) {
                    nt = base + __ffs(m) - 1;
                    break;
                }
            }
            t = nt;
            continue;
        }
        // passing start: rebuild the running sums and the start plane (the
        // verdict is known; cert[t] may since hold a growth-plane certificate,
        // which remains a valid proof for later union tests)
        double acc = 0.0;
        fold_tile(ch, g, A.tg, t, sm, acc, pf);
        double a, b, c;
        solve_round(acc, A.cond_limit, a, b, c);
        const int s = t;
        int e = t + 1;
        while (e < g.tx) {
            double saved = acc;
            int add = fold_tile(ch, g, A.tg, e, sm, acc, pf);
            if (add == 0) {  // unchanged sums -> same plane -> same verdict
                if (lane == 0) {  // certificate: no pixels, passes under any plane
                    ch.cert[CERT_F4 * e] = make_float4(0.f, 0.f, 0.f, CERT_EMPTY);
                }
                e += 1;
                continue;
            }
            double na, nb, nc;
            bool ok2 = solve_round(acc, A.cond_limit, na, nb, nc);
            if (ok2) ok2 = union_fits(ch, g, A.tg, s, e, na, nb, nc, A.tau, A.r_max);
            if (!ok2) {
                acc = saved;
                break;
            }
            a = na; b = nb; c = nc;
            e += 1;
        }
        if (lane == 0) {
            rs[n_runs] = (uint16_t)s;
            rl[n_runs] = (uint16_t)(e - s);
            rabc[3 * n_runs] = (float)a;
            rabc[3 * n_runs + 1] = (float)b;
            rabc[3 * n_runs + 2] = (float)c;
        }
        for (int tt = s + lane; tt < e; tt += 32)
            if (!(ch.skip1 && crow[tt] == 1)) crow[tt] = run_cls;
        n_runs += 1;
        t = e;
    }
    if (lane == 0) A.n_runs[slot] = n_runs;
}

// ---------------------------------------------------------------------------
// Lock-step variant for tiles of <= 16 pixels (4x4 and smaller): two chains
// per warp, 16 lanes each.  A 4x4 tile's fold and pixel test need exactly 16
// lanes, so pairing chains costs no extra iterations while the solve, the
// control flow and the certificate logic serve two chains per instruction.
// Each iteration advances every live chain by one step of the same state
// machine (scan to the next start tile | fold + solve | test + certificates |
// update); per-chain differences are predicated.
// ---------------------------------------------------------------------------
constexpr int PG = 16;

__device__ __forceinline__ unsigned group_min(unsigned v, int sub, unsigned neutral)
{
    const unsigned r0 = __reduce_min_sync(STPC_FULL, sub == 0 ? v : neutral);
    const unsigned r1 = __reduce_min_sync(STPC_FULL, sub == 1 ? v : neutral);
    return sub ? r1 : r0;
}
__device__ __forceinline__ unsigned group_max(unsigned v, int sub, unsigned neutral)
{
    const unsigned r0 = __reduce_max_sync(STPC_FULL, sub == 0 ? v : neutral);
    const unsigned r1 = __reduce_max_sync(STPC_FULL, sub == 1 ? v : neutral);
    return sub ? r1 : r0;
}

// Pixel test of tile `tile` for every active chain of the warp; on pass the
// group's lane 0 stores the certificate.  Returns this chain's verdict.
// One pixel per lane, so each certificate statistic of a lane is its own
// pixel's value (or the reduction's neutral element): no per-lane min/max and
// no clamping (a passing pixel has 0 < r_hat <= r_max).  The margin, r_hat
// lower bound and r_max headroom share one field, the pixel's slack
// X = min(tau - |r - r_hat|, r_hat, r_max - r_hat): the three tests
// B < m, B < rmin, B < r_max - rmax become B < X.
// `has`: the lane holds a valid pixel (r, direction) of the tile.
__device__ __forceinline__ bool test_px_pair(bool active, bool has, double r, double dx, double dy, double dz,
                                             const Chain& ch, int tile, double a, double b, double c,
                                             double tau, double r_max, double ybias, float4* stage = nullptr)
{
    const int lane = threadIdx.x & 31;
    const int sub = lane >> 4, gl = lane & 15;
    const unsigned gmask = 0xffffu << (sub * 16);
    const unsigned NEUT_MIN = 0xffffffffu, NEUT_MAX = 0u;
    unsigned kx = NEUT_MIN, kd = NEUT_MIN, ky0 = NEUT_MIN, ky1 = NEUT_MAX, kz0 = NEUT_MIN, kz1 = NEUT_MAX;
    bool bad = false;
    {
        if (has) {
            const double den = (dx + a * dy) + b * dz;
            const double ad = fabs(den);
            if (ad < STPC_PARALLEL_EPS) {
                bad = true;
            } else {
                const double r_hat = c / den;
                const double err = fabs(r - r_hat);
                if (r_hat <= 0.0 || r_hat > r_max || err > tau) {
                    bad = true;
                } else {
                    kx = __float_as_uint(__double2float_rd(fmin(fmin(tau - err, r_hat), r_max - r_hat)));
                    kd = __float_as_uint(__double2float_rd(ad));
                    const double yh = r_hat * dy, zh = r_hat * dz;
                    // |yh|, |zh| <= r_max <= ybias / 2: biased, they are positive
                    // floats, whose bit patterns order like their values (no
                    // order-preserving key transform on either side of the REDUX)
                    ky0 = __float_as_uint(__double2float_rd(__dadd_rd(yh, ybias)));
                    ky1 = __float_as_uint(__double2float_ru(__dadd_ru(yh, ybias)));
                    kz0 = __float_as_uint(__double2float_rd(__dadd_rd(zh, ybias)));
                    kz1 = __float_as_uint(__double2float_ru(__dadd_ru(zh, ybias)));
                }
            }
        }
    }
    const bool fail = (__ballot_sync(STPC_FULL, bad) & gmask) != 0;
    if (!__any_sync(STPC_FULL, active && !fail)) return false;
    // X, dmin >= 0: their float bit patterns order like their values
    const unsigned ux = group_min(kx, sub, NEUT_MIN);
    const unsigned ud = group_min(kd, sub, NEUT_MIN);
    ky0 = group_min(ky0, sub, NEUT_MIN);
    ky1 = group_max(ky1, sub, NEUT_MAX);
    kz0 = group_min(kz0, sub, NEUT_MIN);
    kz1 = group_max(kz1, sub, NEUT_MAX);
    const bool pass = active && !fail;
    if (pass && gl == 0) {
        float4* ce = stage ? stage : ch.cert + CERT_F4 * tile;
        // a tile whose pixels are all invalid certifies as empty (no neutral
        // keys leak into the float fields)
        const float xf = ux == NEUT_MIN ? CERT_EMPTY : __uint_as_float(ux);
        const float bf = (float)ybias;  // a power of two: the subtractions are exact
        cert_store(ce, (float)a, (float)b, (float)c, xf, __uint_as_float(ud), __fsub_rd(__uint_as_float(ky0), bf),
                   __fsub_ru(__uint_as_float(ky1), bf), __fsub_rd(__uint_as_float(kz0), bf),
                   __fsub_ru(__uint_as_float(kz1), bf));
    }
    return pass;
}

// Tile shape of the pair kernel: F44 = every tile is a full 4x4 (tile 4x4,
// w and h multiples of 4, e.g. every BASELINE 4x4 config): lane gl's pixel is
// (gl >> 2, gl & 3) with no runtime divide; otherwise the general shape.
template <bool F44>
__device__ __forceinline__ bool tile_px(const Chain& ch, const Geometry& g, int u0, int gl, int& dv, int& du)
{
    if constexpr (F44) {
        dv = gl >> 2;
        du = gl & 3;
        return true;
    } else {
        const int cols = min(g.tw, g.w - u0);
        if (gl >= ch.rows * cols) return false;
        divmod_small(gl, cols, __frcp_rn((float)cols), dv, du);
        return true;
    }
}

// test_px_pair with the lane's pixel of `tile` loaded from global memory.
template <bool F44>
__device__ bool test_tile_pair(bool active, const Chain& ch, const Geometry& g, const Trig& tg, int tile,
                               double a, double b, double c, double tau, double r_max, double ybias)
{
    const int gl = threadIdx.x & 15;
    bool has = false;
    double r = 0.0, dx = 0.0, dy = 0.0, dz = 0.0;
    if (active) {
        const int u0 = tile * g.tw;
        int dv, du;
        if (tile_px<F44>(ch, g, u0, gl, dv, du)) {
            const int v = ch.v0 + dv, u = u0 + du;
            r = ch.img[v * g.w + u];
            if (isfinite(r)) {
                ray_dir(tg, v, u, dx, dy, dz);
                has = true;
            }
        }
    }
    return test_px_pair(active, has, r, dx, dy, dz, ch, tile, a, b, c, tau, r_max, ybias);
}

// plane_from_sums for a half-warp (see plane_from_sums_lanes).
__device__ __forceinline__ bool plane_from_sums_pair(double acc, int sub, int gl, double cond_limit, double& a,
                                                     double& b, double& c)
{
    return plane_from_sums_lanes(acc, sub * PG, gl, cond_limit, a, b, c);
}

// Asynchronous global -> shared copy (cp.async): a prefetch that holds no
// register across the step.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

#ifndef STPC_PAIR_MINB
#define STPC_PAIR_MINB 8  // measured (fit_p): 5 -> 28.5 ms, 6 -> 29.1, 7 -> 26.5, 8 -> 26.3, 10 -> 29.8; re-measured after the slimmer step: 6 -> 22.7, 7 -> 22.1, 8 -> 21.9, 9 -> 22.1
#endif
#ifndef STPC_PAIR44_MINB
#define STPC_PAIR44_MINB 7  // the full-4x4 instantiation (fit_p): 8 -> 19.6-19.9 ms (110 B spilled), 7 -> 19.4 (34 B)
#endif
template <bool F44> constexpr int pair_minb() { return F44 ? STPC_PAIR44_MINB : STPC_PAIR_MINB; }
#ifdef STPC_FIT_STATS
// diagnostic build only (tools/fit_stats.py): chain-step counters
__device__ unsigned long long g_fit_stats[8];
#define FIT_STAT(i, pred)                                                               \
    do {                                                                                \
        const unsigned m_ = __ballot_sync(STPC_FULL, (pred));                          \
        if ((threadIdx.x & 31) == 0 && m_) atomicAdd(&g_fit_stats[i], (unsigned long long)__popc(m_)); \
    } while (0)
extern "C" int stpc_debug_fit_stats(unsigned long long* out)
{
    return cudaMemcpyFromSymbol(out, g_fit_stats, sizeof(g_fit_stats)) == cudaSuccess ? 0 : 1;
}
extern "C" int stpc_debug_fit_stats_reset()
{
    unsigned long long z[8] = {0};
    return cudaMemcpyToSymbol(g_fit_stats, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
#else
#define FIT_STAT(i, pred) ((void)0)
#endif
template <bool F44>
__global__ void __launch_bounds__(FIT_WARPS * 32, pair_minb<F44>()) fit_pair_kernel(FitArgs A)
{
    __shared__ double smem[FIT_WARPS][2][PG * 9];
    __shared__ float4 cstage[FIT_WARPS][2][CERT_F4];  // the growth tile's certificate until the union verdict
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int sub = lane >> 4, gl = lane & 15;
    const unsigned gmask = 0xffffu << (sub * 16);
    const long long n_chains = (long long)A.n_jobs * g.ty;
    const uint8_t run_cls = A.mode == 0 ? 1 : 2;
    double* sm = smem[wib][sub];
    const int kk = gl < 9 ? gl : 8;

    // Work stealing: each half-warp pulls chains from a global counter, so a
    // half whose chain finished early never idles beside a longer partner.
    // Chain state is kept lean (64 registers at 8 blocks per SM): the
    // per-chain arrays are addressed from `slot` on use.
    bool finished = false;  // no chains left for this half
    bool done = true;       // current chain complete
    unsigned sb = 0;        // (frame * ty + tile-row) * tx: the chain's first tile (32-bit: host-checked)
    Chain ch;
    ch.skip1 = A.mode != 0;
    int t = 0, s = 0, n_runs = 0;
    bool grow = false;
    double acc = 0.0;
    float a = 0.f, b = 0.f, c = 0.f;  // the run's plane: f32-exact by construction, kept as floats (3 registers, not 6)
    int pf_t = -1;
    __shared__ double pf_slot[FIT_WARPS * 32];  // the lane's prefetched pixel (cp.async: no register)
    double& pf_s = pf_slot[threadIdx.x];
#ifdef STPC_PAIR_PTRS
    uint8_t* crowp = nullptr;
    const uint8_t* sokp = nullptr;
    float4* certp = nullptr;
#define CROW crowp
#define SOK sokp
#define CERT certp
#else
#define CROW (A.cls + sb)
#define SOK (A.start_ok + sb)
#define CERT (A.cert + (size_t)sb * CERT_F4)
#endif
    auto take_chain = [&](long long cid) {
        if (cid >= n_chains) {
            finished = true;
            done = true;
            return;
        }
        const int job = (int)(cid / g.ty);
        const int tr = (int)(cid % g.ty);
        int frame;
        if (A.mode == 0) {
            frame = job * A.n_frames_group + A.k;
        } else {
            int np = A.n_frames_group - 1;
            int grp = job / np, i = job % np;
            frame = grp * A.n_frames_group + (i < A.k ? i : i + 1);
        }
        const long long slot = (long long)frame * g.ty + tr;
        sb = (unsigned)(slot * g.tx);
#ifdef STPC_PAIR_PTRS
        crowp = A.cls + sb;
        sokp = A.start_ok + sb;
        certp = A.cert + (size_t)sb * CERT_F4;
#endif
        ch.img = A.best + (long long)frame * g.P;
        ch.v0 = tr * g.th;
        ch.rows = min(g.th, g.h - ch.v0);
        t = 0;
        s = 0;
        n_runs = 0;
        grow = false;
        acc = 0.0;
        pf_t = -1;
        done = false;
    };
    {
        long long nc = 0;
        if (gl == 0) nc = (long long)atomicAdd(A.chain_counter, 1u);
        take_chain(__shfl_sync(STPC_FULL, nc, sub * 16));
    }
    // record run [s, e) with the current plane; class its tiles (pass 2 keeps
    // the temporally covered ones)
    auto emit_run = [&](int e_) {
        if (gl == 0) {
            A.run_s[sb + n_runs] = (uint16_t)s;
            A.run_len[sb + n_runs] = (uint16_t)(e_ - s);
            float* rabc = A.run_abc + (size_t)(sb + n_runs) * 3;
            rabc[0] = a;
            rabc[1] = b;
            rabc[2] = c;
        }
        for (int tt = s + gl; tt < e_; tt += PG)
            if (!(ch.skip1 && CROW[tt] == 1)) CROW[tt] = run_cls;
        n_runs += 1;
    };

    while (__any_sync(STPC_FULL, !finished)) {
        // ---- (1) chains between runs jump to their next start tile
        const bool scan = !done && !grow;
        bool jumped = false;
        {
            bool found = false;
            int nt = g.tx;
            int base = t;
            while (__any_sync(STPC_FULL, scan && !found && base < g.tx)) {
                const int j = base + gl;
                // pass 2: a temporally covered tile is never a start (its start
                // verdict may predate the refit that covered it)
                const bool f = scan && !found && j < g.tx && SOK[j] == 1 && !(ch.skip1 && CROW[j] == 1);
                const unsigned mm = (__ballot_sync(STPC_FULL, f) & gmask) >> (sub * 16);
                if (mm && !found) {
                    nt = base + __ffs(mm) - 1;
                    found = true;
                }
                base += PG;
            }
            if (scan) {
                if (found) t = nt;
                else done = true;
                jumped = found;
            }
        }
        // ---- (1a) start: the start verdict already folded the start tile from
        // zero (its sums) and fixed its plane (its certificate's a, b, c are
        // the f32-rounded solve), so the chain takes both and goes on, in
        // this same iteration, to grow into the next tile (a start needs no
        // fold, solve or test of its own; a start iteration of its own was
        // ~21% of the steps)
        if (jumped) {
            const float4 c0 = CERT[CERT_F4 * t];
            a = c0.x;
            b = c0.y;
            c = c0.z;
            s = t;
            grow = true;
            t += 1;
            if (t >= g.tx) {  // a one-tile run at the row end
                emit_run(g.tx);
                grow = false;
                done = true;
                jumped = false;
            }
        }
        FIT_STAT(1, jumped && gl == 0);  // start steps (taken with the next growth step)
        if (jumped) {
            // the start tile's sums, folded from zero by the start verdict
            acc = A.start_sums[kk * A.sums_stride + sb + s];
            // prefetch tile t's pixel for the growth fold below
            const int nu0 = t * g.tw;
            int pv, pu;
            cp_async_wait_all();
            if (tile_px<F44>(ch, g, nu0, gl, pv, pu)) {
                cp_async8(&pf_s, ch.img + ((ch.v0 + pv) * g.w + nu0 + pu));
            } else {
                pf_s = __longlong_as_double(0x7ff0000000000000ll);
            }
            cp_async_commit();
            pf_t = t;
        }
        // ---- (2) fold tile t (every live chain is growing here)
        bool live = !done;
        const double INF = __longlong_as_double(0x7ff0000000000000ll);
        double r = INF;
        int dv = 0, du = 0;
        if (live && tile_px<F44>(ch, g, t * g.tw, gl, dv, du)) {
            if (pf_t == t) {
                cp_async_wait_all();
                r = pf_s;
            } else {
                r = ch.img[(ch.v0 + dv) * g.w + t * g.tw + du];
            }
        }
        int cnt = __popc(__ballot_sync(STPC_FULL, isfinite(r)) & gmask);
        // ---- (2a) a tile without valid pixels (none in the frame -- its start
        // verdict marked it 2 -- or, in pass 2, temporally covered) changes
        // neither the run's sums, plane nor verdict: skip the whole stretch of
        // such tiles at once, certifying them empty, and fold the next tile in
        // this same iteration (an empty growth step of its own was ~18% of the
        // steps)
        const bool emp = live && cnt == 0;
        if (__any_sync(STPC_FULL, emp)) {
            int nt = g.tx;
            bool found = false;
            int base = t + 1;
            while (__any_sync(STPC_FULL, emp && !found && base < g.tx)) {
                const int j = base + gl;
                const bool f = emp && !found && j < g.tx && SOK[j] != 2 && !(ch.skip1 && CROW[j] == 1);
                const unsigned mm = (__ballot_sync(STPC_FULL, f) & gmask) >> (sub * 16);
                if (mm && !found) {
                    nt = base + __ffs(mm) - 1;
                    found = true;
                }
                base += PG;
            }
            if (emp) {
                for (int tt = t + gl; tt < nt; tt += PG)
                    CERT[CERT_F4 * tt] = make_float4(0.f, 0.f, 0.f, CERT_EMPTY);
                t = nt;
                r = INF;
                if (t >= g.tx) {  // the run reaches the row end
                    emit_run(g.tx);
                    grow = false;
                    done = true;
                    live = false;
                } else if (tile_px<F44>(ch, g, t * g.tw, gl, dv, du)) {
                    r = ch.img[(ch.v0 + dv) * g.w + t * g.tw + du];
                }
            }
            cnt = __popc(__ballot_sync(STPC_FULL, isfinite(r)) & gmask);
        }
        double x = 0.0, y = 0.0, z = 0.0, one = 0.0;
        double fr = 0.0, fdx = 0.0, fdy = 0.0, fdz = 0.0;  // the lane's pixel, kept for the tile test
        if (isfinite(r)) {
            double dx, dy, dz;
            ray_dir(A.tg, ch.v0 + dv, t * g.tw + du, dx, dy, dz);
            x = r * dx;
            y = r * dy;
            z = r * dz;
            one = 1.0;
            fr = r;
            fdx = dx;
            fdy = dy;
            fdz = dz;
        }
        double* row = sm + gl * 9;
        row[0] = y * y;
        row[1] = y * z;
        row[2] = z * z;
        row[3] = y;
        row[4] = z;
        row[5] = x * y;
        row[6] = x * z;
        row[7] = x;
        row[8] = one;
        __syncwarp();
        if (live) {
#pragma unroll
            for (int j = 0; j < PG; ++j) acc += sm[j * 9 + kk];  // zeros beyond npx: exact
        }
        __syncwarp();
        // the lane's pixel stays in its own transpose row for this step's tile test
        row[0] = fr;
        row[1] = fdx;
        row[2] = fdy;
        row[3] = fdz;
        // prefetch the next tile's pixel gl
        if (live && t + 1 < g.tx) {
            const int nu0 = (t + 1) * g.tw;
            cp_async_wait_all();  // an unconsumed earlier copy into the slot has landed
            if (tile_px<F44>(ch, g, nu0, gl, dv, du)) {
                cp_async8(&pf_s, ch.img + ((ch.v0 + dv) * g.w + nu0 + du));
            } else {
                pf_s = __longlong_as_double(0x7ff0000000000000ll);
            }
            cp_async_commit();
            pf_t = t + 1;
        }
        // ---- (3) solve: starts (verdict known ok) and growing chains with new pixels
        FIT_STAT(0, live && gl == 0);                      // chain steps
        FIT_STAT(2, live && grow && cnt == 0 && gl == 0);  // empty growth steps
        const bool need = live && (!grow || cnt > 0);
        // the new plane, f32-rounded (_kernels.py:196-198): held as floats and
        // widened (exactly) where the fp64 tests use it
        float naf = 0.f, nbf = 0.f, ncf = 0.f;
        bool ok = false;
        {
            double pa, pb, pc;
            const bool solved = plane_from_sums_pair(acc, sub, gl, A.cond_limit, pa, pb, pc);
            if (need && solved) {
                naf = __double2float_rn(pa);
                nbf = __double2float_rn(pb);
                ncf = __double2float_rn(pc);
                ok = true;
            }
        }
        // ---- (4) growing chains: test tile t, then certificates of [s, t)
        const bool testing = live && grow && cnt > 0 && ok;
        bool pass = false;
        if (__any_sync(STPC_FULL, testing)) {
            ch.cert = CERT;
            // the first certificate batch of [s, t) does not depend on the new
            // tile's verdict: its loads and checks are issued before the pixel
            // test so the two latency chains overlap
            const bool weak0 = testing && s + gl < t && !cert_holds_f(ch.cert, s + gl, naf, nbf, ncf);
            // the new tile's certificate is staged and stored only if the
            // whole union passes: a failed growth leaves tile t's start
            // certificate (whose plane (1a) takes as the start plane) intact
            pass = test_px_pair(testing, testing && one != 0.0, row[0], row[1], row[2], row[3], ch, t, (double)naf,
                                (double)nbf, (double)ncf,
                                A.tau, A.r_max, A.ybias, cstage[wib][sub]);
            FIT_STAT(5, testing && gl == 0);        // growth tests
            FIT_STAT(6, testing && pass && gl == 0);  // growth tests passed (new tile)
            int base = s;
            while (__any_sync(STPC_FULL, pass && base < t)) {
                const int j = base + gl;
                const bool weak =
                    pass && j < t && (base == s ? weak0 : !cert_holds_f(ch.cert, j, naf, nbf, ncf));
                FIT_STAT(3, pass && j < t);  // certificate checks
                FIT_STAT(4, weak);           // weak certificates -> full re-test
                unsigned wm = (__ballot_sync(STPC_FULL, weak) & gmask) >> (sub * 16);
                while (__any_sync(STPC_FULL, pass && wm != 0)) {
                    const bool act = pass && wm != 0;
                    const int jj = act ? base + __ffs(wm) - 1 : 0;
                    if (act) wm &= wm - 1;
                    const bool r = test_tile_pair<F44>(act, ch, g, A.tg, jj, (double)naf, (double)nbf, (double)ncf, A.tau,
                                                       A.r_max, A.ybias);
                    FIT_STAT(7, act && !r && gl == 0);  // re-tests that fail the union
                    if (act && !r) pass = false;
                }
                base += PG;
            }
            __syncwarp();
            if (pass && gl < CERT_F4) CERT[CERT_F4 * t + gl] = cstage[wib][sub][gl];
        }
        // ---- (5) state update (uniform within each chain's 16 lanes)
        if (!done) {  // every live chain is growing here (starts are taken in (1a))
            int emit_e = -1;
            if (cnt == 0) {
                if (gl == 0) CERT[CERT_F4 * t] = make_float4(0.f, 0.f, 0.f, CERT_EMPTY);
                t += 1;
            } else if (pass) {
                a = naf; b = nbf; c = ncf;
                t += 1;
            } else {
                emit_e = t;  // close [s, t); t becomes a start candidate again
                grow = false;
            }
            if (t >= g.tx) {
                if (grow) {
                    emit_e = g.tx;
                    grow = false;
                }
                done = true;
            }
            if (emit_e >= 0) emit_run(emit_e);
        }
        // ---- (6) hand-over: a finished chain records its run count and its
        // half-warp steals the next chain
        const bool handover = done && !finished;
        if (handover && gl == 0) A.n_runs[sb / g.tx] = n_runs;
        if (__any_sync(STPC_FULL, handover)) {
            long long nc = 0;
            if (handover && gl == 0) nc = (long long)atomicAdd(A.chain_counter, 1u);
            nc = __shfl_sync(STPC_FULL, nc, sub * 16);
            if (handover) take_chain(nc);
        }
    }
#undef CROW
#undef SOK
#undef CERT
}

void launch_start_tiles(const FitArgs& a, cudaStream_t s)
{
    long long tiles = (long long)a.n_jobs * a.g.ty * a.g.tx;
    if (tiles <= 0) return;
    STPC_LAUNCH();
    const long long chains = (long long)a.n_jobs * a.g.ty;
    const long long bpc = (a.g.tx + START_TPB - 1) / START_TPB;
    if (a.g.tw == 4 && a.g.th <= 4) {
        start_tiles_staged_kernel<4><<<(unsigned)(chains * bpc), START_TPB, 0, s>>>(a);
    } else if (a.g.tw == 2 && a.g.th <= 8) {
        start_tiles_staged_kernel<2><<<(unsigned)(chains * bpc), START_TPB, 0, s>>>(a);
    } else {
        start_tiles_kernel<0, 0><<<(unsigned)((tiles + 255) / 256), 256, 0, s>>>(a);
    }
}

static bool pair_full44(const Geometry& g) { return g.tw == 4 && g.th == 4 && g.w % 4 == 0 && g.h % 4 == 0; }

void launch_fit_chains(const FitArgs& a, cudaStream_t s)
{
    long long warps = (long long)a.n_jobs * a.g.ty;
    if (warps <= 0) return;
    STPC_LAUNCH();
    if (a.g.tw * a.g.th <= PG) {
        // work-stealing grid: STPC_PAIR_MINB resident blocks per SM, capped by the chain count
        long long pairs = (warps + 1) / 2;
        const bool f44 = pair_full44(a.g);
        long long blocks = std::min<long long>((pairs + FIT_WARPS - 1) / FIT_WARPS,
                                               148LL * (f44 ? STPC_PAIR44_MINB : STPC_PAIR_MINB));
        launch_zero(a.chain_counter, sizeof(unsigned), s);
        if (f44)
            fit_pair_kernel<true><<<(unsigned)blocks, FIT_WARPS * 32, 0, s>>>(a);
        else
            fit_pair_kernel<false><<<(unsigned)blocks, FIT_WARPS * 32, 0, s>>>(a);
    } else {
        fit_rows_kernel<<<(unsigned)((warps + FIT_WARPS - 1) / FIT_WARPS), FIT_WARPS * 32, 0, s>>>(a);
    }
}

// Does running the P-frame start verdicts beside the key-frame fit pay?
// Measured (frames/s, overlapped vs serial): configs[3] 1024 groups 145.2k vs
// 143.4k (16 k key chains: the fit's last wave leaves slots idle) and
// configs[2] with 16x16 tiles 36.5k vs 33.2k (fit_rows: one warp per chain
// leaves SMs idle) win; with fewer key chains than the pair kernel's resident
// slots the verdicts' blocks slow the latency-bound chains, which stay the
// critical path: configs[1] 102.6k vs 106.1k, configs[2] 4x4 26.3k vs 27.3k.
bool fit_overlap_pays(const Geometry& g, long long key_chains)
{
    if (g.tw * g.th > PG) return true;
    return key_chains > 148LL * (pair_full44(g) ? STPC_PAIR44_MINB : STPC_PAIR_MINB) * FIT_WARPS * 2;
}

void launch_fit_rows(const FitArgs& a, cudaStream_t s)
{
    launch_start_tiles(a, s);
    launch_fit_chains(a, s);
}

// K3a: the temporal offset refit (refit_kernel below) and a second tiny
// kernel that sizes each key chain's temporal records (18 B + presence bits +
// 4 B per present P channel, bitstream.py:222-245).
#ifndef STPC_REFIT_MINB
#define STPC_REFIT_MINB 10  // measured: unbounded 5.74 ms, 10 -> 5.66, 16 -> 5.65 (latency-bound; more warps beat a few spills)
#endif
// One run's span [U0, U0 + U) x rows of one P channel, full warp: c' = f32
// of the v-major ordered mean of r (d . n) over the valid pixels, then the
// span re-test (refit_spans, _kernels.py:231-279).  Returns ok, sets c.
__device__ __forceinline__ bool refit_span(const RefitArgs& A, const double* img, double* sm, int v0, int rows,
                                           int U0, int U, double a, double b, double& c)
{
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const int npx = rows * U;
    const float ru = __frcp_rn((float)U);
    double acc = 0.0;
    int cnt = 0;
    for (int base = 0; base < npx; base += 32) {
        int p = base + lane;
        double prod = 0.0;
        bool valid = false;
        if (p < npx) {
            int dv, du;
            divmod_small(p, U, ru, dv, du);
            int v = v0 + dv, u = U0 + du;
            double r = img[(long long)v * g.w + u];
            if (isfinite(r)) {
                double dx, dy, dz;
                ray_dir(A.tg, v, u, dx, dy, dz);
                double den = (dx + a * dy) + b * dz;
                prod = r * den;
                valid = true;
            }
        }
        cnt += __popc(__ballot_sync(STPC_FULL, valid));
        sm[lane] = prod;  // +0.0 for invalid pixels: exact (see fit_rows)
        __syncwarp();
        // lanes past the span hold +0.0, so a fixed-length unrolled fold
        // is exact; a one-tile span (16 pixels of 4x4) adds 16 terms
        if (npx - base > 16) {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) acc += sm[jj];
        } else {
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) acc += sm[jj];
        }
        __syncwarp();
    }
    c = 0.0;
    if (cnt == 0) return false;
    c = f32_round(acc / (double)cnt);
    bool ok = true;
    for (int base = 0; base < npx && ok; base += 32) {
        int p = base + lane;
        bool bad = false;
        if (p < npx) {
            int dv, du;
            divmod_small(p, U, ru, dv, du);
            int v = v0 + dv, u = U0 + du;
            double r = img[(long long)v * g.w + u];
            if (isfinite(r)) {
                double dx, dy, dz;
                ray_dir(A.tg, v, u, dx, dy, dz);
                bad = !pixel_fits(r, dx, dy, dz, a, b, c, A.tau, A.r_max);
            }
        }
        ok = !__any_sync(STPC_FULL, bad);
    }
    return ok;
}

// Spans of at most 16 pixels (one 4x4 tile), two channels at once: half h of
// the warp refits channel h of the pair with the same arithmetic and order.
__device__ __forceinline__ bool refit_span_pair(const RefitArgs& A, const double* img, double* sm, int v0, int U0,
                                                int U, int npx, double a, double b, double& c)
{
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    const unsigned hmask = 0xffffu << (half * 16);
    double r = 0.0, dx = 0.0, dy = 0.0, dz = 0.0, prod = 0.0;
    bool valid = false;
    if (hl < npx) {
        int dv, du;
        divmod_small(hl, U, __frcp_rn((float)U), dv, du);
        const int v = v0 + dv, u = U0 + du;
        r = img[(long long)v * g.w + u];
        if (isfinite(r)) {
            ray_dir(A.tg, v, u, dx, dy, dz);
            prod = r * ((dx + a * dy) + b * dz);
            valid = true;
        }
    }
    const int cnt = __popc(__ballot_sync(STPC_FULL, valid) & hmask);
    sm[lane] = prod;
    __syncwarp();
    double acc = 0.0;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) acc += sm[half * 16 + jj];  // +0.0 past the span: exact
    __syncwarp();
    c = cnt > 0 ? f32_round(acc / (double)cnt) : 0.0;
    const bool bad = valid && !pixel_fits(r, dx, dy, dz, a, b, c, A.tau, A.r_max);
    const unsigned bm = __ballot_sync(STPC_FULL, bad);  // every lane votes (no short-circuit)
    return cnt > 0 && (bm & hmask) == 0;
}

// K3a: one warp per (key-frame chain, pair of P channels); for each run of the
// chain, c' = f32(mean over the channel's valid span pixels of r * (d . n)),
// folded v-major over the whole span in the reference's order, then the span
// re-test with (a, b, c').  One-tile spans refit both channels of the pair at
// once (half a warp each); longer spans take the full warp per channel.
// Spans that pass mark their tiles class 1 in the channel and poison the
// channel's pixels there (+inf) for pass 2.
__global__ void __launch_bounds__(128, STPC_REFIT_MINB) refit_kernel(RefitArgs A)
{
    __shared__ double smem[4][32];
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31, half = lane >> 4;
    double* sm = smem[threadIdx.x >> 5];
    const int np = A.n - 1;
    // pairs of channels only where one-tile spans fit half a warp; larger
    // tiles keep one warp per channel (twice the warps in flight)
    const int per = g.tw * g.th <= 16 ? 2 : 1;
    const int npairs = (np + per - 1) / per;
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (np < 1 || wid >= (long long)A.n_groups * g.ty * npairs) return;
    const long long kc = wid / npairs;  // key chain
    const int q = (int)(wid % npairs);
    const int np_here = min(per, np - per * q);  // channels of this warp
    const int grp = (int)(kc / g.ty);
    const int tr = (int)(kc % g.ty);
    const long long kslot = ((long long)grp * A.n + A.k) * g.ty + tr;
    const int nr = A.n_runs[kslot];
    const int v0 = tr * g.th;
    const int rows = min(g.th, g.h - v0);
    int chn[2];
    for (int h = 0; h < 2; ++h) {
        const int pi = min(per * q + h, np - 1);
        chn[h] = pi < A.k ? pi : pi + 1;
    }
    for (int j = 0; j < nr; ++j) {
        const long long ri = kslot * g.tx + j;
        const int s = A.run_s[ri], len = A.run_len[ri];
        const double a = (double)A.run_abc[3 * ri], b = (double)A.run_abc[3 * ri + 1];
        const int U0 = s * g.tw;
        const int U = min((s + len) * g.tw, g.w) - U0;
        const int npx = rows * U;
        const long long rj = (kc * g.tx + j) * A.n;
        if (lane == 0 && q == 0) A.ref_ok[rj + A.k] = 1;
        bool ok[2] = {false, false};
        double cc[2] = {0.0, 0.0};
        if (npx <= 16 && np_here == 2) {
            const int frame = grp * A.n + chn[half];
            double c;
            const bool okh = refit_span_pair(A, A.best + (long long)frame * g.P, sm, v0, U0, U, npx, a, b, c);
            ok[0] = __shfl_sync(STPC_FULL, okh, 0);
            ok[1] = __shfl_sync(STPC_FULL, okh, 16);
            cc[0] = __shfl_sync(STPC_FULL, c, 0);
            cc[1] = __shfl_sync(STPC_FULL, c, 16);
        } else {
            for (int h = 0; h < np_here; ++h) {
                const int frame = grp * A.n + chn[h];
                ok[h] = refit_span(A, A.best + (long long)frame * g.P, sm, v0, rows, U0, U, a, b, cc[h]);
            }
        }
        for (int h = 0; h < np_here; ++h) {
            const int frame = grp * A.n + chn[h];
            if (lane == 0) {
                A.ref_ok[rj + chn[h]] = ok[h];
                A.ref_c[rj + chn[h]] = (float)cc[h];
            }
            if (ok[h]) {
                uint8_t* crow = A.cls + ((long long)frame * g.ty + tr) * g.tx;
                double* img = A.best + (long long)frame * g.P;
                for (int tt = s + lane; tt < s + len; tt += 32) crow[tt] = 1;
                const float ru = __frcp_rn((float)U);
                for (int p = lane; p < npx; p += 32) {
                    int dv, du;
                    divmod_small(p, U, ru, dv, du);
                    img[(long long)(v0 + dv) * g.w + U0 + du] = __longlong_as_double(0x7ff0000000000000ll);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K3a, channel-batched (the product path; refit_kernel above is the
// -DSTPC_REFIT_V1 A/B baseline).  One warp per (key chain, slice of its runs)
// refits a run against ALL P channels at once: a lane owns a pixel position of
// the span, and the ray, the denominator (dx + a dy) + b dz and the pixel
// index are the same for every channel, so they are computed once per pixel
// and each channel costs one load and one product.  The ordered fold, which a
// warp can only do with every lane repeating the same sequential adds, now
// serves up to RF_CB channels per instruction: lane c folds channel c's terms
// from shared memory (the same v-major order and +0.0 padding as refit_span).
// Two consecutive one-tile runs (<= 16 pixels each) are taken side by side,
// one per half-warp.  Arithmetic and order per (run, channel) are
// refit_spans' (_kernels.py:231-279), so the bits are the per-channel
// kernel's.
// ---------------------------------------------------------------------------
#ifndef STPC_REFIT2_MINB
#define STPC_REFIT2_MINB 6  // measured (refit, split 1): 5 -> 3.46 ms, 6 -> 3.12-3.18, 7 -> 3.36, 8 -> 3.22-3.61
#endif
#ifndef STPC_REFIT_SPLIT_MIN
#define STPC_REFIT_SPLIT_MIN 1  // measured at 16 k key chains: split 1 -> 3.12 ms, 2 -> 3.44, 4 -> 4.3
#endif
#ifndef STPC_REFIT2_WPB
#define STPC_REFIT2_WPB 2  // warps per block (a block's slot is held until its slowest warp ends); measured 1 -> 3.18 ms, 2 -> 3.12, 4 -> 3.17
#endif
constexpr int RF_WPB = STPC_REFIT2_WPB;
constexpr long long REFIT_TARGET_WARPS = 148LL * STPC_REFIT2_MINB * 4 * 4;  // four waves of resident warps
constexpr int RF_CB = 8;    // P channels per pass (n - 1 <= 8: one pass)
constexpr int RF_ROW = 33;  // 32 terms per channel + 1 of padding (conflict-free folds)

__global__ void __launch_bounds__(32 * RF_WPB, STPC_REFIT2_MINB * 4 / RF_WPB) refit_all_kernel(RefitArgs A, int split)
{
    __shared__ double smem[RF_WPB][RF_CB * RF_ROW];
    __shared__ double s_pf[RF_WPB][2][RF_CB * 32];  // the lanes' prefetched pixels, two visits deep: [buffer][channel][lane]
    __shared__ double s_cc[RF_WPB][2 * RF_CB];
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    const int wib = threadIdx.x >> 5;
    double* sm = smem[wib];
    double* scc = s_cc[wib];
    double* pf = &s_pf[wib][0][lane];  // buffer b, channel ch: pf[b * RF_CB * 32 + ch * 32]
    const int np = A.n - 1;
    const long long wid = (long long)blockIdx.x * RF_WPB + wib;
    if (np < 1 || wid >= (long long)A.n_groups * g.ty * split) return;
    const long long kc = wid / split;  // key chain
    const int q = (int)(wid % split);
    const int grp = (int)(kc / g.ty);
    const int tr = (int)(kc % g.ty);
    const long long kslot = ((long long)grp * A.n + A.k) * g.ty + tr;
    const int nr = A.n_runs[kslot];
    const int j0 = (int)((long long)nr * q / split), j1 = (int)((long long)nr * (q + 1) / split);
    if (j0 >= j1) return;
    const int v0 = tr * g.th;
    const int rows = min(g.th, g.h - v0);
    const int P = (int)g.P;  // pixel indices are ints (host-checked: n * P < 2^31)
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    double* gbase = A.best + (long long)grp * A.n * g.P;  // the group's frames
#define RF_CHN(pi) ((pi) < A.k ? (pi) : (pi) + 1)
    // pointer step from P channel pi to pi + 1 (the key frame lies between k - 1 and k)
#define RF_STEP(pi) ((pi) + 1 == A.k ? 2 * P : P)
    auto load_run = [&](int jr, int& s_, int& len_, float& af_, float& bf_) {
        const long long ri = kslot * g.tx + min(jr, j1 - 1);
        s_ = A.run_s[ri];
        len_ = A.run_len[ri];
        af_ = A.run_abc[3 * ri];
        bf_ = A.run_abc[3 * ri + 1];
    };
    auto span_px = [&](int s_, int len_) { return rows * (min((s_ + len_) * g.tw, g.w) - s_ * g.tw); };
    // pixel index of position p of run (s_, len_)'s span in v-major order; -1 past the span
    auto px_index = [&](int s_, int len_, int p) -> int {
        const int U0 = s_ * g.tw;
        const int U = min((s_ + len_) * g.tw, g.w) - U0;
        if (p >= rows * U) return -1;
        int dv, du;
        divmod_small(p, U, __frcp_rn((float)U), dv, du);
        return (v0 + dv) * g.w + U0 + du;
    };
    for (int cb = 0; cb < np; cb += RF_CB) {
        const int nch = min(RF_CB, np - cb);
        double* const img0 = gbase + (long long)RF_CHN(cb) * P;  // the pass's first channel
        // Visits of chunks alternate between the two prefetch buffers: a visit
        // first issues the copies of the next visit in the stream (the next
        // chunk, the re-test's first chunk of a long span, or the next run's
        // first chunk) into the other buffer, then works on its own, so a
        // visit's DRAM latency hides behind the previous visit's arithmetic.
        int vb = 0;
        auto pf_issue = [&](int idx, int buf) {
            if (idx >= 0) {
                double* d = pf + buf * (RF_CB * 32);
                const double* src = img0 + idx;
#pragma unroll 1
                for (int ch = 0; ch < nch; ++ch) {
                    cp_async8(d, src);
                    d += 32;
                    src += RF_STEP(cb + ch);
                }
            }
            cp_async_commit();
        };
        int j = j0;
        // candidates: half 0 holds run j, half 1 run j + 1 (cs..), and runs
        // j + 2, j + 3 behind them (ns..), loaded an iteration ahead
        int cs, clen, ns, nlen;
        float caf, cbf, naf, nbf;
        load_run(j + half, cs, clen, caf, cbf);
        load_run(j + 2 + half, ns, nlen, naf, nbf);
        {
            const bool pr = __all_sync(STPC_FULL, span_px(cs, clen) <= 16) && j + 1 < j1;
            const int s0 = pr ? cs : __shfl_sync(STPC_FULL, cs, 0);
            const int l0 = pr ? clen : __shfl_sync(STPC_FULL, clen, 0);
            pf_issue(px_index(s0, l0, pr ? hl : lane), vb);
        }
        while (j < j1) {
            // two one-tile runs side by side (one per half-warp), else run j alone
            const bool paired = __all_sync(STPC_FULL, span_px(cs, clen) <= 16) && j + 1 < j1;
            int s = cs, len = clen;
            float af = caf, bf = cbf;
            if (!paired) {
                s = __shfl_sync(STPC_FULL, s, 0);
                len = __shfl_sync(STPC_FULL, len, 0);
                af = __shfl_sync(STPC_FULL, af, 0);
                bf = __shfl_sync(STPC_FULL, bf, 0);
            }
            const int U0 = s * g.tw;
            const int U = min((s + len) * g.tw, g.w) - U0;
            const int npx = rows * U;
            const int gw = paired ? 16 : 32;    // lanes per run
            const int gl = paired ? hl : lane;  // lane within the run's group
            const int gsh = paired ? half : 0;  // group index
            const unsigned gmask = paired ? 0xffffu << (half * 16) : STPC_FULL;
            const double a = (double)af, b = (double)bf;
            const float ru = __frcp_rn((float)U);
            const long long rj = (kc * g.tx + (paired ? j + half : j)) * A.n;
            if (cb == 0 && gl == 0) A.ref_ok[rj + A.k] = 1;
            const int nchunks = paired ? 1 : (npx + 31) >> 5;

            // the next iteration's candidates and the lane's first pixel there
            const int jn = j + (paired ? 2 : 1);
            if (paired) {
                cs = ns; clen = nlen; caf = naf; cbf = nbf;
            } else {
                const int t_s = __shfl_sync(STPC_FULL, cs, 16), t_l = __shfl_sync(STPC_FULL, clen, 16);
                const float t_a = __shfl_sync(STPC_FULL, caf, 16), t_b = __shfl_sync(STPC_FULL, cbf, 16);
                const int u_s = __shfl_sync(STPC_FULL, ns, 0), u_l = __shfl_sync(STPC_FULL, nlen, 0);
                const float u_a = __shfl_sync(STPC_FULL, naf, 0), u_b = __shfl_sync(STPC_FULL, nbf, 0);
                cs = half ? u_s : t_s;
                clen = half ? u_l : t_l;
                caf = half ? u_a : t_a;
                cbf = half ? u_b : t_b;
            }
            load_run(jn + 2 + half, ns, nlen, naf, nbf);
            int nidx0 = -1;
            if (jn < j1) {
                const bool pr = __all_sync(STPC_FULL, span_px(cs, clen) <= 16) && jn + 1 < j1;
                const int s0 = pr ? cs : __shfl_sync(STPC_FULL, cs, 0);
                const int l0 = pr ? clen : __shfl_sync(STPC_FULL, clen, 0);
                nidx0 = px_index(s0, l0, pr ? hl : lane);
            }

            // the lane's pixel of chunk ck: index and denominator (dx + a dy) + b dz
            auto pixel = [&](int ck, int& idx, double& den) {
                const int p = ck * 32 + gl;
                idx = -1;
                den = 0.0;
                if (p < npx) {
                    int dv, du;
                    divmod_small(p, U, ru, dv, du);
                    const int v = v0 + dv, u = U0 + du;
                    double dx, dy, dz;
                    ray_dir(A.tg, v, u, dx, dy, dz);
                    den = (dx + a * dy) + b * dz;
                    idx = v * g.w + u;
                }
            };

            // ---- pass 1: the channels' ordered sums of r * (d . n)
            double acc = 0.0;
            int mycnt = 0;
            int idx0 = -1;
            double den0 = 0.0;
#pragma unroll 1
            for (int ck = 0; ck < nchunks; ++ck) {
                int idx;
                double den;
                pixel(ck, idx, den);
                if (ck == 0) {
                    idx0 = idx;
                    den0 = den;
                }
                // the next visit: next chunk | the re-test's first chunk | the next run
                pf_issue(ck + 1 < nchunks ? px_index(s, len, ck * 32 + 32 + gl) : nchunks > 1 ? idx0 : nidx0, vb ^ 1);
                asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // this visit's copies have landed
                const double* rp = pf + vb * (RF_CB * 32);
#pragma unroll 1
                for (int ch = 0; ch < nch; ++ch) {
                    double prod = 0.0;  // +0.0 for invalid pixels and lanes past the span: exact
                    bool valid = false;
                    if (idx >= 0) {
                        const double r = rp[ch * 32];
                        if (isfinite(r)) {
                            prod = r * den;
                            valid = true;
                        }
                    }
                    const unsigned bm = __ballot_sync(STPC_FULL, valid) & gmask;
                    if (gl == ch) mycnt += __popc(bm);
                    sm[ch * RF_ROW + lane] = prod;
                }
                __syncwarp();
                if (gl < nch) {  // lane c of the group folds channel c
                    const double* row = sm + gl * RF_ROW + (paired ? half * 16 : 0);
                    const int nf = (paired || npx - ck * 32 <= 16) ? 16 : 32;
#pragma unroll 8
                    for (int jj = 0; jj < nf; ++jj) acc += row[jj];
                }
                __syncwarp();
                vb ^= 1;
            }
            double cme = 0.0;
            if (gl < nch) {
                if (mycnt > 0) cme = f32_round(acc / (double)mycnt);
                scc[gsh * RF_CB + gl] = cme;
            }
            __syncwarp();

            // ---- pass 2: the span re-test with (a, b, c') per channel.  A
            // one-chunk span re-reads its pass-1 buffer; a longer span streams
            // its chunks through the buffers again.
            unsigned failed = 0;  // bit ch: channel ch failed (uniform within the group)
            const int rb = nchunks == 1 ? vb ^ 1 : vb;  // pass 1 left vb at the next visit's buffer
#pragma unroll 1
            for (int ck = 0; ck < nchunks; ++ck) {
                int idx = idx0;
                double den = den0;
                if (ck > 0) pixel(ck, idx, den);
                int cur = rb;
                if (nchunks > 1) {
                    pf_issue(ck + 1 < nchunks ? px_index(s, len, ck * 32 + 32 + gl) : nidx0, vb ^ 1);
                    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
                    cur = vb;
                    vb ^= 1;
                }
                const double* rp = pf + cur * (RF_CB * 32);
                const bool par = fabs(den) < STPC_PARALLEL_EPS;
                unsigned bad = 0;
                if (idx >= 0) {
#pragma unroll 1
                    for (int ch = 0; ch < nch; ++ch) {
                        if ((failed >> ch) & 1) continue;
                        const double r = rp[ch * 32];
                        if (isfinite(r)) {
                            bool fits = !par;
                            if (fits) {
                                const double r_hat = scc[gsh * RF_CB + ch] / den;
                                fits = !(r_hat <= 0.0 || r_hat > A.r_max) && !(fabs(r - r_hat) > A.tau);
                            }
                            if (!fits) bad |= 1u << ch;
                        }
                    }
                }
                const unsigned red = __reduce_or_sync(STPC_FULL, bad << (gsh * RF_CB));
                failed |= (red >> (gsh * RF_CB)) & 0xffu;
                if (!paired && failed == (1u << nch) - 1u && ck + 1 < nchunks) {
                    // uniform: every channel failed; the copies in flight are
                    // this run's next chunk: replace them with the next run's
                    cp_async_wait_all();
                    pf_issue(nidx0, vb);
                    break;
                }
            }

            // ---- results, classes and poisoning
            bool okc = false;
            if (gl < nch) {
                okc = mycnt > 0 && !((failed >> gl) & 1);
                const int chn = RF_CHN(cb + gl);
                A.ref_ok[rj + chn] = okc;
                A.ref_c[rj + chn] = (float)cme;
            }
            const unsigned okb = __ballot_sync(STPC_FULL, okc);
            const unsigned okmask = (okb >> (gsh * 16)) & 0xffu;
            if (okmask) {
                uint8_t* crow = A.cls + (((long long)grp * A.n + RF_CHN(cb)) * g.ty + tr) * g.tx;
#pragma unroll 1
                for (int ch = 0; ch < nch; ++ch) {
                    if ((okmask >> ch) & 1)
                        for (int tt = s + gl; tt < s + len; tt += gw) crow[tt] = 1;
                    crow += (long long)(RF_STEP(cb + ch) / P) * g.ty * g.tx;
                }
#pragma unroll 1
                for (int ck = 0; ck < nchunks; ++ck) {
                    const int idx = ck == 0 ? idx0 : px_index(s, len, ck * 32 + gl);
                    if (idx >= 0) {
                        double* dst = img0 + idx;
#pragma unroll 1
                        for (int ch = 0; ch < nch; ++ch) {
                            if ((okmask >> ch) & 1) *dst = INF;
                            dst += RF_STEP(cb + ch);
                        }
                    }
                }
            }
            j = jn;
        }
        cp_async_wait_all();
    }
#undef RF_CHN
#undef RF_STEP
}

// temporal record bytes per key chain: lanes over runs, popcount of present P channels
__global__ void __launch_bounds__(128) record_bytes_kernel(RefitArgs A)
{
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const long long kc = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (kc >= (long long)A.n_groups * g.ty) return;
    const int grp = (int)(kc / g.ty), tr = (int)(kc % g.ty);
    const long long kslot = ((long long)grp * A.n + A.k) * g.ty + tr;
    const int nr = A.n_runs[kslot];
    const int pm = (A.n + 7) / 8;
    long long tb = 0;
    for (int j = lane; j < nr; j += 32) {
        const uint8_t* okv = A.ref_ok + (kc * g.tx + j) * A.n;
        int present = 0;
        for (int c = 0; c < A.n; ++c) present += (c != A.k) && okv[c];
        tb += 18 + pm + 4 * present;
        if (A.n == 1) A.ref_ok[(kc * g.tx + j) * A.n + A.k] = 1;
    }
    for (int o = 16; o > 0; o >>= 1) tb += __shfl_xor_sync(STPC_FULL, tb, o);
    if (lane == 0) A.chain_tbytes[kc] = tb;
}

void launch_refit(const RefitArgs& a, cudaStream_t s)
{
    long long kchains = (long long)a.n_groups * a.g.ty;
    if (kchains <= 0) return;
#ifdef STPC_REFIT_V1
    const int per = a.g.tw * a.g.th <= 16 ? 2 : 1;  // P channels per warp (refit_kernel)
    long long warps = kchains * ((a.n - 1 + per - 1) / per);
    if (warps > 0) {
        STPC_LAUNCH();
        refit_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(a);
    }
#else
    if (a.n > 1) {
        // warps per key chain (contiguous slices of its runs): enough warps to
        // fill the machine a few times over when the batch has few chains
        static const int forced = getenv("STPC_REFIT_SPLIT") ? atoi(getenv("STPC_REFIT_SPLIT")) : 0;
        int split = forced > 0 ? forced : (int)std::min<long long>(32, std::max<long long>(STPC_REFIT_SPLIT_MIN, (REFIT_TARGET_WARPS + kchains - 1) / kchains));
        const long long warps = kchains * split;
        STPC_LAUNCH();
        refit_all_kernel<<<(unsigned)((warps + RF_WPB - 1) / RF_WPB), 32 * RF_WPB, 0, s>>>(a, split);
    }
#endif
    STPC_LAUNCH();
    record_bytes_kernel<<<(unsigned)((kchains + 3) / 4), 128, 0, s>>>(a);
}

}  // namespace stpc
