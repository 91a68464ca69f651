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

namespace stpc {

constexpr int FIT_WARPS = 4;  // warps per block

struct Chain {
    const double* img;    // frame's best grid (covered pixels already +inf in pass 2)
    const uint8_t* crow;  // tile classes of this tile-row
    bool skip1;           // pass 2: tiles of class 1 are fully masked
    int v0, rows;
};

// Fold the valid pixels of tile t onto the lane-owned running sums (lane k<9
// owns sum k; lanes >= 9 shadow sum 8).  Returns the valid count (uniform).
__device__ __forceinline__ int fold_tile(const Chain& ch, const Geometry& g, const Trig& tg, int t,
                                         double* sm, double& acc)
{
    if (ch.skip1 && ch.crow[t] == 1) return 0;
    const int lane = threadIdx.x & 31;
    const int kk = lane < 9 ? lane : 8;
    const int u0 = t * g.tw;
    const int cols = min(g.tw, g.w - u0);
    const int npx = ch.rows * cols;
    int cnt = 0;
    for (int base = 0; base < npx; base += 32) {
        int p = base + lane;
        double x = 0.0, y = 0.0, z = 0.0, one = 0.0;
        if (p < npx) {
            int v = ch.v0 + p / cols;
            int u = u0 + p % cols;
            double r = ch.img[(long long)v * g.w + u];
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
#pragma unroll 4
        for (int j = 0; j < nj; ++j) acc += sm[j * 9 + kk];
        __syncwarp();
    }
    return cnt;
}

// True iff every valid pixel of tiles [t0, t1) reconstructs within tau.
__device__ __forceinline__ bool span_fits(const Chain& ch, const Geometry& g, const Trig& tg, int t0,
                                          int t1, double a, double b, double c, double tau, double r_max)
{
    const int lane = threadIdx.x & 31;
    const int U0 = t0 * g.tw;
    const int U1 = min(t1 * g.tw, g.w);
    const int U = U1 - U0;
    const int npx = ch.rows * U;
    for (int base = 0; base < npx; base += 32) {
        int p = base + lane;
        bool bad = false;
        if (p < npx) {
            int v = ch.v0 + p / U;
            int u = U0 + p % U;
            double r = ch.img[(long long)v * g.w + u];
            if (isfinite(r)) {
                double dx, dy, dz;
                ray_dir(tg, v, u, dx, dy, dz);
                bad = !pixel_fits(r, dx, dy, dz, a, b, c, tau, r_max);
            }
        }
        if (__any_sync(STPC_FULL, bad)) return false;
    }
    return true;
}

__device__ __forceinline__ bool solve_round(double acc, double cond_limit, double& a, double& b, double& c)
{
    double s[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) s[k] = shfl_d(acc, k);
    if (!plane_from_sums(s, cond_limit, a, b, c)) return false;
    a = f32_round(a);
    b = f32_round(b);
    c = f32_round(c);
    return true;
}

__global__ void __launch_bounds__(FIT_WARPS * 32, 6) fit_rows_kernel(FitArgs A)
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
    while (t < g.tx) {
        double acc = 0.0;
        int cnt = fold_tile(ch, g, A.tg, t, sm, acc);
        bool ok = false;
        double a = 0.0, b = 0.0, c = 0.0;
        if (cnt >= 3) {  // sums[8] >= 3.0
            ok = solve_round(acc, A.cond_limit, a, b, c);
            if (ok) ok = span_fits(ch, g, A.tg, t, t + 1, a, b, c, A.tau, A.r_max);
        }
        if (!ok) {  // residual tile (class 0 stays; covered tiles keep class 1)
            t += 1;
            continue;
        }
        const int s = t;
        int e = t + 1;
        while (e < g.tx) {
            double saved = acc;
            int add = fold_tile(ch, g, A.tg, e, sm, acc);
            if (add == 0) {  // unchanged sums -> same plane -> same verdict
                e += 1;
                continue;
            }
            double na, nb, nc;
            bool ok2 = solve_round(acc, A.cond_limit, na, nb, nc);
            if (ok2) ok2 = span_fits(ch, g, A.tg, s, e + 1, na, nb, nc, A.tau, A.r_max);
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

void launch_fit_rows(const FitArgs& a, cudaStream_t s)
{
    long long warps = (long long)a.n_jobs * a.g.ty;
    if (warps <= 0) return;
    STPC_LAUNCH();
    fit_rows_kernel<<<(unsigned)((warps + FIT_WARPS - 1) / FIT_WARPS), FIT_WARPS * 32, 0, s>>>(a);
}

// K3a: one warp per key-frame chain; for each of its runs and each P channel,
// c' = f32(mean over valid span pixels of r * (d . n)), folded v-major over the
// whole span in the reference's order, then the span re-test with (a, b, c').
// Spans that pass mark their tiles class 1 in the channel and poison the
// channel's pixels there (+inf) for pass 2.
__global__ void __launch_bounds__(128) refit_kernel(RefitArgs A)
{
    __shared__ double smem[4][32];
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    double* sm = smem[threadIdx.x >> 5];
    const long long kc = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (kc >= (long long)A.n_groups * g.ty) return;
    const int grp = (int)(kc / g.ty);
    const int tr = (int)(kc % g.ty);
    const int kframe = grp * A.n + A.k;
    const long long kslot = (long long)kframe * g.ty + tr;
    const int nr = A.n_runs[kslot];
    const int v0 = tr * g.th;
    const int rows = min(g.th, g.h - v0);
    const int pm = (A.n + 7) / 8;
    long long tbytes = 0;
    for (int j = 0; j < nr; ++j) {
        const long long ri = kslot * g.tx + j;
        const int s = A.run_s[ri], len = A.run_len[ri];
        const double a = (double)A.run_abc[3 * ri], b = (double)A.run_abc[3 * ri + 1];
        const int U0 = s * g.tw;
        const int U1 = min((s + len) * g.tw, g.w);
        const int U = U1 - U0;
        const int npx = rows * U;
        uint8_t* okv = A.ref_ok + (kc * g.tx + j) * A.n;
        float* cv = A.ref_c + (kc * g.tx + j) * A.n;
        int present = 0;
        for (int chn = 0; chn < A.n; ++chn) {
            if (chn == A.k) continue;
            const int frame = grp * A.n + chn;
            double* img = A.best + (long long)frame * g.P;
            double acc = 0.0;
            int cnt = 0;
            for (int base = 0; base < npx; base += 32) {
                int p = base + lane;
                double prod = 0.0;
                bool valid = false;
                if (p < npx) {
                    int v = v0 + p / U;
                    int u = U0 + p % U;
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
                const int nj = min(32, npx - base);
#pragma unroll 8
                for (int jj = 0; jj < nj; ++jj) acc += sm[jj];
                __syncwarp();
            }
            bool ok = false;
            double c = 0.0;
            if (cnt > 0) {
                c = f32_round(acc / (double)cnt);
                ok = true;
                for (int base = 0; base < npx && ok; base += 32) {
                    int p = base + lane;
                    bool bad = false;
                    if (p < npx) {
                        int v = v0 + p / U;
                        int u = U0 + p % U;
                        double r = img[(long long)v * g.w + u];
                        if (isfinite(r)) {
                            double dx, dy, dz;
                            ray_dir(A.tg, v, u, dx, dy, dz);
                            bad = !pixel_fits(r, dx, dy, dz, a, b, c, A.tau, A.r_max);
                        }
                    }
                    ok = !__any_sync(STPC_FULL, bad);
                }
            }
            if (lane == 0) {
                okv[chn] = ok;
                cv[chn] = (float)c;
            }
            if (ok) {
                present += 1;
                uint8_t* crow = A.cls + ((long long)frame * g.ty + tr) * g.tx;
                for (int tt = s + lane; tt < s + len; tt += 32) crow[tt] = 1;
                for (int p = lane; p < npx; p += 32) {
                    int v = v0 + p / U;
                    int u = U0 + p % U;
                    img[(long long)v * g.w + u] = __longlong_as_double(0x7ff0000000000000ll);
                }
            }
        }
        if (lane == 0) okv[A.k] = 1;
        tbytes += 18 + pm + 4 * present;
    }
    if (lane == 0) A.chain_tbytes[kc] = tbytes;
}

void launch_refit(const RefitArgs& a, cudaStream_t s)
{
    long long warps = (long long)a.n_groups * a.g.ty;
    if (warps <= 0) return;
    STPC_LAUNCH();
    refit_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(a);
}

}  // namespace stpc
