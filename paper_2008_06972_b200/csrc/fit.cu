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
//   * moments: lanes compute x, y, z of up to 32 pixels at once; the 9 running
//     sums (lane k owns sum k) then fold the pixels in raster order through
//     shuffles -- the reference's rounding sequence, not a tree (SURVEY.md
//     §0 item 3: a shuffle tree flips run decisions);
//   * union re-test: order-independent AND over pixels, 32 lanes at a time
//     with an early-out vote (the reference's early return gives the same
//     verdict);
//   * the 3x3 solve runs redundantly in every lane (warp-uniform branches).
#include "kernels.cuh"

namespace stpc {

struct Chain {
    const double* img;    // frame's best grid
    const uint8_t* crow;  // tile classes of this tile-row
    int excl;             // class value that masks a tile out (-1: none)
    int v0, rows;
};

// Fold the valid pixels of tile t onto the lane-owned running sums.
// Returns the tile's valid pixel count (warp-uniform).
__device__ __forceinline__ int fold_tile(const Chain& ch, const Geometry& g, const Trig& tg, int t,
                                         int psel, int qsel, double& acc)
{
    if (ch.excl >= 0 && ch.crow[t] == ch.excl) return 0;
    const int lane = threadIdx.x & 31;
    const int u0 = t * g.tw;
    const int cols = min(g.tw, g.w - u0);
    const int npx = ch.rows * cols;
    int cnt = 0;
    for (int base = 0; base < npx; base += 32) {
        int p = base + lane;
        double x = 0.0, y = 0.0, z = 0.0;
        bool valid = false;
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
                valid = true;
            }
        }
        uint32_t m = __ballot_sync(STPC_FULL, valid);
        cnt += __popc(m);
        while (m) {
            int j = __ffs(m) - 1;
            m &= m - 1;
            double xj = shfl_d(x, j), yj = shfl_d(y, j), zj = shfl_d(z, j);
            double P = psel == 0 ? xj : psel == 1 ? yj : psel == 2 ? zj : 1.0;
            double Q = qsel == 0 ? xj : qsel == 1 ? yj : qsel == 2 ? zj : 1.0;
            acc += P * Q;  // y*1.0 == y and 1.0*1.0 == 1.0 exactly
        }
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
            bool valid = isfinite(r) && !(ch.excl >= 0 && ch.crow[u / g.tw] == ch.excl);
            if (valid) {
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

__global__ void __launch_bounds__(128) fit_rows_kernel(FitArgs A)
{
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
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
    ch.excl = A.mode == 0 ? -1 : 1;
    ch.v0 = tr * g.th;
    ch.rows = min(g.th, g.h - ch.v0);
    const uint8_t run_cls = A.mode == 0 ? 1 : 2;

    // lane k accumulates sum k of [Syy, Syz, Szz, Sy, Sz, Sxy, Sxz, Sx, N]
    const int PS[9] = {1, 1, 2, 1, 2, 0, 0, 0, 3};
    const int QS[9] = {1, 2, 2, 3, 3, 1, 2, 3, 3};
    const int psel = lane < 9 ? PS[lane] : 3;
    const int qsel = lane < 9 ? QS[lane] : 3;

    uint16_t* rs = A.run_s + slot * g.tx;
    uint16_t* rl = A.run_len + slot * g.tx;
    float* rabc = A.run_abc + slot * g.tx * 3;
    int n_runs = 0;
    int t = 0;
    while (t < g.tx) {
        double acc = 0.0;
        int cnt = fold_tile(ch, g, A.tg, t, psel, qsel, acc);
        bool ok = false;
        double a = 0.0, b = 0.0, c = 0.0;
        if (cnt >= 3) {  // sums[8] >= 3.0
            ok = solve_round(acc, A.cond_limit, a, b, c);
            if (ok) ok = span_fits(ch, g, A.tg, t, t + 1, a, b, c, A.tau, A.r_max);
        }
        if (!ok) {  // residual tile (class 0 stays; excluded tiles keep theirs)
            t += 1;
            continue;
        }
        const int s = t;
        int e = t + 1;
        while (e < g.tx) {
            double saved = acc;
            int add = fold_tile(ch, g, A.tg, e, psel, qsel, acc);
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
            if (!(ch.excl >= 0 && crow[tt] == ch.excl)) crow[tt] = run_cls;
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
    fit_rows_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(a);
}

// K3a: one warp per key-frame chain; for each of its runs and each P channel,
// c' = f32(mean over valid span pixels of r * (d . n)), folded v-major over the
// whole span in the reference's order, then the span re-test with (a, b, c').
__global__ void __launch_bounds__(128) refit_kernel(RefitArgs A)
{
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
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
            const double* img = A.best + (long long)frame * g.P;
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
                uint32_t m = __ballot_sync(STPC_FULL, valid);
                cnt += __popc(m);
                while (m) {
                    int jj = __ffs(m) - 1;
                    m &= m - 1;
                    acc += shfl_d(prod, jj);
                }
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
