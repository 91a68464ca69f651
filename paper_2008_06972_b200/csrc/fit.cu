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

// q, r = p / d, p % d for 0 <= p < 2^24 without an integer divide: float
// reciprocal estimate, then an exact +-1 correction.
__device__ __forceinline__ void divmod_small(int p, int d, float rcp, int& q, int& r)
{
    q = __float2int_rz(((float)p + 0.5f) * rcp);
    r = p - q * d;
    if (r < 0) { q -= 1; r += d; }
    else if (r >= d) { q += 1; r -= d; }
}

// G lanes per chain, 32/G chains per warp.  All chains of a warp advance in
// lock-step through one state-machine step per iteration (fold one tile,
// optionally solve + test, update), so every warp instruction serves 32/G
// chains; per-chain differences (union sizes, branch outcomes) are handled
// with predicates and warp-uniform loop bounds.
//
// Per chain (== one encode_tile_row call):
//   START mode: sums = fold(tile t) from zero; if N >= 3 and the solve is ok,
//               round through f32 and test tile t alone; pass -> GROW with
//               s = t, fail -> tile t is residual; t += 1.
//   GROW mode:  sums += fold(tile t); an empty tile extends the run (same
//               sums, same plane, same verdict); otherwise solve and test
//               the union [s, t]; pass -> keep plane, t += 1; fail -> emit run
//               [s, t) and restart in START mode at the same t.
//   t == tiles_x closes an open run.
template <int G>
__global__ void __launch_bounds__(FIT_WARPS * 32, 5) fit_rows_kernel(FitArgs A)
{
    constexpr int CPW = 32 / G;
    __shared__ double smem[FIT_WARPS][CPW][G * 8];
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int sub = lane / G;
    const int gl = lane % G;
    const unsigned gmask = G == 32 ? STPC_FULL : (((1u << G) - 1u) << (sub * G));
    const long long n_chains = (long long)A.n_jobs * g.ty;
    const long long cid = ((long long)blockIdx.x * FIT_WARPS + wib) * CPW + sub;
    bool done = cid >= n_chains;
    if (__all_sync(STPC_FULL, done)) return;

    // chain setup
    int frame = 0, tr = 0;
    if (!done) {
        const int job = (int)(cid / g.ty);
        tr = (int)(cid % g.ty);
        if (A.mode == 0) {
            frame = job * A.n_frames_group + A.k;
        } else {
            int np = A.n_frames_group - 1;
            int grp = job / np, i = job % np;
            frame = grp * A.n_frames_group + (i < A.k ? i : i + 1);
        }
    }
    const long long slot = (long long)frame * g.ty + tr;
    const double* img = A.best + (long long)frame * g.P;
    uint8_t* crow = A.cls + slot * g.tx;
    const bool skip1 = A.mode != 0;
    const int v0 = tr * g.th;
    const int rows = min(g.th, g.h - v0);
    const uint8_t run_cls = A.mode == 0 ? 1 : 2;
    double* sm = smem[wib][sub];
    uint16_t* rs = A.run_s + slot * g.tx;
    uint16_t* rl = A.run_len + slot * g.tx;
    float* rabc = A.run_abc + slot * g.tx * 3;

    // lane gl < 8 owns sum gl of [Syy, Syz, Szz, Sy, Sz, Sxy, Sxz, Sx]; N is
    // the exact valid count (the reference's N += 1.0 fold equals it).
    double acc = 0.0;
    int nsum = 0;
    int t = 0, s = 0, n_runs = 0;
    bool grow = false;
    double a = 0.0, b = 0.0, c = 0.0;

    while (__any_sync(STPC_FULL, !done)) {
        // ---- fold tile t of every live chain onto its running sums
        if (!done && !grow) { acc = 0.0; nsum = 0; }
        const bool masked = done || (skip1 && crow[t] == 1);
        const int u0 = t * g.tw;
        const int cols = done ? 1 : min(g.tw, g.w - u0);
        const int npx = masked ? 0 : rows * cols;
        const float rc = __frcp_rn((float)cols);
        int cnt = 0;
        for (int base = 0; __any_sync(STPC_FULL, base < npx); base += G) {
            const int p = base + gl;
            double x = 0.0, y = 0.0, z = 0.0;
            bool valid = false;
            if (p < npx) {
                int dv, du;
                divmod_small(p, cols, rc, dv, du);
                const int v = v0 + dv, u = u0 + du;
                const double r = img[(long long)v * g.w + u];
                if (isfinite(r)) {
                    double dx, dy, dz;
                    ray_dir(A.tg, v, u, dx, dy, dz);
                    x = r * dx;
                    y = r * dy;
                    z = r * dz;
                    valid = true;
                }
            }
            cnt += __popc(__ballot_sync(STPC_FULL, valid) & gmask);
            double* row = sm + gl * 8;
            row[0] = y * y;
            row[1] = y * z;
            row[2] = z * z;
            row[3] = y;
            row[4] = z;
            row[5] = x * y;
            row[6] = x * z;
            row[7] = x;
            __syncwarp();
            const int nj = min(G, npx - base);  // <= 0 for finished chains
            if (gl < 8)
                for (int j = 0; j < nj; ++j) acc += sm[j * 8 + gl];  // +0.0 for invalid: exact
            __syncwarp();
        }
        nsum += cnt;

        // ---- solve (chains that need it), round through f32
        const bool need = !done && (grow ? cnt > 0 : nsum >= 3);
        double na = 0.0, nb = 0.0, nc = 0.0;
        bool ok = false;
        {
            double sv[9];
#pragma unroll
            for (int k = 0; k < 8; ++k) sv[k] = __shfl_sync(STPC_FULL, acc, sub * G + k);
            sv[8] = (double)nsum;
            if (need && plane_from_sums(sv, A.cond_limit, na, nb, nc)) {
                na = f32_round(na);
                nb = f32_round(nb);
                nc = f32_round(nc);
                ok = true;
            }
        }

        // ---- test the union (START: tile t; GROW: tiles [s, t])
        {
            const int t0 = grow ? s : t;
            const int U0 = t0 * g.tw;
            const int U = min((t + 1) * g.tw, g.w) - U0;
            const int tpx = ok ? rows * U : 0;
            const float ru = __frcp_rn((float)(U > 0 ? U : 1));
            bool bad_any = false;
            for (int base = 0; __any_sync(STPC_FULL, base < tpx && !bad_any); base += G) {
                const int p = base + gl;
                bool bad = false;
                if (p < tpx && !bad_any) {
                    int dv, du;
                    divmod_small(p, U, ru, dv, du);
                    const int v = v0 + dv, u = U0 + du;
                    const double r = img[(long long)v * g.w + u];
                    if (isfinite(r)) {
                        double dx, dy, dz;
                        ray_dir(A.tg, v, u, dx, dy, dz);
                        bad = !pixel_fits(r, dx, dy, dz, na, nb, nc, A.tau, A.r_max);
                    }
                }
                // ballot unconditionally: every lane must reach the full-mask collective
                const unsigned bb = __ballot_sync(STPC_FULL, bad) & gmask;
                bad_any = bad_any || bb != 0;
            }
            ok = ok && !bad_any;
        }

        // ---- state update (uniform within each chain's lane group)
        if (!done) {
            int emit_e = -1;
            if (!grow) {
                if (ok) {
                    s = t;
                    a = na; b = nb; c = nc;
                    grow = true;
                }
                t += 1;
            } else if (cnt == 0 || ok) {
                if (ok) { a = na; b = nb; c = nc; }
                t += 1;
            } else {
                emit_e = t;  // close [s, t); t restarts as a start tile
                grow = false;
            }
            if (t >= g.tx) {
                if (grow) { emit_e = g.tx; grow = false; }
                done = true;
            }
            if (emit_e >= 0) {
                if (gl == 0) {
                    rs[n_runs] = (uint16_t)s;
                    rl[n_runs] = (uint16_t)(emit_e - s);
                    rabc[3 * n_runs] = (float)a;
                    rabc[3 * n_runs + 1] = (float)b;
                    rabc[3 * n_runs + 2] = (float)c;
                }
                for (int tt = s + gl; tt < emit_e; tt += G)
                    if (!(skip1 && crow[tt] == 1)) crow[tt] = run_cls;
                n_runs += 1;
            }
        }
    }
    if (cid < n_chains && gl == 0) A.n_runs[slot] = n_runs;
}

void launch_fit_rows(const FitArgs& a, cudaStream_t s)
{
    long long chains = (long long)a.n_jobs * a.g.ty;
    if (chains <= 0) return;
    const int tpx = a.g.tw * a.g.th;
    STPC_LAUNCH();
    if (tpx <= 32) {
        long long warps = (chains + 3) / 4;
        fit_rows_kernel<8><<<(unsigned)((warps + FIT_WARPS - 1) / FIT_WARPS), FIT_WARPS * 32, 0, s>>>(a);
    } else if (tpx <= 128) {
        long long warps = (chains + 1) / 2;
        fit_rows_kernel<16><<<(unsigned)((warps + FIT_WARPS - 1) / FIT_WARPS), FIT_WARPS * 32, 0, s>>>(a);
    } else {
        fit_rows_kernel<32><<<(unsigned)((chains + FIT_WARPS - 1) / FIT_WARPS), FIT_WARPS * 32, 0, s>>>(a);
    }
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
        const float ru = __frcp_rn((float)U);
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
                    int dv, du;
                    divmod_small(p, U, ru, dv, du);
                    int v = v0 + dv, u = U0 + du;
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
