// K3c -- residual compaction and .stpc v1 payload assembly on the device.
//
// Replaces residual_pixels_for_tiles + the residual/run/fallback sections of
// serialize (/root/reference/pkg/src/stpc/spatial.py:160-168;
// /root/reference/pkg/src/stpc/temporal.py:206-245;
// /root/reference/pkg/src/stpc/bitstream.py:193-278, 176-190) and the
// coverage counts (/root/reference/pkg/src/stpc/temporal.py:269-290).
//
// Payload layout per group (pkg/README.md:79-120, bitstream.py:204-276):
//   config(57) | transforms n*48 | validity bitmaps n*ceil(P/8) |
//   u32 #runs, runs <HHH fff> + presence bits + f32 per present P channel |
//   per channel: u32 #rows, rows <HH> + runs <HH fff> |
//   per channel: u32 count [, LEB128 deltas, u16 codes, u32 #esc, f32 escapes]
//
// Residual pixels of a channel are the valid pixels of class-0 tiles in flat
// (row-major) order; one warp walks one image row 32 pixels at a time, the
// per-row counts are chained across rows by the plan kernel (delta coding
// crosses row boundaries), then the emit pass writes each row's bytes at its
// final offsets.
#include "kernels.cuh"

namespace stpc {

__device__ __forceinline__ uint32_t load_bits(const uint8_t* bm, long long word)
{
    return natural_bits(__ldg(reinterpret_cast<const uint32_t*>(bm) + word));
}

struct RowWalk {
    long long rb, re;  // flat pixel range of the row
    long long w0, w1;  // bitmap words overlapping it
};

__device__ __forceinline__ RowWalk row_walk(const Geometry& g, int v)
{
    RowWalk rw;
    rw.rb = (long long)v * g.w;
    rw.re = rw.rb + g.w;
    rw.w0 = rw.rb >> 5;
    rw.w1 = (rw.re + 31) >> 5;
    return rw;
}

// residual / class masks of one 32-pixel word of one row
__device__ __forceinline__ void word_masks(const Geometry& g, const uint8_t* vb, const uint8_t* crow,
                                           const RowWalk& rw, long long wd, int v, uint32_t& res,
                                           uint32_t& tmp, uint32_t& fb)
{
    const int lane = threadIdx.x & 31;
    long long pix = wd * 32 + lane;
    uint32_t valid = load_bits(vb, wd);
    int cls = 255;
    if (pix >= rw.rb && pix < rw.re && ((valid >> lane) & 1u)) {
        const int u = (int)(pix - rw.rb);
        // u / tw without an integer divide (exact +-1 correction)
        int q = __float2int_rz(((float)u + 0.5f) * __frcp_rn((float)g.tw));
        const int r = u - q * g.tw;
        q += r < 0 ? -1 : (r >= g.tw ? 1 : 0);
        cls = crow[q];
    }
    res = __ballot_sync(STPC_FULL, cls == 0);
    tmp = __ballot_sync(STPC_FULL, cls == 1);
    fb = __ballot_sync(STPC_FULL, cls == 2);
}


// Lane-per-word view: the residual / temporal / fallback masks of bitmap word
// wd restricted to image row [rb, re).  Tile classes are applied per tile span
// (<= 32/tw + 1 spans per word), not per pixel.
__device__ __forceinline__ void word_classes(const Geometry& g, const uint8_t* crow, uint32_t valid, long long rb,
                                             long long re, long long wd, uint32_t& res, uint32_t& tmp, uint32_t& fb)
{
    res = tmp = fb = 0;
    const long long p0 = wd * 32;
    const int lo = (int)max(0LL, rb - p0), hi = (int)min(32LL, re - p0);
    if (lo >= hi) return;
    if (g.tw == 4 && (g.w & 15) == 0 && lo == 0 && hi == 32) {
        // a whole word of 4-pixel tiles (w % 16 == 0 makes its first tile
        // index a multiple of 4): eight class bytes by two aligned loads,
        // compared four at a time, each byte spread to its tile's nibble
        const int t0 = (int)(p0 - rb) >> 2;
        const uint32_t c0 = *reinterpret_cast<const uint32_t*>(crow + t0);
        const uint32_t c1 = *reinterpret_cast<const uint32_t*>(crow + t0 + 4);
        auto nib = [](uint32_t m) {  // 0xFF / 0x00 per byte -> 0xF / 0x0 per nibble
            return (m & 0xFu) | ((m >> 4) & 0xF0u) | ((m >> 8) & 0xF00u) | ((m >> 12) & 0xF000u);
        };
        res = (nib(__vcmpeq4(c0, 0u)) | (nib(__vcmpeq4(c1, 0u)) << 16)) & valid;
        tmp = (nib(__vcmpeq4(c0, 0x01010101u)) | (nib(__vcmpeq4(c1, 0x01010101u)) << 16)) & valid;
        fb = (nib(__vcmpeq4(c0, 0x02020202u)) | (nib(__vcmpeq4(c1, 0x02020202u)) << 16)) & valid;
        return;
    }
    int u = (int)(p0 + lo - rb);  // column of bit lo
    int tile = __float2int_rz(((float)u + 0.5f) * __frcp_rn((float)g.tw));
    {
        const int r = u - tile * g.tw;
        tile += r < 0 ? -1 : (r >= g.tw ? 1 : 0);
    }
    int bit = lo;
    while (bit < hi) {
        const int nb = min(hi - bit, (tile + 1) * g.tw - u);
        const uint32_t m = (nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u)) << bit;
        const uint8_t c = crow[tile];
        if (c == 0) res |= m;
        else if (c == 1) tmp |= m;
        else if (c == 2) fb |= m;
        bit += nb;
        u += nb;
        tile += 1;
    }
    res &= valid;
    tmp &= valid;
    fb &= valid;
}

__device__ __forceinline__ long long warp_excl_max(long long v, long long ident)
{
    const int lane = threadIdx.x & 31;
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long t = __shfl_up_sync(STPC_FULL, inc, o);
        if (lane >= o) inc = max(inc, t);
    }
    long long ex = __shfl_up_sync(STPC_FULL, inc, 1);
    return lane == 0 ? ident : ex;
}

// Warp per (frame, row): counts, varint bytes (excluding the row's first
// delta), first/last residual flat index, coverage counters.
#ifndef STPC_ROWSTATS_MINB
#define STPC_ROWSTATS_MINB 1
#endif
__global__ void __launch_bounds__(256, STPC_ROWSTATS_MINB) rowstats_kernel(PlanArgs A)
{
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long F = (long long)A.n_groups * A.n;
    if (wid >= F * g.h) return;
    const int f = (int)(wid / g.h);
    const int v = (int)(wid % g.h);
    const uint8_t* vb = A.vbits + (long long)f * g.pbs;
    const uint8_t* eb = A.ebits + (long long)f * g.pbs;
    const uint8_t* crow = A.cls + ((long long)f * g.ty + v / g.th) * g.tx;
    RowWalk rw = row_walk(g, v);
    int cnt = 0, nesc = 0, vbytes = 0, ntmp = 0, nfb = 0;
    long long first = -1, last = -1;  // carried across word batches
    for (long long base = rw.w0; base < rw.w1; base += 32) {
        const long long wd = base + lane;
        uint32_t res = 0, tmp = 0, fb = 0, esc = 0;
        if (wd < rw.w1) {
            word_classes(g, crow, load_bits(vb, wd), rw.rb, rw.re, wd, res, tmp, fb);
            if (res) esc = load_bits(eb, wd) & res;
        }
        const long long wfirst = res ? wd * 32 + (__ffs(res) - 1) : -1;
        const long long wlast = res ? wd * 32 + (31 - __clz(res)) : -1;
        // previous residual before this word within the row (or none)
        long long prev = warp_excl_max(wlast, -1);
        prev = max(prev, last);
        int len = 0;
        if (res) len = (__popc(res) - 1) + (prev >= 0 ? varint_len((uint32_t)(wfirst - prev)) : 0);
        len = __reduce_add_sync(STPC_FULL, len);
        const int c = __reduce_add_sync(STPC_FULL, __popc(res)), e = __reduce_add_sync(STPC_FULL, __popc(esc));
        const int t1 = __reduce_add_sync(STPC_FULL, __popc(tmp)), f2 = __reduce_add_sync(STPC_FULL, __popc(fb));
        // batch first/last
        const unsigned nz = __ballot_sync(STPC_FULL, res != 0);
        if (nz) {
            const long long bf = __shfl_sync(STPC_FULL, wfirst, __ffs(nz) - 1);
            const long long bl = __shfl_sync(STPC_FULL, wlast, 31 - __clz(nz));
            if (first < 0) first = bf;
            last = bl;
        }
        vbytes += len;
        cnt += c;
        nesc += e;
        ntmp += t1;
        nfb += f2;
    }
    if (lane == 0) {
        RowStat st;
        st.cnt = cnt;
        st.nesc = nesc;
        st.vb = vbytes;
        st.first = (int)first;
        st.last = (int)last;
        A.rowstat[wid] = st;
        long long* fs = A.fstats + (long long)f * FS_COUNT;
        if (ntmp) atomicAdd((unsigned long long*)&fs[FS_TEMPORAL], (unsigned long long)ntmp);
        if (nfb) atomicAdd((unsigned long long*)&fs[FS_FALLBACK], (unsigned long long)nfb);
        if (cnt) atomicAdd((unsigned long long*)&fs[FS_RESIDUAL], (unsigned long long)cnt);
        if (nesc) atomicAdd((unsigned long long*)&fs[FS_ESCAPES], (unsigned long long)nesc);
    }
}

void launch_rowstats(const PlanArgs& a, cudaStream_t s)
{
    long long warps = (long long)a.n_groups * a.n * a.g.h;
    if (warps <= 0) return;
    STPC_LAUNCH();
    rowstats_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(a);
}

// Block per group: chain the per-row residual counts into per-frame sections,
// lay out the fallback rows and temporal records, and size the payload.
__global__ void plan_kernel(PlanArgs A)
{
    const Geometry& g = A.g;
    const int grp = blockIdx.x;
    const int n = A.n;
    const int tid = threadIdx.x;
    const long long PB = (g.P + 7) / 8;
    // per-frame residual chaining and fallback row layout (thread per frame)
    for (int i = tid; i < n; i += blockDim.x) {
        const long long f = (long long)grp * n + i;
        long long cnt = 0, vbt = 0, esc = 0, prev = -1;
        for (int v = 0; v < g.h; ++v) {
            RowStat st = A.rowstat[f * g.h + v];
            RowOff ro;
            ro.cnt_off = (int)cnt;
            ro.vb_off = (int)vbt;
            ro.esc_off = (int)esc;
            ro.prev = (int)(prev < 0 ? 0 : prev);
            if (st.cnt) {
                vbt += st.vb + varint_len((uint32_t)(st.first - ro.prev));
                cnt += st.cnt;
                esc += st.nesc;
                prev = st.last;
            }
            A.rowoff[f * g.h + v] = ro;
        }
        A.res_cnt[f] = cnt;
        A.res_vb[f] = vbt;
        A.res_esc[f] = esc;
        long long rows = 0;
        if (i != A.k) {
            for (int tr = 0; tr < g.ty; ++tr) rows += A.n_runs[f * g.ty + tr] > 0;
        }
        A.fb_rows[f] = rows;
    }
    __syncthreads();
    if (tid != 0) return;
    long long* sec = A.sec + (long long)grp * (2 + 2 * n);
    long long off = 57 + 48LL * n + PB * n;
    // temporal section
    sec[0] = off;
    off += 4;
    const long long kf = (long long)grp * n + A.k;
    long long nruns = 0;
    for (int tr = 0; tr < g.ty; ++tr) {
        long long kc = (long long)grp * g.ty + tr;
        A.chain_off[kf * g.ty + tr] = off;
        off += A.chain_tbytes[kc];
        nruns += A.n_runs[kf * g.ty + tr];
    }
    sec[1] = nruns;
    // fallback sections
    for (int i = 0; i < n; ++i) {
        const long long f = (long long)grp * n + i;
        sec[2 + i] = off;
        off += 4;
        if (i == A.k) continue;
        for (int tr = 0; tr < g.ty; ++tr) {
            int nr = A.n_runs[f * g.ty + tr];
            A.chain_off[f * g.ty + tr] = off;
            if (nr > 0) off += 4 + 16LL * nr;
        }
    }
    // residual sections
    for (int i = 0; i < n; ++i) {
        const long long f = (long long)grp * n + i;
        sec[2 + n + i] = off;
        off += 4;
        if (A.res_cnt[f]) off += A.res_vb[f] + 2 * A.res_cnt[f] + 4 + 4 * A.res_esc[f];
    }
    A.payload_len[grp] = off;
}

void launch_plan(const PlanArgs& a, cudaStream_t s)
{
    if (a.n_groups <= 0) return;
    STPC_LAUNCH();
    plan_kernel<<<a.n_groups, 64, 0, s>>>(a);
}

// Single-block exclusive scan over group lengths (rounded up to `align`).
__global__ void group_scan_kernel(const long long* lens, long long* offs, int G, int align, long long add)
{
    __shared__ long long carry;
    __shared__ long long wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < G; base += blockDim.x) {
        int i = base + threadIdx.x;
        long long v = 0;
        if (i < G) {
            v = lens[i] + add;
            v = (v + align - 1) / align * align;
        }
        long long inc = warp_incl_scan_ll(v);
        if (lane == 31) wsum[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            long long ws = lane < (blockDim.x >> 5) ? wsum[lane] : 0;
            long long wi = warp_incl_scan_ll(ws);
            if (lane < (blockDim.x >> 5)) wsum[lane] = wi - ws;
        }
        __syncthreads();
        long long excl = carry + wsum[wid] + inc - v;
        if (i < G) offs[i] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) offs[G] = carry;
}

void launch_group_scan(const long long* lens, long long* offs, int G, int align, long long add, cudaStream_t s)
{
    STPC_LAUNCH();
    group_scan_kernel<<<1, 1024, 0, s>>>(lens, offs, G, align, add);
}

// ---------------------------------------------------------------------------
// emission
// ---------------------------------------------------------------------------

// config, transforms, section counts; block per group
__global__ void emit_header_kernel(EmitArgs E)
{
    const PlanArgs& A = E.p;
    const int grp = blockIdx.x;
    const int n = A.n;
    uint8_t* out = E.payload + A.payload_off[grp];
    const long long* sec = A.sec + (long long)grp * (2 + 2 * n);
    for (int i = threadIdx.x; i < 57; i += blockDim.x) out[i] = E.cfg_bytes[i];
    for (int i = threadIdx.x; i < 12 * n; i += blockDim.x) {
        int fi = i / 12, j = i % 12;
        put_f32(out + 57 + 4 * i, (float)E.xf[((long long)grp * n + fi) * 12 + j]);
    }
    if (threadIdx.x == 0) put_u32(out + sec[0], (uint32_t)sec[1]);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const long long f = (long long)grp * n + i;
        put_u32(out + sec[2 + i], (uint32_t)A.fb_rows[f]);
        put_u32(out + sec[2 + n + i], (uint32_t)A.res_cnt[f]);
        if (A.res_cnt[f]) {
            long long o = sec[2 + n + i] + 4 + A.res_vb[f] + 2 * A.res_cnt[f];
            put_u32(out + o, (uint32_t)A.res_esc[f]);
        }
    }
}

// validity bitmaps: frame bytes [0, PB) copied into the payload
// Validity bitmaps into the payload (packbits, bitstream.py:219-220): block
// per frame; the destination sits at an arbitrary byte offset, so head and
// tail bytes are stored singly and every aligned 32-bit destination word is
// assembled from two source words by a funnel shift.
__global__ void __launch_bounds__(256) emit_bitmaps_kernel(EmitArgs E)
{
    const PlanArgs& A = E.p;
    const Geometry& g = A.g;
    const int f = blockIdx.x;
    const int grp = f / A.n, i = f % A.n;
    const long long PB = (g.P + 7) / 8;
    uint8_t* out = E.payload + A.payload_off[grp] + 57 + 48LL * A.n + PB * i;
    const uint8_t* src = A.vbits + (long long)f * g.pbs;  // 4-byte aligned, pbs % 4 == 0
    const uint32_t* src32 = reinterpret_cast<const uint32_t*>(src);
    const long long nsw = g.pbs / 4;
    const int head = (int)((4 - ((unsigned long long)out & 3)) & 3);
    if (head > PB) {
        for (long long b = threadIdx.x; b < PB; b += blockDim.x) out[b] = src[b];
        return;
    }
    if (threadIdx.x < head) out[threadIdx.x] = src[threadIdx.x];
    const long long nw = (PB - head) / 4;
    uint32_t* dst32 = reinterpret_cast<uint32_t*>(out + head);
    const int sh = 8 * head;
    for (long long j = threadIdx.x; j < nw; j += blockDim.x) {
        const long long sw = (head + 4 * j) >> 2;  // head < 4: source word holding the first byte
        const uint32_t lo = __ldg(src32 + sw);
        const uint32_t hi = sw + 1 < nsw ? __ldg(src32 + sw + 1) : 0u;
        dst32[j] = sh ? __funnelshift_r(lo, hi, sh) : lo;
    }
    for (long long b = head + 4 * nw + threadIdx.x; b < PB; b += blockDim.x) out[b] = src[b];
}

// temporal runs: warp per key chain
__global__ void __launch_bounds__(128) emit_temporal_kernel(EmitArgs E)
{
    const PlanArgs& A = E.p;
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const long long kc = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (kc >= (long long)A.n_groups * g.ty) return;
    const int grp = (int)(kc / g.ty), tr = (int)(kc % g.ty);
    const int n = A.n, k = A.k, pm = (n + 7) / 8;
    const long long kslot = ((long long)grp * n + k) * g.ty + tr;
    const int nr = A.n_runs[kslot];
    uint8_t* out = E.payload + A.payload_off[grp];
    long long pos = A.chain_off[kslot];
    for (int base = 0; base < nr; base += 32) {
        int j = base + lane;
        int size = 0;
        const uint8_t* okv = nullptr;
        if (j < nr) {
            okv = E.ref_ok + (kc * g.tx + j) * n;
            int present = 0;
            for (int c = 0; c < n; ++c) present += (c != k) && okv[c];
            size = 18 + pm + 4 * present;
        }
        int inc = warp_incl_scan(size);
        if (j < nr) {
            uint8_t* o = out + pos + inc - size;
            const long long ri = kslot * g.tx + j;
            put_u16(o, tr);
            put_u16(o + 2, E.run_s[ri]);
            put_u16(o + 4, E.run_len[ri]);
            put_f32(o + 6, E.run_abc[3 * ri]);
            put_f32(o + 10, E.run_abc[3 * ri + 1]);
            put_f32(o + 14, E.run_abc[3 * ri + 2]);
            uint8_t* bits = o + 18;
            for (int b = 0; b < pm; ++b) bits[b] = 0;
            const float* cv = E.ref_c + (kc * g.tx + j) * n;
            int q = 0;
            for (int c = 0; c < n; ++c) {
                bool pres = (c == k) || okv[c];
                if (pres) bits[c >> 3] |= (uint8_t)(1u << (c & 7));
                if (pres && c != k) put_f32(o + 18 + pm + 4 * q++, cv[c]);
            }
        }
        pos += __shfl_sync(STPC_FULL, inc, 31);
    }
}

// fallback rows: warp per P chain
__global__ void __launch_bounds__(128) emit_fallback_kernel(EmitArgs E)
{
    const PlanArgs& A = E.p;
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long F = (long long)A.n_groups * A.n;
    if (wid >= F * g.ty) return;
    const long long f = wid / g.ty;
    const int tr = (int)(wid % g.ty);
    const int grp = (int)(f / A.n), i = (int)(f % A.n);
    if (i == A.k) return;
    const int nr = A.n_runs[wid];
    if (nr == 0) return;
    uint8_t* o = E.payload + A.payload_off[grp] + A.chain_off[wid];
    if (lane == 0) {
        put_u16(o, tr);
        put_u16(o + 2, nr);
    }
    for (int j = lane; j < nr; j += 32) {
        const long long ri = wid * g.tx + j;
        uint8_t* r = o + 4 + 16LL * j;
        put_u16(r, E.run_s[ri]);
        put_u16(r + 2, E.run_len[ri]);
        put_f32(r + 4, E.run_abc[3 * ri]);
        put_f32(r + 8, E.run_abc[3 * ri + 1]);
        put_f32(r + 12, E.run_abc[3 * ri + 2]);
    }
}

// residual rows: warp per (frame, row) with residual pixels.  Lane per bitmap
// word for the class masks (32 words at a time), then the emission is
// transposed to lane per pixel, one word at a time: the previous residual
// index comes from the word mask, varint offsets from a warp scan and code /
// escape slots from popcounts, so every byte, code, escape store and range
// load of the warp is coalesced.
#ifndef STPC_EMIT_MINB
#define STPC_EMIT_MINB 8  // measured: 1 -> 5.14 ms, 6 -> 4.08, 8 -> 3.82 (latency-bound)
#endif
__global__ void __launch_bounds__(256, STPC_EMIT_MINB) emit_residual_kernel(EmitArgs E)
{
    const PlanArgs& A = E.p;
    const Geometry& g = A.g;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long F = (long long)A.n_groups * A.n;
    if (wid >= F * g.h) return;
    const RowStat st = A.rowstat[wid];
    if (st.cnt == 0) return;
    const RowOff ro = A.rowoff[wid];
    const long long f = wid / g.h;
    const int v = (int)(wid % g.h);
    const int grp = (int)(f / A.n), i = (int)(f % A.n);
    const long long* sec = A.sec + (long long)grp * (2 + 2 * A.n);
    uint8_t* base = E.payload + A.payload_off[grp] + sec[2 + A.n + i] + 4;
    const long long total = A.res_cnt[f];
    uint8_t* vptr = base + ro.vb_off;
    uint8_t* cptr = base + A.res_vb[f] + 2LL * ro.cnt_off;
    uint8_t* eptr = base + A.res_vb[f] + 2 * total + 4 + 4LL * ro.esc_off;
    const uint8_t* vb = A.vbits + f * g.pbs;
    const uint8_t* eb = A.ebits + f * g.pbs;
    const uint8_t* crow = A.cls + (f * g.ty + v / g.th) * g.tx;
    const double* img = E.best + f * g.P;
    RowWalk rw = row_walk(g, v);
    long long last = ro.prev;  // previous residual of the frame (0 if none)
    for (long long wbase = rw.w0; wbase < rw.w1; wbase += 32) {
        const long long wd = wbase + lane;
        uint32_t res = 0, tmp, fb, esc = 0;
        if (wd < rw.w1) {
            word_classes(g, crow, load_bits(vb, wd), rw.rb, rw.re, wd, res, tmp, fb);
            if (res) esc = load_bits(eb, wd) & res;
        }
        unsigned todo = __ballot_sync(STPC_FULL, res != 0);
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t m = __shfl_sync(STPC_FULL, res, j);
            const uint32_t em = __shfl_sync(STPC_FULL, esc, j);
            const long long w0px = (wbase + j) * 32;
            const bool has = (m >> lane) & 1u;
            const uint32_t below = m & lt;
            const long long prev = below ? w0px + (31 - __clz(below)) : last;
            const long long idx = w0px + lane;
            uint32_t d = (uint32_t)(idx - prev);
            const int len = has ? varint_len(d) : 0;
            // one-byte deltas everywhere (dense residual words): the varint
            // offsets are a popcount, not a scan
            const int vinc = __all_sync(STPC_FULL, len <= 1) ? __popc(m & (lt | (1u << lane)))
                                                             : warp_incl_scan(len);
            if (has) {
                uint8_t* vo = vptr + (vinc - len);
                while (d >= 0x80u) {
                    *vo++ = (uint8_t)((d & 0x7f) | 0x80);
                    d >>= 7;
                }
                *vo = (uint8_t)d;
                const double r = img[idx];
                uint32_t code = 0xFFFFu;
                if ((em >> lane) & 1u) {
                    put_f32(eptr + 4 * __popc(em & lt), (float)r);
                } else {
                    // rint(r / q) (bitstream.py:178): reciprocal estimate, exact
                    // IEEE division only when the estimate is near a .5 boundary
                    const double qa = r * E.inv_quant;
                    const double fr = qa - floor(qa);
                    code = fabs(fr - 0.5) > 1e-6 ? (uint32_t)(long long)rint(qa)
                                                 : (uint32_t)(long long)rint(r / E.range_quant);
                }
                put_u16(cptr + 2 * __popc(below), code);
            }
            vptr += __shfl_sync(STPC_FULL, vinc, 31);
            cptr += 2 * __popc(m);
            eptr += 4 * __popc(em);
            last = w0px + (31 - __clz(m));
        }
    }
}

// Compacted variant: per batch of 32 bitmap words (lane per word for the
// class masks, as above), the batch's residual pixels are first listed in
// shared memory in pixel order (10-bit offset within the batch, escape flag
// in bit 15), then emitted lane per *residual pixel*, 32 at a time -- every
// lane of the varint / range-load / code / escape stores does useful work,
// instead of one lane per pixel slot of a word (~1/3 residual on the bench
// workload).
constexpr int EC_WARPS = 8;
#ifndef STPC_EMITC_MINB
#define STPC_EMITC_MINB 6  // measured with the range loads issued a round ahead: 4 -> 3.38 ms, 5 -> 3.11, 6 -> 2.98, 7 -> 3.50, 8 -> 3.61 (without: 8 -> 3.26, 6 -> 3.20)
#endif
__global__ void __launch_bounds__(EC_WARPS * 32, STPC_EMITC_MINB) emit_residual_compact_kernel(EmitArgs E)
{
    const PlanArgs& A = E.p;
    const Geometry& g = A.g;
    __shared__ uint16_t s_list[EC_WARPS][1024];
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    uint16_t* list = s_list[threadIdx.x >> 5];
    const long long wid = (long long)blockIdx.x * EC_WARPS + (threadIdx.x >> 5);
    const long long F = (long long)A.n_groups * A.n;
    if (wid >= F * g.h) return;
    const RowStat st = A.rowstat[wid];
    if (st.cnt == 0) return;
    const RowOff ro = A.rowoff[wid];
    const long long f = wid / g.h;
    const int v = (int)(wid % g.h);
    const int grp = (int)(f / A.n), i = (int)(f % A.n);
    const long long* sec = A.sec + (long long)grp * (2 + 2 * A.n);
    uint8_t* base = E.payload + A.payload_off[grp] + sec[2 + A.n + i] + 4;
    const long long total = A.res_cnt[f];
    uint8_t* vptr = base + ro.vb_off;
    uint8_t* cptr = base + A.res_vb[f] + 2LL * ro.cnt_off;
    uint8_t* eptr = base + A.res_vb[f] + 2 * total + 4 + 4LL * ro.esc_off;
    const uint8_t* vb = A.vbits + f * g.pbs;
    const uint8_t* eb = A.ebits + f * g.pbs;
    const uint8_t* crow = A.cls + (f * g.ty + v / g.th) * g.tx;
    const double* img = E.best + f * g.P;
    RowWalk rw = row_walk(g, v);
    int last = ro.prev;  // previous residual of the frame (0 if none); pixel indices fit 32 bits (P < 2^31)
    for (long long wbase = rw.w0; wbase < rw.w1; wbase += 32) {
        const long long wd = wbase + lane;
        uint32_t res = 0, tmp, fb, esc = 0;
        if (wd < rw.w1) {
            word_classes(g, crow, load_bits(vb, wd), rw.rb, rw.re, wd, res, tmp, fb);
            if (res) esc = load_bits(eb, wd) & res;
        }
        const int cnt = __popc(res);
        const int incl = warp_incl_scan(cnt);
        const int n = __shfl_sync(STPC_FULL, incl, 31);
        if (n == 0) continue;
        // list the batch's residual pixels in order
        unsigned todo = __ballot_sync(STPC_FULL, res != 0);
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t m = __shfl_sync(STPC_FULL, res, j);
            const uint32_t em = __shfl_sync(STPC_FULL, esc, j);
            const int o = __shfl_sync(STPC_FULL, incl - cnt, j);
            if ((m >> lane) & 1u)
                list[o + __popc(m & lt)] = (uint16_t)((j * 32 + lane) | (((em >> lane) & 1u) << 15));
        }
        __syncwarp();
        // emit them, lane per residual pixel
        const int p0 = (int)(wbase * 32);
        // the ranges are scattered DRAM reads: each round's load is issued a
        // round ahead, so its latency hides behind the previous round's stores
        unsigned e_n = lane < n ? list[lane] : 0u;
        double r_n = lane < n ? img[p0 + (e_n & 1023u)] : 0.0;
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            const bool act = k < n;
            const int na = min(32, n - k0);
            const unsigned e = e_n;
            const double r = r_n;
            if (k0 + 32 < n) {
                const bool an = k + 32 < n;
                e_n = an ? list[k + 32] : 0u;
                r_n = an ? img[p0 + (e_n & 1023u)] : 0.0;
            }
            const int idx = p0 + (int)(e & 1023u);
            const bool isesc = act && (e >> 15);
            const int pl = __shfl_up_sync(STPC_FULL, idx, 1);
            const int prev = lane == 0 ? last : pl;
            uint32_t d = (uint32_t)(idx - prev);
            const int len = act ? varint_len(d) : 0;
            // one-byte deltas everywhere: the offsets are the lane numbers
            const int vinc = __all_sync(STPC_FULL, len <= 1) ? lane + 1 : warp_incl_scan(len);
            const unsigned eball = __ballot_sync(STPC_FULL, isesc);
            if (act) {
                uint8_t* vo = vptr + (vinc - len);
                while (d >= 0x80u) {
                    *vo++ = (uint8_t)((d & 0x7f) | 0x80);
                    d >>= 7;
                }
                *vo = (uint8_t)d;
                uint32_t code = 0xFFFFu;
                if (isesc) {
                    put_f32(eptr + 4 * __popc(eball & lt), (float)r);
                } else {
                    // rint(r / q) (bitstream.py:178): reciprocal estimate, exact
                    // IEEE division only when the estimate is near a .5 boundary
                    const double qa = r * E.inv_quant;
                    const double fr = qa - floor(qa);
                    code = fabs(fr - 0.5) > 1e-6 ? (uint32_t)(long long)rint(qa)
                                                 : (uint32_t)(long long)rint(r / E.range_quant);
                }
                put_u16(cptr + 2 * lane, code);
            }
            vptr += __shfl_sync(STPC_FULL, vinc, na - 1);
            cptr += 2 * na;
            eptr += 4 * __popc(eball);
            last = __shfl_sync(STPC_FULL, idx, na - 1);
        }
        __syncwarp();  // the list is rewritten by the next batch
    }
}

void launch_emit(const EmitArgs& E, cudaStream_t s)
{
    const PlanArgs& A = E.p;
    const Geometry& g = A.g;
    if (A.n_groups <= 0) return;
    const long long F = (long long)A.n_groups * A.n;
    STPC_LAUNCH();
    emit_header_kernel<<<A.n_groups, 128, 0, s>>>(E);
    STPC_LAUNCH();
    emit_bitmaps_kernel<<<(unsigned)F, 256, 0, s>>>(E);
    long long kwarps = (long long)A.n_groups * g.ty;
    STPC_LAUNCH();
    emit_temporal_kernel<<<(unsigned)((kwarps + 3) / 4), 128, 0, s>>>(E);
    long long fwarps = F * g.ty;
    STPC_LAUNCH();
    emit_fallback_kernel<<<(unsigned)((fwarps + 3) / 4), 128, 0, s>>>(E);
    long long rwarps = F * g.h;
    STPC_LAUNCH();
#ifndef STPC_EMIT_PERWORD
    emit_residual_compact_kernel<<<(unsigned)((rwarps + EC_WARPS - 1) / EC_WARPS), EC_WARPS * 32, 0, s>>>(E);
#else
    emit_residual_kernel<<<(unsigned)((rwarps + 7) / 8), 256, 0, s>>>(E);
#endif
}

}  // namespace stpc
