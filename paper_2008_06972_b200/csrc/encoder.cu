// Native runtime + C-ABI of libstpc_b200: owns the device workspace of a batch
// of K+P groups and sequences the hot-path kernels on one CUDA stream.
//
// Pipeline per call:
//   K1 convert -> bitmaps -> K2 fit (key frames) -> K3a refit -> K3b fit (P
//   frames, temporally covered tiles masked) -> residual row stats -> plan
//   [sync: payload sizes] -> payload emission -> histogram -> Huffman code
//   lengths [sync: blob sizes] -> bit packing -> CRC + header.
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>

#include <cmath>
#include "kernels.cuh"
#include "runtime.cuh"
#include "../../include/stpc_b200.h"

using namespace stpc;

unsigned long long stpc::g_launch_count = 0;

#ifdef STPC_GUARD
#include <mutex>
#include <set>
namespace {
std::mutex g_guard_mu;
std::set<DevBuf*> g_guard_bufs;
constexpr unsigned char GUARD_BYTE = 0xA5;

__global__ void guard_count_kernel(const unsigned char* p, long long n, unsigned long long* bad)
{
    unsigned long long c = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        c += p[i] != GUARD_BYTE;
    if (c) atomicAdd(bad, c);
}
}  // namespace

void stpc::guard_arm(DevBuf* b, size_t from)
{
    cudaDeviceSynchronize();
    if (b->cap > from) cudaMemset((char*)b->p + from, GUARD_BYTE, b->cap - from);
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(g_guard_mu);
    g_guard_bufs.insert(b);
}

void stpc::guard_forget(DevBuf* b)
{
    std::lock_guard<std::mutex> lk(g_guard_mu);
    g_guard_bufs.erase(b);
}

// Canary bytes changed past each live workspace's requested size; a report
// line per damaged buffer goes to `report`.
extern "C" int64_t stpc_debug_guard_check(char* report, int32_t cap)
{
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(g_guard_mu);
    unsigned long long* d_bad = nullptr;
    cudaMalloc(&d_bad, sizeof(unsigned long long));
    std::string rep;
    long long total = 0;
    for (DevBuf* b : g_guard_bufs) {
        if (!b->p || b->cap <= b->used) continue;
        cudaMemset(d_bad, 0, sizeof(unsigned long long));
        guard_count_kernel<<<148, 256>>>((const unsigned char*)b->p + b->used, (long long)(b->cap - b->used), d_bad);
        unsigned long long bad = 0;
        cudaMemcpy(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost);
        if (bad) {
            total += (long long)bad;
            rep += "buffer " + std::to_string((unsigned long long)(uintptr_t)b->p) + " used " + std::to_string(b->used) +
                   " cap " + std::to_string(b->cap) + ": " + std::to_string(bad) + " bytes past the end changed\n";
        }
    }
    cudaFree(d_bad);
    if (report && cap > 0) {
        strncpy(report, rep.c_str(), (size_t)cap - 1);
        report[cap - 1] = 0;
    }
    return cudaGetLastError() == cudaSuccess ? total : -1;
}

extern "C" int32_t stpc_debug_guard_buffers(void)
{
    std::lock_guard<std::mutex> lk(g_guard_mu);
    return (int32_t)g_guard_bufs.size();
}
#endif
static thread_local std::string g_err;
void stpc::set_last_error(const std::string& msg) { g_err = msg; }

// pipeline stages timed with CUDA events when profiling is enabled
enum Stage { ST_INIT, ST_CONVERT, ST_BITMAP, ST_START_K, ST_FIT_K, ST_REFIT, ST_START_P, ST_FIT_P,
             ST_PLAN, ST_EMIT, ST_HUFF, ST_PACK, ST_CRC, ST_COUNT };
static const char* kStageNames[ST_COUNT] = {"init", "convert", "bitmaps", "start_key", "fit_key", "refit",
                                            "start_p", "fit_p", "plan", "emit", "huffman", "pack", "crc"};

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            g_err = std::string(#x) + ": " + cudaGetErrorString(e_);                  \
            return STPC_ERR_CUDA;                                                     \
        }                                                                             \
    } while (0)


struct stpc_encoder {
    stpc_config cfg;
    Geometry g;
    int n, k;
    DevBuf trig;  // sin_t | cos_t | sin_p | cos_p
    DevBuf cfg_bytes;
    // inputs
    DevBuf pts, pt_off, xf;
    DevBuf q_count, q_idx, q_frame;  // convert's exact-path queue
    HostBuf h_stage;  // pinned staging: pt_off | xf
    // frame level.  The range grid is double-buffered: the pack kernel of a
    // call (which runs after the last reader of its grid) also +inf-fills the
    // other buffer with background stores, so the next call starts on a
    // prefilled grid; the last call's grid stays readable (STPC_BUF_BEST).
    DevBuf best2[2];
    int best_cur = 0, best_last = 0;
    long long best_filled[2] = {0, 0};  // +inf-filled elements (valid once ev_fill[i] completes)
    cudaEvent_t ev_fill[2] = {};
    DevBuf vbits, ebits, cls, fstats;
    // chain level
    DevBuf cert, start_ok, start_sums, chain_counter;
    DevBuf run_s, run_len, run_abc, n_runs, ref_ok, ref_c, chain_tbytes, chain_off;
    // plan
    DevBuf rowstat, rowoff, res_cnt, res_vb, res_esc, fb_rows, sec, payload_len, payload_off;
    DevBuf payload;
    // entropy
    DevBuf hist, lens, codes, enc_len, blob_off, chunk_bits, seg_crc, blobs;
    // last result (host)
    int G = 0;
    std::vector<long long> h_payload_len, h_blob_off, h_enc_len;
    HostBuf h_sizes;
    // chunked host pipeline (stpc_encode_host)
    DevBuf pts2[2];
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_done[2] = {};
    bool host_result = false;            // last result assembled on the host
    HostBuf gstage[2];                   // pinned gather staging (stpc_encode_host_gather)
    HostBuf hout;                        // encoder-owned pinned blob arena (gather path)
    bool own_host_blobs = false;         // last host result lives in hout
    std::vector<long long> acc_payload;  // per group raw payload lengths
    HostBuf acc_stats;                   // pinned [F][FS_COUNT]
    // high-priority stream for the key-frame fit; the P-frame start verdicts
    // run beside it on the caller's stream (see encode_impl)
    cudaStream_t hi = nullptr;
    cudaEvent_t ev_hi_in = nullptr, ev_hi_out = nullptr, ev_ovl[5] = {};
    // profiling
    int profile = 0;
    cudaEvent_t ev[ST_COUNT + 1] = {};
    double stage_ms[ST_COUNT] = {};
    long long profiled_calls = 0;
    ~stpc_encoder()
    {
        for (auto& x : ev)
            if (x) cudaEventDestroy(x);
        for (int i = 0; i < 2; ++i) {
            if (ev_h2d[i]) cudaEventDestroy(ev_h2d[i]);
            if (ev_done[i]) cudaEventDestroy(ev_done[i]);
        }
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (hi) cudaStreamDestroy(hi);
        for (cudaEvent_t x : {ev_hi_in, ev_hi_out, ev_ovl[0], ev_ovl[1], ev_ovl[2], ev_ovl[3], ev_ovl[4]})
            if (x) cudaEventDestroy(x);
        for (auto& x : ev_fill)
            if (x) cudaEventDestroy(x);
    }
    void mark(int st, cudaStream_t s)
    {
        if (profile) cudaEventRecord(ev[st], s);
    }
};

static Trig trig_of(const stpc_encoder* e)
{
    const double* t = e->trig.as<double>();
    Trig tg;
    tg.sin_t = t;
    tg.cos_t = t + e->g.w;
    tg.sin_p = t + 2 * e->g.w;
    tg.cos_p = t + 2 * e->g.w + e->g.h;
    return tg;
}

// config block of the payload: struct.pack("<Bd HH ddd II HH d", ...)
// (/root/reference/pkg/src/stpc/bitstream.py:142-157)
static void pack_config(const stpc_config& c, uint8_t out[57])
{
    size_t o = 0;
    auto put = [&](const void* p, size_t n) {
        memcpy(out + o, p, n);
        o += n;
    };
    uint8_t mode = (uint8_t)c.mode;
    uint16_t tw = (uint16_t)c.tile_w, th = (uint16_t)c.tile_h;
    uint32_t w = (uint32_t)c.w, h = (uint32_t)c.h;
    uint16_t nf = (uint16_t)c.n_frames, ki = (uint16_t)c.k_index;
    put(&mode, 1);
    put(&c.tau, 8);
    put(&tw, 2);
    put(&th, 2);
    put(&c.theta_r, 8);
    put(&c.phi_r, 8);
    put(&c.phi_offset, 8);
    put(&w, 4);
    put(&h, 4);
    put(&nf, 2);
    put(&ki, 2);
    put(&c.range_quant, 8);
}

extern "C" {

const char* stpc_last_error(void) { return g_err.c_str(); }
const char* stpc_version(void) { return "stpc_b200 0.1 (sm_100a)"; }

int stpc_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int stpc_malloc(void** dev_ptr, int64_t bytes)
{
    if (!dev_ptr || bytes < 0) return STPC_ERR_ARG;
    CK(cudaMalloc(dev_ptr, (size_t)std::max<int64_t>(bytes, 1)));
    return STPC_OK;
}

int stpc_free(void* dev_ptr)
{
    if (dev_ptr) CK(cudaFree(dev_ptr));
    return STPC_OK;
}

int stpc_memcpy_d2h(void* dst, const void* src, int64_t bytes)
{
    if (bytes <= 0) return STPC_OK;
    CK(cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost));
    return STPC_OK;
}

int stpc_memcpy_h2d(void* dst, const void* src, int64_t bytes)
{
    if (bytes <= 0) return STPC_OK;
    CK(cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyHostToDevice));
    return STPC_OK;
}

int stpc_encoder_create(const stpc_config* cfg, const double* sin_theta, const double* cos_theta,
                        const double* sin_phi, const double* cos_phi, stpc_encoder** out)
{
    if (!cfg || !out || !sin_theta || !cos_theta || !sin_phi || !cos_phi) {
        g_err = "null argument";
        return STPC_ERR_ARG;
    }
    const stpc_config& c = *cfg;
    if (c.w < 1 || c.h < 1 || c.tile_w < 1 || c.tile_h < 1 || c.n_frames < 1 || c.k_index < 0 ||
        c.k_index >= c.n_frames || !(c.tau > 0) || !(c.range_quant > 0)) {
        g_err = "invalid config";
        return STPC_ERR_ARG;
    }
    int tx = (c.w + c.tile_w - 1) / c.tile_w, ty = (c.h + c.tile_h - 1) / c.tile_h;
    if (tx > 0xFFFF || ty > 0xFFFF) {
        g_err = "tile grid exceeds the format's u16 indices";
        return STPC_ERR_ARG;
    }
    stpc_encoder* e = new stpc_encoder();
    e->cfg = c;
    e->n = c.n_frames;
    e->k = c.k_index;
    Geometry& g = e->g;
    g.w = c.w;
    g.h = c.h;
    g.tw = c.tile_w;
    g.th = c.tile_h;
    g.tx = tx;
    g.ty = ty;
    g.P = (long long)c.w * c.h;
    long long pb = (g.P + 7) / 8;
    g.pbs = (int)((pb + 127) / 128 * 128);
    g.theta_r = c.theta_r;
    g.phi_r = c.phi_r;
    g.phi_offset = c.phi_offset;
    int rc = e->trig.ensure(sizeof(double) * (2 * c.w + 2 * c.h));
    if (!rc) rc = e->cfg_bytes.ensure(64);
    if (rc) {
        delete e;
        return rc;
    }
    double* t = e->trig.as<double>();
    cudaMemcpy(t, sin_theta, sizeof(double) * c.w, cudaMemcpyHostToDevice);
    cudaMemcpy(t + c.w, cos_theta, sizeof(double) * c.w, cudaMemcpyHostToDevice);
    cudaMemcpy(t + 2 * c.w, sin_phi, sizeof(double) * c.h, cudaMemcpyHostToDevice);
    cudaMemcpy(t + 2 * c.w + c.h, cos_phi, sizeof(double) * c.h, cudaMemcpyHostToDevice);
    uint8_t cb[57];
    pack_config(c, cb);
    cudaError_t ce = cudaMemcpy(e->cfg_bytes.p, cb, 57, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
        g_err = std::string("encoder upload: ") + cudaGetErrorString(ce);
        delete e;
        return STPC_ERR_CUDA;
    }
    *out = e;
    return STPC_OK;
}

void stpc_encoder_destroy(stpc_encoder* enc) { delete enc; }

#define ENS(buf, bytes)                    \
    do {                                   \
        int r_ = (buf).ensure(bytes);      \
        if (r_) return r_;                 \
    } while (0)

// d_off/d_xf: the same offsets/transforms already in device memory (the
// pipelined host path uploads them once, so no H2D is queued behind the big
// point copies), or nullptr to upload here.
static int encode_impl(stpc_encoder* e, int G, const void* d_points, const int64_t* h_off,
                       const double* h_xf, cudaStream_t s, const long long* d_off = nullptr,
                       const double* d_xf = nullptr)
{
    const Geometry& g = e->g;
    const int n = e->n, k = e->k;
    const long long F = (long long)G * n;
    const long long TT = (long long)g.tx * g.ty;
    // the chain kernels index a batch's tiles with 32-bit offsets
    if (F * TT >= (1LL << 32)) return STPC_ERR_ARG;
    // the refit indexes the pixels of one group's frames with 32-bit offsets
    if ((long long)n * g.P >= (1LL << 31)) return STPC_ERR_ARG;
    e->mark(ST_INIT, s);
    // --- inputs (offsets + transforms through pinned staging)
    long long max_pts = 0;
    for (long long f = 0; f < F; ++f) max_pts = std::max<long long>(max_pts, h_off[f + 1] - h_off[f]);
    const long long* dev_off = d_off;
    const double* dev_xf = d_xf;
    if (!dev_off) {
        ENS(e->h_stage, sizeof(long long) * (F + 1) + sizeof(double) * 12 * F);
        long long* st_off = e->h_stage.as<long long>();
        double* st_xf = reinterpret_cast<double*>(st_off + F + 1);
        for (long long f = 0; f <= F; ++f) st_off[f] = h_off[f];
        memcpy(st_xf, h_xf, sizeof(double) * 12 * F);
        ENS(e->pt_off, sizeof(long long) * (F + 1));
        ENS(e->xf, sizeof(double) * 12 * F);
        CK(cudaMemcpyAsync(e->pt_off.p, st_off, sizeof(long long) * (F + 1), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(e->xf.p, st_xf, sizeof(double) * 12 * F, cudaMemcpyHostToDevice, s));
        dev_off = e->pt_off.as<long long>();
        dev_xf = e->xf.as<double>();
    }
    // --- workspace
    const int bi = e->best_cur;
    DevBuf& best = e->best2[bi];
    // both grids sized to an even element count: the pack kernels' prefill
    // of the other grid stores 16 bytes at a time
    const long long PE = (F * g.P + 1) / 2 * 2;
    {
        void* before = best.p;
        ENS(best, sizeof(double) * PE);
        if (best.p != before) e->best_filled[bi] = 0;
    }
    ENS(e->vbits, (size_t)F * g.pbs);
    ENS(e->ebits, (size_t)F * g.pbs);
    ENS(e->cls, (size_t)F * TT);
    ENS(e->fstats, sizeof(long long) * F * FS_COUNT);
    ENS(e->run_s, sizeof(uint16_t) * F * TT);
    ENS(e->run_len, sizeof(uint16_t) * F * TT);
    ENS(e->run_abc, sizeof(float) * 3 * F * TT);
    ENS(e->n_runs, sizeof(int) * F * g.ty);
    ENS(e->cert, sizeof(float4) * CERT_F4 * F * TT);
    ENS(e->start_ok, (size_t)F * TT);
    const bool keep_sums = g.tw * g.th <= 16;  // the pair chains take a start's sums from its verdict
    if (keep_sums) ENS(e->start_sums, sizeof(double) * 9 * F * TT);
    ENS(e->chain_counter, 64);
    ENS(e->ref_ok, (size_t)G * TT * n);
    ENS(e->ref_c, sizeof(float) * G * TT * n);
    ENS(e->chain_tbytes, sizeof(long long) * G * g.ty);
    ENS(e->chain_off, sizeof(long long) * F * g.ty);
    ENS(e->rowstat, sizeof(RowStat) * F * g.h);
    ENS(e->rowoff, sizeof(RowOff) * F * g.h);
    ENS(e->res_cnt, sizeof(long long) * F);
    ENS(e->res_vb, sizeof(long long) * F);
    ENS(e->res_esc, sizeof(long long) * F);
    ENS(e->fb_rows, sizeof(long long) * F);
    ENS(e->sec, sizeof(long long) * G * (2 + 2 * n));
    ENS(e->payload_len, sizeof(long long) * G);
    ENS(e->payload_off, sizeof(long long) * (G + 1));
    ENS(e->hist, sizeof(unsigned) * 256 * G);
    ENS(e->lens, 256 * (size_t)G);
    ENS(e->codes, sizeof(unsigned) * 256 * G);
    ENS(e->enc_len, sizeof(long long) * G);
    ENS(e->blob_off, sizeof(long long) * (G + 1));
    ENS(e->h_sizes, sizeof(long long) * (3 * G + 2));

    launch_zero(e->fstats.p, sizeof(long long) * F * FS_COUNT, s);
    launch_zero(e->cls.p, (long long)F * TT, s);
    if (e->best_filled[bi] >= F * g.P) {
        CK(cudaStreamWaitEvent(s, e->ev_fill[bi], 0));  // prefilled during the previous call's entropy stage
    } else {
        launch_fill_u64(best.as<unsigned long long>(), 0x7ff0000000000000ull, F * g.P, s);
    }
    e->best_filled[bi] = 0;  // consumed by this call

    e->mark(ST_CONVERT, s);
    // --- K1
    ConvertArgs ca;
    ca.pts = d_points;
    ca.pts_f64 = e->cfg.points_f64;
    ca.pt_off = dev_off;
    ca.xf = dev_xf;
    ca.n_frames = (int)F;
    ca.g = g;
    ca.best = best.as<unsigned long long>();
    ca.win = nullptr;
    ca.fstats = e->fstats.as<long long>();
    {
        long long npts = h_off[F] - h_off[0];
        long long cap = npts / 8 + 4096;
        ENS(e->q_count, CONVERT_QCOUNT_BYTES);
        ENS(e->q_idx, sizeof(long long) * cap);
        ENS(e->q_frame, sizeof(int) * cap);
        ca.q_count = e->q_count.as<unsigned long long>();
        ca.q_idx = e->q_idx.as<long long>();
        ca.q_frame = e->q_frame.as<int>();
        ca.q_cap = cap;
    }
    launch_convert(ca, (int)max_pts, s);
    e->mark(ST_BITMAP, s);
    launch_bitmaps(best.as<double>(), (int)F, g, e->cfg.range_quant, e->vbits.as<uint8_t>(),
                   e->ebits.as<uint8_t>(), e->fstats.as<long long>(), s);

    // --- K2 / K3a / K3b
    Trig tg = trig_of(e);
    FitArgs fa;
    fa.best = best.as<double>();
    fa.tg = tg;
    fa.g = g;
    fa.tau = e->cfg.tau;
    fa.r_max = e->cfg.r_max;
    fa.cond_limit = e->cfg.cond_limit;
    fa.ybias = std::exp2(std::ceil(std::log2(std::max(fa.r_max, 1.0))) + 1.0);  // power of two >= 2 r_max
    fa.n_frames_group = n;
    fa.k = k;
    fa.mode = 0;
    fa.n_jobs = G;
    fa.cls = e->cls.as<uint8_t>();
    fa.run_s = e->run_s.as<uint16_t>();
    fa.run_len = e->run_len.as<uint16_t>();
    fa.run_abc = e->run_abc.as<float>();
    fa.n_runs = e->n_runs.as<int>();
    fa.cert = e->cert.as<float4>();
    fa.start_ok = e->start_ok.as<uint8_t>();
    fa.start_sums = g.tw * g.th <= 16 ? e->start_sums.as<double>() : nullptr;
    fa.sums_stride = F * TT;
    fa.chain_counter = e->chain_counter.as<unsigned>();
    RefitArgs ra;
    ra.best = best.as<double>();
    ra.tg = tg;
    ra.g = g;
    ra.tau = fa.tau;
    ra.r_max = fa.r_max;
    ra.n = n;
    ra.k = k;
    ra.n_groups = G;
    ra.run_s = fa.run_s;
    ra.run_len = fa.run_len;
    ra.run_abc = fa.run_abc;
    ra.n_runs = fa.n_runs;
    ra.ref_ok = e->ref_ok.as<uint8_t>();
    ra.ref_c = e->ref_c.as<float>();
    ra.cls = fa.cls;
    ra.chain_tbytes = e->chain_tbytes.as<long long>();

#ifndef STPC_SERIAL_FIT
    // The key-frame fit leaves part of the GPU idle in its last wave of
    // chains.  It runs on a high-priority stream, and the P-frame start
    // verdicts -- which need only the P grids (a tile that the refit later
    // covers is masked by its class in fit_p's scan) -- run beside it on the
    // caller's stream, filling the idle slots.  Joined before the refit, the
    // first writer of P-frame pixels and classes.  (Running the refit on the
    // high-priority stream too starved the verdicts: 143.6k vs 145.3k
    // frames/s; without priorities the two kernels only time-share.)
    const bool ovl = n > 1 && fit_overlap_pays(g, (long long)G * g.ty);
#else
    const bool ovl = false;
#endif
    if (ovl) {
        if (!e->hi) {
            int least = 0, greatest = 0;
            CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            CK(cudaStreamCreateWithPriority(&e->hi, cudaStreamNonBlocking, greatest));
            CK(cudaEventCreateWithFlags(&e->ev_hi_in, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&e->ev_hi_out, cudaEventDisableTiming));
            for (auto& x : e->ev_ovl) CK(cudaEventCreate(&x));
        }
        CK(cudaEventRecord(e->ev_hi_in, s));
        CK(cudaStreamWaitEvent(e->hi, e->ev_hi_in, 0));
        if (e->profile) cudaEventRecord(e->ev_ovl[0], e->hi);
        launch_start_tiles(fa, e->hi);
        if (e->profile) cudaEventRecord(e->ev_ovl[1], e->hi);
        launch_fit_chains(fa, e->hi);
        if (e->profile) cudaEventRecord(e->ev_ovl[2], e->hi);
        CK(cudaEventRecord(e->ev_hi_out, e->hi));
        e->mark(ST_START_K, s);
        FitArgs fp = fa;
        fp.mode = 1;
        fp.n_jobs = G * (n - 1);
        if (e->profile) cudaEventRecord(e->ev_ovl[3], s);
        launch_start_tiles(fp, s);
        if (e->profile) cudaEventRecord(e->ev_ovl[4], s);
        e->mark(ST_FIT_K, s);
        CK(cudaStreamWaitEvent(s, e->ev_hi_out, 0));
    } else {
        e->mark(ST_START_K, s);
        launch_start_tiles(fa, s);
        e->mark(ST_FIT_K, s);
        launch_fit_chains(fa, s);
    }

    e->mark(ST_REFIT, s);
    launch_refit(ra, s);

    e->mark(ST_START_P, s);
    if (n > 1) {
        fa.mode = 1;
        fa.n_jobs = G * (n - 1);
        if (!ovl) launch_start_tiles(fa, s);
    }
    e->mark(ST_FIT_P, s);
    if (n > 1) launch_fit_chains(fa, s);

    e->mark(ST_PLAN, s);
    // --- residual stats + plan
    PlanArgs pa;
    pa.g = g;
    pa.n = n;
    pa.k = k;
    pa.n_groups = G;
    pa.vbits = e->vbits.as<uint8_t>();
    pa.ebits = e->ebits.as<uint8_t>();
    pa.cls = fa.cls;
    pa.n_runs = fa.n_runs;
    pa.chain_tbytes = ra.chain_tbytes;
    pa.rowstat = e->rowstat.as<RowStat>();
    pa.rowoff = e->rowoff.as<RowOff>();
    pa.fstats = e->fstats.as<long long>();
    pa.res_cnt = e->res_cnt.as<long long>();
    pa.res_vb = e->res_vb.as<long long>();
    pa.res_esc = e->res_esc.as<long long>();
    pa.fb_rows = e->fb_rows.as<long long>();
    pa.chain_off = e->chain_off.as<long long>();
    pa.sec = e->sec.as<long long>();
    pa.payload_len = e->payload_len.as<long long>();
    pa.payload_off = e->payload_off.as<long long>();
    launch_rowstats(pa, s);
    launch_plan(pa, s);
    launch_group_scan(pa.payload_len, pa.payload_off, G, 16, 0, s);

    long long* hs = e->h_sizes.as<long long>();
    CK(cudaMemcpyAsync(hs, pa.payload_len, sizeof(long long) * G, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hs + G, pa.payload_off + G, sizeof(long long), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    e->h_payload_len.assign(hs, hs + G);
    long long payload_total = hs[G];
    long long max_payload = 0;
    for (int i = 0; i < G; ++i) max_payload = std::max(max_payload, hs[i]);

    e->mark(ST_EMIT, s);
    ENS(e->payload, (size_t)payload_total + 16);
    EmitArgs ea;
    ea.p = pa;
    ea.best = fa.best;
    ea.range_quant = e->cfg.range_quant;
    ea.inv_quant = 1.0 / e->cfg.range_quant;
    ea.cfg_bytes = e->cfg_bytes.as<uint8_t>();
    ea.xf = dev_xf;
    ea.run_s = fa.run_s;
    ea.run_len = fa.run_len;
    ea.run_abc = fa.run_abc;
    ea.ref_ok = ra.ref_ok;
    ea.ref_c = ra.ref_c;
    ea.payload = e->payload.as<uint8_t>();
    launch_emit(ea, s);
    e->mark(ST_HUFF, s);
    // --- entropy stage
    EntropyArgs en;
    en.G = G;
    en.payload = ea.payload;
    // this call's grid is dead after emit (the entropy stage never reads it):
    // the pack blocks +inf-fill the other buffer for the next call
    const int nb = 1 - bi;
    DevBuf& nxt_best = e->best2[nb];
    {
        void* before = nxt_best.p;
        ENS(nxt_best, sizeof(double) * PE);
        if (nxt_best.p != before) e->best_filled[nb] = 0;
    }
    en.prefill = nxt_best.as<unsigned long long>();
    en.prefill_n = PE;
    en.payload_off = pa.payload_off;
    en.payload_len = pa.payload_len;
    en.hist = e->hist.as<unsigned>();
    en.lens = e->lens.as<uint8_t>();
    en.codes = e->codes.as<unsigned>();
    en.enc_len = e->enc_len.as<long long>();
    en.blob_off = e->blob_off.as<long long>();
    en.max_chunks = (int)((max_payload + PACK_CHUNK - 1) / PACK_CHUNK);
    launch_zero(en.hist, sizeof(unsigned) * 256 * G, s);
    launch_histogram(en, (int)max_payload, s);
    launch_code_lengths(en, s);
    launch_group_scan(en.enc_len, en.blob_off, G, 16, HDR, s);
    CK(cudaMemcpyAsync(hs, en.enc_len, sizeof(long long) * G, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hs + G, en.blob_off, sizeof(long long) * (G + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    e->h_enc_len.assign(hs, hs + G);
    e->h_blob_off.assign(hs + G, hs + 2 * G + 1);
    long long blob_total = e->h_blob_off[G];
    long long max_enc = 0;
    for (int i = 0; i < G; ++i) max_enc = std::max(max_enc, e->h_enc_len[i]);
    en.max_segs = (int)((max_enc + CRC_SEG - 1) / CRC_SEG);
    ENS(e->chunk_bits, sizeof(long long) * (size_t)G * std::max(en.max_chunks, 1));
    ENS(e->seg_crc, sizeof(unsigned) * (size_t)G * std::max(en.max_segs, 1));
    ENS(e->blobs, (size_t)blob_total + 16);
    en.chunk_bits = e->chunk_bits.as<long long>();
    en.seg_crc = e->seg_crc.as<unsigned>();
    en.blobs = e->blobs.as<uint8_t>();
    e->mark(ST_PACK, s);
    launch_pack(en, s);
    if (!e->ev_fill[0]) for (auto& x : e->ev_fill) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    CK(cudaEventRecord(e->ev_fill[nb], s));
    e->best_filled[nb] = en.max_chunks > 0 ? F * g.P : 0;  // pack ran: the next grid is +inf
    e->best_last = bi;
    e->best_cur = nb;
    e->mark(ST_CRC, s);
    launch_crc(en, s);
    CK(cudaGetLastError());
    e->G = G;
    e->host_result = false;
    if (e->profile) {
        cudaEventRecord(e->ev[ST_COUNT], s);
        CK(cudaEventSynchronize(e->ev[ST_COUNT]));
        for (int i = 0; i < ST_COUNT; ++i) {
            float ms = 0.f;
            cudaEvent_t a = e->ev[i], b = e->ev[i + 1];
            if (ovl && i == ST_START_K) a = e->ev_ovl[0], b = e->ev_ovl[1];  // overlapped stages: own events
            if (ovl && i == ST_FIT_K) a = e->ev_ovl[1], b = e->ev_ovl[2];
            if (ovl && i == ST_START_P) a = e->ev_ovl[3], b = e->ev_ovl[4];
            if (cudaEventElapsedTime(&ms, a, b) == cudaSuccess) e->stage_ms[i] += ms;
        }
        e->profiled_calls += 1;
    }
    return STPC_OK;
}

int stpc_encoder_profile(stpc_encoder* enc, int32_t enable)
{
    if (!enc) return STPC_ERR_ARG;
    if (enable && !enc->ev[0])
        for (auto& x : enc->ev) CK(cudaEventCreate(&x));
    enc->profile = enable ? 1 : 0;
    for (auto& m : enc->stage_ms) m = 0.0;
    enc->profiled_calls = 0;
    return STPC_OK;
}

int32_t stpc_encoder_stage_ms(const stpc_encoder* enc, double* ms, int32_t n)
{
    if (!enc || !ms) return 0;
    int m = n < ST_COUNT ? n : ST_COUNT;
    for (int i = 0; i < m; ++i) ms[i] = enc->stage_ms[i];
    return ST_COUNT;
}

const char* stpc_stage_name(int32_t i) { return (i >= 0 && i < ST_COUNT) ? kStageNames[i] : ""; }

uint64_t stpc_launch_count(void) { return stpc::g_launch_count; }

int stpc_encode_device(stpc_encoder* enc, int32_t n_groups, const void* d_points,
                       const int64_t* point_offsets, const double* transforms, void* stream)
{
    if (!enc || n_groups < 1 || !point_offsets || !transforms || (!d_points && point_offsets[(long long)n_groups * enc->n] > 0)) {
        g_err = "invalid arguments";
        return STPC_ERR_ARG;
    }
    if ((uintptr_t)d_points % (enc->cfg.points_f64 ? 8 : 4)) {
        g_err = "device points are not aligned to their element size";
        return STPC_ERR_ARG;
    }
    return encode_impl(enc, n_groups, d_points, (const int64_t*)point_offsets, transforms, (cudaStream_t)stream);
}

}  // extern "C"

// copy frames [f0, f1) (host pointers fptrs[f], counts from the offsets) to
// dst in order, frames spread over host threads
static void gather_frames(char* dst, const void* const* fptrs, const int64_t* point_offsets, long long f0,
                          long long f1, size_t esz)
{
    const long long nf = f1 - f0;
    if (nf <= 0) return;
    const unsigned nt = (unsigned)std::max<long long>(1, std::min<long long>(
        std::min<long long>(16, std::max(1u, std::thread::hardware_concurrency())), nf));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        th.emplace_back([=] {
            for (long long f = f0 + nf * t / nt; f < f0 + nf * (t + 1) / nt; ++f) {
                const long long cnt = point_offsets[f + 1] - point_offsets[f];
                if (cnt > 0)
                    memcpy(dst + esz * 3 * (point_offsets[f] - point_offsets[f0]), fptrs[f], esz * 3 * (size_t)cnt);
            }
        });
    }
    for (auto& x : th) x.join();
}

// Blob i of a host arena (src + offsets[i], lengths[i] bytes) to dst[i], the
// blobs spread over host threads by bytes.  The Python layer passes the
// buffers of freshly allocated bytes objects, so materialising a batch's
// blobs is one parallel copy instead of one serial copy per blob.
extern "C" int stpc_host_scatter(const uint8_t* src, const int64_t* offsets, const int64_t* lengths,
                                 uint8_t* const* dst, int32_t n)
{
    if (n < 0 || (n > 0 && (!src || !offsets || !lengths || !dst))) {
        g_err = "invalid arguments";
        return STPC_ERR_ARG;
    }
    long long total = 0;
    for (int i = 0; i < n; ++i) total += lengths[i];
    const unsigned nt = (unsigned)std::max<long long>(1, std::min<long long>(
        std::min<long long>(16, std::max(1u, std::thread::hardware_concurrency())), (total >> 20) + 1));
    if (nt == 1) {
        for (int i = 0; i < n; ++i)
            if (lengths[i] > 0) memcpy(dst[i], src + offsets[i], (size_t)lengths[i]);
        return STPC_OK;
    }
    // thread t copies the byte range [total t / nt, total (t+1) / nt) of the
    // concatenated blobs, split at blob boundaries inside the range
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        th.emplace_back([=] {
            const long long lo = total * t / nt, hi = total * (t + 1) / nt;
            long long pos = 0;
            for (int i = 0; i < n && pos < hi; ++i) {
                const long long b0 = pos, b1 = pos + lengths[i];
                pos = b1;
                const long long c0 = std::max(b0, lo), c1 = std::min(b1, hi);
                if (c1 > c0) memcpy(dst[i] + (c0 - b0), src + offsets[i] + (c0 - b0), (size_t)(c1 - c0));
            }
        });
    }
    for (auto& x : th) x.join();
    return STPC_OK;
}

// Host-memory encode.  Points come from one contiguous buffer (hp) or from
// per-frame pointers (fptrs, gathered into pinned staging).  Blobs go to
// h_out, or (own_out) to the encoder's pinned arena, or stay on the device.
static int encode_host_impl(stpc_encoder* enc, int32_t n_groups, const char* hp, const void* const* fptrs,
                            const int64_t* point_offsets, const double* transforms, uint8_t* h_out,
                            int64_t out_cap, void* stream, bool own_out)
{
    if (!enc || n_groups < 1 || !point_offsets || !transforms || (!hp && !fptrs)) {
        g_err = "invalid arguments";
        return STPC_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int n = enc->n;
    const long long F = (long long)n_groups * n;
    const size_t esz = enc->cfg.points_f64 ? sizeof(double) : sizeof(float);
    enc->own_host_blobs = false;
    // Small batches: one H2D + encode + D2H.
    // measured on the bench workload (1024 groups): 8 chunks 232.5 ms,
    // 16: 227.7, 24: 226.8, 32: 239.4 -- the tail (last chunk's encode + blob
    // D2H) shrinks with chunk size until per-chunk syncs and launches dominate;
    // re-measured after the fit trims: 16: 227.5, 24: 225.7, 32: 227.6
    int n_chunks = n_groups >= 384 ? 24 : n_groups >= 128 ? 16 : (n_groups >= 64 ? 8 : 1);
    if (n_chunks > 1 && getenv("STPC_PIPE_CHUNKS")) {  // tuning knob
        n_chunks = std::max(2, std::min(atoi(getenv("STPC_PIPE_CHUNKS")), n_groups / 8));
    }
    if (n_chunks == 1 || (!h_out && !own_out)) {
        long long npts = point_offsets[F] - point_offsets[0];
        ENS(enc->pts, esz * 3 * std::max<long long>(npts, 1));
        const char* src = hp ? hp + esz * 3 * point_offsets[0] : nullptr;
        if (!hp) {
            ENS(enc->gstage[0], esz * 3 * std::max<long long>(npts, 1));
            gather_frames(enc->gstage[0].as<char>(), fptrs, point_offsets, 0, F, esz);
            src = enc->gstage[0].as<char>();
        }
        if (npts > 0) CK(cudaMemcpyAsync(enc->pts.p, src, esz * 3 * npts, cudaMemcpyHostToDevice, s));
        std::vector<int64_t> off(point_offsets, point_offsets + F + 1);
        for (auto& o : off) o -= point_offsets[0];
        int rc = encode_impl(enc, n_groups, enc->pts.p, off.data(), transforms, s);
        if (rc) return rc;
        if (h_out) {
            rc = stpc_result_copy_blobs(enc, h_out, out_cap, stream);
            if (rc) return rc;
        }
        CK(cudaStreamSynchronize(s));
        return STPC_OK;
    }
    // Pipelined: the H2D of chunk c+1 (copy stream, double-buffered device
    // points) overlaps the encode and blob D2H of chunk c (stream s).
    if (!enc->copy_stream) {
        CK(cudaStreamCreateWithFlags(&enc->copy_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&enc->ev_h2d[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&enc->ev_done[i], cudaEventDisableTiming));
        }
    }
    const int gc = (n_groups + n_chunks - 1) / n_chunks;
    long long max_pts = 1;
    for (int c = 0; c < n_chunks; ++c) {
        int g0 = c * gc, g1 = std::min(n_groups, g0 + gc);
        if (g0 >= g1) break;
        max_pts = std::max<long long>(max_pts, point_offsets[(long long)g1 * n] - point_offsets[(long long)g0 * n]);
    }
    ENS(enc->pts2[0], esz * 3 * max_pts);
    ENS(enc->pts2[1], esz * 3 * max_pts);
    ENS(enc->acc_stats, sizeof(long long) * FS_COUNT * F);
    // all chunks' (rebased) offsets and transforms go up once, before the big
    // point copies, so encode_impl queues no H2D behind them
    ENS(enc->h_stage, sizeof(long long) * (F + n_chunks) + sizeof(double) * 12 * F);
    ENS(enc->pt_off, sizeof(long long) * (F + n_chunks));
    ENS(enc->xf, sizeof(double) * 12 * F);
    {
        long long* st_off = enc->h_stage.as<long long>();
        double* st_xf = reinterpret_cast<double*>(st_off + F + n_chunks);
        for (int c = 0; c < n_chunks; ++c) {
            const int g0 = c * gc, g1 = std::min(n_groups, g0 + gc);
            if (g0 >= g1) break;
            const long long f0 = (long long)g0 * n, f1 = (long long)g1 * n;
            for (long long f = f0; f <= f1; ++f) st_off[f + c] = point_offsets[f] - point_offsets[f0];
        }
        memcpy(st_xf, transforms, sizeof(double) * 12 * F);
        CK(cudaMemcpyAsync(enc->pt_off.p, st_off, sizeof(long long) * (F + n_chunks), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(enc->xf.p, st_xf, sizeof(double) * 12 * F, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    std::vector<long long> blob_off(n_groups + 1, 0), enc_len(n_groups, 0), payload(n_groups, 0);
    // gather (per-frame mode): host threads copy chunk c into pinned stage
    // c&1 once that stage's previous H2D (chunk c-2) has drained; runs on a
    // helper thread one chunk ahead, concurrently with encode_impl(c - 1)
    if (!hp) {
        ENS(enc->gstage[0], esz * 3 * max_pts);
        ENS(enc->gstage[1], esz * 3 * max_pts);
    }
    auto gather = [&](int c) -> int {
        const int b = c & 1;
        const int g0 = c * gc, g1 = std::min(n_groups, g0 + gc);
        if (c >= 2 && cudaEventSynchronize(enc->ev_h2d[b]) != cudaSuccess) return STPC_ERR_CUDA;
        auto gt0 = std::chrono::steady_clock::now();
        gather_frames(enc->gstage[b].as<char>(), fptrs, point_offsets, (long long)g0 * n, (long long)g1 * n, esz);
        if (getenv("STPC_PIPE_TRACE"))
            fprintf(stderr, "host: gather(%d) %.2f ms\n", c,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - gt0).count());
        return STPC_OK;
    };
    auto h2d = [&](int c) -> int {
        const int b = c & 1;
        const int g0 = c * gc, g1 = std::min(n_groups, g0 + gc);
        const long long p0 = point_offsets[(long long)g0 * n], p1 = point_offsets[(long long)g1 * n];
        CK(cudaStreamWaitEvent(enc->copy_stream, enc->ev_done[b], 0));
        const char* src = hp ? hp + esz * 3 * p0 : enc->gstage[b].as<char>();
        if (p1 > p0)
            CK(cudaMemcpyAsync(enc->pts2[b].p, src, esz * 3 * (p1 - p0), cudaMemcpyHostToDevice,
                               enc->copy_stream));
        CK(cudaEventRecord(enc->ev_h2d[b], enc->copy_stream));
        return STPC_OK;
    };
    auto chunk_ok = [&](int c) { return c < n_chunks && c * gc < n_groups; };
    std::thread helper;
    int helper_rc = STPC_OK;
    struct JoinGuard {
        std::thread& t;
        ~JoinGuard()
        {
            if (t.joinable()) t.join();
        }
    } join_guard{helper};
    auto join_helper = [&]() -> int {
        if (helper.joinable()) helper.join();
        return helper_rc;
    };
    // optional timeline (STPC_PIPE_TRACE=1): per chunk H2D end / encode end
    const bool trace = getenv("STPC_PIPE_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    cudaEvent_t t0 = nullptr;
    if (trace) {
        cudaEventCreate(&t0);
        cudaEventRecord(t0, s);
    }
    if (!hp) {
        int grc = gather(0);
        if (grc) return grc;
    }
    int rc = h2d(0);
    if (rc) return rc;
    if (trace) { tev.emplace_back(); cudaEventCreate(&tev.back()); cudaEventRecord(tev.back(), enc->copy_stream); }
    if (!hp && chunk_ok(1)) helper = std::thread([&] { helper_rc = gather(1); });
    long long out_pos = 0;
    if (own_out) ENS(enc->hout, (size_t)(esz * 3 * (point_offsets[F] - point_offsets[0]) / 6 + (1 << 20)));
    for (int c = 0; c < n_chunks; ++c) {
        const int g0 = c * gc, g1 = std::min(n_groups, g0 + gc);
        if (g0 >= g1) break;
        const int b = c & 1;
        if (chunk_ok(c + 1)) {
            auto hA = std::chrono::steady_clock::now();
            if (!hp) {
                rc = join_helper();
                if (rc) return rc;
            }
            rc = h2d(c + 1);
            if (!hp && !rc && chunk_ok(c + 2)) helper = std::thread([&, cc = c + 2] { helper_rc = gather(cc); });
            if (trace)
                fprintf(stderr, "host: h2d(%d) enqueue took %.2f ms\n", c + 1,
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hA).count());
            if (rc) return rc;
            if (trace) { tev.emplace_back(); cudaEventCreate(&tev.back()); cudaEventRecord(tev.back(), enc->copy_stream); }
        }
        CK(cudaStreamWaitEvent(s, enc->ev_h2d[b], 0));
        const long long f0 = (long long)g0 * n, f1 = (long long)g1 * n;
        std::vector<int64_t> off(point_offsets + f0, point_offsets + f1 + 1);
        for (auto& o : off) o -= point_offsets[f0];
        rc = encode_impl(enc, g1 - g0, enc->pts2[b].p, off.data(), transforms + 12 * f0, s,
                         enc->pt_off.as<long long>() + f0 + c, enc->xf.as<double>() + 12 * f0);
        if (rc) return rc;
        CK(cudaEventRecord(enc->ev_done[b], s));
        if (trace) { tev.emplace_back(); cudaEventCreate(&tev.back()); cudaEventRecord(tev.back(), s); }
        const long long total = enc->h_blob_off[g1 - g0];
        if (own_out && out_pos + total > (long long)enc->hout.cap) {
            // grow the encoder's arena, keeping the blobs already copied
            CK(cudaStreamSynchronize(s));
            HostBuf bigger;
            if (bigger.ensure((size_t)((out_pos + total) * 3 / 2 + (1 << 20)))) return STPC_ERR_NOMEM;
            if (out_pos > 0) memcpy(bigger.p, enc->hout.p, (size_t)out_pos);
            std::swap(bigger.p, enc->hout.p);
            std::swap(bigger.cap, enc->hout.cap);
        }
        uint8_t* out_base = own_out ? enc->hout.as<uint8_t>() : h_out;
        if (!own_out && out_pos + total > out_cap) {
            g_err = "output buffer too small";
            return STPC_ERR_ARG;
        }
        if (total > 0) CK(cudaMemcpyAsync(out_base + out_pos, enc->blobs.p, (size_t)total, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(enc->acc_stats.as<long long>() + FS_COUNT * f0, enc->fstats.p,
                           sizeof(long long) * FS_COUNT * (f1 - f0), cudaMemcpyDeviceToHost, s));
        for (int i = 0; i < g1 - g0; ++i) {
            blob_off[g0 + i] = out_pos + enc->h_blob_off[i];
            enc_len[g0 + i] = enc->h_enc_len[i];
            payload[g0 + i] = enc->h_payload_len[i];
        }
        out_pos += total;
    }
    blob_off[n_groups] = out_pos;
    CK(cudaStreamSynchronize(s));
    if (trace) {
        cudaDeviceSynchronize();
        for (size_t i = 0; i < tev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, t0, tev[i]);
            fprintf(stderr, "pipe ev %zu at %.2f ms\n", i, ms);
            cudaEventDestroy(tev[i]);
        }
        cudaEventDestroy(t0);
    }
    enc->G = n_groups;
    enc->h_blob_off = blob_off;
    enc->h_enc_len = enc_len;
    enc->h_payload_len = payload;
    enc->host_result = true;
    enc->own_host_blobs = own_out;
    return STPC_OK;
}

extern "C" {

int stpc_encode_host(stpc_encoder* enc, int32_t n_groups, const void* h_points,
                     const int64_t* point_offsets, const double* transforms, uint8_t* h_out,
                     int64_t out_cap, void* stream)
{
    if (!h_points) {
        g_err = "invalid arguments";
        return STPC_ERR_ARG;
    }
    return encode_host_impl(enc, n_groups, (const char*)h_points, nullptr, point_offsets, transforms, h_out,
                            out_cap, stream, false);
}

int stpc_encode_host_gather(stpc_encoder* enc, int32_t n_groups, const void* const* frame_points,
                            const int64_t* frame_counts, const double* transforms, void* stream)
{
    if (!enc || n_groups < 1 || !frame_points || !frame_counts) {
        g_err = "invalid arguments";
        return STPC_ERR_ARG;
    }
    const long long F = (long long)n_groups * enc->n;
    std::vector<int64_t> off(F + 1, 0);
    for (long long f = 0; f < F; ++f) {
        if (frame_counts[f] < 0 || (frame_counts[f] > 0 && !frame_points[f])) {
            g_err = "invalid frame";
            return STPC_ERR_ARG;
        }
        off[f + 1] = off[f] + frame_counts[f];
    }
    return encode_host_impl(enc, n_groups, nullptr, frame_points, off.data(), transforms, nullptr, 0, stream, true);
}

const uint8_t* stpc_result_host_blobs(const stpc_encoder* enc)
{
    return (enc && enc->host_result && enc->own_host_blobs) ? enc->hout.as<uint8_t>() : nullptr;
}

int stpc_encoder_wait(stpc_encoder* enc, void* stream)
{
    if (!enc) return STPC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (enc->ev_fill[enc->best_cur]) CK(cudaStreamWaitEvent(s, enc->ev_fill[enc->best_cur], 0));
    return STPC_OK;
}

int32_t stpc_result_groups(const stpc_encoder* enc) { return enc ? enc->G : 0; }

int stpc_result_blobs(const stpc_encoder* enc, int64_t* offsets, int64_t* lengths)
{
    if (!enc) return STPC_ERR_ARG;
    for (int i = 0; i < enc->G; ++i) {
        if (offsets) offsets[i] = enc->h_blob_off[i];
        if (lengths) lengths[i] = HDR + enc->h_enc_len[i];
    }
    if (offsets) offsets[enc->G] = enc->G ? enc->h_blob_off[enc->G] : 0;
    return STPC_OK;
}

int stpc_result_payload_lengths(const stpc_encoder* enc, int64_t* raw_lengths)
{
    if (!enc) return STPC_ERR_ARG;
    for (int i = 0; i < enc->G; ++i) raw_lengths[i] = enc->h_payload_len[i];
    return STPC_OK;
}

const uint8_t* stpc_result_device_blobs(const stpc_encoder* enc)
{
    // after a pipelined stpc_encode_host the blobs live in the caller's buffer
    return (enc && !enc->host_result) ? enc->blobs.as<uint8_t>() : nullptr;
}

int stpc_result_copy_blobs(const stpc_encoder* enc, uint8_t* h_dst, int64_t cap, void* stream)
{
    if (!enc || !h_dst) return STPC_ERR_ARG;
    long long total = enc->G ? enc->h_blob_off[enc->G] : 0;
    if (enc->host_result && enc->own_host_blobs) {
        if (total > cap) {
            g_err = "output buffer too small: need " + std::to_string(total);
            return STPC_ERR_ARG;
        }
        memcpy(h_dst, enc->hout.p, (size_t)total);
        return STPC_OK;
    }
    if (enc->host_result) {
        g_err = "blobs of a pipelined host encode are already in the caller's buffer";
        return STPC_ERR_ARG;
    }
    if (total > cap) {
        g_err = "output buffer too small: need " + std::to_string(total);
        return STPC_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (total > 0) CK(cudaMemcpyAsync(h_dst, enc->blobs.p, (size_t)total, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return STPC_OK;
}

int stpc_result_frame_stats(const stpc_encoder* enc, int64_t* out)
{
    if (!enc || !out) return STPC_ERR_ARG;
    const size_t bytes = sizeof(long long) * (size_t)enc->G * enc->n * FS_COUNT;
    if (enc->host_result) {
        memcpy(out, enc->acc_stats.p, bytes);
        return STPC_OK;
    }
    CK(cudaMemcpy(out, enc->fstats.p, bytes, cudaMemcpyDeviceToHost));
    return STPC_OK;
}

int stpc_encoder_buffer(const stpc_encoder* enc, int32_t which, void** dev_ptr, int64_t* bytes)
{
    if (!enc || !dev_ptr) return STPC_ERR_ARG;
    const DevBuf* b = nullptr;
    switch (which) {
    case STPC_BUF_BEST: b = &enc->best2[enc->best_last]; break;
    case STPC_BUF_CLS: b = &enc->cls; break;
    case STPC_BUF_RUN_S: b = &enc->run_s; break;
    case STPC_BUF_RUN_LEN: b = &enc->run_len; break;
    case STPC_BUF_RUN_ABC: b = &enc->run_abc; break;
    case STPC_BUF_N_RUNS: b = &enc->n_runs; break;
    case STPC_BUF_REF_OK: b = &enc->ref_ok; break;
    case STPC_BUF_REF_C: b = &enc->ref_c; break;
    case STPC_BUF_PAYLOAD: b = &enc->payload; break;
    case STPC_BUF_VBITS: b = &enc->vbits; break;
    default: g_err = "unknown buffer"; return STPC_ERR_ARG;
    }
    *dev_ptr = b->p;
    if (bytes) *bytes = (int64_t)b->cap;
    return STPC_OK;
}

// The entropy stage alone on caller-supplied raw payloads (the same kernels
// and launch sequence as encode_impl's entropy stage).
int stpc_entropy_encode(const uint8_t* h_payloads, const int64_t* offsets, int32_t n, uint8_t* h_out,
                        int64_t out_cap, int64_t* out_offsets)
{
    if (n < 1 || !h_payloads || !offsets || !h_out || !out_offsets) {
        g_err = "invalid arguments";
        return STPC_ERR_ARG;
    }
    cudaStream_t s = nullptr;
    std::vector<long long> len(n), poff(n + 1, 0);
    long long max_payload = 0;
    for (int i = 0; i < n; ++i) {
        len[i] = offsets[i + 1] - offsets[i];
        if (len[i] < 0) {
            g_err = "invalid offsets";
            return STPC_ERR_ARG;
        }
        poff[i + 1] = poff[i] + (len[i] + 15) / 16 * 16;  // 16-byte aligned like the encoder's arena
        max_payload = std::max(max_payload, len[i]);
    }
    DevBuf payload, plen, pofs, hist, lens, codes, enc_len, blob_off, chunk_bits, seg_crc, blobs;
    ENS(payload, (size_t)poff[n] + 16);
    ENS(plen, sizeof(long long) * n);
    ENS(pofs, sizeof(long long) * (n + 1));
    ENS(hist, sizeof(unsigned) * 256 * n);
    ENS(lens, 256 * (size_t)n);
    ENS(codes, sizeof(unsigned) * 256 * n);
    ENS(enc_len, sizeof(long long) * n);
    ENS(blob_off, sizeof(long long) * (n + 1));
    for (int i = 0; i < n; ++i)
        if (len[i]) CK(cudaMemcpy(payload.as<uint8_t>() + poff[i], h_payloads + offsets[i], (size_t)len[i],
                                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(plen.p, len.data(), sizeof(long long) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(pofs.p, poff.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice));
    EntropyArgs en;
    en.G = n;
    en.payload = payload.as<uint8_t>();
    en.payload_off = pofs.as<long long>();
    en.payload_len = plen.as<long long>();
    en.hist = hist.as<unsigned>();
    en.lens = lens.as<uint8_t>();
    en.codes = codes.as<unsigned>();
    en.enc_len = enc_len.as<long long>();
    en.blob_off = blob_off.as<long long>();
    en.max_chunks = (int)((max_payload + PACK_CHUNK - 1) / PACK_CHUNK);
    launch_zero(en.hist, sizeof(unsigned) * 256 * n, s);
    launch_histogram(en, (int)max_payload, s);
    launch_code_lengths(en, s);
    launch_group_scan(en.enc_len, en.blob_off, n, 16, HDR, s);
    std::vector<long long> el(n), bo(n + 1);
    CK(cudaMemcpy(el.data(), en.enc_len, sizeof(long long) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(bo.data(), en.blob_off, sizeof(long long) * (n + 1), cudaMemcpyDeviceToHost));
    long long max_enc = 0;
    for (int i = 0; i < n; ++i) max_enc = std::max(max_enc, el[i]);
    en.max_segs = (int)((max_enc + CRC_SEG - 1) / CRC_SEG);
    ENS(chunk_bits, sizeof(long long) * (size_t)n * std::max(en.max_chunks, 1));
    ENS(seg_crc, sizeof(unsigned) * (size_t)n * std::max(en.max_segs, 1));
    ENS(blobs, (size_t)bo[n] + 16);
    en.chunk_bits = chunk_bits.as<long long>();
    en.seg_crc = seg_crc.as<unsigned>();
    en.blobs = blobs.as<uint8_t>();
    launch_pack(en, s);
    launch_crc(en, s);
    CK(cudaGetLastError());
    long long total = 0;
    for (int i = 0; i < n; ++i) total += HDR + el[i];
    if (total > out_cap) {
        g_err = "output buffer too small: need " + std::to_string(total);
        return STPC_ERR_ARG;
    }
    CK(cudaStreamSynchronize(s));
    out_offsets[0] = 0;
    for (int i = 0; i < n; ++i) {
        CK(cudaMemcpy(h_out + out_offsets[i], blobs.as<uint8_t>() + bo[i], (size_t)(HDR + el[i]),
                      cudaMemcpyDeviceToHost));
        out_offsets[i + 1] = out_offsets[i] + HDR + el[i];
    }
    return STPC_OK;
}

int stpc_project(const void* d_points, int32_t points_f64, const int64_t* point_offsets, int32_t n_frames,
                 const double* transforms, int32_t w, int32_t h, double theta_r, double phi_r,
                 double phi_offset, double* d_best, int64_t* d_win, int64_t* h_counts, void* stream)
{
    if (n_frames < 1 || w < 1 || h < 1 || !point_offsets || !transforms || !d_best || !h_counts) {
        g_err = "invalid arguments";
        return STPC_ERR_ARG;
    }
    if ((uintptr_t)d_points % (points_f64 ? 8 : 4)) {
        g_err = "device points are not aligned to their element size";
        return STPC_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    Geometry g{};
    g.w = w;
    g.h = h;
    g.P = (long long)w * h;
    g.theta_r = theta_r;
    g.phi_r = phi_r;
    g.phi_offset = phi_offset;
    long long max_pts = 0;
    for (int f = 0; f < n_frames; ++f) max_pts = std::max<long long>(max_pts, point_offsets[f + 1] - point_offsets[f]);
    DevBuf off, xf, fs, qc, qi, qf;
    long long npts = point_offsets[n_frames] - point_offsets[0];
    long long cap = npts / 8 + 4096;
    ENS(qc, CONVERT_QCOUNT_BYTES);
    ENS(qi, sizeof(long long) * cap);
    ENS(qf, sizeof(int) * cap);
    ENS(off, sizeof(long long) * (n_frames + 1));
    ENS(xf, sizeof(double) * 12 * n_frames);
    ENS(fs, sizeof(long long) * FS_COUNT * n_frames);
    CK(cudaMemcpyAsync(off.p, point_offsets, sizeof(long long) * (n_frames + 1), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(xf.p, transforms, sizeof(double) * 12 * n_frames, cudaMemcpyHostToDevice, s));
    launch_zero(fs.p, sizeof(long long) * FS_COUNT * n_frames, s);
    launch_fill_u64((unsigned long long*)d_best, 0x7ff0000000000000ull, n_frames * g.P, s);
    ConvertArgs ca;
    ca.pts = d_points;
    ca.pts_f64 = points_f64;
    ca.pt_off = off.as<long long>();
    ca.xf = xf.as<double>();
    ca.n_frames = n_frames;
    ca.g = g;
    ca.best = (unsigned long long*)d_best;
    ca.win = (long long*)d_win;
    ca.fstats = fs.as<long long>();
    ca.q_count = qc.as<unsigned long long>();
    ca.q_idx = qi.as<long long>();
    ca.q_frame = qf.as<int>();
    ca.q_cap = cap;
    if (max_pts > 0) launch_convert(ca, (int)max_pts, s);
    if (d_win) launch_convert_win(ca, (int)std::max<long long>(max_pts, 1), s);
    std::vector<long long> hfs((size_t)FS_COUNT * n_frames);
    CK(cudaMemcpyAsync(hfs.data(), fs.p, sizeof(long long) * hfs.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int f = 0; f < n_frames; ++f)
        for (int j = 0; j < 3; ++j) h_counts[3 * f + j] = hfs[(size_t)f * FS_COUNT + j];
    return STPC_OK;
}

}  // extern "C"
