// Internal kernel interfaces of libstpc_b200 (not part of the C-ABI).
//
// Device data model for a batch of G groups of n frames (F = G*n), frame f =
// g*n + i, key frame i = k ("flat SoA device arrays"):
//
//   best   f64  [F][P]        project_kernel's min-range grid, +inf = empty
//   vbits  u8   [F][PBs]      packbits(valid), MSB-first (payload-ready)
//   ebits  u8   [F][PBs]      pixels whose u16 quantisation escapes
//   cls    u8   [F][TY][TX]   tile class: 0 residual, 1 temporal, 2 fallback
//   runs   [F*TY][TX]         s/len u16, abc f32x3 (f32-exact by construction)
//   ref    [G*TY][TX][n]      refit ok flag + f32 offset per K-run x channel
//
// P = w*h, PBs = round_up(ceil(P/8), 16), TX/TY = tiles per row / column.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace stpc {

// kernel launches issued by this library (bench.py's gpu_launches claim)
extern unsigned long long g_launch_count;
#define STPC_LAUNCH() (++::stpc::g_launch_count)

enum FrameStat {
    FS_REJECTED = 0,  // non-finite or zero-norm points
    FS_DROPPED,       // polar row outside [0, h)
    FS_KEPT,          // binned points
    FS_VALID,         // occupied pixels
    FS_TEMPORAL,      // valid pixels in temporal-run tiles
    FS_FALLBACK,      // valid pixels in fallback-run tiles
    FS_RESIDUAL,      // residual pixels
    FS_ESCAPES,       // residual pixels stored as raw f32
    FS_EPS_BAND,      // points binned within 1e-9 of a bin edge (report-only)
    FS_COUNT
};

struct Geometry {
    int w, h, tw, th, tx, ty;
    long long P;
    int pbs;  // bitmap stride (bytes)
    double theta_r, phi_r, phi_offset;
};

struct ConvertArgs {
    const void* pts;          // float32 or float64 xyz (pts_f64)
    int pts_f64;
    const long long* pt_off;  // device [F+1]
    const double* xf;         // device [F][12]
    int n_frames;
    Geometry g;
    unsigned long long* best;  // [F][P] as u64 bit patterns
    long long* win;            // nullable [F][P]
    long long* fstats;         // [F][FS_COUNT]
    // exact-path queue of points the fp32 fast path could not decide
    unsigned long long* q_count;
    long long* q_idx;
    int* q_frame;
    long long q_cap;
    int* q_bcount = nullptr;  // staged kernel: per-CTA queue counts (set by launch_convert)
    // fp32 fast-path constants, set by launch_convert: a point is decided in
    // fp32 when |frac(q) - 1/2| < hu (azimuth) and < hv (elevation)
    float inv_tr = 0.f, inv_pr = 0.f, phi_off = 0.f, hu = 0.f, hv = 0.f;
};

// The staged convert's persistent grid cap: the exact-path queue counter
// buffer holds 8 + 4 * CONVERT_MAX_GRID bytes (q_count, then q_bcount).
constexpr int CONVERT_MAX_GRID = 148 * 8;
constexpr size_t CONVERT_QCOUNT_BYTES = 8 + 4 * CONVERT_MAX_GRID;

void launch_fill_u64(unsigned long long* p, unsigned long long v, long long n, cudaStream_t s);
void launch_zero(void* p, long long bytes, cudaStream_t s);
void launch_convert(const ConvertArgs& a, int max_pts, cudaStream_t s);
void launch_convert_win(const ConvertArgs& a, int max_pts, cudaStream_t s);
void launch_bitmaps(const double* best, int n_frames, const Geometry& g, double range_quant,
                    uint8_t* vbits, uint8_t* ebits, long long* fstats, cudaStream_t s);

// float4 per tile certificate: (a, b, c, slack), (min |den|, box centre y, z, packed radii)
constexpr int CERT_F4 = 2;

struct FitArgs {
    const double* best;
    Trig tg;
    Geometry g;
    double tau, r_max, cond_limit;
    double ybias = 0.0;     // power of two >= 2 r_max: biases the certificates' box coordinates positive (pair kernel)
    int n_frames_group, k;  // group layout
    int mode;               // 0: key frames (pass 1), 1: P frames (pass 2)
    int n_jobs;             // frames in this pass
    uint8_t* cls;
    uint16_t* run_s;
    uint16_t* run_len;
    float* run_abc;
    int* n_runs;
    float4* cert;       // [F*TY][TX][CERT_F4] per-tile test certificates (scratch)
    uint8_t* start_ok;  // [F*TY][TX] start verdicts (scratch)
    double* start_sums;  // [9][F*TY*TX] a passing start tile's moment sums (scratch; null: not kept)
    long long sums_stride;  // F*TY*TX
    unsigned* chain_counter;  // work-stealing counter (scratch)
};
void launch_fit_rows(const FitArgs& a, cudaStream_t s);  // = start_tiles + fit_chains
void launch_start_tiles(const FitArgs& a, cudaStream_t s);
void launch_fit_chains(const FitArgs& a, cudaStream_t s);
bool fit_overlap_pays(const Geometry& g, long long key_chains);  // key fit beside the P start verdicts?

struct RefitArgs {
    double* best;  // covered P-frame pixels are overwritten with +inf
    Trig tg;
    Geometry g;
    double tau, r_max;
    int n, k, n_groups;
    const uint16_t* run_s;
    const uint16_t* run_len;
    const float* run_abc;
    const int* n_runs;
    uint8_t* ref_ok;     // [G*TY][TX][n]
    float* ref_c;        // [G*TY][TX][n]
    uint8_t* cls;
    long long* chain_tbytes;  // [G*TY] temporal record bytes per key chain
};
void launch_refit(const RefitArgs& a, cudaStream_t s);

// Residual rows: per (frame, image row) counts for the payload plan.
struct RowStat {
    int cnt, nesc, vb, first, last;
};
struct RowOff {
    int cnt_off, vb_off, esc_off, prev;
};

struct PlanArgs {
    Geometry g;
    int n, k, n_groups;
    const uint8_t* vbits;
    const uint8_t* ebits;
    const uint8_t* cls;
    const int* n_runs;
    const long long* chain_tbytes;
    RowStat* rowstat;  // [F][h]
    RowOff* rowoff;    // [F][h]
    long long* fstats;
    // per frame
    long long* res_cnt;   // [F]
    long long* res_vb;    // [F]
    long long* res_esc;   // [F]
    long long* fb_rows;   // [F] non-empty fallback rows
    long long* chain_off;  // [F*TY] key chains: temporal record base; P chains: fallback row offset
    // per group
    long long* sec;        // [G][2 + 2n]: temporal, total runs, fb[n], res[n]  (offsets in group payload)
    long long* payload_len;  // [G]
    long long* payload_off;  // [G] (filled by launch_group_scan)
};
void launch_rowstats(const PlanArgs& a, cudaStream_t s);
void launch_plan(const PlanArgs& a, cudaStream_t s);
// Exclusive scan of lens[G] (rounded up to `align`) into offs; offs[G] = total.
void launch_group_scan(const long long* lens, long long* offs, int G, int align, long long add, cudaStream_t s);

struct EmitArgs {
    PlanArgs p;
    const double* best;
    double range_quant, inv_quant;
    const uint8_t* cfg_bytes;  // device [57]
    const double* xf;          // device [F][12]
    const uint16_t* run_s;
    const uint16_t* run_len;
    const float* run_abc;
    const uint8_t* ref_ok;
    const float* ref_c;
    uint8_t* payload;  // arena
};
void launch_emit(const EmitArgs& a, cudaStream_t s);

struct EntropyArgs {
    int G;
    const uint8_t* payload;
    const long long* payload_off;  // [G+1]
    const long long* payload_len;  // [G]
    unsigned int* hist;            // [G][256]
    uint8_t* lens;                 // [G][256]
    unsigned int* codes;           // [G][256]
    long long* enc_len;            // [G]
    long long* blob_off;           // [G+1]
    uint8_t* blobs;                // arena
    long long* chunk_bits;         // [G][max_chunks]
    unsigned int* seg_crc;         // [G][max_segs]
    int max_chunks, max_segs;
    // +inf prefill of the next call's range grid, spread over the pack
    // blocks (background stores behind the instruction-bound packing)
    unsigned long long* prefill = nullptr;
    long long prefill_n = 0;  // u64 elements (even)
    long long prefill_per = 0;  // 16-byte elements per pack block (set by launch_pack)
};
constexpr int PACK_CHUNK = 4096;  // payload bytes per pack block
constexpr int CRC_PIECE = 256;    // bytes per CRC thread
constexpr int CRC_SEG = 32 * CRC_PIECE;  // bytes per CRC warp
struct CrcConsts {
    unsigned int x256[5];  // x^(8*256*2^l) mod P
    unsigned int seg;      // x^(8*CRC_SEG) mod P
};
constexpr int HDR = 284;          // header + code-length table
void launch_histogram(const EntropyArgs& a, int max_payload, cudaStream_t s);
void launch_code_lengths(const EntropyArgs& a, cudaStream_t s);
void launch_pack(const EntropyArgs& a, cudaStream_t s);
void launch_crc(const EntropyArgs& a, cudaStream_t s);

}  // namespace stpc
