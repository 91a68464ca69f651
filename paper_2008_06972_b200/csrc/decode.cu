// Decoder: the device side of decompress().
//
// Replaces the reference decoder (/root/reference/pkg/src/stpc/bitstream.py:
// 388-519, 605-631) end to end on the GPU, batched over blobs:
//
//   phase 1  stpc_decoder_load     header + code-table checks (host, :398-409,
//                                  huffman.py:80-104), zlib.crc32 (:410-411)
//                                  -> crc_blob_kernel, canonical Huffman decode
//                                  (huffman.py:121-137, _kernels.py:385-417)
//                                  -> huff_decode_kernel
//   phase 2  stpc_decoder_frames   record sections of deserialize (:428-519)
//                                  -> parse_kernel (validation + per-tile plane
//                                  maps + residual section bounds);
//                                  decode_stream_images (temporal.py:293-343)
//                                  with reconstruct_span (_kernels.py:282-308)
//                                  -> reconstruct_kernel, residual_kernel;
//                                  point counts -> count/scan kernels
//   phase 3  stpc_decoder_points   unproject (range_image.py:214-221) + the
//                                  inverse frame transform (motion.py:78-79,
//                                  70-72) -> unproject_kernel
//
// Structural errors carry a key (reader position << 8 | order << 4 | kind);
// the smallest key per blob is the error the reference's sequential reader
// (_Reader, bitstream.py:333-353) raises first.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "kernels.cuh"
#include "runtime.cuh"
#include "../../include/stpc_b200.h"

namespace stpc {

constexpr unsigned long long DEC_NONE = ~0ull;
// "no point" marker of the range scratch: a signalling NaN whose low mantissa
// bit is set, which neither a float32 escape range widened to float64 (low 29
// bits zero) nor a reconstructed range (positive, finite) can produce.
constexpr long long DEC_NOPT = 0x7ff4000000000001ll;
constexpr int DEC_HEADER = 284;

struct DecGeom {
    int w, h, tw, th, tx, ty, n, k, pm;
    long long P, nb;
    long long bits_off;  // 57 + 48 n: first validity bitmap
    long long runs_off;  // bits_off + n nb: temporal run count
    double quant, r_max;
    double rw, rtw, rth, rn;  // fl(1 / w), 1 / tw, 1 / th, 1 / n for dmod
    // x / tw and x / th as __umulhi(x, m) (exact for x, divisor < 2^16:
    // m = ceil(2^32 / d) overshoots by less than d per unit, so x (m d - 2^32)
    // < 2^32); both 0 when the geometry is too large or a divisor is 1 (dmod)
    unsigned mtw, mth;
};

// q, r = p / d, p % d for 0 <= p < 2^50 through the double reciprocal rd =
// fl(1 / d): the estimate is off by at most one, fixed exactly (per-pixel
// 64-bit integer divides dominated the pixel kernels' instruction counts).
__device__ __forceinline__ long long dmod(long long p, long long d, double rd, long long& r)
{
    long long q = (long long)((double)p * rd);
    r = p - q * d;
    if (r < 0) {
        q -= 1;
        r += d;
    } else if (r >= d) {
        q += 1;
        r -= d;
    }
    return q;
}

struct ResSec {
    long long pos_var;   // first varint byte
    long long cnt;       // residual pixels
    long long pos_code;  // u16 codes
    long long pos_esc;   // f32 escape ranges
};

__device__ __forceinline__ unsigned dec_u8(const uint8_t* p) { return __ldg(p); }
__device__ __forceinline__ unsigned dec_u16(const uint8_t* p) { return dec_u8(p) | (dec_u8(p + 1) << 8); }
__device__ __forceinline__ unsigned dec_u32(const uint8_t* p) { return dec_u16(p) | (dec_u16(p + 2) << 16); }
__device__ __forceinline__ float dec_f32(const uint8_t* p) { return __uint_as_float(dec_u32(p)); }
__device__ __forceinline__ unsigned long long dec_key(long long pos, int order, int kind)
{
    return ((unsigned long long)pos << 8) | ((unsigned)order << 4) | (unsigned)kind;
}

// ---------------------------------------------------------------- block scans

template <int NT>
__device__ __forceinline__ long long block_excl_scan(long long v, long long& total)
{
    __shared__ long long ws[NT / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(STPC_FULL, x, o);
        if (lane >= o) x += t;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    long long before = 0, tot = 0;
    for (int w = 0; w < NT / 32; ++w) {
        if (w < wid) before += ws[w];
        tot += ws[w];
    }
    __syncthreads();
    total = tot;
    return before + x - v;
}

// ---------------------------------------------------------------- CRC-32

__host__ __device__ __forceinline__ unsigned int dec_multmodp(unsigned int a, unsigned int b)
{
    unsigned int m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = b & 1 ? (b >> 1) ^ 0xedb88320u : b >> 1;
    }
    return p;
}

__host__ __device__ __forceinline__ unsigned int dec_x8nmodp(unsigned long long nbytes)
{
    unsigned int p = 1u << 31, sq = 1u << 23;
    while (nbytes) {
        if (nbytes & 1) p = dec_multmodp(sq, p);
        sq = dec_multmodp(sq, sq);
        nbytes >>= 1;
    }
    return p;
}

#ifndef STPC_DC_PIECE
#define STPC_DC_PIECE 64  // 16 KB chunks: 1024 blobs fit one wave (load 26.0 -> 24.8 ms); 32 -> 25.8
#endif
constexpr int DC_PIECE = STPC_DC_PIECE;          // bytes per thread
constexpr int DC_CHUNK = 256 * DC_PIECE;          // bytes per block pass

struct DecCrcK {
    unsigned int lvl[8];  // x^(8 * DC_PIECE * 2^l) mod P, l = 0..7
    unsigned int chunk;   // x^(8 * DC_CHUNK)
};

// Block per blob.  Each pass stages a 32 KB chunk of the entropy payload in
// shared memory (coalesced 32-bit loads from the aligned base), every thread
// folds a 128-byte piece with the byte table, and the pieces are combined
// in order by a shuffle tree (crc(A|B) = x^(8|B|) crc(A) ^ crc(B) for the
// zero-initialised register).  A short last chunk is end-aligned in its
// frame: leading zero bytes leave a zero register unchanged.  crc_bad =
// (zlib.crc32(encoded) != header CRC), bitstream.py:410-411.
__global__ void __launch_bounds__(256) crc_blob_kernel(const uint8_t* blobs, const long long* blob_off,
                                                       const int* skip, DecCrcK K, int* crc_bad)
{
    if (skip[blockIdx.x]) return;
    if ((((unsigned long long)(blobs + blob_off[blockIdx.x] + DEC_HEADER)) & 3) == 0) return;  // crc_dseg_kernel's
    __shared__ unsigned int tab[256];
    __shared__ unsigned int stage[DC_CHUNK / 4 + 2];
    __shared__ unsigned int wpart[8];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    {
        unsigned int c = tid;
        for (int k = 0; k < 8; ++k) c = c & 1 ? (c >> 1) ^ 0xedb88320u : c >> 1;
        tab[tid] = c;
    }
    const uint8_t* blob = blobs + blob_off[blockIdx.x];
    unsigned long long enc_len = 0;
    for (int b = 0; b < 8; ++b) enc_len |= (unsigned long long)blob[16 + b] << (8 * b);
    const unsigned int want = dec_u32(blob + 24);
    const uint8_t* enc = blob + DEC_HEADER;
    const unsigned long long addr = (unsigned long long)enc;
    const int mis = (int)(addr & 3);
    const unsigned int* wbase = (const unsigned int*)(addr - mis);
    const long long last_byte = mis + (long long)enc_len - 1;  // relative to wbase
    unsigned int raw = 0;
    for (long long base = 0; base < (long long)enc_len; base += DC_CHUNK) {
        const long long nb = min((long long)DC_CHUNK, (long long)enc_len - base);
        const long long w0 = (mis + base) >> 2;
        const long long w1 = (mis + base + nb - 1) >> 2;
        __syncthreads();
        for (long long i = tid; w0 + i <= w1; i += 256) {
            const long long w = w0 + i;
            unsigned int v;
            if (4 * w + 3 <= last_byte) {
                v = __ldg(wbase + w);
            } else {  // the stream's last word: no read past its final byte
                v = 0;
                const uint8_t* bp = (const uint8_t*)wbase + 4 * w;
                for (int k = 0; k < 4 && 4 * w + k <= last_byte; ++k) v |= (unsigned)dec_u8(bp + k) << (8 * k);
            }
            stage[i] = v;
        }
        __syncthreads();
        // piece tid covers frame bytes [tid*128, +128); frame byte f is stream
        // byte base + f - (DC_CHUNK - nb); earlier frame bytes are zeros
        const long long lead = DC_CHUNK - nb;
        const uint8_t* sb = (const uint8_t*)stage + ((mis + base) - 4 * w0);
        unsigned int c = 0;
        const long long f0 = (long long)tid * DC_PIECE;
        for (int i = 0; i < DC_PIECE; ++i) {
            const long long f = f0 + i;
            if (f < lead) continue;
            c = tab[(c ^ sb[f - lead]) & 0xff] ^ (c >> 8);
        }
        for (int l = 0; l < 5; ++l) {
            const unsigned int other = __shfl_down_sync(STPC_FULL, c, 1 << l);
            if ((lane & ((2 << l) - 1)) == 0) c = dec_multmodp(K.lvl[l], c) ^ other;
        }
        if (lane == 0) wpart[wid] = c;
        __syncthreads();
        if (tid == 0) {
            unsigned int ch = 0;
            for (int w = 0; w < 8; ++w) ch = dec_multmodp(K.lvl[5], ch) ^ wpart[w];
            raw = dec_multmodp(nb == DC_CHUNK ? K.chunk : dec_x8nmodp((unsigned long long)nb), raw) ^ ch;
        }
    }
    if (tid == 0) {
        const unsigned int crc = ~(raw ^ dec_multmodp(dec_x8nmodp(enc_len), 0xffffffffu));
        crc_bad[blockIdx.x] = crc != want;
    }
}

// Fast path of the same check for entropy payloads that start on a 4-byte
// boundary (every blob the encoder writes: 16-byte-aligned blobs + the
// 284-byte header; other blobs keep crc_blob_kernel), spread over many warps
// per blob (the encoder's CRC scheme, entropy.cu): each lane folds one
// 256-byte piece slice-by-4 (four table lookups per word), staged through a
// padded shared tile 64 bytes of every piece at a time so the global loads
// stay coalesced; a warp's 32 pieces merge by a shuffle tree into a segment
// CRC, and crc_dfinish combines the segments with x^(8n) multipliers.  Both
// paths skip the other's blobs.
struct DecCrcTab4 {
    unsigned int t[4][256];
};
constexpr DecCrcTab4 make_dec_crc_tab4()
{
    DecCrcTab4 r{};
    for (unsigned int i = 0; i < 256; ++i) {
        unsigned int c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? (c >> 1) ^ 0xedb88320u : c >> 1;
        r.t[0][i] = c;
    }
    for (unsigned int i = 0; i < 256; ++i) {
        unsigned int c = r.t[0][i];
        for (int k = 1; k < 4; ++k) {
            c = (c >> 8) ^ r.t[0][c & 0xff];
            r.t[k][i] = c;
        }
    }
    return r;
}
__device__ const DecCrcTab4 kDecCrcTab4 = make_dec_crc_tab4();

constexpr int DCF_PIECE = 256;  // bytes per lane
constexpr int DCF_SUB = 64;     // bytes per piece per staging round

struct DecCrcF {
    unsigned int x256[5];  // x^(8 * 256 * 2^l) mod P
    unsigned int warp;     // x^(8 * 32 * 256): one segment
};

constexpr int DCF_WARPS = 8;
constexpr int DCF_SEGS_PER_WARP = 4;  // segments per warp (amortises the table copy)
constexpr int DCF_SEG = 32 * DCF_PIECE;  // bytes per segment (a warp's 32 pieces)

// grid (segments / (DCF_WARPS * DCF_SEGS_PER_WARP), blobs): warp-segments of
// 32 pieces of 256 B from the payload's start; only full pieces here (the
// < 256 B tail is crc_dfinish's).  The last segment's pieces are end-aligned
// in the 32-slot tree (missing leading slots = zero prefix).
__global__ void __launch_bounds__(DCF_WARPS * 32) crc_dseg_kernel(const uint8_t* blobs, const long long* blob_off,
                                                                  const int* skip, DecCrcF K, int max_segs,
                                                                  unsigned* seg_crc)
{
    const int b = blockIdx.y;
    if (skip[b]) return;
    const uint8_t* blob = blobs + blob_off[b];
    const uint8_t* encb = blob + DEC_HEADER;
    if (((unsigned long long)encb) & 3) return;  // crc_blob_kernel's blob
    __shared__ unsigned int T[4][256];
    __shared__ unsigned int stg[DCF_WARPS][32][DCF_SUB / 4 + 1];
    {
        const unsigned int* src = &kDecCrcTab4.t[0][0];
        for (int i = threadIdx.x; i < 1024; i += blockDim.x) (&T[0][0])[i] = __ldg(src + i);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned long long enc_len = 0;
    for (int i = 0; i < 8; ++i) enc_len |= (unsigned long long)blob[16 + i] << (8 * i);
    const long long npieces = (long long)(enc_len / DCF_PIECE);
    const long long nseg = (npieces + 31) / 32;
    const uint32_t* enc = reinterpret_cast<const uint32_t*>(encb);
    unsigned int (*tile)[DCF_SUB / 4 + 1] = stg[wib];
    for (int rep = 0; rep < DCF_SEGS_PER_WARP; ++rep) {
        const long long sgi = ((long long)blockIdx.x * DCF_SEGS_PER_WARP + rep) * DCF_WARPS + wib;
        if (sgi >= nseg) return;
        const long long first = sgi * 32;
        const int np = (int)min(32LL, npieces - first);
        const int slot_piece = lane - (32 - np);  // end-aligned
        unsigned int crc = 0;
        for (int r = 0; r < DCF_PIECE / DCF_SUB; ++r) {
#pragma unroll
            for (int it = 0; it < DCF_SUB / 4; ++it) {  // 32 pieces x 16 words, 2 pieces per load
                const int widx = it * 32 + lane;
                const int k = widx >> 4, wd = widx & 15;
                const int pk = k - (32 - np);
                tile[k][wd] = pk >= 0 ? __ldg(enc + ((first + pk) * DCF_PIECE + r * DCF_SUB) / 4 + wd) : 0u;
            }
            __syncwarp();
            if (slot_piece >= 0) {
#pragma unroll
                for (int i = 0; i < DCF_SUB / 4; ++i) {
                    const unsigned int x = crc ^ tile[lane][i];
                    crc = T[3][x & 0xff] ^ T[2][(x >> 8) & 0xff] ^ T[1][(x >> 16) & 0xff] ^ T[0][x >> 24];
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int l = 0; l < 5; ++l) {
            const unsigned int right = __shfl_down_sync(STPC_FULL, crc, 1 << l);
            if ((lane & ((2 << l) - 1)) == 0) crc = dec_multmodp(K.x256[l], crc) ^ right;
        }
        if (lane == 0) seg_crc[(long long)b * max_segs + sgi] = crc;
    }
}

// block per blob (one thread): the segment CRCs in order, then the < 256 B
// tail byte-wise, then the comparison with the header's CRC
__global__ void crc_dfinish_kernel(const uint8_t* blobs, const long long* blob_off, const int* skip, DecCrcF K,
                                   int max_segs, const unsigned* seg_crc, int* crc_bad)
{
    const int b = blockIdx.x;
    if (skip[b] || threadIdx.x != 0) return;
    const uint8_t* blob = blobs + blob_off[b];
    const uint8_t* encb = blob + DEC_HEADER;
    if (((unsigned long long)encb) & 3) return;
    unsigned long long enc_len = 0;
    for (int i = 0; i < 8; ++i) enc_len |= (unsigned long long)blob[16 + i] << (8 * i);
    const unsigned int want = dec_u32(blob + 24);
    const long long npieces = (long long)(enc_len / DCF_PIECE);
    const long long nseg = (npieces + 31) / 32;
    unsigned int raw = 0;
    for (long long sgi = 0; sgi < nseg; ++sgi) {
        const long long np = min(32LL, npieces - sgi * 32);
        const unsigned int X = np == 32 ? K.warp : dec_x8nmodp((unsigned long long)np * DCF_PIECE);
        raw = dec_multmodp(X, raw) ^ seg_crc[(long long)b * max_segs + sgi];
    }
    const long long tb = npieces * DCF_PIECE;
    if (tb < (long long)enc_len) {
        raw = dec_multmodp(dec_x8nmodp((unsigned long long)(enc_len - tb)), raw);
        unsigned int t = 0;
        for (long long i = tb; i < (long long)enc_len; ++i) {
            unsigned int c = (t ^ dec_u8(encb + i)) & 0xff;
            for (int k = 0; k < 8; ++k) c = c & 1 ? (c >> 1) ^ 0xedb88320u : c >> 1;
            t = c ^ (t >> 8);
        }
        raw ^= t;
    }
    const unsigned int crc = ~(raw ^ dec_multmodp(dec_x8nmodp(enc_len), 0xffffffffu));
    crc_bad[b] = crc != want;
}

// ---------------------------------------------------------------- Huffman

constexpr int HD_THREADS = 256;
constexpr int HD_SUB = 4;                     // sub-segments per thread
constexpr int HD_NSEG = HD_THREADS * HD_SUB;  // sub-segments per blob (max)
constexpr int HD_LUT = 12;                    // first-level table bits
constexpr long long HD_SEG_MIN = 2048;        // bits per sub-segment (min)

struct HuffDev {
    unsigned short lut[1 << HD_LUT];  // (len << 8) | symbol; 0 = longer code
    unsigned long long first[33];
    int count[33];
    int index[33];
    unsigned char sym[256];
};

// codes longer than the first-level table (rare): canonical first-code search
// over lengths HD_LUT+1..32 (huffman_decode_kernel's per-length test)
__device__ __noinline__ unsigned huff_long(const HuffDev& T, unsigned w)
{
    // returns (len << 8) | symbol, 0 when no code matches (by value: a
    // reference argument would force the caller's symbol through local memory)
    for (int l = HD_LUT + 1; l <= 32; ++l) {
        if (T.count[l]) {
            const unsigned long long c = (unsigned long long)w >> (32 - l);
            if (c >= T.first[l] && c - T.first[l] < (unsigned long long)T.count[l])
                return ((unsigned)l << 8) | T.sym[T.index[l] + (int)(c - T.first[l])];
        }
    }
    return 0u;
}

// Lean reader for the decode loops: a 64-bit MSB-aligned window refilled by
// one 32-bit big-endian word whenever fewer than 32 bits remain (one word
// prefetched ahead); positions are 32-bit offsets from the start of the
// sub-segment, so the per-symbol work stays in 32-bit integer ops.
struct BitRd {
    const uint32_t* words;
    long long wlast, wi;
    unsigned long long cur;
    int nb, used, avail;
    uint32_t nxt;
    __device__ __forceinline__ uint32_t ldw(long long i) const
    {
        return i <= wlast ? __byte_perm(__ldg(words + i), 0, 0x0123) : 0u;
    }
    __device__ __forceinline__ void init(const uint8_t* e, long long elen, long long start)
    {
        const unsigned long long a = (unsigned long long)e;
        const int mis = (int)(a & 3);
        words = (const uint32_t*)(a - mis);
        wlast = elen > 0 ? (mis + elen - 1) / 4 : -1;
        const long long sb = start + 8ll * mis;
        const long long w = sb >> 5;
        const int o = (int)(sb & 31);
        cur = (((unsigned long long)ldw(w) << 32) | ldw(w + 1)) << o;
        nb = 64 - o;
        nxt = ldw(w + 2);
        wi = w + 3;
        used = 0;
        avail = (int)min(elen * 8 - start, (long long)0x7fffffff);
    }
};

// One symbol; returns whether it fit (the caller derives the reference's
// 1 / 2 status from the last `len` once, after its loop).  Branch-free apart
// from the rare long-code search: the refill (every ~5 symbols, at different
// steps in different lanes) is predicated, with the next word's load issued
// under a predicate instead of a divergent branch.
__device__ __forceinline__ bool huff_step(const HuffDev& T, BitRd& r, int& sym, int& len)
{
    const unsigned w = (unsigned)(r.cur >> 32);
    unsigned e = T.lut[w >> (32 - HD_LUT)];
    if (e == 0) e = huff_long(T, w);
    len = (int)(e >> 8);
    sym = (int)(e & 0xff);
    const bool fits = len != 0 && len <= r.avail - r.used;
    const int l = fits ? len : 0;
    r.cur <<= l;
    r.nb -= l;
    r.used += l;
    const bool refill = r.nb < 32;
    r.cur |= refill ? (unsigned long long)r.nxt << (32 - r.nb) : 0ull;
    r.nb += refill ? 32 : 0;
#ifndef STPC_HUFF_BRANCHY
    unsigned nw = r.nxt;
    const int ld = refill && r.wi <= r.wlast;
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.s32 p, %2, 0;\n @p ld.global.nc.u32 %0, [%1];\n}"
        : "+r"(nw)
        : "l"(r.words + r.wi), "r"(ld));
    nw = ld ? __byte_perm(nw, 0, 0x0123) : 0u;
    r.nxt = refill ? nw : r.nxt;
    r.wi += refill ? 1 : 0;
#else
    if (refill) {
        r.nxt = r.ldw(r.wi);
        ++r.wi;
    }
#endif
    return fits;
}

#ifdef STPC_HUFF_STATS
__device__ unsigned long long g_huff_stats[8];
extern "C" int stpc_debug_huff_stats(unsigned long long* out)
{
    return cudaMemcpyFromSymbol(out, g_huff_stats, sizeof(g_huff_stats)) == cudaSuccess ? 0 : 1;
}
#define HUFF_STAT(i, v) atomicAdd(&g_huff_stats[i], (unsigned long long)(v))
#else
#define HUFF_STAT(i, v) ((void)0)
#endif

// Block per blob.  The bitstream is cut into <= 1024 sub-segments (4 per
// thread).  Round 1: each thread parses its sub-segments in sequence from the
// nominal start of its first one (a guess: it may sit inside a codeword).
// Later rounds: a thread whose first start differs from where its left
// neighbour's parse ended re-parses from that end, sub-segment by
// sub-segment, until its new parse reaches a sub-segment end of the old one
// (canonical codes resynchronise within a few symbols), after which the old
// counts stand.  Converged starts are exact by induction from bit 0; a final
// pass writes the symbols at scanned offsets.
#ifndef STPC_HUFF_MINB
#define STPC_HUFF_MINB 8  // measured (load = crc + huffman, 1024 blobs): 1 -> 27.7 ms, 8 -> 26.0
#endif
__global__ void __launch_bounds__(HD_THREADS, STPC_HUFF_MINB) huff_decode_kernel(const uint8_t* blobs, const long long* blob_off,
                                                                 const int* skip, uint8_t* raw,
                                                                 const long long* raw_off, int* status)
{
    const int b = blockIdx.x;
    if (skip[b]) return;
    __shared__ HuffDev T;
    __shared__ long long s_st[HD_NSEG], s_en[HD_NSEG];
    __shared__ int s_cnt[HD_NSEG];
    __shared__ unsigned char s_err[HD_NSEG];
    __shared__ unsigned char s_len[256];
    __shared__ long long s_errpos;
    const int tid = threadIdx.x;
    const uint8_t* blob = blobs + blob_off[b];
    unsigned long long raw_len = 0, enc_len = 0;
    for (int i = 0; i < 8; ++i) {
        raw_len |= (unsigned long long)blob[8 + i] << (8 * i);
        enc_len |= (unsigned long long)blob[16 + i] << (8 * i);
    }
    if (raw_len == 0) {
        if (tid == 0) status[b] = 0;
        return;
    }
    // canonical tables (huffman.py:80-104); the host has checked the lengths
    for (int i = tid; i < (1 << HD_LUT); i += HD_THREADS) T.lut[i] = 0;
    if (tid < 33) T.count[tid] = 0;
    s_len[tid] = blob[28 + tid];
    if (tid == 0) s_errpos = 0x7fffffffffffffffll;
    __syncthreads();
    if (s_len[tid]) atomicAdd(&T.count[s_len[tid]], 1);
    __syncthreads();
    if (tid == 0) {
        unsigned long long code = 0;
        int idx = 0;
        T.first[0] = 0;
        T.index[0] = 0;
        for (int l = 1; l <= 32; ++l) {
            T.first[l] = code;
            T.index[l] = idx;
            code = (code + (unsigned long long)T.count[l]) << 1;
            idx += T.count[l];
        }
    }
    __syncthreads();
    {
        const int l = s_len[tid];
        if (l) {
            int rank = T.index[l];
            for (int s = 0; s < 256; ++s) rank += (s < tid) & (s_len[s] == l);
            T.sym[rank] = (unsigned char)tid;
            if (l <= HD_LUT) {
                const unsigned long long code = T.first[l] + (unsigned long long)(rank - T.index[l]);
                const int lo = (int)(code << (HD_LUT - l)), span = 1 << (HD_LUT - l);
                for (int i = 0; i < span; ++i) T.lut[lo + i] = (unsigned short)((l << 8) | tid);
            }
        }
    }
    __syncthreads();

    const uint8_t* enc = blob + DEC_HEADER;
    const long long total = (long long)enc_len * 8;
    long long nseg = (total + HD_SEG_MIN - 1) / HD_SEG_MIN;
    nseg = nseg < 1 ? 1 : (nseg > HD_NSEG ? HD_NSEG : nseg);
    const long long seg = total > 0 ? (total + nseg - 1) / nseg : 0;
    const int t0 = tid * HD_SUB;
    const int t1 = (int)min((long long)t0 + HD_SUB, nseg);
    auto nominal_end = [&](int t) -> long long { return t == nseg - 1 ? total : min((t + 1) * seg, total); };
    // Parse one sub-segment per lane, all 32 lanes of the warp together: the
    // vote in the loop condition keeps the warp converged every step (a
    // plain per-lane loop lets the lanes drift apart and run one at a time).
    auto parse_sub = [&](bool active, int t, long long start, long long& end, int& cnt) -> int {
        BitRd r;
        r.init(enc, (long long)enc_len, active ? start : 0);
        const int need = active ? (int)(nominal_end(t) - start) : 0;
        int c = 0, len = 1;
        bool fits = true;
        bool go = active && need > 0;
        while (__any_sync(STPC_FULL, go)) {
            if (go) {
                int sym;
                fits = huff_step(T, r, sym, len);
                c += fits ? 1 : 0;
                go = fits && r.used < need;
            }
        }
        end = start + r.used;
        cnt = c;
        if (active) HUFF_STAT(0, c);  // symbols parsed (all rounds)
        return fits ? 0 : (len == 0 && r.avail - r.used >= 33 ? 2 : 1);
    };

    // round 1 (warp-uniform trip count; __syncwarp re-converges the lanes
    // before every sub-segment so the 32 parses run in lock-step)
    {
        long long pos = t0 < nseg ? min(t0 * seg, total) : total;
        bool dead = false;
        for (int k = 0; k < HD_SUB; ++k) {
            __syncwarp();
            const int t = t0 + k;
            const bool act = t < t1 && !dead;
            long long e;
            int c;
            const int rc = parse_sub(act, t, pos, e, c);
            if (t < t1) {
                s_st[t] = pos;
                if (dead) {
                    s_en[t] = pos;
                    s_cnt[t] = 0;
                    s_err[t] = 3;
                } else {
                    s_en[t] = e;
                    s_cnt[t] = c;
                    s_err[t] = (unsigned char)rc;
                    pos = e;
                    dead = rc == 2;
                }
            }
        }
    }
    __syncthreads();  // round-1 ends must be visible before any thread reads its neighbour's
    // correction rounds
    for (;;) {
        long long want = -1;
        if (t0 > 0 && t0 < nseg && s_err[t0 - 1] == 0 && s_en[t0 - 1] != s_st[t0]) want = s_en[t0 - 1];
        __syncthreads();
        long long pos = want;
        bool live = want >= 0, dead = false;
        for (int k = 0; k < HD_SUB; ++k) {
            __syncwarp();
            const int t = t0 + k;
            const bool act = live && t < t1 && !dead;
            long long e;
            int c;
            const int rc = parse_sub(act, t, pos, e, c);
            if (live && t < t1) {
                if (dead) {
                    s_st[t] = pos;
                    s_en[t] = pos;
                    s_cnt[t] = 0;
                    s_err[t] = 3;
                } else {
                    const long long old_en = s_en[t];
                    const int old_err = s_err[t];
                    s_st[t] = pos;
                    s_en[t] = e;
                    s_cnt[t] = c;
                    s_err[t] = (unsigned char)rc;
                    if (rc == 2) dead = true;
                    else if (rc == 0 && old_err == 0 && e == old_en) live = false;  // resynchronised
                    else pos = e;
                }
            }
        }
        if (tid == 0) HUFF_STAT(1, 1);  // correction rounds
        if (want >= 0) HUFF_STAT(2, 1);  // corrected threads
        if (!__syncthreads_or(want >= 0)) break;
    }

    // symbol offsets; the first invalid code (in parse order) and the total
    long long mine = 0;
    for (int t = t0; t < t1; ++t) mine += s_cnt[t];
    long long tot;
    const long long base = block_excl_scan<HD_THREADS>(mine, tot);
    {
        long long o = base;
        for (int t = t0; t < t1; ++t) {
            if (s_err[t] == 2) {
                atomicMin((unsigned long long*)&s_errpos, (unsigned long long)(o + s_cnt[t]));
                break;
            }
            o += s_cnt[t];
        }
    }
    __syncthreads();
    const long long errpos = s_errpos;
    if (errpos < (long long)raw_len) {
        if (tid == 0) status[b] = 2;
        return;
    }
    if (tot < (long long)raw_len) {
        if (tid == 0) status[b] = 1;
        return;
    }
    // write pass (warp-synchronous like parse_sub)
    uint8_t* out = raw + raw_off[b];
    long long o = base;
    for (int k = 0; k < HD_SUB; ++k) {
        const int t = t0 + k;
        const bool act = t < t1 && o < (long long)raw_len;
        BitRd r;
        r.init(enc, (long long)enc_len, act ? s_st[t] : 0);
        const int c = act ? (int)min((long long)s_cnt[t], (long long)raw_len - o) : 0;
        int i = 0;
        bool go = i < c;
        while (__any_sync(STPC_FULL, go)) {
            if (go) {
                int sym, len;
                huff_step(T, r, sym, len);
                out[o + i] = (uint8_t)sym;
                go = ++i < c;
            }
        }
        if (t < t1) o += s_cnt[t];
    }
    if (tid == 0) status[b] = 0;
}

// the 284-byte header of every blob (shorter blobs: what there is, zero-padded)
__global__ void blob_headers_kernel(const uint8_t* blobs, const long long* blob_off, const long long* blob_len,
                                    uint8_t* out)
{
    const int b = blockIdx.x;
    const long long n = min((long long)DEC_HEADER, blob_len[b]);
    for (int i = threadIdx.x; i < DEC_HEADER; i += blockDim.x)
        out[(long long)b * DEC_HEADER + i] = i < n ? blobs[blob_off[b] + i] : 0;
}

// first min(raw_len, cap) bytes of every raw payload (config + transforms)
__global__ void heads_kernel(const uint8_t* raw, const long long* raw_off, const long long* raw_len,
                             const int* ok, int cap, uint8_t* heads)
{
    const int b = blockIdx.x;
    const long long n = ok[b] ? min((long long)cap, raw_len[b]) : 0;
    for (int i = threadIdx.x; i < cap; i += blockDim.x)
        heads[(long long)b * cap + i] = i < n ? raw[raw_off[b] + i] : 0;
}

// ---------------------------------------------------------------- records

constexpr int PK_THREADS = 256;
#ifndef STPC_PK_BATCH
#define STPC_PK_BATCH 512  // records per batch; 512 (with 8 blocks per SM) fits 1024 blobs in one wave: frames 31.9 -> 28.3 ms
#endif
#ifndef STPC_PK_WIN
#define STPC_PK_WIN 16384
#endif
constexpr int PK_BATCH = STPC_PK_BATCH;
constexpr int PK_WIN = STPC_PK_WIN;  // staged bytes of the run section

// Block per blob: validates the record sections in the reference's reading
// order and turns them into per-(frame, tile) plane maps (a, b, c, kind:
// 1 temporal run with this frame's offset, 2 fallback run, 0 none) plus the
// bounds of each frame's residual section.  The variable-length records are
// walked by one thread (a record's size depends on its presence mask) in
// batches that the block then expands in parallel; residual varints are
// scanned block-parallel (terminator bytes < 0x80).
#ifndef STPC_PARSE_MINB
#define STPC_PARSE_MINB 8  // measured (frames phase): 1 -> 35.5 ms, 6 -> 31.7, 8 -> 32.7 (smem-limited to 6 at 1024-record batches); 8 with 512-record batches -> 28.3
#endif
__global__ void __launch_bounds__(PK_THREADS, STPC_PARSE_MINB) parse_kernel(DecGeom G, const uint8_t* raw, const long long* raw_off,
                                                           const long long* raw_len, const int* sel, float4* tmap,
                                                           ResSec* res, unsigned long long* pstat, long long* ovl)
{
    const int j = blockIdx.x;
    const int b = sel[j];
    const uint8_t* p = raw + raw_off[b];
    const long long len = raw_len[b];
    const int tid = threadIdx.x;
    __shared__ unsigned long long st;
    __shared__ long long recs[PK_BATCH];
    __shared__ int fch[PK_BATCH], frow[PK_BATCH], fnr[PK_BATCH];
    __shared__ unsigned win32[PK_WIN / 4];
    __shared__ int s_nrec, s_done;
    __shared__ long long s_pos, s_cnt, s_end, s_left;
    __shared__ int s_ch;
    __shared__ unsigned long long s_flat;
    __shared__ int s_dbad, s_vbad;
    // Run order check.  The encoder emits temporal runs sorted by (row, s)
    // and disjoint, and per frame fallback rows in increasing row order with
    // sorted, disjoint runs; then one plane per (frame, tile) is exact.  Any
    // other order (a hand-made blob the reference's deserialize accepts) may
    // overlap, and the reference's stream-order last-writer semantics
    // (temporal.py:307-331) are replayed by ordered_reconstruct_kernel.
    __shared__ int s_ovl, s_frow;
    __shared__ long long s_tend, s_fbpos;
    if (tid == 0) {
        st = DEC_NONE;
        s_ovl = 0;
        s_tend = -1;
        s_fbpos = 0;
    }
    float4* tm = tmap + (long long)j * G.n * G.ty * G.tx;
    const long long ntile = (long long)G.n * G.ty * G.tx;
    for (long long i = tid; i < ntile; i += PK_THREADS) tm[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    auto fail = [&](long long pos, int order, int kind) { atomicMin(&st, dec_key(pos, order, kind)); };

    // bitmaps (n takes of nb bytes) and the run count
    if (tid == 0) {
        if (len < G.runs_off) {
            fail(G.bits_off + (len - G.bits_off) / G.nb * G.nb, 0, STPC_DEC_TRUNCATED);
        } else if (G.runs_off + 4 > len) {
            fail(G.runs_off, 0, STPC_DEC_TRUNCATED);
        } else {
            s_cnt = dec_u32(p + G.runs_off);
            s_pos = G.runs_off + 4;
        }
    }
    if (__syncthreads_or(tid == 0 && st != DEC_NONE)) goto finish;

    // temporal runs: <HHH fff> + presence mask + f32 per present non-key frame
    {
        const long long n_runs = s_cnt;
        long long done = 0;
        while (done < n_runs) {
            // stage the next window of the run section (coalesced; raw
            // payloads are 16-byte aligned in the arena)
            const long long wbase = s_pos & ~3ll;
            {
                const long long wl = min((long long)PK_WIN, len - wbase);
                const unsigned* src = (const unsigned*)(p + wbase);
                for (long long i = tid; 4 * i < wl; i += PK_THREADS) win32[i] = __ldg(src + i);
            }
            __syncthreads();
            if (tid == 0) {
                const uint8_t* win = (const uint8_t*)win32;
                auto wb = [&](long long x) -> unsigned { return x - wbase < PK_WIN ? win[x - wbase] : dec_u8(p + x); };
                int c = 0;
                long long q = s_pos;
                while (c < PK_BATCH && done + c < n_runs) {
                    if (c > 0 && q + 18 + G.pm > wbase + PK_WIN) break;  // restage
                    if (q + 18 > len) {
                        fail(q, 0, STPC_DEC_TRUNCATED);
                        break;
                    }
                    recs[c++] = q;
                    {
                        const long long key = (long long)(wb(q) | (wb(q + 1) << 8)) * G.tx + (wb(q + 2) | (wb(q + 3) << 8));
                        if (key < s_tend) s_ovl = 1;
                        s_tend = key + (wb(q + 4) | (wb(q + 5) << 8));
                    }
                    if (q + 18 + G.pm > len) {
                        fail(q + 18, 1, STPC_DEC_TRUNCATED);
                        break;
                    }
                    int present = 0;
                    for (int i = 0; i < G.pm; ++i) {
                        unsigned m = wb(q + 18 + i);
                        const int valid_bits = min(8, G.n - 8 * i);
                        if (valid_bits < 8) m &= (1u << valid_bits) - 1u;
                        present += __popc(m);
                    }
                    const int kbit = (wb(q + 18 + (G.k >> 3)) >> (G.k & 7)) & 1;
                    const long long size = 18 + G.pm + 4ll * (present - kbit);
                    if (q + size > len) {
                        const long long o0 = q + 18 + G.pm;
                        fail(o0 + (len - o0) / 4 * 4, 0, STPC_DEC_TRUNCATED);
                        break;
                    }
                    q += size;
                }
                s_nrec = c;
                s_pos = q;
            }
            __syncthreads();
            const int c = s_nrec;
            for (int r = tid; r < c; r += PK_THREADS) {
                const long long q = recs[r];
                const int row = (int)dec_u16(p + q), s = (int)dec_u16(p + q + 2), ln = (int)dec_u16(p + q + 4);
                if (row >= G.ty || ln < 1 || s + ln > G.tx) {
                    fail(q + 18, 0, STPC_DEC_MALFORMED);
                    continue;
                }
                if (q + 18 + G.pm > len) continue;
                const float a = dec_f32(p + q + 6), bb = dec_f32(p + q + 10), cc = dec_f32(p + q + 14);
                long long o = q + 18 + G.pm;
                bool havek = false, trunc = false;
                for (int ch = 0; ch < G.n; ++ch) {
                    if (!((dec_u8(p + q + 18 + (ch >> 3)) >> (ch & 7)) & 1)) continue;
                    float off;
                    if (ch == G.k) {
                        off = cc;
                        havek = true;
                    } else {
                        if (o + 4 > len) {
                            trunc = true;
                            break;
                        }
                        off = dec_f32(p + o);
                        o += 4;
                    }
                    float4* dst = tm + ((long long)ch * G.ty + row) * G.tx;
                    for (int t = s; t < s + ln; ++t) dst[t] = make_float4(a, bb, off, 1.f);
                }
                if (!trunc && !havek) fail(o, 0, STPC_DEC_MALFORMED);
            }
            done += c;
            if (__syncthreads_or(st != DEC_NONE)) goto finish;
        }
    }

    // fallback rows per frame: <I> rows, each <HH> + nr x <HH fff>
    if (tid == 0) {
        s_ch = 0;
        s_left = 0;
        s_done = 0;
        s_fbpos = s_pos;
    }
    __syncthreads();
    for (;;) {
        if (tid == 0) {
            int c = 0;
            long long q = s_pos;
            while (c < PK_BATCH) {
                if (s_left == 0) {
                    if (s_ch == G.n) {
                        s_done = 1;
                        break;
                    }
                    if (q + 4 > len) {
                        fail(q, 0, STPC_DEC_TRUNCATED);
                        break;
                    }
                    const long long nrows = dec_u32(p + q);
                    q += 4;
                    if (nrows > G.ty) {
                        fail(q, 0, STPC_DEC_MALFORMED);
                        break;
                    }
                    s_left = nrows;
                    s_frow = -1;
                    ++s_ch;
                    continue;
                }
                if (q + 4 > len) {
                    fail(q, 0, STPC_DEC_TRUNCATED);
                    break;
                }
                const int row = (int)dec_u16(p + q), nr = (int)dec_u16(p + q + 2);
                q += 4;
                if (row <= s_frow) s_ovl = 1;
                s_frow = row;
                if (row >= G.ty || nr > G.tx) {
                    fail(q, 0, STPC_DEC_MALFORMED);
                    break;
                }
                if (q + 16ll * nr > len) {
                    const int avail = (int)((len - q) / 16);
                    fch[c] = s_ch - 1;
                    frow[c] = row;
                    fnr[c] = avail;
                    recs[c++] = q;
                    fail(q + 16ll * avail, 0, STPC_DEC_TRUNCATED);
                    break;
                }
                fch[c] = s_ch - 1;
                frow[c] = row;
                fnr[c] = nr;
                recs[c++] = q;
                q += 16ll * nr;
                --s_left;
            }
            s_nrec = c;
            s_pos = q;
        }
        __syncthreads();
        const int c = s_nrec;
        const int lane = tid & 31, wid = tid >> 5;
        for (int r = wid; r < c; r += PK_THREADS / 32) {
            float4* dst = tm + ((long long)fch[r] * G.ty + frow[r]) * G.tx;
            for (int i = lane; i < fnr[r]; i += 32) {
                const long long rp = recs[r] + 16ll * i;
                const int s = (int)dec_u16(p + rp), ln = (int)dec_u16(p + rp + 2);
                if (ln < 1 || s + ln > G.tx) {
                    fail(rp + 16, 0, STPC_DEC_MALFORMED);
                    continue;
                }
                if (i > 0 && s < (int)dec_u16(p + rp - 16) + (int)dec_u16(p + rp - 14)) s_ovl = 1;
                const float4 v = make_float4(dec_f32(p + rp + 4), dec_f32(p + rp + 8), dec_f32(p + rp + 12), 2.f);
                for (int t = s; t < s + ln; ++t)
                    if (dst[t].w != 1.f) dst[t] = v;  // temporal coverage wins (remaining mask)
            }
        }
        if (__syncthreads_or(st != DEC_NONE)) goto finish;
        if (s_done) break;
        __syncthreads();
    }

    // residual sections per frame
    for (int ch = 0; ch < G.n; ++ch) {
        ResSec* rs = res + (long long)j * G.n + ch;
        if (tid == 0) {
            const long long q = s_pos;
            if (q + 4 > len) {
                fail(q, 0, STPC_DEC_TRUNCATED);
            } else {
                const long long cnt = dec_u32(p + q);
                s_pos = q + 4;
                s_cnt = cnt;
                if (cnt > G.P) fail(q + 4, 0, STPC_DEC_MALFORMED);
                if (cnt == 0) *rs = ResSec{q + 4, 0, q + 4, q + 4};
            }
            s_end = -1;
            s_flat = 0;
            s_dbad = 0;
            s_vbad = 0;
        }
        if (__syncthreads_or(st != DEC_NONE)) goto finish;
        const long long cnt = s_cnt;
        if (cnt == 0) continue;
        // varints: value i ends at the i-th byte < 0x80 (varint_decode_kernel
        // _kernels.py:435-459); deltas checked as bitstream.py:494-498
        const long long base = s_pos;
        long long found = 0;
        for (long long chunk = base;; chunk += 4 * PK_THREADS) {
            const long long x0 = chunk + 4ll * tid;
            int nt = 0;
            for (int i = 0; i < 4; ++i)
                if (x0 + i < len && dec_u8(p + x0 + i) < 128) ++nt;
            long long tot;
            long long vi = found + block_excl_scan<PK_THREADS>(nt, tot);
            unsigned long long dsum = 0;
            for (int i = 0; i < 4; ++i) {
                const long long x = x0 + i;
                if (x >= len) break;
                if (dec_u8(p + x) >= 128) continue;
                if (vi < cnt) {
                    long long y = x;
                    while (y > base && dec_u8(p + y - 1) >= 128 && x - y < 9) --y;
                    unsigned long long v = 0;
                    for (long long z = y; z <= x; ++z)
                        v |= (unsigned long long)(dec_u8(p + z) & 0x7f) << (7 * (z - y));
                    const long long dlt = (long long)v;
                    if ((vi == 0 ? dlt < 0 : dlt < 1) || dlt > G.P) s_dbad = 1;
                    else dsum += (unsigned long long)dlt;
                    if (vi == cnt - 1) s_end = x + 1;
                }
                ++vi;
            }
            // one shared atomic per warp (a per-thread 64-bit atomic on the one
            // address serialised the block: ~45% of the kernel's instructions)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(STPC_FULL, dsum, o);
            if ((tid & 31) == 0 && dsum) atomicAdd(&s_flat, dsum);
            __syncthreads();
            const long long end = s_end;
            const long long lim = end >= 0 ? end : len;
            // an 11th byte of one value: ten continuation bytes in a row (shift > 63)
            for (int i = 0; i < 4; ++i) {
                const long long x = x0 + i;
                if (x >= lim || x - 9 < base || dec_u8(p + x) < 128) continue;
                bool all = true;
                for (int dd = 1; dd <= 9 && all; ++dd) all = dec_u8(p + x - dd) >= 128;
                if (all) s_vbad = 1;
            }
            found += tot;
            if (__syncthreads_or(end >= 0 || chunk + 4 * PK_THREADS >= len)) break;
        }
        if (tid == 0) {
            const long long end = s_end;
            if (end < 0 || s_vbad) {
                fail(base, 1, STPC_DEC_TRUNCATED);
            } else if (s_dbad) {
                fail(end, 1, STPC_DEC_MALFORMED);
            } else if ((long long)s_flat >= G.P) {
                fail(end, 2, STPC_DEC_MALFORMED);
            } else if (end + 2 * cnt > len) {
                fail(end, 3, STPC_DEC_TRUNCATED);
            } else if (end + 2 * cnt + 4 > len) {
                fail(end + 2 * cnt, 0, STPC_DEC_TRUNCATED);
            } else {
                const long long n_esc = dec_u32(p + end + 2 * cnt);
                const long long pe = end + 2 * cnt + 4;
                if (pe + 4 * n_esc > len) {
                    fail(pe + (len - pe) / 4 * 4, 0, STPC_DEC_TRUNCATED);
                } else {
                    *rs = ResSec{base, cnt, end, pe};
                    s_pos = pe + 4 * n_esc;
                    s_cnt = n_esc;
                }
            }
        }
        if (__syncthreads_or(st != DEC_NONE)) goto finish;
        {
            // escape count (bitstream.py:499-501)
            const long long pc = res[(long long)j * G.n + ch].pos_code;
            int ne = 0;
            for (long long i = tid; i < cnt; i += PK_THREADS) ne += dec_u16(p + pc + 2 * i) == 0xFFFFu;
            long long tot;
            block_excl_scan<PK_THREADS>(ne, tot);
            if (tid == 0 && tot != s_cnt) fail(s_pos, 0, STPC_DEC_MALFORMED);
        }
        if (__syncthreads_or(st != DEC_NONE)) goto finish;
    }
    if (tid == 0 && s_pos != len) fail(s_pos, 0, STPC_DEC_MALFORMED);  // trailing bytes

finish:
    __syncthreads();
    if (tid == 0) {
        pstat[j] = st;
        ovl[j] = st == DEC_NONE && s_ovl ? s_fbpos : 0;
    }
}

// Per pixel of every frame: plane reconstruction from the tile map, exactly
// reconstruct_span's arithmetic; failures counted per blob.  Block per
// (frame, 1024-pixel block), 8 warps; warp w handles mask words w, w + 8,
// w + 16, w + 24.  Only pixels that get a plane range are stored (the point
// mask word of every 32 pixels says which; unproject reads nothing else), and
// the mask word is the warp's ballot, later OR-ed with the residual pixels.
constexpr int RC_WARPS = 8;
__global__ void __launch_bounds__(RC_WARPS * 32) reconstruct_kernel(DecGeom G, Trig tg, const uint8_t* raw,
                                                                    const long long* raw_off, const int* sel,
                                                                    const float4* tmap,
                                                                    const unsigned long long* pstat,
                                                                    const long long* ovl, double* out_r,
                                                                    unsigned* pmask, unsigned long long* failed)
{
    const long long f = blockIdx.y;
    long long chl;
    const int j = (int)dmod(f, G.n, G.rn, chl), ch = (int)chl;
    if (pstat[j] != DEC_NONE || ovl[j]) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long W = (G.P + 31) >> 5;
    const long long pb = (long long)blockIdx.x * 1024;
    const uint8_t* vb = raw + raw_off[sel[j]] + G.bits_off + (long long)ch * G.nb;
    const float4* tm = tmap + f * G.ty * G.tx;
    double* dst = out_r + f * G.P;
    long long ul;
    const int v0 = (int)dmod(pb, G.w, G.rw, ul), u0 = (int)ul;
    int nfail = 0;
    for (int k = wid; k < 32; k += RC_WARPS) {
        const long long wd = (pb >> 5) + k;
        if (wd >= W) break;
        const long long p = pb + 32 * k + lane;
        bool have = false;
        if (p < G.P && ((dec_u8(vb + (p >> 3)) >> (7 - (p & 7))) & 1u)) {
            int v, u;
            if (G.w >= 1024) {  // the block spans at most two rows
                u = u0 + 32 * k + lane;
                v = v0;
                if (u >= G.w) {
                    u -= G.w;
                    ++v;
                }
            } else {
                long long uu;
                v = (int)dmod(p, G.w, G.rw, uu);
                u = (int)uu;
            }
            long long tv, tu;
            if (G.mtw) {
                tv = __umulhi((unsigned)v, G.mth);
                tu = __umulhi((unsigned)u, G.mtw);
            } else {
                long long rv, ru;
                tv = dmod(v, G.th, G.rth, rv);
                tu = dmod(u, G.tw, G.rtw, ru);
            }
            const float4 pl = tm[tv * G.tx + tu];
            if (pl.w != 0.0f) {
                double dx, dy, dz;
                ray_dir(tg, v, u, dx, dy, dz);
                const double den = (dx + (double)pl.x * dy) + (double)pl.y * dz;
                if (fabs(den) < STPC_PARALLEL_EPS) {
                    ++nfail;
                } else {
                    const double r_hat = (double)pl.z / den;
                    if (r_hat <= 0.0 || r_hat > G.r_max) {
                        ++nfail;
                    } else {
                        dst[p] = r_hat;
                        have = true;
                    }
                }
            }
        }
        const unsigned m = __ballot_sync(STPC_FULL, have);
        if (lane == 0) pmask[f * W + wd] = m;
    }
    for (int o = 16; o > 0; o >>= 1) nfail += __shfl_xor_sync(STPC_FULL, nfail, o);
    if (lane == 0 && nfail) atomicAdd(failed + j, (unsigned long long)nfail);
}

// Blobs whose runs are not sorted and disjoint (parse_kernel's order check):
// decode_stream_images' loops replayed in stream order (temporal.py:307-331).
// Block per (frame, blob): every thread walks the records (uniform loads);
// each run's pixels are reconstructed block-parallel, a barrier after each
// run, so a later run overwrites an earlier one and a failed reconstruction
// keeps the earlier value; failures count per (run, pixel) like the
// reference's.  Fallback runs see remaining = valid & ~temporal cover (the
// tile map's w == 1 marks, written only by temporal runs).
__global__ void __launch_bounds__(256) ordered_reconstruct_kernel(DecGeom G, Trig tg, const uint8_t* raw,
                                                                  const long long* raw_off, const int* sel,
                                                                  const float4* tmap,
                                                                  const unsigned long long* pstat,
                                                                  const long long* ovl, double* out_r,
                                                                  unsigned long long* failed)
{
    const int ch = blockIdx.x, j = blockIdx.y;
    if (pstat[j] != DEC_NONE || ovl[j] == 0) return;
    const long long f = (long long)j * G.n + ch;
    const uint8_t* p = raw + raw_off[sel[j]];
    const uint8_t* vb = p + G.bits_off + (long long)ch * G.nb;
    double* dst = out_r + f * G.P;
    for (long long pix = threadIdx.x; pix < G.P; pix += blockDim.x) dst[pix] = __longlong_as_double(DEC_NOPT);
    __syncthreads();
    unsigned long long nfail = 0;
    auto apply = [&](int row, int s, int ln, double a, double b, double c, bool fallback) {
        const int v0 = row * G.th, v1 = min(v0 + G.th, G.h);
        const int u0 = s * G.tw, u1 = min((s + ln) * G.tw, G.w);
        const int cols = u1 - u0;
        const long long cnt = (long long)(v1 - v0) * cols;
        for (long long i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int v = v0 + (int)(i / cols), u = u0 + (int)(i % cols);
            const long long pix = (long long)v * G.w + u;
            if (!((dec_u8(vb + (pix >> 3)) >> (7 - (pix & 7))) & 1u)) continue;
            if (fallback && tmap[(f * G.ty + row) * G.tx + u / G.tw].w == 1.f) continue;
            double dx, dy, dz;
            ray_dir(tg, v, u, dx, dy, dz);
            const double den = (dx + a * dy) + b * dz;
            if (fabs(den) < STPC_PARALLEL_EPS) {
                ++nfail;
                continue;
            }
            const double r_hat = c / den;
            if (r_hat <= 0.0 || r_hat > G.r_max) {
                ++nfail;
                continue;
            }
            dst[pix] = r_hat;
        }
        __syncthreads();
    };
    // temporal runs <HHH fff> + presence mask + f32 per present non-key frame
    long long q = G.runs_off;
    const long long n_runs = dec_u32(p + q);
    q += 4;
    for (long long r = 0; r < n_runs; ++r) {
        const int row = (int)dec_u16(p + q), s = (int)dec_u16(p + q + 2), ln = (int)dec_u16(p + q + 4);
        const double a = dec_f32(p + q + 6), b = dec_f32(p + q + 10), c = dec_f32(p + q + 14);
        int extra = 0, before = 0;
        bool pres = false;
        for (int c2 = 0; c2 < G.n; ++c2) {
            if (!((dec_u8(p + q + 18 + (c2 >> 3)) >> (c2 & 7)) & 1u)) continue;
            if (c2 == ch) pres = true;
            if (c2 == G.k) continue;
            if (c2 < ch) ++before;
            ++extra;
        }
        if (pres) apply(row, s, ln, a, b, ch == G.k ? c : (double)dec_f32(p + q + 18 + G.pm + 4 * before), false);
        q += 18 + G.pm + 4ll * extra;
    }
    // fallback rows: per frame <I> rows, each <HH> + nr x <HH fff>
    q = ovl[j];
    for (int c2 = 0; c2 < G.n; ++c2) {
        const long long nrows = dec_u32(p + q);
        q += 4;
        for (long long rr = 0; rr < nrows; ++rr) {
            const int row = (int)dec_u16(p + q), nr = (int)dec_u16(p + q + 2);
            q += 4;
            if (c2 == ch)
                for (int i = 0; i < nr; ++i) {
                    const uint8_t* rp = p + q + 16ll * i;
                    apply(row, (int)dec_u16(rp), (int)dec_u16(rp + 2), dec_f32(rp + 4), dec_f32(rp + 8),
                          dec_f32(rp + 12), true);
                }
            q += 16ll * nr;
        }
    }
    for (int o = 16; o > 0; o >>= 1) nfail += __shfl_xor_sync(STPC_FULL, nfail, o);
    if ((threadIdx.x & 31) == 0 && nfail) atomicAdd(failed + j, nfail);
}

// Residual pixels override (rng_out[vs, us] = ranges, temporal.py:336-338):
// block per (frame, blob); the same terminator scan as parse_kernel, with
// block scans carrying value index, pixel index (cumsum of deltas) and escape
// rank across 1 KB chunks.  The section was validated by parse_kernel.
__global__ void __launch_bounds__(PK_THREADS) residual_kernel(DecGeom G, const uint8_t* raw, const long long* raw_off,
                                                              const int* sel, const ResSec* res,
                                                              const unsigned long long* pstat, double* out_r,
                                                              unsigned* pmask)
{
    const int ch = blockIdx.x, j = blockIdx.y;
    if (pstat[j] != DEC_NONE) return;
    const ResSec rs = res[(long long)j * G.n + ch];
    if (rs.cnt == 0) return;
    const uint8_t* p = raw + raw_off[sel[j]];
    double* dst = out_r + ((long long)j * G.n + ch) * G.P;
    unsigned* pm = pmask + ((long long)j * G.n + ch) * ((G.P + 31) >> 5);
    const int tid = threadIdx.x;
    long long c_idx = 0, c_flat = 0, c_esc = 0;
    for (long long chunk = rs.pos_var; chunk < rs.pos_code; chunk += 4 * PK_THREADS) {
        const long long x0 = chunk + 4ll * tid;
        long long dv[4];
        int term[4];
        int nv = 0;
        long long dsum = 0;
        int ne = 0;
        for (int i = 0; i < 4; ++i) {
            const long long x = x0 + i;
            term[i] = 0;
            if (x >= rs.pos_code || dec_u8(p + x) >= 128) continue;
            long long y = x;
            while (y > rs.pos_var && dec_u8(p + y - 1) >= 128) --y;
            unsigned long long v = 0;
            for (long long z = y; z <= x; ++z) v |= (unsigned long long)(dec_u8(p + z) & 0x7f) << (7 * (z - y));
            dv[i] = (long long)v;
            term[i] = 1;
            ++nv;
            dsum += (long long)v;
        }
        // value count and delta sum in one scan: nv sums to at most 4 *
        // PK_THREADS < 2^11 per chunk, so it never carries into the sum
        long long t_idx, t_flat, t_esc, t_pk;
        const long long b_pk = block_excl_scan<PK_THREADS>((dsum << 11) | nv, t_pk);
        const long long b_idx = c_idx + (b_pk & 2047);
        const long long b_flat = c_flat + (b_pk >> 11);
        t_idx = t_pk & 2047;
        t_flat = t_pk >> 11;
        // escape flags need the value index, so count them after the index scan
        {
            long long vi = b_idx;
            for (int i = 0; i < 4; ++i)
                if (term[i]) ne += dec_u16(p + rs.pos_code + 2 * vi++) == 0xFFFFu;
        }
        const long long b_esc = c_esc + block_excl_scan<PK_THREADS>(ne, t_esc);
        long long vi = b_idx, flat = b_flat, ei = b_esc;
        long long cw = -1;
        unsigned bits = 0;
        for (int i = 0; i < 4; ++i) {
            if (!term[i]) continue;
            flat += dv[i];
            const unsigned code = dec_u16(p + rs.pos_code + 2 * vi);
            double r;
            if (code == 0xFFFFu) r = (double)dec_f32(p + rs.pos_esc + 4 * ei++);
            else r = (double)code * G.quant;
            if (flat >= 0 && flat < G.P) {
                dst[flat] = r;
                if ((flat >> 5) != cw) {  // one atomic per distinct mask word of this thread's values
                    if (cw >= 0) atomicOr(pm + cw, bits);
                    cw = flat >> 5;
                    bits = 0;
                }
                bits |= 1u << (flat & 31);
            }
            ++vi;
        }
        if (cw >= 0) atomicOr(pm + cw, bits);
        c_idx += t_idx;
        c_flat += t_flat;
        c_esc += t_esc;
    }
}

// points per (frame, 1024-pixel block) = popcounts of the block's 32 point
// mask words (blocks never straddle frames); blobs whose runs overlap have
// no mask (ordered_reconstruct_kernel) and are counted from the range image
__global__ void __launch_bounds__(256) count_points_kernel(DecGeom G, const double* out_r, const unsigned* pmask,
                                                           const unsigned long long* pstat, const long long* ovl,
                                                           long long bpf, long long F, int* blk_count)
{
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= bpf * F) return;
    const long long f = id / bpf, bk = id - f * bpf;
    long long fch;
    const int j = (int)dmod(f, G.n, G.rn, fch);
    int t = 0;
    if (pstat[j] == DEC_NONE) {
        const long long W = (G.P + 31) >> 5;
        const long long w0 = bk * 32, w1 = min(w0 + 32, W);
        if (ovl[j]) {
            for (long long p = w0 * 32; p < min(w1 * 32, G.P); ++p)
                t += __double_as_longlong(out_r[f * G.P + p]) != DEC_NOPT;
        } else {
            for (long long w = w0; w < w1; ++w) t += __popc(pmask[f * W + w]);
        }
    }
    blk_count[id] = t;
}

// warp per frame: exclusive scan of its block counts in place + frame total
__global__ void frame_scan_kernel(int* blk_count, long long bpf, long long F, long long* frame_count)
{
    const long long f = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (f >= F) return;
    const int lane = threadIdx.x & 31;
    int* c = blk_count + f * bpf;
    int carry = 0;
    for (long long i0 = 0; i0 < bpf; i0 += 32) {
        const long long i = i0 + lane;
        const int v = i < bpf ? c[i] : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(STPC_FULL, x, o);
            if (lane >= o) x += t;
        }
        if (i < bpf) c[i] = carry + x - v;
        carry += __shfl_sync(STPC_FULL, x, 31);
    }
    if (lane == 0) frame_count[f] = carry;
}

// single block: exclusive scan over the frame totals
__global__ void __launch_bounds__(1024) frame_offset_kernel(const long long* frame_count, long long F,
                                                            long long* frame_off)
{
    long long carry = 0;
    for (long long i0 = 0; i0 < F; i0 += 1024) {
        const long long i = i0 + threadIdx.x;
        const long long v = i < F ? frame_count[i] : 0;
        long long tot;
        const long long e = block_excl_scan<1024>(v, tot);
        if (i < F) frame_off[i] = carry + e;
        carry += tot;
    }
}

// points = r * d in row-major pixel order per frame, then
// p' = R^-1 p + T^-1 as fma(z, r2, fma(y, r1, x r0)) + t (xform_coord).
// Block per (frame, 1024-pixel block), 8 warps; warp w handles mask words
// w, w + 8, w + 16, w + 24 of the block.  The block's 32 point-mask words
// (for blobs with overlapping runs: ballots over the range image) and their
// exclusive popcount scan give every word's output offset up front, so the
// per-word work is the points alone; the inverse transform, the output base
// and the block's first pixel coordinates are loaded once per block.
constexpr int UP_WARPS = 8;
#ifndef STPC_UP_MINB
#define STPC_UP_MINB 5
#endif
// Block per 1024 pixels of one frame; warp w owns the block's words 4w..4w+3
// (128 consecutive pixels).  Every point of the block lands in a shared
// staging area at its rank within the block (the block's points are
// contiguous in the output), then the block writes its 3 x count doubles
// with 16-byte stores.  Each lane issues the range loads of all four of its
// words before any arithmetic.
__global__ void __launch_bounds__(UP_WARPS * 32, STPC_UP_MINB) unproject_kernel(DecGeom G, Trig tg, const double* out_r,
                                                                  const unsigned* pmask,
                                                                  const unsigned long long* pstat,
                                                                  const long long* ovl, const int* blk_off,
                                                                  const long long* frame_off, const double* xf_inv,
                                                                  double* pts)
{
    const long long f = blockIdx.y;
    long long fch;
    const int j = (int)dmod(f, G.n, G.rn, fch);
    if (pstat[j] != DEC_NONE) return;
    __shared__ unsigned s_m[32];
    __shared__ int s_off[33];
    __shared__ double s_R[12];
    __shared__ long long s_base;
    __shared__ __align__(16) double stage[3 * 1024 + 2];  // the block's points, xyz interleaved
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long W = (G.P + 31) >> 5;
    const long long pb = (long long)blockIdx.x * 1024;  // the block's first pixel
    const bool ord = ovl[j] != 0;
    for (int k = wid; k < 32; k += UP_WARPS) {
        const long long wd = (pb >> 5) + k;
        unsigned m = 0;
        if (ord) {
            const long long p = pb + 32 * k + lane;
            m = __ballot_sync(STPC_FULL, p < G.P && __double_as_longlong(out_r[f * G.P + p]) != DEC_NOPT);
        } else if (wd < W) {
            m = pmask[f * W + wd];
        }
        if (lane == 0) s_m[k] = m;
    }
    if (threadIdx.x < 12) s_R[threadIdx.x] = xf_inv[12 * f + threadIdx.x];
    if (threadIdx.x == 12) s_base = frame_off[f] + blk_off[f * gridDim.x + blockIdx.x];
    __syncthreads();
    if (wid == 0) {
        const int c = __popc(s_m[lane]);
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(STPC_FULL, x, o);
            if (lane >= o) x += t;
        }
        s_off[lane] = x - c;
        if (lane == 31) s_off[32] = x;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    const double* img = out_r + f * G.P;
    double r[4];
    unsigned mk[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = 4 * wid + i;
        mk[i] = s_m[k];
        r[i] = (mk[i] >> lane) & 1u ? img[pb + 32 * k + lane] : 0.0;
    }
    long long ul;
    const int v0 = (int)dmod(pb, G.w, G.rw, ul), u0 = (int)ul;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = 4 * wid + i;
        if ((mk[i] >> lane) & 1u) {
            int v, u;
            if (G.w >= 1024) {  // the block spans at most two rows
                u = u0 + 32 * k + lane;
                v = v0;
                if (u >= G.w) {
                    u -= G.w;
                    ++v;
                }
            } else {
                long long uu;
                v = (int)dmod(pb + 32 * k + lane, G.w, G.rw, uu);
                u = (int)uu;
            }
            double dx, dy, dz;
            ray_dir(tg, v, u, dx, dy, dz);
            const double x = r[i] * dx, y = r[i] * dy, z = r[i] * dz;
            double* o = stage + 3 * (s_off[k] + __popc(mk[i] & lt));
            o[0] = xform_coord(x, y, z, s_R[0], s_R[1], s_R[2], s_R[9]);
            o[1] = xform_coord(x, y, z, s_R[3], s_R[4], s_R[5], s_R[10]);
            o[2] = xform_coord(x, y, z, s_R[6], s_R[7], s_R[8], s_R[11]);
        }
    }
    __syncthreads();
    // 3 x count doubles to pts + 3 s_base: a leading double when that start is
    // odd, then 16-byte stores
    const int nd = 3 * s_off[32];
    if (nd == 0) return;
    double* dst = pts + 3 * s_base;
    const int head = (int)((reinterpret_cast<uintptr_t>(dst) >> 3) & 1);
    if (head && threadIdx.x == 0) dst[0] = stage[0];
    const int n2 = (nd - head) >> 1;
    double2* d2 = reinterpret_cast<double2*>(dst + head);
    for (int q = threadIdx.x; q < n2; q += blockDim.x) d2[q] = make_double2(stage[head + 2 * q], stage[head + 2 * q + 1]);
    if (((nd - head) & 1) && threadIdx.x == 0) dst[nd - 1] = stage[nd - 1];
}

}  // namespace stpc

using namespace stpc;

#define DCK(x)                                                                        \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            set_last_error(std::string(#x) + ": " + cudaGetErrorString(e_));          \
            return STPC_ERR_CUDA;                                                     \
        }                                                                             \
    } while (0)
#define DRET(x)                  \
    do {                         \
        int r_ = (x);            \
        if (r_) return r_;       \
    } while (0)

struct stpc_decoder {
    // phase 1
    int n = 0;
    std::vector<long long> raw_len, raw_off;
    std::vector<int> ok;
    const uint8_t* d_blob_base = nullptr;
    DevBuf blobs, boff, skip, raw, roff, rlen, crcbad, hstat, okdev, heads, segcrc;
    // phase 2
    int m = 0;
    DecGeom G{};
    long long F = 0, bpf = 0, total = 0;
    DevBuf sel, tmap, res, pstat, ovl, outr, pmask, trig, xfi, blkcnt, fcnt, foff, failed, pts;
    std::vector<unsigned long long> h_pstat;
    const double* last_points = nullptr;
    // host output path: pinned double buffer + copy threads
    HostBuf stage[2];
    HostBuf stage_in;  // gathered host blobs (stpc_decoder_load_gather)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~stpc_decoder()
    {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
};

namespace {

// memcpy with the destination's page faults spread over host threads (a
// fresh numpy array is first touched here)
void parallel_memcpy(uint8_t* dst, const uint8_t* src, size_t n)
{
    const size_t min_part = 8u << 20;
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    nt = (unsigned)std::max<size_t>(1, std::min<size_t>(nt, n / min_part));
    if (nt <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t part = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const size_t b = t * part, e = std::min(n, b + part);
        if (b < e) th.emplace_back([=] { std::memcpy(dst + b, src + b, e - b); });
    }
    for (auto& x : th) x.join();
}

// header checks of deserialize in the reference's order (bitstream.py:398-409)
int check_header(const uint8_t* hdr, long long blob_len, long long& raw_len, long long& enc_len)
{
    if (blob_len < DEC_HEADER) return STPC_DEC_TRUNCATED;
    if (std::memcmp(hdr, "STPC", 4) != 0) return STPC_DEC_MALFORMED;
    const unsigned version = hdr[4] | (hdr[5] << 8);
    if (version != 1) return STPC_DEC_VERSION;
    unsigned long long rl = 0, el = 0;
    for (int i = 0; i < 8; ++i) {
        rl |= (unsigned long long)hdr[8 + i] << (8 * i);
        el |= (unsigned long long)hdr[16 + i] << (8 * i);
    }
    if (rl > (1ull << 30)) return STPC_DEC_MALFORMED;
    if (el > (unsigned long long)(blob_len - DEC_HEADER)) return STPC_DEC_TRUNCATED;
    raw_len = (long long)rl;
    enc_len = (long long)el;
    return 0;
}

// decode_tables (huffman.py:80-104) checks; only consulted when raw_len > 0
int check_table(const uint8_t* lens)
{
    long long count[33] = {0};
    int nsym = 0;
    for (int s = 0; s < 256; ++s) {
        if (lens[s] > 32) return STPC_DEC_MALFORMED;
        if (lens[s]) {
            ++count[lens[s]];
            ++nsym;
        }
    }
    unsigned long long code = 0;
    for (int l = 1; l <= 32; ++l) {
        if (code + (unsigned long long)count[l] > (1ull << l)) return STPC_DEC_MALFORMED;
        code = (code + (unsigned long long)count[l]) << 1;
    }
    if (nsym == 0) return STPC_DEC_MALFORMED;
    return 0;
}

}  // namespace

extern "C" {

// RigidTransform validation and inverse of the decoded transforms, on the
// host in native code (decode.py's _transforms_batch, which it replaces, spent
// ~3 ms of numpy per 8192 frames).  The same expressions as the numpy path:
// R^T R, R^T T and the cofactor determinant as explicit left-to-right sums of
// exact float32 x float32 products (no FMA: plain x86-64 code), so the bits
// are identical.  States: 0 passes, 1 fails, 2 within 1e-12 / 1e-9 of the
// tolerance or non-finite -- the caller re-checks those frames with the
// reference's own numpy expressions (motion.py:52-62).
int stpc_decode_transforms(const uint8_t* heads, int64_t head_stride, const int64_t* rows, int32_t m,
                           int32_t n_frames, int32_t offset, double atol, double* xf_inv, int8_t* orth_state,
                           int8_t* det_state)
{
    if (m < 0 || n_frames < 0 || (m > 0 && (!heads || !rows || !xf_inv || !orth_state || !det_state))) {
        set_last_error("invalid arguments");
        return STPC_ERR_ARG;
    }
    for (int32_t j = 0; j < m; ++j) {
        const uint8_t* h = heads + rows[j] * head_stride + offset;
        for (int32_t f = 0; f < n_frames; ++f) {
            float v[12];
            std::memcpy(v, h + 48 * f, 48);  // little-endian float32 (bitstream.py:207-210)
            double R[3][3], T[3];
            for (int a = 0; a < 3; ++a) {
                for (int b = 0; b < 3; ++b) R[a][b] = (double)v[3 * a + b];
                T[a] = (double)v[9 + a];
            }
            bool finite = true;
            for (int a = 0; a < 9; ++a) finite = finite && std::isfinite((double)v[a]);
            bool orth = true, near = !finite;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    const double mab = (R[0][a] * R[0][b] + R[1][a] * R[1][b]) + R[2][a] * R[2][b];
                    const double eye = a == b ? 1.0 : 0.0;
                    const double dev = std::fabs(mab - eye);
                    const double thr = atol + 1e-5 * eye;  // allclose: atol + rtol * |b|
                    orth = orth && dev <= thr;
                    near = near || std::fabs(dev - thr) < 1e-12;
                }
            const double det = (R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) -
                                R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0])) +
                               R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
            const double dtol = atol + 1e-5;
            const bool det_near = !(std::fabs(std::fabs(det - 1.0) - dtol) > 1e-9) || !std::isfinite(det);
            const long long o = ((long long)j * n_frames + f);
            orth_state[o] = near ? 2 : (orth ? 0 : 1);
            det_state[o] = det_near ? 2 : (std::fabs(det - 1.0) <= dtol ? 0 : 1);
            double* x = xf_inv + 12 * o;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) x[3 * a + b] = R[b][a];
            for (int a = 0; a < 3; ++a) x[9 + a] = -((R[0][a] * T[0] + R[1][a] * T[1]) + R[2][a] * T[2]);
        }
    }
    return STPC_OK;
}

int stpc_decoder_create(stpc_decoder** out)
{
    if (!out) return STPC_ERR_ARG;
    *out = new stpc_decoder();
    return STPC_OK;
}

void stpc_decoder_destroy(stpc_decoder* d) { delete d; }

}  // extern "C"

// Phase 1 body.  Blob i starts at offsets[i]; its length is lengths[i] when
// given (gathered, padded layout) else offsets[i+1] - offsets[i].
static int decoder_load_impl(stpc_decoder* d, const uint8_t* blobs, int32_t blobs_on_device, const int64_t* offsets,
                             const int64_t* lengths, int32_t n, int32_t* status, void* stream)
{
    if (!d || !blobs || !offsets || !status || n < 1) return STPC_ERR_ARG;
    auto blen_of = [&](int i) -> long long { return lengths ? lengths[i] : offsets[i + 1] - offsets[i]; };
    cudaStream_t s = (cudaStream_t)stream;
    d->n = n;
    d->m = 0;
    const long long arena = offsets[n];
    // headers (on the host already, or a small gather)
    std::vector<uint8_t> hdr((size_t)n * DEC_HEADER, 0);
    if (blobs_on_device) {
        std::vector<long long> blen(n);
        for (int i = 0; i < n; ++i) blen[i] = blen_of(i);
        DRET(d->boff.ensure(sizeof(long long) * 2 * n));
        DRET(d->heads.ensure((size_t)n * DEC_HEADER));
        DCK(cudaMemcpyAsync(d->boff.p, offsets, sizeof(long long) * n, cudaMemcpyHostToDevice, s));
        DCK(cudaMemcpyAsync(d->boff.as<long long>() + n, blen.data(), sizeof(long long) * n, cudaMemcpyHostToDevice,
                            s));
        STPC_LAUNCH();
        blob_headers_kernel<<<n, 128, 0, s>>>(blobs, d->boff.as<long long>(), d->boff.as<long long>() + n,
                                              d->heads.as<uint8_t>());
        DCK(cudaGetLastError());
        DCK(cudaMemcpyAsync(hdr.data(), d->heads.p, (size_t)n * DEC_HEADER, cudaMemcpyDeviceToHost, s));
        DCK(cudaStreamSynchronize(s));
    } else {
        for (int i = 0; i < n; ++i) {
            const long long len = std::min<long long>(blen_of(i), DEC_HEADER);
            if (len > 0) std::memcpy(hdr.data() + (size_t)i * DEC_HEADER, blobs + offsets[i], len);
        }
    }
    d->raw_len.assign(n, 0);
    d->raw_off.assign(n + 1, 0);
    d->ok.assign(n, 0);
    std::vector<int> pre(n, 0), skip(n, 1), table(n, 0);
    std::vector<long long> hdr_enc(n, 0);
    long long ro = 0;
    for (int i = 0; i < n; ++i) {
        long long rl = 0, el = 0;
        const uint8_t* h = hdr.data() + (size_t)i * DEC_HEADER;
        pre[i] = check_header(h, blen_of(i), rl, el);
        hdr_enc[i] = el;
        d->raw_off[i] = ro;
        if (!pre[i]) {
            d->raw_len[i] = rl;
            table[i] = rl > 0 ? check_table(h + 28) : 0;
            skip[i] = 0;
            ro += (rl + 15) / 16 * 16;
        }
    }
    d->raw_off[n] = ro;
    // device buffers
    if (blobs_on_device) {
        d->d_blob_base = blobs;
    } else {
        DRET(d->blobs.ensure(std::max<long long>(arena, 1)));
        DCK(cudaMemcpyAsync(d->blobs.p, blobs, arena, cudaMemcpyHostToDevice, s));
        d->d_blob_base = d->blobs.as<uint8_t>();
    }
    // per-blob tables for the CRC/Huffman kernels: skip = header or table error
    std::vector<int> skip_huff(n);
    for (int i = 0; i < n; ++i) skip_huff[i] = skip[i] || table[i];
    DRET(d->boff.ensure(sizeof(long long) * 2 * n));
    DRET(d->skip.ensure(sizeof(int) * 2 * n));
    DRET(d->roff.ensure(sizeof(long long) * (n + 1)));
    DRET(d->rlen.ensure(sizeof(long long) * n));
    DRET(d->crcbad.ensure(sizeof(int) * 2 * n));
    DRET(d->raw.ensure(std::max<long long>(ro, 16)));
    DCK(cudaMemcpyAsync(d->boff.p, offsets, sizeof(long long) * n, cudaMemcpyHostToDevice, s));
    DCK(cudaMemcpyAsync(d->skip.p, skip.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    DCK(cudaMemcpyAsync(d->skip.as<int>() + n, skip_huff.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    DCK(cudaMemcpyAsync(d->roff.p, d->raw_off.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, s));
    DCK(cudaMemcpyAsync(d->rlen.p, d->raw_len.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, s));
    DCK(cudaMemsetAsync(d->crcbad.p, 0, sizeof(int) * 2 * n, s));
    DecCrcK ck;
    for (int l = 0; l < 8; ++l) ck.lvl[l] = dec_x8nmodp((unsigned long long)DC_PIECE << l);
    ck.chunk = dec_x8nmodp((unsigned long long)DC_CHUNK);
    STPC_LAUNCH();
    crc_blob_kernel<<<n, 256, 0, s>>>(d->d_blob_base, d->boff.as<long long>(), d->skip.as<int>(), ck,
                                      d->crcbad.as<int>());
    {
        DecCrcF kf;
        for (int l = 0; l < 5; ++l) kf.x256[l] = dec_x8nmodp((unsigned long long)DCF_PIECE << l);
        kf.warp = dec_x8nmodp(32ull * DCF_PIECE);
        long long max_enc = 0;
        for (int i = 0; i < n; ++i)
            if (!skip[i]) max_enc = std::max<long long>(max_enc, hdr_enc[i]);
        const int max_segs = (int)std::max<long long>(1, (max_enc / DCF_PIECE + 31) / 32);
        DRET(d->segcrc.ensure(sizeof(unsigned) * (size_t)n * max_segs));
        const int per_block = DCF_WARPS * DCF_SEGS_PER_WARP;
        STPC_LAUNCH();
        crc_dseg_kernel<<<dim3((unsigned)((max_segs + per_block - 1) / per_block), (unsigned)n), DCF_WARPS * 32, 0,
                          s>>>(d->d_blob_base, d->boff.as<long long>(), d->skip.as<int>(), kf, max_segs,
                               d->segcrc.as<unsigned>());
        STPC_LAUNCH();
        crc_dfinish_kernel<<<n, 32, 0, s>>>(d->d_blob_base, d->boff.as<long long>(), d->skip.as<int>(), kf, max_segs,
                                            d->segcrc.as<unsigned>(), d->crcbad.as<int>());
    }
    STPC_LAUNCH();
    huff_decode_kernel<<<n, HD_THREADS, 0, s>>>(d->d_blob_base, d->boff.as<long long>(), d->skip.as<int>() + n,
                                                d->raw.as<uint8_t>(), d->roff.as<long long>(),
                                                d->crcbad.as<int>() + n);
    DCK(cudaGetLastError());
    std::vector<int> res(2 * (size_t)n);
    DCK(cudaMemcpyAsync(res.data(), d->crcbad.p, sizeof(int) * 2 * n, cudaMemcpyDeviceToHost, s));
    DCK(cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i) {
        int st = pre[i];
        if (!st && res[i]) st = STPC_DEC_CHECKSUM;
        if (!st && table[i]) st = table[i];
        if (!st && res[n + i]) st = res[n + i] == 1 ? STPC_DEC_TRUNCATED : STPC_DEC_MALFORMED;
        status[i] = st;
        d->ok[i] = st == 0;
    }
    DRET(d->okdev.ensure(sizeof(int) * n));
    DCK(cudaMemcpyAsync(d->okdev.p, d->ok.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    return STPC_OK;
}

extern "C" {

int stpc_decoder_load(stpc_decoder* d, const uint8_t* blobs, int32_t blobs_on_device, const int64_t* offsets,
                      int32_t n, int32_t* status, void* stream)
{
    return decoder_load_impl(d, blobs, blobs_on_device, offsets, nullptr, n, status, stream);
}

int stpc_decoder_load_gather(stpc_decoder* d, const uint8_t* const* blobs, const int64_t* lengths, int32_t n,
                             int32_t* status, void* stream)
{
    if (!d || !blobs || !lengths || !status || n < 1) return STPC_ERR_ARG;
    std::vector<int64_t> off(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        if (lengths[i] < 0 || (!blobs[i] && lengths[i] > 0)) return STPC_ERR_ARG;
        off[i + 1] = off[i] + (lengths[i] + 15) / 16 * 16;
    }
    DRET(d->stage_in.ensure((size_t)std::max<int64_t>(off[n], 16)));
    uint8_t* dst = d->stage_in.as<uint8_t>();
    // threads over contiguous runs of blobs; each blob's tail pad is zeroed
    const unsigned nt = std::max(1u, std::min(16u, std::min((unsigned)n, std::thread::hardware_concurrency())));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        th.emplace_back([&, t] {
            for (int i = (int)((long long)n * t / nt); i < (int)((long long)n * (t + 1) / nt); ++i) {
                if (lengths[i] > 0) std::memcpy(dst + off[i], blobs[i], (size_t)lengths[i]);
                std::memset(dst + off[i] + lengths[i], 0, (size_t)(off[i + 1] - off[i] - lengths[i]));
            }
        });
    }
    for (auto& x : th) x.join();
    // blob i occupies [off[i], off[i] + lengths[i]) of the pinned arena: the
    // H2D of the whole arena runs at pinned speed, headers are read in place
    return decoder_load_impl(d, dst, 0, off.data(), lengths, n, status, stream);
}

int stpc_decoder_heads(stpc_decoder* d, int32_t head_cap, uint8_t* h_heads, int64_t* h_raw_len, void* stream)
{
    if (!d || d->n < 1 || head_cap < 1 || !h_heads) return STPC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    DRET(d->heads.ensure((size_t)d->n * head_cap));
    STPC_LAUNCH();
    heads_kernel<<<d->n, 256, 0, s>>>(d->raw.as<uint8_t>(), d->roff.as<long long>(), d->rlen.as<long long>(),
                                      d->okdev.as<int>(), head_cap, d->heads.as<uint8_t>());
    DCK(cudaGetLastError());
    DCK(cudaMemcpyAsync(h_heads, d->heads.p, (size_t)d->n * head_cap, cudaMemcpyDeviceToHost, s));
    DCK(cudaStreamSynchronize(s));
    if (h_raw_len)
        for (int i = 0; i < d->n; ++i) h_raw_len[i] = d->raw_len[i];
    return STPC_OK;
}

int stpc_decoder_frames(stpc_decoder* d, const stpc_decode_geom* g, const int32_t* sel, int32_t m,
                        const double* sin_theta, const double* cos_theta, const double* sin_phi,
                        const double* cos_phi, const double* xf_inv, int64_t* frame_counts, int64_t* status,
                        int64_t* failed, void* stream)
{
    if (!d || !g || !sel || m < 1 || !sin_theta || !cos_theta || !sin_phi || !cos_phi || !xf_inv ||
        !frame_counts || !status || !failed)
        return STPC_ERR_ARG;
    if (g->w < 1 || g->h < 1 || g->tile_w < 1 || g->tile_h < 1 || g->n_frames < 1 || g->k_index < 0 ||
        g->k_index >= g->n_frames)
        return STPC_ERR_ARG;
    for (int j = 0; j < m; ++j)
        if (sel[j] < 0 || sel[j] >= d->n || !d->ok[sel[j]]) return STPC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    DecGeom& G = d->G;
    G.w = g->w;
    G.h = g->h;
    G.tw = g->tile_w;
    G.th = g->tile_h;
    G.tx = (g->w + g->tile_w - 1) / g->tile_w;
    G.ty = (g->h + g->tile_h - 1) / g->tile_h;
    G.n = g->n_frames;
    G.k = g->k_index;
    G.pm = (g->n_frames + 7) / 8;
    G.P = (long long)g->w * g->h;
    G.nb = (G.P + 7) / 8;
    G.bits_off = 57 + 48ll * G.n;
    G.runs_off = G.bits_off + (long long)G.n * G.nb;
    G.quant = g->range_quant;
    G.r_max = g->r_max;
    G.rw = 1.0 / G.w;
    G.rtw = 1.0 / G.tw;
    G.rth = 1.0 / G.th;
    G.rn = 1.0 / G.n;
    // (a divisor of 1 would need m = 2^32: those geometries keep dmod)
    const bool small = G.w < 65536 && G.h < 65536 && G.tw < 65536 && G.th < 65536 && G.tw > 1 && G.th > 1;
    G.mtw = small ? (unsigned)((0x100000000ull + G.tw - 1) / G.tw) : 0u;
    G.mth = small ? (unsigned)((0x100000000ull + G.th - 1) / G.th) : 0u;
    d->m = m;
    d->F = (long long)m * G.n;
    d->bpf = (G.P + 1023) / 1024;
    const long long F = d->F, bpf = d->bpf;
    DRET(d->sel.ensure(sizeof(int) * m));
    DRET(d->tmap.ensure(sizeof(float4) * F * G.ty * G.tx));
    DRET(d->res.ensure(sizeof(ResSec) * F));
    DRET(d->pstat.ensure(sizeof(unsigned long long) * m));
    DRET(d->ovl.ensure(sizeof(long long) * m));
    DRET(d->outr.ensure(sizeof(double) * F * G.P));
    DRET(d->pmask.ensure(sizeof(unsigned) * F * ((G.P + 31) >> 5)));
    DRET(d->trig.ensure(sizeof(double) * 2 * (G.w + G.h)));
    DRET(d->xfi.ensure(sizeof(double) * 12 * F));
    DRET(d->blkcnt.ensure(sizeof(int) * F * bpf));
    DRET(d->fcnt.ensure(sizeof(long long) * F));
    DRET(d->foff.ensure(sizeof(long long) * F));
    DRET(d->failed.ensure(sizeof(unsigned long long) * m));
    DCK(cudaMemcpyAsync(d->sel.p, sel, sizeof(int) * m, cudaMemcpyHostToDevice, s));
    double* tr = d->trig.as<double>();
    DCK(cudaMemcpyAsync(tr, sin_theta, sizeof(double) * G.w, cudaMemcpyHostToDevice, s));
    DCK(cudaMemcpyAsync(tr + G.w, cos_theta, sizeof(double) * G.w, cudaMemcpyHostToDevice, s));
    DCK(cudaMemcpyAsync(tr + 2 * G.w, sin_phi, sizeof(double) * G.h, cudaMemcpyHostToDevice, s));
    DCK(cudaMemcpyAsync(tr + 2 * G.w + G.h, cos_phi, sizeof(double) * G.h, cudaMemcpyHostToDevice, s));
    DCK(cudaMemcpyAsync(d->xfi.p, xf_inv, sizeof(double) * 12 * F, cudaMemcpyHostToDevice, s));
    DCK(cudaMemsetAsync(d->failed.p, 0, sizeof(unsigned long long) * m, s));
    Trig tg{tr, tr + G.w, tr + 2 * G.w, tr + 2 * G.w + G.h};
    const uint8_t* raw = d->raw.as<uint8_t>();
    const long long* roff = d->roff.as<long long>();
    const unsigned long long* pst = d->pstat.as<unsigned long long>();
    STPC_LAUNCH();
    parse_kernel<<<m, PK_THREADS, 0, s>>>(G, raw, roff, d->rlen.as<long long>(), d->sel.as<int>(),
                                          d->tmap.as<float4>(), d->res.as<ResSec>(),
                                          d->pstat.as<unsigned long long>(), d->ovl.as<long long>());
    const dim3 fg((unsigned)bpf, (unsigned)F);
    STPC_LAUNCH();
    reconstruct_kernel<<<fg, RC_WARPS * 32, 0, s>>>(G, tg, raw, roff, d->sel.as<int>(), d->tmap.as<float4>(), pst,
                                           d->ovl.as<long long>(), d->outr.as<double>(), d->pmask.as<unsigned>(),
                                           d->failed.as<unsigned long long>());
    STPC_LAUNCH();
    ordered_reconstruct_kernel<<<dim3((unsigned)G.n, (unsigned)m), 256, 0, s>>>(
        G, tg, raw, roff, d->sel.as<int>(), d->tmap.as<float4>(), pst, d->ovl.as<long long>(),
        d->outr.as<double>(), d->failed.as<unsigned long long>());
    STPC_LAUNCH();
    residual_kernel<<<dim3((unsigned)G.n, (unsigned)m), PK_THREADS, 0, s>>>(G, raw, roff, d->sel.as<int>(),
                                                                            d->res.as<ResSec>(), pst,
                                                                            d->outr.as<double>(),
                                                                            d->pmask.as<unsigned>());
    STPC_LAUNCH();
    count_points_kernel<<<(unsigned)((F * bpf + 255) / 256), 256, 0, s>>>(
        G, d->outr.as<double>(), d->pmask.as<unsigned>(), pst, d->ovl.as<long long>(), bpf, F, d->blkcnt.as<int>());
    STPC_LAUNCH();
    frame_scan_kernel<<<(unsigned)((F + 7) / 8), 256, 0, s>>>(d->blkcnt.as<int>(), bpf, F, d->fcnt.as<long long>());
    STPC_LAUNCH();
    frame_offset_kernel<<<1, 1024, 0, s>>>(d->fcnt.as<long long>(), F, d->foff.as<long long>());
    DCK(cudaGetLastError());
    d->h_pstat.resize(m);
    std::vector<unsigned long long> hf(m);
    DCK(cudaMemcpyAsync(frame_counts, d->fcnt.p, sizeof(long long) * F, cudaMemcpyDeviceToHost, s));
    DCK(cudaMemcpyAsync(d->h_pstat.data(), d->pstat.p, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost, s));
    DCK(cudaMemcpyAsync(hf.data(), d->failed.p, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost, s));
    DCK(cudaStreamSynchronize(s));
    d->total = 0;
    for (int j = 0; j < m; ++j) {
        status[j] = d->h_pstat[j] == DEC_NONE ? 0 : (int64_t)d->h_pstat[j];
        failed[j] = (int64_t)hf[j];
    }
    for (long long f = 0; f < F; ++f) d->total += frame_counts[f];
    return STPC_OK;
}

int64_t stpc_decoder_total_points(const stpc_decoder* d) { return d ? d->total : -1; }

const double* stpc_decoder_device_points(const stpc_decoder* d) { return d ? d->last_points : nullptr; }

int stpc_decoder_points(stpc_decoder* d, double* dst, int32_t dst_on_device, int64_t cap_points, void* stream)
{
    if (!d || d->m < 1 || (!dst && !dst_on_device && d->total > 0) || (dst && cap_points < d->total))
        return STPC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    double* out = dst;
    if (!dst_on_device || !dst) {
        DRET(d->pts.ensure(sizeof(double) * 3 * std::max<long long>(d->total, 1)));
        out = d->pts.as<double>();
    }
    Trig tg;
    const double* tr = d->trig.as<double>();
    tg = Trig{tr, tr + d->G.w, tr + 2 * d->G.w, tr + 2 * d->G.w + d->G.h};
    STPC_LAUNCH();
    unproject_kernel<<<dim3((unsigned)d->bpf, (unsigned)d->F), UP_WARPS * 32, 0, s>>>(
        d->G, tg, d->outr.as<double>(), d->pmask.as<unsigned>(), d->pstat.as<unsigned long long>(),
        d->ovl.as<long long>(), d->blkcnt.as<int>(), d->foff.as<long long>(), d->xfi.as<double>(), out);
    DCK(cudaGetLastError());
    if (!dst_on_device && d->total > 0) {
        // D2H through two pinned 128 MB stages; the copy of chunk k into the
        // caller's (pageable) array overlaps the D2H of chunk k+1
        const size_t total_bytes = sizeof(double) * 3 * (size_t)d->total;
        const size_t CH = 128u << 20;
        const size_t nch = (total_bytes + CH - 1) / CH;
        for (int i = 0; i < 2; ++i) {
            DRET(d->stage[i].ensure(std::min(CH, total_bytes)));
            if (!d->ev[i]) DCK(cudaEventCreateWithFlags(&d->ev[i], cudaEventDisableTiming));
        }
        auto issue = [&](size_t k) -> cudaError_t {
            const size_t o = k * CH, n = std::min(CH, total_bytes - o);
            cudaError_t e = cudaMemcpyAsync(d->stage[k & 1].p, (const uint8_t*)out + o, n, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaEventRecord(d->ev[k & 1], s);
            return e;
        };
        DCK(issue(0));
        for (size_t k = 0; k < nch; ++k) {
            DCK(cudaEventSynchronize(d->ev[k & 1]));
            if (k + 1 < nch) DCK(issue(k + 1));
            const size_t o = k * CH, n = std::min(CH, total_bytes - o);
            parallel_memcpy((uint8_t*)dst + o, d->stage[k & 1].as<uint8_t>(), n);
        }
    }
    d->last_points = out;
    DCK(cudaStreamSynchronize(s));
    return STPC_OK;
}

}  // extern "C"
