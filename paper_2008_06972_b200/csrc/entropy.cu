// K3d -- the lossless stage on the device: payload byte histogram, canonical
// Huffman code lengths, MSB-first bit packing, CRC-32 and the blob header.
//
// Replaces huffman.encode_bytes (np.bincount histogram :112,
// code_lengths_from_counts :23-60, canonical_codes :63-77) and
// huffman_encode_kernel (/root/reference/pkg/src/stpc/_kernels.py:363-382),
// plus the header of serialize (/root/reference/pkg/src/stpc/bitstream.py:
// 279-289, zlib.crc32).
#include "kernels.cuh"

namespace stpc {

// ---------------------------------------------------------------- histogram
// grid (chunks, groups); 256-bin shared histogram per block.
// Byte histogram of the raw payload (np.bincount, huffman.py:112): 64 KB per
// block read as 16-byte vectors; 16 private sub-histograms (per warp x lane
// parity) keep same-bin collisions of the skewed payload bytes low.
constexpr int HIST_CHUNK = 65536;
__global__ void __launch_bounds__(256) histogram_kernel(EntropyArgs E)
{
    __shared__ unsigned int h[16][256];
    const int grp = blockIdx.y;
    for (int i = threadIdx.x; i < 16 * 256; i += 256) (&h[0][0])[i] = 0;
    __syncthreads();
    const long long len = E.payload_len[grp];
    const uint8_t* p = E.payload + E.payload_off[grp];  // 16-byte aligned
    const long long b = (long long)blockIdx.x * HIST_CHUNK;
    const long long e = min(b + HIST_CHUNK, len);
    unsigned int* hh = h[((threadIdx.x >> 5) << 1) | (threadIdx.x & 1)];
    for (long long i = b + 16LL * threadIdx.x; i < e; i += 16LL * 256) {
        if (i + 16 <= e) {
            const uint4 v = *reinterpret_cast<const uint4*>(p + i);
            const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 16; ++q) atomicAdd(&hh[(w[q >> 2] >> (8 * (q & 3))) & 0xff], 1u);
        } else {
            for (long long j = i; j < e; ++j) atomicAdd(&hh[p[j]], 1u);
        }
    }
    __syncthreads();
    unsigned int t = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) t += h[k][threadIdx.x];
    if (t) atomicAdd(&E.hist[grp * 256 + threadIdx.x], t);
}

void launch_histogram(const EntropyArgs& E, int max_payload, cudaStream_t s)
{
    if (E.G <= 0) return;
    dim3 grid((max_payload + HIST_CHUNK - 1) / HIST_CHUNK > 0 ? (max_payload + HIST_CHUNK - 1) / HIST_CHUNK : 1, E.G);
    STPC_LAUNCH();
    histogram_kernel<<<grid, 256, 0, s>>>(E);
}

// ------------------------------------------------------------- code lengths
// One warp per group.  Node keys are (weight << 10 | serial): leaves carry
// their symbol as serial, merged nodes 256, 257, ... -- the exact (weight,
// tiebreak) order of the reference's heapq (huffman.py:37-48).
__global__ void __launch_bounds__(32) code_lengths_kernel(EntropyArgs E)
{
    __shared__ unsigned long long key[512];
    __shared__ short parent[512];
    __shared__ uint8_t L[256];
    const int grp = blockIdx.x;
    const int lane = threadIdx.x;
    const unsigned int* hist = E.hist + grp * 256;
    const unsigned long long INACTIVE = ~0ull;
    int nsym = 0;
    for (int i = lane; i < 512; i += 32) {
        unsigned long long k = INACTIVE;
        if (i < 256 && hist[i]) k = ((unsigned long long)hist[i] << 10) | (unsigned)i;
        key[i] = k;
        parent[i] = -1;
        nsym += (i < 256 && hist[i]) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) nsym += __shfl_xor_sync(STPC_FULL, nsym, o);
    __syncwarp();

    // The heap's pops in (weight, serial) order without a heap: the leaves
    // are sorted once (bitonic, in shared memory), and merged nodes are
    // created in non-decreasing (weight, serial) order, so the smallest node
    // is always at the head of one of two queues -- the classic two-queue
    // construction, with the reference's tie-break (a leaf's serial is its
    // symbol < 256 <= any merged node's) decided by the same key compare.
    for (int k = 2; k <= 256; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = lane; t < 128; t += 32) {
                const int i = 2 * j * (t / j) + (t % j), p = i + j;
                const unsigned long long x = key[i], y = key[p];
                const bool up = (i & k) == 0;
                if ((x > y) == up) {
                    key[i] = y;
                    key[p] = x;
                }
            }
            __syncwarp();
        }
    }
    if (lane == 0) {
        int q1 = 0, q2 = 256;  // heads of the leaf queue [0, nsym) and the merged-node queue [256, 256 + m)
        for (int m = 0; m + 1 < nsym; ++m) {
            const int node = 256 + m;
            unsigned long long wsum = 0;
            for (int q = 0; q < 2; ++q) {
                const unsigned long long k1 = q1 < nsym ? key[q1] : INACTIVE;
                const unsigned long long k2 = q2 < node ? key[q2] : INACTIVE;
                const unsigned long long best = k1 < k2 ? k1 : k2;
                if (k1 < k2) ++q1;
                else ++q2;
                parent[(int)(best & 1023u)] = (short)node;
                wsum += best >> 10;
            }
            key[node] = (wsum << 10) | (unsigned)node;
        }
    }
    __syncwarp();
    // depth = merges a leaf's subtree took part in = hops to the root
    int maxlen = 0;
    for (int s = lane; s < 256; s += 32) {
        int d = 0;
        if (hist[s]) {
            if (nsym == 1) d = 1;
            else
                for (int x = parent[s]; x >= 0; x = parent[x]) ++d;
        }
        L[s] = (uint8_t)(d > 255 ? 255 : d);
        maxlen = max(maxlen, d);
    }
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(STPC_FULL, maxlen, o));
    __syncwarp();
    if (lane == 0) {
        if (maxlen > 32) {
            // 32-bit cap repair (huffman.py:52-59); Kraft sum in units of 2^-32 is exact
            unsigned long long kraft = 0;
            for (int s = 0; s < 256; ++s) {
                if (L[s] > 32) L[s] = 32;
                if (L[s]) kraft += 1ull << (32 - L[s]);
            }
            while (kraft > (1ull << 32)) {
                int pick = -1, pl = 0;
                for (int s = 0; s < 256; ++s)
                    if (L[s] > 0 && L[s] < 32 && L[s] > pl) { pl = L[s]; pick = s; }
                kraft -= 1ull << (32 - L[pick]);
                L[pick] += 1;
                kraft += 1ull << (32 - L[pick]);
            }
        }
        // canonical codes (huffman.py:63-77), DEFLATE-style next_code table
        unsigned int bl[34] = {0};
        for (int s = 0; s < 256; ++s) bl[L[s]]++;
        unsigned long long next[34];
        unsigned long long code = 0;
        bl[0] = 0;
        for (int b = 1; b <= 33; ++b) {
            code = (code + bl[b - 1]) << 1;
            next[b] = code;
        }
        unsigned long long bits = 0;
        for (int s = 0; s < 256; ++s) {
            int l = L[s];
            E.lens[grp * 256 + s] = (uint8_t)l;
            unsigned int c = 0;
            if (l) c = (unsigned int)(next[l]++);
            E.codes[grp * 256 + s] = c;
            bits += (unsigned long long)hist[s] * l;
        }
        E.enc_len[grp] = (long long)((bits + 7) / 8);
    }
}

void launch_code_lengths(const EntropyArgs& E, cudaStream_t s)
{
    if (E.G <= 0) return;
    STPC_LAUNCH();
    code_lengths_kernel<<<E.G, 32, 0, s>>>(E);
}

// ------------------------------------------------------------------ packing
constexpr int PACK_THREADS = 256;
constexpr int PACK_PER_THREAD = PACK_CHUNK / PACK_THREADS;  // 16 bytes

__device__ __forceinline__ void chunk_range(const EntropyArgs& E, int grp, int c, long long& b, long long& e)
{
    long long len = E.payload_len[grp];
    b = (long long)c * PACK_CHUNK;
    e = min(b + PACK_CHUNK, len);
}

// phase A: bits per chunk
__global__ void __launch_bounds__(PACK_THREADS) pack_count_kernel(EntropyArgs E)
{
    const int grp = blockIdx.y, c = blockIdx.x;
    long long b, e;
    chunk_range(E, grp, c, b, e);
    if (b >= e) return;
    __shared__ uint8_t lens[256];
    lens[threadIdx.x] = E.lens[grp * 256 + threadIdx.x];
    __syncthreads();
    const uint8_t* p = E.payload + E.payload_off[grp];
    // the same 16-byte-per-thread layout as pack_write (vector loads)
    const long long tb = b + (long long)threadIdx.x * PACK_PER_THREAD;
    const int nq = (int)max(0LL, min((long long)PACK_PER_THREAD, e - tb));
    long long bits = 0;
    if (nq == PACK_PER_THREAD) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(p + tb);
        const uint32_t wv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int q = 0; q < PACK_PER_THREAD; ++q) bits += lens[(wv[q >> 2] >> (8 * (q & 3))) & 0xff];
    } else {
        for (int q = 0; q < nq; ++q) bits += lens[p[tb + q]];
    }
    for (int o = 16; o > 0; o >>= 1) bits += __shfl_xor_sync(STPC_FULL, bits, o);
    __shared__ long long ws[PACK_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = bits;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < PACK_THREADS / 32; ++w) t += ws[w];
        E.chunk_bits[(long long)grp * E.max_chunks + c] = t;
    }
}

// phase B: per-group exclusive scan over chunks (block per group)
__global__ void pack_scan_kernel(EntropyArgs E)
{
    const int grp = blockIdx.x;
    const long long nch = (E.payload_len[grp] + PACK_CHUNK - 1) / PACK_CHUNK;
    long long* cb = E.chunk_bits + (long long)grp * E.max_chunks;
    const int lane = threadIdx.x;  // one warp per group
    // pack_write ORs a chunk's first and last word into the blob (a word can
    // be shared with the neighbouring chunk) and stores the words in between:
    // only those boundary words need to start at zero, so they are cleared
    // here instead of the whole blob arena
    unsigned int* gw = reinterpret_cast<unsigned int*>(E.blobs + E.blob_off[grp] + HDR);
    long long run = 0;
    for (long long base = 0; base < nch; base += 32) {
        const long long c = base + lane;
        const long long v = c < nch ? cb[c] : 0;
        const long long inc = warp_incl_scan_ll(v);
        if (c < nch) {
            const long long O = run + inc - v;
            cb[c] = O;
            gw[O >> 5] = 0u;
            if (v > 0) gw[(O + v - 1) >> 5] = 0u;
        }
        run += __shfl_sync(STPC_FULL, inc, 31);
    }
}

// phase C: compose each chunk's bits in shared memory (big-endian u32 words),
// store interior words, atomicOr the two boundary words shared with
// neighbouring chunks (pack_scan zeroes exactly those words beforehand).
#ifndef STPC_PACK_MINB
#define STPC_PACK_MINB 8  // measured: 1 -> 2.98 ms (pack stage), 8 -> 2.87
#endif
__global__ void __launch_bounds__(PACK_THREADS, STPC_PACK_MINB) pack_write_kernel(EntropyArgs E)
{
    const int grp = blockIdx.y, c = blockIdx.x;
    if (E.prefill) {  // this block's slice of the next grid's +inf fill (16-byte stores)
        const long long bid = (long long)blockIdx.y * gridDim.x + blockIdx.x;
        const long long lo = bid * E.prefill_per;  // 16-byte elements per block: host-computed (no 64-bit divide here)
        const long long cntl = max(0LL, min(E.prefill_per, (E.prefill_n >> 1) - lo));
        ulonglong2* dst = reinterpret_cast<ulonglong2*>(E.prefill) + lo;
        const ulonglong2 inf2 = make_ulonglong2(0x7ff0000000000000ull, 0x7ff0000000000000ull);
        if (cntl <= 0x7fffffffLL) {  // 32-bit loop (always, in practice)
            const int cnt = (int)cntl;
            for (int i = threadIdx.x; i < cnt; i += PACK_THREADS) dst[i] = inf2;
        } else {
            for (long long i = threadIdx.x; i < cntl; i += PACK_THREADS) dst[i] = inf2;
        }
    }
    long long b, e;
    chunk_range(E, grp, c, b, e);
    if (b >= e) return;
    __shared__ uint8_t lens[256];
    __shared__ uint2 cl[256];  // (code, length): one 8-byte load per symbol in the assembly pass
    __shared__ unsigned int buf[PACK_CHUNK + 2];  // 32 bits per byte worst case
    __shared__ int wsum[PACK_THREADS / 32];
    {
        const uint8_t l = E.lens[grp * 256 + threadIdx.x];
        lens[threadIdx.x] = l;
        cl[threadIdx.x] = make_uint2(E.codes[grp * 256 + threadIdx.x], l);
    }
    __syncthreads();
    const uint8_t* p = E.payload + E.payload_off[grp];
    const long long O = E.chunk_bits[(long long)grp * E.max_chunks + c];  // chunk's first bit
    const int lead = (int)(O & 31);
    // each thread owns PACK_PER_THREAD consecutive bytes (a chunk holds at
    // most 4096 * 32 bits: 32-bit counts throughout)
    const long long tb = b + (long long)threadIdx.x * PACK_PER_THREAD;
    const int nq = (int)max(0LL, min((long long)PACK_PER_THREAD, e - tb));
    uint32_t wv[4] = {0u, 0u, 0u, 0u};
    if (nq == PACK_PER_THREAD) {  // 16-byte aligned (payload offsets are 16-aligned)
        const uint4 v4 = *reinterpret_cast<const uint4*>(p + tb);
        wv[0] = v4.x;
        wv[1] = v4.y;
        wv[2] = v4.z;
        wv[3] = v4.w;
    } else {
        for (int q = 0; q < nq; ++q) wv[q >> 2] |= (uint32_t)p[tb + q] << (8 * (q & 3));
    }
    int mybits = 0;
    if (nq == PACK_PER_THREAD) {  // every chunk but a payload's last: no per-byte bound
#pragma unroll
        for (int q = 0; q < PACK_PER_THREAD; ++q) mybits += lens[(wv[q >> 2] >> (8 * (q & 3))) & 0xff];
    } else {
#pragma unroll
        for (int q = 0; q < PACK_PER_THREAD; ++q)
            mybits += q < nq ? lens[(wv[q >> 2] >> (8 * (q & 3))) & 0xff] : 0;
    }
    const int inc = warp_incl_scan(mybits);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    int wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < PACK_THREADS / 32; ++w) {
        const int x = wsum[w];
        wbase += w < wid ? x : 0;
        total += x;
    }
    // zero only the words this chunk fills (~6 bits per byte, not the
    // 32-bit worst case the buffer is sized for)
    const int nwords = (lead + total + 31) >> 5;
    for (int i = threadIdx.x; i < nwords + 1; i += PACK_THREADS) buf[i] = 0;
    __syncthreads();
    // Big-endian word assembly: the accumulator starts with `fill` zero bits
    // (the neighbour's share of the first word); a code is <= 32 bits and
    // fewer than 32 bits are pending, so each symbol emits at most one word.
    // Words strictly inside this thread's bits are plain stores; the first
    // and the last can be shared with a neighbour (atomicOr).
    if (nq > 0) {
        const int pos = lead + wbase + inc - mybits;
        int wi = pos >> 5;
        const int w0 = wi;
        unsigned long long acc = 0;
        int nacc = pos & 31;
#pragma unroll
        for (int q = 0; q < PACK_PER_THREAD; ++q) {
            if (q < nq) {
                const unsigned s = (wv[q >> 2] >> (8 * (q & 3))) & 0xff;
                const uint2 e = cl[s];
                const int l = (int)e.y;
                acc = (acc << l) | e.x;
                nacc += l;
                if (nacc >= 32) {
                    nacc -= 32;
                    const unsigned int word = (unsigned int)(acc >> nacc);
                    if (wi == w0) atomicOr(&buf[wi], word);
                    else buf[wi] = word;
                    ++wi;
                }
            }
        }
        if (nacc > 0) atomicOr(&buf[wi], (unsigned int)(acc << (32 - nacc)));
    }
    __syncthreads();
    unsigned int* gw = reinterpret_cast<unsigned int*>(E.blobs + E.blob_off[grp] + HDR) + (O >> 5);
    for (int i = threadIdx.x; i < nwords; i += PACK_THREADS) {
        const unsigned int le = __byte_perm(buf[i], 0, 0x0123);
        if (i == 0 || i == nwords - 1) {
            if (le) atomicOr(gw + i, le);
        } else {
            gw[i] = le;
        }
    }
}

void launch_pack(const EntropyArgs& E, cudaStream_t s)
{
    if (E.G <= 0 || E.max_chunks <= 0) return;
    dim3 grid(E.max_chunks, E.G);
    STPC_LAUNCH();
    pack_count_kernel<<<grid, PACK_THREADS, 0, s>>>(E);
    STPC_LAUNCH();
    pack_scan_kernel<<<E.G, 32, 0, s>>>(E);
    STPC_LAUNCH();
    EntropyArgs W = E;
    if (W.prefill) {
        const long long nblk = (long long)grid.x * grid.y, n2 = W.prefill_n / 2;
        W.prefill_per = (n2 + nblk - 1) / nblk;
    }
    pack_write_kernel<<<grid, PACK_THREADS, 0, s>>>(W);
}

// --------------------------------------------------------------------- CRC
// zlib CRC-32 (reflected 0xEDB88320).  The encoded payload is cut into
// 256-byte pieces aligned to its END (a virtual zero prefix leaves an
// init-0 CRC register unchanged), each piece's raw CRC is computed by one
// thread, and pieces/segments are combined with x^(8*len) multipliers; the
// 0xFFFFFFFF init is folded in at the end by linearity.
__device__ __forceinline__ unsigned int multmodp(unsigned int a, unsigned int b)
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

__device__ __forceinline__ unsigned int x8nmodp(unsigned long long nbytes)
{
    // x^(8*nbytes) mod p by square-and-multiply
    unsigned int p = 1u << 31;      // x^0
    unsigned int sq = 1u << 23;     // x^8
    while (nbytes) {
        if (nbytes & 1) p = multmodp(sq, p);
        sq = multmodp(sq, sq);
        nbytes >>= 1;
    }
    return p;
}

// slice-by-4 tables for the reflected CRC (T[0] is the classic byte table)
// Slice-by-4 CRC-32 tables (zlib polynomial), built at compile time and
// copied into shared memory per block with coalesced loads.
struct CrcTab4 {
    unsigned int t[4][256];
};
constexpr CrcTab4 make_crc_tab4()
{
    CrcTab4 r{};
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
__device__ const CrcTab4 kCrcTab4 = make_crc_tab4();

__device__ __forceinline__ void crc_tables4(unsigned int (*T)[256])
{
    const unsigned int* src = &kCrcTab4.t[0][0];
    unsigned int* dst = &T[0][0];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
}

constexpr int CRC_WARPS = 8;
constexpr int CRC_SEGS_PER_WARP = 4;  // segments per warp (amortises the table copy)

// grid (segments / CRC_WARPS, groups): warp w of block x handles segment
// x*CRC_WARPS + w = 32 pieces of 256 B of the encoded payload, counted from
// its START; only full pieces are covered here (the < 256 B tail is folded
// in by crc_finish).  The last segment's pieces are end-aligned in the
// 32-slot tree: the missing leading slots act as a zero prefix, which leaves
// an init-0 CRC register unchanged.
// Each lane folds one 256-byte piece; the warp stages the pieces through
// shared memory in 4 rounds of 64 bytes per piece (two pieces per load
// instruction, every sector fully used) into a padded [32][17] word tile, so
// the lane-per-piece fold reads conflict-free shared memory instead of
// 256-byte-strided global words.
constexpr int CRC_SUB = 64;  // bytes per piece per staging round
__global__ void __launch_bounds__(CRC_WARPS * 32) crc_segment_kernel(EntropyArgs E, CrcConsts K)
{
    __shared__ unsigned int T[4][256];
    __shared__ unsigned int stg[CRC_WARPS][32][CRC_SUB / 4 + 1];
    crc_tables4(T);
    const int grp = blockIdx.y;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long L = E.enc_len[grp];
    const long long npieces = L / CRC_PIECE;
    const long long nseg = (npieces + 31) / 32;
    const uint32_t* enc = reinterpret_cast<const uint32_t*>(E.blobs + E.blob_off[grp] + HDR);  // 4-byte aligned
    unsigned int (*tile)[CRC_SUB / 4 + 1] = stg[wib];
    for (int rep = 0; rep < CRC_SEGS_PER_WARP; ++rep) {
        const long long sgi = ((long long)blockIdx.x * CRC_SEGS_PER_WARP + rep) * CRC_WARPS + wib;
        if (sgi >= nseg) return;
        const long long first = sgi * 32;
        const int np = (int)min(32LL, npieces - first);
        const int slot_piece = lane - (32 - np);  // end-aligned
        unsigned int crc = 0;
        for (int r = 0; r < CRC_PIECE / CRC_SUB; ++r) {
#pragma unroll
            for (int it = 0; it < CRC_SUB / 4; ++it) {  // 32 pieces x 16 words, 2 pieces per load
                const int widx = it * 32 + lane;
                const int k = widx >> 4, wd = widx & 15;
                const int pk = k - (32 - np);
                tile[k][wd] = pk >= 0 ? __ldg(enc + ((first + pk) * CRC_PIECE + r * CRC_SUB) / 4 + wd) : 0u;
            }
            __syncwarp();
            if (slot_piece >= 0) {
#pragma unroll
                for (int i = 0; i < CRC_SUB / 4; ++i) {
                    const unsigned int x = crc ^ tile[lane][i];
                    crc = T[3][x & 0xff] ^ T[2][(x >> 8) & 0xff] ^ T[1][(x >> 16) & 0xff] ^ T[0][x >> 24];
                }
            }
            __syncwarp();
        }
        // tree: level l merges blocks of 2^l pieces (256 * 2^l bytes)
#pragma unroll
        for (int l = 0; l < 5; ++l) {
            const unsigned int right = __shfl_down_sync(STPC_FULL, crc, 1 << l);
            if ((lane & ((2 << l) - 1)) == 0) crc = multmodp(K.x256[l], crc) ^ right;
        }
        if (lane == 0) E.seg_crc[(long long)grp * E.max_segs + sgi] = crc;
    }
}

__global__ void crc_finish_kernel(EntropyArgs E, CrcConsts K)
{
    const int grp = blockIdx.x;
    uint8_t* blob = E.blobs + E.blob_off[grp];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) blob[28 + i] = E.lens[grp * 256 + i];
    if (threadIdx.x >= 32) return;
    const long long L = E.enc_len[grp];
    const long long npieces = L / CRC_PIECE;
    const long long nseg = (npieces + 31) / 32;
    // the segments' CRCs combine by Horner's rule; lane l folds a contiguous
    // range of them, weights its partial by x^(8 * bytes of the pieces after
    // the range), and the partials XOR together (CRC is linear)
    unsigned int raw = 0;
    {
        const long long per = (nseg + 31) / 32;
        const long long s0 = threadIdx.x * per, s1 = min(nseg, s0 + per);
        unsigned int r = 0;
        for (long long sgi = s0; sgi < s1; ++sgi) {
            const long long np = min(32LL, npieces - sgi * 32);
            const unsigned int X = np == 32 ? K.seg : x8nmodp((unsigned long long)np * CRC_PIECE);
            r = multmodp(X, r) ^ E.seg_crc[(long long)grp * E.max_segs + sgi];
        }
        if (s0 < s1) {
            const long long after = npieces - min(npieces, s1 * 32);
            r = multmodp(x8nmodp((unsigned long long)after * CRC_PIECE), r);
        }
        raw = __reduce_xor_sync(STPC_FULL, r);
    }
    if (threadIdx.x != 0) return;
    // tail (< 256 bytes) byte-wise
    const uint8_t* enc = blob + HDR;
    const long long tb = npieces * CRC_PIECE;
    if (tb < L) {
        raw = multmodp(x8nmodp((unsigned long long)(L - tb)), raw);
        unsigned int t = 0;
        for (long long i = tb; i < L; ++i) {
            unsigned int c = (t ^ enc[i]) & 0xff;
            for (int k = 0; k < 8; ++k) c = c & 1 ? (c >> 1) ^ 0xedb88320u : c >> 1;
            t = c ^ (t >> 8);
        }
        raw ^= t;
    }
    unsigned int crc = ~(raw ^ multmodp(x8nmodp((unsigned long long)L), 0xffffffffu));
    blob[0] = 'S'; blob[1] = 'T'; blob[2] = 'P'; blob[3] = 'C';
    put_u16(blob + 4, 1);
    put_u16(blob + 6, 0);
    unsigned long long raw_len = (unsigned long long)E.payload_len[grp];
    put_u32(blob + 8, (uint32_t)raw_len);
    put_u32(blob + 12, (uint32_t)(raw_len >> 32));
    put_u32(blob + 16, (uint32_t)L);
    put_u32(blob + 20, (uint32_t)((unsigned long long)L >> 32));
    put_u32(blob + 24, crc);
}

// host-side x^(8n) mod P (same arithmetic as the device helpers)
static unsigned int h_multmodp(unsigned int a, unsigned int b)
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
static unsigned int h_x8nmodp(unsigned long long n)
{
    unsigned int p = 1u << 31, sq = 1u << 23;
    while (n) {
        if (n & 1) p = h_multmodp(sq, p);
        sq = h_multmodp(sq, sq);
        n >>= 1;
    }
    return p;
}

void launch_crc(const EntropyArgs& E, cudaStream_t s)
{
    if (E.G <= 0) return;
    CrcConsts K;
    for (int l = 0; l < 5; ++l) K.x256[l] = h_x8nmodp((unsigned long long)CRC_PIECE << l);
    K.seg = h_x8nmodp(32ull * CRC_PIECE);
    if (E.max_segs > 0) {
        STPC_LAUNCH();
        const long long per_block = (long long)CRC_WARPS * CRC_SEGS_PER_WARP;
        crc_segment_kernel<<<dim3((unsigned)((E.max_segs + per_block - 1) / per_block), E.G), CRC_WARPS * 32, 0, s>>>(E, K);
    }
    STPC_LAUNCH();
    crc_finish_kernel<<<E.G, 64, 0, s>>>(E, K);
}

}  // namespace stpc
