// Decoder kernels: the device side of decompress().
//
// Replaces the heavy loops of the reference decoder
// (/root/reference/pkg/src/stpc/bitstream.py:388-519, 605-631):
//   * zlib.crc32 of the entropy payload (:410-411)       -> crc_blob_kernel
//   * huffman_decode_kernel (_kernels.py:385-417)       -> huff_decode_kernel
//   * decode_stream_images + reconstruct_span
//     (temporal.py:293-343, _kernels.py:282-308)        -> reconstruct_kernel
//   * unproject (range_image.py:214-221) + the inverse
//     frame transform (motion.py:78-79, 70-72)          -> unproject_kernel
// Record-level parsing (runs, fallback rows, residual varints: O(records))
// stays in the host mirror (decode.py), which builds per-tile plane maps.
#include <vector>

#include "kernels.cuh"
#include "../../include/stpc_b200.h"

namespace stpc {

__device__ __forceinline__ unsigned int dec_multmodp(unsigned int a, unsigned int b)
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

__device__ __forceinline__ unsigned int dec_x8nmodp(unsigned long long nbytes)
{
    unsigned int p = 1u << 31, sq = 1u << 23;
    while (nbytes) {
        if (nbytes & 1) p = dec_multmodp(sq, p);
        sq = dec_multmodp(sq, sq);
        nbytes >>= 1;
    }
    return p;
}

// block per blob: threads CRC 1 KB pieces of the encoded payload, thread 0
// combines them in order (a few hundred pieces per blob).
__global__ void __launch_bounds__(256) crc_blob_kernel(const uint8_t* blobs, const long long* blob_off,
                                                       unsigned int* crc_out)
{
    __shared__ unsigned int tab[256];
    __shared__ unsigned int part[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        unsigned int c = i;
        for (int k = 0; k < 8; ++k) c = c & 1 ? (c >> 1) ^ 0xedb88320u : c >> 1;
        tab[i] = c;
    }
    __syncthreads();
    const uint8_t* blob = blobs + blob_off[blockIdx.x];
    unsigned long long enc_len = 0;
    for (int b = 0; b < 8; ++b) enc_len |= (unsigned long long)blob[16 + b] << (8 * b);
    const uint8_t* enc = blob + 284;
    const long long piece = 1024;
    const long long npieces = ((long long)enc_len + piece - 1) / piece;
    unsigned int raw = 0;
    for (long long base = 0; base < npieces; base += 256) {
        const long long pi = base + threadIdx.x;
        unsigned int c = 0;
        if (pi < npieces) {
            const long long e = min((pi + 1) * piece, (long long)enc_len);
            for (long long i = pi * piece; i < e; ++i) c = tab[(c ^ enc[i]) & 0xff] ^ (c >> 8);
        }
        part[threadIdx.x] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned int X = dec_x8nmodp(piece);
            for (int t = 0; t < 256 && base + t < npieces; ++t) {
                const long long len = min(piece, (long long)enc_len - (base + t) * piece);
                raw = dec_multmodp(len == piece ? X : dec_x8nmodp(len), raw) ^ part[t];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        crc_out[blockIdx.x] = ~(raw ^ dec_multmodp(dec_x8nmodp(enc_len), 0xffffffffu));
}

// One thread per blob: bit-serial canonical Huffman decode with the
// reference's per-length first-code search (batches decode many blobs in
// parallel).  status: 0 ok, 1 out of bits, 2 bad code.
__global__ void huff_decode_kernel(const uint8_t* blobs, const long long* blob_off, int n, uint8_t* out,
                                   const long long* out_off, int* status)
{
    const int bi = blockIdx.x * blockDim.x + threadIdx.x;
    if (bi >= n) return;
    const uint8_t* blob = blobs + blob_off[bi];
    unsigned long long raw_len = 0, enc_len = 0;
    for (int b = 0; b < 8; ++b) {
        raw_len |= (unsigned long long)blob[8 + b] << (8 * b);
        enc_len |= (unsigned long long)blob[16 + b] << (8 * b);
    }
    const uint8_t* lens = blob + 28;
    const uint8_t* enc = blob + 284;
    // canonical tables (huffman.py:80-104)
    int count[33] = {0};
    for (int s = 0; s < 256; ++s) count[lens[s]] += 1;
    count[0] = 0;
    unsigned int first[33], index[33];
    unsigned int code = 0, idx = 0;
    for (int l = 1; l <= 32; ++l) {
        first[l] = code;
        index[l] = idx;
        code = (code + count[l]) << 1;
        idx += count[l];
    }
    uint8_t sym_sorted[256];
    {
        int fill[33];
        for (int l = 1; l <= 32; ++l) fill[l] = index[l];
        for (int s = 0; s < 256; ++s)
            if (lens[s]) sym_sorted[fill[lens[s]]++] = (uint8_t)s;
    }
    uint8_t* o = out + out_off[bi];
    const unsigned long long total_bits = enc_len * 8;
    unsigned long long bitpos = 0;
    int st = 0;
    for (unsigned long long i = 0; i < raw_len; ++i) {
        unsigned int c = 0;
        int l = 0;
        for (;;) {
            if (bitpos >= total_bits) { st = 1; break; }
            const unsigned int bit = (enc[bitpos >> 3] >> (7 - (bitpos & 7))) & 1u;
            ++bitpos;
            c = (c << 1) | bit;
            ++l;
            if (l > 32) { st = 2; break; }
            if (count[l] > 0 && c - first[l] < (unsigned)count[l]) {
                o[i] = sym_sorted[index[l] + (c - first[l])];
                break;
            }
        }
        if (st) break;
    }
    status[bi] = st;
}

// Per pixel of every frame: plane reconstruction from the per-tile plane map
// (kind 1 = temporal run with this channel's offset, kind 2 = fallback run
// over the channel's remaining pixels), exactly reconstruct_span's
// arithmetic; then residual pixels override.  out_r: +inf = no point.
__global__ void reconstruct_kernel(Geometry g, Trig tg, int n_frames, const uint8_t* vbits, long long vstride,
                                   const float4* tmap, const double* r_max_p, double* out_r,
                                   unsigned long long* failed)
{
    const long long P = g.P;
    const long long total = (long long)n_frames * P;
    const double r_max = *r_max_p;
    unsigned int nfail = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long f = i / P, p = i - f * P;
        const int v = (int)(p / g.w), u = (int)(p - (long long)v * g.w);
        const bool valid = (vbits[f * vstride + (p >> 3)] >> (7 - (p & 7))) & 1u;
        double r = __longlong_as_double(0x7ff0000000000000ll);
        if (valid) {
            const float4 pl = tmap[(f * g.ty + v / g.th) * g.tx + u / g.tw];
            if (pl.w != 0.0f) {
                double dx, dy, dz;
                ray_dir(tg, v, u, dx, dy, dz);
                const double den = (dx + (double)pl.x * dy) + (double)pl.y * dz;
                if (fabs(den) < STPC_PARALLEL_EPS) {
                    ++nfail;
                } else {
                    const double r_hat = (double)pl.z / den;
                    if (r_hat <= 0.0 || r_hat > r_max) ++nfail;
                    else r = r_hat;
                }
            }
        }
        out_r[i] = r;
    }
    for (int o = 16; o > 0; o >>= 1) nfail += __shfl_xor_sync(STPC_FULL, nfail, o);
    if ((threadIdx.x & 31) == 0 && nfail) atomicAdd(failed, (unsigned long long)nfail);
}

__global__ void residual_scatter_kernel(const long long* flat, const double* ranges, long long n, long long P,
                                        const int* frame_of, double* out_r)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out_r[(long long)frame_of[i] * P + flat[i]] = ranges[i];
}

// count points per (frame, 1024-pixel block) -- grid (blocks per frame,
// frames) so blocks never straddle frames -- for the row-major compaction
__global__ void count_points_kernel(const double* out_r, long long P, int* blk_count)
{
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long i = (long long)blockIdx.y * P + p;
    const bool have = p < P && isfinite(out_r[i]);
    const unsigned m = __ballot_sync(STPC_FULL, have);
    __shared__ int ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
        blk_count[(long long)blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// points = r * d in row-major pixel order per frame, then p' = R^-1 p + T^-1
// with fma(z, r2, fma(y, r1, x r0)) + t (motion.py:70-72 on the inverse transform).
__global__ void unproject_kernel(Geometry g, Trig tg, const double* out_r, const long long* blk_off,
                                 const double* xf_inv, double* pts)
{
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long f = blockIdx.y;
    const long long i = f * g.P + p;
    const bool have = p < g.P && isfinite(out_r[i]);
    const unsigned m = __ballot_sync(STPC_FULL, have);
    __shared__ int ws[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) ws[wid] = __popc(m);
    __syncthreads();
    int before = 0;
    for (int w = 0; w < wid; ++w) before += ws[w];
    if (!have) return;
    const long long o = blk_off[f * gridDim.x + blockIdx.x] + before + __popc(m & ((1u << lane) - 1u));
    const int v = (int)(p / g.w), u = (int)(p - (long long)v * g.w);
    double dx, dy, dz;
    ray_dir(tg, v, u, dx, dy, dz);
    const double r = out_r[i];
    const double x = r * dx, y = r * dy, z = r * dz;
    const double* R = xf_inv + 12 * f;
    // numpy's pts @ Rinv.T is a K=3 dgemm: the BLAS micro-kernel accumulates
    // k = 0,1,2 with fused multiply-adds (checked bit-for-bit against the
    // reference's decompress output, tests/golden dec_sha256); + T is a
    // separate add.  -fmad=false keeps every other op unfused.
    pts[3 * o] = xform_coord(x, y, z, R[0], R[1], R[2], R[9]);
    pts[3 * o + 1] = xform_coord(x, y, z, R[3], R[4], R[5], R[10]);
    pts[3 * o + 2] = xform_coord(x, y, z, R[6], R[7], R[8], R[11]);
}

}  // namespace stpc

using namespace stpc;

extern "C" {

int stpc_crc32_blobs(const uint8_t* d_blobs, const int64_t* d_blob_off, int32_t n, uint32_t* h_crc, void* stream)
{
    if (n < 1 || !d_blobs || !d_blob_off || !h_crc) return STPC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned int* d_crc = nullptr;
    if (cudaMalloc(&d_crc, sizeof(unsigned) * n) != cudaSuccess) return STPC_ERR_NOMEM;
    STPC_LAUNCH();
    crc_blob_kernel<<<n, 256, 0, s>>>(d_blobs, (const long long*)d_blob_off, d_crc);
    cudaError_t e = cudaMemcpyAsync(h_crc, d_crc, sizeof(unsigned) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d_crc);
    return e == cudaSuccess ? STPC_OK : STPC_ERR_CUDA;
}

int stpc_huffman_decode_blobs(const uint8_t* d_blobs, const int64_t* d_blob_off, int32_t n, uint8_t* d_out,
                              const int64_t* d_out_off, int32_t* h_status, void* stream)
{
    if (n < 1 || !d_blobs || !d_out || !h_status) return STPC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    int* d_st = nullptr;
    if (cudaMalloc(&d_st, sizeof(int) * n) != cudaSuccess) return STPC_ERR_NOMEM;
    STPC_LAUNCH();
    huff_decode_kernel<<<(n + 63) / 64, 64, 0, s>>>(d_blobs, (const long long*)d_blob_off, n, d_out,
                                                     (const long long*)d_out_off, d_st);
    cudaError_t e = cudaMemcpyAsync(h_status, d_st, sizeof(int) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d_st);
    return e == cudaSuccess ? STPC_OK : STPC_ERR_CUDA;
}

int stpc_reconstruct_frames(int32_t w, int32_t h, int32_t tile_w, int32_t tile_h, const double* d_trig,
                            int32_t n_frames, const uint8_t* d_vbits, int64_t vstride, const float* d_tile_map,
                            const int64_t* d_res_flat, const double* d_res_range, const int32_t* d_res_frame,
                            int64_t n_res, const double* d_xf_inv, double r_max, double* d_scratch,
                            double* d_points, int64_t points_cap, int64_t* h_frame_counts, int64_t* h_failed,
                            void* stream)
{
    if (n_frames < 1 || w < 1 || h < 1 || !d_trig || !d_vbits || !d_tile_map || !d_scratch || !h_frame_counts)
        return STPC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    Geometry g{};
    g.w = w;
    g.h = h;
    g.tw = tile_w;
    g.th = tile_h;
    g.tx = (w + tile_w - 1) / tile_w;
    g.ty = (h + tile_h - 1) / tile_h;
    g.P = (long long)w * h;
    Trig tg;
    tg.sin_t = d_trig;
    tg.cos_t = d_trig + w;
    tg.sin_p = d_trig + 2 * w;
    tg.cos_p = d_trig + 2 * w + h;
    const long long bpf = (g.P + 1023) / 1024;  // blocks per frame
    const long long nblk = bpf * n_frames;
    void* tmp = nullptr;
    const size_t tmp_bytes = 16 + sizeof(int) * nblk + 8 + sizeof(long long) * nblk;
    if (cudaMalloc(&tmp, tmp_bytes) != cudaSuccess) return STPC_ERR_NOMEM;
    unsigned long long* d_failed = (unsigned long long*)tmp;
    double* d_rmax = (double*)(d_failed + 1);
    int* d_cnt = (int*)(d_rmax + 1);
    long long* d_off = (long long*)(((uintptr_t)(d_cnt + nblk) + 7) & ~(uintptr_t)7);
    cudaError_t e = cudaMemsetAsync(d_failed, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_rmax, &r_max, sizeof(double), cudaMemcpyHostToDevice, s);
    STPC_LAUNCH();
    reconstruct_kernel<<<148 * 8, 256, 0, s>>>(g, tg, n_frames, d_vbits, vstride, (const float4*)d_tile_map,
                                                d_rmax, d_scratch, d_failed);
    if (n_res > 0) {
        STPC_LAUNCH();
        residual_scatter_kernel<<<148 * 4, 256, 0, s>>>((const long long*)d_res_flat, d_res_range, n_res, g.P,
                                                         d_res_frame, d_scratch);
    }
    STPC_LAUNCH();
    count_points_kernel<<<dim3((unsigned)bpf, (unsigned)n_frames), 1024, 0, s>>>(d_scratch, g.P, d_cnt);
    std::vector<int> hc(nblk);
    std::vector<long long> ho(nblk + 1);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), d_cnt, sizeof(int) * nblk, cudaMemcpyDeviceToHost, s);
    unsigned long long hfail = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hfail, d_failed, sizeof(hfail), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        cudaFree(tmp);
        return STPC_ERR_CUDA;
    }
    ho[0] = 0;
    for (long long b = 0; b < nblk; ++b) ho[b + 1] = ho[b] + hc[b];
    for (int f = 0; f < n_frames; ++f) h_frame_counts[f] = ho[(long long)(f + 1) * bpf] - ho[(long long)f * bpf];
    if (ho[nblk] > points_cap || (!d_points && ho[nblk] > 0)) {
        cudaFree(tmp);
        return STPC_ERR_ARG;
    }
    e = cudaMemcpyAsync(d_off, ho.data(), sizeof(long long) * nblk, cudaMemcpyHostToDevice, s);
    STPC_LAUNCH();
    unproject_kernel<<<dim3((unsigned)bpf, (unsigned)n_frames), 1024, 0, s>>>(g, tg, d_scratch, d_off, d_xf_inv,
                                                                              d_points);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(tmp);
    if (h_failed) *h_failed = (int64_t)hfail;
    return e == cudaSuccess ? STPC_OK : STPC_ERR_CUDA;
}

}  // extern "C"
