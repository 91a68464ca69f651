/*
 * libstpc_b200 -- C-ABI of the B200-native stpc compression hot path.
 *
 * The drop-in boundary for the reference package's compress() path
 * (/root/reference/pkg/src/stpc/bitstream.py:527-602).  The reference's only
 * native boundary is the set of numba kernels in
 * /root/reference/pkg/src/stpc/_kernels.py (positional arrays in,
 * caller-allocated outputs, scalar status, no exceptions, GIL released); this
 * ABI keeps those conventions at batch granularity: plain pointers and sizes,
 * int status (0 = ok), no torch types, no global mutable state (one encoder
 * per thread/stream).  See INTEGRATION.md for the ctypes binding.
 *
 * Entry point          replaces (reference file:line)
 * ------------------   ---------------------------------------------------
 * stpc_encode_device   compress() minus host glue: build_stack (motion.py:258-284,
 * stpc_encode_host       project_kernel _kernels.py:311-355), encode_stream
 *                        (temporal.py:105-266: encode_tile_row :151-228,
 *                        refit_spans :231-279), serialize (bitstream.py:193-289:
 *                        huffman.encode_bytes huffman.py:107-118,
 *                        huffman_encode_kernel _kernels.py:363-382, zlib.crc32)
 * stpc_project         project(..., return_indices=True) (range_image.py:165-211)
 *                        fused with RigidTransform.apply (motion.py:70-72)
 * stpc_decoder_*       decompress (bitstream.py:605-631): deserialize,
 *                        decode_stream_images, unproject (see below)
 */
#ifndef STPC_B200_H
#define STPC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STPC_OK 0
#define STPC_ERR_CUDA 1
#define STPC_ERR_ARG 2
#define STPC_ERR_NOMEM 3

/* CodecConfig (/root/reference/pkg/src/stpc/bitstream.py:87-126) plus the
 * fixed fit constants (range_image.py:34 r_max = 200, plane.py:26 cond = 1e8). */
typedef struct stpc_config {
    int32_t mode; /* 0 = single, 1 = stream */
    int32_t tile_w, tile_h;
    int32_t w, h;
    int32_t n_frames, k_index;
    int32_t points_f64; /* input xyz dtype: 0 = float32, 1 = float64 */
    double tau;
    double theta_r, phi_r, phi_offset;
    double range_quant;
    double r_max;
    double cond_limit;
} stpc_config;

/* Per-frame statistics (ProjectionStats range_image.py:58-70, coverage_counts
 * temporal.py:269-290). */
#define STPC_STAT_REJECTED 0
#define STPC_STAT_DROPPED 1
#define STPC_STAT_KEPT 2
#define STPC_STAT_VALID 3
#define STPC_STAT_TEMPORAL 4
#define STPC_STAT_FALLBACK 5
#define STPC_STAT_RESIDUAL 6
#define STPC_STAT_ESCAPES 7
#define STPC_STAT_EPS_BAND 8
#define STPC_NSTAT 9

typedef struct stpc_encoder stpc_encoder;

/* Trig tables of pixel_ray_grid (range_image.py:141-147), computed by the host
 * with the reference's own numpy expressions: sin/cos of theta_u =
 * (u+0.5)*theta_r (w entries) and of phi_v = phi_offset+(v+0.5)*phi_r (h). */
int stpc_encoder_create(const stpc_config* cfg, const double* sin_theta, const double* cos_theta,
                        const double* sin_phi, const double* cos_phi, stpc_encoder** out);
void stpc_encoder_destroy(stpc_encoder* enc);

/* Encode n_groups independent K+P groups (n_frames each, frame f = g*n + i).
 * d_points: device float32 (or float64 if cfg.points_f64) xyz, frames concatenated; point_offsets: host
 * int64[F+1] (point index of each frame's start); transforms: host
 * double[F][12] frame -> key-frame R (row-major) | T, already rounded through
 * float32 (round_f32, motion.py:87-92).  stream: cudaStream_t (NULL = legacy).
 * Blobs stay in the encoder's device arena until the next call. */
int stpc_encode_device(stpc_encoder* enc, int32_t n_groups, const void* d_points,
                       const int64_t* point_offsets, const double* transforms, void* stream);

/* End-to-end variant from host memory: H2D of the points (pinned memory
 * recommended), encode, D2H of every blob into h_out (capacity out_cap).
 * Batches of >= 64 groups are pipelined in 8 chunks (16 from 128 groups): the H2D of chunk c+1
 * overlaps the encode and blob D2H of chunk c; stpc_result_blobs then gives
 * offsets into h_out and stpc_result_device_blobs returns NULL. */
int stpc_encode_host(stpc_encoder* enc, int32_t n_groups, const void* h_points,
                     const int64_t* point_offsets, const double* transforms, uint8_t* h_out,
                     int64_t out_cap, void* stream);

/* Host encode from per-frame arrays (no concatenation on the caller's side):
 * frame f's xyz at frame_points[f] (float32, or float64 if cfg.points_f64),
 * frame_counts[f] points.  Frames are gathered by host threads into pinned
 * staging per pipeline chunk (overlapping the previous chunk's H2D and
 * encode); blobs land in the encoder's own pinned arena
 * (stpc_result_host_blobs / stpc_result_copy_blobs). */
int stpc_encode_host_gather(stpc_encoder* enc, int32_t n_groups, const void* const* frame_points,
                            const int64_t* frame_counts, const double* transforms, void* stream);
const uint8_t* stpc_result_host_blobs(const stpc_encoder* enc);

/* Make `stream` wait for the encoder's pending side-stream work (the +inf
 * prefill of the next call's range grid, which overlaps the entropy stage of
 * the last call).  Timing code calls it before its closing event so that a
 * window of K calls contains exactly K prefills. */
int stpc_encoder_wait(stpc_encoder* enc, void* stream);

/* Results of the last encode. offsets: int64[G+1] (blob start in the arena;
 * offsets[G] = arena bytes), lengths: int64[G]. */
int32_t stpc_result_groups(const stpc_encoder* enc);
int stpc_result_blobs(const stpc_encoder* enc, int64_t* offsets, int64_t* lengths);
const uint8_t* stpc_result_device_blobs(const stpc_encoder* enc);
int stpc_result_copy_blobs(const stpc_encoder* enc, uint8_t* h_dst, int64_t cap, void* stream);
int stpc_result_frame_stats(const stpc_encoder* enc, int64_t* out /* F * STPC_NSTAT */);
int stpc_result_payload_lengths(const stpc_encoder* enc, int64_t* raw_lengths /* G */);

/* Device pointer + size of an intermediate buffer of the last encode (for
 * parity tests): see STPC_BUF_*. */
#define STPC_BUF_BEST 0    /* f64 [F][h*w], +inf = empty */
#define STPC_BUF_CLS 1     /* u8 [F][tiles_y][tiles_x] */
#define STPC_BUF_RUN_S 2   /* u16 [F*tiles_y][tiles_x] */
#define STPC_BUF_RUN_LEN 3 /* u16 [F*tiles_y][tiles_x] */
#define STPC_BUF_RUN_ABC 4 /* f32 [F*tiles_y][tiles_x][3] */
#define STPC_BUF_N_RUNS 5  /* i32 [F*tiles_y] */
#define STPC_BUF_REF_OK 6  /* u8 [G*tiles_y][tiles_x][n] */
#define STPC_BUF_REF_C 7   /* f32 [G*tiles_y][tiles_x][n] */
#define STPC_BUF_PAYLOAD 8 /* u8 raw payload arena */
#define STPC_BUF_VBITS 9   /* u8 [F][pbs] */
int stpc_encoder_buffer(const stpc_encoder* enc, int32_t which, void** dev_ptr, int64_t* bytes);

/* Per-stage device time (CUDA events on the encode stream) accumulated over
 * the calls since profiling was (re-)enabled; stage names via stpc_stage_name.
 * stpc_launch_count: kernels this library has launched (process-wide). */
int stpc_encoder_profile(stpc_encoder* enc, int32_t enable);
int32_t stpc_encoder_stage_ms(const stpc_encoder* enc, double* ms, int32_t n);
const char* stpc_stage_name(int32_t i);
uint64_t stpc_launch_count(void);

/* Standalone K1 for project(..., return_indices=True) parity: d_best
 * f64[F][h*w] (+inf empty), d_win int64[F][h*w] (-1 empty, nullable),
 * h_counts int64[F][3] = rejected, dropped, kept. */
int stpc_project(const void* d_points, int32_t points_f64, const int64_t* point_offsets, int32_t n_frames,
                 const double* transforms, int32_t w, int32_t h, double theta_r, double phi_r,
                 double phi_offset, double* d_best, int64_t* d_win, int64_t* h_counts, void* stream);

/* The entropy stage alone (huffman.encode_bytes huffman.py:107-118 with the
 * 32-bit cap repair :51-58, canonical codes :63-77, huffman_encode_kernel
 * _kernels.py:363-382, header + zlib.crc32 bitstream.py:279-289) on n raw
 * payloads in host memory (payload i = h_payloads[offsets[i], offsets[i+1])):
 * blob i lands at h_out[out_offsets[i], out_offsets[i+1]).  The kernels are
 * the ones stpc_encode_* run; this entry exists so a payload of any byte
 * statistics (e.g. a Fibonacci histogram that forces the cap repair) can be
 * coded on the device. */
int stpc_entropy_encode(const uint8_t* h_payloads, const int64_t* offsets, int32_t n, uint8_t* h_out,
                        int64_t out_cap, int64_t* out_offsets);

/* Decoder (decompress / decompress_full, bitstream.py:605-631; SURVEY.md
 * §8(f) rank 3), batched over blobs, all on the GPU:
 *
 * stpc_decoder_load    replaces deserialize's header checks (bitstream.py:
 *                        398-409), zlib.crc32 (:410-411), decode_tables and
 *                        huffman.decode_bytes (huffman.py:80-137,
 *                        huffman_decode_kernel _kernels.py:385-417).  blobs:
 *                        host or device bytes, blob i at [offsets[i],
 *                        offsets[i+1]).  status[i]: STPC_DEC_* of the first
 *                        failing check, in the reference's order.
 * stpc_decoder_load_gather  the same from n separate host buffers (blob i at
 *                        blobs[i], lengths[i] bytes): gathered into pinned
 *                        staging by host threads, one H2D.
 * stpc_decoder_heads   first head_cap bytes of each raw payload (config block
 *                        + float32 transforms, bitstream.py:413-426) for the
 *                        host-side config checks.
 * stpc_decoder_frames  replaces the record sections of deserialize (:428-519),
 *                        decode_stream_images (temporal.py:293-343) and
 *                        reconstruct_span (_kernels.py:282-308) for the loaded
 *                        blobs sel[0..m) sharing one configuration; trig tables
 *                        as for the encoder; xf_inv: double[m*n][12]
 *                        R^-1 | T^-1 (RigidTransform.inverse, motion.py:78-79).
 *                        frame_counts[m*n]: points per frame; status[m]: 0 or
 *                        (reader position << 8 | order << 4 | STPC_DEC_*) of
 *                        the first structural error; failed[m]: failed
 *                        reconstructions (DecodeReport).
 * stpc_decoder_points  unproject (range_image.py:214-221) + inverse transform
 *                        (motion.py:70-72): float64 xyz of every frame of the
 *                        last stpc_decoder_frames, concatenated, into dst (host
 *                        or device, capacity cap_points points); dst NULL with
 *                        dst_on_device = 1 keeps them in the decoder's own
 *                        device buffer (stpc_decoder_device_points). */
#define STPC_DEC_TRUNCATED 1 /* TruncatedBlobError */
#define STPC_DEC_MALFORMED 2 /* MalformedBlobError */
#define STPC_DEC_CHECKSUM 3  /* ChecksumError */
#define STPC_DEC_VERSION 4   /* UnknownVersionError */

typedef struct stpc_decode_geom {
    int32_t w, h, tile_w, tile_h, n_frames, k_index;
    double range_quant, r_max;
} stpc_decode_geom;

typedef struct stpc_decoder stpc_decoder;
int stpc_decoder_create(stpc_decoder** out);
void stpc_decoder_destroy(stpc_decoder* dec);
int stpc_decoder_load(stpc_decoder* dec, const uint8_t* blobs, int32_t blobs_on_device, const int64_t* offsets,
                      int32_t n, int32_t* status, void* stream);
int stpc_decoder_load_gather(stpc_decoder* dec, const uint8_t* const* blobs, const int64_t* lengths, int32_t n,
                             int32_t* status, void* stream);
int stpc_decoder_heads(stpc_decoder* dec, int32_t head_cap, uint8_t* h_heads, int64_t* h_raw_len, void* stream);
/* stpc_decode_transforms  host-side RigidTransform checks (motion.py:52-62:
 *                        allclose(R.T @ R, I, atol), isclose(det R, 1)) and
 *                        inverses (motion.py:78-79) of the float32 transforms
 *                        of blobs rows[0..m) of a stpc_decoder_heads array
 *                        (head_stride bytes per blob, transforms at `offset`):
 *                        xf_inv double[m*n][12] (R^T | -R^T T), orth_state /
 *                        det_state int8[m*n]: 0 passes, 1 fails, 2 too close to
 *                        the tolerance or non-finite (the caller re-checks with
 *                        the reference's numpy expressions). */
int stpc_decode_transforms(const uint8_t* heads, int64_t head_stride, const int64_t* rows, int32_t m,
                           int32_t n_frames, int32_t offset, double atol, double* xf_inv, int8_t* orth_state,
                           int8_t* det_state);
int stpc_decoder_frames(stpc_decoder* dec, const stpc_decode_geom* geom, const int32_t* sel, int32_t m,
                        const double* sin_theta, const double* cos_theta, const double* sin_phi,
                        const double* cos_phi, const double* xf_inv, int64_t* frame_counts, int64_t* status,
                        int64_t* failed, void* stream);
int64_t stpc_decoder_total_points(const stpc_decoder* dec);
int stpc_decoder_points(stpc_decoder* dec, double* dst, int32_t dst_on_device, int64_t cap_points, void* stream);
const double* stpc_decoder_device_points(const stpc_decoder* dec);

/* Utilities so FFI callers need no CUDA runtime binding of their own. */
int stpc_malloc(void** dev_ptr, int64_t bytes);
int stpc_free(void* dev_ptr);
int stpc_memcpy_d2h(void* dst, const void* src, int64_t bytes);
int stpc_memcpy_h2d(void* dst, const void* src, int64_t bytes);
/* Host copy of n blobs (src + offsets[i], lengths[i] bytes) to dst[i] with
 * host threads: how compress_groups fills its bytes objects.  Replaces the
 * per-blob bytes(...) of the reference's result assembly
 * (/root/reference/pkg/src/stpc/bitstream.py:289-290, one blob per compress). */
int stpc_host_scatter(const uint8_t* src, const int64_t* offsets, const int64_t* lengths, uint8_t* const* dst,
                      int32_t n);
int stpc_device_count(void);
const char* stpc_last_error(void);
const char* stpc_version(void);

#ifdef __cplusplus
}
#endif
#endif
