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
 * Batches of >= 64 groups are pipelined in 8 chunks: the H2D of chunk c+1
 * overlaps the encode and blob D2H of chunk c; stpc_result_blobs then gives
 * offsets into h_out and stpc_result_device_blobs returns NULL. */
int stpc_encode_host(stpc_encoder* enc, int32_t n_groups, const void* h_points,
                     const int64_t* point_offsets, const double* transforms, uint8_t* h_out,
                     int64_t out_cap, void* stream);

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

/* Decoder (decompress).  d_blob_off: device int64[n]
 * blob starts in d_blobs.  stpc_crc32_blobs: zlib CRC-32 of each blob's entropy
 * payload (bitstream.py:410-411).  stpc_huffman_decode_blobs: raw payload of
 * each blob into d_out + d_out_off[i] (huffman_decode_kernel, _kernels.py:
 * 385-417); h_status 0 ok / 1 truncated / 2 invalid code.
 * stpc_reconstruct_frames: per-tile plane maps (float4 a, b, c, kind; kind 0 =
 * none) + validity bitmaps + residual pixels -> points (float64 xyz, row-major
 * per frame, inverse-transformed with d_xf_inv [F][12] = R^-1 | T^-1)
 * (decode_stream_images temporal.py:293-343, reconstruct_span _kernels.py:
 * 282-308, unproject range_image.py:214-221).  d_scratch: f64 [F][h*w]. */
int stpc_crc32_blobs(const uint8_t* d_blobs, const int64_t* d_blob_off, int32_t n, uint32_t* h_crc, void* stream);
int stpc_huffman_decode_blobs(const uint8_t* d_blobs, const int64_t* d_blob_off, int32_t n, uint8_t* d_out,
                              const int64_t* d_out_off, int32_t* h_status, void* stream);
int stpc_reconstruct_frames(int32_t w, int32_t h, int32_t tile_w, int32_t tile_h, const double* d_trig,
                            int32_t n_frames, const uint8_t* d_vbits, int64_t vstride, const float* d_tile_map,
                            const int64_t* d_res_flat, const double* d_res_range, const int32_t* d_res_frame,
                            int64_t n_res, const double* d_xf_inv, double r_max, double* d_scratch,
                            double* d_points, int64_t points_cap, int64_t* h_frame_counts, int64_t* h_failed,
                            void* stream);

/* Utilities so FFI callers need no CUDA runtime binding of their own. */
int stpc_malloc(void** dev_ptr, int64_t bytes);
int stpc_free(void* dev_ptr);
int stpc_memcpy_d2h(void* dst, const void* src, int64_t bytes);
int stpc_memcpy_h2d(void* dst, const void* src, int64_t bytes);
int stpc_device_count(void);
const char* stpc_last_error(void);
const char* stpc_version(void);

#ifdef __cplusplus
}
#endif
#endif
