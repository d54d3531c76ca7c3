/* include/stereo.h — C ABI of the B200-native stereo hot path.
 *
 * Implements the data-parallel pipeline of Chang & Maruyama, "Real-Time
 * High-Quality Stereo Matching System on a GPU" (arXiv 2212.00488), §III and
 * §IV Steps 1-8, as hand-written CUDA kernels for sm_100a:
 *
 *   SD (Eq. 2)  -> mini-census + cross arms
 *   -> cost + x aggregation, both bases (Eqs. 3-7; Step3 P:418-457)
 *   -> y aggregation + WTA, both bases (Eqs. 8-9; Step5 P:474-502)
 *   -> cross-check (Eq. 10) + 3x3 median (Step7)
 *   -> bilateral fill of non-GCPs (§III.E; Step7 P:516-525)
 *   -> bilateral/linear scale-up (Step8)
 *
 * Plain C linkage: no C++ types, no torch types, no exceptions cross this
 * boundary.  Pointers are either DEVICE pointers (cudaMalloc'd or torch CUDA
 * tensor storage on the handle's device) or HOST pointers, as stated per call.
 * Streams are passed as `void*` holding a cudaStream_t (NULL = legacy default
 * stream).
 *
 * Numerics (DESIGN.md §2 reading R12c): every cost term is quantised once to
 * fixed point, Q = floor(c * 2^f + 0.5), f = largest value <= 25 with
 * (2 w_x + 1) 2^(f+1) < 2^32; all aggregation is then exact integer arithmetic
 * (u32 modular prefix sums along x, u64 along y), so the result is bit-exact
 * with the CPU oracle's fixed mode and within 0.5*2^-f/c_AD(1) <= 1.2e-6
 * relative of the IEEE-double definition on every aggregated cost.
 *
 * Errors: every function returns STEREO_OK (0) or a negative STEREO_E* code and
 * never aborts; stereo_last_error() returns a thread-local message naming the
 * first violated invariant or the failing CUDA call.  Asynchronous kernel
 * faults surface at the caller's next synchronisation of the stream.
 */
#ifndef STEREO_B200_H
#define STEREO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STEREO_ABI_VERSION 3u

enum {
  STEREO_OK = 0,
  STEREO_EINVAL = -1,       /* invalid argument / parameter invariant violated */
  STEREO_ENOMEM = -2,       /* device or host allocation failed */
  STEREO_ECUDA = -3,        /* a CUDA runtime call or launch failed */
  STEREO_EUNSUPPORTED = -4  /* valid per the paper, outside this build's limits */
};

/* Method parameters.  Defaults (stereo_default_params) are the paper's values
 * where it gives them: lambda_AD = 0.3, lambda_MC = 2.3, T = 3,
 * W_x = 21, W_y = 31, K = 2, 3x3 mean pool;
 * delta = 20 (the paper never states it, reading R13);
 * census pattern (0,-2)(-1,-1)(+1,-1)(-1,+1)(+1,+1)(0,+2) (Fig. 3 is missing;
 * SPEC S:92, reading R8). */
typedef struct {
  uint32_t abi_version;  /* must equal STEREO_ABI_VERSION */
  double lambda_ad;      /* Eq. 4 scale; AD uses |dI|/255 (reading R12), > 0 */
  double lambda_mc;      /* Eq. 5 scale on the raw Hamming distance, > 0 */
  int32_t t_fill;        /* T: continuity threshold of §III.E; SU uses K*T; >= 0 */
  int32_t w_x, w_y;      /* per-side arm caps W_x, W_y; 0..254 */
  int32_t delta;         /* arm similarity |dI| < delta (strict); > 0 */
  int32_t k_scale;       /* K: 2 (scale down/up) or 1 (no scaling path) */
  int32_t m_pool;        /* mean-pool radius m of Eq. 2; 0..3 */
  int8_t census_dx[6];   /* the six mini-census offsets, |dx|,|dy| <= 2, */
  int8_t census_dy[6];   /* distinct and non-zero; bit i <-> offset i */
  /* ABI 2: the NEXT-3 method variants */
  int32_t w_x_r;         /* x arm cap of the RIGHT-base map D^R: "(W_x, W_y) can be
                            changed when calculating D^L and D^R", W_y common
                            (P:613-619); -1 = w_x (default); else 0..254 */
  int32_t fill_mode;     /* non-GCP filling, §III.E: STEREO_FILL_* (default 0) */
} stereo_params;

/* Non-GCP filling modes (§III.E). */
enum {
  STEREO_FILL_BILATERAL = 0,    /* the paper's method, steps 1-3, Eq. 11
                                   read as the interpolation (reading E6) */
  STEREO_FILL_NEAREST = 1,      /* Fig. 6(a): the closer GCP's disparity (tie: left) */
  STEREO_FILL_SMALLER = 2,      /* Fig. 6(b): the smaller of the two disparities */
  STEREO_FILL_EQ11_LITERAL = 3  /* steps 1-3 with Eq. 11 exactly as printed:
                                   D(x-i) + i (D(x-i) - D(x+j)) / (i+j) */
};

/* Derived sizes and resources of a handle (filled by stereo_get_info). */
typedef struct {
  int32_t W, H, D;        /* original width, height, maximum disparity */
  int32_t Ws, Hs, Ds;     /* scaled: W/K, H/K (floor), ceil(D/K) */
  int32_t frac_bits;      /* f of the fixed-point cost */
  int32_t device;         /* CUDA device ordinal the handle is bound to */
  uint64_t device_bytes;  /* total device scratch owned by the handle */
  uint64_t cax_bytes;     /* bytes of ONE CA_x volume (u32 [ceil(Ds/2)][Hs][cax_pitch][2]) */
  int32_t launches_per_frame; /* kernels enqueued by one launch sequence (one
                                 stereo_compute, or one chunk of max_frames frames) */
  int32_t ypass_block_rows;   /* output rows per y-aggregation tile */
  int32_t cax_pitch;          /* row pitch (elements) of the CA_x volumes */
  /* ABI 3 */
  int32_t max_frames;         /* frames one launch sequence serves (stereo_create_batch) */
  int32_t band;               /* 1: a row-band handle (stereo_create_band) */
  int32_t band_y0_org, band_rows_org;          /* band: own original rows */
  int32_t band_halo_top_org, band_halo_bot_org; /* band: halo rows above / below */
  int32_t ypass_rows;         /* scaled rows the y aggregation + WTA computes per frame
                                 (band: own rows + the cross-check / median / Step8 cone) */
} stereo_info;

typedef struct stereo_s stereo_t; /* opaque; owns ALL device scratch */

/* Fill *p with the defaults above.  p must be non-NULL. */
void stereo_default_params(stereo_params* p);

/* Create a handle for W x H u8 gray inputs and maximum disparity D (candidates
 * d = 0..D-1) at ORIGINAL resolution, on the current CUDA device.
 * Validates, in order: lambda_ad > 0, lambda_mc > 0, delta > 0,
 * t_fill >= 0, w_x >= 0, w_y >= 0, k_scale >= 1, D >= 1, W >= 1, H >= 1,
 * W/K >= 1, H/K >= 1, six distinct non-zero census offsets -> STEREO_EINVAL.
 * STEREO_EUNSUPPORTED for K not in {1,2}, ceil(D/K) > 255 (u8 maps use 255 as
 * INVALID), w_x or w_x_r > 254 (u8 arms), w_y > 112 (the y-aggregation tile
 * holds B + 2*w_y <= 240 rows), census offsets beyond +-2, m_pool > 3, and
 * scaled widths W/K > 2016 (the x pass keeps a row in 32 lane chunks of at
 * most 63 columns).
 * STEREO_EINVAL also for w_x_r < -1 and fill_mode outside STEREO_FILL_*.
 * Allocates every device buffer (dominant: two u32 CA_x volumes of
 * Ds*Hs*Ws*4 bytes each), builds the fixed-point cost tables on the host in
 * double precision and uploads them.  No kernel runs.  On success *out owns
 * the handle (release with stereo_destroy).  The handle is bound to the CUDA
 * device current at create: every later call switches to that device for its
 * own work and restores the caller's current device before returning. */
int stereo_create(int W, int H, int D, const stereo_params* p, stereo_t** out);

/* Enqueue one frame on `stream` and return without synchronising.
 * L, R: DEVICE u8 [H][W], row pitch W (rectified left/right gray images).
 * disp_out: DEVICE f32 [H][W], receives D^{fL_org}, the left-based
 * disparity in original-resolution pixels, range [0, K*(Ds-1)]; every pixel is
 * written, INVALID is never emitted.  L, R and disp_out stay owned by the
 * caller and must remain valid until the stream work completes.  A handle is
 * not re-entrant: use one handle per concurrently running stream.
 * STEREO_EINVAL for NULL pointers or a band handle (stereo_compute_band). */
int stereo_compute(stereo_t* h, const uint8_t* L, const uint8_t* R, float* disp_out,
                   void* stream);

/* As stereo_create, with buffers for up to max_frames frames (>= 1) so that
 * stereo_compute_batch enqueues each kernel ONCE per chunk of max_frames
 * frames (SD / census+arms / C+CA_x / CA+WTA / CC+median+fill+SU: five
 * launches per chunk, K = 2; four for K = 1) instead of once per frame.
 * Device memory grows linearly with max_frames (stereo_info.device_bytes).
 * STEREO_EINVAL for max_frames < 1; STEREO_EUNSUPPORTED if
 * max_frames * H/K > 2^20.  Stage access (debug up/download, run_stage,
 * set_debug) needs max_frames == 1. */
int stereo_create_batch(int W, int H, int D, const stereo_params* p, int max_frames,
                        stereo_t** out);

/* `nframes` (>= 0; 0 is a no-op that accepts NULL buffers) frames back to
 * back; L, R: DEVICE u8 [nframes][H][W];
 * disp_out: DEVICE f32 [nframes][H][W].  Processed in chunks of the handle's
 * max_frames, one launch sequence per chunk.  Same contract as
 * stereo_compute (enqueued on `stream`, no synchronisation, no allocation). */
int stereo_compute_batch(stereo_t* h, const uint8_t* L, const uint8_t* R, int nframes,
                         float* disp_out, void* stream);

/* End-to-end variant with HOST buffers: copies L and R (HOST u8 [H][W]) into
 * handle-owned device staging, computes, copies the result into disp_out
 * (HOST f32 [H][W]), all enqueued on `stream`; returns without synchronising.
 * Host buffers should be page-locked (cudaHostAlloc / torch pin_memory) for
 * the copies to be asynchronous; the caller must synchronise the stream
 * before reading disp_out or reusing L/R.  The FIRST host-buffer call on a
 * handle allocates the device staging (6*W*H*max_frames bytes, counted in
 * device_bytes); later calls never allocate. */
int stereo_compute_host(stereo_t* h, const uint8_t* L, const uint8_t* R, float* disp_out,
                        void* stream);

/* stereo_compute_host for `nframes` (>= 0; 0 is a no-op) frames back to
 * back: HOST L, R u8 [nframes][H][W], HOST disp_out f32 [nframes][H][W]; per
 * chunk of max_frames frames one copy in per image, one launch sequence, one
 * copy out, all enqueued on `stream`; the first host-buffer call allocates
 * the staging for max_frames frames (6*W*H*max_frames bytes).  Same rules as
 * stereo_compute_host. */
int stereo_compute_host_batch(stereo_t* h, const uint8_t* L, const uint8_t* R, int nframes,
                              float* disp_out, void* stream);

/* Synchronise the device, then free every buffer and the handle.  NULL is a
 * no-op. */
void stereo_destroy(stereo_t* h);

/* Thread-local description of the last error on this thread ("" if none). */
const char* stereo_last_error(void);

/* Derived sizes and resources of the handle (HOST struct). */
int stereo_get_info(const stereo_t* h, stereo_info* info);

/* Copy the handle's fixed-point tables to HOST arrays: qad[256] (indexed by
 * |dI|), qmc[7] (indexed by Hamming distance); *border = 2^(f+1). */
int stereo_get_tables(const stereo_t* h, uint32_t* qad, uint32_t* qmc, uint32_t* border);

/* ---- stage-level access (parity tests, profiling) ------------------------
 * Buffer ids and their layouts (all row-major, scaled resolution unless noted):
 *   STEREO_BUF_PIX_L/R : u16 [Hs][Ws]  = I | census << 8  (scaled image + code)
 *   STEREO_BUF_ARM_L/R : u32 [Hs][Ws]  = m | n << 8 | M << 16 | N << 24
 *                        (m, n: -x/+x arms; M, N: -y/+y arms)
 *   STEREO_BUF_CAX_L/R : u32 [ceil(Ds/2)][Hs][Wp][2]  Eq. 7 (fixed point),
 *                        disparities 2j and 2j+1 interleaved per pixel (the
 *                        x pass stores, the y pass TMA-loads disparity pairs);
 *                        Wp = cax_pitch = Ws rounded up to 32 (columns >= Ws
 *                        and the odd-Ds tail slot are undefined)
 *   STEREO_BUF_CA_L/R  : u64 [Ds][Hs][Ws]  Eq. 8, only after
 *                        stereo_set_debug(h, STEREO_DEBUG_CA, 1)
 *   STEREO_BUF_DL/DR   : u8  [Hs][Ws]  Eq. 9 WTA maps
 *   STEREO_BUF_MASKED  : u8  [Hs][Ws]  D^L with non-GCPs = 255 (Eq. 10)
 *   STEREO_BUF_MEDIAN  : u8  [Hs][Ws]  after the 3x3 median
 *   STEREO_BUF_FILL    : f32 [Hs][Ws]  D^{+L}
 *   STEREO_BUF_ROWS    : i32 [4][Hs]   per median-map row: first valid x, last
 *                        valid x, value at first, value at last (-1 = none)
 * stereo_debug_download synchronises the device; `bytes` must equal the
 * buffer size exactly (STEREO_EINVAL otherwise). */
enum {
  STEREO_BUF_PIX_L = 0, STEREO_BUF_PIX_R, STEREO_BUF_ARM_L, STEREO_BUF_ARM_R,
  STEREO_BUF_CAX_L, STEREO_BUF_CAX_R, STEREO_BUF_CA_L, STEREO_BUF_CA_R,
  STEREO_BUF_DL, STEREO_BUF_DR, STEREO_BUF_MASKED, STEREO_BUF_MEDIAN,
  STEREO_BUF_FILL, STEREO_BUF_ROWS, STEREO_BUF_COUNT
};
int stereo_debug_download(stereo_t* h, int buf_id, void* host_dst, size_t bytes);
int stereo_debug_upload(stereo_t* h, int buf_id, const void* host_src, size_t bytes);

/* Debug switches: STEREO_DEBUG_CA (allocate + store the CA volumes). */
enum { STEREO_DEBUG_CA = 1 };
int stereo_set_debug(stereo_t* h, int what, int enable);

/* Run ONE stage on the handle's buffers (after stereo_debug_upload of its
 * inputs).  L, R: DEVICE u8 [H][W] originals (used by SD and, for K = 1, by
 * PREP); disp_out: DEVICE f32 [H][W] (written by POST).  Stage ids follow the
 * paper's Table II taxonomy: SD | W^{LR}_+- and W^{*LR}_+- (PREP) |
 * C+CA_x (XPASS) | CA (YPASS) | CC + Post + SU (POST). */
enum {
  STEREO_STAGE_SD = 0,     /* Eq. 2 (K = 2 only; no-op for K = 1) */
  STEREO_STAGE_PREP,       /* census + x/y cross arms, both images (also writes the
                              x-pass row arrays, internal, not a debug buffer) */
  STEREO_STAGE_XPASS,      /* C + CA_x, both bases (reads PREP's internal row
                              arrays: run PREP first, uploads of PIX/ARM are not seen) */
  STEREO_STAGE_YPASS,      /* CA + WTA, both bases */
  STEREO_STAGE_POST,       /* cross-check + median + bilateral fill + scale-up */
  STEREO_STAGE_COUNT
};
int stereo_run_stage(stereo_t* h, int stage_id, const uint8_t* L, const uint8_t* R,
                     float* disp_out, void* stream);

/* Gray front end, §III list item 1 ("the two input images are
 * gray-scaled"; the formula is unstated -> BT.601 luma rounded half up,
 * reading R31): gray = floor((299 R + 587 G + 114 B + 500) / 1000).
 * rgb: DEVICE u8 [H][W][3] interleaved; gray: DEVICE u8 [H][W]; enqueued on
 * `stream` (cudaStream_t, NULL = legacy default).  STEREO_EINVAL for NULL
 * pointers or W, H < 1. */
int stereo_rgb_to_gray(const uint8_t* rgb, uint8_t* gray, int W, int H, void* stream);

/* stereo_compute for colour inputs: L_rgb, R_rgb DEVICE u8 [H][W][3]; the
 * gray conversion runs into handle-owned buffers, then the normal pipeline.
 * Same ownership / error rules as stereo_compute. */
int stereo_compute_rgb(stereo_t* h, const uint8_t* L_rgb, const uint8_t* R_rgb,
                       float* disp_out, void* stream);

/* Depth from disparity, Eq. 1: Z = f B / d with fB = f*B given
 * as one binary32 value; Z = fl32(fB / d) (one correctly rounded division),
 * d <= 0 -> +infinity ("d = 0 means that the object is at infinity",
 * P:107-108).  disp, Z: DEVICE f32 [n] (e.g. disp_out of stereo_compute,
 * n = W*H; Z may alias disp); enqueued on `stream`.  STEREO_EINVAL for NULL
 * pointers or n < 0. */
int stereo_disparity_to_depth(const float* disp, float* Z, int n, float fB, void* stream);

/* ---- row bands -------------------------------
 * One frame split into horizontal bands, one per GPU.  A band owns original
 * rows [y0_org, y0_org + rows_org) of the W x H frame.  Its handle computes
 * SD, census, arms and C + CA_x over the band plus a halo of rows that covers
 * the dependency cone of the own rows (Eq. 8's vertical window w_y, P:229-233;
 * the census pattern's vertical reach; Eq. 2's pool radius; one scaled row
 * for the cross-check/median and for Step8's odd rows),
 * but CA + WTA only for the own scaled rows + 3 (the cross-check / median /
 * Step8 cone) and POST only for the own rows.  Borders follow the FRAME
 * (arms, census and Step8 see the real image edges), so the assembled bands
 * equal the whole-frame result bit for bit.  The only frame-wide rule is fill
 * rule (d) (reading R25b: a row with no valid pixel takes the last valid value
 * of the nearest row above that has one, else the first of the nearest row
 * below, else 0): it is resolved ON DEVICE from a frame-wide
 * int32 [H/K][2] summary that the caller assembles with one element-wise MAX
 * all-reduce (NCCL) — no host synchronisation anywhere in the band path.
 *
 * Per frame:  stereo_compute_band -> stereo_band_summary(summ) ->
 *             all_reduce(summ, MAX) -> stereo_band_finish(summ), all on one
 * stream. */

/* The library's partition of a frame of H rows into nbands bands (scaled rows
 * split as evenly as possible, band b gets rows [b*Hs/n, (b+1)*Hs/n) of the
 * Hs = H/K scaled rows; the last band also owns the extra row of an odd H).
 * Pure host arithmetic.  STEREO_EINVAL if nbands is not in 1..H/K or band is
 * not in 0..nbands-1; p supplies k_scale. */
int stereo_band_rows(int H, const stereo_params* p, int nbands, int band, int* y0_org,
                     int* rows_org);

/* Create the handle of the band [y0_org, y0_org + rows_org) of a W x H frame
 * (same validation as stereo_create, on the frame).  y0_org must be a
 * multiple of K and y0_org + rows_org a multiple of K or H, else
 * STEREO_EINVAL.  Buffers are sized for the band's sub-image (own rows +
 * halo), allocated here. */
int stereo_create_band(int W, int H, int D, const stereo_params* p, int y0_org, int rows_org,
                       stereo_t** out);

/* Halo rows the band [y0_org, y0_org + rows_org) of a frame of H rows needs
 * above / below its own rows (fewer at the frame's top / bottom edge), for
 * the parameters p (k_scale, w_y, m_pool, census_dy).  Pure host arithmetic
 * (no device needed); HOST outputs.  The same rules as stereo_create_band. */
int stereo_band_halo(int H, const stereo_params* p, int y0_org, int rows_org, int* halo_top_org,
                     int* halo_bot_org);

/* One frame of the band.  L_band, R_band: DEVICE u8 [halo_top + rows_org +
 * halo_bot][W], the frame's rows [y0_org - halo_top, y0_org + rows_org +
 * halo_bot) (the caller exchanges the halo rows with the neighbouring bands).
 * out_band: DEVICE f32 [rows_org][W], receives the band's own rows of
 * D^{fL_org}, final unless fill rule (d) applies to one of them (see
 * stereo_band_finish).  y0_org / rows_org / halos must equal the handle's
 * (STEREO_EINVAL otherwise).  Enqueued on `stream`; no synchronisation. */
int stereo_compute_band(stereo_t* h, const uint8_t* L_band, const uint8_t* R_band, int y0_org,
                        int rows_org, int halo_top_org, int halo_bot_org, float* out_band,
                        void* stream);

/* Write the band's per-row fill summaries into summ: DEVICE int32 [H/K][2]
 * over the whole frame, (last valid value, first valid value) of each own
 * scaled row after the median (-1 = no valid pixel), and -1 in every other
 * row, so that an element-wise MAX over the bands assembles the frame.
 * Enqueued on `stream` after the band's stereo_compute_band. */
int stereo_band_summary(stereo_t* h, int32_t* summ_dev, void* stream);

/* Resolve fill rule (d) for the rows the band's output reads, from the
 * frame-wide summ (DEVICE int32 [H/K][2], all bands assembled), and recompute
 * Step8 for the own output rows that read a patched row.  L_band / out_band
 * as in stereo_compute_band.  One small kernel that returns at once when no
 * such row is all-invalid.  Enqueued on `stream`. */
int stereo_band_finish(stereo_t* h, const int32_t* summ_dev, const uint8_t* L_band,
                       float* out_band, void* stream);

/* Per-stage device timing with CUDA events recorded on the compute stream.
 * stereo_set_timing(h, 1) resets the accumulators and starts recording around
 * every stage of every subsequent stereo_compute*; stereo_stage_times_ms
 * synchronises on the recorded events and returns, per stage id, the summed
 * milliseconds over *nframes frames recorded since the reset. */
int stereo_set_timing(stereo_t* h, int enable);
int stereo_stage_times_ms(stereo_t* h, double* ms_per_stage /* [STEREO_STAGE_COUNT] */,
                          int* nframes);

#ifdef __cplusplus
}
#endif
#endif /* STEREO_B200_H */
