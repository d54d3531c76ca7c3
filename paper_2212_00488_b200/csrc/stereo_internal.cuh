// stereo_internal.cuh — internal declarations shared by the kernels and the
// host ABI of libstereo_b200.so (never exposed through include/stereo.h).
#pragma once
#include <cuda.h>  // CUtensorMap (the driver entry point is resolved at run time)
#include <cuda_runtime.h>
#include <stdint.h>

namespace stereo {

constexpr int kInvalid = 255;  // INVALID disparity in u8 maps

// Geometry and derived constants of one handle (all sizes in elements).
struct Geom {
  int W, H, D;      // original size and max disparity
  int K, m_pool;    // scale factor, mean-pool radius
  int Ws, Hs, Ds;   // scaled sizes
  int Wp;           // row pitch (elements) of the CA_x volumes: Ws rounded up to 32
  int w_x, w_y, delta, t_fill;
  int w_x_r;        // right-base x arm cap (resolved: >= 0)
  int w_x_max;      // max(w_x, w_x_r): x halos and the fixed-point width
  int fill_mode;    // STEREO_FILL_*
  int f;            // fixed-point fraction bits
  uint32_t border;  // 2^(f+1): the BORDER cost (reading R12b)
  int8_t cdx[6], cdy[6];
  // frame batch: buffers hold NB frames; one launch of every kernel serves up
  // to NB frames (SD / PREP / POST index the frame by blockIdx.z; the x and
  // y passes see the batch as one image of NB*Hs rows: both are row-local or
  // window-local, and no window crosses a frame border since the arms stop at
  // the frame's own borders)
  int NB = 1;
  // row-band mode (stereo_create_band; W x H above is then the band's
  // sub-image: own rows + halo): own scaled rows [pa, pb) and the rows whose
  // D^L / D^R POST reads, [ya, yb), in sub-image coordinates; s0 = global
  // scaled row of sub-image row 0; Hs_g = the frame's scaled height
  bool band = false;
  int pa = 0, pb = 0, ya = 0, yb = 0;
  int s0 = 0, Hs_g = 0, H_g = 0;
  int y0_org = 0, rows_org = 0, top = 0, bot = 0;  // own original rows, halo rows
};

// Device buffers owned by a handle.
struct Buffers {
  uint8_t* Ls = nullptr;     // scaled left  u8 [Hs][Ws] (K=2 only)
  uint8_t* Rs = nullptr;     // scaled right u8 [Hs][Ws] (K=2 only)
  uint16_t* pixL = nullptr;  // I | census << 8
  uint16_t* pixR = nullptr;
  uint32_t* armL = nullptr;  // m | n<<8 | M<<16 | N<<24
  uint32_t* armR = nullptr;
  uint32_t* xrow = nullptr;  // u32 [4][Hs][Wp] x-pass rows: code L, code R (census | I << 24),
                             // window byte offsets L, R (4(x-m) | 4(x+n+1) << 16)
  uint32_t* caxL = nullptr;  // u32 [ceil(Ds/2)][Hs][Wp][2] (disparity pairs interleaved)
  uint32_t* caxR = nullptr;
  uint64_t* caL = nullptr;   // debug only: u64 [Ds][Hs][Ws]
  uint64_t* caR = nullptr;
  uint8_t* DL = nullptr;
  uint8_t* DR = nullptr;
  uint8_t* masked = nullptr;
  uint8_t* median = nullptr;
  int32_t* rowFirst = nullptr;  // int32 [NB][4][Hs]: first valid x, last valid x, their values (-1 = none)
  unsigned* counter = nullptr;  // POST last-block counters, one per frame (self-resetting)
  float* fill = nullptr;        // f32 [Hs][Ws]
  uint32_t* qad = nullptr;      // u32 [256]
  uint32_t* qmc = nullptr;      // u32 [7]
  uint32_t* qtab = nullptr;     // u32 [(256 + 64) * 32]: Q_AD[a] and Q_MC[popc(i)] replicated per bank
  // staging for stereo_compute_host
  uint8_t* inL = nullptr;
  uint8_t* inR = nullptr;
  float* outF = nullptr;
  // gray front end of stereo_compute_rgb: u8 [H][W] x 2
  uint8_t* grayL = nullptr;
  uint8_t* grayR = nullptr;
};

// Launch configuration chosen at create time.
struct Plan {
  int xpass_C = 0;  // lane chunk (odd), Ws <= 32*C
  int xpass_grid = 0;
  int xpass_smem = 0;
  int xpass_PL = 0;  // per-warp prefix buffer length
  bool xpass_fixpl = false;  // PL = 32C + 128 at compile time (small D_s + w_x)
  int xpass_warps = 0;
  int xpass_slots = 3;  // row slots of the bulk-copy ring
  int ypass_ver = 1;  // 1: 16-column strips, 2 CTAs/SM; 2: 32-column strips, 16 warps (ypass2_kernel)
  int ypass_B = 0;   // output rows per tile (<= 8*kYRPT)
  int ypass_nb = 0;  // tiles per column strip
  int ypass_SEG = 0; // tile rows per warp; TMA box height = 8*SEG
  int ypass_smem = 0;
  int l2_bands = 0;  // > 1: C+CA_x / CA+WTA interleaved over this many row bands (NEXT-1 prototype)
  int l2_band_rows = 0;
  CUtensorMap tmL, tmR;  // 3-D u64 maps over the CA_x volumes {Wp, Hs, ceil(Ds/2)}
  bool fused = false;   // NEXT-1 prototype: fused_kernel instead of the x and y passes
  int fused_smem = 0;
  int post_smem = 0;
  int post_rows = 2;     // scaled rows per POST CTA
  int post_threads = 512;
  int sd_smem = 0;
  int prep_smem = 0;
  int prep_rows = 1;  // pixel rows per PREP thread (tile 32 x 8*prep_rows)
};

// Launchers (stereo_kernels.cu).  All enqueue on `s` and return the launch
// error.  nfr = frames of this launch (1..g.NB), stored at frame slots 0..nfr-1
// of the handle's buffers; Lorg / Rorg / out hold nfr frames back to back.
cudaError_t launch_sd(const Geom& g, const Plan& p, const uint8_t* Lorg, const uint8_t* Rorg,
                      uint8_t* Ls, uint8_t* Rs, int nfr, cudaStream_t s);
// padded: Ls / Rs are handle buffers with >= 3 bytes of tail padding (word loads)
cudaError_t launch_prep(const Geom& g, const Plan& p, const uint8_t* Ls, const uint8_t* Rs, bool padded,
                        Buffers& b, int nfr, cudaStream_t s);
cudaError_t launch_xpass(const Geom& g, const Plan& p, Buffers& b, int nfr, cudaStream_t s);
// rows [row0, row0 + rows) of the batch image only; first discards rows
// [disc0, disc1) of both CA_x volumes from L2 (L2 band staging)
cudaError_t launch_xpass_rows(const Geom& g, const Plan& p, Buffers& b, int row0, int rows,
                              int disc0, int disc1, cudaStream_t s);
// output rows [y0, y1) of the batch image only (L2 band staging)
cudaError_t launch_ypass_rows(const Geom& g, const Plan& p, Buffers& b, int y0, int y1,
                              cudaStream_t s);
cudaError_t launch_ypass(const Geom& g, const Plan& p, Buffers& b, bool store_ca, int nfr,
                         cudaStream_t s);
// NEXT-1 prototype: cost + CA_x + CA + WTA in one kernel (CA_x stays on chip)
cudaError_t launch_fused(const Geom& g, const Plan& p, Buffers& b, cudaStream_t s);
// band mode: out = the caller's band output (own original rows only)
cudaError_t launch_post(const Geom& g, const Plan& p, Buffers& b, const uint8_t* Lorg,
                        float* out, int nfr, cudaStream_t s);
cudaError_t launch_depth(const float* disp, float* Z, int n, float fB, cudaStream_t s);
cudaError_t launch_gray(const uint8_t* rgb0, const uint8_t* rgb1, uint8_t* g0, uint8_t* g1,
                        int W, int H, cudaStream_t s);
// band mode: own-row summaries into the frame-wide int32 [Hs_g][2] buffer
// (last valid value, first valid value; -1 elsewhere) / rule (d) from the
// frame-wide summaries, then Step8 again for the output rows that read a
// patched row (a no-op kernel when the band has no all-invalid row)
cudaError_t launch_band_summary(const Geom& g, Buffers& b, int32_t* summ, cudaStream_t s);
cudaError_t launch_band_finish(const Geom& g, Buffers& b, const int32_t* summ,
                               const uint8_t* Lorg, float* out, cudaStream_t s);

// Plan helpers
int xpass_chunk_for(int Ws);  // 0 if unsupported
cudaError_t plan_kernels(const Geom& g, Plan& p, Buffers& b, int device);

}  // namespace stereo
