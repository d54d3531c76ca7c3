// stereo_abi.cu — host side of the C ABI declared in include/stereo.h.
//
// Owns validation (SPEC S:59-61 order), the fixed-point table builder, the
// buffer planner, the per-frame launch sequence (Step1..Step8 order)
// and the CUDA-event stage timers.  No kernel runs at create time.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/stereo.h"
#include "stereo_internal.cuh"

using namespace stereo;

namespace {
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                 \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return fail(e_ == cudaErrorMemoryAllocation ? STEREO_ENOMEM : STEREO_ECUDA, \
                  "%s: %s", #call, cudaGetErrorString(e_));                      \
  } while (0)

constexpr int kMaxMarks = 140;  // launches per sequence (L2 band staging: 2 per band)

struct TimedFrame {
  cudaEvent_t ev[kMaxMarks + 1];
  int stage[kMaxMarks];
  int n;
  int frames;  // frames of this launch sequence (a batch chunk)
};

// Entry points run on the handle's device whatever the calling thread's
// current device is (buffers, tensor maps and planned attributes live there).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

struct stereo_s {
  Geom g{};
  Plan plan{};
  Buffers b{};
  stereo_params params{};
  int device = 0;
  bool debug_ca = false;
  int l2_tail0 = -1, l2_tail1 = -1;  // L2 band staging: CA_x rows still to discard
  uint32_t qad_h[256];
  uint32_t qmc_h[7];
  std::vector<void*> allocs;
  uint64_t bytes = 0;  // device bytes owned (every allocation, padding included)
  // timing
  bool timing = false;
  std::vector<TimedFrame> pending;
  std::vector<cudaEvent_t> pool;
  double acc_ms[STEREO_STAGE_COUNT] = {0};
  int acc_frames = 0;
};

namespace {

int alloc(stereo_t* h, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess)
    return fail(STEREO_ENOMEM, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
  h->allocs.push_back(*p);
  h->bytes += bytes;
  // defined contents from the start: the tail paddings that the word loads of
  // PREP / POST over-read are then initialised (compute-sanitizer initcheck)
  e = cudaMemset(*p, 0, bytes);
  if (e != cudaSuccess) return fail(STEREO_ECUDA, "cudaMemset: %s", cudaGetErrorString(e));
  return STEREO_OK;
}

// Eq. 4 / Eq. 5 evaluated in IEEE double, then quantised once:
// Q = floor(c * 2^f + 0.5)  (reading R12c).
void build_tables(const stereo_params& p, int f, uint32_t qad[256], uint32_t qmc[7]) {
  const double scale = std::ldexp(1.0, f);
  for (int a = 0; a < 256; ++a) {
    const double c = 1.0 - std::exp(-((static_cast<double>(a) / 255.0) / p.lambda_ad));
    qad[a] = static_cast<uint32_t>(std::floor(c * scale + 0.5));
  }
  for (int k = 0; k < 7; ++k) {
    const double c = 1.0 - std::exp(-(static_cast<double>(k) / p.lambda_mc));
    qmc[k] = static_cast<uint32_t>(std::floor(c * scale + 0.5));
  }
}

int frac_bits(int w_x) {
  for (int f = 25; f >= 0; --f)
    if ((static_cast<uint64_t>(2 * w_x + 1) << (f + 1)) < (1ull << 32)) return f;
  return -1;
}

int validate(int W, int H, int D, const stereo_params* p) {
  if (!p) return fail(STEREO_EINVAL, "params must not be NULL");
  if (p->abi_version != STEREO_ABI_VERSION)
    return fail(STEREO_EINVAL, "abi_version %u != %u", p->abi_version, STEREO_ABI_VERSION);
  if (!(p->lambda_ad > 0)) return fail(STEREO_EINVAL, "lambda_ad must be > 0");
  if (!(p->lambda_mc > 0)) return fail(STEREO_EINVAL, "lambda_mc must be > 0");
  if (p->delta <= 0) return fail(STEREO_EINVAL, "delta must be > 0");
  if (p->t_fill < 0) return fail(STEREO_EINVAL, "t_fill must be >= 0");
  if (p->w_x < 0) return fail(STEREO_EINVAL, "w_x must be >= 0");
  if (p->w_y < 0) return fail(STEREO_EINVAL, "w_y must be >= 0");
  if (p->w_x_r < -1) return fail(STEREO_EINVAL, "w_x_r must be -1 (= w_x) or >= 0");
  if (p->k_scale < 1) return fail(STEREO_EINVAL, "k_scale must be >= 1");
  if (D < 1) return fail(STEREO_EINVAL, "D (d_max_org) must be >= 1");
  if (W < 1 || H < 1) return fail(STEREO_EINVAL, "W and H must be >= 1");
  if (p->m_pool < 0) return fail(STEREO_EINVAL, "m_pool must be >= 0");
  for (int i = 0; i < 6; ++i) {
    if (p->census_dx[i] == 0 && p->census_dy[i] == 0)
      return fail(STEREO_EINVAL, "census offset %d is zero", i);
    for (int j = 0; j < i; ++j)
      if (p->census_dx[i] == p->census_dx[j] && p->census_dy[i] == p->census_dy[j])
        return fail(STEREO_EINVAL, "census offsets %d and %d are not distinct", j, i);
  }
  if (p->fill_mode < STEREO_FILL_BILATERAL || p->fill_mode > STEREO_FILL_EQ11_LITERAL)
    return fail(STEREO_EINVAL, "fill_mode must be one of STEREO_FILL_*");
  if (p->k_scale > 2) return fail(STEREO_EUNSUPPORTED, "k_scale must be 1 or 2");
  if (W / p->k_scale < 1 || H / p->k_scale < 1)
    return fail(STEREO_EINVAL, "scaled image is empty (W/K or H/K < 1)");
  if ((D + p->k_scale - 1) / p->k_scale > 255)
    return fail(STEREO_EUNSUPPORTED, "ceil(D/K) must be <= 255 (u8 disparity maps)");
  if (p->w_x > 254 || p->w_y > 254 || p->w_x_r > 254)
    return fail(STEREO_EUNSUPPORTED, "w_x, w_x_r, w_y must be <= 254");
  if (p->m_pool > 3) return fail(STEREO_EUNSUPPORTED, "m_pool must be <= 3");
  for (int i = 0; i < 6; ++i)
    if (p->census_dx[i] < -2 || p->census_dx[i] > 2 || p->census_dy[i] < -2 || p->census_dy[i] > 2)
      return fail(STEREO_EUNSUPPORTED, "census offsets must lie within +-2");
  return STEREO_OK;
}

cudaEvent_t get_event(stereo_t* h) {
  if (!h->pool.empty()) {
    cudaEvent_t e = h->pool.back();
    h->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

int drain_one(stereo_t* h, size_t idx) {
  TimedFrame& f = h->pending[idx];
  CU(cudaEventSynchronize(f.ev[f.n]));
  for (int i = 0; i < f.n; ++i) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, f.ev[i], f.ev[i + 1]));
    h->acc_ms[f.stage[i]] += ms;
  }
  for (int i = 0; i <= f.n; ++i) h->pool.push_back(f.ev[i]);
  h->acc_frames += f.frames;
  return STEREO_OK;
}

// nfr frames (1..NB, back to back in L, R, out): the Step1..Step8 launch
// sequence, each kernel launched ONCE for all nfr frames.
int enqueue_frames(stereo_t* h, const uint8_t* L, const uint8_t* R, float* out, int nfr,
                   cudaStream_t s) {
  const Geom& g = h->g;
  Buffers& b = h->b;
  TimedFrame tf{};
  tf.frames = nfr;
  if (h->timing) {
    tf.ev[0] = get_event(h);
    cudaEventRecord(tf.ev[0], s);
  }
  auto mark = [&](int stage) {
    if (!h->timing || tf.n >= kMaxMarks) return;
    tf.stage[tf.n] = stage;
    tf.ev[tf.n + 1] = get_event(h);
    cudaEventRecord(tf.ev[tf.n + 1], s);
    tf.n += 1;
  };
  const uint8_t* Ls = L;
  const uint8_t* Rs = R;
  if (g.K == 2) {
    CU(launch_sd(g, h->plan, L, R, b.Ls, b.Rs, nfr, s));
    mark(STEREO_STAGE_SD);
    Ls = b.Ls;
    Rs = b.Rs;
  }
  const bool padded = (Ls == b.Ls && Rs == b.Rs) || (Ls == b.grayL && Rs == b.grayR);
  CU(launch_prep(g, h->plan, Ls, Rs, padded, b, nfr, s));
  mark(STEREO_STAGE_PREP);
  const Plan& p = h->plan;
  if (p.fused && !h->debug_ca) {
    // NEXT-1 prototype: one kernel from the PREP outputs to D^L, D^R
    CU(launch_fused(g, p, b, s));
    mark(STEREO_STAGE_YPASS);
  } else if (p.l2_bands > 1 && !h->debug_ca) {
    // L2 band staging (NEXT-1 prototype): x pass of band k's
    // rows (+ w_y rows ahead), then the y pass of band k's outputs, which
    // reads CA_x rows written moments before (L2 hits); rows no later band
    // reads are discarded from L2 by the next x-pass launch (no write-back)
    const int R = nfr * g.Hs, Bb = p.l2_band_rows, wy = g.w_y;
    for (int k = 0, xa = 0; k * Bb < R; ++k) {
      const int xb = std::min(R, (k + 1) * Bb + wy);
      int d0 = std::max(0, (k - 1) * Bb - wy), d1 = std::max(0, k * Bb - wy);
      if (k == 0) {  // the previous frame's tail, when disjoint from the rows written now
        d0 = d1 = 0;
        if (h->l2_tail0 >= xb && h->l2_tail1 > h->l2_tail0) { d0 = h->l2_tail0; d1 = h->l2_tail1; }
      }
      if (xb > xa || d1 > d0) CU(launch_xpass_rows(g, p, b, xa, xb - xa, d0, d1, s));
      mark(STEREO_STAGE_XPASS);
      xa = xb;
      CU(launch_ypass_rows(g, p, b, k * Bb, std::min(R, (k + 1) * Bb), s));
      mark(STEREO_STAGE_YPASS);
      h->l2_tail0 = std::max(0, k * Bb - wy);
      h->l2_tail1 = R;
    }
  } else {
    CU(launch_xpass(g, p, b, nfr, s));
    mark(STEREO_STAGE_XPASS);
    CU(launch_ypass(g, p, b, h->debug_ca, nfr, s));
    mark(STEREO_STAGE_YPASS);
  }
  CU(launch_post(g, h->plan, b, L, out, nfr, s));
  mark(STEREO_STAGE_POST);
  if (h->timing) {
    h->pending.push_back(tf);
    if (h->pending.size() > 4096) {  // bound the event pool; the GPU is far behind anyway
      int rc = drain_one(h, 0);
      h->pending.erase(h->pending.begin());
      if (rc) return rc;
    }
  }
  return STEREO_OK;
}

struct BufView {
  void* p;
  size_t bytes;
};

BufView buf_view(stereo_t* h, int id) {
  const Geom& g = h->g;
  const size_t n = (size_t)g.Ws * g.Hs;
  const size_t vol = (size_t)((g.Ds + 1) / 2) * 2 * g.Hs * g.Wp;  // disparity pairs (u32 x 2)
  switch (id) {
    case STEREO_BUF_PIX_L: return {h->b.pixL, n * 2};
    case STEREO_BUF_PIX_R: return {h->b.pixR, n * 2};
    case STEREO_BUF_ARM_L: return {h->b.armL, n * 4};
    case STEREO_BUF_ARM_R: return {h->b.armR, n * 4};
    case STEREO_BUF_CAX_L: return {h->b.caxL, vol * 4};
    case STEREO_BUF_CAX_R: return {h->b.caxR, vol * 4};
    case STEREO_BUF_CA_L: return {h->b.caL, h->b.caL ? n * g.Ds * 8 : 0};
    case STEREO_BUF_CA_R: return {h->b.caR, h->b.caR ? n * g.Ds * 8 : 0};
    case STEREO_BUF_DL: return {h->b.DL, n};
    case STEREO_BUF_DR: return {h->b.DR, n};
    case STEREO_BUF_MASKED: return {h->b.masked, n};
    case STEREO_BUF_MEDIAN: return {h->b.median, n};
    case STEREO_BUF_FILL: return {h->b.fill, n * 4};
    case STEREO_BUF_ROWS: return {h->b.rowFirst, (size_t)g.Hs * 16};
    default: return {nullptr, 0};
  }
}

}  // namespace

extern "C" {

void stereo_default_params(stereo_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof *p);
  p->abi_version = STEREO_ABI_VERSION;
  p->lambda_ad = 0.3;
  p->lambda_mc = 2.3;
  p->t_fill = 3;
  p->w_x = 21;
  p->w_y = 31;
  p->delta = 20;
  p->k_scale = 2;
  p->m_pool = 1;
  p->w_x_r = -1;
  p->fill_mode = STEREO_FILL_BILATERAL;
  const int8_t dx[6] = {0, -1, 1, -1, 1, 0}, dy[6] = {-2, -1, -1, 1, 1, 2};
  for (int i = 0; i < 6; ++i) {
    p->census_dx[i] = dx[i];
    p->census_dy[i] = dy[i];
  }
}

const char* stereo_last_error(void) { return g_err.c_str(); }

}  // extern "C"

namespace {

// Band geometry: the sub-image of original rows
// [r0, r1) whose own scaled rows [ys0, ys1) come out exactly as in the whole
// frame.  The dependency cone, in scaled rows: POST's own rows read D^L / D^R
// rows [ys0 - 1, ys1 + 1 + (K == 2)) (median +-1, Step8's odd rows read fill
// row y + 1); those maps read CA_x rows +-w_y (Eq. 8) and the y arms of their
// own rows (<= w_y rows away); CA_x rows read census rows +-cy (the pattern's
// vertical reach); Eq. 2 reads original rows 2y - m .. 2y + m.
struct BandGeom {
  int ys0, ys1, ya, yb, sa, sb, r0, r1;
};

int band_geom(int H, const stereo_params* p, int y0_org, int rows_org, BandGeom& bg) {
  const int K = p->k_scale, Hs = H / K;
  int cy = 0;
  for (int i = 0; i < 6; ++i) cy = std::max(cy, std::abs((int)p->census_dy[i]));
  if (y0_org < 0 || rows_org < 1 || y0_org + rows_org > H)
    return fail(STEREO_EINVAL, "band rows [%d, %d) outside the frame's %d rows", y0_org,
                y0_org + rows_org, H);
  const int end = y0_org + rows_org;
  if (y0_org % K || (end % K && end != H))
    return fail(STEREO_EINVAL, "band rows must start and end on multiples of K=%d (or end at H)", K);
  bg.ys0 = y0_org / K;
  bg.ys1 = end == H ? Hs : end / K;
  if (bg.ys1 <= bg.ys0 || bg.ys0 >= Hs)
    return fail(STEREO_EINVAL, "band [%d, %d) holds no scaled row", y0_org, end);
  bg.ya = std::max(0, bg.ys0 - 1);
  bg.yb = std::min(Hs, bg.ys1 + 1 + (K == 2 ? 1 : 0));
  bg.sa = std::max(0, bg.ya - p->w_y - cy);
  bg.sb = std::min(Hs, bg.yb + p->w_y + cy);
  if (K == 2) {
    bg.r0 = std::max(0, 2 * bg.sa - p->m_pool);
    bg.r0 -= bg.r0 & 1;  // even: the scaled grids coincide
    bg.r1 = bg.sb == Hs ? H : std::min(H, std::max(2 * (bg.sb - 1) + p->m_pool + 1, 2 * bg.sb));
  } else {
    bg.r0 = bg.sa;
    bg.r1 = bg.sb == Hs ? H : bg.sb;
  }
  return STEREO_OK;
}

int create_impl(int W, int H, int D, const stereo_params* p, int nb, const BandGeom* bg,
                int Hframe, int y0_org, int rows_org, stereo_t** out) {
  stereo_t* h = new (std::nothrow) stereo_t();
  if (!h) return fail(STEREO_ENOMEM, "host allocation failed");
  int rc;
  h->params = *p;
  Geom& g = h->g;
  g.W = W; g.H = H; g.D = D; g.K = p->k_scale; g.m_pool = p->m_pool;
  g.Ws = W / g.K; g.Hs = H / g.K; g.Ds = (D + g.K - 1) / g.K;
  g.NB = nb;
  g.Wp = 32 * xpass_chunk_for(g.Ws);  // CA_x pitch = the x pass's lane-chunk span
  g.w_x = p->w_x; g.w_y = p->w_y; g.delta = p->delta; g.t_fill = p->t_fill;
  g.w_x_r = p->w_x_r < 0 ? p->w_x : p->w_x_r;
  g.w_x_max = g.w_x > g.w_x_r ? g.w_x : g.w_x_r;
  g.fill_mode = p->fill_mode;
  g.f = frac_bits(g.w_x_max);
  g.border = 1u << (g.f + 1);
  for (int i = 0; i < 6; ++i) { g.cdx[i] = p->census_dx[i]; g.cdy[i] = p->census_dy[i]; }
  if (bg) {
    g.band = true;
    g.H_g = Hframe;
    g.Hs_g = Hframe / g.K;
    g.s0 = bg->r0 / g.K;
    g.pa = bg->ys0 - g.s0; g.pb = bg->ys1 - g.s0;
    g.ya = bg->ya - g.s0; g.yb = bg->yb - g.s0;
    g.y0_org = y0_org; g.rows_org = rows_org;
    g.top = y0_org - bg->r0; g.bot = bg->r1 - (y0_org + rows_org);
  }
  if (!xpass_chunk_for(g.Ws)) {
    delete h;
    return fail(STEREO_EUNSUPPORTED, "scaled width %d exceeds 2016", g.Ws);
  }
  if (g.w_y > 112) {
    delete h;
    return fail(STEREO_EUNSUPPORTED, "w_y > 112 not supported by the y-aggregation tile");
  }
  cudaError_t e = cudaGetDevice(&h->device);
  if (e != cudaSuccess) {
    delete h;
    return fail(STEREO_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  }
  build_tables(*p, g.f, h->qad_h, h->qmc_h);
  const size_t n = (size_t)g.Ws * g.Hs * nb;  // per-frame buffers x NB frames
  const size_t vol = (size_t)((g.Ds + 1) / 2) * 2 * g.Hs * nb * g.Wp;  // disparity pairs (u32 x 2)
  Buffers& b = h->b;
  struct A { void** p; size_t bytes; } as[] = {
      {(void**)&b.pixL, n * 2 + 16}, {(void**)&b.pixR, n * 2 + 16}, {(void**)&b.armL, n * 4},
      {(void**)&b.armR, n * 4}, {(void**)&b.caxL, vol * 4}, {(void**)&b.caxR, vol * 4},
      {(void**)&b.xrow, (size_t)4 * g.Hs * nb * g.Wp * 4},
      {(void**)&b.grayL, (size_t)W * H + 16}, {(void**)&b.grayR, (size_t)W * H + 16},
      {(void**)&b.DL, n + 16}, {(void**)&b.DR, n + 16}, {(void**)&b.masked, n}, {(void**)&b.median, n},
      {(void**)&b.rowFirst, (size_t)g.Hs * 16 * nb},
      {(void**)&b.counter, (size_t)4 * nb + 16},
      {(void**)&b.fill, n * 4}, {(void**)&b.qad, 256 * 4}, {(void**)&b.qmc, 7 * 4},
      {(void**)&b.qtab, (size_t)(256 + 64) * 32 * 4},
  };
  for (auto& a : as) {
    if ((rc = alloc(h, a.p, a.bytes))) { stereo_destroy(h); return rc; }
  }
  if (g.K == 2) {
    // + 16: PREP reads these rows as unaligned words (3-byte over-read)
    if ((rc = alloc(h, (void**)&b.Ls, n + 16)) || (rc = alloc(h, (void**)&b.Rs, n + 16))) {
      stereo_destroy(h);
      return rc;
    }
  }
  e = cudaMemcpy(b.qad, h->qad_h, sizeof h->qad_h, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(b.qmc, h->qmc_h, sizeof h->qmc_h, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {  // the x pass's shared-memory table image (one copy per bank)
    std::vector<uint32_t> tab((256 + 64) * 32);
    for (int i = 0; i < 256 * 32; ++i) tab[i] = h->qad_h[i >> 5];
    for (int i = 0; i < 64 * 32; ++i) tab[256 * 32 + i] = h->qmc_h[__builtin_popcount(i >> 5)];
    e = cudaMemcpy(b.qtab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = plan_kernels(g, h->plan, b, h->device);
  if (e != cudaSuccess) {
    stereo_destroy(h);
    return fail(STEREO_ECUDA, "setup: %s", cudaGetErrorString(e));
  }
  *out = h;
  return STEREO_OK;
}

}  // namespace

extern "C" {

int stereo_create(int W, int H, int D, const stereo_params* p, stereo_t** out) {
  return stereo_create_batch(W, H, D, p, 1, out);
}

int stereo_create_batch(int W, int H, int D, const stereo_params* p, int max_frames,
                        stereo_t** out) {
  g_err.clear();
  if (!out) return fail(STEREO_EINVAL, "out must not be NULL");
  *out = nullptr;
  int rc = validate(W, H, D, p);
  if (rc) return rc;
  if (max_frames < 1) return fail(STEREO_EINVAL, "max_frames must be >= 1");
  if ((size_t)max_frames * (H / p->k_scale) > (1u << 20))
    return fail(STEREO_EUNSUPPORTED, "max_frames * H/K must be <= 2^20 rows");
  return create_impl(W, H, D, p, max_frames, nullptr, 0, 0, 0, out);
}

int stereo_band_rows(int H, const stereo_params* p, int nbands, int band, int* y0_org,
                     int* rows_org) {
  g_err.clear();
  if (!p || !y0_org || !rows_org) return fail(STEREO_EINVAL, "NULL argument");
  if (p->k_scale < 1 || p->k_scale > 2) return fail(STEREO_EUNSUPPORTED, "k_scale must be 1 or 2");
  const int K = p->k_scale, Hs = H / K;
  if (H < 1 || nbands < 1 || nbands > Hs || band < 0 || band >= nbands)
    return fail(STEREO_EINVAL, "cannot split %d scaled rows into %d bands (band %d)", Hs, nbands, band);
  const int ys0 = (int)((long long)band * Hs / nbands), ys1 = (int)((long long)(band + 1) * Hs / nbands);
  *y0_org = K * ys0;
  *rows_org = (ys1 == Hs ? H : K * ys1) - K * ys0;
  return STEREO_OK;
}

int stereo_create_band(int W, int H, int D, const stereo_params* p, int y0_org, int rows_org,
                       stereo_t** out) {
  g_err.clear();
  if (!out) return fail(STEREO_EINVAL, "out must not be NULL");
  *out = nullptr;
  int rc = validate(W, H, D, p);
  if (rc) return rc;
  BandGeom bg;
  if ((rc = band_geom(H, p, y0_org, rows_org, bg))) return rc;
  return create_impl(W, bg.r1 - bg.r0, D, p, 1, &bg, H, y0_org, rows_org, out);
}

int stereo_band_halo(int H, const stereo_params* p, int y0_org, int rows_org, int* halo_top_org,
                     int* halo_bot_org) {
  g_err.clear();
  if (!p || !halo_top_org || !halo_bot_org) return fail(STEREO_EINVAL, "NULL argument");
  if (p->k_scale < 1 || p->k_scale > 2) return fail(STEREO_EUNSUPPORTED, "k_scale must be 1 or 2");
  if (p->w_y < 0 || p->m_pool < 0) return fail(STEREO_EINVAL, "w_y and m_pool must be >= 0");
  BandGeom bg;
  int rc = band_geom(H, p, y0_org, rows_org, bg);
  if (rc) return rc;
  *halo_top_org = y0_org - bg.r0;
  *halo_bot_org = bg.r1 - (y0_org + rows_org);
  return STEREO_OK;
}

void stereo_destroy(stereo_t* h) {
  if (!h) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (auto& f : h->pending)
    for (int i = 0; i <= f.n; ++i) cudaEventDestroy(f.ev[i]);
  for (auto e : h->pool) cudaEventDestroy(e);
  for (void* p : h->allocs) cudaFree(p);
  if (h->b.caL) cudaFree(h->b.caL);
  if (h->b.caR) cudaFree(h->b.caR);
  cudaSetDevice(cur);
  delete h;
}

int stereo_compute(stereo_t* h, const uint8_t* L, const uint8_t* R, float* disp_out,
                   void* stream) {
  if (!h || !L || !R || !disp_out) return fail(STEREO_EINVAL, "NULL handle or buffer");
  if (h->g.band) return fail(STEREO_EINVAL, "band handle: use stereo_compute_band");
  DeviceGuard dg(h->device);
  return enqueue_frames(h, L, R, disp_out, 1, (cudaStream_t)stream);
}

int stereo_rgb_to_gray(const uint8_t* rgb, uint8_t* gray, int W, int H, void* stream) {
  g_err.clear();
  if (!rgb || !gray) return fail(STEREO_EINVAL, "NULL buffer");
  if (W < 1 || H < 1) return fail(STEREO_EINVAL, "W and H must be >= 1");
  CU(launch_gray(rgb, nullptr, gray, nullptr, W, H, (cudaStream_t)stream));
  return STEREO_OK;
}

int stereo_disparity_to_depth(const float* disp, float* Z, int n, float fB, void* stream) {
  g_err.clear();
  if (!disp || !Z) return fail(STEREO_EINVAL, "NULL buffer");
  if (n < 0) return fail(STEREO_EINVAL, "n must be >= 0");
  CU(launch_depth(disp, Z, n, fB, (cudaStream_t)stream));
  return STEREO_OK;
}

int stereo_compute_rgb(stereo_t* h, const uint8_t* L_rgb, const uint8_t* R_rgb, float* disp_out,
                       void* stream) {
  if (!h || !L_rgb || !R_rgb || !disp_out) return fail(STEREO_EINVAL, "NULL handle or buffer");
  if (h->g.band) return fail(STEREO_EINVAL, "band handle: use stereo_compute_band");
  DeviceGuard dg(h->device);
  const cudaStream_t s = (cudaStream_t)stream;
  CU(launch_gray(L_rgb, R_rgb, h->b.grayL, h->b.grayR, h->g.W, h->g.H, s));
  return enqueue_frames(h, h->b.grayL, h->b.grayR, disp_out, 1, s);
}

int stereo_compute_batch(stereo_t* h, const uint8_t* L, const uint8_t* R, int nframes,
                         float* disp_out, void* stream) {
  if (!h || nframes < 0) return fail(STEREO_EINVAL, "NULL handle or negative nframes");
  if (nframes == 0) return STEREO_OK;  // nothing to enqueue (buffers may be NULL)
  if (!L || !R || !disp_out) return fail(STEREO_EINVAL, "NULL buffer");
  if (h->g.band) return fail(STEREO_EINVAL, "band handle: use stereo_compute_band");
  DeviceGuard dg(h->device);
  const size_t in = (size_t)h->g.W * h->g.H;
  // chunks of NB frames: five launches per chunk, whatever the chunk size
  for (int i = 0; i < nframes; i += h->g.NB) {
    const int nfr = std::min(h->g.NB, nframes - i);
    int rc = enqueue_frames(h, L + i * in, R + i * in, disp_out + i * in, nfr, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return STEREO_OK;
}

}  // extern "C"

namespace {
// device staging of the host-buffer calls: max_frames frames, allocated by
// the first such call on the handle (never again)
int host_staging(stereo_t* h) {
  if (h->b.inL) return STEREO_OK;
  const size_t in = (size_t)h->g.W * h->g.H * h->g.NB;
  int rc;
  if ((rc = alloc(h, (void**)&h->b.inL, in)) || (rc = alloc(h, (void**)&h->b.inR, in)) ||
      (rc = alloc(h, (void**)&h->b.outF, in * 4)))
    return rc;
  return STEREO_OK;
}
}  // namespace

extern "C" {

int stereo_compute_host(stereo_t* h, const uint8_t* L, const uint8_t* R, float* disp_out,
                        void* stream) {
  if (!h || !L || !R || !disp_out) return fail(STEREO_EINVAL, "NULL handle or buffer");
  if (h->g.band) return fail(STEREO_EINVAL, "band handle: use stereo_compute_band");
  DeviceGuard dg(h->device);
  const size_t in = (size_t)h->g.W * h->g.H;
  int rc;
  if ((rc = host_staging(h))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  CU(cudaMemcpyAsync(h->b.inL, L, in, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(h->b.inR, R, in, cudaMemcpyHostToDevice, s));
  if ((rc = enqueue_frames(h, h->b.inL, h->b.inR, h->b.outF, 1, s))) return rc;
  CU(cudaMemcpyAsync(disp_out, h->b.outF, in * 4, cudaMemcpyDeviceToHost, s));
  return STEREO_OK;
}

int stereo_compute_host_batch(stereo_t* h, const uint8_t* L, const uint8_t* R, int nframes,
                              float* disp_out, void* stream) {
  if (!h || nframes < 0) return fail(STEREO_EINVAL, "NULL handle or negative nframes");
  if (nframes == 0) return STEREO_OK;
  if (!L || !R || !disp_out) return fail(STEREO_EINVAL, "NULL buffer");
  if (h->g.band) return fail(STEREO_EINVAL, "band handle: use stereo_compute_band");
  DeviceGuard dg(h->device);
  const size_t in = (size_t)h->g.W * h->g.H;
  int rc;
  if ((rc = host_staging(h))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  // per chunk of max_frames frames: one copy in per image, one launch
  // sequence, one copy out (the staging is reused in stream order)
  for (int i = 0; i < nframes; i += h->g.NB) {
    const int nfr = std::min(h->g.NB, nframes - i);
    CU(cudaMemcpyAsync(h->b.inL, L + i * in, nfr * in, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(h->b.inR, R + i * in, nfr * in, cudaMemcpyHostToDevice, s));
    if ((rc = enqueue_frames(h, h->b.inL, h->b.inR, h->b.outF, nfr, s))) return rc;
    CU(cudaMemcpyAsync(disp_out + i * in, h->b.outF, nfr * in * 4, cudaMemcpyDeviceToHost, s));
  }
  return STEREO_OK;
}

int stereo_get_info(const stereo_t* h, stereo_info* info) {
  if (!h || !info) return fail(STEREO_EINVAL, "NULL handle or info");
  const Geom& g = h->g;
  info->W = g.W; info->H = g.H; info->D = g.D;
  info->Ws = g.Ws; info->Hs = g.Hs; info->Ds = g.Ds;
  info->frac_bits = g.f;
  info->device = h->device;
  const size_t vol = (size_t)((g.Ds + 1) / 2) * 2 * g.Hs * g.Wp;  // disparity pairs (u32 x 2)
  info->device_bytes = h->bytes + (h->b.caL ? 2 * (size_t)g.Ds * g.Hs * g.Ws * 8 : 0);
  info->cax_bytes = vol * 4;
  {
    const Plan& p = h->plan;
    const int agg = p.l2_bands > 1 ? 2 * ((g.NB * g.Hs + p.l2_band_rows - 1) / p.l2_band_rows) : 2;
    info->launches_per_frame = (g.K == 2 ? 3 : 2) + agg;  // per launch sequence (max_frames frames)
  }
  info->ypass_block_rows = h->plan.ypass_B;
  info->cax_pitch = g.Wp;
  info->max_frames = g.NB;
  info->band = g.band ? 1 : 0;
  info->band_y0_org = g.y0_org;
  info->band_rows_org = g.rows_org;
  info->band_halo_top_org = g.top;
  info->band_halo_bot_org = g.bot;
  info->ypass_rows = g.band ? g.yb - g.ya : g.Hs;
  return STEREO_OK;
}

int stereo_get_tables(const stereo_t* h, uint32_t* qad, uint32_t* qmc, uint32_t* border) {
  if (!h || !qad || !qmc || !border) return fail(STEREO_EINVAL, "NULL argument");
  std::memcpy(qad, h->qad_h, sizeof h->qad_h);
  std::memcpy(qmc, h->qmc_h, sizeof h->qmc_h);
  *border = h->g.border;
  return STEREO_OK;
}

int stereo_debug_download(stereo_t* h, int buf_id, void* host_dst, size_t bytes) {
  if (!h || !host_dst) return fail(STEREO_EINVAL, "NULL argument");
  if (h->g.NB != 1) return fail(STEREO_EINVAL, "stage access needs a handle of batch capacity 1");
  DeviceGuard dg(h->device);
  BufView v = buf_view(h, buf_id);
  if (!v.p) return fail(STEREO_EINVAL, "buffer %d not available", buf_id);
  if (bytes != v.bytes) return fail(STEREO_EINVAL, "buffer %d has %zu bytes, not %zu", buf_id, v.bytes, bytes);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(host_dst, v.p, bytes, cudaMemcpyDeviceToHost));
  return STEREO_OK;
}

int stereo_debug_upload(stereo_t* h, int buf_id, const void* host_src, size_t bytes) {
  if (!h || !host_src) return fail(STEREO_EINVAL, "NULL argument");
  if (h->g.NB != 1) return fail(STEREO_EINVAL, "stage access needs a handle of batch capacity 1");
  DeviceGuard dg(h->device);
  BufView v = buf_view(h, buf_id);
  if (!v.p) return fail(STEREO_EINVAL, "buffer %d not available", buf_id);
  if (bytes != v.bytes) return fail(STEREO_EINVAL, "buffer %d has %zu bytes, not %zu", buf_id, v.bytes, bytes);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(v.p, host_src, bytes, cudaMemcpyHostToDevice));
  return STEREO_OK;
}

int stereo_set_debug(stereo_t* h, int what, int enable) {
  if (!h) return fail(STEREO_EINVAL, "NULL handle");
  if (what != STEREO_DEBUG_CA) return fail(STEREO_EINVAL, "unknown debug switch %d", what);
  if (h->g.NB != 1) return fail(STEREO_EINVAL, "stage access needs a handle of batch capacity 1");
  DeviceGuard dg(h->device);
  h->l2_tail0 = h->l2_tail1 = -1;
  if (enable && !h->b.caL) {
    const size_t bytes = (size_t)h->g.Ds * h->g.Hs * h->g.Ws * 8;
    CU(cudaMalloc(&h->b.caL, bytes));
    CU(cudaMalloc(&h->b.caR, bytes));
  }
  h->debug_ca = enable != 0;
  return STEREO_OK;
}

int stereo_run_stage(stereo_t* h, int stage_id, const uint8_t* L, const uint8_t* R,
                     float* disp_out, void* stream) {
  if (!h) return fail(STEREO_EINVAL, "NULL handle");
  if (h->g.NB != 1) return fail(STEREO_EINVAL, "stage access needs a handle of batch capacity 1");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const Geom& g = h->g;
  Buffers& b = h->b;
  switch (stage_id) {
    case STEREO_STAGE_SD:
      if (g.K == 2) {
        if (!L || !R) return fail(STEREO_EINVAL, "SD needs L and R");
        CU(launch_sd(g, h->plan, L, R, b.Ls, b.Rs, 1, s));
      }
      return STEREO_OK;
    case STEREO_STAGE_PREP:
      if (g.K == 1 && (!L || !R)) return fail(STEREO_EINVAL, "PREP with K=1 needs L and R");
      CU(launch_prep(g, h->plan, g.K == 2 ? b.Ls : L, g.K == 2 ? b.Rs : R, g.K == 2, b, 1, s));
      return STEREO_OK;
    case STEREO_STAGE_XPASS: CU(launch_xpass(g, h->plan, b, 1, s)); return STEREO_OK;
    case STEREO_STAGE_YPASS: CU(launch_ypass(g, h->plan, b, h->debug_ca, 1, s)); return STEREO_OK;
    case STEREO_STAGE_POST:
      if (!disp_out || (g.K == 2 && !L)) return fail(STEREO_EINVAL, "POST needs disp_out (and L when K=2)");
      CU(launch_post(g, h->plan, b, L, disp_out, 1, s));
      return STEREO_OK;
    default: return fail(STEREO_EINVAL, "unknown stage %d", stage_id);
  }
}

int stereo_compute_band(stereo_t* h, const uint8_t* L_band, const uint8_t* R_band, int y0_org,
                        int rows_org, int halo_top_org, int halo_bot_org, float* out_band,
                        void* stream) {
  if (!h || !L_band || !R_band || !out_band) return fail(STEREO_EINVAL, "NULL handle or buffer");
  const Geom& g = h->g;
  if (!g.band) return fail(STEREO_EINVAL, "not a band handle (stereo_create_band)");
  if (y0_org != g.y0_org || rows_org != g.rows_org || halo_top_org != g.top || halo_bot_org != g.bot)
    return fail(STEREO_EINVAL,
                "band (y0 %d, rows %d, halo %d/%d) differs from the handle's (y0 %d, rows %d, halo %d/%d)",
                y0_org, rows_org, halo_top_org, halo_bot_org, g.y0_org, g.rows_org, g.top, g.bot);
  DeviceGuard dg(h->device);
  return enqueue_frames(h, L_band, R_band, out_band, 1, (cudaStream_t)stream);
}

int stereo_band_summary(stereo_t* h, int32_t* summ_dev, void* stream) {
  if (!h || !summ_dev) return fail(STEREO_EINVAL, "NULL handle or buffer");
  if (!h->g.band) return fail(STEREO_EINVAL, "not a band handle (stereo_create_band)");
  DeviceGuard dg(h->device);
  CU(launch_band_summary(h->g, h->b, summ_dev, (cudaStream_t)stream));
  return STEREO_OK;
}

int stereo_band_finish(stereo_t* h, const int32_t* summ_dev, const uint8_t* L_band,
                       float* out_band, void* stream) {
  if (!h || !summ_dev || !L_band || !out_band) return fail(STEREO_EINVAL, "NULL handle or buffer");
  if (!h->g.band) return fail(STEREO_EINVAL, "not a band handle (stereo_create_band)");
  DeviceGuard dg(h->device);
  CU(launch_band_finish(h->g, h->b, summ_dev, L_band, out_band, (cudaStream_t)stream));
  return STEREO_OK;
}

int stereo_set_timing(stereo_t* h, int enable) {
  if (!h) return fail(STEREO_EINVAL, "NULL handle");
  DeviceGuard dg(h->device);
  for (size_t i = 0; i < h->pending.size(); ++i) {
    cudaEventSynchronize(h->pending[i].ev[h->pending[i].n]);
    for (int k = 0; k <= h->pending[i].n; ++k) h->pool.push_back(h->pending[i].ev[k]);
  }
  h->pending.clear();
  for (double& v : h->acc_ms) v = 0;
  h->acc_frames = 0;
  h->timing = enable != 0;
  // pre-create the events of ~512 frames so the timed loop never calls cudaEventCreate
  while (h->timing && h->pool.size() < 512 * (STEREO_STAGE_COUNT + 1)) {
    cudaEvent_t e = nullptr;
    CU(cudaEventCreate(&e));
    h->pool.push_back(e);
  }
  return STEREO_OK;
}

int stereo_stage_times_ms(stereo_t* h, double* ms, int* nframes) {
  if (!h || !ms) return fail(STEREO_EINVAL, "NULL argument");
  DeviceGuard dg(h->device);
  for (size_t i = 0; i < h->pending.size(); ++i) {
    int rc = drain_one(h, i);
    if (rc) return rc;
  }
  h->pending.clear();
  for (int i = 0; i < STEREO_STAGE_COUNT; ++i) ms[i] = h->acc_ms[i];
  if (nframes) *nframes = h->acc_frames;
  return STEREO_OK;
}

}  // extern "C"
