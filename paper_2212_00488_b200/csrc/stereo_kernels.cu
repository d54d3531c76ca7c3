// stereo_kernels.cu — sm_100a kernels of the stereo hot path (v1).
//
// One kernel per Table II stage.  Every kernel cites the passage it
// implements; DESIGN.md §4 gives each one's data layout, roofline and
// algorithmic bytes.  Integer/fixed-point throughout up to WTA (bit-exact with
// the oracle's fixed mode); binary32 with explicit round-to-nearest intrinsics
// (no FMA contraction) for the fill and scale-up.
#include <climits>
#include <cstdio>

#include "stereo_internal.cuh"

namespace stereo {

namespace {
constexpr unsigned kFull = 0xffffffffu;
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }
}  // namespace

// ============================================================================
// SD — Eq. 2, Step1: L(x,y) = mean of the (2m+1)^2
// block of L_org around (Kx, Ky), border-clamped, rounded half up:
// floor((2*sum + n) / (2n)), n = (2m+1)^2.  K = 2 only (K = 1: no scaling).
// HBM-bound: reads 2*W*H bytes, writes 2*Ws*Hs bytes.
// ============================================================================
__global__ void __launch_bounds__(128) sd_kernel(const uint8_t* __restrict__ Lorg,
                                                 const uint8_t* __restrict__ Rorg,
                                                 uint8_t* __restrict__ Ls,
                                                 uint8_t* __restrict__ Rs, int W, int H,
                                                 int Ws, int Hs, int m) {
  const uint8_t* src = blockIdx.z ? Rorg : Lorg;
  uint8_t* dst = blockIdx.z ? Rs : Ls;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= Ws) return;
  const int n = (2 * m + 1) * (2 * m + 1);
  int sum = 0;
  for (int j = -m; j <= m; ++j) {
    const uint8_t* row = src + (size_t)clampi(2 * y + j, 0, H - 1) * W;
    for (int i = -m; i <= m; ++i) sum += __ldg(row + clampi(2 * x + i, 0, W - 1));
  }
  dst[(size_t)y * Ws + x] = (uint8_t)((2 * sum + n) / (2 * n));
}

cudaError_t launch_sd(const Geom& g, const uint8_t* Lorg, const uint8_t* Rorg, uint8_t* Ls,
                      uint8_t* Rs, cudaStream_t s) {
  dim3 grid((g.Ws + 127) / 128, g.Hs, 2);
  sd_kernel<<<grid, 128, 0, s>>>(Lorg, Rorg, Ls, Rs, g.W, g.H, g.Ws, g.Hs, g.m_pool);
  return cudaGetLastError();
}

// ============================================================================
// PREP — mini-census (Fig. 3; pattern is a parameter, reading R8)
// and the four cross arms (Steps 2 and 4)
// of both scaled images in one pass.  A 32x8 pixel tile is staged in shared
// memory as two strips: a vertical one (rows +-max(w_y,2), cols +-2) for the
// census and the y arms, a horizontal one (rows +-2, cols +-max(w_x,2)) for
// the x arms.  Coordinates are clamped on load (census border rule R11); arm
// scans stop at the real image border (R16) and at the first |dI| >= delta.
// Output: pix = I | code << 8 (u16), arm = m | n<<8 | M<<16 | N<<24 (u32).
// Also resets the per-row first/last-valid records used by FILL rule (d).
// ============================================================================
struct PrepArgs {
  const uint8_t* img[2];
  uint16_t* pix[2];
  uint32_t* arm[2];
  int32_t* rowFirst;
  int32_t* rowLast;
  int Ws, Hs, w_x, w_y, delta;
  int8_t cdx[6], cdy[6];
};

__global__ void __launch_bounds__(256) prep_kernel(PrepArgs a) {
  extern __shared__ uint8_t psm[];
  const int hy = max(a.w_y, 2), hx = max(a.w_x, 2);
  const int AW = 36, AH = 8 + 2 * hy;
  const int BW = 32 + 2 * hx, BH = 12;
  uint8_t* sA = psm;
  uint8_t* sB = psm + AW * AH;
  const uint8_t* img = blockIdx.z ? a.img[1] : a.img[0];
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 8;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int i = tid; i < AW * AH; i += 256) {
    int r = i / AW, c = i % AW;
    sA[i] = __ldg(img + (size_t)clampi(y0 - hy + r, 0, a.Hs - 1) * a.Ws +
                  clampi(x0 - 2 + c, 0, a.Ws - 1));
  }
  for (int i = tid; i < BW * BH; i += 256) {
    int r = i / BW, c = i % BW;
    sB[i] = __ldg(img + (size_t)clampi(y0 - 2 + r, 0, a.Hs - 1) * a.Ws +
                  clampi(x0 - hx + c, 0, a.Ws - 1));
  }
  __syncthreads();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x = x0 + tx, y = y0 + ty;
  if (blockIdx.x == 0 && blockIdx.z == 0 && tx == 0 && y < a.Hs) {
    a.rowFirst[y] = INT_MAX;
    a.rowLast[y] = -1;
  }
  if (x >= a.Ws || y >= a.Hs) return;
  const int c = sA[(ty + hy) * AW + tx + 2];
  int code = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i)
    code |= (sA[(ty + hy + a.cdy[i]) * AW + tx + 2 + a.cdx[i]] < c) << i;
  const uint8_t* rowB = sB + (ty + 2) * BW + tx + hx;
  int n = 0;
  while (n < a.w_x && x + n + 1 <= a.Ws - 1 && abs((int)rowB[n + 1] - c) < a.delta) ++n;
  int m = 0;
  while (m < a.w_x && x - m - 1 >= 0 && abs((int)rowB[-m - 1] - c) < a.delta) ++m;
  const uint8_t* colA = sA + (ty + hy) * AW + tx + 2;
  int N = 0;
  while (N < a.w_y && y + N + 1 <= a.Hs - 1 && abs((int)colA[(N + 1) * AW] - c) < a.delta) ++N;
  int M = 0;
  while (M < a.w_y && y - M - 1 >= 0 && abs((int)colA[-(M + 1) * AW] - c) < a.delta) ++M;
  const size_t o = (size_t)y * a.Ws + x;
  uint16_t* pix = blockIdx.z ? a.pix[1] : a.pix[0];
  uint32_t* armo = blockIdx.z ? a.arm[1] : a.arm[0];
  pix[o] = (uint16_t)(c | (code << 8));
  armo[o] = (uint32_t)m | ((uint32_t)n << 8) | ((uint32_t)M << 16) | ((uint32_t)N << 24);
}

cudaError_t launch_prep(const Geom& g, const uint8_t* Ls, const uint8_t* Rs, Buffers& b,
                        cudaStream_t s) {
  PrepArgs a;
  a.img[0] = Ls; a.img[1] = Rs;
  a.pix[0] = b.pixL; a.pix[1] = b.pixR;
  a.arm[0] = b.armL; a.arm[1] = b.armR;
  a.rowFirst = b.rowFirst; a.rowLast = b.rowLast;
  a.Ws = g.Ws; a.Hs = g.Hs; a.w_x = g.w_x; a.w_y = g.w_y; a.delta = g.delta;
  for (int i = 0; i < 6; ++i) { a.cdx[i] = g.cdx[i]; a.cdy[i] = g.cdy[i]; }
  const int hy = g.w_y > 2 ? g.w_y : 2, hx = g.w_x > 2 ? g.w_x : 2;
  const size_t smem = 36 * (8 + 2 * hy) + 12 * (32 + 2 * hx);
  dim3 grid((g.Ws + 31) / 32, (g.Hs + 7) / 8, 2);
  prep_kernel<<<grid, dim3(32, 8), smem, s>>>(a);
  return cudaGetLastError();
}

// ============================================================================
// XPASS — cost (Eqs. 3-5) + x aggregation (Eq. 7) for
// BOTH bases, Step3.  The right base reuses the left cost line
// (Eq. 6): C^R(x,d) = C^L(x+d,d), so ONE exclusive prefix row
//   P[k] = sum_{x'<k} Q(x',d)   (u32, modular: window sums < 2^32 are exact)
// gives  CA^L_x(x,d) = P[x+n_L+1] - P[x-m_L]
//        CA^R_x(x,d) = P[x+d+n_R+1] - P[x+d-m_R]   (P extended by BORDER
//                                                    beyond Ws)
// replacing the paper's O(W_x) direct sums by O(1) differences.
// Work unit = (row y, 16 consecutive d); each warp owns one d at a time:
//   phase A: lane l scans its contiguous chunk [lC, lC+C) (C odd -> shared
//            loads at stride C are bank-conflict free); costs from the fixed
//            tables Q_AD[|dI|] and Q_MC[cL ^ cR] (popc folded into a 64-entry
//            table), both replicated per bank (index*32 + lane);
//   warp scan of the 32 lane totals (shuffles) -> P into shared memory;
//   phase C: lanes interleaved over x -> two coalesced 128-B stores per warp.
// Output layout: u32 [Ds][Hs][Wp] (Wp = Ws rounded up to 32).
// Bound: HBM writes (8 B per (x,y,d)) vs shared-memory wavefronts.
// ============================================================================
struct XArgs {
  const uint16_t* pixL;
  const uint16_t* pixR;
  const uint32_t* armL;
  const uint32_t* armR;
  const uint32_t* qad;
  const uint32_t* qmc;
  uint32_t* caxL;
  uint32_t* caxR;
  int Ws, Hs, Ds, Wp;
  uint32_t border;
};

constexpr int kXWarps = 8;
constexpr int kXDPerUnit = 16;

template <int C>
__global__ void __launch_bounds__(kXWarps * 32) xpass_kernel(XArgs a) {
  extern __shared__ uint32_t xsm[];
  uint32_t* sQAD = xsm;              // [256][32]
  uint32_t* sQMC = sQAD + 256 * 32;  // [64][32], indexed by cL ^ cR
  uint32_t* sL = sQMC + 64 * 32;     // [32C] pixL row (u32)
  uint32_t* sR = sL + 32 * C;        // [32C] pixR row
  uint32_t* sA = sR + 32 * C;        // [32C] mL | nL<<8 | mR<<16 | nR<<24
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* P = sA + 32 * C + warp * (32 * C + 1);  // [32C+1] exclusive prefix

  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sQAD[i] = __ldg(a.qad + (i >> 5));
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) sQMC[i] = __ldg(a.qmc + __popc(i >> 5));

  const int nch = (a.Ds + kXDPerUnit - 1) / kXDPerUnit;
  const int units = a.Hs * nch;
  const int Ws = a.Ws;
  const uint32_t border = a.border;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int y = u / nch, d0 = (u % nch) * kXDPerUnit;
    __syncthreads();  // previous unit finished with the row buffers
    for (int x = threadIdx.x; x < 32 * C; x += blockDim.x) {
      if (x < Ws) {
        const size_t o = (size_t)y * Ws + x;
        sL[x] = __ldg(a.pixL + o);
        sR[x] = __ldg(a.pixR + o);
        sA[x] = (__ldg(a.armL + o) & 0xffffu) | (__ldg(a.armR + o) << 16);
      } else {
        sL[x] = 0; sR[x] = 0; sA[x] = 0;
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int j = 0; j < kXDPerUnit / kXWarps; ++j) {
      const int d = d0 + j * kXWarps + warp;
      if (d >= a.Ds) break;
      // ---- phase A: costs of the lane's chunk + local inclusive prefix
      uint32_t pref[C];
      uint32_t run = 0;
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int x = lane * C + k;
        uint32_t q = border;  // x - d < 0: out of the right image (reading R12b)
        if (x >= d) {
          const uint32_t pl = sL[x], pr = sR[x - d];
          const int ad = abs((int)(pl & 255u) - (int)(pr & 255u));
          const uint32_t hx = ((pl ^ pr) >> 8) & 63u;
          q = sQAD[ad * 32 + lane] + sQMC[hx * 32 + lane];
        }
        run += q;
        pref[k] = run;
      }
      uint32_t incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t off = incl - run;
#pragma unroll
      for (int k = 0; k < C; ++k) P[lane * C + k + 1] = pref[k] + off;
      if (lane == 0) P[0] = 0;
      __syncwarp();
      // ---- phase C: window differences, coalesced stores
      const uint32_t PW = P[Ws];
      uint32_t* outL = a.caxL + ((size_t)d * a.Hs + y) * a.Wp;
      uint32_t* outR = a.caxR + ((size_t)d * a.Hs + y) * a.Wp;
#pragma unroll 4
      for (int i = 0; i < C; ++i) {
        const int x = lane + 32 * i;
        if (x < Ws) {
          const uint32_t ar = sA[x];
          const int mL = ar & 255u, nL = (ar >> 8) & 255u, mR = (ar >> 16) & 255u, nR = ar >> 24;
          const uint32_t caL = P[x + nL + 1] - P[x - mL];
          const int hi = x + d + nR + 1, lo = x + d - mR;
          const uint32_t Phi = hi <= Ws ? P[hi] : PW + (uint32_t)(hi - Ws) * border;
          const uint32_t Plo = lo <= Ws ? P[lo] : PW + (uint32_t)(lo - Ws) * border;
          outL[x] = caL;
          outR[x] = Phi - Plo;
        }
      }
      __syncwarp();
    }
  }
}

int xpass_chunk_for(int Ws) {
  static const int cs[] = {3, 7, 15, 23, 31, 47, 63};
  for (int c : cs)
    if (32 * c >= Ws) return c;
  return 0;
}

static size_t xpass_smem_bytes(int C) {
  return sizeof(uint32_t) * ((size_t)256 * 32 + 64 * 32 + 3 * 32 * C + kXWarps * (32 * C + 1));
}

template <int C>
static cudaError_t launch_xpass_c(const Geom& g, const Plan& p, Buffers& b, cudaStream_t s) {
  XArgs a{b.pixL, b.pixR, b.armL, b.armR, b.qad, b.qmc, b.caxL, b.caxR,
          g.Ws, g.Hs, g.Ds, g.Wp, g.border};
  xpass_kernel<C><<<p.xpass_grid, kXWarps * 32, p.xpass_smem, s>>>(a);
  return cudaGetLastError();
}

template <int C>
static cudaError_t setup_xpass_c(int smem) {
  return cudaFuncSetAttribute(xpass_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

template <int C>
static int occ_xpass_c(int smem) {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, xpass_kernel<C>, kXWarps * 32, smem);
  return n;
}

#define XPASS_DISPATCH(C_, EXPR) \
  switch (C_) {                  \
    case 3: { constexpr int CC = 3; EXPR; } break;   \
    case 7: { constexpr int CC = 7; EXPR; } break;   \
    case 15: { constexpr int CC = 15; EXPR; } break; \
    case 23: { constexpr int CC = 23; EXPR; } break; \
    case 31: { constexpr int CC = 31; EXPR; } break; \
    case 47: { constexpr int CC = 47; EXPR; } break; \
    case 63: { constexpr int CC = 63; EXPR; } break; \
    default: break;              \
  }

cudaError_t launch_xpass(const Geom& g, const Plan& p, Buffers& b, cudaStream_t s) {
  cudaError_t e = cudaErrorInvalidValue;
  XPASS_DISPATCH(p.xpass_C, e = launch_xpass_c<CC>(g, p, b, s));
  return e;
}

// ============================================================================
// YPASS — y aggregation (Eq. 8) + WTA (Eq. 9) for one
// base, Step5.  CTA = 32-column strip x B output rows; loops over
// d.  Per d the CTA loads the tile rows [y0-w_y, y0+B+w_y) of CA_x (coalesced
// 128-B rows), builds the exact u64 column prefix E (each warp a row segment
// serially in registers, segment offsets via shared memory), then every
// output pixel takes CA = E[y+N+1] - E[y-M] (O(1) instead of O(W_y)) and keeps
// the running minimum with the paper's strict "<": ties keep the
// smallest d.  Double-buffered prefix -> two barriers per d.
// ============================================================================
struct YArgs {
  const uint32_t* cax[2];
  const uint32_t* arm[2];
  uint8_t* Dmap[2];
  uint64_t* ca[2];  // debug (may be null)
  int Ws, Hs, Ds, Wp, w_y, B, T;
};

constexpr int kYWarps = 8;

template <int S, int RPT>
__global__ void __launch_bounds__(kYWarps * 32) ypass_kernel(YArgs a) {
  extern __shared__ uint64_t ysm[];
  const int T = a.T;
  uint64_t* sE = ysm;                        // [2][T+1][32]
  uint64_t* sTot = ysm + 2 * (T + 1) * 32;   // [2][kYWarps][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int base = blockIdx.z;
  const uint32_t* cax = base ? a.cax[1] : a.cax[0];
  const uint32_t* armp = base ? a.arm[1] : a.arm[0];
  uint64_t* cadbg = base ? a.ca[1] : a.ca[0];
  uint8_t* dmap = base ? a.Dmap[1] : a.Dmap[0];
  const int x = blockIdx.x * 32 + lane;
  const int y0 = blockIdx.y * a.B;
  const int yt0 = y0 - a.w_y;
  const bool xin = x < a.Ws;

  // output rows of this thread and their window indices into E
  int ia[RPT], ib[RPT];
  uint64_t best[RPT];
  int bd[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int y = y0 + w * RPT + r;
    ia[r] = 0; ib[r] = 0; best[r] = ~0ull; bd[r] = 0;
    if (xin && y < a.Hs && w * RPT + r < a.B) {
      const uint32_t arm = __ldg(armp + (size_t)y * a.Ws + x);
      const int M = (arm >> 16) & 255u, N = arm >> 24;
      ia[r] = y - M - yt0;
      ib[r] = y + N + 1 - yt0;
    }
  }
  const int seg0 = w * S;
  uint32_t v[S];
  auto load = [&](int d) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int yg = yt0 + seg0 + s;
      v[s] = 0;
      if (seg0 + s < T && yg >= 0 && yg < a.Hs)
        v[s] = __ldg(cax + ((size_t)d * a.Hs + yg) * a.Wp + x);
    }
  };
  load(0);
  for (int d = 0; d < a.Ds; ++d) {
    const int buf = d & 1;
    uint64_t loc[S];
    uint64_t acc = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      acc += v[s];
      loc[s] = acc;
    }
    sTot[(buf * kYWarps + w) * 32 + lane] = acc;
    __syncthreads();
    uint64_t off = 0;
    for (int q = 0; q < w; ++q) off += sTot[(buf * kYWarps + q) * 32 + lane];
    uint64_t* E = sE + (size_t)buf * (T + 1) * 32;
    if (w == 0) E[lane] = 0;
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (seg0 + s < T) E[(seg0 + s + 1) * 32 + lane] = loc[s] + off;
    if (d + 1 < a.Ds) load(d + 1);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const uint64_t ca = E[ib[r] * 32 + lane] - E[ia[r] * 32 + lane];
      if (ca < best[r]) { best[r] = ca; bd[r] = d; }
      if (cadbg) {
        const int y = y0 + w * RPT + r;
        if (xin && y < a.Hs && w * RPT + r < a.B) cadbg[((size_t)d * a.Hs + y) * a.Ws + x] = ca;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int y = y0 + w * RPT + r;
    if (xin && y < a.Hs && w * RPT + r < a.B) dmap[(size_t)y * a.Ws + x] = (uint8_t)bd[r];
  }
}

constexpr int kYRPT = 8;
constexpr int kYB = kYWarps * kYRPT;  // 64 output rows per tile

static size_t ypass_smem_bytes(int T) {
  return sizeof(uint64_t) * ((size_t)2 * (T + 1) * 32 + 2 * kYWarps * 32);
}

#define YPASS_DISPATCH(S_, EXPR)                             \
  switch (S_) {                                              \
    case 8: { constexpr int SS = 8; EXPR; } break;           \
    case 16: { constexpr int SS = 16; EXPR; } break;         \
    case 24: { constexpr int SS = 24; EXPR; } break;         \
    case 32: { constexpr int SS = 32; EXPR; } break;         \
    default: break;                                          \
  }

static int ypass_S_for(int T) {
  const int need = (T + kYWarps - 1) / kYWarps;
  for (int s : {8, 16, 24, 32})
    if (s >= need) return s;
  return 0;
}

cudaError_t launch_ypass(const Geom& g, const Plan& p, Buffers& b, bool store_ca,
                         cudaStream_t s) {
  YArgs a;
  a.cax[0] = b.caxL; a.cax[1] = b.caxR;
  a.arm[0] = b.armL; a.arm[1] = b.armR;
  a.Dmap[0] = b.DL; a.Dmap[1] = b.DR;
  a.ca[0] = store_ca ? b.caL : nullptr;
  a.ca[1] = store_ca ? b.caR : nullptr;
  a.Ws = g.Ws; a.Hs = g.Hs; a.Ds = g.Ds; a.Wp = g.Wp; a.w_y = g.w_y;
  a.B = p.ypass_B; a.T = p.ypass_T;
  dim3 grid((g.Ws + 31) / 32, (g.Hs + p.ypass_B - 1) / p.ypass_B, 2);
  cudaError_t e = cudaErrorInvalidValue;
  YPASS_DISPATCH(ypass_S_for(p.ypass_T),
                 (ypass_kernel<SS, kYRPT><<<grid, kYWarps * 32, p.ypass_smem, s>>>(a),
                  e = cudaGetLastError()));
  return e;
}

// ============================================================================
// CCMED — cross-check (Eq. 10; Step6 P:504-511; reading E5: the
// partner is D^R[y][x-k]) fused with the 3x3 median on the masked left map
// (Step7 first half; readings R21-R23).  A 34x10 masked tile (1-px
// clamped halo) is built in shared memory; each pixel sorts its 9 clamped
// neighbours with a 25-comparator network in registers (INVALID = 255 sorts
// last) and takes sorted[(n_valid-1)/2].  Per-row first/last valid column are
// recorded (warp ballot + one atomic per warp) for FILL rule (d).
// ============================================================================
__device__ __forceinline__ void cswap(int& a, int& b) {
  const int lo = min(a, b), hi = max(a, b);
  a = lo; b = hi;
}

__global__ void __launch_bounds__(256) ccmed_kernel(const uint8_t* __restrict__ DL,
                                                    const uint8_t* __restrict__ DR,
                                                    uint8_t* __restrict__ masked,
                                                    uint8_t* __restrict__ median,
                                                    int32_t* rowFirst, int32_t* rowLast,
                                                    int Ws, int Hs) {
  __shared__ uint8_t t[10][34];
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 8;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int i = tid; i < 340; i += 256) {
    const int r = i / 34, c = i % 34;
    const int yy = clampi(y0 - 1 + r, 0, Hs - 1), xx = clampi(x0 - 1 + c, 0, Ws - 1);
    const int k = __ldg(DL + (size_t)yy * Ws + xx);
    const bool gcp = (xx - k >= 0) && (__ldg(DR + (size_t)yy * Ws + xx - k) == k);
    t[r][c] = gcp ? (uint8_t)k : (uint8_t)kInvalid;
  }
  __syncthreads();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x = x0 + tx, y = y0 + ty;
  const bool in = x < Ws && y < Hs;
  int out = kInvalid;
  if (in) {
    const int c = t[ty + 1][tx + 1];
    if (c != kInvalid) {
      int v0 = t[ty][tx], v1 = t[ty][tx + 1], v2 = t[ty][tx + 2];
      int v3 = t[ty + 1][tx], v4 = c, v5 = t[ty + 1][tx + 2];
      int v6 = t[ty + 2][tx], v7 = t[ty + 2][tx + 1], v8 = t[ty + 2][tx + 2];
      const int n = (v0 != kInvalid) + (v1 != kInvalid) + (v2 != kInvalid) + (v3 != kInvalid) +
                    1 + (v5 != kInvalid) + (v6 != kInvalid) + (v7 != kInvalid) + (v8 != kInvalid);
      // 9-input sorting network (25 compare-exchanges)
      cswap(v0, v1); cswap(v3, v4); cswap(v6, v7);
      cswap(v1, v2); cswap(v4, v5); cswap(v7, v8);
      cswap(v0, v1); cswap(v3, v4); cswap(v6, v7);
      cswap(v0, v3); cswap(v3, v6); cswap(v0, v3);
      cswap(v1, v4); cswap(v4, v7); cswap(v1, v4);
      cswap(v2, v5); cswap(v5, v8); cswap(v2, v5);
      cswap(v1, v3); cswap(v5, v7); cswap(v2, v6);
      cswap(v4, v6); cswap(v2, v4); cswap(v2, v3);
      cswap(v5, v6);
      const int k = (n - 1) >> 1;  // 0..4
      out = k == 0 ? v0 : k == 1 ? v1 : k == 2 ? v2 : k == 3 ? v3 : v4;
    }
    const size_t o = (size_t)y * Ws + x;
    masked[o] = (uint8_t)c;
    median[o] = (uint8_t)out;
  }
  const unsigned bal = __ballot_sync(kFull, in && out != kInvalid);
  if (tx == 0 && bal && y < Hs) {
    atomicMin(rowFirst + y, x0 + __ffs(bal) - 1);
    atomicMax(rowLast + y, x0 + 31 - __clz(bal));
  }
}

cudaError_t launch_ccmed(const Geom& g, Buffers& b, cudaStream_t s) {
  dim3 grid((g.Ws + 31) / 32, (g.Hs + 7) / 8);
  ccmed_kernel<<<grid, dim3(32, 8), 0, s>>>(b.DL, b.DR, b.masked, b.median, b.rowFirst,
                                             b.rowLast, g.Ws, g.Hs);
  return cudaGetLastError();
}

// ============================================================================
// FILL — bilateral estimation of non-GCPs (§III.E steps 1-3; Step7
// P:516-525), one warp per row.  Nearest valid neighbours by ballot scans
// (left: forward pass with carry; right: backward pass), then
//  (a) |Dl-Dr| <= T: (Dl*j + Dr*i)/(i+j), one IEEE binary32 division (R26; the
//      sign of Eq. 11 as printed is reading E6);
//  (b) else the side whose scaled-L brightness is closer (tie -> left, R24);
//  (c) one-sided -> that side;  (d) all-invalid row -> last valid value of the
//      nearest row above, else first valid of the nearest row below, else 0.
// ============================================================================
__global__ void __launch_bounds__(256) fill_kernel(const uint8_t* __restrict__ median,
                                                   const uint16_t* __restrict__ pixL,
                                                   const int32_t* __restrict__ rowFirst,
                                                   const int32_t* __restrict__ rowLast,
                                                   float* __restrict__ out, int Ws, int Hs,
                                                   int T) {
  extern __shared__ int16_t fsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int y = blockIdx.x * 8 + w;
  if (y >= Hs) return;
  int16_t* sLeft = fsm + w * Ws;
  const uint8_t* med = median + (size_t)y * Ws;
  const uint16_t* pix = pixL + (size_t)y * Ws;
  float* o = out + (size_t)y * Ws;
  const int nch = (Ws + 31) / 32;
  int carry = -1;
  for (int c = 0; c < nch; ++c) {
    const int x = c * 32 + lane;
    const bool valid = x < Ws && med[x] != kInvalid;
    const unsigned mask = __ballot_sync(kFull, valid);
    const unsigned below = mask & ((1u << lane) - 1u);
    if (x < Ws) sLeft[x] = (int16_t)(below ? c * 32 + 31 - __clz(below) : carry);
    if (mask) carry = c * 32 + 31 - __clz(mask);
  }
  if (carry < 0) {  // rule (d): no valid pixel in this row
    int v = 0;
    if (lane == 0) {
      bool found = false;
      for (int yy = y - 1; yy >= 0 && !found; --yy)
        if (rowLast[yy] >= 0 && rowLast[yy] < Ws) { v = median[(size_t)yy * Ws + rowLast[yy]]; found = true; }
      for (int yy = y + 1; yy < Hs && !found; ++yy)
        if (rowFirst[yy] >= 0 && rowFirst[yy] < Ws) { v = median[(size_t)yy * Ws + rowFirst[yy]]; found = true; }
    }
    v = __shfl_sync(kFull, v, 0);
    for (int x = lane; x < Ws; x += 32) o[x] = (float)v;
    return;
  }
  __syncwarp();
  int rcarry = -1;
  for (int c = nch - 1; c >= 0; --c) {
    const int x = c * 32 + lane;
    const bool valid = x < Ws && med[x] != kInvalid;
    const unsigned mask = __ballot_sync(kFull, valid);
    const unsigned above = lane == 31 ? 0u : (mask & ~((2u << lane) - 1u));
    const int ri = above ? c * 32 + __ffs(above) - 1 : rcarry;
    if (x < Ws) {
      float val;
      if (valid) {
        val = (float)med[x];
      } else {
        const int li = sLeft[x];
        if (li >= 0 && ri >= 0) {
          const int Dl = med[li], Dr = med[ri];
          const int i = x - li, j = ri - x;
          if (abs(Dl - Dr) <= T) {
            val = __fdiv_rn((float)(Dl * j + Dr * i), (float)(i + j));
          } else {
            const int cI = pix[x] & 255, lI = pix[li] & 255, rI = pix[ri] & 255;
            val = (abs(lI - cI) <= abs(rI - cI)) ? (float)Dl : (float)Dr;
          }
        } else if (li >= 0) {
          val = (float)med[li];
        } else {
          val = (float)med[ri];
        }
      }
      o[x] = val;
    }
    if (mask) rcarry = c * 32 + __ffs(mask) - 1;
  }
}

cudaError_t launch_fill(const Geom& g, Buffers& b, float* out, cudaStream_t s) {
  const size_t smem = sizeof(int16_t) * 8 * g.Ws;
  fill_kernel<<<(g.Hs + 7) / 8, 256, smem, s>>>(b.median, b.pixL, b.rowFirst, b.rowLast, out,
                                                g.Ws, g.Hs, g.t_fill);
  return cudaGetLastError();
}

// ============================================================================
// SU — Step8: values x K on the even grid (R27); odd columns of
// seeded rows by the bilateral rule with i = j = 1 and threshold K*T (R28),
// brightness from L_org; odd rows linear (mean of the neighbouring seeded
// rows, R30); a missing successor copies its predecessor.  One thread per
// output pixel, each recomputing the seeded-row values it needs (idempotent,
// binary32 round-to-nearest intrinsics: bit-identical to the oracle).
// ============================================================================
__device__ __forceinline__ float su_xval(const float* __restrict__ v,
                                         const uint8_t* __restrict__ Lorg, int X, int y, int W,
                                         int Ws, float thr) {
  const float* row = v + (size_t)y * Ws;
  if ((X & 1) == 0) {
    if ((X >> 1) < Ws) return 2.0f * __ldg(row + (X >> 1));
    X -= 1;  // extra last column of an odd width: copy the predecessor
  }
  const float a = 2.0f * __ldg(row + ((X - 1) >> 1));
  if (X + 1 < W && ((X + 1) >> 1) < Ws) {
    const float b = 2.0f * __ldg(row + ((X + 1) >> 1));
    if (fabsf(__fsub_rn(a, b)) <= thr) return __fmul_rn(__fadd_rn(a, b), 0.5f);
    const uint8_t* lr = Lorg + (size_t)(2 * y) * W;
    const int c = __ldg(lr + X);
    return (abs((int)__ldg(lr + X - 1) - c) <= abs((int)__ldg(lr + X + 1) - c)) ? a : b;
  }
  return a;
}

__global__ void __launch_bounds__(256) su_kernel(const float* __restrict__ v,
                                                 const uint8_t* __restrict__ Lorg,
                                                 float* __restrict__ out, int W, int H, int Ws,
                                                 int Hs, float thr) {
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  const int Y = blockIdx.y;
  if (X >= W) return;
  float r;
  if ((Y & 1) == 0 && (Y >> 1) < Hs) {
    r = su_xval(v, Lorg, X, Y >> 1, W, Ws, thr);
  } else if ((Y & 1) == 1 && Y + 1 < H && ((Y + 1) >> 1) < Hs) {
    r = __fmul_rn(__fadd_rn(su_xval(v, Lorg, X, (Y - 1) >> 1, W, Ws, thr),
                            su_xval(v, Lorg, X, (Y + 1) >> 1, W, Ws, thr)), 0.5f);
  } else {
    r = su_xval(v, Lorg, X, Hs - 1 < ((Y - 1) >> 1) ? Hs - 1 : ((Y - 1) >> 1), W, Ws, thr);
  }
  out[(size_t)Y * W + X] = r;
}

cudaError_t launch_su(const Geom& g, const float* fill, const uint8_t* Lorg, float* out,
                      cudaStream_t s) {
  dim3 grid((g.W + 255) / 256, g.H);
  su_kernel<<<grid, 256, 0, s>>>(fill, Lorg, out, g.W, g.H, g.Ws, g.Hs,
                                 (float)(g.K * g.t_fill));
  return cudaGetLastError();
}

// ============================================================================
// Launch planning (create time)
// ============================================================================
cudaError_t plan_kernels(const Geom& g, Plan& p, int device) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return e;
  p.xpass_C = xpass_chunk_for(g.Ws);
  if (!p.xpass_C) return cudaErrorInvalidValue;
  p.xpass_smem = (int)xpass_smem_bytes(p.xpass_C);
  int occ = 0;
  XPASS_DISPATCH(p.xpass_C, (e = setup_xpass_c<CC>(p.xpass_smem), occ = occ_xpass_c<CC>(p.xpass_smem)));
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int units = g.Hs * ((g.Ds + kXDPerUnit - 1) / kXDPerUnit);
  p.xpass_grid = units < occ * prop.multiProcessorCount ? units : occ * prop.multiProcessorCount;

  p.ypass_B = kYB;
  p.ypass_T = kYB + 2 * g.w_y;
  if (!ypass_S_for(p.ypass_T)) return cudaErrorInvalidValue;
  p.ypass_smem = (int)ypass_smem_bytes(p.ypass_T);
  YPASS_DISPATCH(ypass_S_for(p.ypass_T),
                 e = cudaFuncSetAttribute(ypass_kernel<SS, kYRPT>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          p.ypass_smem));
  return e;
}

}  // namespace stereo
