// stereo_kernels.cu — sm_100a kernels of the stereo hot path.
//
// Five kernels per frame, one per Table II group:
//   sd_kernel    SD                      (Eq. 2)
//   prep_kernel  W^{LR}_+- and W^{*LR}_+- (census + cross arms)
//   xpass_kernel C + CA_x                (Eqs. 3-7, both bases from one prefix row)
//   ypass_kernel CA + WTA                (Eqs. 8-9; TMA tile loads)
//   post_kernel  CC + Post + SU          (Eq. 10, median, Eq. 11 fill, Step8)
// Every kernel cites the passage it implements; DESIGN.md §4 gives each one's
// layout, roofline and algorithmic bytes.  Integer / fixed point up to WTA
// (bit-exact with the oracle's fixed mode); binary32 with explicit
// round-to-nearest intrinsics (no FMA contraction) for the fill and scale-up.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include "stereo_common.cuh"

namespace stereo {


// ============================================================================
// SD — Eq. 2, Step1: L(x,y) = mean of the (2m+1)^2
// block of L_org around (2x, 2y), border-clamped, rounded half up:
// floor((2*sum + n) / (2n)), n = (2m+1)^2.  One CTA per output row and image:
// the 2m+1 source rows are staged in shared memory with 4-byte loads.
// ============================================================================
template <int M>
__global__ void __launch_bounds__(256) sd_kernel(const uint8_t* __restrict__ Lorg,
                                                 const uint8_t* __restrict__ Rorg,
                                                 uint8_t* __restrict__ Ls,
                                                 uint8_t* __restrict__ Rs, int W, int H,
                                                 int Ws, int Hs) {
  extern __shared__ uint32_t sdm32[];
  uint8_t* sdm = reinterpret_cast<uint8_t*>(sdm32);
  constexpr int NR = 2 * M + 1, N = NR * NR;
  // blockIdx.z: frame of the batch (frames back to back in both buffers)
  const uint8_t* src = (blockIdx.y ? Rorg : Lorg) + (size_t)blockIdx.z * W * H;
  uint8_t* dst = (blockIdx.y ? Rs : Ls) + (size_t)blockIdx.z * Ws * Hs;
  const int y = blockIdx.x;
  const int Wq = (W + 3) & ~3;
  const bool vec = ((W & 3) == 0) && ((reinterpret_cast<uintptr_t>(src) & 3) == 0);
  if (M == 1 && vec) {
    // 3x3 case on aligned rows: stage the three-row COLUMN sums (u16, two per
    // word, summed as u16x2 lanes: <= 765, no carries), then every output is
    // cs(2x-1) + cs(2x) + cs(2x+1) (cs(-1) = cs(0); 2x+1 <= W-1 always)
    uint16_t* cs = reinterpret_cast<uint16_t*>(sdm32);
    const uint32_t* r0 = reinterpret_cast<const uint32_t*>(src + (size_t)clampi(2 * y - 1, 0, H - 1) * W);
    const uint32_t* r1 = reinterpret_cast<const uint32_t*>(src + (size_t)(2 * y) * W);
    const uint32_t* r2 = reinterpret_cast<const uint32_t*>(src + (size_t)clampi(2 * y + 1, 0, H - 1) * W);
    for (int i = threadIdx.x; i < (W >> 2); i += blockDim.x) {
      const uint32_t a = __ldg(r0 + i), b = __ldg(r1 + i), c = __ldg(r2 + i);
      const uint32_t ev = __byte_perm(a, 0, 0x4240) + __byte_perm(b, 0, 0x4240) + __byte_perm(c, 0, 0x4240);
      const uint32_t od = __byte_perm(a, 0, 0x4341) + __byte_perm(b, 0, 0x4341) + __byte_perm(c, 0, 0x4341);
      reinterpret_cast<uint2*>(cs)[i] = make_uint2(__byte_perm(ev, od, 0x5410), __byte_perm(ev, od, 0x7632));
    }
    __syncthreads();
    for (int t = threadIdx.x; 2 * t < Ws; t += blockDim.x) {
      const uint2 q = reinterpret_cast<const uint2*>(cs)[t];  // cs(4t .. 4t+3)
      const int c0 = q.x & 0xffff, c1 = q.x >> 16, c2 = q.y & 0xffff, c3 = q.y >> 16;
      const int cm = t ? cs[4 * t - 1] : c0;
      const int s0 = cm + c0 + c1, s1 = c1 + c2 + c3;
      const uint32_t o0 = (uint32_t)((2 * s0 + N) / (2 * N)), o1 = (uint32_t)((2 * s1 + N) / (2 * N));
      uint8_t* d = dst + (size_t)y * Ws + 2 * t;
      if (2 * t + 1 < Ws && (Ws & 1) == 0) {
        *reinterpret_cast<uint16_t*>(d) = (uint16_t)(o0 | o1 << 8);
      } else {
        d[0] = (uint8_t)o0;
        if (2 * t + 1 < Ws) d[1] = (uint8_t)o1;
      }
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const uint8_t* row = src + (size_t)clampi(2 * y + j - M, 0, H - 1) * W;
    if (vec) {
      const uint32_t* r4 = reinterpret_cast<const uint32_t*>(row);
      for (int i = threadIdx.x; i < (W >> 2); i += blockDim.x) sdm32[j * (Wq >> 2) + i] = __ldg(r4 + i);
    } else {
      for (int i = threadIdx.x; i < W; i += blockDim.x) sdm[j * Wq + i] = __ldg(row + i);
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < Ws; x += blockDim.x) {
    int sum = 0;
#pragma unroll
    for (int j = 0; j < NR; ++j)
#pragma unroll
      for (int i = -M; i <= M; ++i) sum += sdm[j * Wq + clampi(2 * x + i, 0, W - 1)];
    dst[(size_t)y * Ws + x] = (uint8_t)((2 * sum + N) / (2 * N));
  }
}

cudaError_t launch_sd(const Geom& g, const Plan& p, const uint8_t* Lorg, const uint8_t* Rorg,
                      uint8_t* Ls, uint8_t* Rs, int nfr, cudaStream_t s) {
  dim3 grid(g.Hs, 2, nfr);
  switch (g.m_pool) {
    case 0: sd_kernel<0><<<grid, 256, p.sd_smem, s>>>(Lorg, Rorg, Ls, Rs, g.W, g.H, g.Ws, g.Hs); break;
    case 1: sd_kernel<1><<<grid, 256, p.sd_smem, s>>>(Lorg, Rorg, Ls, Rs, g.W, g.H, g.Ws, g.Hs); break;
    case 2: sd_kernel<2><<<grid, 256, p.sd_smem, s>>>(Lorg, Rorg, Ls, Rs, g.W, g.H, g.Ws, g.Hs); break;
    default: sd_kernel<3><<<grid, 256, p.sd_smem, s>>>(Lorg, Rorg, Ls, Rs, g.W, g.H, g.Ws, g.Hs); break;
  }
  return cudaGetLastError();
}

// ============================================================================
// PREP — mini-census (Fig. 3; pattern is a parameter, reading R8)
// and the four cross arms (Steps 2 and 4)
// of both scaled images.  Tile: 32 columns x TH rows, 8*TH threads, every
// thread owning FOUR pixels so that the byte-SIMD video instructions work on
// four pixels at once:
//  * a horizontal strip (rows +-2, columns +-P4) serves the census and the
//    x arms of the four consecutive pixels (x0+4g .. +3, y) of thread (y, g);
//  * a TRANSPOSED vertical strip (column-major, rows +-Q4) serves the y arms of
//    the four consecutive pixels (x, y0+4q .. +3) of thread (x, q);
// census bit i of a pixel = [I(clamp(p + o_i)) < I(p)] (R9-R11; vcmpltu4 of
// the four neighbour bytes at offset o_i against the four centre bytes).
// An arm is the count of leading similar steps k = 1, 2, ...: per step one
// funnel shift brings the four neighbour bytes at distance k, |dI| by
// vabsdiffu4, the byte-SIMD ">= delta" test, an "alive" mask that stays 0
// after the first dissimilar step (R15, R16) and a byte add.  Counts are
// capped per pixel at min(w, distance to the image border) (R14, R16) with
// one vminu4.  Coordinates are clamped on load (census border R11); source
// rows are read as unaligned words (aligned pairs + funnel shift) when the
// source is a handle buffer with tail padding, else bytewise.
// Output: pix = I | code << 8 (u16), arm = m | n<<8 | M<<16 | N<<24 (u32),
// and the x-pass rows (pitch Wp): code word census | I << 24 and the x-window
// byte offsets 4(x-m) | 4(x+n+1) << 16.
// ============================================================================
struct PrepArgs {
  const uint8_t* img0;
  const uint8_t* img1;
  uint16_t* pix0;
  uint16_t* pix1;
  uint32_t* arm0;
  uint32_t* arm1;
  uint32_t* xrow;  // [4][NB*Hs][Wp]: x-pass code L, R; window offsets L, R
  int Ws, Hs, Wp, w_x, w_x_r, w_y, delta;  // w_x: left image (D^L) x cap, w_x_r: right
  int plane_rows;  // NB*Hs: rows of one xrow plane (frame f at rows f*Hs ..)
  int P4, BW, Q4, AV;  // strip pads and pitches in bytes (prep_geometry)
  int8_t cdx[6], cdy[6];
};

// one step of four arm scans: `alive` keeps bit 7 of a pixel's byte while
// every step so far was similar; cnt counts the similar steps per byte.
// The ">= delta" test on |dI| bytes (1 <= delta <= 255): dl4 replicates
// delta (delta < 128) or delta - 128 (BIG, delta >= 128);
// lo = ((diff & 0x7f) | 0x80) - dl never borrows across bytes, and bit 7 of
// (BIG ? lo & diff : lo | diff) is set iff diff >= delta.  BIG is a template
// parameter so that the test and the alive update fold into one three-input
// logic op (alive carries bit 7 only: no final mask).
template <bool BIG>
struct ArmStep {
  uint32_t c4, dl4, alive, cnt;
  __device__ __forceinline__ uint32_t kill(uint32_t nb4) const {  // bit 7: dissimilar
    const uint32_t diff = __vabsdiffu4(nb4, c4);
    const uint32_t lo = ((diff & 0x7f7f7f7fu) | 0x80808080u) - dl4;
    return BIG ? (lo & diff) : (lo | diff);
  }
  __device__ __forceinline__ void operator()(uint32_t nb4) {
    alive &= ~kill(nb4);
    cnt += alive >> 7;
  }
  __device__ __forceinline__ void sat(uint32_t nb4) {  // per-byte saturating count
    alive &= ~kill(nb4);
    cnt = __vaddus4(cnt, alive >> 7);
  }
};

// Leading similar steps k = 1 .. 4*ceil(kmax/4) of the four pixels whose
// centre bytes are word cw of s, towards higher byte addresses (fwd) or lower
// (bwd); per-byte counts, capped by the caller.  The loop bound is
// warp-uniform; the warp stops once none of its pixels is still alive.
// (Byte counts stay <= 252 in the loop; caps above 252, allowed up to 254,
// take one more group with saturating adds.)
template <bool BIG>
__device__ __forceinline__ uint32_t arm4_fwd(const uint32_t* s, int cw, ArmStep<BIG> st, int kmax) {
  uint32_t lo = s[cw];
  int q = 0;
  for (; 4 * q < min(kmax, 252); ++q) {
    const uint32_t hi = s[cw + q + 1];
    st(__funnelshift_r(lo, hi, 8));
    st(__funnelshift_r(lo, hi, 16));
    st(__funnelshift_r(lo, hi, 24));
    st(hi);
    lo = hi;
    if (!__any_sync(kFull, st.alive)) return st.cnt;
  }
  if (kmax > 252) {
    const uint32_t hi = s[cw + q + 1];
    st.sat(__funnelshift_r(lo, hi, 8));
    st.sat(__funnelshift_r(lo, hi, 16));
    st.sat(__funnelshift_r(lo, hi, 24));
    st.sat(hi);
  }
  return st.cnt;
}
template <bool BIG>
__device__ __forceinline__ uint32_t arm4_bwd(const uint32_t* s, int cw, ArmStep<BIG> st, int kmax) {
  uint32_t hi = s[cw];
  int q = 0;
  for (; 4 * q < min(kmax, 252); ++q) {
    const uint32_t lo = s[cw - q - 1];
    st(__funnelshift_r(lo, hi, 24));
    st(__funnelshift_r(lo, hi, 16));
    st(__funnelshift_r(lo, hi, 8));
    st(lo);
    hi = lo;
    if (!__any_sync(kFull, st.alive)) return st.cnt;
  }
  if (kmax > 252) {
    const uint32_t lo = s[cw - q - 1];
    st.sat(__funnelshift_r(lo, hi, 24));
    st.sat(__funnelshift_r(lo, hi, 16));
    st.sat(__funnelshift_r(lo, hi, 8));
    st.sat(lo);
  }
  return st.cnt;
}

// both arms of the four pixels at word cw of s (fwd -> f, bwd -> b)
__device__ __forceinline__ void arms4(const uint32_t* s, int cw, uint32_t dl4, int delta, int kmax,
                                      uint32_t& f, uint32_t& b) {
  if (delta > 255) {  // |dI| <= 255 < delta: every step similar, the caps decide
    f = b = 0xffffffffu;
  } else if (delta >= 128) {
    const ArmStep<true> st{s[cw], dl4, 0x80808080u, 0u};
    f = arm4_fwd(s, cw, st, kmax);
    b = arm4_bwd(s, cw, st, kmax);
  } else {
    const ArmStep<false> st{s[cw], dl4, 0x80808080u, 0u};
    f = arm4_fwd(s, cw, st, kmax);
    b = arm4_bwd(s, cw, st, kmax);
  }
}

// four bytes starting at p (any alignment): aligned word + successor (the
// source buffer must allow a 3-byte over-read)
__device__ __forceinline__ uint32_t ldg_u32_unaligned(const uint8_t* p) {
  const uintptr_t ad = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(ad & ~(uintptr_t)3);
  const uint32_t lo = __ldg(w);
  const int sh = 8 * (int)(ad & 3);
  return sh ? __funnelshift_r(lo, __ldg(w + 1), sh) : lo;
}

// per-byte caps min(w, dist_i), dist_i = base + step * i (clamped at 0)
__device__ __forceinline__ uint32_t caps4(int w, int base, int step) {
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) c |= (uint32_t)max(0, min(w, base + step * i)) << (8 * i);
  return c;
}

template <int TH, bool WORDS>
__global__ void __launch_bounds__(256) prep_kernel(PrepArgs a) {
  extern __shared__ uint32_t psm32[];
  const int BW = a.BW, AV = a.AV, P4 = a.P4, Q4 = a.Q4, Ws = a.Ws, Hs = a.Hs;
  uint8_t* sB = reinterpret_cast<uint8_t*>(psm32);  // [TH+4][BW] horizontal strip
  uint8_t* sV = sB + (TH + 4) * BW;                   // [32][AV]  vertical strip, column-major
  uint8_t* sYM = sV + 32 * AV;                        // [TH][32]  M (up) of the tile pixels
  uint8_t* sYN = sYM + TH * 32;                       // [TH][32]  N (down)
  // blockIdx.z = 2 * frame + image (0: left, 1: right)
  const int im = blockIdx.z & 1, fr = blockIdx.z >> 1;
  const size_t foff = (size_t)fr * Ws * Hs;
  const uint8_t* img = (im ? a.img1 : a.img0) + foff;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * TH;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  constexpr int NW = TH / 4;  // warps

  // ---- horizontal strip: rows y0-2 .. y0+TH+1, columns x0-P4 .. x0-P4+BW-1
  {
    const int cx0 = x0 - P4;
    if (WORDS && cx0 >= 0 && cx0 + BW <= Ws) {
      uint32_t* sB32 = reinterpret_cast<uint32_t*>(sB);
      const int nwr = BW >> 2;
      for (int r = warp; r < TH + 4; r += NW) {
        const uint8_t* row = img + (size_t)clampi(y0 - 2 + r, 0, Hs - 1) * Ws + cx0;
        for (int w = lane; w < nwr; w += 32) sB32[r * nwr + w] = ldg_u32_unaligned(row + 4 * w);
      }
    } else {
      for (int r = warp; r < TH + 4; r += NW) {
        const uint8_t* row = img + (size_t)clampi(y0 - 2 + r, 0, Hs - 1) * Ws;
        for (int c = lane; c < BW; c += 32) sB[r * BW + c] = __ldg(row + clampi(cx0 + c, 0, Ws - 1));
      }
    }
  }
  // ---- vertical strip: tile column c at byte c*AV, strip row j = image row
  // y0 - Q4 + j (clamped), j < TH + 2 Q4
  {
    const int nrow = TH + 2 * Q4;
    if (WORDS && x0 + 32 <= Ws) {
      // 4x4 byte blocks: four unaligned row words -> four column words
      uint32_t* sV32 = reinterpret_cast<uint32_t*>(sV);
      const int AVw = AV >> 2;
      for (int i = t; i < (nrow >> 2) * 8; i += 8 * TH) {
        const int jb = i >> 3, cb = i & 7;
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          w[k] = ldg_u32_unaligned(img + (size_t)clampi(y0 - Q4 + 4 * jb + k, 0, Hs - 1) * Ws +
                                   x0 + 4 * cb);
        const uint32_t l01 = __byte_perm(w[0], w[1], 0x5140), h01 = __byte_perm(w[0], w[1], 0x7362);
        const uint32_t l23 = __byte_perm(w[2], w[3], 0x5140), h23 = __byte_perm(w[2], w[3], 0x7362);
        sV32[(4 * cb + 0) * AVw + jb] = __byte_perm(l01, l23, 0x5410);
        sV32[(4 * cb + 1) * AVw + jb] = __byte_perm(l01, l23, 0x7632);
        sV32[(4 * cb + 2) * AVw + jb] = __byte_perm(h01, h23, 0x5410);
        sV32[(4 * cb + 3) * AVw + jb] = __byte_perm(h01, h23, 0x7632);
      }
    } else {
      const int col = clampi(x0 + lane, 0, Ws - 1);
      for (int j = warp; j < nrow; j += NW)
        sV[lane * AV + j] = __ldg(img + (size_t)clampi(y0 - Q4 + j, 0, Hs - 1) * Ws + col);
    }
  }
  __syncthreads();

  const uint32_t dl4 = (uint32_t)(a.delta >= 128 ? a.delta - 128 : a.delta) * 0x01010101u;
  const int wx = im ? a.w_x_r : a.w_x;  // per-base x cap

  // ---- y arms: thread (column x0 + lane, rows y0 + 4 warp .. +3)
  {
    const uint32_t* colV = reinterpret_cast<const uint32_t*>(sV + lane * AV);
    const int cwv = (Q4 >> 2) + warp;
    const int yb = y0 + 4 * warp;
    uint32_t N4, M4;
    arms4(colV, cwv, dl4, a.delta, a.w_y, N4, M4);
    N4 = __vminu4(N4, caps4(a.w_y, Hs - 1 - yb, -1));
    M4 = __vminu4(M4, caps4(a.w_y, yb, 1));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      sYN[(4 * warp + i) * 32 + lane] = (uint8_t)(N4 >> (8 * i));
      sYM[(4 * warp + i) * 32 + lane] = (uint8_t)(M4 >> (8 * i));
    }
  }

  // ---- census + x arms: thread (row y0 + r, pixels x0 + 4g .. +3)
  const int r = t >> 3, g = t & 7;
  const uint32_t* rowB = reinterpret_cast<const uint32_t*>(sB + (r + 2) * BW);
  const int cw = (P4 >> 2) + g;
  const uint32_t c4 = rowB[cw];
  uint32_t code4 = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(sB + (r + 2 + a.cdy[i]) * BW);
    const int bo = 4 * cw + a.cdx[i];
    const int wi = bo >> 2, sh = 8 * (bo & 3);
    const uint32_t nb4 = __funnelshift_r(rw[wi], rw[wi + 1], sh);
    code4 |= (__vcmpltu4(nb4, c4) & 0x01010101u) << i;
  }
  const int xb = x0 + 4 * g;
  uint32_t n4, m4;
  arms4(rowB, cw, dl4, a.delta, wx, n4, m4);
  n4 = __vminu4(n4, caps4(wx, Ws - 1 - xb, -1));
  m4 = __vminu4(m4, caps4(wx, xb, 1));
  __syncthreads();

  // ---- outputs of the thread's four pixels
  const int y = y0 + r;
  if (y >= Hs) return;
  const uint32_t M4 = *reinterpret_cast<const uint32_t*>(sYM + r * 32 + 4 * g);
  const uint32_t N4 = *reinterpret_cast<const uint32_t*>(sYN + r * 32 + 4 * g);
  const size_t plane = (size_t)a.plane_rows * a.Wp;
  uint32_t* xr = a.xrow + im * plane + ((size_t)fr * Hs + y) * a.Wp + xb;  // 16-B aligned (Wp = 32C)
  const uint32_t mnl = __byte_perm(m4, n4, 0x5140), mnh = __byte_perm(m4, n4, 0x7362);
  const uint32_t MNl = __byte_perm(M4, N4, 0x5140), MNh = __byte_perm(M4, N4, 0x7362);
  const uint32_t armw[4] = {__byte_perm(mnl, MNl, 0x5410), __byte_perm(mnl, MNl, 0x7632),
                            __byte_perm(mnh, MNh, 0x5410), __byte_perm(mnh, MNh, 0x7632)};
  const uint32_t pixw[2] = {__byte_perm(c4, code4, 0x5140), __byte_perm(c4, code4, 0x7362)};
  uint32_t codew[4], offw[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t x = (uint32_t)(xb + i);
    codew[i] = ((code4 >> (8 * i)) & 0xffu) | ((c4 >> (8 * i)) << 24);
    const uint32_t m = (m4 >> (8 * i)) & 0xffu, n = (n4 >> (8 * i)) & 0xffu;
    offw[i] = 4u * (x - m) | (4u * (x + n + 1)) << 16;
  }
  if (xb + 3 < Ws) {
    uint16_t* pix = (im ? a.pix1 : a.pix0) + foff + (size_t)y * Ws + xb;
    uint32_t* arm = (im ? a.arm1 : a.arm0) + foff + (size_t)y * Ws + xb;
    *reinterpret_cast<uint4*>(xr) = make_uint4(codew[0], codew[1], codew[2], codew[3]);
    *reinterpret_cast<uint4*>(xr + 2 * plane) = make_uint4(offw[0], offw[1], offw[2], offw[3]);
#pragma unroll
    for (int i = 0; i < 4; ++i) arm[i] = armw[i];
    if ((reinterpret_cast<uintptr_t>(pix) & 3) == 0) {
      reinterpret_cast<uint32_t*>(pix)[0] = pixw[0];
      reinterpret_cast<uint32_t*>(pix)[1] = pixw[1];
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) pix[i] = (uint16_t)(pixw[i >> 1] >> (16 * (i & 1)));
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x = xb + i;
      if (x < Ws) {
        xr[i] = codew[i];
        xr[2 * plane + i] = offw[i];
        (im ? a.arm1 : a.arm0)[foff + (size_t)y * Ws + x] = armw[i];
        (im ? a.pix1 : a.pix0)[foff + (size_t)y * Ws + x] = (uint16_t)(pixw[i >> 1] >> (16 * (i & 1)));
      } else if (x < a.Wp) {  // pitch padding of the x-pass rows: harmless windows, never read
        xr[i] = 0u;
        xr[2 * plane + i] = 4u * x | (4u * (x + 1)) << 16;
      }
    }
  }
}

static int prep_rows_for(const Geom& g, int nsm) {
  for (int pr : {4, 2})
    if ((long long)(g.Wp / 32) * ((g.Hs + 8 * pr - 1) / (8 * pr)) * 2 * g.NB >= 4LL * nsm) return pr;
  return 1;
}

// Strip geometry (bytes): P4 / Q4 = pads, multiples of 4 covering the arm cap
// rounded up to the 4-step granularity of the scans (and the census
// footprint); BW = horizontal strip pitch with BW/4 = 8 or 24 (mod 32), so the
// four rows a warp reads fall in distinct bank octets; AV = vertical strip
// pitch with AV/4 odd (conflict-free column accesses).
static void prep_geometry(const Geom& g, int th, int& P4, int& BW, int& Q4, int& AV) {
  const int hx = g.w_x_max > 2 ? g.w_x_max : 2;
  const int hy = g.w_y > 2 ? g.w_y : 2;
  P4 = 4 * ((hx + 3) / 4) + 4;
  BW = 32 + 2 * P4;
  while ((BW / 4) % 32 != 8 && (BW / 4) % 32 != 24) BW += 4;
  Q4 = 4 * ((hy + 3) / 4) + 4;
  AV = th + 2 * Q4;
  if (((AV >> 2) & 1) == 0) AV += 4;
}

static int prep_smem_bytes(int th, int BW, int AV) { return (th + 4) * BW + 32 * AV + 2 * th * 32 + 16; }

cudaError_t launch_prep(const Geom& g, const Plan& p, const uint8_t* Ls, const uint8_t* Rs,
                        bool padded, Buffers& b, int nfr, cudaStream_t s) {
  PrepArgs a;
  a.img0 = Ls; a.img1 = Rs;
  a.pix0 = b.pixL; a.pix1 = b.pixR;
  a.arm0 = b.armL; a.arm1 = b.armR;
  a.xrow = b.xrow;
  a.Ws = g.Ws; a.Hs = g.Hs; a.Wp = g.Wp; a.w_x = g.w_x; a.w_x_r = g.w_x_r; a.w_y = g.w_y;
  a.delta = g.delta;
  a.plane_rows = g.NB * g.Hs;
  const int th = 8 * p.prep_rows;
  prep_geometry(g, th, a.P4, a.BW, a.Q4, a.AV);
  for (int i = 0; i < 6; ++i) { a.cdx[i] = g.cdx[i]; a.cdy[i] = g.cdy[i]; }
  dim3 grid(g.Wp / 32, (g.Hs + th - 1) / th, 2 * nfr);
  const int smem = p.prep_smem;
  if (th == 32) {
    if (padded) prep_kernel<32, true><<<grid, 256, smem, s>>>(a);
    else prep_kernel<32, false><<<grid, 256, smem, s>>>(a);
  } else if (th == 16) {
    if (padded) prep_kernel<16, true><<<grid, 128, smem, s>>>(a);
    else prep_kernel<16, false><<<grid, 128, smem, s>>>(a);
  } else {
    if (padded) prep_kernel<8, true><<<grid, 64, smem, s>>>(a);
    else prep_kernel<8, false><<<grid, 64, smem, s>>>(a);
  }
  return cudaGetLastError();
}

// ============================================================================
// YPASS — y aggregation (Eq. 8) + WTA (Eq. 9) for one
// base, Step5.  CTA = 16-column strip x B output rows, looping over
// disparity pairs.  Per pair a TMA 3-D box {16 columns, TB = 16*SEG rows,
// 1 pair} of u64 (d, d+1) elements of the CA_x volume starting at row y0 - w_y
// lands in shared memory (rows outside the image are zero-filled by the TMA
// unit: they never enter a window); two stages, mbarrier-completed, refilled
// as soon as a stage is consumed.  Thread (col = t & 15, seg = t >> 4) scans
// SEG rows of its column serially in registers (split precision, exact, see
// below); the two segments of a warp combine by shuffle, the eight warp
// totals through shared memory; the exact column prefix E lands in shared
// memory and every output pixel takes CA = E[y+N+1] - E[y-M] (O(1) instead of
// O(W_y)) and keeps the running minimum with the paper's strict "<":
// ties keep the smallest d.  SEG is odd so the two half-warps' hi-prefix
// stores fall in disjoint banks; 16-column strips allow tall tiles (small
// halo ratio TB/B) at good grid balance.
// ============================================================================
struct YArgs {
  const uint32_t* arm0;
  const uint32_t* arm1;
  uint8_t* D0;
  uint8_t* D1;
  uint64_t* ca0;  // debug (may be null)
  uint64_t* ca1;
  int Ws, Hs, Ds, w_y, B;
  int y_begin, y_end;  // output rows of this launch (tiles of B rows from y_begin)
  uint32_t e52;  // kYExp52
};

constexpr int kYThreads = 256;
constexpr int kYSegs = 16;   // row segments per CTA (2 per warp)
constexpr int kYRPT = 12;    // output rows per thread (B <= 192)
constexpr int kYStages = 2;

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// Two disparities per iteration in split precision.  Every CA_x value is
// < 2^32 (choice of f, R12c); split it as x = hi*2^24 + lo with lo < 2^24:
// over any window of <= 2 w_y + 1 <= 225 rows the lo sum is < 2^32 and the hi
// sum < 2^16, so the column prefixes can be kept modulo 2^32 (lo of d and
// d+1) and modulo 2^16 (hi of d in the low half, of d+1 in the high half of one
// u32) and every window difference is still exact:
// CA = (lo_b - lo_a) + ((hi_b - hi_a) << 24).  12 bytes of prefix per two
// disparities instead of 16, i.e. fewer shared-memory wavefronts per output.
// The argmin key CA << 8 | d (CA < 2^40, d < 256) is then two 32-bit words
// {lo << 8 | d, (lo >> 24) + hi}: two ALU operations, no 64-bit shifts; the
// minimum of the keys is the paper's strict-< scan with ties to the smallest
// d.
constexpr int kYSplit = 24;  // = byte 3: the hi parts are extracted by byte permutes

// The running minimum is kept as the IEEE double 2^52 + key (key < 2^48 is
// exact and the map is monotone): one DSETP.MIN + two selects per candidate
// instead of a 64-bit integer compare-and-select.  `hib` is the hi window sum
// with the exponent bits 0x433 (2^52) already OR-ed in (hi < 2^16 + 2^8).
constexpr uint32_t kYExp52 = 0x43300000u;
__device__ __forceinline__ void ypass_take(double& best, uint32_t lo, uint32_t hib, int d) {
  uint32_t klo;  // lo << 8 | d as one multiply-add (d < 256)
  asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(klo) : "r"(lo), "r"(d));
  const uint32_t khi = (lo >> 24) + hib;
  const double kd = __hiloint2double((int)khi, (int)klo);
  if (kd < best) best = kd;  // never NaN: no fmin NaN fix-ups
}

// WTA over the window sums of d (and d+1 if TWO) for the thread's outputs
// r < NR (NR warp-uniform: straight-line code the scheduler can interleave).
// `z` is an opaque per-iteration zero: it keeps the optimiser from hoisting
// four d-invariant addresses per output out of the d loop (register spills).
template <int NR, bool TWO>
__device__ __forceinline__ void ypass_wta(double (&best)[kYRPT], const uint32_t (&oab)[kYRPT],
                                          const uint8_t* EloB, const uint8_t* EhiB, uint32_t z,
                                          uint32_t e52, int d) {
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const uint32_t v = oab[r] + z;
    const uint32_t ia = v & 0xffffu, ib = v >> 16;
    const uint2 la = *reinterpret_cast<const uint2*>(EloB + ia);
    const uint2 lb = *reinterpret_cast<const uint2*>(EloB + ib);
    const uint32_t dh = *reinterpret_cast<const uint32_t*>(EhiB + (ib >> 1)) -
                        *reinterpret_cast<const uint32_t*>(EhiB + (ia >> 1));
    uint32_t hib0;  // (dh & 0xffff) | e52 as one three-input logic op
    asm("lop3.b32 %0, %1, 0xffff, %2, 0xea;" : "=r"(hib0) : "r"(dh), "r"(e52));
    ypass_take(best[r], lb.x - la.x, hib0, d);
    if (TWO) ypass_take(best[r], lb.y - la.y, (dh >> 16) + e52, d + 1);
  }
}

template <bool TWO>
__device__ __forceinline__ void ypass_wta_n(int nr, double (&best)[kYRPT],
                                            const uint32_t (&oab)[kYRPT], const uint8_t* EloB,
                                            const uint8_t* EhiB, int d, uint32_t e52) {
  uint32_t z;  // opaque zero (see ypass_wta)
  asm volatile("mov.u32 %0, 0;" : "=r"(z));
  // e52 (= kYExp52) arrives as a kernel parameter so that it sits in a
  // register: the hi-word builds are then single three-input ops
  switch (nr) {  // warp-uniform (depends on the row segment only)
    case 12: ypass_wta<12, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 11: ypass_wta<11, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 10: ypass_wta<10, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 9: ypass_wta<9, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 8: ypass_wta<8, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 7: ypass_wta<7, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 6: ypass_wta<6, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 5: ypass_wta<5, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 4: ypass_wta<4, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 3: ypass_wta<3, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 2: ypass_wta<2, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    case 1: ypass_wta<1, TWO>(best, oab, EloB, EhiB, z, e52, d); break;
    default: break;
  }
}

// Debug volume (STEREO_DEBUG_CA): the exact window sums of d (and d+1) of the
// thread's own rows, from the same prefix rows the WTA read.  A plain loop
// (debug builds of the kernel only).
__device__ __noinline__ void ypass_debug_store(const uint32_t* oab, int nr, const uint8_t* EloB,
                                               const uint8_t* EhiB, int d, bool two,
                                               uint64_t* cadbg, int Hs, int Ws, int yrow0,
                                               int x) {
  if (x >= Ws) return;
  for (int r = 0; r < nr; ++r) {
    const uint32_t ia = oab[r] & 0xffffu, ib = oab[r] >> 16;
    const uint2 la = *reinterpret_cast<const uint2*>(EloB + ia);
    const uint2 lb = *reinterpret_cast<const uint2*>(EloB + ib);
    const uint32_t dh = *reinterpret_cast<const uint32_t*>(EhiB + (ib >> 1)) -
                        *reinterpret_cast<const uint32_t*>(EhiB + (ia >> 1));
    const size_t o = ((size_t)d * Hs + yrow0 + 16 * r) * Ws + x;
    cadbg[o] = (uint64_t)(lb.x - la.x) + ((uint64_t)(dh & 0xffffu) << kYSplit);
    if (two) cadbg[o + (size_t)Hs * Ws] = (uint64_t)(lb.y - la.y) + ((uint64_t)(dh >> 16) << kYSplit);
  }
}

template <int SEG, bool DBG>
__global__ void __launch_bounds__(kYThreads, 2)
    ypass_kernel(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
                 YArgs a) {
  static_assert(SEG & 1, "SEG must be odd (bank-disjoint half-warps)");
  constexpr int TB = kYSegs * SEG;                 // tile rows = TMA box height
  constexpr uint32_t kTileBytes = 2 * TB * 16 * 4;  // box {16 columns, TB rows, 1 pair} of u64
  extern __shared__ __align__(128) uint8_t ysm[];  // TMA destinations need 128-B alignment
  uint32_t* tile = reinterpret_cast<uint32_t*>(ysm);                      // [kYStages][2][TB][16]
  uint2* Elo = reinterpret_cast<uint2*>(ysm + kYStages * kTileBytes);      // [TB+1][16]
  uint32_t* Ehi = reinterpret_cast<uint32_t*>(Elo + (TB + 1) * 16);       // [TB+1][16]
  uint4* tot = reinterpret_cast<uint4*>(Ehi + (TB + 1) * 16);             // [8][16]
  uint64_t* bar = reinterpret_cast<uint64_t*>(tot + 8 * 16);              // [kYStages]
  const int tid = threadIdx.x, w = tid >> 5;
  const int col = tid & 15, seg = tid >> 4, upper = (tid >> 4) & 1;
  const int base = blockIdx.z;
  const CUtensorMap* tm = base ? &tm1 : &tm0;
  const uint32_t* armp = base ? a.arm1 : a.arm0;
  uint8_t* dmap = base ? a.D1 : a.D0;
  uint64_t* cadbg = base ? a.ca1 : a.ca0;
  const int x0 = blockIdx.x * 16, x = x0 + col;
  const int y0 = a.y_begin + blockIdx.y * a.B, yt0 = y0 - a.w_y;
  const int Ds = a.Ds;
  // output rows of this thread: y0 + seg + 16 r, r < nr (interleaved, so the
  // rows past B are whole trailing iterations, mostly warp-uniform)
  const int nrow = min(a.B, a.y_end - y0);
  const int nr = max(0, (nrow - seg + 15) >> 4);  // same for both segments of a warp if B even
  // (B odd: the two half-warps may differ by one row; the warp then runs the
  // larger count and the extra row reads a harmless window, never stored)
  const int nrw = max(nr, __shfl_xor_sync(kFull, nr, 16));

  if (tid == 0) {
    for (int s = 0; s < kYStages; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the initialising thread may use the barriers at once: first tiles in
    // flight before the CTA barrier
    for (int s = 0; s < kYStages && 2 * s < Ds; ++s) {
      mbar_expect_tx(bar + s, kTileBytes);
      tma_load_3d(tile + s * 2 * TB * 16, tm, bar + s, x0, yt0, s);
    }
  }
  __syncthreads();
  if (tid < 16) {
    Elo[tid] = make_uint2(0u, 0u);
    Ehi[tid] = 0u;
  }

  // window byte offsets into Elo (Ehi: half of it), packed a | b << 16
  // (< 2^16: (TB+1)*16*8 <= 30848), and the running minimum keys
  uint32_t oab[kYRPT];
  double best[kYRPT];
#pragma unroll
  for (int r = 0; r < kYRPT; ++r) {
    const int y = y0 + seg + 16 * r;
    oab[r] = 0u;
    best[r] = __hiloint2double(0x7ff00000, 0);  // +inf
    if (r < nr && x < a.Ws) {
      const uint32_t arm = __ldg(armp + (size_t)y * a.Ws + x);
      const int M = (arm >> 16) & 255u, N = arm >> 24;
      oab[r] = (((uint32_t)(y - M - yt0) * 16u + col) * 8u) |
               ((((uint32_t)(y + N + 1 - yt0) * 16u + col) * 8u) << 16);
    }
  }
  const uint8_t* EloB = reinterpret_cast<const uint8_t*>(Elo);
  const uint8_t* EhiB = reinterpret_cast<const uint8_t*>(Ehi);
  uint2* Ew = Elo + (seg * SEG + 1) * 16 + col;
  uint32_t* Hw = Ehi + (seg * SEG + 1) * 16 + col;
  constexpr uint32_t kLoMask = (1u << kYSplit) - 1u;

#pragma unroll 1
  for (int d = 0; d < Ds; d += 2) {
    const int it = d >> 1, st = it & 1;
    mbar_wait(bar + st, (it >> 1) & 1);
    // tile rows hold (d, d+1) pairs per column: one 8-B load per element
    const uint2* t01 = reinterpret_cast<const uint2*>(tile + st * 2 * TB * 16) + seg * SEG * 16 + col;
    uint32_t l0[SEG], l1[SEG], lh[SEG];
    uint32_t a0 = 0, a1 = 0, ah = 0;
#pragma unroll
    for (int s = 0; s < SEG; ++s) {
      const uint2 v = t01[s * 16];
      const uint32_t v0 = v.x, v1 = v.y;
      a0 += v0 & kLoMask;
      a1 += v1 & kLoMask;
      ah += __byte_perm(v0, 0u, 0x4443u) + __byte_perm(v1, 0u, 0x4344u);  // v0.b3 | v1.b3 << 16
      l0[s] = a0; l1[s] = a1; lh[s] = ah;
    }
    // the warp's two segments: the upper half adds the lower half's totals
    const uint32_t b0 = __shfl_sync(kFull, a0, col), b1 = __shfl_sync(kFull, a1, col),
                   bh = __shfl_sync(kFull, ah, col);
    if (upper) tot[w * 16 + col] = make_uint4(b0 + a0, b1 + a1, bh + ah, 0u);
    __syncthreads();  // (1) tile[st] consumed, warp totals visible
    if (tid == 0 && d + 2 * kYStages < Ds) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar + st, kTileBytes);
      tma_load_3d(tile + st * 2 * TB * 16, tm, bar + st, x0, yt0, (d >> 1) + kYStages);
    }
    uint32_t o0 = upper ? b0 : 0u, o1 = upper ? b1 : 0u, oh = upper ? bh : 0u;
    // earlier warps' totals: unrolled, warp-uniform predicates, so that all
    // loads issue back to back (one shared-memory latency, not w of them)
#pragma unroll
    for (int q = 0; q < kYThreads / 32 - 1; ++q) {
      if (q < w) {
        const uint4 t = tot[q * 16 + col];
        o0 += t.x; o1 += t.y; oh += t.z;
      }
    }
#pragma unroll
    for (int s = 0; s < SEG; ++s) {
      Ew[s * 16] = make_uint2(l0[s] + o0, l1[s] + o1);
      Hw[s * 16] = lh[s] + oh;
    }
    __syncthreads();  // (2) column prefixes complete
    if (d + 1 < Ds)
      ypass_wta_n<true>(nrw, best, oab, EloB, EhiB, d, a.e52);
    else
      ypass_wta_n<false>(nrw, best, oab, EloB, EhiB, d, a.e52);
    if (DBG) ypass_debug_store(oab, nr, EloB, EhiB, d, d + 1 < Ds, cadbg, a.Hs, a.Ws, y0 + seg, x);
  }
#pragma unroll
  for (int r = 0; r < kYRPT; ++r)
    if (r < nr && x < a.Ws) dmap[(size_t)(y0 + seg + 16 * r) * a.Ws + x] = (uint8_t)(__double2loint(best[r]) & 255);
}

// ============================================================================
// FUSED (NEXT-1 prototype, STEREO_FUSED=1): cost + CA_x + CA + WTA in ONE
// kernel, CA_x never leaves the SM.  The y stage is v1's (same tile, split
// prefix, WTA); instead of a TMA load, the CTA computes its tile of CA_x
// itself for each disparity pair: warp w takes tile rows w, w+8, ...; per row
// the 64 cost columns [x0 - 24, x0 + 40) that the 16 output columns' x
// windows can reach (w_x, w_x_r <= 24) -- Eqs. 3-5 from the PREP code words
// and the bank-replicated fixed-point tables (BORDER outside the right /
// left image, R12b) -- a warp-scan exclusive prefix into per-warp shared
// scratch, then Eq. 7's window difference for the 16 columns (lanes 0-15:
// d, lanes 16-31: d+1).  The right base evaluates its own costs
// C^R(x', d) = C(x'+d, d) (Eq. 6): nothing is shared between the bases and
// each output needs (16 + 48) / 16 x TB / B cost evaluations (vs 0.5 staged).
// ============================================================================
struct FArgs {
  const uint32_t* xrow;  // [4][Hs][Wp]: code L, code R (census | I << 24)
  const uint32_t* qtab;  // the replicated tables (40 KB)
  uint32_t border;
  int Wp;
};
constexpr int kFHalo = 24;  // max x arm of the fused prototype

template <int SEG>
__global__ void __launch_bounds__(kYThreads, 1)
    fused_kernel(YArgs a, FArgs f) {
  constexpr int TB = kYSegs * SEG;
  extern __shared__ __align__(128) uint8_t ysm[];
  uint32_t* sQAD = reinterpret_cast<uint32_t*>(ysm);          // [256][32]
  uint32_t* sQMC = sQAD + 256 * 32;                           // [64][32]
  uint32_t* tile = sQMC + 64 * 32;                            // [TB][16] x u64 (d, d+1)
  uint2* Elo = reinterpret_cast<uint2*>(tile + 2 * TB * 16);   // [TB+1][16]
  uint32_t* Ehi = reinterpret_cast<uint32_t*>(Elo + (TB + 1) * 16);
  uint4* tot = reinterpret_cast<uint4*>(Ehi + (TB + 1) * 16); // [8][16]
  uint32_t* scr = reinterpret_cast<uint32_t*>(tot + 8 * 16);  // [8 warps][2][65] row prefixes
  uint64_t* bar = reinterpret_cast<uint64_t*>(scr + 8 * 2 * 72);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int col = tid & 15, seg = tid >> 4, upper = (tid >> 4) & 1;
  const int base = blockIdx.z;
  const uint32_t* armp = base ? a.arm1 : a.arm0;
  uint8_t* dmap = base ? a.D1 : a.D0;
  const int x0 = blockIdx.x * 16, x = x0 + col;
  const int y0 = a.y_begin + blockIdx.y * a.B, yt0 = y0 - a.w_y;
  const int Ds = a.Ds, Ws = a.Ws, Hs = a.Hs;
  const size_t plane = (size_t)Hs * f.Wp;
  const uint32_t* codeL = f.xrow;
  const uint32_t* codeR = f.xrow + plane;

  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    constexpr uint32_t kTabBytes = (256 + 64) * 32 * 4;
    mbar_expect_tx(bar, kTabBytes);
    bulk_g2s(sQAD, f.qtab, kTabBytes, bar);
  }
  __syncthreads();
  if (tid < 16) {
    Elo[tid] = make_uint2(0u, 0u);
    Ehi[tid] = 0u;
  }
  const int nrow = min(a.B, a.y_end - y0);
  const int nr = max(0, (nrow - seg + 15) >> 4);
  const int nrw = max(nr, __shfl_xor_sync(kFull, nr, 16));
  uint32_t oab[kYRPT];
  double best[kYRPT];
#pragma unroll
  for (int r = 0; r < kYRPT; ++r) {
    const int y = y0 + seg + 16 * r;
    oab[r] = 0u;
    best[r] = __hiloint2double(0x7ff00000, 0);
    if (r < nr && x < Ws) {
      const uint32_t arm = __ldg(armp + (size_t)y * Ws + x);
      const int M = (arm >> 16) & 255u, N = arm >> 24;
      oab[r] = (((uint32_t)(y - M - yt0) * 16u + col) * 8u) |
               ((((uint32_t)(y + N + 1 - yt0) * 16u + col) * 8u) << 16);
    }
  }
  mbar_wait(bar, 0u);
  const char* qadb = reinterpret_cast<const char*>(sQAD + lane);
  const char* qmcb = reinterpret_cast<const char*>(sQMC + lane);
  const uint2* t01 = reinterpret_cast<const uint2*>(tile) + seg * SEG * 16 + col;
  uint2* Ew = Elo + (seg * SEG + 1) * 16 + col;
  uint32_t* Hw = Ehi + (seg * SEG + 1) * 16 + col;
  uint32_t* sp = scr + w * 2 * 72;  // this warp's two prefix rows (d, d+1), 65 entries each
  constexpr uint32_t kLoMask = (1u << kYSplit) - 1u;
  const int cb = x0 - kFHalo;          // first cost column of the row window
  const int c0 = cb + 2 * lane;        // this lane's two cost columns c0, c0 + 1

#pragma unroll 1
  for (int d = 0; d < Ds; d += 2) {
    // ---- x stage: this pair's CA_x tile, rows yt0 .. yt0 + TB - 1
    for (int r = w; r < TB; r += 8) {
      const int yy = yt0 + r;
      uint2* trow = reinterpret_cast<uint2*>(tile) + r * 16;
      if (yy < 0 || yy >= Hs) {  // outside the image: zero rows (never inside a window)
        if (lane < 16) trow[lane] = make_uint2(0u, 0u);
        continue;
      }
      const uint32_t* cl = codeL + (size_t)yy * f.Wp;
      const uint32_t* cr = codeR + (size_t)yy * f.Wp;
      uint32_t cost[2][2];  // [column][disparity]
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int c = c0 + k;
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const int dd = d + n;
          // left base: C(c, dd) = Q[L(c), R(c - dd)]; right base: C(c + dd, dd) = Q[L(c + dd), R(c)]
          const int xl = base ? c + dd : c, xr = base ? c : c - dd;
          const bool out = base ? (xl >= Ws) : (xr < 0);  // BORDER (R12b)
          const uint32_t pl = __ldg(cl + clampi(xl, 0, Ws - 1));
          const uint32_t pr = __ldg(cr + clampi(xr, 0, Ws - 1));
          const uint32_t qa = *reinterpret_cast<const uint32_t*>(qadb + (__vabsdiffu4(pl, pr) >> 17));
          const uint32_t qm = *reinterpret_cast<const uint32_t*>(qmcb + (((pl ^ pr) & 63u) << 7));
          cost[k][n] = out ? f.border : qa + qm;
        }
      }
      // exclusive prefix over the 64 columns (two per lane), both disparities
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        const uint32_t loc = cost[0][n] + cost[1][n];
        uint32_t inc = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += t;
        }
        const uint32_t ex = inc - loc;
        sp[n * 72 + 2 * lane] = ex;
        sp[n * 72 + 2 * lane + 1] = ex + cost[0][n];
        if (lane == 31) sp[n * 72 + 64] = inc;
      }
      __syncwarp();
      // Eq. 7: lanes 0-15 the window of column x0 + lane at d, lanes 16-31 at d + 1
      {
        const int j = lane & 15, n = lane >> 4, xx = x0 + j;
        uint32_t v = 0u;
        if (xx < Ws && d + n < Ds) {
          const uint32_t arm = __ldg((base ? a.arm1 : a.arm0) + (size_t)yy * Ws + xx);
          const int m = arm & 255u, nn = (arm >> 8) & 255u;
          v = sp[n * 72 + j + kFHalo + nn + 1] - sp[n * 72 + j + kFHalo - m];
        }
        reinterpret_cast<uint32_t*>(trow + j)[n] = v;
      }
      __syncwarp();
    }
    __syncthreads();  // (0) tile complete
    // ---- y stage (v1): column prefix in split precision, then the WTA
    uint32_t l0[SEG], l1[SEG], lh[SEG];
    uint32_t a0 = 0, a1 = 0, ah = 0;
#pragma unroll
    for (int s = 0; s < SEG; ++s) {
      const uint2 v = t01[s * 16];
      a0 += v.x & kLoMask;
      a1 += v.y & kLoMask;
      ah += __byte_perm(v.x, 0u, 0x4443u) + __byte_perm(v.y, 0u, 0x4344u);
      l0[s] = a0; l1[s] = a1; lh[s] = ah;
    }
    const uint32_t b0 = __shfl_sync(kFull, a0, col), b1 = __shfl_sync(kFull, a1, col),
                   bh = __shfl_sync(kFull, ah, col);
    if (upper) tot[w * 16 + col] = make_uint4(b0 + a0, b1 + a1, bh + ah, 0u);
    __syncthreads();  // (1) tile consumed, warp totals visible
    uint32_t o0 = upper ? b0 : 0u, o1 = upper ? b1 : 0u, oh = upper ? bh : 0u;
#pragma unroll
    for (int q = 0; q < kYThreads / 32 - 1; ++q) {
      if (q < w) {
        const uint4 t = tot[q * 16 + col];
        o0 += t.x; o1 += t.y; oh += t.z;
      }
    }
#pragma unroll
    for (int s = 0; s < SEG; ++s) {
      Ew[s * 16] = make_uint2(l0[s] + o0, l1[s] + o1);
      Hw[s * 16] = lh[s] + oh;
    }
    __syncthreads();  // (2) column prefixes complete
    const uint8_t* EloB = reinterpret_cast<const uint8_t*>(Elo);
    const uint8_t* EhiB = reinterpret_cast<const uint8_t*>(Ehi);
    if (d + 1 < Ds)
      ypass_wta_n<true>(nrw, best, oab, EloB, EhiB, d, a.e52);
    else
      ypass_wta_n<false>(nrw, best, oab, EloB, EhiB, d, a.e52);
    // (the next pair's E stores follow its barrier (0), which every warp
    // reaches only after this WTA)
  }
#pragma unroll
  for (int r = 0; r < kYRPT; ++r)
    if (r < nr && x < Ws) dmap[(size_t)(y0 + seg + 16 * r) * Ws + x] = (uint8_t)(__double2loint(best[r]) & 255);
}

static int fused_smem_bytes(int SEG) {
  const int TB = kYSegs * SEG;
  return (256 + 64) * 32 * 4 + 2 * TB * 16 * 4 + (TB + 1) * 16 * 12 + 8 * 16 * 16 + 8 * 2 * 72 * 4 + 16;
}


// Wide-strip variant (v2): CTA = 32-column strip x B output rows, 16 warps,
// warp w = tile row segment w (SEG rows) across all 32 columns.  Every warp
// access of the prefix arrays then lies in ONE tile row (32 consecutive
// columns): the hi prefixes (4 B per column) are one conflict-free wavefront
// per access instead of the two half-warps' rows meeting in the same bank half
// (v1: ~20% of the y pass's wavefronts were such conflicts).  Same arithmetic,
// same layouts, same WTA as v1; the segment offsets come from the earlier
// warps' column totals (independent loads, issued back to back).
constexpr int kY2Threads = 512;
constexpr int kY2Cols = 32;

template <int SEG, bool DBG>
__global__ void __launch_bounds__(kY2Threads, 1)
    ypass2_kernel(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
                  YArgs a) {
  constexpr int TB = kYSegs * SEG;                        // tile rows = TMA box height
  constexpr uint32_t kTileBytes = 2 * TB * kY2Cols * 4;   // box {32 columns, TB rows, 1 pair} of u64
  extern __shared__ __align__(128) uint8_t ysm[];
  uint32_t* tile = reinterpret_cast<uint32_t*>(ysm);                          // [kYStages][TB][32] x u64
  uint2* Elo = reinterpret_cast<uint2*>(ysm + kYStages * kTileBytes);          // [TB+1][32]
  uint32_t* Ehi = reinterpret_cast<uint32_t*>(Elo + (TB + 1) * kY2Cols);      // [TB+1][32]
  uint4* tot = reinterpret_cast<uint4*>(Ehi + (TB + 1) * kY2Cols);            // [16][32]
  uint64_t* bar = reinterpret_cast<uint64_t*>(tot + kYSegs * kY2Cols);        // [kYStages]
  const int tid = threadIdx.x, col = tid & 31, seg = tid >> 5;
  const int base = blockIdx.z;
  const CUtensorMap* tm = base ? &tm1 : &tm0;
  const uint32_t* armp = base ? a.arm1 : a.arm0;
  uint8_t* dmap = base ? a.D1 : a.D0;
  uint64_t* cadbg = base ? a.ca1 : a.ca0;
  const int x0 = blockIdx.x * kY2Cols, x = x0 + col;
  const int y0 = a.y_begin + blockIdx.y * a.B, yt0 = y0 - a.w_y;
  const int Ds = a.Ds;
  // output rows of this thread: y0 + seg + 16 r, r < nr (warp-uniform)
  const int nrow = min(a.B, a.y_end - y0);
  const int nr = max(0, (nrow - seg + 15) >> 4);

  if (tid == 0) {
    for (int s = 0; s < kYStages; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kYStages && 2 * s < Ds; ++s) {
      mbar_expect_tx(bar + s, kTileBytes);
      tma_load_3d(tile + s * 2 * TB * kY2Cols, tm, bar + s, x0, yt0, s);
    }
  }
  __syncthreads();
  if (tid < kY2Cols) {
    Elo[tid] = make_uint2(0u, 0u);
    Ehi[tid] = 0u;
  }
  // window byte offsets into Elo (Ehi: half of it), packed a | b << 16
  // (< 2^16: (TB+1)*32*8 <= 61696), and the running minimum keys
  uint32_t oab[kYRPT];
  double best[kYRPT];
#pragma unroll
  for (int r = 0; r < kYRPT; ++r) {
    const int y = y0 + seg + 16 * r;
    oab[r] = 0u;
    best[r] = __hiloint2double(0x7ff00000, 0);  // +inf
    if (r < nr && x < a.Ws) {
      const uint32_t arm = __ldg(armp + (size_t)y * a.Ws + x);
      const int M = (arm >> 16) & 255u, N = arm >> 24;
      oab[r] = (((uint32_t)(y - M - yt0) * kY2Cols + col) * 8u) |
               ((((uint32_t)(y + N + 1 - yt0) * kY2Cols + col) * 8u) << 16);
    }
  }
  const uint8_t* EloB = reinterpret_cast<const uint8_t*>(Elo);
  const uint8_t* EhiB = reinterpret_cast<const uint8_t*>(Ehi);
  uint2* Ew = Elo + (seg * SEG + 1) * kY2Cols + col;
  uint32_t* Hw = Ehi + (seg * SEG + 1) * kY2Cols + col;
  constexpr uint32_t kLoMask = (1u << kYSplit) - 1u;

#pragma unroll 1
  for (int d = 0; d < Ds; d += 2) {
    const int it = d >> 1, st = it & 1;
    mbar_wait(bar + st, (it >> 1) & 1);
    const uint2* t01 = reinterpret_cast<const uint2*>(tile + st * 2 * TB * kY2Cols) + seg * SEG * kY2Cols + col;
    uint32_t l0[SEG], l1[SEG], lh[SEG];
    uint32_t a0 = 0, a1 = 0, ah = 0;
#pragma unroll
    for (int s = 0; s < SEG; ++s) {
      const uint2 v = t01[s * kY2Cols];
      a0 += v.x & kLoMask;
      a1 += v.y & kLoMask;
      ah += __byte_perm(v.x, 0u, 0x4443u) + __byte_perm(v.y, 0u, 0x4344u);  // v.x.b3 | v.y.b3 << 16
      l0[s] = a0; l1[s] = a1; lh[s] = ah;
    }
    tot[seg * kY2Cols + col] = make_uint4(a0, a1, ah, 0u);
    __syncthreads();  // (1) tile[st] consumed, segment totals visible
    if (tid == 0 && d + 2 * kYStages < Ds) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar + st, kTileBytes);
      tma_load_3d(tile + st * 2 * TB * kY2Cols, tm, bar + st, x0, yt0, (d >> 1) + kYStages);
    }
    uint32_t o0 = 0u, o1 = 0u, oh = 0u;
#pragma unroll
    for (int q = 0; q < kYSegs - 1; ++q) {
      if (q < seg) {  // warp-uniform
        const uint4 t = tot[q * kY2Cols + col];
        o0 += t.x; o1 += t.y; oh += t.z;
      }
    }
#pragma unroll
    for (int s = 0; s < SEG; ++s) {
      Ew[s * kY2Cols] = make_uint2(l0[s] + o0, l1[s] + o1);
      Hw[s * kY2Cols] = lh[s] + oh;
    }
    __syncthreads();  // (2) column prefixes complete
    if (d + 1 < Ds)
      ypass_wta_n<true>(nr, best, oab, EloB, EhiB, d, a.e52);
    else
      ypass_wta_n<false>(nr, best, oab, EloB, EhiB, d, a.e52);
    if (DBG) ypass_debug_store(oab, nr, EloB, EhiB, d, d + 1 < Ds, cadbg, a.Hs, a.Ws, y0 + seg, x);
  }
#pragma unroll
  for (int r = 0; r < kYRPT; ++r)
    if (r < nr && x < a.Ws) dmap[(size_t)(y0 + seg + 16 * r) * a.Ws + x] = (uint8_t)(__double2loint(best[r]) & 255);
}

static int ypass2_smem_bytes(int SEG) {
  const int TB = kYSegs * SEG;
  return kYStages * 2 * TB * kY2Cols * 4 + (TB + 1) * kY2Cols * 12 + kYSegs * kY2Cols * 16 + kYStages * 8;
}

#define YPASS2_DISPATCH(S_, EXPR)                      \
  switch (S_) {                                        \
    case 4: { constexpr int SS = 4; EXPR; } break;     \
    case 5: { constexpr int SS = 5; EXPR; } break;     \
    case 6: { constexpr int SS = 6; EXPR; } break;     \
    case 7: { constexpr int SS = 7; EXPR; } break;     \
    case 8: { constexpr int SS = 8; EXPR; } break;     \
    case 9: { constexpr int SS = 9; EXPR; } break;     \
    case 10: { constexpr int SS = 10; EXPR; } break;   \
    case 11: { constexpr int SS = 11; EXPR; } break;   \
    case 12: { constexpr int SS = 12; EXPR; } break;   \
    case 13: { constexpr int SS = 13; EXPR; } break;   \
    case 14: { constexpr int SS = 14; EXPR; } break;   \
    case 15: { constexpr int SS = 15; EXPR; } break;   \
    default: break;                                    \
  }

#define YPASS_DISPATCH(S_, EXPR)                       \
  switch (S_) {                                        \
    case 5: { constexpr int SS = 5; EXPR; } break;     \
    case 7: { constexpr int SS = 7; EXPR; } break;     \
    case 9: { constexpr int SS = 9; EXPR; } break;     \
    case 11: { constexpr int SS = 11; EXPR; } break;   \
    case 13: { constexpr int SS = 13; EXPR; } break;   \
    case 15: { constexpr int SS = 15; EXPR; } break;   \
    default: break;                                    \
  }

cudaError_t launch_fused(const Geom& g, const Plan& p, Buffers& b, cudaStream_t s) {
  YArgs a;
  a.arm0 = b.armL; a.arm1 = b.armR;
  a.D0 = b.DL; a.D1 = b.DR;
  a.ca0 = a.ca1 = nullptr;
  a.Ws = g.Ws; a.Hs = g.Hs; a.Ds = g.Ds; a.w_y = g.w_y; a.B = p.ypass_B;
  a.y_begin = 0;
  a.y_end = g.Hs;
  a.e52 = kYExp52;
  FArgs f{b.xrow, b.qtab, g.border, g.Wp};
  dim3 grid((g.Ws + 15) / 16, (g.Hs + p.ypass_B - 1) / p.ypass_B, 2);
  cudaError_t e = cudaErrorInvalidValue;
  YPASS_DISPATCH(p.ypass_SEG, (fused_kernel<SS><<<grid, kYThreads, p.fused_smem, s>>>(a, f),
                               e = cudaGetLastError()))
  return e;
}

static int ypass_seg_for(int T, int ver) {
  const int need = (T + kYSegs - 1) / kYSegs;
  if (ver == 2) return need <= 15 ? std::max(need, 4) : 0;
  for (int s : {5, 7, 9, 11, 13, 15})
    if (s >= need) return s;
  return 0;
}

static int ypass_smem_bytes(int SEG) {
  const int TB = kYSegs * SEG;
  return kYStages * 2 * TB * 16 * 4 + (TB + 1) * 16 * 12 + 8 * 16 * 16 + kYStages * 8;
}



static cudaError_t launch_ypass_range(const Geom& g, const Plan& p, Buffers& b, bool store_ca,
                                      int y_begin, int y_end, cudaStream_t s);

cudaError_t launch_ypass(const Geom& g, const Plan& p, Buffers& b, bool store_ca, int nfr,
                         cudaStream_t s) {
  // whole frames (the batch as one image of nfr*Hs rows), or in band mode
  // only the rows whose D^L / D^R the band's POST reads
  return launch_ypass_range(g, p, b, store_ca, g.band ? g.ya : 0, g.band ? g.yb : nfr * g.Hs, s);
}

cudaError_t launch_ypass_rows(const Geom& g, const Plan& p, Buffers& b, int y0, int y1,
                              cudaStream_t s) {
  return launch_ypass_range(g, p, b, false, y0, y1, s);
}

static cudaError_t launch_ypass_range(const Geom& g, const Plan& p, Buffers& b, bool store_ca,
                                      int y_begin, int y_end, cudaStream_t s) {
  YArgs a;
  a.arm0 = b.armL; a.arm1 = b.armR;
  a.D0 = b.DL; a.D1 = b.DR;
  a.ca0 = store_ca ? b.caL : nullptr;
  a.ca1 = store_ca ? b.caR : nullptr;
  a.Ws = g.Ws; a.Hs = g.Hs; a.Ds = g.Ds; a.w_y = g.w_y; a.B = p.ypass_B;
  a.y_begin = y_begin;
  a.y_end = y_end;
  a.e52 = kYExp52;
  const int cols = p.ypass_ver == 2 ? kY2Cols : 16;
  dim3 grid((g.Ws + cols - 1) / cols, (a.y_end - a.y_begin + p.ypass_B - 1) / p.ypass_B, 2);
  cudaError_t e = cudaErrorInvalidValue;
  if (p.ypass_ver == 2) {
    if (store_ca)
      YPASS2_DISPATCH(p.ypass_SEG,
                      (ypass2_kernel<SS, true><<<grid, kY2Threads, p.ypass_smem, s>>>(p.tmL, p.tmR, a),
                       e = cudaGetLastError()))
    else
      YPASS2_DISPATCH(p.ypass_SEG,
                      (ypass2_kernel<SS, false><<<grid, kY2Threads, p.ypass_smem, s>>>(p.tmL, p.tmR, a),
                       e = cudaGetLastError()))
    return e;
  }
  if (store_ca)
    YPASS_DISPATCH(p.ypass_SEG,
                   (ypass_kernel<SS, true><<<grid, kYThreads, p.ypass_smem, s>>>(p.tmL, p.tmR, a),
                    e = cudaGetLastError()))
  else
    YPASS_DISPATCH(p.ypass_SEG,
                   (ypass_kernel<SS, false><<<grid, kYThreads, p.ypass_smem, s>>>(p.tmL, p.tmR, a),
                    e = cudaGetLastError()))
  return e;
}

// ============================================================================
// POST — one CTA per scaled row y:
//  * cross-check (Eq. 10; Step6 P:504-511; reading E5: the partner
//    is D^R[y][x-k]) for the masked rows y-1 .. y+2 (clamped);
//  * 3x3 median of the valid values (Step7 first half; R21-R23)
//    for rows y and y+1, a 25-comparator sorting network in registers with
//    INVALID = 255 sorting last, output sorted[(n_valid-1)/2];
//  * bilateral fill (§III.E steps 1-3; Step7 P:516-525) of rows y
//    and y+1: nearest valid neighbours from per-32-pixel ballot masks and a
//    warp scan over the chunk summaries, then (a) (Dl*j + Dr*i)/(i+j) as one
//    IEEE binary32 division (R26, sign reading E6), (b) brightness-closer
//    side (tie -> left, R24), (c) one-sided copy;
//  * scale-up (Step8; R27-R30) of output rows 2y, 2y+1 (K = 2), or
//    the fill row itself as the output (K = 1).
// Rows without any valid pixel (rule (d)) are patched by the last CTA to
// finish (grid-wide counter), which sees every row's first/last valid column.
// ============================================================================
// POST row pitch in shared memory: room for the clamp byte at Ws and the
// word over-reads of the SIMD median, a multiple of 32 (ballot chunks)
static int post_pitch(int Ws) { return (Ws + 8 + 31) & ~31; }

struct PostArgs {
  const uint8_t* DL;
  const uint8_t* DR;
  const uint16_t* pixL;
  const uint8_t* Lorg;
  uint8_t* masked;
  uint8_t* median;
  float* fill;
  float* out;
  int32_t* rowFirst;  // [4][Hs] of this frame: first x, last x, first value, last value
  int32_t* rowLast;   // = rowFirst + Hs
  unsigned* counter;
  int W, H, Ws, Hs, K, T;
  int fill_mode;  // STEREO_FILL_*
  int Wsp;  // smem row pitch, post_pitch(Ws)
  int Wx;   // W rounded up to 4
  int y_lo, y_hi;  // scaled rows owned by this launch (band mode: the band's own rows)
  int out_row0;    // original row held by out[0] (band mode: the first own row)
  int rule_d;      // resolve fill rule (d) in-kernel (whole frames; band mode: stereo_band_finish)
};

// the frame `fr` of a batch launch: every per-frame buffer offset by its slot
__device__ __forceinline__ PostArgs post_frame(PostArgs a, int fr) {
  const size_t n = (size_t)a.Ws * a.Hs, N = (size_t)a.W * a.H;
  a.DL += fr * n; a.DR += fr * n; a.pixL += fr * n;
  a.masked += fr * n; a.median += fr * n; a.fill += fr * n;
  a.Lorg += fr * N; a.out += fr * N;
  a.rowFirst += (size_t)fr * 4 * a.Hs;
  a.rowLast = a.rowFirst + a.Hs;
  a.counter += fr;
  return a;
}

// u16x2 helpers of the SIMD median (lanes hold values 0..255, INVALID = 255)
__device__ __forceinline__ void cswap16(uint32_t& a, uint32_t& b) {
  const uint32_t lo = __vminu2(a, b), hi = __vmaxu2(a, b);
  a = lo;
  b = hi;
}
// 0xffff in the lanes of w equal to 255 (bit 15 of w + 0x7f01, replicated)
// (prmt sign-replicate mode via PTX: __byte_perm keeps only 3 selector bits)
__device__ __forceinline__ uint32_t inv16(uint32_t w) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0xbb99;" : "=r"(r) : "r"(w + 0x7f017f01u));
  return r;
}
// per lane: key valid (< 255) ? val : cur
__device__ __forceinline__ uint32_t sel16_valid(uint32_t key, uint32_t val, uint32_t cur) {
  const uint32_t m = inv16(key);
  return (cur & m) | (val & ~m);
}
// bytes 2h, 2h+1 of w as u16x2 lanes
__device__ __forceinline__ uint32_t u16x2_of(uint32_t w, int h) {
  return h ? __byte_perm(w, 0, 0x4342) : __byte_perm(w, 0, 0x4140);
}

// Step8 x rule on seeded row `f` (fill values) with original-resolution row `L`
__device__ __forceinline__ float su_xval(const float* f, const uint8_t* __restrict__ L, int X,
                                         int W, int Ws, float thr) {
  if ((X & 1) == 0) {
    if ((X >> 1) < Ws) return 2.0f * f[X >> 1];
    X -= 1;  // extra last column of an odd width copies its predecessor
  }
  const float av = 2.0f * f[(X - 1) >> 1];
  if (X + 1 < W && ((X + 1) >> 1) < Ws) {
    const float bv = 2.0f * f[(X + 1) >> 1];
    if (fabsf(__fsub_rn(av, bv)) <= thr) return __fmul_rn(__fadd_rn(av, bv), 0.5f);
    const int c = __ldg(L + X);
    return (abs((int)__ldg(L + X - 1) - c) <= abs((int)__ldg(L + X + 1) - c)) ? av : bv;
  }
  return av;
}

// fill value of pixel x given its nearest valid neighbours li / ri (§III.E):
// mode 0 the bilateral estimation, 1 / 2 the Fig. 6 baselines (nearest /
// smaller disparity), 3 Eq. 11 as printed -- every rational
// result rounded once (__fdiv_rn of exact integers, |numerator| < 2^24)
__device__ __forceinline__ float fill_value(const uint8_t* md, const uint16_t* pix,
                                            int x, int li, int ri, int T, int mode) {
  if (li >= 0 && ri >= 0) {
    const int Dl = md[li], Dr = md[ri];
    const int i = x - li, j = ri - x;
    if (mode == 1) return (float)(i <= j ? Dl : Dr);  // equal distances -> left
    if (mode == 2) return (float)min(Dl, Dr);
    if (abs(Dl - Dr) <= T)
      return mode == 3 ? __fdiv_rn((float)(Dl * (i + j) + i * (Dl - Dr)), (float)(i + j))
                       : __fdiv_rn((float)(Dl * j + Dr * i), (float)(i + j));
    const int cI = pix[x] & 255, lI = pix[li] & 255, rI = pix[ri] & 255;
    return (abs(lI - cI) <= abs(rI - cI)) ? (float)Dl : (float)Dr;
  }
  if (li >= 0) return (float)md[li];
  if (ri >= 0) return (float)md[ri];
  return 0.0f;  // no valid pixel in the row: patched by rule (d)
}

// rule (d) value for an all-invalid row r (reads other rows: global memory)
__device__ float rule_d_value(const PostArgs& a, int r) {
  for (int yy = r - 1; yy >= 0; --yy) {
    const int l = __ldcg(a.rowLast + yy);
    if (l >= 0) return (float)__ldcg(a.median + (size_t)yy * a.Ws + l);
  }
  for (int yy = r + 1; yy < a.Hs; ++yy) {
    const int f = __ldcg(a.rowFirst + yy);
    if (f >= 0) return (float)__ldcg(a.median + (size_t)yy * a.Ws + f);
  }
  return 0.0f;
}

// scale-up of output row Y from the (global) fill buffer — used by the rule-(d) patch
__device__ void su_row_global(const PostArgs& a, int Y, float thr) {
  const int Hs = a.Hs;
  int ya, yb = -1;
  if ((Y & 1) == 0 && (Y >> 1) < Hs) {
    ya = Y >> 1;
  } else if ((Y & 1) == 1 && Y + 1 < a.H && ((Y + 1) >> 1) < Hs) {
    ya = (Y - 1) >> 1;
    yb = (Y + 1) >> 1;
  } else {
    ya = min((Y - 1) >> 1, Hs - 1);
  }
  for (int X = threadIdx.x; X < a.W; X += blockDim.x) {
    float v = su_xval(a.fill + (size_t)ya * a.Ws, a.Lorg + (size_t)(2 * ya) * a.W, X, a.W, a.Ws, thr);
    if (yb >= 0)
      v = __fmul_rn(__fadd_rn(v, su_xval(a.fill + (size_t)yb * a.Ws,
                                         a.Lorg + (size_t)(2 * yb) * a.W, X, a.W, a.Ws, thr)),
                    0.5f);
    a.out[(size_t)(Y - a.out_row0) * a.W + X] = v;
  }
}

// n bytes from global src (any alignment) to 4-byte aligned shared dst with
// one aligned word load (+ its successor, when misaligned) and one word store
// per 4 bytes; reads up to 7 bytes past src + n when src is misaligned
__device__ __forceinline__ void stage_row(uint8_t* dst, const uint8_t* src, int n, int tid,
                                          int nthreads) {
  const uintptr_t ad = reinterpret_cast<uintptr_t>(src);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(ad & ~(uintptr_t)3);
  const int sh = 8 * (int)(ad & 3);
  uint32_t* d = reinterpret_cast<uint32_t*>(dst);
  const int nw = (n + 3) >> 2;
  if (sh == 0) {
    for (int t = tid; t < nw; t += nthreads) d[t] = __ldg(w + t);
  } else {
    for (int t = tid; t < nw; t += nthreads) d[t] = __funnelshift_r(__ldg(w + t), __ldg(w + t + 1), sh);
  }
}

template <int R>  // scaled rows owned per CTA
__global__ void __launch_bounds__(512) post_kernel(PostArgs a0) {
  const PostArgs a = post_frame(a0, blockIdx.z);
  extern __shared__ uint32_t psm_[];
  const int Ws = a.Ws, Wsp = a.Wsp, nch = Wsp >> 5, W = a.W, Wx = a.Wx;
  uint8_t* mk = reinterpret_cast<uint8_t*>(psm_);                  // [R+3][Wsp] masked rows
  uint8_t* md = mk + (R + 3) * Wsp;                                // [R+1][Wsp] median rows
  float* fv = reinterpret_cast<float*>(md + (R + 1) * Wsp);        // [R+1][Wsp] fill rows
  float* xr = fv + (R + 1) * Wsp;                                  // [R+1][Wx]  x-filled rows (K=2)
  uint32_t* cmask = reinterpret_cast<uint32_t*>(xr + (R + 1) * Wx); // [R+1][64]
  int* prevLast = reinterpret_cast<int*>(cmask + (R + 1) * 64);    // [R+1][64]
  int* nextFirst = prevLast + (R + 1) * 64;                        // [R+1][64]
  uint16_t* sPix = reinterpret_cast<uint16_t*>(nextFirst + (R + 1) * 64);  // [R+1][Wsp]
  uint8_t* sDL = reinterpret_cast<uint8_t*>(sPix + (R + 1) * Wsp);         // [R+3][Wsp]
  uint8_t* sDR = sDL + (R + 3) * Wsp;                                      // [R+3][Wsp]
  uint8_t* sLo = sDR + (R + 3) * Wsp;                                      // [R+1][Wx] L_org rows
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int y0 = a.y_lo + blockIdx.x * R;
  const int nr = min(R, a.y_hi - y0);                        // owned scaled rows
  const int nf = a.K == 2 ? min(nr + 1, a.Hs - y0) : nr;     // fill rows needed (SU reads y+1)
  const float thr = (float)(a.K * a.T);

  // 0. stage every input row in shared memory, one warp per row (rows are
  // re-aligned with a funnel shift; the handle's own buffers carry 16 bytes
  // of tail padding for the over-read): D^L, D^R rows y0-1 .. y0+nf (clamped),
  // pix rows y0 .. y0+nf-1, L_org rows 2(y0+j) (K = 2)
  {
    const int nwarp = blockDim.x >> 5;
    const int nmap = nf + 2, nrows = 2 * nmap + nf + (a.K == 2 ? nf : 0);
    for (int q = warp; q < nrows; q += nwarp) {
      if (q < 2 * nmap) {
        const int r = q < nmap ? q : q - nmap;
        const size_t o = (size_t)clampi(y0 - 1 + r, 0, a.Hs - 1) * Ws;
        stage_row(q < nmap ? sDL + r * Wsp : sDR + r * Wsp, (q < nmap ? a.DL : a.DR) + o, Ws, lane, 32);
      } else if (q < 2 * nmap + nf) {
        const int j = q - 2 * nmap;
        stage_row(reinterpret_cast<uint8_t*>(sPix + j * Wsp),
                  reinterpret_cast<const uint8_t*>(a.pixL + (size_t)(y0 + j) * Ws), 2 * Ws, lane, 32);
      } else {
        const int j = q - 2 * nmap - nf;
        const uint8_t* src = a.Lorg + (size_t)(2 * (y0 + j)) * W;
        if (((reinterpret_cast<uintptr_t>(src) | (uintptr_t)W) & 3) == 0)  // caller buffer:
          stage_row(sLo + j * Wx, src, W, lane, 32);                       // no over-read
        else
          for (int X = lane; X < W; X += 32) sLo[j * Wx + X] = __ldg(src + X);
      }
    }
  }
  __syncthreads();
  // 1. masked rows y0-1 .. y0+nf (clamped), Eq. 10; four pixels per thread.
  // Byte Ws of every row repeats byte Ws-1 (the clamped right neighbour of
  // the median below).
  const int nq = (Ws + 3) >> 2;
  for (int r = 0; r < nf + 2; ++r)
    for (int q = tid; q < nq; q += blockDim.x) {
      const int x = 4 * q;
      const uint32_t k4 = *reinterpret_cast<const uint32_t*>(sDL + r * Wsp + x);
      const uint8_t* dr = sDR + r * Wsp;
      uint32_t m4 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = (k4 >> (8 * i)) & 255;
        const bool gcp = (x + i - k >= 0) && (dr[max(x + i - k, 0)] == k);
        m4 |= (uint32_t)(gcp ? k : kInvalid) << (8 * i);
      }
      *reinterpret_cast<uint32_t*>(mk + r * Wsp + x) = m4;
      if (x + 4 >= Ws) mk[r * Wsp + Ws] = mk[r * Wsp + Ws - 1];  // (this thread wrote Ws-1)
    }
  __syncthreads();
  // 2. median rows y0 .. y0+nf-1: the 25-comparator 9-sorting network on two
  // pixels at a time (u16x2 lanes, native VIMNMX.U16x2), four pixels per
  // thread.  INVALID (255) sorts last, so with n valid neighbours the median
  // sorted[(n-1)/2] is s0, then s1 if s2 is valid, s2 if s4 is, s3 if s6 is,
  // s4 if s8 is (R21-R23); an INVALID centre stays INVALID.
  for (int j = 0; j < nf; ++j) {
    for (int q = tid; q < nq; q += blockDim.x) {
      const int x = 4 * q;
      uint32_t v[2][9];
      uint32_t cword = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(mk + (j + k) * Wsp + x);
        const uint32_t wb = w[0], wc = w[1];
        // bytes x-1 .. x+2 (x-1 clamped to x at the left border) and x+1 .. x+4
        const uint32_t W0 = x ? __funnelshift_r(w[-1], wb, 24) : __byte_perm(wb, 0, 0x2100);
        const uint32_t W1 = __funnelshift_r(wb, wc, 8);
        v[0][3 * k + 0] = __byte_perm(W0, 0, 0x4140);  // (x-1, x)
        v[0][3 * k + 1] = __byte_perm(W0, 0, 0x4241);  // (x, x+1)
        v[0][3 * k + 2] = __byte_perm(W0, 0, 0x4342);  // (x+1, x+2)
        v[1][3 * k + 0] = __byte_perm(W1, 0, 0x4140);  // (x+1, x+2)
        v[1][3 * k + 1] = __byte_perm(W1, 0, 0x4241);  // (x+2, x+3)
        v[1][3 * k + 2] = __byte_perm(W1, 0, 0x4342);  // (x+3, x+4)
        if (k == 1) cword = wb;
      }
      uint32_t out[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t* u = v[h];
        cswap16(u[0], u[1]); cswap16(u[3], u[4]); cswap16(u[6], u[7]);
        cswap16(u[1], u[2]); cswap16(u[4], u[5]); cswap16(u[7], u[8]);
        cswap16(u[0], u[1]); cswap16(u[3], u[4]); cswap16(u[6], u[7]);
        cswap16(u[0], u[3]); cswap16(u[3], u[6]); cswap16(u[0], u[3]);
        cswap16(u[1], u[4]); cswap16(u[4], u[7]); cswap16(u[1], u[4]);
        cswap16(u[2], u[5]); cswap16(u[5], u[8]); cswap16(u[2], u[5]);
        cswap16(u[1], u[3]); cswap16(u[5], u[7]); cswap16(u[2], u[6]);
        cswap16(u[4], u[6]); cswap16(u[2], u[4]); cswap16(u[2], u[3]);
        cswap16(u[5], u[6]);
        uint32_t med = u[0];
        med = sel16_valid(u[2], u[1], med);
        med = sel16_valid(u[4], u[2], med);
        med = sel16_valid(u[6], u[3], med);
        med = sel16_valid(u[8], u[4], med);
        out[h] = med | inv16(u16x2_of(cword, h));  // INVALID centre stays INVALID
      }
      const uint32_t o4 = __byte_perm(out[0], out[1], 0x6420);
      *reinterpret_cast<uint32_t*>(md + j * Wsp + x) = o4;
      if (j < nr) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (x + i < Ws) {
            a.masked[(size_t)(y0 + j) * Ws + x + i] = (uint8_t)(cword >> (8 * i));
            a.median[(size_t)(y0 + j) * Ws + x + i] = (uint8_t)(o4 >> (8 * i));
          }
      }
    }
  }
  __syncthreads();
  // 3. per-32-pixel validity masks
  for (int j = 0; j < nf; ++j)
    for (int cc = warp; cc < nch; cc += blockDim.x >> 5) {
      const int x = cc * 32 + lane;
      const unsigned m = __ballot_sync(kFull, x < Ws && md[j * Wsp + x] != kInvalid);
      if (lane == 0) cmask[j * 64 + cc] = m;
    }
  __syncthreads();
  // 4. warp j: exclusive max-scan of chunk last-valid, reverse min-scan of first-valid
  if (warp < nf) {
    const int j = warp;
    int carry = -1;
    for (int base = 0; base < nch; base += 32) {
      const int cc = base + lane;
      const unsigned m = cc < nch ? cmask[j * 64 + cc] : 0u;
      int v = m ? cc * 32 + 31 - __clz(m) : -1;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v = max(v, t);
      }
      const int prev = __shfl_up_sync(kFull, v, 1);
      if (cc < nch) prevLast[j * 64 + cc] = lane == 0 ? carry : max(carry, prev);
      carry = max(carry, __shfl_sync(kFull, v, 31));
    }
    int rc = INT_MAX;  // INT_MAX = none
    for (int base = ((nch - 1) >> 5) << 5; base >= 0; base -= 32) {
      const int cc = base + lane;
      const unsigned m = cc < nch ? cmask[j * 64 + cc] : 0u;
      int v = m ? cc * 32 + __ffs(m) - 1 : INT_MAX;
      for (int o = 1; o < 32; o <<= 1) {  // inclusive min-scan toward lower lanes
        const int t = __shfl_down_sync(kFull, v, o);
        if (lane + o < 32) v = min(v, t);
      }
      const int nxt = __shfl_down_sync(kFull, v, 1);
      const int excl = lane == 31 ? rc : min(nxt, rc);
      if (cc < nch) nextFirst[j * 64 + cc] = excl == INT_MAX ? -1 : excl;
      rc = min(rc, __shfl_sync(kFull, v, 0));
    }
    if (j < nr && lane == 0) {  // per-row summary [first x, last x, first value, last value]
      const int y = y0 + j, first = rc == INT_MAX ? -1 : rc;
      a.rowLast[y] = carry;
      a.rowFirst[y] = first;
      a.rowFirst[2 * a.Hs + y] = first >= 0 ? md[j * Wsp + first] : -1;
      a.rowFirst[3 * a.Hs + y] = carry >= 0 ? md[j * Wsp + carry] : -1;
    }
  }
  __syncthreads();
  // 5. fill values of rows y0 .. y0+nf-1
  for (int j = 0; j < nf; ++j) {
    const uint8_t* mdr = md + j * Wsp;
    const uint16_t* pix = sPix + j * Wsp;
    for (int x = tid; x < Ws; x += blockDim.x) {
      float v;
      if (mdr[x] != kInvalid) {
        v = (float)mdr[x];
      } else {
        const int cc = x >> 5, ln = x & 31;
        const unsigned m = cmask[j * 64 + cc];
        const unsigned below = m & ((1u << ln) - 1u);
        const unsigned above = ln == 31 ? 0u : (m & ~((2u << ln) - 1u));
        const int li = below ? cc * 32 + 31 - __clz(below) : prevLast[j * 64 + cc];
        const int ri = above ? cc * 32 + __ffs(above) - 1 : nextFirst[j * 64 + cc];
        v = fill_value(mdr, pix, x, li, ri, a.T, a.fill_mode);
      }
      fv[j * Wsp + x] = v;
      if (j < nr) {
        if (a.K == 2) a.fill[(size_t)(y0 + j) * Ws + x] = v;
        else a.out[(size_t)(y0 + j - a.out_row0) * Ws + x] = v;
      }
    }
  }
  if (a.K == 2) {
    __syncthreads();
    // 6a. x pass of Step8 on the seeded rows: xr[j][X] for X < W (pairs 2p, 2p+1)
    for (int j = 0; j < nf; ++j) {
      const float* f = fv + j * Wsp;
      const uint8_t* L = sLo + j * Wx;
      float* o = xr + j * Wx;
      for (int p = tid; 2 * p < W; p += blockDim.x) {
        if (p < Ws) {
          const float av = 2.0f * f[p];
          o[2 * p] = av;
          if (2 * p + 1 < W) {
            float v = av;
            if (p + 1 < Ws) {
              const float bv = 2.0f * f[p + 1];
              if (fabsf(__fsub_rn(av, bv)) <= thr) {
                v = __fmul_rn(__fadd_rn(av, bv), 0.5f);
              } else {
                const int c = L[2 * p + 1];
                v = (abs((int)L[2 * p] - c) <= abs((int)L[2 * p + 2] - c)) ? av : bv;
              }
            }
            o[2 * p + 1] = v;
          }
        } else {  // odd W: the extra last column copies its predecessor (an odd column = av)
          o[2 * p] = 2.0f * f[Ws - 1];
        }
      }
    }
    __syncthreads();
    // 6b. output rows 2y, 2y+1 (+ the extra last row of an odd H): y pass, linear
    for (int j = 0; j < nr; ++j) {
      const int y = y0 + j;
      const float* x0r = xr + j * Wx;
      const float* x1r = xr + (j + 1) * Wx;
      const bool down = j + 1 < nf;
      float* o0 = a.out + (size_t)(2 * y - a.out_row0) * W;
      float* o1 = o0 + W;
      const bool has1 = 2 * y + 1 < a.H;
      const bool extra = (y == a.Hs - 1) && (2 * y + 2 < a.H);
      for (int X = tid; X < W; X += blockDim.x) {
        const float v0 = x0r[X];
        o0[X] = v0;
        if (has1) {
          const float v1 = down ? __fmul_rn(__fadd_rn(v0, x1r[X]), 0.5f) : v0;
          o1[X] = v1;
          if (extra) o1[W + X] = v1;
        }
      }
    }
  }
  // 7. rule (d): the last CTA patches rows with no valid pixel
  if (!a.rule_d) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  int mine = 0;  // parallel check first: almost always no row needs patching
  for (int r = tid; r < a.Hs; r += blockDim.x) mine |= __ldcg(a.rowLast + r) < 0;
  if (!__syncthreads_or(mine)) {
    if (tid == 0) *a.counter = 0u;
    return;
  }
  bool any = false;
  for (int r = 0; r < a.Hs; ++r) {
    if (__ldcg(a.rowLast + r) >= 0) continue;
    any = true;
    const float v = rule_d_value(a, r);
    float* dst = (a.K == 2 ? a.fill : a.out) + (size_t)r * Ws;
    for (int x = tid; x < Ws; x += blockDim.x) dst[x] = v;
  }
  if (any && a.K == 2) {
    __threadfence();
    __syncthreads();
    for (int r = 0; r < a.Hs; ++r) {
      if (__ldcg(a.rowLast + r) >= 0) continue;
      for (int Y = max(2 * r - 1, 0); Y <= min(2 * r + 2, a.H - 1); ++Y) su_row_global(a, Y, thr);
    }
  }
  if (tid == 0) *a.counter = 0u;
}

// Band mode: the frame-wide per-row summary that fill rule (d)
// needs (R25b: an all-invalid row takes the last valid value of the nearest
// row above that has one, else the first valid value of the nearest row
// below, else 0).  summ: int32 [Hs_g][2] = (last valid value, first valid
// value), -1 = none; this band writes its own rows and -1 everywhere else, so
// an element-wise MAX over the bands (one NCCL all_reduce) assembles the frame.
__global__ void __launch_bounds__(256) band_summary_kernel(const int32_t* __restrict__ rowFirst,
                                                           int32_t* __restrict__ summ, int Hs,
                                                           int s0, int Hs_g, int pa, int pb) {
  for (int yg = blockIdx.x * blockDim.x + threadIdx.x; yg < Hs_g; yg += gridDim.x * blockDim.x) {
    const int y = yg - s0;
    int2 v = make_int2(-1, -1);
    if (y >= pa && y < pb) v = make_int2(rowFirst[3 * Hs + y], rowFirst[2 * Hs + y]);
    reinterpret_cast<int2*>(summ)[yg] = v;
  }
}

// Rule (d) for the rows this band's output reads (own rows and, K = 2, the
// next band's first row, which Step8's odd rows read), from the frame-wide
// summaries; then Step8 again for the own output rows that read a patched
// fill row.  One CTA; returns at once when no such row is all-invalid.
__global__ void __launch_bounds__(256) band_finish_kernel(PostArgs a, const int32_t* __restrict__ summ,
                                                          int s0, int Hs_g, int out_rows) {
  const int pa = a.y_lo, pb = a.y_hi;
  const int hi = min(pb + (a.K == 2 ? 1 : 0), Hs_g - s0);
  int mine = 0;
  for (int y = pa + threadIdx.x; y < hi; y += blockDim.x) mine |= summ[2 * (y + s0)] < 0;
  if (!__syncthreads_or(mine)) return;
  for (int y = pa; y < hi; ++y) {
    if (summ[2 * (y + s0)] >= 0) continue;
    float v = 0.0f;
    int yy = y + s0 - 1;
    while (yy >= 0 && summ[2 * yy] < 0) --yy;
    if (yy >= 0) {
      v = (float)summ[2 * yy];
    } else {
      yy = y + s0 + 1;
      while (yy < Hs_g && summ[2 * yy + 1] < 0) ++yy;
      if (yy < Hs_g) v = (float)summ[2 * yy + 1];
    }
    if (a.K == 2) {
      for (int x = threadIdx.x; x < a.Ws; x += blockDim.x) a.fill[(size_t)y * a.Ws + x] = v;
    } else if (y < pb) {
      for (int x = threadIdx.x; x < a.Ws; x += blockDim.x) a.out[(size_t)(y - a.out_row0) * a.Ws + x] = v;
    }
  }
  if (a.K != 2) return;
  __threadfence_block();
  __syncthreads();
  const float thr = (float)(a.K * a.T);
  const int Y0 = a.out_row0, Y1 = a.out_row0 + out_rows;  // own output rows (sub-image coordinates)
  for (int y = pa; y < hi; ++y) {
    if (summ[2 * (y + s0)] >= 0) continue;
    for (int Y = max(2 * y - 1, Y0); Y <= min(2 * y + 2, Y1 - 1); ++Y) su_row_global(a, Y, thr);
  }
}

static PostArgs post_args(const Geom& g, Buffers& b, const uint8_t* Lorg, float* out);

cudaError_t launch_band_summary(const Geom& g, Buffers& b, int32_t* summ, cudaStream_t s) {
  band_summary_kernel<<<(g.Hs_g + 255) / 256, 256, 0, s>>>(b.rowFirst, summ, g.Hs, g.s0, g.Hs_g,
                                                            g.pa, g.pb);
  return cudaGetLastError();
}

cudaError_t launch_band_finish(const Geom& g, Buffers& b, const int32_t* summ,
                               const uint8_t* Lorg, float* out, cudaStream_t s) {
  band_finish_kernel<<<1, 256, 0, s>>>(post_args(g, b, Lorg, out), summ, g.s0, g.Hs_g, g.rows_org);
  return cudaGetLastError();
}

static PostArgs post_args(const Geom& g, Buffers& b, const uint8_t* Lorg, float* out) {
  PostArgs a;
  a.DL = b.DL; a.DR = b.DR; a.pixL = b.pixL; a.Lorg = Lorg;
  a.masked = b.masked; a.median = b.median; a.fill = b.fill; a.out = out;
  a.rowFirst = b.rowFirst; a.rowLast = b.rowFirst + g.Hs; a.counter = b.counter;
  a.W = g.W; a.H = g.H; a.Ws = g.Ws; a.Hs = g.Hs; a.K = g.K; a.T = g.t_fill;
  a.fill_mode = g.fill_mode;
  a.Wsp = post_pitch(g.Ws);
  a.Wx = (g.W + 3) & ~3;
  a.y_lo = g.band ? g.pa : 0;
  a.y_hi = g.band ? g.pb : g.Hs;
  a.out_row0 = g.band ? g.top : 0;
  a.rule_d = g.band ? 0 : 1;
  return a;
}

cudaError_t launch_post(const Geom& g, const Plan& p, Buffers& b, const uint8_t* Lorg,
                        float* out, int nfr, cudaStream_t s) {
  const PostArgs a = post_args(g, b, Lorg, out);
  const int R = p.post_rows, nt = p.post_threads, rows = a.y_hi - a.y_lo;
  const dim3 grid((rows + R - 1) / R, 1, nfr);
  if (R == 1) post_kernel<1><<<grid, nt, p.post_smem, s>>>(a);
  else if (R == 2) post_kernel<2><<<grid, nt, p.post_smem, s>>>(a);
  else if (R == 4) post_kernel<4><<<grid, nt, p.post_smem, s>>>(a);
  else post_kernel<8><<<grid, nt, p.post_smem, s>>>(a);
  return cudaGetLastError();
}

// ============================================================================
// GRAY — §III list item 1, BT.601 luma rounded half up (reading R31,
// S:117): floor((299 R + 587 G + 114 B + 500) / 1000), exact integers.
// rgb u8 [H][W][3] -> u8 [H][W]; blockIdx.y selects the image (L / R).
// ============================================================================
__global__ void __launch_bounds__(256) gray_kernel(const uint8_t* __restrict__ rgb0,
                                                   const uint8_t* __restrict__ rgb1,
                                                   uint8_t* __restrict__ g0,
                                                   uint8_t* __restrict__ g1, int n) {
  const uint8_t* rgb = blockIdx.y ? rgb1 : rgb0;
  uint8_t* g = blockIdx.y ? g1 : g0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t r = __ldg(rgb + 3 * (size_t)k), gg = __ldg(rgb + 3 * (size_t)k + 1),
                   b = __ldg(rgb + 3 * (size_t)k + 2);
    g[k] = (uint8_t)((299u * r + 587u * gg + 114u * b + 500u) / 1000u);
  }
}

cudaError_t launch_gray(const uint8_t* rgb0, const uint8_t* rgb1, uint8_t* g0, uint8_t* g1,
                        int W, int H, cudaStream_t s) {
  const int n = W * H;
  const int blocks = std::min((n + 255) / 256, 148 * 8);
  gray_kernel<<<dim3(blocks, rgb1 ? 2 : 1), 256, 0, s>>>(rgb0, rgb1, g0, g1, n);
  return cudaGetLastError();
}

// ============================================================================
// DEPTH — Eq. 1: Z = fl32(fB / d), d <= 0 -> +infinity
// ============================================================================
__global__ void __launch_bounds__(256) depth_kernel(const float* disp, float* Z, int n,
                                                    float fB) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const float d = disp[k];
    Z[k] = d > 0.0f ? __fdiv_rn(fB, d) : __int_as_float(0x7f800000);
  }
}

cudaError_t launch_depth(const float* disp, float* Z, int n, float fB, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int blocks = std::min((n + 255) / 256, 148 * 8);
  depth_kernel<<<blocks, 256, 0, s>>>(disp, Z, n, fB);
  return cudaGetLastError();
}

// ============================================================================
// Launch planning (create time)
// ============================================================================
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 3-D map over a CA_x volume as u64 elements (the (d, d+1) pair of a pixel):
// {Wp columns, Hs rows, ceil(Ds/2) pairs}; box {box_cols columns, box_rows, 1 pair}
static cudaError_t make_tmap(CUtensorMap* m, void* base, const Geom& g, int box_cols, int box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess) return e;
    if (q != cudaDriverEntryPointSuccess || !f) return cudaErrorNotSupported;
    fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  const cuuint64_t rows = (cuuint64_t)g.NB * g.Hs;  // the batch as one tall image
  cuuint64_t dims[3] = {(cuuint64_t)g.Wp, rows, (cuuint64_t)((g.Ds + 1) / 2)};
  cuuint64_t strides[2] = {(cuuint64_t)g.Wp * 8, (cuuint64_t)g.Wp * rows * 8};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t plan_kernels(const Geom& g, Plan& p, Buffers& b, int device) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return e;
  const int nsm = prop.multiProcessorCount;
  // SD / PREP / POST dynamic shared memory
  p.sd_smem = (2 * g.m_pool + 1) * ((g.W + 3) & ~3) + 16;
  {
    p.prep_rows = env_int("STEREO_PREP_ROWS", prep_rows_for(g, nsm), 1, 4);
    if (p.prep_rows == 3) p.prep_rows = 2;
    int P4, BW, Q4, AV;
    prep_geometry(g, 8 * p.prep_rows, P4, BW, Q4, AV);
    p.prep_smem = prep_smem_bytes(8 * p.prep_rows, BW, AV);
  }
  const int Wsp = post_pitch(g.Ws);
  const int Wx = (g.W + 3) & ~3;
  // 4 rows x 384 threads per CTA: best throughput with frames in flight at c2
  // and c3 among {1,2,4,8} x {256,384,512} (a lone frame is ~2% slower than
  // with 2 x 512)
  p.post_rows = env_int("STEREO_POST_ROWS", 4, 1, 8);
  if (p.post_rows == 3) p.post_rows = 2;
  if (p.post_rows > 4) p.post_rows = 8;
  p.post_threads = env_int("STEREO_POST_THREADS", 384, 128, 512) & ~127;
  // step 4 of POST runs one warp per fill row (R + 1 of them)
  p.post_threads = std::max(p.post_threads, (32 * (p.post_rows + 1) + 127) & ~127);
  {
    const int R = p.post_rows;
    p.post_smem = (R + 3) * Wsp + (R + 1) * Wsp + (R + 1) * Wsp * 4 + (R + 1) * Wx * 4 +
                  3 * (R + 1) * 64 * 4 + (R + 1) * Wsp * 2 + 2 * (R + 3) * Wsp + (R + 1) * Wx + 64;
  }
  for (auto fn : {prep_kernel<32, true>, prep_kernel<32, false>, prep_kernel<16, true>,
                  prep_kernel<16, false>, prep_kernel<8, true>, prep_kernel<8, false>}) {
    if (p.prep_smem > 48 * 1024 &&
        (e = raise_smem(fn, p.prep_smem)))
      return e;
    if ((e = max_carveout(fn))) return e;
  }
  for (auto fn : {post_kernel<1>, post_kernel<2>, post_kernel<4>, post_kernel<8>})
    if ((e = max_carveout(fn))) return e;
  for (auto fn : {sd_kernel<0>, sd_kernel<1>, sd_kernel<2>, sd_kernel<3>})
    if ((e = max_carveout(fn))) return e;
  if (p.post_smem > 48 * 1024) {
    for (auto fn : {post_kernel<1>, post_kernel<2>, post_kernel<4>, post_kernel<8>})
      if ((e = raise_smem(fn, p.post_smem)))
        return e;
  }
  if (p.sd_smem > 48 * 1024) {
    switch (g.m_pool) {
      case 0: e = raise_smem(sd_kernel<0>, p.sd_smem); break;
      case 1: e = raise_smem(sd_kernel<1>, p.sd_smem); break;
      case 2: e = raise_smem(sd_kernel<2>, p.sd_smem); break;
      default: e = raise_smem(sd_kernel<3>, p.sd_smem); break;
    }
    if (e != cudaSuccess) return e;
  }
  // YPASS: choose the number of tiles per strip balancing halo cost and waves
  // (per-CTA shared wavefronts per d ~ 1.25*TB + 1.75*B + tot exchange)
  // rows of one launch: a whole batch of NB frames (one tall image), or in
  // band mode the rows whose maps the band's POST reads
  const int yrows0 = g.band ? g.yb - g.ya : g.NB * g.Hs;
  // L2 band staging (NEXT-1 prototype, STEREO_L2_BANDS = n > 1): the x and y
  // passes alternate over n row bands so that a band's CA_x is read back from
  // L2 and discarded there (never written to HBM); off in band mode
  p.l2_bands = g.band ? 0 : env_int("STEREO_L2_BANDS", 0, 0, 64);
  if (p.l2_bands > 1) p.l2_band_rows = (yrows0 + p.l2_bands - 1) / p.l2_bands;
  else p.l2_bands = 0;
  const int yrows = p.l2_bands ? p.l2_band_rows : yrows0;
  // version 1 (16-column strips, two CTAs per SM); STEREO_YPASS_V=2 selects
  // the 32-column strips (conflict-free prefix reads, one 16-warp CTA per
  // SM: measured 2.1x slower at c3, 88 -> 183 us); tiles per
  // strip balance the halo cost against waves
  p.ypass_ver = env_int("STEREO_YPASS_V", 1, 1, 2);
  const int cols = p.ypass_ver == 2 ? kY2Cols : 16;
  const int strips = (g.Ws + cols - 1) / cols;
  const int nb0 = (yrows + kYSegs * kYRPT - 1) / (kYSegs * kYRPT);
  double best = 1e30;
  p.ypass_nb = 0;
  const int nb_force = env_int("STEREO_YPASS_NB", 0, 0, yrows);
  for (int nb = nb0; nb <= yrows; ++nb) {
    if (nb_force && nb != nb_force) continue;
    const int B = (yrows + nb - 1) / nb;
    const int SEG = ypass_seg_for(B + 2 * g.w_y, p.ypass_ver);
    if (!SEG) continue;
    const int smem = p.ypass_ver == 2 ? ypass2_smem_bytes(SEG) : ypass_smem_bytes(SEG);
    // v2: one 512-thread CTA per SM (registers); v1: two when shared memory allows
    const int per_sm = p.ypass_ver == 2 ? 1 : (smem * 2 <= 227 * 1024 ? 2 : 1);
    const int ctas = strips * nb * 2;
    const double waves = (double)((ctas + nsm * per_sm - 1) / (nsm * per_sm));
    // shared-memory wavefronts per CTA and disparity pair (v1 in 16-column
    // units: tile + split prefix ~1.25 TB, windows ~1.75 B; v2 in 32-column
    // units: TMA write + read + prefix 7 TB, windows 6 B, segment totals)
    const double cost = p.ypass_ver == 2 ? waves * (7.0 * kYSegs * SEG + 6.0 * B + 60.0)
                                         : waves * per_sm * (1.25 * kYSegs * SEG + 1.75 * B + 20.0);
    if (cost < best - 1e-9) {
      best = cost;
      p.ypass_nb = nb; p.ypass_B = B; p.ypass_SEG = SEG; p.ypass_smem = smem;
    }
  }
  if (!p.ypass_nb) return cudaErrorInvalidValue;
  if (p.ypass_ver == 2) {
    YPASS2_DISPATCH(p.ypass_SEG, e = max_carveout(ypass2_kernel<SS, false>));
    if (e != cudaSuccess) return e;
    YPASS2_DISPATCH(p.ypass_SEG, e = max_carveout(ypass2_kernel<SS, true>));
    if (e != cudaSuccess) return e;
    YPASS2_DISPATCH(p.ypass_SEG, e = raise_smem(ypass2_kernel<SS, false>, p.ypass_smem));
    if (e != cudaSuccess) return e;
    YPASS2_DISPATCH(p.ypass_SEG, e = raise_smem(ypass2_kernel<SS, true>, p.ypass_smem));
    if (e != cudaSuccess) return e;
  } else {
    YPASS_DISPATCH(p.ypass_SEG, e = max_carveout(ypass_kernel<SS, false>));
    if (e != cudaSuccess) return e;
    YPASS_DISPATCH(p.ypass_SEG, e = max_carveout(ypass_kernel<SS, true>));
    if (e != cudaSuccess) return e;
    YPASS_DISPATCH(p.ypass_SEG, e = raise_smem(ypass_kernel<SS, false>, p.ypass_smem));
    if (e != cudaSuccess) return e;
    YPASS_DISPATCH(p.ypass_SEG, e = raise_smem(ypass_kernel<SS, true>, p.ypass_smem));
    if (e != cudaSuccess) return e;
  }
  // FUSED (NEXT-1 prototype): whole frames of a batch-capacity-1 handle whose x arms fit the
  // 24-column halo; same tiles as the y pass
  p.fused = !g.band && g.NB == 1 && g.w_x_max <= kFHalo && env_int("STEREO_FUSED", 0, 0, 1) == 1;
  if (p.fused) {
    p.fused_smem = fused_smem_bytes(p.ypass_SEG);
    YPASS_DISPATCH(p.ypass_SEG, e = max_carveout(fused_kernel<SS>));
    if (e != cudaSuccess) return e;
    YPASS_DISPATCH(p.ypass_SEG, e = raise_smem(fused_kernel<SS>, p.fused_smem));
    if (e != cudaSuccess) return e;
  }
  // XPASS: one persistent CTA per SM, as many warps (<= 16) as shared memory allows
  p.xpass_C = xpass_chunk_for(g.Ws);
  if (!p.xpass_C) return cudaErrorInvalidValue;
  p.xpass_fixpl = g.Ds + g.w_x_max + 3 <= kXFixExt;
  p.xpass_PL = p.xpass_fixpl ? 32 * p.xpass_C + kXFixExt : 32 * p.xpass_C + g.Ds + g.w_x_max + 3;
  {
    const int nd = p.xpass_C <= 2 * kXMaxC2 ? 2 : 1;
    // Co-residency: with frames in flight on several streams, an x pass of one
    // frame and a y pass of another share each SM when one x-pass CTA of 8
    // warps with a 2-slot ring fits beside one y-pass CTA (registers: 8 + 8
    // warps of <= 128; shared memory: both footprints + the per-CTA reserve).
    // Measured at c3: 143.5 vs 148 us per frame with 6 frames in flight
    // (16 warps / 3 slots alone); a lone frame is ~5% slower.
    const int nd0 = p.xpass_C <= 2 * kXMaxC2 ? 2 : 1;
    const size_t co = sizeof(uint32_t) * ((size_t)256 * 32 + 64 * 32 + (size_t)2 * 4 * 32 * p.xpass_C +
                                          (size_t)8 * nd0 * p.xpass_PL) +
                      kXMaxSlots * (8 + 8 + 4) + 8;
    const bool coresident = co + (size_t)p.ypass_smem + 2 * 1024 <= (size_t)prop.sharedMemPerMultiprocessor;
    const size_t per_warp = sizeof(uint32_t) * (size_t)nd * p.xpass_PL;
    const size_t cap = (size_t)prop.sharedMemPerBlockOptin;
    auto fixed_for = [&](int slots) {
      return sizeof(uint32_t) * ((size_t)256 * 32 + 64 * 32 + (size_t)slots * 4 * 32 * p.xpass_C) +
             kXMaxSlots * (8 + 8 + 4) + 8;
    };
    // alone: 3 slots, unless shared memory then holds fewer warps than with 2
    // (wide rows; c5: 2 slots measured 5% faster)
    int slots_alone = 3;
    if (fixed_for(3) + per_warp <= cap && fixed_for(2) + per_warp <= cap &&
        std::min<size_t>(kXMaxWarps, (cap - fixed_for(2)) / per_warp) >
            std::min<size_t>(kXMaxWarps, (cap - fixed_for(3)) / per_warp))
      slots_alone = 2;
    p.xpass_slots = env_int("STEREO_XPASS_SLOTS", coresident ? 2 : slots_alone, 2, kXMaxSlots);
    const size_t fixed = fixed_for(p.xpass_slots);
    if (fixed + per_warp > cap) return cudaErrorInvalidConfiguration;
    p.xpass_warps = (int)std::min<size_t>(kXMaxWarps, (cap - fixed) / per_warp);
    p.xpass_warps = std::min(p.xpass_warps, env_int("STEREO_XPASS_WARPS", coresident ? 8 : kXMaxWarps, 1, kXMaxWarps));
    p.xpass_smem = (int)(fixed + per_warp * p.xpass_warps);
    e = setup_xpass(p.xpass_C, p.xpass_smem);
    if (e != cudaSuccess) return e;
    p.xpass_grid = nsm;
  }
  const int box_cols = p.ypass_ver == 2 ? kY2Cols : 16;
  if ((e = make_tmap(&p.tmL, b.caxL, g, box_cols, kYSegs * p.ypass_SEG))) return e;
  if ((e = make_tmap(&p.tmR, b.caxR, g, box_cols, kYSegs * p.ypass_SEG))) return e;
  return cudaSuccess;
}

}  // namespace stereo
