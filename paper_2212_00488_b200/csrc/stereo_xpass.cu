// stereo_xpass.cu — the C + CA_x kernel (Step3) in its own translation unit
// (31 lane-chunk instantiations x 2: the slowest file to compile).
#include "stereo_common.cuh"

namespace stereo {

// ============================================================================
// XPASS — cost (Eqs. 3-5) + x aggregation (Eq. 7) for
// BOTH bases, Step3.  The right base reuses the left cost line
// (Eq. 6): C^R(x,d) = C^L(x+d,d), so ONE exclusive prefix row
//   P[k] = sum_{x'<k} Q(x',d)   (u32, modular: window sums < 2^32 are exact)
// gives  CA^L_x(x,d) = P[x+n_L+1] - P[x-m_L]
//        CA^R_x(x,d) = P[x+d+n_R+1] - P[x+d-m_R]
// with P extended by BORDER = 2^(f+1) per column beyond Ws, replacing
// the paper's O(W_x) direct sums by O(1) differences.
// Persistent: one CTA per SM owns a contiguous range of work items
// (row y, disparity group of ND); every warp takes items independently.  The
// four PREP row arrays of a row (codes, window offsets; pitch Wp) arrive by
// bulk asynchronous copies into a ring of `slots` row slots, completed on an
// mbarrier; the warp that finishes the last item of a row in the range
// refills its slot with the row `slots` ahead, so row loads overlap compute
// and no CTA-wide barrier is needed after the start.  Per item:
//   phase A: lane l scans its contiguous chunk [lC, lC+C) (C odd -> shared
//            loads at stride C are bank-conflict free); costs from the fixed
//            tables Q_AD[|dI|] and Q_MC[cL ^ cR] (popc folded into a 64-entry
//            table), both replicated per bank (index*32 + lane); branch-free
//            BORDER select for x < d;
//   warp scan of the 32 lane totals (shuffles) -> P into shared memory;
//   phase C: lanes interleaved over x -> two coalesced 128-B stores per warp
//            and disparity.
// ND = 2: two consecutive disparities d, d+1 per item.  The right pixel of
// (x, d+1) is the one of (x-1, d), so both cost rows come from the same C + 1
// shared loads per lane, both window sets from the same offsets, and the two
// shuffle scans overlap.
// Output layout: u32 [ceil(Ds/2)][Hs][Wp][2] (disparity pairs interleaved; Wp = 32C).
// ============================================================================
struct XArgs {
  const uint32_t* xrow;  // [4][Hs][Wp]
  const uint32_t* qad;
  const uint32_t* qmc;
  uint32_t* caxL;
  uint32_t* caxR;
  int Ws, Hs, Ds, Wp, PL, ext;  // Hs: row stride of the planes (NB frames x scaled rows)
  int rows;                     // rows of this launch (frames x scaled rows; rows are independent)
  uint32_t border;
  int slots;  // row slots in the ring (2..kXMaxSlots)
  uint32_t mc_mask;  // 63, as a parameter (see the Q_MC address below)
  const uint32_t* qtab;  // the replicated tables as laid out in shared memory (40 KB)
  // L2 band staging (NEXT-1 prototype): rows [disc0, disc1) of
  // both whole volumes whose last reader (a y pass) has run are discarded
  // from L2 (no write-back to HBM) by this launch, before its own items
  const uint32_t* discL;
  const uint32_t* discR;
  int disc0, disc1;
};


// one row's four arrays into a slot (single thread)
__device__ __forceinline__ void xpass_load_row(uint32_t* slot, uint64_t* bar, const XArgs& a,
                                               int row) {
  const uint32_t bytes = (uint32_t)a.Wp * 4u;
  const size_t plane = (size_t)a.Hs * a.Wp;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(4u * bytes)
               : "memory");
  for (int k = 0; k < 4; ++k)
    bulk_g2s(slot + k * a.Wp, a.xrow + k * plane + (size_t)row * a.Wp, bytes, bar);
}

// Phase C of an item: CA_x of the lane's columns x = lane + 32 i for both
// bases from the exclusive prefix rows (L: P_d, P_{d+1}; R: the same rows
// shifted by d, resp. d + 1); the pair (d, d+1) of a pixel is one 8-B store
// (CA_x layout u32 [Ds/2][Hs][Wp][2]), 256 coalesced bytes per warp.
// MODE 2: disparities d and d+1 (one 8-B store per pixel); 1: d only, the
// d+1 slot zero (odd-Ds tail of the two-disparity kernel); 0: d only, a 4-B
// store into slot d & 1 (the one-disparity kernel for very wide images).
template <int C, int MODE>
__device__ __forceinline__ void xpass_windows(const uint32_t* sAL, const uint32_t* sAR,
                                              const char* P0, const char* P0d, const char* P1,
                                              const char* P1d, uint2* outL, uint2* outR, int lane,
                                              int slot) {
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const uint32_t al = sAL[lane + 32 * i], ar = sAR[lane + 32 * i];
    const uint32_t alo = al & 0xffffu, ahi = al >> 16, arlo = ar & 0xffffu, arhi = ar >> 16;
    const uint32_t caL = *reinterpret_cast<const uint32_t*>(P0 + ahi) -
                         *reinterpret_cast<const uint32_t*>(P0 + alo);
    const uint32_t caR = *reinterpret_cast<const uint32_t*>(P0d + arhi) -
                         *reinterpret_cast<const uint32_t*>(P0d + arlo);
    // pitch Wp = 32C: padding columns are written, never read
    if (MODE == 0) {
      reinterpret_cast<uint32_t*>(outL + 32 * i)[slot] = caL;
      reinterpret_cast<uint32_t*>(outR + 32 * i)[slot] = caR;
    } else {
      uint32_t caL1 = 0u, caR1 = 0u;
      if (MODE == 2) {
        caL1 = *reinterpret_cast<const uint32_t*>(P1 + ahi) - *reinterpret_cast<const uint32_t*>(P1 + alo);
        caR1 = *reinterpret_cast<const uint32_t*>(P1d + arhi) - *reinterpret_cast<const uint32_t*>(P1d + arlo);
      }
      outL[32 * i] = make_uint2(caL, caL1);
      outR[32 * i] = make_uint2(caR, caR1);
    }
  }
}

// FIXPL: the per-disparity prefix rows have the compile-time pitch 32C + 128
// (usable when D_s + w_x + 3 <= 128), so that P_{d+1} = P_d + constant folds
// into the shared-load immediates instead of one add per window read.
template <int C, int ND, bool FIXPL>
__global__ void __launch_bounds__(kXMaxWarps * 32, 1) xpass_kernel(XArgs a) {
  static_assert(ND == 1 || ND == 2, "one or two disparities per item");
  const int PL = FIXPL ? 32 * C + kXFixExt : a.PL;
  extern __shared__ __align__(128) uint32_t xsm[];
  uint32_t* sQAD = xsm;                // [256][32]  Q_AD[|dI|], one copy per bank
  uint32_t* sQMC = sQAD + 256 * 32;    // [64][32]   Q_MC[popc(cL ^ cR)], indexed by cL ^ cR
  uint32_t* ring = sQMC + 64 * 32;     // [slots][4][32C] row slots
  const int nw = blockDim.x >> 5;
  const int nslot = a.slots;
  uint32_t* Pall = ring + nslot * 4 * 32 * C;  // [nw][ND][PL] exclusive prefixes (+ BORDER)
  uint64_t* full = reinterpret_cast<uint64_t*>(Pall + (size_t)nw * ND * PL);  // [slots]
  uint64_t* empty = full + kXMaxSlots;                                          // [slots]
  uint64_t* tabbar = empty + kXMaxSlots;                                        // [1]
  unsigned* done = reinterpret_cast<unsigned*>(tabbar + 1);                     // [slots]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* P = Pall + warp * ND * PL;

  // this CTA's item range [i0, i1) of the Hs * npairs items, and its rows
  const int npairs = (a.Ds + ND - 1) / ND;
  const long long total = (long long)a.rows * npairs;
  const int i0 = (int)(total * blockIdx.x / gridDim.x);
  const int i1 = (int)(total * (blockIdx.x + 1) / gridDim.x);
  if (i0 >= i1) return;
  const int rfirst = i0 / npairs, rlast = (i1 - 1) / npairs;
  const int skip0 = i0 - rfirst * npairs;  // items of the first row owned by earlier CTAs

  if (threadIdx.x == 0) {
    for (int k = 0; k < nslot; ++k) {
      xbar_init(full + k);
      // one arrival per item of the slot's row: orders every warp's reads of
      // the slot before its refill (the counter below only elects the refiller)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + k)), "r"(npairs)
                   : "memory");
      done[k] = 0u;
    }
    if (skip0)  // items of the first row owned by earlier CTAs
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(empty)),
                   "r"(skip0)
                   : "memory");
    xbar_init(tabbar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the bank-replicated tables arrive pre-built (one 40 KB bulk copy)
    constexpr uint32_t kTabBytes = (256 + 64) * 32 * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(tabbar)),
                 "r"(kTabBytes)
                 : "memory");
    bulk_g2s(sQAD, a.qtab, kTabBytes, tabbar);
    for (int k = 0; k < nslot && rfirst + k <= rlast; ++k)
      xpass_load_row(ring + k * 4 * 32 * C, full + k, a, rfirst + k);
  }
  if (a.disc1 > a.disc0) {  // overlaps the table and first-row copies in flight
    const int lpr = a.Wp * 8 / 128;  // 128-B lines per row of one disparity-pair plane
    const int nrow = a.disc1 - a.disc0;
    const long long nl = (long long)npairs * nrow * lpr;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nl;
         i += (long long)gridDim.x * blockDim.x) {
      const int l = (int)(i % lpr);
      const long long pr = i / lpr;
      const int r = (int)(pr % nrow), pp = (int)(pr / nrow);
      const size_t off = (((size_t)pp * a.Hs + a.disc0 + r) * a.Wp * 8) + (size_t)l * 128;
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<const char*>(a.discL) + off) : "memory");
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<const char*>(a.discR) + off) : "memory");
    }
  }
  __syncthreads();  // barrier inits visible
  xbar_wait(tabbar, 0u);
  // with pixels encoded as census | I << 24, |dI|*128 = vabsdiffu4(pl, pr) >> 17 and
  // (cL ^ cR)*128 = ((pl ^ pr) & 63) << 7: table addresses in two ALU operations.
  const char* qadb = reinterpret_cast<const char*>(sQAD + lane);
  const char* qmcb = reinterpret_cast<const char*>(sQMC + lane);
  // the census mask arrives as a kernel parameter so that it sits in a
  // register: (pl ^ pr) & mask is then one 3-input LOP3 and the table address
  // one LEA (a literal 63 lets the compiler shift first and mask 0x1f80 after)
  const uint32_t mcm = a.mc_mask;
  const char* Pb = reinterpret_cast<const char*>(P);
  const int PLb = 4 * PL;
  const int Ws = a.Ws;
  const uint32_t border = a.border;

  // one item (row y, pair pidx) whose row sits in ring slot `slot`, lap `lap`
  auto item = [&](int y, int pidx, int slot, int lap) {
    const int d = pidx * ND;
    xbar_wait(full + slot, (uint32_t)lap & 1u);
    const uint32_t* sL = ring + slot * 4 * 32 * C;
    const uint32_t* sR = sL + 32 * C;
    const uint32_t* sAL = sR + 32 * C;
    const uint32_t* sAR = sAL + 32 * C;
    const bool two = ND == 2 && d + 1 < a.Ds;
    // ---- phase A: costs of the lane's chunk + local inclusive prefixes
    const uint32_t* Lr = sL + lane * C;
    // elements k < nb have x - d < 0 and take BORDER; their loads land before
    // sR (in the slot's sL or the tables: d <= 255) and are unused
    const int nb = d - lane * C;
    const uint32_t* Rr = sR + lane * C - d;
    // Register passes of CH columns: one pass when the 2C prefix registers fit
    // (C <= kXMaxC2), else two (wide rows, C <= 2 kXMaxC2): the first pass's
    // local prefixes go to shared memory right away and get the lane offset
    // added after the warp scan (one read-modify-write per element).
    constexpr int CH = C <= kXMaxC2 ? C : (C + 1) / 2;
    uint32_t pref[ND][CH];
    uint32_t run[ND] = {};
    uint32_t prv = ND == 2 ? Rr[-1] : 0u;  // right pixel of (x, d+1) = of (x-1, d)
    auto costs = [&](int k0, int kn) {
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (j < kn) {
          const int k = k0 + j;
          const uint32_t pl = Lr[k], pr = Rr[k];
          const uint32_t qa = *reinterpret_cast<const uint32_t*>(qadb + (__vabsdiffu4(pl, pr) >> 17));
          const uint32_t qm = *reinterpret_cast<const uint32_t*>(qmcb + (((pl ^ pr) & mcm) << 7));
          run[0] += (k < nb) ? border : qa + qm;  // reading R12b: out of the right image
          pref[0][j] = run[0];
          if (ND == 2) {
            const uint32_t qa1 = *reinterpret_cast<const uint32_t*>(qadb + (__vabsdiffu4(pl, prv) >> 17));
            const uint32_t qm1 = *reinterpret_cast<const uint32_t*>(qmcb + (((pl ^ prv) & mcm) << 7));
            run[ND - 1] += (k < nb + 1) ? border : qa1 + qm1;
            pref[ND - 1][j] = run[ND - 1];
            prv = pr;
          }
        }
      }
    };
    if (CH < C) {  // first pass, stored without the lane offset
      costs(0, CH);
#pragma unroll
      for (int n = 0; n < ND; ++n) {
        uint32_t* Pl = P + n * PL + lane * C + 1;
#pragma unroll
        for (int j = 0; j < CH; ++j) Pl[j] = pref[n][j];
      }
    }
    costs(C - CH == 0 ? 0 : CH, C - (CH < C ? CH : 0));
    uint32_t incl[ND];
#pragma unroll
    for (int n = 0; n < ND; ++n) incl[n] = run[n];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int n = 0; n < ND; ++n) {
        const uint32_t t = __shfl_up_sync(kFull, incl[n], o);
        if (lane >= o) incl[n] += t;
      }
    }
#pragma unroll
    for (int n = 0; n < ND; ++n) {
      const uint32_t off = incl[n] - run[n];
      uint32_t* Pl = P + n * PL + lane * C + 1;
      if (CH < C) {
#pragma unroll
        for (int j = 0; j < CH; ++j) Pl[j] += off;  // first pass: add the offset
#pragma unroll
        for (int j = 0; j < C - CH; ++j) Pl[CH + j] = pref[n][j] + off;
      } else {
#pragma unroll
        for (int k = 0; k < C; ++k) Pl[k] = pref[n][k] + off;
      }
    }
    if (lane < ND) P[lane * PL] = 0;
    __syncwarp();
    uint32_t PW[ND];
#pragma unroll
    for (int n = 0; n < ND; ++n) PW[n] = P[n * PL + Ws];
    for (int e = lane; e < a.ext; e += 32) {
#pragma unroll
      for (int n = 0; n < ND; ++n) P[n * PL + Ws + 1 + e] = PW[n] + (uint32_t)(e + 1) * border;
    }
    __syncwarp();
    // ---- phase C: window differences (precomputed byte offsets), coalesced stores
    uint2* outL = reinterpret_cast<uint2*>(a.caxL) + ((size_t)(d >> 1) * a.Hs + y) * a.Wp + lane;
    uint2* outR = reinterpret_cast<uint2*>(a.caxR) + ((size_t)(d >> 1) * a.Hs + y) * a.Wp + lane;
    const char* Pdb = Pb + 4 * d;
    if (ND == 1)
      xpass_windows<C, 0>(sAL, sAR, Pb, Pdb, Pb, Pdb, outL, outR, lane, d & 1);
    else if (two)  // (the single-disparity tail item exists only for odd Ds)
      xpass_windows<C, 2>(sAL, sAR, Pb, Pdb, Pb + PLb, Pdb + PLb + 4, outL, outR, lane, 0);
    else
      xpass_windows<C, 1>(sAL, sAR, Pb, Pdb, Pb, Pdb, outL, outR, lane, 0);
  };
#ifndef STEREO_RACECHECK
  // item -> (row y, pair p), row -> (ring slot, lap): one division at the
  // start, then incremental updates (a warp's items are nw apart, nw < npairs
  // is not assumed: the row advance is a short loop)
  int y = (i0 + warp) / npairs, pidx = i0 + warp - y * npairs;
  int slot = (y - rfirst) % nslot, lap = (y - rfirst) / nslot;
#pragma unroll 1
  for (int it = i0 + warp; it < i1; it += nw) {
    item(y, pidx, slot, lap);
    __syncwarp();
    // ---- release the row slot: the warp finishing the row's last item of
    // this range refills the slot with the row `slots` ahead
    if (lane == 0) {
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + slot))
                   : "memory");
      const unsigned target = (unsigned)((lap + 1) * npairs - (slot == 0 ? skip0 : 0));
      const unsigned prev = atomicAdd(done + slot, 1u);
      if (prev + 1u == target && y + nslot <= rlast) {
        xbar_wait(empty + slot, (uint32_t)lap & 1u);  // complete: this was the last item
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        xpass_load_row(ring + slot * 4 * 32 * C, full + slot, a, y + nslot);
      }
    }
    for (pidx += nw; pidx >= npairs; pidx -= npairs) {  // next item of this warp
      ++y;
      if (++slot == nslot) { slot = 0; ++lap; }
    }
  }
#else
  // Sanitizer build (-DSTEREO_RACECHECK, tools/sanitize.sh): the same items
  // in rounds of one item per warp (rw <= npairs, so a round spans at most two
  // rows), a CTA barrier after every round, and the ring refills issued by
  // thread 0 after that barrier once a row's items are all done -- the
  // ordering compute-sanitizer's racecheck models.  Identical results.
  const int rw = min(nw, npairs);
  int next = rfirst;  // (thread 0) first row whose slot has not been refilled
#pragma unroll 1
  for (int base = i0; base < i1; base += rw) {
    const int it = base + warp;
    if (warp < rw && it < i1) {
      const int y = it / npairs;
      item(y, it - y * npairs, (y - rfirst) % nslot, (y - rfirst) / nslot);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int done_to = min(i1, base + rw);  // every item < done_to is complete
      while (next + nslot <= rlast && min(i1, (next + 1) * npairs) <= done_to) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        xpass_load_row(ring + ((next - rfirst) % nslot) * 4 * 32 * C, full + (next - rfirst) % nslot, a,
                       next + nslot);
        ++next;
      }
    }
  }
#endif
}

int xpass_chunk_for(int Ws) {
  for (int c = 3; c <= 63; c += 2)
    if (32 * c >= Ws) return c;
  return 0;
}

// two disparities per item while the prefix registers of one or two register
// passes (2 * ceil(C/2)) fit
template <int C>
constexpr int xpass_nd() { return C <= 2 * kXMaxC2 ? 2 : 1; }

template <int C>
static cudaError_t launch_xpass_c(const Geom& g, const Plan& p, Buffers& b, int row0, int rows,
                                  int disc0, int disc1, cudaStream_t s) {
  // rows [row0, row0 + rows) of the (batch) image: the row arrays and both
  // volumes are addressed from row0 on (rows are independent)
  XArgs a{b.xrow + (size_t)row0 * g.Wp, b.qad, b.qmc, b.caxL + (size_t)row0 * g.Wp * 2,
          b.caxR + (size_t)row0 * g.Wp * 2, g.Ws, g.NB * g.Hs, g.Ds, g.Wp, p.xpass_PL,
          g.Ds + g.w_x_max, rows, g.border, p.xpass_slots, 63u, b.qtab,
          b.caxL, b.caxR, disc0, disc1};
  if (p.xpass_fixpl)
    xpass_kernel<C, xpass_nd<C>(), true><<<p.xpass_grid, p.xpass_warps * 32, p.xpass_smem, s>>>(a);
  else
    xpass_kernel<C, xpass_nd<C>(), false><<<p.xpass_grid, p.xpass_warps * 32, p.xpass_smem, s>>>(a);
  return cudaGetLastError();
}


template <int C>
static cudaError_t setup_xpass_c(int smem) {
  cudaError_t e = raise_smem(xpass_kernel<C, xpass_nd<C>(), true>, smem);
  if (e == cudaSuccess) e = max_carveout(xpass_kernel<C, xpass_nd<C>(), true>);
  if (e == cudaSuccess)
    e = raise_smem(xpass_kernel<C, xpass_nd<C>(), false>, smem);
  if (e == cudaSuccess) e = max_carveout(xpass_kernel<C, xpass_nd<C>(), false>);
  return e;
}

#define XPASS_DISPATCH(C_, EXPR)                        \
  switch (C_) {                                         \
    case 3: { constexpr int CC = 3; EXPR; } break;   \
    case 5: { constexpr int CC = 5; EXPR; } break;   \
    case 7: { constexpr int CC = 7; EXPR; } break;   \
    case 9: { constexpr int CC = 9; EXPR; } break;   \
    case 11: { constexpr int CC = 11; EXPR; } break;   \
    case 13: { constexpr int CC = 13; EXPR; } break;   \
    case 15: { constexpr int CC = 15; EXPR; } break;   \
    case 17: { constexpr int CC = 17; EXPR; } break;   \
    case 19: { constexpr int CC = 19; EXPR; } break;   \
    case 21: { constexpr int CC = 21; EXPR; } break;   \
    case 23: { constexpr int CC = 23; EXPR; } break;   \
    case 25: { constexpr int CC = 25; EXPR; } break;   \
    case 27: { constexpr int CC = 27; EXPR; } break;   \
    case 29: { constexpr int CC = 29; EXPR; } break;   \
    case 31: { constexpr int CC = 31; EXPR; } break;   \
    case 33: { constexpr int CC = 33; EXPR; } break;   \
    case 35: { constexpr int CC = 35; EXPR; } break;   \
    case 37: { constexpr int CC = 37; EXPR; } break;   \
    case 39: { constexpr int CC = 39; EXPR; } break;   \
    case 41: { constexpr int CC = 41; EXPR; } break;   \
    case 43: { constexpr int CC = 43; EXPR; } break;   \
    case 45: { constexpr int CC = 45; EXPR; } break;   \
    case 47: { constexpr int CC = 47; EXPR; } break;   \
    case 49: { constexpr int CC = 49; EXPR; } break;   \
    case 51: { constexpr int CC = 51; EXPR; } break;   \
    case 53: { constexpr int CC = 53; EXPR; } break;   \
    case 55: { constexpr int CC = 55; EXPR; } break;   \
    case 57: { constexpr int CC = 57; EXPR; } break;   \
    case 59: { constexpr int CC = 59; EXPR; } break;   \
    case 61: { constexpr int CC = 61; EXPR; } break;   \
    case 63: { constexpr int CC = 63; EXPR; } break;   \
    default: break;                                     \
  }

cudaError_t launch_xpass(const Geom& g, const Plan& p, Buffers& b, int nfr, cudaStream_t s) {
  return launch_xpass_rows(g, p, b, 0, nfr * g.Hs, 0, 0, s);
}

cudaError_t launch_xpass_rows(const Geom& g, const Plan& p, Buffers& b, int row0, int rows,
                              int disc0, int disc1, cudaStream_t s) {
  cudaError_t e = cudaErrorInvalidValue;
  XPASS_DISPATCH(p.xpass_C, e = launch_xpass_c<CC>(g, p, b, row0, rows, disc0, disc1, s));
  return e;
}

cudaError_t setup_xpass(int C, int smem) {
  cudaError_t e = cudaErrorInvalidValue;
  XPASS_DISPATCH(C, e = setup_xpass_c<CC>(smem));
  return e;
}

}  // namespace stereo
