/* oracle/stereo_oracle.c — plain CPU oracle of the stereo hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see stereo_oracle.h).  Never linked into, called
 * by, or sharing code with the CUDA product path.
 *
 * Every function is a literal transcription of the paper passage it cites
 * (P:n = PAPER.md line n, S:n = SPEC.md line n), with the readings listed in
 * DESIGN.md §2 (R1..R31) where the paper is silent or garbled.  No prefix
 * sums, no fusion, no reordering: aggregation is direct summation over the
 * cross arms exactly as Step3/Step5 describe it.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * (closed forms, paper/SPEC worked examples under tests/golden/, brute-force
 * enumeration in oracle/brute.py, invariants).  The one documented gap is
 * or_pipeline's real-scene ACCURACY (bad-2.0), which needs Middlebury
 * data: parity unpinned for that property only.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 */
#include "stereo_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static int iabs(int v) { return v < 0 ? -v : v; }

/* S:65-73 "scaled_max_disparity": ceil(D/K) (reading R1: "reduced to half",
 * P:75, rounds up so that every original disparity stays reachable). */
int or_scaled_max_disparity(int D, int K) { return (D + K - 1) / K; }

/* Reading R12c: fixed-point fraction bits.  f = the largest
 * value <= 25 such that a full x window of BORDER costs, (2 w_x + 1) * 2^(f+1),
 * stays below 2^32; f >= 22 for every w_x <= 254, which keeps the relative
 * error of any aggregated cost below 0.5*2^-f / c_AD(1) < 1e-5. */
int or_fixed_bits(int w_x) {
  for (int f = 25; f >= 0; --f) {
    unsigned long long v = (unsigned long long)(2 * w_x + 1) << (f + 1);
    if (v < (1ull << 32)) return f;
  }
  return -1;
}

/* Eq. 4: C_AD = 1 - exp(-|L - R| / lambda_AD), with brightness
 * normalised to [0,1] (reading R12): argument (|dI|/255)/lambda_AD. */
double or_cost_ad(int absdiff, double lambda_ad) {
  return 1.0 - exp(-(((double)absdiff / 255.0) / lambda_ad));
}

/* Eq. 5: C_MC = 1 - exp(-MC / lambda_MC), MC = Hamming distance. */
double or_cost_mc(int hamming, double lambda_mc) {
  return 1.0 - exp(-((double)hamming / lambda_mc));
}

/* Reading R12c: each cost term quantised ONCE, Q = floor(c * 2^f + 0.5). */
void or_fixed_tables(double lambda_ad, double lambda_mc, int f, uint32_t qad[256],
                     uint32_t qmc[7]) {
  double s = ldexp(1.0, f);
  for (int a = 0; a < 256; ++a) qad[a] = (uint32_t)floor(or_cost_ad(a, lambda_ad) * s + 0.5);
  for (int h = 0; h < 7; ++h) qmc[h] = (uint32_t)floor(or_cost_mc(h, lambda_mc) * s + 0.5);
}

/* P:177-178 "MC(alpha, beta) is the Hamming distance": count differing bits. */
int or_hamming6(int a, int b) {
  int x = a ^ b, n = 0;
  for (int i = 0; i < 6; ++i) n += (x >> i) & 1;
  return n;
}

/* Eq. 2 and Step1: mean of the (2m+1)^2 block around
 * (K x, K y).  Readings: R4 border -> clamp; R5 round half up,
 * floor((2*sum + n) / (2n)) with n = (2m+1)^2; R3 odd sizes -> floor
 * (S:142); R7 K = 1 is the "no scaling path" (BASELINE.json c1, c2): identity. */
void or_downscale(const uint8_t* org, int W, int H, int K, int m, uint8_t* out) {
  int Ws = W / K, Hs = H / K;
  if (K == 1) {
    memcpy(out, org, (size_t)W * H);
    return;
  }
  int n = (2 * m + 1) * (2 * m + 1);
  for (int y = 0; y < Hs; ++y)
    for (int x = 0; x < Ws; ++x) {
      int sum = 0;
      for (int j = -m; j <= m; ++j)
        for (int i = -m; i <= m; ++i)
          sum += org[(size_t)clampi(K * y + j, 0, H - 1) * W + clampi(K * x + i, 0, W - 1)];
      out[(size_t)y * Ws + x] = (uint8_t)((2 * sum + n) / (2 * n));
    }
}

/* Mini-census, P:177-182 (Fig. 3 missing): bit i = [I(x+dx_i, y+dy_i) < I(x,y)].
 * Readings: R8 pattern is a parameter (default); R9 strict <; R10 bit i
 * <-> offset i; R11 border -> clamp. */
void or_census(const uint8_t* img, int W, int H, const int32_t* dx, const int32_t* dy,
               uint8_t* out) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int c = img[(size_t)y * W + x], code = 0;
      for (int i = 0; i < 6; ++i) {
        int v = img[(size_t)clampi(y + dy[i], 0, H - 1) * W + clampi(x + dx[i], 0, W - 1)];
        if (v < c) code |= 1 << i;
      }
      out[(size_t)y * W + x] = (uint8_t)code;
    }
}

/* Cross arms, P:226-228 (x) and P:234-237 (y): the number of continuous pixels
 * with |I(c) - I(c + k)| < delta on each side, capped by W_x ("dx=1,W_x")
 * and by the image border (R16).  Strict < (R15). */
void or_arms_x(const uint8_t* img, int W, int H, int delta, int w, uint8_t* minus,
               uint8_t* plus) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int c = img[(size_t)y * W + x];
      int n = 0;
      while (n < w && x + n + 1 <= W - 1 && iabs(img[(size_t)y * W + x + n + 1] - c) < delta) ++n;
      int m = 0;
      while (m < w && x - m - 1 >= 0 && iabs(img[(size_t)y * W + x - m - 1] - c) < delta) ++m;
      plus[(size_t)y * W + x] = (uint8_t)n;
      minus[(size_t)y * W + x] = (uint8_t)m;
    }
}

void or_arms_y(const uint8_t* img, int W, int H, int delta, int w, uint8_t* minus,
               uint8_t* plus) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int c = img[(size_t)y * W + x];
      int n = 0;
      while (n < w && y + n + 1 <= H - 1 && iabs(img[(size_t)(y + n + 1) * W + x] - c) < delta) ++n;
      int m = 0;
      while (m < w && y - m - 1 >= 0 && iabs(img[(size_t)(y - m - 1) * W + x] - c) < delta) ++m;
      plus[(size_t)y * W + x] = (uint8_t)n;
      minus[(size_t)y * W + x] = (uint8_t)m;
    }
}

/* Eq. 3: C^L(x,y,d) = C_AD + C_MC between L(x,y) and R(x-d,y).
 * Reading R12b: a candidate outside the image (x - d < 0) costs BORDER = 2.0,
 * the supremum of the cost range. */
void or_cost_left_double(const uint8_t* L, const uint8_t* R, const uint8_t* cL,
                         const uint8_t* cR, int W, int H, int d, double lad, double lmc,
                         double* out) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      if (x - d < 0) { out[i] = 2.0; continue; }
      size_t j = (size_t)y * W + (x - d);
      out[i] = or_cost_ad(iabs(L[i] - R[j]), lad) + or_cost_mc(or_hamming6(cL[i], cR[j]), lmc);
    }
}

/* Eq. 6, middle expression, computed INDEPENDENTLY of C^L:
 * C^R(x,y,d) = C_AD(R(x,y), L(x+d,y)) + C_MC(R(x,y), L(x+d,y)); BORDER when
 * x + d >= W. */
void or_cost_right_double(const uint8_t* L, const uint8_t* R, const uint8_t* cL,
                          const uint8_t* cR, int W, int H, int d, double lad, double lmc,
                          double* out) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      if (x + d >= W) { out[i] = 2.0; continue; }
      size_t j = (size_t)y * W + (x + d);
      out[i] = or_cost_ad(iabs(R[i] - L[j]), lad) + or_cost_mc(or_hamming6(cR[i], cL[j]), lmc);
    }
}

void or_cost_left_fixed(const uint8_t* L, const uint8_t* R, const uint8_t* cL,
                        const uint8_t* cR, int W, int H, int d, const uint32_t* qad,
                        const uint32_t* qmc, uint32_t border, uint32_t* out) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      if (x - d < 0) { out[i] = border; continue; }
      size_t j = (size_t)y * W + (x - d);
      out[i] = qad[iabs(L[i] - R[j])] + qmc[or_hamming6(cL[i], cR[j])];
    }
}

void or_cost_right_fixed(const uint8_t* L, const uint8_t* R, const uint8_t* cL,
                         const uint8_t* cR, int W, int H, int d, const uint32_t* qad,
                         const uint32_t* qmc, uint32_t border, uint32_t* out) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      if (x + d >= W) { out[i] = border; continue; }
      size_t j = (size_t)y * W + (x + d);
      out[i] = qad[iabs(R[i] - L[j])] + qmc[or_hamming6(cR[i], cL[j])];
    }
}

/* Eq. 7 in Step3's order: CA_x[x] = C[x]; add C[x+dx]
 * for dx = 1..n; add C[x-dx] for dx = 1..m. */
void or_aggregate_x_double(const double* C, const uint8_t* minus, const uint8_t* plus,
                           int W, int H, double* out) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      double s = C[i];
      for (int dx = 1; dx <= plus[i]; ++dx) s += C[i + dx];
      for (int dx = 1; dx <= minus[i]; ++dx) s += C[i - dx];
      out[i] = s;
    }
}

/* Eq. 8 in Step5's order: CA[y] = CA_x[y]; add
 * CA_x[y+dy] for dy = 1..N; add CA_x[y-dy] for dy = 1..M.  Reading E3: Step5(a)
 * "CA^{*L}[d][x][y]" means CA^{*L}_x. */
void or_aggregate_y_double(const double* C, const uint8_t* minus, const uint8_t* plus,
                           int W, int H, double* out) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      double s = C[i];
      for (int dy = 1; dy <= plus[i]; ++dy) s += C[i + (size_t)dy * W];
      for (int dy = 1; dy <= minus[i]; ++dy) s += C[i - (size_t)dy * W];
      out[i] = s;
    }
}

void or_aggregate_x_u64(const uint64_t* C, const uint8_t* minus, const uint8_t* plus,
                        int W, int H, uint64_t* out) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      uint64_t s = C[i];
      for (int dx = 1; dx <= plus[i]; ++dx) s += C[i + dx];
      for (int dx = 1; dx <= minus[i]; ++dx) s += C[i - dx];
      out[i] = s;
    }
}

void or_aggregate_y_u64(const uint64_t* C, const uint8_t* minus, const uint8_t* plus,
                        int W, int H, uint64_t* out) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      uint64_t s = C[i];
      for (int dy = 1; dy <= plus[i]; ++dy) s += C[i + (size_t)dy * W];
      for (int dy = 1; dy <= minus[i]; ++dy) s += C[i - (size_t)dy * W];
      out[i] = s;
    }
}

/* Eq. 9 with Step5's update rule: Min = MAX_VALUE,
 * "If CA[y] < Min[y] then Min[y] = CA[y] and D_map[y] = d", d = 0..D-1 (R2).
 * Reading E4: Eq. 9 prints min, means argmin; strict < keeps the smallest d. */
void or_wta_double(const double* vol, int W, int H, int D, uint8_t* out) {
  size_t n = (size_t)W * H;
  for (size_t i = 0; i < n; ++i) {
    double best = HUGE_VAL;
    int bd = 0;
    for (int d = 0; d < D; ++d)
      if (vol[(size_t)d * n + i] < best) { best = vol[(size_t)d * n + i]; bd = d; }
    out[i] = (uint8_t)bd;
  }
}

void or_wta_u64(const uint64_t* vol, int W, int H, int D, uint8_t* out) {
  size_t n = (size_t)W * H;
  for (size_t i = 0; i < n; ++i) {
    uint64_t best = UINT64_MAX;
    int bd = 0;
    for (int d = 0; d < D; ++d)
      if (vol[(size_t)d * n + i] < best) { best = vol[(size_t)d * n + i]; bd = d; }
    out[i] = (uint8_t)bd;
  }
}

/* Eq. 10: with k = D^L(x,y), (x,y) is a GCP iff D^R(x-k,y) = k.
 * Readings: E5 Step6's "D^R_map[y][+k]" means [y][x-k]; R19 x-k < 0
 * is not a GCP; R20 exact equality.  Non-GCPs become INVALID. */
void or_cross_check(const uint8_t* DL, const uint8_t* DR, int W, int H, uint8_t* masked) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      int k = DL[(size_t)y * W + x];
      int gcp = (x - k >= 0) && (DR[(size_t)y * W + (x - k)] == k);
      masked[(size_t)y * W + x] = gcp ? (uint8_t)k : (uint8_t)OR_INVALID;
    }
}

/* Step7, first half: median filter on the left map.
 * Readings: R21 3x3, border clamped; R22 a valid pixel takes the
 * lower median of the VALID values among its 9 clamped neighbours (centre
 * included); INVALID stays INVALID; R23 before the fill. */
void or_median3x3(const uint8_t* in, int W, int H, uint8_t* out) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x;
      if (in[i] == OR_INVALID) { out[i] = OR_INVALID; continue; }
      int v[9], n = 0;
      for (int j = -1; j <= 1; ++j)
        for (int k = -1; k <= 1; ++k) {
          int a = in[(size_t)clampi(y + j, 0, H - 1) * W + clampi(x + k, 0, W - 1)];
          if (a != OR_INVALID) v[n++] = a;
        }
      for (int p = 1; p < n; ++p)       /* insertion sort */
        for (int q = p; q > 0 && v[q - 1] > v[q]; --q) { int t = v[q]; v[q] = v[q - 1]; v[q - 1] = t; }
      out[i] = (uint8_t)v[(n - 1) / 2];
    }
}

/* Bilateral estimation, §III.E steps 1-3 and Step7,
 * on the median output, guided by the scaled left image.  Per INVALID pixel:
 * D_l = nearest valid to the left at distance i, D_r nearest valid to the right
 * at distance j.
 *  (a) |D_l - D_r| <= T: linear interpolation (reading E6: Eq. 11 as printed
 *      moves away from D_r; the prose "changing continuously" fixes the sign)
 *      = (D_l*j + D_r*i)/(i+j), ONE correctly-rounded binary32 division (R26);
 *  (b) else D_l if |L(x-i) - L(x)| <= |L(x+j) - L(x)| else D_r (R24: tie -> left);
 *  (c) one side only -> that side (R25);
 *  (d) a row with no valid pixel -> the nearest valid value preceding it in
 *      raster order (the last valid pixel of the nearest row above that has
 *      one); if none, the first valid pixel of the nearest such row below; if
 *      the whole map is invalid, 0 (reading R25b). */
void or_fill_bilateral(const uint8_t* med, const uint8_t* Limg, int W, int H, int T,
                       int mode, float* out) {
  for (int y = 0; y < H; ++y) {
    const uint8_t* row = med + (size_t)y * W;
    const uint8_t* lrow = Limg + (size_t)y * W;
    float* orow = out + (size_t)y * W;
    int any = 0;
    for (int x = 0; x < W; ++x) any |= (row[x] != OR_INVALID);
    if (!any) continue; /* rule (d), below */
    for (int x = 0; x < W; ++x) {
      if (row[x] != OR_INVALID) { orow[x] = (float)row[x]; continue; }
      int i = 1, j = 1;
      while (x - i >= 0 && row[x - i] == OR_INVALID) ++i;
      while (x + j < W && row[x + j] == OR_INVALID) ++j;
      int hl = x - i >= 0, hr = x + j < W;
      if (hl && hr) {
        int Dl = row[x - i], Dr = row[x + j];
        if (mode == OR_FILL_NEAREST) {          /* Fig. 6(a); tie -> left */
          orow[x] = (float)(i <= j ? Dl : Dr);
        } else if (mode == OR_FILL_SMALLER) {   /* Fig. 6(b) */
          orow[x] = (float)(Dl < Dr ? Dl : Dr);
        } else if (iabs(Dl - Dr) <= T) {
          if (mode == OR_FILL_EQ11_LITERAL)     /* D(x-i) + i (D(x-i) - D(x+j)) / (i+j), P:292,
                                                   as one exact rational rounded once */
            orow[x] = (float)(Dl * (i + j) + i * (Dl - Dr)) / (float)(i + j);
          else
            orow[x] = (float)(Dl * j + Dr * i) / (float)(i + j);
        } else {
          int c = lrow[x];
          orow[x] = (iabs(lrow[x - i] - c) <= iabs(lrow[x + j] - c)) ? (float)Dl : (float)Dr;
        }
      } else if (hl) {
        orow[x] = (float)row[x - i];
      } else {
        orow[x] = (float)row[x + j];
      }
    }
  }
  for (int y = 0; y < H; ++y) {
    const uint8_t* row = med + (size_t)y * W;
    int any = 0;
    for (int x = 0; x < W; ++x) any |= (row[x] != OR_INVALID);
    if (any) continue;
    float v = 0.0f;
    int found = 0;
    for (int yy = y - 1; yy >= 0 && !found; --yy)
      for (int x = W - 1; x >= 0; --x)
        if (med[(size_t)yy * W + x] != OR_INVALID) { v = (float)med[(size_t)yy * W + x]; found = 1; break; }
    for (int yy = y + 1; yy < H && !found; ++yy)
      for (int x = 0; x < W; ++x)
        if (med[(size_t)yy * W + x] != OR_INVALID) { v = (float)med[(size_t)yy * W + x]; found = 1; break; }
    for (int x = 0; x < W; ++x) out[(size_t)y * W + x] = v;
  }
}

void or_rgb_to_gray(const uint8_t* rgb, int W, int H, uint8_t* gray) {
  for (size_t k = 0; k < (size_t)W * H; ++k) {
    const int r = rgb[3 * k], g = rgb[3 * k + 1], b = rgb[3 * k + 2];
    gray[k] = (uint8_t)((299 * r + 587 * g + 114 * b + 500) / 1000);
  }
}

void or_depth(const float* disp, int n, float fB, float* Z) {
  for (int k = 0; k < n; ++k) Z[k] = disp[k] > 0.0f ? fB / disp[k] : INFINITY;
}

/* Step8: scale up x K (K = 2), bilateral along x (the §III.E rule
 * again, with i = j = 1), linear along y.  Readings: R27 values scaled by K
 * (S:449); R28 threshold K*T; R29 seeds on the even grid, x
 * pass first; R30 "linear" along y = mean of the rows above and
 * below, copy of the row above at the bottom edge; the extra last column/row
 * of an odd size copies its predecessor.  All arithmetic binary32. */
void or_scale_up(const float* v, int Ws, int Hs, const uint8_t* Lorg, int W, int H,
                 int K, int T, float* out) {
  if (K == 1) {
    memcpy(out, v, sizeof(float) * (size_t)W * H);
    return;
  }
  const float thr = (float)(K * T);
  /* (1)+(2): seeded rows Y = 2y, y < Hs */
  for (int y = 0; y < Hs; ++y) {
    int Y = 2 * y;
    float* o = out + (size_t)Y * W;
    const uint8_t* lo = Lorg + (size_t)Y * W;
    for (int X = 0; X < W; X += 2)
      if (X / 2 < Ws) o[X] = (float)K * v[(size_t)y * Ws + X / 2];
    for (int X = 1; X < W; X += 2) {
      float a = o[X - 1];
      if (X + 1 < W && (X + 1) / 2 < Ws) {
        float b = o[X + 1];
        if (fabsf(a - b) <= thr) {
          o[X] = (a + b) * 0.5f;
        } else {
          int c = lo[X];
          o[X] = (iabs(lo[X - 1] - c) <= iabs(lo[X + 1] - c)) ? a : b;
        }
      } else {
        o[X] = a;
      }
    }
    for (int X = 0; X < W; X += 2)
      if (X / 2 >= Ws) o[X] = o[X - 1];
  }
  /* (3): every other row, top to bottom */
  for (int Y = 0; Y < H; ++Y) {
    if (Y % 2 == 0 && Y / 2 < Hs) continue;
    float* o = out + (size_t)Y * W;
    const float* up = out + (size_t)(Y - 1) * W;
    int has_down = (Y % 2 == 1) && (Y + 1 < H) && ((Y + 1) / 2 < Hs);
    if (has_down) {
      const float* dn = out + (size_t)(Y + 1) * W;
      for (int X = 0; X < W; ++X) o[X] = (up[X] + dn[X]) * 0.5f;
    } else {
      for (int X = 0; X < W; ++X) o[X] = up[X];
    }
  }
}

static int validate(int W, int H, int D, const or_params* p) {
  if (!(p->lambda_ad > 0) || !(p->lambda_mc > 0) || p->delta <= 0 || p->t_fill < 0 ||
      p->w_x < 0 || p->w_y < 0 || p->k_scale < 1 || D < 1 || W < 1 || H < 1)
    return -1;
  if (p->k_scale > 2 || p->m_pool < 0) return -1;
  if (W / p->k_scale < 1 || H / p->k_scale < 1) return -1;
  if (or_scaled_max_disparity(D, p->k_scale) > 255) return -1;
  if (p->w_x > 254 || p->w_y > 254 || p->w_x_r > 254) return -1;
  if (p->fill_mode < OR_FILL_BILATERAL || p->fill_mode > OR_FILL_EQ11_LITERAL) return -1;
  return 0;
}

/* Full pipeline in the §IV order: SD -> census/arms -> per d:
 * cost, CA_x, CA, WTA (both bases) -> CC -> median -> fill -> SU. */
int or_pipeline(const uint8_t* Lorg, const uint8_t* Rorg, int W, int H, int D,
                const or_params* p, int mode, int nthreads, or_outputs* o) {
  if (validate(W, H, D, p)) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  const int K = p->k_scale, Ws = W / K, Hs = H / K, Ds = or_scaled_max_disparity(D, K);
  const size_t n = (size_t)Ws * Hs;
  uint8_t* buf = (uint8_t*)calloc(n, 16);
  uint8_t *Ls = buf, *Rs = buf + n, *cL = buf + 2 * n, *cR = buf + 3 * n;
  uint8_t *aL = buf + 4 * n, *aR = buf + 8 * n; /* m, n, M, N */
  uint8_t *DL = buf + 12 * n, *DR = buf + 13 * n, *msk = buf + 14 * n, *med = buf + 15 * n;

  or_downscale(Lorg, W, H, K, p->m_pool, Ls);
  or_downscale(Rorg, W, H, K, p->m_pool, Rs);
  or_census(Ls, Ws, Hs, p->census_dx, p->census_dy, cL);
  or_census(Rs, Ws, Hs, p->census_dx, p->census_dy, cR);
  or_arms_x(Ls, Ws, Hs, p->delta, p->w_x, aL, aL + n);
  or_arms_y(Ls, Ws, Hs, p->delta, p->w_y, aL + 2 * n, aL + 3 * n);
  const int wxr = p->w_x_r < 0 ? p->w_x : p->w_x_r;
  or_arms_x(Rs, Ws, Hs, p->delta, wxr, aR, aR + n);
  or_arms_y(Rs, Ws, Hs, p->delta, p->w_y, aR + 2 * n, aR + 3 * n);

  if (mode == OR_MODE_FIXED) {
    const int f = or_fixed_bits(p->w_x > wxr ? p->w_x : wxr);
    uint32_t qad[256], qmc[7];
    or_fixed_tables(p->lambda_ad, p->lambda_mc, f, qad, qmc);
    const uint32_t border = (uint32_t)1 << (f + 1);
    uint32_t* c32 = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint64_t* c64 = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* ax = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* ca = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* bestL = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* bestR = (uint64_t*)malloc(n * sizeof(uint64_t));
    for (size_t i = 0; i < n; ++i) { bestL[i] = UINT64_MAX; bestR[i] = UINT64_MAX; DL[i] = 0; DR[i] = 0; }
    for (int d = 0; d < Ds; ++d) {
      for (int base = 0; base < 2; ++base) {
        const uint8_t* arm = base ? aR : aL;
        if (base == 0)
          or_cost_left_fixed(Ls, Rs, cL, cR, Ws, Hs, d, qad, qmc, border, c32);
        else
          or_cost_right_fixed(Ls, Rs, cL, cR, Ws, Hs, d, qad, qmc, border, c32);
        for (size_t i = 0; i < n; ++i) c64[i] = c32[i];
        or_aggregate_x_u64(c64, arm, arm + n, Ws, Hs, ax);
        or_aggregate_y_u64(ax, arm + 2 * n, arm + 3 * n, Ws, Hs, ca);
        uint32_t* dax = base ? o->caxR : o->caxL;
        uint64_t* dca = base ? o->caR : o->caL;
        if (dax) for (size_t i = 0; i < n; ++i) dax[(size_t)d * n + i] = (uint32_t)ax[i];
        if (dca) memcpy(dca + (size_t)d * n, ca, n * sizeof(uint64_t));
        uint64_t* best = base ? bestR : bestL;
        uint8_t* Dm = base ? DR : DL;
        for (size_t i = 0; i < n; ++i)
          if (ca[i] < best[i]) { best[i] = ca[i]; Dm[i] = (uint8_t)d; }
      }
    }
    free(c32); free(c64); free(ax); free(ca); free(bestL); free(bestR);
  } else {
    double* c = (double*)malloc(n * sizeof(double));
    double* ax = (double*)malloc(n * sizeof(double));
    double* ca = (double*)malloc(n * sizeof(double));
    double* bestL = (double*)malloc(n * sizeof(double));
    double* bestR = (double*)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) { bestL[i] = HUGE_VAL; bestR[i] = HUGE_VAL; DL[i] = 0; DR[i] = 0; }
    for (int d = 0; d < Ds; ++d) {
      for (int base = 0; base < 2; ++base) {
        const uint8_t* arm = base ? aR : aL;
        if (base == 0)
          or_cost_left_double(Ls, Rs, cL, cR, Ws, Hs, d, p->lambda_ad, p->lambda_mc, c);
        else
          or_cost_right_double(Ls, Rs, cL, cR, Ws, Hs, d, p->lambda_ad, p->lambda_mc, c);
        or_aggregate_x_double(c, arm, arm + n, Ws, Hs, ax);
        or_aggregate_y_double(ax, arm + 2 * n, arm + 3 * n, Ws, Hs, ca);
        double* dax = base ? o->caxR_d : o->caxL_d;
        double* dca = base ? o->caR_d : o->caL_d;
        if (dax) memcpy(dax + (size_t)d * n, ax, n * sizeof(double));
        if (dca) memcpy(dca + (size_t)d * n, ca, n * sizeof(double));
        double* best = base ? bestR : bestL;
        uint8_t* Dm = base ? DR : DL;
        for (size_t i = 0; i < n; ++i)
          if (ca[i] < best[i]) { best[i] = ca[i]; Dm[i] = (uint8_t)d; }
      }
    }
    free(c); free(ax); free(ca); free(bestL); free(bestR);
  }

  or_cross_check(DL, DR, Ws, Hs, msk);
  or_median3x3(msk, Ws, Hs, med);
  float* fill = (float*)malloc(n * sizeof(float));
  or_fill_bilateral(med, Ls, Ws, Hs, p->t_fill, p->fill_mode, fill);
  if (o->out) {
    if (K == 1) memcpy(o->out, fill, n * sizeof(float));
    else or_scale_up(fill, Ws, Hs, Lorg, W, H, K, p->t_fill, o->out);
  }
  if (o->Ls) memcpy(o->Ls, Ls, n);
  if (o->Rs) memcpy(o->Rs, Rs, n);
  if (o->cenL) memcpy(o->cenL, cL, n);
  if (o->cenR) memcpy(o->cenR, cR, n);
  if (o->armL) memcpy(o->armL, aL, 4 * n);
  if (o->armR) memcpy(o->armR, aR, 4 * n);
  if (o->DL) memcpy(o->DL, DL, n);
  if (o->DR) memcpy(o->DR, DR, n);
  if (o->masked) memcpy(o->masked, msk, n);
  if (o->median) memcpy(o->median, med, n);
  if (o->fill) memcpy(o->fill, fill, n * sizeof(float));
  free(fill);
  free(buf);
  return 0;
}
