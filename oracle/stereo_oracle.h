/* oracle/stereo_oracle.h — the CPU oracle's OWN header.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or run anything
 * under oracle/.  The CUDA product path (paper_2212_00488_b200/, include/)
 * shares no code, header, table or constant generator with this file.
 *
 * Plain, slow, literal CPU implementation of Chang & Maruyama, "Real-Time
 * High-Quality Stereo Matching System on a GPU" (arXiv 2212.00488), PAPER.md
 * §III, with the readings of SURVEY.md §8(c) / DESIGN.md §2.
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n.
 *
 * Two cost modes share everything but the cost arithmetic:
 *   OR_MODE_FIXED  (0): every cost term quantised once to Q = floor(c*2^f+0.5),
 *                       all sums exact integers -> the bit-exact contract;
 *   OR_MODE_DOUBLE (1): Eqs. 3-8 in IEEE double, direct summation in the
 *                       paper's Step3/Step5 order (centre, +d asc., -d asc.).
 * Layout of every 2-D map: row-major [y][x].  Volumes: [d][y][x].
 * INVALID disparity in u8 maps: 255.
 */
#ifndef STEREO_ORACLE_H
#define STEREO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_INVALID 255
#define OR_MODE_FIXED 0
#define OR_MODE_DOUBLE 1

typedef struct {
  double lambda_ad;     /* 0.3; AD on |dI|/255 */
  double lambda_mc;     /* 2.3; raw Hamming distance */
  int32_t t_fill;       /* T = 3 */
  int32_t w_x, w_y;     /* 21, 31 per-side caps */
  int32_t delta;        /* similarity threshold, strict <, P:227 (value: S:90) */
  int32_t k_scale;      /* K = 2; 1 = no scaling */
  int32_t m_pool;       /* m = 1 */
  int32_t census_dx[6], census_dy[6];  /* mini-census pattern */
  int32_t w_x_r;        /* x cap of the RIGHT-base arms, < 0 = w_x: "(W_x, W_y) can be
                           changed when calculating D^L and D^R", W_y common */
  int32_t fill_mode;    /* OR_FILL_*: non-GCP filling, §III.E */
} or_params;

/* non-GCP filling (§III.E): the bilateral estimation (Eq. 11 read
 * as the interpolation, reading E6), the two baselines of Fig. 6
 * and Eq. 11 exactly as printed (NEXT-3) */
#define OR_FILL_BILATERAL 0
#define OR_FILL_NEAREST 1
#define OR_FILL_SMALLER 2
#define OR_FILL_EQ11_LITERAL 3

typedef struct {          /* every pointer may be NULL (= not requested) */
  uint8_t *Ls, *Rs;       /* scaled images [Hs][Ws] */
  uint8_t *cenL, *cenR;   /* 6-bit census codes */
  uint8_t *armL, *armR;   /* arms [4][Hs][Ws]: m(-x), n(+x), M(-y), N(+y) */
  uint32_t *caxL, *caxR;  /* FIXED CA_x [Ds][Hs][Ws] */
  uint64_t *caL, *caR;    /* FIXED CA   [Ds][Hs][Ws] */
  double *caxL_d, *caxR_d;/* DOUBLE CA_x [Ds][Hs][Ws] */
  double *caL_d, *caR_d;  /* DOUBLE CA   [Ds][Hs][Ws] */
  uint8_t *DL, *DR;       /* WTA maps */
  uint8_t *masked;        /* D^L with non-GCPs = 255 */
  uint8_t *median;        /* after the 3x3 valid-only median */
  float *fill;            /* D^{+L} [Hs][Ws] */
  float *out;             /* D^{fL_org} [H][W] (K=1: equals fill) */
} or_outputs;

int or_scaled_max_disparity(int D, int K);
int or_fixed_bits(int w_x);
double or_cost_ad(int absdiff, double lambda_ad);
double or_cost_mc(int hamming, double lambda_mc);
void or_fixed_tables(double lambda_ad, double lambda_mc, int f,
                     uint32_t qad[256], uint32_t qmc[7]);
int or_hamming6(int a, int b);

void or_downscale(const uint8_t* org, int W, int H, int K, int m, uint8_t* out);
void or_census(const uint8_t* img, int W, int H, const int32_t* dx,
               const int32_t* dy, uint8_t* out);
void or_arms_x(const uint8_t* img, int W, int H, int delta, int w,
               uint8_t* minus, uint8_t* plus);
void or_arms_y(const uint8_t* img, int W, int H, int delta, int w,
               uint8_t* minus, uint8_t* plus);

/* cost slices C^L(.,.,d) and C^R(.,.,d) (Eqs. 3-6) */
void or_cost_left_double(const uint8_t* L, const uint8_t* R, const uint8_t* cL,
                         const uint8_t* cR, int W, int H, int d,
                         double lad, double lmc, double* out);
void or_cost_right_double(const uint8_t* L, const uint8_t* R, const uint8_t* cL,
                          const uint8_t* cR, int W, int H, int d,
                          double lad, double lmc, double* out);
void or_cost_left_fixed(const uint8_t* L, const uint8_t* R, const uint8_t* cL,
                        const uint8_t* cR, int W, int H, int d,
                        const uint32_t* qad, const uint32_t* qmc, uint32_t border,
                        uint32_t* out);
void or_cost_right_fixed(const uint8_t* L, const uint8_t* R, const uint8_t* cL,
                         const uint8_t* cR, int W, int H, int d,
                         const uint32_t* qad, const uint32_t* qmc, uint32_t border,
                         uint32_t* out);
/* Eq. 7 / Eq. 8 on one slice */
void or_aggregate_x_double(const double* C, const uint8_t* minus, const uint8_t* plus,
                           int W, int H, double* out);
void or_aggregate_y_double(const double* C, const uint8_t* minus, const uint8_t* plus,
                           int W, int H, double* out);
void or_aggregate_x_u64(const uint64_t* C, const uint8_t* minus, const uint8_t* plus,
                        int W, int H, uint64_t* out);
void or_aggregate_y_u64(const uint64_t* C, const uint8_t* minus, const uint8_t* plus,
                        int W, int H, uint64_t* out);
/* Eq. 9 over a [D][H][W] volume */
void or_wta_double(const double* vol, int W, int H, int D, uint8_t* out);
void or_wta_u64(const uint64_t* vol, int W, int H, int D, uint8_t* out);
/* Eq. 10 */
void or_cross_check(const uint8_t* DL, const uint8_t* DR, int W, int H, uint8_t* masked);
/* Step7 */
void or_median3x3(const uint8_t* in, int W, int H, uint8_t* out);
void or_fill_bilateral(const uint8_t* med, const uint8_t* Limg, int W, int H, int T,
                       int mode, float* out);
/* §III list item 1 "the two input images are gray-scaled"; formula
 * unstated -> BT.601 luma, round half up (reading R31):
 * gray = floor((299 R + 587 G + 114 B + 500) / 1000); rgb is [H][W][3] */
void or_rgb_to_gray(const uint8_t* rgb, int W, int H, uint8_t* gray);
/* Eq. 1: Z = f B / d, d = 0 -> +infinity ("at infinity",
 * P:107-108); fB = f*B given as one binary32 value, Z = fl32(fB / d) */
void or_depth(const float* disp, int n, float fB, float* Z);
/* Step8 */
void or_scale_up(const float* v, int Ws, int Hs, const uint8_t* Lorg, int W, int H,
                 int K, int T, float* out);

/* Full pipeline.  Returns 0, or -1 on invalid parameters. */
int or_pipeline(const uint8_t* Lorg, const uint8_t* Rorg, int W, int H, int D,
                const or_params* p, int mode, int nthreads, or_outputs* o);

#ifdef __cplusplus
}
#endif
#endif
