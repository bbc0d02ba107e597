// Exact-integer tensor-core filter for the 1-NN parents (dci.py:527-543),
// tcgen05 (kind::i8, accumulators in TMEM).  Included by build.cu.
//
// The reference picks each point's parent as the fp64 argmin over the next
// level's points of d2 = |c|^2 - 2 p.c (first index on ties).  This filter
// lists, per point, every candidate that can be that argmin; nn_verify_kernel
// then evaluates the listed ones with the reference's fp64 FMA chain.
//
// Quantisation.  Every lifted fp64 row x (dim + 1 <= 129 coordinates, |x| = 1)
// is scaled by u = max|x_i| / 32639 and rounded: X_i = rint(x_i / u), |X_i| <=
// 32639, split into two signed bytes X = 256 hi + lo (lo in [-128, 127], hi in
// [-127, 127]).  Then, exactly in int32 on the tensor cores,
//   S11 = sum hi_p hi_c,  S12 = sum (hi_p lo_c + lo_p hi_c),  S22 = sum lo_p lo_c
// (three TMEM accumulators; S12 is one accumulation over both cross products),
// and X_p . X_c = 65536 S11 + 256 S12 + S22.  Nothing here is rounded, so the
// only errors are the quantisation and the fp32 epilogue:
//   |p.c - u_p u_c X_p.X_c| <= e_p ||c||_1 + e_c ||p~||_1,
// with e = max_i |x_i - u X_i| and the L1 norms measured per row (fp64), and
// the candidate terms bounded by their maxima over the tree.  Per point
//   E = 2 (e_p L1c_max + e_c,max L1p~) + 2^-18  (epilogue fp32 roundings, csq
//       to fp32, and the fp64 chain's own rounding, all far below 2^-18),
// and, as in the f16 filter, the exact argmin j* and all of its exact ties
// satisfy d2~(j*) <= m~ + 2E.  The epilogue keeps a running minimum m and
// lists j whenever d2~(j) <= m + 2E; the running minimum is never below the
// final one, so the list is a superset of the final window.  On 128-d lifted
// keys e ~ 5e-6 and L1 ~ 9: the window is ~3e-4 wide, against 6.5e-3 for the
// f16 filter (whose windows overflow at 128k points).
//
// Tiles.  A CTA owns 128 consecutive point entries (the M = 128 rows of the
// MMA = the 128 TMEM lanes); their digits sit in TMEM as the MMAs' A operand
// (80 columns, loaded once), so shared memory only carries the candidates.
// It streams the candidate tiles of the rows' level(s), 64 candidates per
// tile (N = 64), K = 160 bytes per digit (5 MMA k-steps of 32).  Candidate
// tiles are stored in global memory already in the canonical no-swizzle
// K-major UMMA layout (8-row x 16-byte core matrices; LBO = 128 B between the
// two core matrices of a k-step, SBO = 1280 B between 8-row groups), so one
// 1-D bulk copy moves a tile.  Warp roles (one CTA per SM): warp 0 bulk
// copies (6-stage ring), warp 1 issues the 20 MMAs of a tile (one thread)
// into one of two accumulator stages (3 x 64 TMEM columns each), warps 2-9
// drain TMEM (tcgen05.ld; two warps per 32-lane quarter, 32 columns each) and
// run the window test.
#pragma once

namespace icb {

constexpr int TC_M = 128;                    // point rows per CTA = TMEM lanes
constexpr int TC_N = 64;                     // candidates per tile (MMA N)
constexpr int TC_KB = 160;                   // int8 coordinates per digit row (dim + 1 <= 129, padded)
constexpr int TC_KSTEPS = TC_KB / 32;        // MMA k-steps per digit pair
constexpr int TC_SBO = (TC_KB / 16) * 128;   // bytes between 8-row core-matrix groups
constexpr int TC_AROW = 2 * TC_KB;           // one point row: both digit planes, row-major (TMEM A operand)
constexpr int TC_BDIG = TC_N * TC_KB;        // one digit plane of a candidate tile
constexpr int TC_BTILE = 2 * TC_BDIG;        // 20 KB
constexpr int TC_STAGES = 6;
constexpr int TC_EPI_WARPS = 8;              // two per TMEM lane quarter, 32 columns each
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;
constexpr int TC_QMAX = 32639;               // |X| <= 127 * 256 + 127
constexpr int TC_A_COLS = TC_KB / 4 * 2;     // A digits in TMEM: 4 int8 per 32-bit column, two planes
constexpr int TC_ACC0 = 128;                 // first accumulator column
constexpr int TC_ACC_COLS = 3 * TC_N;        // S11, S12, S22
constexpr int TC_TMEM_COLS = 512;            // A (80) + two accumulator stages (384); one CTA per SM
constexpr float TC_ERND = 3.814697265625e-06f;   // 2^-18
constexpr int TC_MAX_SEG = 64;
static_assert(TC_A_COLS <= TC_ACC0 && TC_ACC0 + 2 * TC_ACC_COLS <= TC_TMEM_COLS, "TMEM budget");

// byte offset of (row r, coordinate k) inside one digit plane
__device__ __forceinline__ int tc_off(int r, int k) {
  return (r >> 3) * TC_SBO + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

// Quantise one lifted fp64 row (one warp) into its two digit planes.
// Returns (on every lane) u, e = max |x - u X| and the L1 norms of x~ and x.
__device__ __forceinline__ void tc_quant_row(const double* x, int D1, int lane, signed char* hi_plane,
                                             signed char* lo_plane, int r, double& u, double& err, double& l1q,
                                             double& l1x, bool umma_layout = true) {
  double v[TC_KB / 32];
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < TC_KB / 32; ++q) {
    const int i = lane + 32 * q;
    v[q] = i < D1 ? x[i] : 0.0;
    s = fmax(s, fabs(v[q]));
  }
  for (int o = 16; o; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  u = s / (double)TC_QMAX;
  double e = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int q = 0; q < TC_KB / 32; ++q) {
    const int i = lane + 32 * q;
    int X = 0;
    if (u > 0.0) {
      double z = rint(v[q] / u);
      z = fmin(fmax(z, -(double)TC_QMAX), (double)TC_QMAX);
      X = (int)z;
    }
    const double xq = (double)X * u;
    e = fmax(e, fabs(v[q] - xq));
    a1 += fabs(xq);
    a2 += fabs(v[q]);
    const int lo = ((X + 128) & 255) - 128;
    const int hi = (X - lo) >> 8;
    const int o = umma_layout ? tc_off(r, i) : i;
    hi_plane[o] = (signed char)hi;
    lo_plane[o] = (signed char)lo;
  }
  for (int o = 16; o; o >>= 1) {
    e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  // fp64 rounding of the products and sums above: a relative 2^-40 margin
  err = e * (1.0 + 0x1p-40) + 0x1p-60;
  l1q = a1 * (1.0 + 0x1p-40);
  l1x = a2 * (1.0 + 0x1p-40);
}

// per tree: tile offset of each level's candidate tiles (levels 1 .. L-1)
__global__ void tc_tile_offsets_kernel(ForestView F, BuildArgs A, const int* cand_off, int* ct_off) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  const int L = F.meta[A.trees[b]].levels;
  int acc = 0;
  for (int lv = 0; lv < 64; ++lv) {
    ct_off[b * 64 + lv] = acc;
    if (lv >= 1 && lv < L) acc += (cand_off[b * 64 + lv + 1] - cand_off[b * 64 + lv] + TC_N - 1) / TC_N;
  }
}

// point rows: the fp64 lifted row (for the verify kernel) and its digits,
// row-major (the filter copies them into TMEM); pmeta[e] = (u, e, L1 of x~)
__global__ void tc_prep_points_kernel(ForestView F, BuildArgs A, const double* nsq, const int* pts,
                                      const int* pts_off, double* p64, signed char* aimg, size_t a_rows,
                                      double* pmeta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int t = A.trees[b];
  const int L = F.meta[t].levels;
  if (L < 2) return;
  const int r = blockIdx.x * 8 + warp;
  if (r >= pts_off[(size_t)b * 64 + L]) return;
  double* row = p64 + ((size_t)b * A.n_points + r) * (ICB_DPAD + 1);
  lift64_row(F, A, b, pts[(size_t)b * A.n_points + r], F.meta[t].c, nsq, row, lane, 32);
  __syncwarp();
  signed char* arow = aimg + ((size_t)b * a_rows + r) * TC_AROW;
  double u, e, l1q, l1x;
  tc_quant_row(row, F.dim + 1, lane, arow, arow + TC_KB, 0, u, e, l1q, l1x, false);
  if (lane == 0) {
    double* m = pmeta + ((size_t)b * A.n_points + r) * 3;
    m[0] = u; m[1] = e; m[2] = l1q;
  }
}

// candidate rows: digits into the level's tiles; cmeta[slot] = (u, |c|^2) as
// fp32; per-tree maxima of e and of the L1 norm of c (cmax[b][0..1], bits of
// non-negative doubles)
__global__ void tc_prep_cands_kernel(ForestView F, BuildArgs A, const int* cand_off, const int* ct_off,
                                     const double* cand64, const double* cand_sq, int stride, signed char* bimg,
                                     size_t b_tiles, float2* cmeta, unsigned long long* cmax) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int t = A.trees[b];
  const int L = F.meta[t].levels;
  if (L < 2) return;
  const int j = blockIdx.x * 8 + warp;
  if (j >= cand_off[(size_t)b * 64 + L] || j >= stride) return;
  int lv = 1;
  while (lv < L - 1 && cand_off[(size_t)b * 64 + lv + 1] <= j) ++lv;
  const int jl = j - cand_off[(size_t)b * 64 + lv];
  const size_t tile = (size_t)ct_off[b * 64 + lv] + jl / TC_N;
  if (tile >= b_tiles) return;   // cannot happen: b_tiles bounds every tree's tiles
  signed char* tp = bimg + ((size_t)b * b_tiles + tile) * TC_BTILE;
  double u, e, l1q, l1x;
  tc_quant_row(cand64 + ((size_t)b * stride + j) * (ICB_DPAD + 1), F.dim + 1, lane, tp, tp + TC_BDIG, jl % TC_N,
               u, e, l1q, l1x);
  if (lane == 0) {
    cmeta[((size_t)b * b_tiles + tile) * TC_N + jl % TC_N] =
        make_float2((float)u, (float)cand_sq[(size_t)b * stride + j]);
    atomicMax(cmax + (size_t)b * 2 + 0, (unsigned long long)__double_as_longlong(e));
    atomicMax(cmax + (size_t)b * 2 + 1, (unsigned long long)__double_as_longlong(l1x));
  }
}

// ---------------------------------------------------------------- tcgen05 helpers
__device__ __forceinline__ unsigned long long tc_desc(unsigned saddr) {
  // K-major, no swizzle: start >> 4, LBO = 128 B, SBO = TC_SBO, version 1 (sm_100)
  return (unsigned long long)((saddr >> 4) & 0x3FFF) | ((unsigned long long)(128 >> 4) << 16) |
         ((unsigned long long)(TC_SBO >> 4) << 32) | (1ull << 46);
}
// kind::i8 instruction descriptor: s32 accumulate, s8 x s8, K-major A and B, M = 128, N = TC_N
constexpr unsigned TC_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(TC_N >> 3) << 17) |
                              ((unsigned)(TC_M >> 4) << 24);

// D[tmem] += A[tmem] . B[smem]^T (A: 128 lanes x 32 int8 in 8 columns)
__device__ __forceinline__ void tc_mma_ts(unsigned tmem_d, unsigned tmem_a, unsigned long long db) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.eq.u32 p, 1, 1;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(TC_IDESC));
}
__device__ __forceinline__ void tc_st8(unsigned taddr, const uint4& a, const uint4& b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(a.x),
               "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
__device__ __forceinline__ void tc_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_ld16(unsigned taddr, unsigned (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_st16(unsigned taddr, unsigned v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ unsigned long long pk2(unsigned lo, unsigned hi) {
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

struct TcSeg {
  int lv, e_begin, e_end, ntile, tile0;
};

template <typename IdxT>
__global__ void __launch_bounds__(TC_THREADS, 1)
    nn_tc_filter_kernel(ForestView F, BuildArgs A, const int* pts_off, const int* cand_off, const int* ct_off,
                        const signed char* aimg, size_t a_rows, const signed char* bimg, size_t b_tiles,
                        const double* pmeta, const float2* cmeta, const unsigned long long* cmax, IdxT* list,
                        int* cnt, float* list_d2, float* thr) {
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  unsigned char* sB = (unsigned char*)(((size_t)tc_raw + 1023) & ~(size_t)1023);
  __shared__ __align__(8) unsigned long long full_bar[TC_STAGES], empty_bar[TC_STAGES], tfull[2], tempty[2];
  __shared__ unsigned s_tmem;
  __shared__ TcSeg seg[TC_MAX_SEG];
  __shared__ int s_nseg;
  __shared__ __align__(16) float s_cm[TC_EPI_WARPS][2 * 64];   // per epilogue warp: (-2 u_c, |c|^2) of two tiles
  __shared__ int s_cnt[TC_M];          // window hits per row (both halves)
  __shared__ float s_min[2][TC_M];     // running minimum per row and half
  const int b = blockIdx.y;
  const int t = A.trees[b];
  const int L = F.meta[t].levels;
  if (L < 2) return;
  const int npts = pts_off[(size_t)b * 64 + L];
  const int e0 = blockIdx.x * TC_M;
  if (e0 >= npts) return;
  const int e1 = min(npts, e0 + TC_M);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    // the levels present among entries [e0, e1) (entries are ordered by level)
    int ns = 0;
    for (int lv = 1; lv < L && ns < TC_MAX_SEG; ++lv) {
      const int a = max(e0, pts_off[(size_t)b * 64 + lv]), z = min(e1, pts_off[(size_t)b * 64 + lv + 1]);
      if (a >= z) continue;
      const int nc = cand_off[(size_t)b * 64 + lv + 1] - cand_off[(size_t)b * 64 + lv];
      seg[ns++] = TcSeg{lv, a, z, (nc + TC_N - 1) / TC_N, ct_off[b * 64 + lv]};
    }
    s_nseg = ns;
    for (int s = 0; s < TC_STAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], TC_EPI_WARPS); }
    mbar_fence_init();
  }
  if (threadIdx.x < TC_M) {
    s_cnt[threadIdx.x] = 0;
    s_min[0][threadIdx.x] = INFINITY;
    s_min[1][threadIdx.x] = INFINITY;
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "n"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = s_tmem;
  const int nseg = s_nseg;
  const signed char* btree = bimg + (size_t)b * b_tiles * TC_BTILE;

  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (int sg = 0; sg < nseg; ++sg)
        for (int k = 0; k < seg[sg].ntile; ++k, ++i) {
          const int s = i % TC_STAGES;
          if (i >= TC_STAGES) mbar_wait(&empty_bar[s], ((i / TC_STAGES) - 1) & 1);
          mbar_expect_tx(&full_bar[s], TC_BTILE);
          bulk_g2s(sB + s * TC_BTILE, btree + (size_t)(seg[sg].tile0 + k) * TC_BTILE, TC_BTILE, &full_bar[s]);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int i = 0;
      for (int sg = 0; sg < nseg; ++sg)
        for (int k = 0; k < seg[sg].ntile; ++k, ++i) {
          const int s = i % TC_STAGES, a = i & 1;
          mbar_wait(&full_bar[s], (i / TC_STAGES) & 1);
          mbar_wait(&tempty[a], (i >> 1) & 1);   // phase 0: the epilogue's initialisation (and A in TMEM)
          tc_fence_after();
          const unsigned b_hi = smem_u32(sB + s * TC_BTILE), b_lo = b_hi + TC_BDIG;
          const unsigned d = tmem + TC_ACC0 + a * TC_ACC_COLS;
          const unsigned a_hi = tmem, a_lo = tmem + TC_A_COLS / 2;
#pragma unroll
          for (int ks = 0; ks < TC_KSTEPS; ++ks) tc_mma_ts(d, a_hi + ks * 8, tc_desc(b_hi + ks * 256));
#pragma unroll
          for (int ks = 0; ks < TC_KSTEPS; ++ks) tc_mma_ts(d + TC_N, a_hi + ks * 8, tc_desc(b_lo + ks * 256));
#pragma unroll
          for (int ks = 0; ks < TC_KSTEPS; ++ks) tc_mma_ts(d + TC_N, a_lo + ks * 8, tc_desc(b_hi + ks * 256));
#pragma unroll
          for (int ks = 0; ks < TC_KSTEPS; ++ks) tc_mma_ts(d + 2 * TC_N, a_lo + ks * 8, tc_desc(b_lo + ks * 256));
          tc_commit(&empty_bar[s]);
          tc_commit(&tfull[a]);
        }
    }
  } else {
    // epilogue: warp w drains TMEM lanes 32 (w % 4) .. +31, columns half * 32 .. +31 of each accumulator
    const int q4 = warp & 3, half = (warp - 2) >> 2, ew = warp - 2;
    const int row = q4 * 32 + lane;
    const int e = e0 + row;
    const bool valid = e < e1;
    float up = 0.f, W = 0.f;
    if (valid) {
      const double* pm = pmeta + ((size_t)b * A.n_points + e) * 3;
      const double ec = __longlong_as_double((long long)cmax[(size_t)b * 2 + 0]);
      const double l1c = __longlong_as_double((long long)cmax[(size_t)b * 2 + 1]);
      const double E = 2.0 * (pm[1] * l1c + ec * pm[2]) + (double)TC_ERND;
      up = (float)pm[0];
      W = (float)(2.0 * E * (1.0 + 0x1p-20) + 0x1p-21);   // + fl(m + W) rounding (|m| <= 4)
    }
    const unsigned tl = tmem + ((unsigned)(q4 * 32) << 16);
    if (half == 0) {
      // the point rows' digits into TMEM (the MMAs' A operand): row e -> lane,
      // 4 int8 per column, hi plane then lo plane
      const uint4* src = reinterpret_cast<const uint4*>(aimg + ((size_t)b * a_rows + e) * TC_AROW);
#pragma unroll
      for (int c = 0; c < TC_A_COLS / 8; ++c) {
        uint4 x = make_uint4(0, 0, 0, 0), y = make_uint4(0, 0, 0, 0);
        if (valid) { x = src[2 * c]; y = src[2 * c + 1]; }
        tc_st8(tl + c * 8, x, y);
      }
    }
    // accumulators start at the bits of M = 1.5 * 2^23, so an int32 sum S
    // (|S| < 2^22: dim + 1 <= 129 coordinates of digit products <= 32512)
    // reads back as the float M + S, exactly: no int -> float conversions
    const unsigned mb = 0x4B400000u;
    auto init_stage = [&](int a) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) tc_st16(tl + TC_ACC0 + a * TC_ACC_COLS + c * TC_N + half * 32 + h * 16, mb);
    };
    init_stage(0);
    init_stage(1);
    tc_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) { mbar_arrive(&tempty[0]); mbar_arrive(&tempty[1]); }
    // per warp: its 32 candidates of the tile as (-2 u_c, |c|^2) column pairs,
    // staged from a coalesced register prefetch of the next tile
    float* cbuf = s_cm[ew];
    const float2* cm = cmeta + (size_t)b * b_tiles * TC_N + half * 32;
    int nsg = 0, nk = 0;   // next tile to prefetch
    float2 pre = make_float2(0.f, 0.f);
    auto prefetch = [&]() {
      if (nsg < nseg) {
        pre = cm[(size_t)(seg[nsg].tile0 + nk) * TC_N + lane];
        if (++nk == seg[nsg].ntile) { ++nsg; nk = 0; }
      }
    };
    prefetch();
    const unsigned long long M2 = 0x4B4000004B400000ull, C256 = 0x4380000043800000ull,
                             C64K = 0x4780000047800000ull;
    const unsigned long long UP2 = pk2(__float_as_uint(up), __float_as_uint(up));
    IdxT* lst = list + ((size_t)b * A.n_points + e) * NF_CAP;
    float* ld2 = list_d2 + ((size_t)b * A.n_points + e) * NF_CAP;
    int i = 0;
    for (int sg = 0; sg < nseg; ++sg) {
      const bool mine = valid && e >= seg[sg].e_begin && e < seg[sg].e_end;
      float m = INFINITY;   // this half's running minimum (>= the row's)
      for (int k = 0; k < seg[sg].ntile; ++k, ++i) {
        const int a = i & 1;
        float* cb = cbuf + a * 64;
        __syncwarp();
        cb[(lane >> 1) * 4 + (lane & 1)] = -2.f * pre.x;        // NaN padding stays NaN
        cb[(lane >> 1) * 4 + 2 + (lane & 1)] = pre.y;
        __syncwarp();
        prefetch();
        mbar_wait(&tfull[a], (i >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          unsigned s11[16], s12[16], s22[16];
          const unsigned col = tl + TC_ACC0 + a * TC_ACC_COLS + half * 32 + h * 16;
          tc_ld16(col, s11);
          tc_ld16(col + TC_N, s12);
          tc_ld16(col + 2 * TC_N, s22);
          tc_wait_ld();
          float d2[16];
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            const unsigned long long a2 = fsub2(pk2(s11[q], s11[q + 1]), M2);
            const unsigned long long b2 = fsub2(pk2(s12[q], s12[q + 1]), M2);
            const unsigned long long c2 = fsub2(pk2(s22[q], s22[q + 1]), M2);
            const unsigned long long x2 = fmul2(ffma2(a2, C64K, ffma2(b2, C256, c2)), UP2);
            const float4 kc = *reinterpret_cast<const float4*>(cb + (h * 8 + (q >> 1)) * 4);
            const unsigned long long r2 =
                ffma2(pk2(__float_as_uint(kc.x), __float_as_uint(kc.y)), x2,
                      pk2(__float_as_uint(kc.z), __float_as_uint(kc.w)));
            d2[q] = __uint_as_float((unsigned)r2);
            d2[q + 1] = __uint_as_float((unsigned)(r2 >> 32));
          }
          float mn = d2[0];
#pragma unroll
          for (int q = 1; q < 16; ++q) mn = fminf(mn, d2[q]);
          m = fminf(m, mn);
          if (mine && mn <= m + W) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (d2[q] <= m + W) {   // both halves of the row list into it: one shared counter
                const int slot = atomicAdd(&s_cnt[row], 1);
                if (slot < NF_CAP) {
                  lst[slot] = (IdxT)(k * TC_N + half * 32 + h * 16 + q);
                  ld2[slot] = d2[q];
                }
              }
          }
        }
        init_stage(a);
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
        // the row's two halves share their running minima (a tighter window)
        // (any value read is a minimum over candidates already seen: >= the final one)
        if (mine) {
          s_min[half][row] = m;
          m = fminf(m, s_min[half ^ 1][row]);
        }
      }
    }
    // every epilogue warp is done with its rows: publish the hit counts
    asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_EPI_WARPS) : "memory");
    if (half == 0 && valid) {
      cnt[(size_t)b * A.n_points + e] = s_cnt[row];
      // the row's final window: the verify kernel skips listed entries above it
      thr[(size_t)b * A.n_points + e] = fminf(s_min[0][row], s_min[1][row]) + W;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TMEM_COLS));
  }
}

}  // namespace icb
