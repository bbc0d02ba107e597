// Batch DCI-tree build on the device: dci_indexing (dci.py:479-568).
//
//  K1 build_norms   : fp64 |k|^2 in NumPy pairwise order, per-tree max (KeyScale, geometry.py:47-56)
//  K1 build_lift    : lifted rows k/c (fp64 divide -> fp32 store) + tail, clamps (dci.py:517-523)
//  K1 build_levels  : level draws from the tree's PCG64 stream + empty-level compaction (dci.py:511-515)
//  K2 nn_parent     : exact fp64 1-NN parent per level, fixed FMA order (dci.py:527-543)
//  K3 node build    : one 64-bit radix sort of (tree, level desc, first appearance, position)
//                     gives node ids and member order (dci.py:545-558)
//  K4 pages         : leaves in node-id order fill pages of s; page ids continue the store
//                     counter; token->page map and K/V scatter (dci.py:560-567, :368-381)
#include "icb.cuh"
#include "internal.h"
#include <cub/cub.cuh>
#include <cuda_fp16.h>
#include <climits>

namespace icb {

// ---------------------------------------------------------------- K1
__global__ void build_norms_kernel(ForestView F, BuildArgs A, double* nsq, unsigned long long* maxbits) {
  __shared__ double sq[8][ICB_DPAD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int i = blockIdx.x * 8 + warp;
  if (i >= A.n_points) return;
  const float* k = A.keys + ((size_t)b * A.n_points + i) * F.dim;
  for (int j = lane; j < F.dim; j += 32) {
    double x = (double)k[j];
    sq[warp][j] = __dmul_rn(x, x);
  }
  __syncwarp();
  if (lane == 0) {
    double s = pairwise_sum(sq[warp], F.dim);
    nsq[(size_t)b * A.n_points + i] = s;
    atomicMax(maxbits + b, (unsigned long long)__double_as_longlong(s));
  }
}

__global__ void build_scale_kernel(ForestView F, BuildArgs A, const unsigned long long* maxbits) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= A.n) return;
  TreeMeta* m = F.meta + A.trees[b];
  double c;
  if (A.scales) {
    c = A.scales[b];
  } else {
    double mx = sqrt(__longlong_as_double((long long)maxbits[b]));
    if (mx == 0.0) mx = 1.0;
    c = __dmul_rn(1.05, mx);
  }
  m->c = c;
}

__global__ void build_lift_kernel(ForestView F, BuildArgs A, const double* nsq) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int i = blockIdx.x * 8 + warp;
  if (i >= A.n_points) return;
  const int t = A.trees[b];
  TreeMeta* m = F.meta + t;
  const int tok = A.tokens[(size_t)b * A.n_points + i];
  if (tok < 0 || tok >= F.tok_cap) {
    if (lane == 0) set_err(m, ICB_ERR_CAP_TOKENS);
    return;
  }
  const double c = m->c;
  const double norm = sqrt(nsq[(size_t)b * A.n_points + i]);
  const bool over = norm > c;
  const double safe = over ? norm : c;
  const float* k = A.keys + ((size_t)b * A.n_points + i) * F.dim;
  float* row = F.lift + F.tk(t, tok) * ICB_ROWF;
  for (int j = lane; j < ICB_DPAD; j += 32)
    row[j] = j < F.dim ? __double2float_rn(__ddiv_rn((double)k[j], safe)) : 0.0f;
  if (lane < ICB_ROWF - ICB_DPAD) row[ICB_DPAD + lane] = 0.0f;
  __syncwarp();
  if (lane == 0) {
    double ratio = __ddiv_rn(norm, safe);
    double rad = __dsub_rn(1.0, __dmul_rn(ratio, ratio));
    const float tl = __double2float_rn(sqrt(rad > 0.0 ? rad : 0.0));
    F.tail[F.tk(t, tok)] = tl;
    if (ICB_ROWF > ICB_DPAD) row[ICB_DPAD] = tl;
    if (over) atomicAdd(&m->scale_clamps, 1ull);
    int old = atomicCAS(F.tok2page + F.tk(t, tok), -1, -2);
    if (old != -1) set_err(m, ICB_ERR_DUP_ID);
  }
}

// Level draws in input order from the tree's continuing stream (assign_level,
// dci.py:81-88): point i consumes uniforms until the first one >= r (its
// "stop"); its level is the number of draws it consumed.  One CTA per tree
// walks the stream in chunks of NT * LV_K draws -- each thread LV_K
// consecutive draws from a jump-ahead state -- and assigns the stops to
// points with a block scan; level = gap to the previous stop.  The stream is
// left just past point P-1's stop, as the sequential draw leaves it.
#define LV_K 4
template <int NT>
__global__ void __launch_bounds__(NT) build_levels_kernel(ForestView F, BuildArgs A, int* drawn,
                                                          unsigned long long* occ) {
  __shared__ int sm[NT / 32 + 1];
  __shared__ long long smx[NT / 32 + 1];
  __shared__ unsigned long long s_mask;
  __shared__ long long s_last;          // draw index of the last stop so far (-1: none)
  __shared__ int s_done;                // points assigned so far
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  TreeMeta* m = F.meta + A.trees[b];
  const Pcg64 g0 = m->rng;
  const int P = A.n_points;
  // threshold on the 53-bit integer: u < r  <=>  (x >> 11) < ceil(r * 2^53)
  // exactly, since u = (x >> 11) * 2^-53 is exact; compare doubles to be literal
  const double r = F.r;
  icb_u128 At, Ct, Ach, Cch;
  icb_pcg_jump((unsigned long long)tid * LV_K, g0.inc, At, Ct);
  icb_pcg_jump((unsigned long long)NT * LV_K, g0.inc, Ach, Cch);
  if (tid == 0) { s_mask = 0; s_last = -1; s_done = 0; }
  __syncthreads();
  icb_u128 base = g0.state;             // state before the chunk's first draw
  long long d0 = 0;                     // index of the chunk's first draw
  while (s_done < P) {
    icb_u128 st = At * base + Ct;
    unsigned stops = 0;                 // bit k: draw d0 + tid*K + k is a stop
    for (int k = 0; k < LV_K; ++k) {
      st = st * icb_pcg_mult() + g0.inc;
      const double u = (double)(icb_pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
      if (!(u < r)) stops |= 1u << k;
    }
    const int nst = __popc(stops);
    int tot;
    const int ex = block_exclusive_scan<NT>(nst, sm, tot);
    // previous stop before this thread's draws: max over lower threads' last stop
    long long mylast = stops ? d0 + (long long)tid * LV_K + (31 - __clz(stops)) : -1;
    long long inc = mylast;
    for (int o = 1; o < 32; o <<= 1) {
      long long v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o && v > inc) inc = v;
    }
    if (lane == 31) smx[wid] = inc;
    __syncthreads();
    long long prev = s_last;
    for (int w = 0; w < wid; ++w) prev = smx[w] > prev ? smx[w] : prev;
    {
      long long v = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane > 0 && v > prev) prev = v;
    }
    const int done = s_done;
    unsigned long long mask = 0;
    int idx = done + ex;
    for (int k = 0; k < LV_K; ++k) {
      if (!(stops >> k & 1u)) continue;
      const long long d = d0 + (long long)tid * LV_K + k;
      if (idx < P) {
        int lv = (int)(d - prev);
        if (lv > 62) lv = 62;
        drawn[(size_t)b * P + idx] = lv;
        mask |= 1ull << lv;
        if (idx == P - 1) {             // leave the stream just past this stop
          icb_u128 Aj, Cj;
          icb_pcg_jump((unsigned long long)(d + 1), g0.inc, Aj, Cj);
          m->rng.state = Aj * g0.state + Cj;
        }
      }
      prev = d;
      ++idx;
    }
    if (mask) atomicOr(&s_mask, mask);
    __syncthreads();
    if (tid == NT - 1) {
      long long last = smx[0];
      for (int w = 1; w < NT / 32; ++w) last = smx[w] > last ? smx[w] : last;
      if (last > s_last) s_last = last;
      s_done = done + tot;
    }
    base = Ach * base + Cch;
    d0 += (long long)NT * LV_K;
    __syncthreads();
  }
  if (tid == 0) {
    occ[b] = s_mask;
    m->levels = __popcll(s_mask);
    m->n_points = P;
    m->top_node = 0;
    if (P == 0) m->rng = g0;
  }
}

__global__ void build_compact_kernel(ForestView F, BuildArgs A, int* drawn, const unsigned long long* occ) {
  int b = blockIdx.y;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_points) return;
  int t = A.trees[b];
  size_t e = (size_t)b * A.n_points + i;
  int lv = drawn[e];
  int c = __popcll(occ[b] & ((2ull << lv) - 1ull));
  drawn[e] = c;
  int tok = A.tokens[e];
  if (tok >= 0 && tok < F.tok_cap) F.level[F.tk(t, tok)] = (int8_t)c;
}

// ---------------------------------------------------------------- level lists
// Per tree (one CTA): own_base scan, per-level point lists (top == lv) and
// candidate lists (top > lv), in input order.  Positions are input indices.
template <int NT>
__global__ void build_lists_kernel(ForestView F, BuildArgs A, const int* top, int* own_base_pos,
                                   int* pts, int* pts_off, int* cands, int* cand_off, int* ent_cnt) {
  __shared__ int sm[NT / 32 + 1];
  __shared__ int carry;
  const int b = blockIdx.x;
  const int t = A.trees[b];
  const int P = A.n_points;
  const int L = F.meta[t].levels;
  const int* tp = top + (size_t)b * P;
  // own_base: exclusive scan of (top - 1)
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < P; base += NT) {
    int i = base + threadIdx.x;
    int v = i < P ? tp[i] - 1 : 0;
    int tot;
    int ex = block_exclusive_scan<NT>(v, sm, tot);
    if (i < P) {
      own_base_pos[(size_t)b * P + i] = carry + ex;
      int tok = A.tokens[(size_t)b * P + i];
      F.own_base[F.tk(t, tok)] = carry + ex;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    F.meta[t].own_top = carry;
    if (carry > F.own_cap) set_err(F.meta + t, ICB_ERR_CAP_OWN);
    ent_cnt[b] = carry + P;  // sum of top levels = entries for node construction
  }
  __syncthreads();
  // per level lists
  int* pb = pts + (size_t)b * P;
  int* cb = cands + (size_t)b * P;   // sum over lv of |top > lv| = own_top <= P*? (bounded by capacity check)
  int pcur = 0, ccur = 0;
  for (int lv = 1; lv < L; ++lv) {
    if (threadIdx.x == 0) { pts_off[(size_t)b * 64 + lv] = pcur; cand_off[(size_t)b * 64 + lv] = ccur; }
    for (int base = 0; base < P; base += NT) {
      int i = base + threadIdx.x;
      int tv = i < P ? tp[i] : 0;
      int tot1, tot2;
      int e1 = block_exclusive_scan<NT>(tv == lv ? 1 : 0, sm, tot1);
      int e2 = block_exclusive_scan<NT>(tv > lv ? 1 : 0, sm, tot2);
      if (i < P && tv == lv) pb[pcur + e1] = i;
      if (i < P && tv > lv) {
        if (ccur + e2 < P) cb[ccur + e2] = i;
        else set_err(F.meta + t, ICB_ERR_CAP_OWN);
      }
      pcur += tot1;
      ccur += tot2;
    }
  }
  if (threadIdx.x == 0) {
    pts_off[(size_t)b * 64 + L] = pcur;
    cand_off[(size_t)b * 64 + L] = ccur;
    pts_off[(size_t)b * 64 + 0] = L;  // slot 0 stores the level count
  }
}

// fp64 lifted row of input point i of build slot b, written to dst[dim+1]
__device__ __forceinline__ void lift64_row(const ForestView& F, const BuildArgs& A, int b, int i,
                                           double c, const double* nsq, double* dst, int lane, int nl) {
  const double norm = sqrt(nsq[(size_t)b * A.n_points + i]);
  const double safe = norm > c ? norm : c;
  const float* k = A.keys + ((size_t)b * A.n_points + i) * F.dim;
  for (int j = lane; j < F.dim; j += nl) dst[j] = __ddiv_rn((double)k[j], safe);
  if (lane == 0) {
    double ratio = __ddiv_rn(norm, safe);
    double rad = __dsub_rn(1.0, __dmul_rn(ratio, ratio));
    dst[F.dim] = sqrt(rad > 0.0 ? rad : 0.0);
  }
}

// candidate fp64 rows + squared norms (sequential FMA chain)
__global__ void build_cand64_kernel(ForestView F, BuildArgs A, const double* nsq, const int* cands,
                                    const int* cand_off, double* cand64, double* cand_sq, int stride) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int t = A.trees[b];
  const int L = F.meta[t].levels;
  const int total = L > 1 ? cand_off[(size_t)b * 64 + L] : 0;
  const int j = blockIdx.x * 8 + warp;
  if (j >= total || j >= stride) return;
  const int i = cands[(size_t)b * A.n_points + j];
  double* dst = cand64 + ((size_t)b * stride + j) * (ICB_DPAD + 1);
  lift64_row(F, A, b, i, F.meta[t].c, nsq, dst, lane, 32);
  __syncwarp();
  if (lane == 0) {
    double acc = 0.0;
    for (int u = 0; u <= F.dim; ++u) acc = __fma_rn(dst[u], dst[u], acc);
    cand_sq[(size_t)b * stride + j] = acc;
  }
}

// K2: exact 1-NN, fp64.  Block = 64 points x all candidates of their level,
// candidates streamed in tiles of 64 with k-chunks of 32 coordinates.
#define NN_BM 64
#define NN_BN 64
#define NN_KC 32
__global__ void __launch_bounds__(256) nn_parent_kernel(ForestView F, BuildArgs A, const double* nsq,
                                                        const int* pts, const int* pts_off,
                                                        const int* cands, const int* cand_off,
                                                        const double* cand64, const double* cand_sq,
                                                        int stride, int* parent_pos, const int* ovf_cnt = nullptr,
                                                        int ovf_cap = 0) {
  extern __shared__ double smem[];
  double* sp = smem;                              // [NN_BM][dim+1 padded]
  const int D1 = F.dim + 1;
  const int PS = D1 | 1;                          // odd stride
  double* sc = sp + NN_BM * PS;                   // [NN_BN][NN_KC + 1]
  __shared__ int s_lv[NN_BM];
  __shared__ double s_best[NN_BM][16];
  __shared__ int s_arg[NN_BM][16];
  const int b = blockIdx.y;
  const int t = A.trees[b];
  const int L = F.meta[t].levels;
  if (L < 2) return;
  const int npts = pts_off[(size_t)b * 64 + L];
  const int e0 = blockIdx.x * NN_BM;
  if (e0 >= npts) return;
  const int e1 = min(npts, e0 + NN_BM);
  const double c = F.meta[t].c;
  const int tid = threadIdx.x;
  if (ovf_cnt) {
    // after the filter: only blocks holding a point whose window overflowed
    __shared__ int s_any;
    if (tid == 0) s_any = 0;
    __syncthreads();
    for (int e = e0 + tid; e < e1; e += blockDim.x)
      if (ovf_cnt[(size_t)b * A.n_points + e] > ovf_cap) s_any = 1;
    __syncthreads();
    if (!s_any) return;
  }
  // levels of block entries
  for (int e = e0 + tid; e < e1; e += blockDim.x) {
    int lv = 1;
    while (lv < L - 1 && pts_off[(size_t)b * 64 + lv + 1] <= e) ++lv;
    s_lv[e - e0] = lv;
  }
  // lifted fp64 rows of the block's points
  for (int r = tid >> 5; r < e1 - e0; r += blockDim.x >> 5)
    lift64_row(F, A, b, pts[(size_t)b * A.n_points + e0 + r], c, nsq, sp + r * PS, tid & 31, 32);
  __syncthreads();
  const int ty = tid >> 4, tx = tid & 15;   // thread: points ty*4..+3, cands tx + 16*j
  int seg = e0;
  while (seg < e1) {
    const int lv = s_lv[seg - e0];
    int segend = seg;
    while (segend < e1 && s_lv[segend - e0] == lv) ++segend;
    const int c0 = cand_off[(size_t)b * 64 + lv];
    const int nc = cand_off[(size_t)b * 64 + lv + 1] - c0;   // points with top > lv
    double best[4];
    int arg[4];
    for (int u = 0; u < 4; ++u) { best[u] = 0.0; arg[u] = -1; }
    for (int cb = 0; cb < nc; cb += NN_BN) {
      double acc[4][4];
      for (int u = 0; u < 4; ++u)
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
      for (int kc = 0; kc < D1; kc += NN_KC) {
        const int kn = min(NN_KC, D1 - kc);
        __syncthreads();
        for (int x = tid; x < NN_BN * NN_KC; x += blockDim.x) {
          int rr = x / NN_KC, cc = x % NN_KC;
          double v = 0.0;
          if (cb + rr < nc && cc < kn) v = cand64[((size_t)b * stride + c0 + cb + rr) * (ICB_DPAD + 1) + kc + cc];
          sc[rr * (NN_KC + 1) + cc] = v;
        }
        __syncthreads();
        for (int u = 0; u < kn; ++u) {
          double pv[4], cv[4];
          for (int q = 0; q < 4; ++q) pv[q] = sp[(ty * 4 + q) * PS + kc + u];
          for (int q = 0; q < 4; ++q) cv[q] = sc[(tx + 16 * q) * (NN_KC + 1) + u];
          for (int q = 0; q < 4; ++q)
            for (int w = 0; w < 4; ++w) acc[q][w] = __fma_rn(pv[q], cv[w], acc[q][w]);
        }
      }
      // d2 = |c|^2 - 2 p.c, argmin with first-index tie break
      for (int w = 0; w < 4; ++w) {
        int j = cb + tx + 16 * w;
        if (j >= nc) continue;
        double csq = cand_sq[(size_t)b * stride + c0 + j];
        for (int q = 0; q < 4; ++q) {
          double d2 = __dsub_rn(csq, __dmul_rn(2.0, acc[q][w]));
          if (arg[q] < 0 || d2 < best[q] || (d2 == best[q] && j < arg[q])) { best[q] = d2; arg[q] = j; }
        }
      }
    }
    // reduce over the 16 tx threads of each point
    for (int q = 0; q < 4; ++q) { s_best[ty * 4 + q][tx] = best[q]; s_arg[ty * 4 + q][tx] = arg[q]; }
    __syncthreads();
    if (tid < NN_BM) {
      int e = e0 + tid;
      if (e >= seg && e < segend) {
        double bb = 0.0;
        int ba = -1;
        for (int x = 0; x < 16; ++x) {
          int a = s_arg[tid][x];
          double d = s_best[tid][x];
          if (a < 0) continue;
          if (ba < 0 || d < bb || (d == bb && a < ba)) { bb = d; ba = a; }
        }
        parent_pos[(size_t)b * A.n_points + pts[(size_t)b * A.n_points + e]] =
            cands[(size_t)b * A.n_points + c0 + ba];
      }
    }
    __syncthreads();
    seg = segend;
  }
}

// ---------------------------------------------------------------- K2' filtered exact 1-NN
// The argmin of nn_parent_kernel, found without evaluating every candidate in
// fp64.  Two passes over the candidates of the point's level:
//  pass 0: tensor-core (mma.sync f16 x f16 -> f32) approximate
//          d2~ = |c|^2 - 2 p.c and its per-point minimum m~;
//  pass 1: the same d2~ again; every candidate with d2~ <= m~ + W gets the
//          exact fp64 d2 of nn_parent_kernel (the same sequential FMA chain,
//          evaluated by the thread holding that accumulator), and the exact
//          (d2, index) minimum wins, first index on ties.
// Exactness: lifted rows have norm <= 1, so |d2~ - d2| <= E with
//   E = 2 * (2^-10 [f16 rounding of both operands] + 129 * 2^-18 [f32 tensor
//   accumulation, generous]) + 2^-20 [epilogue] < 3.0e-3.
// The exact argmin j* satisfies d2~(j*) <= d2(j*) + E <= d2(j~) + E <= m~ + 2E,
// and so does every exact tie of it, so W = 2E rounded up keeps them all.  The
// window costs nothing in correctness, only verification work (on clustered
// 128-d keys about 80 candidates per point fall inside it, of ~3k).
#define NF_K 144                 // (dim + 1) padded to a multiple of 16
#define NF_KS (NF_K + 8)         // smem row stride (halves): conflict-free ldmatrix
#define NF_BM 64
#define NF_BN 128
#define NF_WINDOW 6.5e-3f
#define NF_CAP 256               // window hits kept per point; more -> verify all candidates

// ICB_PROF diagnostics: points verified, exact chains run, windows that overflowed
__device__ unsigned long long g_build_prof[4];

// one warp per row: lifted fp64 point rows (p64, for verification) and f16
// copies of point and candidate rows, zero padded to NF_K
__global__ void nn_half_kernel(ForestView F, BuildArgs A, const double* nsq, const int* pts,
                               const int* pts_off, const double* cand64, const int* cand_off, int stride,
                               double* p64, __half* p16, __half* c16) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int t = A.trees[b];
  const int L = F.meta[t].levels;
  if (L < 2) return;
  const int r = blockIdx.x * 8 + warp;
  const int npts = pts_off[(size_t)b * 64 + L];
  const int ncand = cand_off[(size_t)b * 64 + L];
  if (r < npts) {
    double* row = p64 + ((size_t)b * A.n_points + r) * (ICB_DPAD + 1);
    lift64_row(F, A, b, pts[(size_t)b * A.n_points + r], F.meta[t].c, nsq, row, lane, 32);
    __syncwarp();
    __half* dst = p16 + ((size_t)b * A.n_points + r) * NF_K;
    for (int u = lane; u < NF_K; u += 32) dst[u] = __double2half(u <= F.dim ? row[u] : 0.0);
  }
  if (r < ncand && r < stride) {
    const double* src = cand64 + ((size_t)b * stride + r) * (ICB_DPAD + 1);
    __half* dst = c16 + ((size_t)b * stride + r) * NF_K;
    for (int u = lane; u < NF_K; u += 32) dst[u] = __double2half(u <= F.dim ? src[u] : 0.0);
  }
}

__device__ __forceinline__ void ldsm_x4(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const unsigned* a, unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ int f2ord(float f) {   // order-preserving float -> int
  int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__device__ __forceinline__ void nn_better(double d, int j, double& best, int& arg) {
  if (arg < 0 || d < best || (d == best && j < arg)) { best = d; arg = j; }
}

struct NfSmem {
  __half a[NF_BM][NF_KS];
  __half bt[2][NF_BN][NF_KS];
  float csq[2][NF_BN];
  int rmin[NF_BM];
  int lv[NF_BM];
  int cnt[NF_BM];                  // window hits per row
};

constexpr int NV_W = 8;   // verify: warps (points) per CTA
constexpr int NV_R = 8;   // verify: candidates per round (the windows hold ~2 after pruning)

// One warp per point entry: the exact fp64 d2 of nn_parent_kernel over the
// point's window hits (all of its level's candidates when the window held more
// than NF_CAP), first index on ties.  The point row is broadcast from smem.
template <typename IdxT>
__global__ void __launch_bounds__(NV_W * 32) nn_verify_kernel(ForestView F, BuildArgs A, const int* pts,
                                                        const int* pts_off, const int* cands, const int* cand_off,
                                                        const double* p64, const double* cand64,
                                                        const double* cand_sq, int stride, const IdxT* list,
                                                        const int* cnt, int* parent_pos,
                                                        unsigned long long* prof, const float* list_d2 = nullptr,
                                                        const float* thr = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int s_keep[NV_W][NF_CAP];   // the listed candidates inside the final window (list_d2 given)
  const int b = blockIdx.y;
  const int t = A.trees[b];
  const int L = F.meta[t].levels;
  if (L < 2) return;
  const int e = blockIdx.x * NV_W + warp;
  const int npts = pts_off[(size_t)b * 64 + L];
  if (e >= npts) return;
  // per warp: the point row (broadcast) and two NV_R-candidate x 32-coordinate
  // chunks of candidate rows (cp.async double buffer over the flattened
  // (round of NV_R candidates, coordinate chunk) sequence); every lane runs one
  // candidate's sequential chain through the chunks, acc in its register
  extern __shared__ double nv_smem[];
  double* p = nv_smem + warp * (ICB_DPAD + 1);
  double (*T)[NV_R][33] = reinterpret_cast<double (*)[NV_R][33]>(nv_smem + NV_W * (ICB_DPAD + 1)) + warp * 2;
  const int D1 = F.dim + 1;
  const double* src = p64 + ((size_t)b * A.n_points + e) * (ICB_DPAD + 1);
  for (int u = lane; u < D1; u += 32) p[u] = src[u];
  int lv = 1;
  while (lv < L - 1 && pts_off[(size_t)b * 64 + lv + 1] <= e) ++lv;
  const int c0 = cand_off[(size_t)b * 64 + lv];
  const int nc = cand_off[(size_t)b * 64 + lv + 1] - c0;
  const int c = cnt[(size_t)b * A.n_points + e];
  const bool all = c > NF_CAP;   // overflowed windows: nn_parent_kernel's shared tiles do those points
  int m = all ? 0 : c;
  const double* c64base = cand64 + ((size_t)b * stride + c0) * (ICB_DPAD + 1);
  const IdxT* lst = list + ((size_t)b * A.n_points + e) * NF_CAP;
  // The tensor-core filter lists against a running minimum; with its d2~ per
  // entry and the row's final threshold, only the entries inside the final
  // window need the exact chain (the argmin and its ties are among them).
  const bool pruned = list_d2 != nullptr && !all;
  if (pruned) {
    const float th = thr[(size_t)b * A.n_points + e];
    const float* ld = list_d2 + ((size_t)b * A.n_points + e) * NF_CAP;
    int mm = 0;
    for (int i0 = 0; i0 < m; i0 += 32) {
      const int i = i0 + lane;
      const bool keep = i < m && ld[i] <= th;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) s_keep[warp][mm + __popc(bal & ((1u << lane) - 1))] = (int)lst[i];
      mm += __popc(bal);
    }
    __syncwarp();
    m = mm;
  }
  if (prof && lane == 0) {
    atomicAdd(prof + 0, 1ull);
    atomicAdd(prof + 1, (unsigned long long)m);
    atomicAdd(prof + 2, all ? 1ull : 0ull);
  }
  double best = 0.0;
  int arg = -1;
  // chunks of 32 coordinates; a final remainder of 1 joins the last chunk (33 wide)
  const int nch = D1 > 32 && D1 % 32 == 1 ? D1 >> 5 : (D1 + 31) >> 5;
  auto chunk_w = [&](int ch) { return ch == nch - 1 ? D1 - ch * 32 : 32; };
  const int steps = (m + NV_R - 1) / NV_R * nch;
  auto cand = [&](int rd) -> int {
    const int i = rd * NV_R + lane;
    return lane < NV_R && i < m ? (all ? i : pruned ? s_keep[warp][i] : (int)lst[i]) : 0;
  };
  auto issue = [&](int st) {
    const int rd = st / nch, u0 = (st - rd * nch) * 32;
    const int nr = min(NV_R, m - rd * NV_R), un = chunk_w(st - rd * nch);
    const int jl = cand(rd);
    double (*B)[33] = T[st & 1];
    for (int r = 0; r < nr; ++r) {
      const int j = __shfl_sync(0xffffffffu, jl, r);
      const double* row = c64base + (size_t)j * (ICB_DPAD + 1) + u0;
      if (lane < un)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(&B[r][lane])), "l"(row + lane));
      if (lane == 0 && un == 33)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(&B[r][32])), "l"(row + 32));
    }
    asm volatile("cp.async.commit_group;\n");
  };
  if (steps > 0) issue(0);
  int jr = cand(0);
  double acc = 0.0;
  for (int st = 0; st < steps; ++st) {
    if (st + 1 < steps) {
      issue(st + 1);
      asm volatile("cp.async.wait_group 1;\n");
    } else {
      asm volatile("cp.async.wait_group 0;\n");
    }
    __syncwarp();
    const int rd = st / nch, ch = st - rd * nch, u0 = ch * 32;
    const int nr = min(NV_R, m - rd * NV_R), un = chunk_w(ch);
    if (ch == 0) { acc = 0.0; jr = cand(rd); }
    const double (*B)[33] = T[st & 1];
    if (lane < nr) {
      if (un == 32) {
#pragma unroll
        for (int u = 0; u < 32; ++u) acc = __fma_rn(p[u0 + u], B[lane][u], acc);
      } else {
        for (int u = 0; u < un; ++u) acc = __fma_rn(p[u0 + u], B[lane][u], acc);
      }
      if (ch == nch - 1)
        nn_better(__dsub_rn(cand_sq[(size_t)b * stride + c0 + jr], __dmul_rn(2.0, acc)), jr, best, arg);
    }
    __syncwarp();   // buffer st & 1 is refilled by issue(st + 2)
  }
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (oa >= 0) nn_better(ob, oa, best, arg);
  }
  if (lane == 0 && arg >= 0)
    parent_pos[(size_t)b * A.n_points + pts[(size_t)b * A.n_points + e]] = cands[(size_t)b * A.n_points + c0 + arg];
}

// Block: NF_BM point entries x all candidates of their level, NF_BN at a time;
// 8 warps = 4 (16 rows) x 2 (64 candidates).
template <typename IdxT>
__global__ void __launch_bounds__(256, 2) nn_filter_kernel(ForestView F, BuildArgs A, const int* pts_off,
                                                          const int* cand_off, const __half* p16,
                                                          const __half* c16, const double* cand_sq, int stride,
                                                          IdxT* list, int* cnt) {
  extern __shared__ __align__(16) unsigned char nf_raw[];
  NfSmem& S = *reinterpret_cast<NfSmem*>(nf_raw);
  const int b = blockIdx.y;
  const int t = A.trees[b];
  const int L = F.meta[t].levels;
  if (L < 2) return;
  const int npts = pts_off[(size_t)b * 64 + L];
  const int e0 = blockIdx.x * NF_BM;
  if (e0 >= npts) return;
  const int e1 = min(npts, e0 + NF_BM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp & 3, wn = warp >> 2;
  for (int e = e0 + tid; e < e0 + NF_BM; e += blockDim.x) {
    int lv = -1;
    if (e < e1) {
      lv = 1;
      while (lv < L - 1 && pts_off[(size_t)b * 64 + lv + 1] <= e) ++lv;
    }
    S.lv[e - e0] = lv;
  }
  // A tile (rows past e1 repeat the last row; masked below)
  for (int x = tid; x < NF_BM * (NF_K / 8); x += blockDim.x) {
    const int r = x / (NF_K / 8), ch = x % (NF_K / 8);
    const int e = min(e0 + r, e1 - 1);
    cp_async16(&S.a[r][ch * 8], p16 + ((size_t)b * A.n_points + e) * NF_K + ch * 8);
  }
  asm volatile("cp.async.commit_group;\n");
  __syncthreads();
  const __half* cbase = c16 + (size_t)b * stride * NF_K;
  const double* sqbase = cand_sq + (size_t)b * stride;
  // rows of this thread's fragments: r_lo = wm*16 + lane/4, r_hi = r_lo + 8
  const int r_lo = wm * 16 + (lane >> 2), r_hi = r_lo + 8;
  int seg = e0;
  while (seg < e1) {
    const int lv = S.lv[seg - e0];
    int segend = seg;
    while (segend < e1 && S.lv[segend - e0] == lv) ++segend;
    const int c0 = cand_off[(size_t)b * 64 + lv];
    const int nc = cand_off[(size_t)b * 64 + lv + 1] - c0;
    const int ntile = (nc + NF_BN - 1) / NF_BN;
    if (ntile == 0) { seg = segend; continue; }
    __syncthreads();
    for (int x = tid; x < NF_BM; x += blockDim.x) {
      S.rmin[x] = INT_MAX;
      S.cnt[x] = 0;
    }
    auto stage = [&](int tile, int buf) {
      const int j0 = tile * NF_BN;
      for (int x = tid; x < NF_BN * (NF_K / 8); x += blockDim.x) {
        const int r = x / (NF_K / 8), ch = x % (NF_K / 8);
        const int j = min(j0 + r, nc - 1);
        cp_async16(&S.bt[buf][r][ch * 8], cbase + (size_t)(c0 + j) * NF_K + ch * 8);
      }
      for (int x = tid; x < NF_BN; x += blockDim.x)
        S.csq[buf][x] = j0 + x < nc ? (float)sqbase[c0 + j0 + x] : 0.f;
      asm volatile("cp.async.commit_group;\n");
    };
    const bool ok_lo = e0 + r_lo >= seg && e0 + r_lo < segend;
    const bool ok_hi = e0 + r_hi >= seg && e0 + r_hi < segend;
    for (int pass = 0; pass < 2; ++pass) {
      float thr_lo = 0.f, thr_hi = 0.f;
      if (pass == 1) {
        thr_lo = ord2f(S.rmin[r_lo]) + NF_WINDOW;
        thr_hi = ord2f(S.rmin[r_hi]) + NF_WINDOW;
      }
      float m_lo = INFINITY, m_hi = INFINITY;
      __syncthreads();
      stage(0, 0);
      for (int tile = 0; tile < ntile; ++tile) {
        const int buf = tile & 1;
        if (tile + 1 < ntile) {
          stage(tile + 1, buf ^ 1);
          asm volatile("cp.async.wait_group 1;\n");
        } else {
          asm volatile("cp.async.wait_group 0;\n");
        }
        __syncthreads();
        float acc[8][4];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
        const int mi = lane >> 3, ri = lane & 7;
#pragma unroll
        for (int k0 = 0; k0 < NF_K; k0 += 16) {
          unsigned a[4];
          ldsm_x4(smem_u32(&S.a[wm * 16 + ri + 8 * (mi & 1)][k0 + 8 * (mi >> 1)]), a[0], a[1], a[2], a[3]);
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            unsigned b0, b1, b2, b3;
            ldsm_x4(smem_u32(&S.bt[buf][wn * 64 + (q + (mi >> 1)) * 8 + ri][k0 + 8 * (mi & 1)]), b0, b1, b2, b3);
            mma16816(acc[q], a, b0, b1);
            mma16816(acc[q + 1], a, b2, b3);
          }
        }
        const int jt = tile * NF_BN;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jl = wn * 64 + q * 8 + 2 * (lane & 3) + h;
            const int j = jt + jl;
            const float cs = S.csq[buf][jl];
            const float d_lo = cs - 2.f * acc[q][h], d_hi = cs - 2.f * acc[q][2 + h];
            if (pass == 0) {
              if (j < nc) {
                m_lo = fminf(m_lo, d_lo);
                m_hi = fminf(m_hi, d_hi);
              }
            } else {
              if (j < nc && ok_lo && d_lo <= thr_lo) {
                const int k = atomicAdd(&S.cnt[r_lo], 1);
                if (k < NF_CAP) list[((size_t)b * A.n_points + e0 + r_lo) * NF_CAP + k] = (IdxT)j;
              }
              if (j < nc && ok_hi && d_hi <= thr_hi) {
                const int k = atomicAdd(&S.cnt[r_hi], 1);
                if (k < NF_CAP) list[((size_t)b * A.n_points + e0 + r_hi) * NF_CAP + k] = (IdxT)j;
              }
            }
          }
        }
        __syncthreads();   // buffer `buf` is restaged by the next iteration
      }
      if (pass == 0) {
        m_lo = fminf(m_lo, __shfl_xor_sync(0xffffffffu, m_lo, 1));
        m_lo = fminf(m_lo, __shfl_xor_sync(0xffffffffu, m_lo, 2));
        m_hi = fminf(m_hi, __shfl_xor_sync(0xffffffffu, m_hi, 1));
        m_hi = fminf(m_hi, __shfl_xor_sync(0xffffffffu, m_hi, 2));
        if ((lane & 3) == 0) {
          atomicMin(&S.rmin[r_lo], f2ord(m_lo));
          atomicMin(&S.rmin[r_hi], f2ord(m_hi));
        }
      }
    }
    __syncthreads();
    if (tid < NF_BM && e0 + tid >= seg && e0 + tid < segend) cnt[(size_t)b * A.n_points + e0 + tid] = S.cnt[tid];
    seg = segend;
  }
}

// ---------------------------------------------------------------- K3 nodes
// entry key: tree(12) | (63 - lv)(6) | firstpos(23) | pos(23)
__device__ __forceinline__ unsigned long long node_key(int b, int lv, int fp, int pos) {
  return ((unsigned long long)b << 52) | ((unsigned long long)(63 - lv) << 46) |
         ((unsigned long long)fp << 23) | (unsigned long long)pos;
}

__global__ void build_firstpos_kernel(ForestView F, BuildArgs A, const int* top, const int* parent_pos,
                                      const int* own_base_pos, int* firstpos) {
  int b = blockIdx.y;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_points) return;
  int t = A.trees[b];
  int L = F.meta[t].levels;
  int T = top[(size_t)b * A.n_points + i];
  for (int lv = 1; lv <= T && lv < L; ++lv) {
    int owner = (T == lv) ? parent_pos[(size_t)b * A.n_points + i] : i;
    int slot = own_base_pos[(size_t)b * A.n_points + owner] + lv - 1;
    atomicMin(firstpos + (size_t)b * A.n_points + slot, i);
  }
}

__global__ void build_entries_kernel(ForestView F, BuildArgs A, const int* top, const int* parent_pos,
                                     const int* own_base_pos, const int* firstpos,
                                     const int* ent_base, unsigned long long* keys) {
  int b = blockIdx.y;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_points) return;
  int t = A.trees[b];
  int L = F.meta[t].levels;
  size_t e = (size_t)b * A.n_points + i;
  int T = top[e];
  int out = ent_base[e];
  for (int lv = 1; lv <= T; ++lv) {
    int fp = 0;
    if (lv < L) {
      int owner = (T == lv) ? parent_pos[e] : i;
      fp = firstpos[(size_t)b * A.n_points + own_base_pos[(size_t)b * A.n_points + owner] + lv - 1];
    }
    keys[out++] = node_key(b, lv, fp, i);
  }
}

// Total entries on the device (no host round trip): padding entries of the
// bound-sized arrays hold ~0 keys and sort last.
__global__ void build_ent_total_kernel(ForestView F, BuildArgs A, const int* ent_base, const int* top, int n_max,
                                       int* n_ent) {
  const size_t last = (size_t)A.n * A.n_points - 1;
  const int tot = ent_base[last] + top[last];
  *n_ent = min(tot, n_max);
  if (tot > n_max)
    for (int b = 0; b < A.n; ++b) set_err(F.meta + A.trees[b], ICB_ERR_CAP_SCRATCH);
}

__global__ void build_flags_kernel(const unsigned long long* keys, int n, int* flags) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  flags[j] = (j == 0 || (keys[j] >> 23) != (keys[j - 1] >> 23)) ? 1 : 0;
}

// gid = inclusive scan of flags; tree_ent0[b] = first entry of tree b
__global__ void build_nodes_kernel(ForestView F, BuildArgs A, const unsigned long long* keys, const int* n_ent_dev,
                                   const int* gid, const int* tree_ent0, const int* top,
                                   const int* own_base_pos) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *n_ent_dev) return;
  unsigned long long k = keys[j];
  int b = (int)(k >> 52);
  int lv = 63 - (int)((k >> 46) & 63);
  int pos = (int)(k & 0x7fffff);
  int t = A.trees[b];
  int g = gid[j] - 1;
  int tok = A.tokens[(size_t)b * A.n_points + pos];
  int local = j - tree_ent0[b];
  if (local >= F.member_cap) { set_err(F.meta + t, ICB_ERR_CAP_MEMBERS); return; }
  F.mem(t)[local] = tok;
  // node-local id needs tree_node0 of this tree: gid at tree_ent0[b]
  int node = g - (gid[tree_ent0[b]] - 1);
  if (node >= F.node_cap) { set_err(F.meta + t, ICB_ERR_CAP_NODES); return; }
  bool boundary = (j == 0) || ((keys[j - 1] >> 23) != (k >> 23));
  if (boundary) {
    F.node_off[F.nd(t, node)] = local;
    F.node_level[F.nd(t, node)] = lv;
    F.node_lastpage[F.nd(t, node)] = -1;
    F.node_dirs[F.nd(t, node)] = -1;
    if (lv == F.meta[t].levels) { F.node_owner[F.nd(t, node)] = ICB_ROOT_OWNER; F.node_parent[F.nd(t, node)] = -1; }
  }
  int T = top[(size_t)b * A.n_points + pos];
  if (lv < F.meta[t].levels && T > lv) {   // this member owns the node
    F.node_owner[F.nd(t, node)] = tok;
    F.node_opos[F.nd(t, node)] = local;   // absolute here; made node-relative by build_summary_kernel
    F.own_list[(size_t)t * F.own_cap + own_base_pos[(size_t)b * A.n_points + pos] + lv - 1] = node;
    if (lv == 1) F.own1[F.tk(t, tok)] = node;
  }
  // node size: count members
  atomicAdd(F.node_size + F.nd(t, node), 1);
}

__global__ void build_tree_totals_kernel(ForestView F, BuildArgs A, const int* gid, const int* tree_ent0,
                                         const int* ent_cnt) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= A.n) return;
  int t = A.trees[b];
  int j0 = tree_ent0[b], j1 = j0 + ent_cnt[b] - 1;
  int n_nodes = gid[j1] - gid[j0] + 1;
  F.meta[t].n_nodes = n_nodes;
  F.meta[t].member_top = ent_cnt[b];
  if (n_nodes > F.node_cap) set_err(F.meta + t, ICB_ERR_CAP_NODES);
}

// node parents + capacities; leaves' page counts.
// parent(node at lv owned by X) = node containing X at lv+1: X's own node
// there if X reaches above lv+1, else the node X joined at its top level,
// i.e. own(parent_of[X], lv+1), or the top node when lv+1 == L.
__global__ void build_parents_kernel(ForestView F, BuildArgs A, int max_nodes, const int* parent_pos,
                                     int* leaf_pages) {
  int b = blockIdx.y;
  int node = blockIdx.x * blockDim.x + threadIdx.x;
  int t = A.trees[b];
  int nn = min(F.meta[t].n_nodes, F.node_cap);
  if (node >= max_nodes) return;
  int np = 0;
  if (node < nn) {
    size_t x = F.nd(t, node);
    F.node_capm[x] = F.node_size[x];
    int lv = F.node_level[x];
    int L = F.meta[t].levels;
    if (lv < L) {
      int X = F.node_owner[x];
      int TX = F.level[F.tk(t, X)];
      int par;
      if (TX > lv + 1) {
        par = F.own(t, X, lv + 1);
      } else if (lv + 1 == L) {
        par = F.meta[t].top_node;
      } else {
        int px = parent_pos[(size_t)b * A.n_points + A.pos_of[(size_t)b * F.tok_cap + X]];
        par = F.own(t, A.tokens[(size_t)b * A.n_points + px], lv + 1);
      }
      F.node_parent[x] = par;
    }
    if (lv == 1) np = (F.node_size[x] + F.s - 1) / F.s;
  }
  leaf_pages[(size_t)b * max_nodes + node] = np;
}

// K4: pages.  leaf_first = exclusive scan over (tree, node) of leaf page counts.
__global__ void build_pages_kernel(ForestView F, BuildArgs A, int max_nodes, const int* leaf_first,
                                   const int* leaf_total) {
  int b = blockIdx.y;
  int node = blockIdx.x;
  int t = A.trees[b];
  if (node >= min(F.meta[t].n_nodes, F.node_cap)) return;
  size_t x = F.nd(t, node);
  if (F.node_level[x] != 1) return;
  const int base = F.meta[t].next_page;   // read before the totals kernel updates it
  const int first = base + leaf_first[(size_t)b * max_nodes + node] - leaf_first[(size_t)b * max_nodes];
  const int off = F.node_off[x], sz = F.node_size[x];
  const int np = (sz + F.s - 1) / F.s;
  if (first + np > F.page_cap) { if (threadIdx.x == 0) set_err(F.meta + t, ICB_ERR_CAP_PAGES); return; }
  if (threadIdx.x == 0) F.node_lastpage[x] = first + np - 1;
  for (int p = threadIdx.x; p < np; p += blockDim.x) {
    F.page_fill[F.pg(t, first + p)] = min(F.s, sz - p * F.s);
    F.page_role[F.pg(t, first + p)] = ICB_ROLE_INDEXED;
  }
  const int* mem = F.mem(t);
  const int P = A.n_points;
  // member u -> page first + u/s, slot u%s.  K/V copy: one warp per member.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int u = warp; u < sz; u += nw) {
    int tok = mem[off + u];
    int page = first + u / F.s, slot = u % F.s;
    if (lane == 0) {
      F.page_tok[F.pg(t, page) * F.s + slot] = tok;
      F.tok2page[F.tk(t, tok)] = page;
    }
    // input position of tok: stored in tok2page scratch? use A.pos_of (token -> pos map)
    int pos = A.pos_of[(size_t)b * F.tok_cap + tok];
    const float* kin = A.keys + ((size_t)b * P + pos) * F.dim;
    const float* vin = A.values ? A.values + ((size_t)b * P + pos) * F.dim_v : nullptr;
    size_t kslot = (F.pg(t, page) * F.s + slot);
    // lane l writes dims 4l..4l+3 (row strides are multiples of 4; padding
    // stays zero): one 8- or 16-byte store per lane, one contiguous row per
    // warp store -- few, large writes also when the store is host memory
    const int j0 = lane * 4;
    float k4[4], v4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      k4[u] = j0 + u < F.dim ? kin[j0 + u] : 0.f;
      v4[u] = (vin && j0 + u < F.dim_v) ? vin[j0 + u] : 0.f;
    }
    if (F.kv_bf16) {
      __nv_bfloat16* K = (__nv_bfloat16*)F.page_k + kslot * F.dkp;
      __nv_bfloat16* V = (__nv_bfloat16*)F.page_v + kslot * F.dvp;
      __nv_bfloat162 k01 = __floats2bfloat162_rn(k4[0], k4[1]), k23 = __floats2bfloat162_rn(k4[2], k4[3]);
      __nv_bfloat162 v01 = __floats2bfloat162_rn(v4[0], v4[1]), v23 = __floats2bfloat162_rn(v4[2], v4[3]);
      if (j0 < F.dkp)
        *reinterpret_cast<uint2*>(K + j0) = make_uint2(*reinterpret_cast<unsigned*>(&k01), *reinterpret_cast<unsigned*>(&k23));
      if (j0 < F.dvp)
        *reinterpret_cast<uint2*>(V + j0) = make_uint2(*reinterpret_cast<unsigned*>(&v01), *reinterpret_cast<unsigned*>(&v23));
    } else {
      float* K = (float*)F.page_k + kslot * F.dkp;
      float* V = (float*)F.page_v + kslot * F.dvp;
      if (j0 < F.dkp) *reinterpret_cast<float4*>(K + j0) = make_float4(k4[0], k4[1], k4[2], k4[3]);
      if (j0 < F.dvp) *reinterpret_cast<float4*>(V + j0) = make_float4(v4[0], v4[1], v4[2], v4[3]);
    }
  }
  (void)leaf_total;
}

__global__ void build_pos_of_kernel(ForestView F, BuildArgs A) {
  int b = blockIdx.y;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_points) return;
  int tok = A.tokens[(size_t)b * A.n_points + i];
  if (tok >= 0 && tok < F.tok_cap) A.pos_of[(size_t)b * F.tok_cap + tok] = i;
}

__global__ void build_page_totals_kernel(ForestView F, BuildArgs A, int max_nodes, const int* leaf_first,
                                         const int* leaf_pages) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= A.n) return;
  int t = A.trees[b];
  size_t last = (size_t)b * max_nodes + max_nodes - 1;
  int total = leaf_first[last] + leaf_pages[last] - leaf_first[(size_t)b * max_nodes];
  F.meta[t].next_page += total;
  if (F.meta[t].next_page > F.page_cap) set_err(F.meta + t, ICB_ERR_CAP_PAGES);
}

// Level summary of a freshly built tree (TreeMeta.lvl_count / lvl_maxnode /
// upper, read by the search's start level): one CTA per tree.
__global__ void __launch_bounds__(256) build_summary_kernel(ForestView F, BuildArgs A) {
  const int b = blockIdx.x, t = A.trees[b];
  TreeMeta* m = F.meta + t;
  __shared__ int cnt[ICB_LV_TRACK], mx[ICB_LV_TRACK], nup, ovf;
  if (threadIdx.x < ICB_LV_TRACK) { cnt[threadIdx.x] = 0; mx[threadIdx.x] = 0; }
  if (threadIdx.x == 0) { nup = 0; ovf = 0; }
  __syncthreads();
  int* up = F.upl(t);
  for (int i = threadIdx.x; i < A.n_points; i += blockDim.x) {
    const int tok = A.tokens[(size_t)b * A.n_points + i];
    if (tok < 0 || tok >= F.tok_cap) continue;
    const int lv = F.level[F.tk(t, tok)];
    if (lv >= ICB_LV_TRACK) { ovf = 1; continue; }
    atomicAdd(&cnt[lv], 1);
    if (lv >= 2) {
      const int pos = atomicAdd(&nup, 1);
      if (pos < F.upper_cap) up[pos] = tok; else ovf = 1;
    }
  }
  for (int x = threadIdx.x; x < min(m->n_nodes, F.node_cap); x += blockDim.x) {
    const int lv = F.node_level[F.nd(t, x)];
    const size_t nx = F.nd(t, x);
    F.node_opos[nx] = F.node_owner[nx] >= 0 ? F.node_opos[nx] - F.node_off[nx] : -1;
    if (lv < ICB_LV_TRACK) atomicMax(&mx[lv], F.node_size[F.nd(t, x)]);
  }
  __syncthreads();
  if (threadIdx.x < ICB_LV_TRACK) { m->lvl_count[threadIdx.x] = cnt[threadIdx.x]; m->lvl_maxnode[threadIdx.x] = mx[threadIdx.x]; }
  if (threadIdx.x == 0) { m->n_upper = min(nup, F.upper_cap); m->lv_ovf = ovf; }
}

}  // namespace icb

#include "nn_tc.cuh"

// ---------------------------------------------------------------- host driver
using namespace icb;

int icb_build_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t n_points, const int32_t* tokens,
                   const float* keys, const float* values, const double* scales, cudaStream_t st) {
  ForestView F = f->view;
  const int P = n_points;
  BuildArgs A{};
  A.trees = trees; A.n = n; A.n_points = P; A.tokens = tokens; A.keys = keys; A.values = values;
  A.scales = scales;
  // scratch
  Scratch S(st);
  {
    // keep build scratch mapped between calls (a prefill issues several builds)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      unsigned long long thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  double* nsq = S.alloc<double>((size_t)n * P);
  unsigned long long* maxbits = S.alloc<unsigned long long>(n);
  int* top = S.alloc<int>((size_t)n * P);
  unsigned long long* occ = S.alloc<unsigned long long>(n);
  int* own_base_pos = S.alloc<int>((size_t)n * P);
  int* pts = S.alloc<int>((size_t)n * P);
  int* cands = S.alloc<int>((size_t)n * P);
  int* pts_off = S.alloc<int>((size_t)n * 64);
  int* cand_off = S.alloc<int>((size_t)n * 64);
  int* ent_cnt = S.alloc<int>(n);
  int* parent_pos = S.alloc<int>((size_t)n * P);
  int* pos_of = S.alloc<int>((size_t)n * F.tok_cap);
  A.pos_of = pos_of;
  if (!S.ok()) return S.fail();
  ICB_CUDA(cudaMemsetAsync(maxbits, 0, sizeof(unsigned long long) * n, st));
  ICB_CUDA(cudaMemsetAsync(cand_off, 0, sizeof(int) * n * 64, st));
  ICB_CUDA(cudaMemsetAsync(pts_off, 0, sizeof(int) * n * 64, st));
  dim3 g8((P + 7) / 8, n);
  build_norms_kernel<<<g8, 256, 0, st>>>(F, A, nsq, maxbits);
  build_scale_kernel<<<(n + 127) / 128, 128, 0, st>>>(F, A, maxbits);
  build_lift_kernel<<<g8, 256, 0, st>>>(F, A, nsq);
  build_levels_kernel<1024><<<n, 1024, 0, st>>>(F, A, top, occ);
  dim3 g256((P + 255) / 256, n);
  build_compact_kernel<<<g256, 256, 0, st>>>(F, A, top, occ);
  build_pos_of_kernel<<<g256, 256, 0, st>>>(F, A);
  build_lists_kernel<1024><<<n, 1024, 0, st>>>(F, A, top, own_base_pos, pts, pts_off, cands, cand_off,
                                               ent_cnt);
  // candidate fp64 rows: sum_lv |top > lv| = own_top <= P (own entries == sum(top-1))
  int stride = P;
  double* cand64 = S.alloc<double>((size_t)n * stride * (ICB_DPAD + 1));
  double* cand_sq = S.alloc<double>((size_t)n * stride);
  if (!S.ok()) return S.fail();
  build_cand64_kernel<<<dim3((stride + 7) / 8, n), 256, 0, st>>>(F, A, nsq, cands, cand_off, cand64,
                                                                 cand_sq, stride);
  static const bool exact_only = getenv("ICB_BUILD_EXACT_NN") != nullptr;   // A/B and test knob
  static const bool f16_filter = getenv("ICB_BUILD_F16_FILTER") != nullptr;  // round-1 filter, A/B
  const int D1 = F.dim + 1, PS = D1 | 1;
  const size_t psm = sizeof(double) * (NN_BM * PS + NN_BN * (NN_KC + 1));
  // exact argmin of the listed candidates; points whose window overflowed
  // NF_CAP: the brute-force tiled kernel, restricted to blocks that contain one
  auto verify = [&](auto* list, const double* p64, int* nf_cnt, const float* list_d2 = nullptr,
                    const float* thr = nullptr) -> int {
    using IdxT = typename std::remove_pointer<decltype(list)>::type;
    unsigned long long* prof = nullptr;
    if (getenv("ICB_PROF")) ICB_CUDA(cudaGetSymbolAddress((void**)&prof, g_build_prof));
    const int nv_sm = (int)sizeof(double) * (NV_W * (ICB_DPAD + 1) + NV_W * 2 * NV_R * 33);
    ICB_CUDA(cudaFuncSetAttribute(nn_verify_kernel<IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize, nv_sm));
    nn_verify_kernel<IdxT><<<dim3((P + NV_W - 1) / NV_W, n), NV_W * 32, nv_sm, st>>>(
        F, A, pts, pts_off, cands, cand_off, p64, cand64, cand_sq, stride, list, nf_cnt, parent_pos, prof, list_d2,
        thr);
    ICB_CUDA(cudaFuncSetAttribute(nn_parent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
    nn_parent_kernel<<<dim3((P + NN_BM - 1) / NN_BM, n), 256, psm, st>>>(
        F, A, nsq, pts, pts_off, cands, cand_off, cand64, cand_sq, stride, parent_pos, nf_cnt, NF_CAP);
    return ICB_OK;
  };
  if (exact_only || D1 > TC_KB || (f16_filter && (D1 > NF_K || P > 98304))) {
    ICB_CUDA(cudaFuncSetAttribute(nn_parent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
    nn_parent_kernel<<<dim3((P + NN_BM - 1) / NN_BM, n), 256, psm, st>>>(
        F, A, nsq, pts, pts_off, cands, cand_off, cand64, cand_sq, stride, parent_pos);
  } else if (!f16_filter) {
    // exact-integer tensor-core filter (tcgen05 kind::i8, nn_tc.cuh), any size
    const size_t a_rows = (size_t)(P + TC_M - 1) / TC_M * TC_M;
    const size_t b_tiles = (size_t)(stride + TC_N - 1) / TC_N + 64;   // + one partial tile per level
    double* p64 = S.alloc<double>((size_t)n * P * (ICB_DPAD + 1));
    signed char* aimg = S.alloc<signed char>((size_t)n * a_rows * TC_AROW);
    signed char* bimg = S.alloc<signed char>((size_t)n * b_tiles * TC_BTILE);
    double* pmeta = S.alloc<double>((size_t)n * P * 3);
    float2* cmeta = S.alloc<float2>((size_t)n * b_tiles * TC_N);
    unsigned long long* cmax = S.alloc<unsigned long long>((size_t)n * 2);
    int* ct_off = S.alloc<int>((size_t)n * 64);
    int* nf_cnt = S.alloc<int>((size_t)n * P);
    float* nf_d2 = S.alloc<float>((size_t)n * P * NF_CAP);   // d2~ of each listed candidate
    float* nf_thr = S.alloc<float>((size_t)n * P);           // each row's final window threshold
    if (!S.ok()) return S.fail();
    ICB_CUDA(cudaMemsetAsync(aimg, 0, (size_t)n * a_rows * TC_AROW, st));
    ICB_CUDA(cudaMemsetAsync(bimg, 0, (size_t)n * b_tiles * TC_BTILE, st));
    ICB_CUDA(cudaMemsetAsync(cmeta, 0xff, sizeof(float2) * n * b_tiles * TC_N, st));   // NaN: padding never listed
    ICB_CUDA(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * n * 2, st));
    ICB_CUDA(cudaMemsetAsync(nf_cnt, 0, sizeof(int) * n * P, st));   // window hits are counted atomically
    tc_tile_offsets_kernel<<<n, 32, 0, st>>>(F, A, cand_off, ct_off);
    tc_prep_points_kernel<<<dim3((P + 7) / 8, n), 256, 0, st>>>(F, A, nsq, pts, pts_off, p64, aimg, a_rows,
                                                               pmeta);
    tc_prep_cands_kernel<<<dim3((stride + 7) / 8, n), 256, 0, st>>>(F, A, cand_off, ct_off, cand64, cand_sq,
                                                                    stride, bimg, b_tiles, cmeta, cmax);
    auto run = [&](auto* list) -> int {
      using IdxT = typename std::remove_pointer<decltype(list)>::type;
      const int sm = TC_STAGES * TC_BTILE + 1024;
      ICB_CUDA(cudaFuncSetAttribute(nn_tc_filter_kernel<IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      nn_tc_filter_kernel<IdxT><<<dim3((unsigned)(a_rows / TC_M), n), TC_THREADS, sm, st>>>(
          F, A, pts_off, cand_off, ct_off, aimg, a_rows, bimg, b_tiles, pmeta, cmeta, cmax, list, nf_cnt, nf_d2,
          nf_thr);
      return verify(list, p64, nf_cnt, nf_d2, nf_thr);
    };
    int rc;
    if (P <= 65536) {
      unsigned short* l16 = S.alloc<unsigned short>((size_t)n * P * NF_CAP);
      if (!S.ok()) return S.fail();
      rc = run(l16);
    } else {
      int* l32 = S.alloc<int>((size_t)n * P * NF_CAP);
      if (!S.ok()) return S.fail();
      rc = run(l32);
    }
    if (rc != ICB_OK) return rc;
  } else {
    // round-1 f16 filter (mma.sync), kept for A/B: ICB_BUILD_F16_FILTER=1
    double* p64 = S.alloc<double>((size_t)n * P * (ICB_DPAD + 1));
    __half* p16 = S.alloc<__half>((size_t)n * P * NF_K);
    __half* c16 = S.alloc<__half>((size_t)n * stride * NF_K);
    int* nf_cnt = S.alloc<int>((size_t)n * P);
    if (!S.ok()) return S.fail();
    nn_half_kernel<<<dim3((P + 7) / 8, n), 256, 0, st>>>(F, A, nsq, pts, pts_off, cand64, cand_off, stride, p64,
                                                         p16, c16);
    // candidate indices of a level are < P: 16-bit lists when they fit
    auto run = [&](auto* list) -> int {
      using IdxT = typename std::remove_pointer<decltype(list)>::type;
      const int sm = (int)sizeof(NfSmem);
      ICB_CUDA(cudaFuncSetAttribute(nn_filter_kernel<IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      nn_filter_kernel<IdxT><<<dim3((P + NF_BM - 1) / NF_BM, n), 256, sm, st>>>(
          F, A, pts_off, cand_off, p16, c16, cand_sq, stride, list, nf_cnt);
      return verify(list, p64, nf_cnt);
    };
    int rc;
    if (P <= 65536) {
      unsigned short* l16 = S.alloc<unsigned short>((size_t)n * P * NF_CAP);
      if (!S.ok()) return S.fail();
      rc = run(l16);
    } else {
      int* l32 = S.alloc<int>((size_t)n * P * NF_CAP);
      if (!S.ok()) return S.fail();
      rc = run(l32);
    }
    if (rc != ICB_OK) return rc;
  }
  // node construction
  int* firstpos = S.alloc<int>((size_t)n * P);
  int* ent_base = S.alloc<int>((size_t)n * P);
  if (!S.ok()) return S.fail();
  ICB_CUDA(cudaMemsetAsync(firstpos, 0x7f, sizeof(int) * (size_t)n * P, st));
  build_firstpos_kernel<<<g256, 256, 0, st>>>(F, A, top, parent_pos, own_base_pos, firstpos);
  // entry offsets: exclusive scan of top over all (b, i)
  {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, top, ent_base, n * P, st);
    void* d_tmp = S.alloc<char>(tmp);
    if (!S.ok()) return S.fail();
    cub::DeviceScan::ExclusiveSum(d_tmp, tmp, top, ent_base, n * P, st);
  }
  // Entries: arrays sized by a bound, the true count stays on the device (no
  // host synchronisation: a build can overlap the caller's work).  Levels
  // beyond the first are geometric(r): their sum concentrates far below twice
  // its mean; a count above the bound sets ICB_ERR_CAP_SCRATCH.
  const double rr = f->cfg.promotion_ratio;
  const size_t np_ = (size_t)n * P;
  const int n_ent = (int)std::min<double>(2.0e9, (double)np_ + std::ceil(2.0 * (double)np_ * rr / (1.0 - rr)) + 4096);
  int* n_ent_dev = S.alloc<int>(1);
  if (!S.ok()) return S.fail();
  build_ent_total_kernel<<<1, 1, 0, st>>>(F, A, ent_base, top, n_ent, n_ent_dev);
  unsigned long long* keys_in = S.alloc<unsigned long long>(n_ent);
  unsigned long long* keys_out = S.alloc<unsigned long long>(n_ent);
  int* flags = S.alloc<int>(n_ent);
  int* gid = S.alloc<int>(n_ent);
  int* tree_ent0 = S.alloc<int>(n);
  if (!S.ok()) return S.fail();
  ICB_CUDA(cudaMemsetAsync(keys_in, 0xff, sizeof(unsigned long long) * (size_t)n_ent, st));   // padding sorts last
  build_entries_kernel<<<g256, 256, 0, st>>>(F, A, top, parent_pos, own_base_pos, firstpos, ent_base, keys_in);
  {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys_in, keys_out, n_ent, 0, 64, st);
    void* d_tmp = S.alloc<char>(tmp);
    if (!S.ok()) return S.fail();
    cub::DeviceRadixSort::SortKeys(d_tmp, tmp, keys_in, keys_out, n_ent, 0, 64, st);
  }
  build_flags_kernel<<<(n_ent + 255) / 256, 256, 0, st>>>(keys_out, n_ent, flags);
  {
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, flags, gid, n_ent, st);
    void* d_tmp = S.alloc<char>(tmp);
    if (!S.ok()) return S.fail();
    cub::DeviceScan::InclusiveSum(d_tmp, tmp, flags, gid, n_ent, st);
  }
  // tree_ent0[b] = ent_base[b * P]  (entries are grouped by tree in sorted order)
  ICB_CUDA(cudaMemcpy2DAsync(tree_ent0, sizeof(int), ent_base, sizeof(int) * P, sizeof(int), n,
                             cudaMemcpyDeviceToDevice, st));
  // zero node sizes of the involved trees
  zero_node_sizes(f, trees, n, st);
  build_nodes_kernel<<<(n_ent + 255) / 256, 256, 0, st>>>(F, A, keys_out, n_ent_dev, gid, tree_ent0, top,
                                                          own_base_pos);
  build_tree_totals_kernel<<<(n + 127) / 128, 128, 0, st>>>(F, A, gid, tree_ent0, ent_cnt);
  // parents, leaf page counts
  const int max_nodes = F.node_cap;
  int* leaf_pages = S.alloc<int>((size_t)n * max_nodes);
  int* leaf_first = S.alloc<int>((size_t)n * max_nodes);
  if (!S.ok()) return S.fail();
  build_parents_kernel<<<dim3((max_nodes + 255) / 256, n), 256, 0, st>>>(F, A, max_nodes, parent_pos,
                                                                       leaf_pages);
  {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, leaf_pages, leaf_first, n * max_nodes, st);
    void* d_tmp = S.alloc<char>(tmp);
    if (!S.ok()) return S.fail();
    cub::DeviceScan::ExclusiveSum(d_tmp, tmp, leaf_pages, leaf_first, n * max_nodes, st);
  }
  build_pages_kernel<<<dim3(max_nodes, n), 256, 0, st>>>(F, A, max_nodes, leaf_first, nullptr);
  build_page_totals_kernel<<<(n + 127) / 128, 128, 0, st>>>(F, A, max_nodes, leaf_first, leaf_pages);
  build_summary_kernel<<<n, 256, 0, st>>>(F, A);
  ICB_CUDA(cudaGetLastError());
  int rc = S.finish();
  if (rc) return rc;
  // P-DCI directions + ladder caches of the nodes decode will visit with P-DCI
  // (the default decode budget's visit cap: 4 x 256)
  return icb_pdci_warm_impl(f, trees, n, 1024, st);
}

extern "C" int icb_build_profile(unsigned long long* out, int reset) {
  ICB_CUDA(cudaDeviceSynchronize());
  ICB_CUDA(cudaMemcpyFromSymbol(out, icb::g_build_prof, sizeof(unsigned long long) * 4));
  if (reset) {
    unsigned long long z[4] = {};
    ICB_CUDA(cudaMemcpyToSymbol(icb::g_build_prof, z, sizeof(z)));
  }
  return ICB_OK;
}
