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

// one thread per tree: draw levels in input order from the continuing stream
__global__ void build_levels_kernel(ForestView F, BuildArgs A, int* drawn, unsigned long long* occ) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= A.n) return;
  TreeMeta* m = F.meta + A.trees[b];
  Pcg64 g = m->rng;
  unsigned long long mask = 0;
  for (int i = 0; i < A.n_points; ++i) {
    int lv = icb_draw_level(g, F.r);
    if (lv > 62) lv = 62;
    drawn[(size_t)b * A.n_points + i] = lv;
    mask |= 1ull << lv;
  }
  m->rng = g;
  occ[b] = mask;
  m->levels = __popcll(mask);
  m->n_points = A.n_points;
  m->top_node = 0;
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
                                                        int stride, int* parent_pos) {
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

__global__ void build_flags_kernel(const unsigned long long* keys, int n, int* flags) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  flags[j] = (j == 0 || (keys[j] >> 23) != (keys[j - 1] >> 23)) ? 1 : 0;
}

// gid = inclusive scan of flags; tree_ent0[b] = first entry of tree b
__global__ void build_nodes_kernel(ForestView F, BuildArgs A, const unsigned long long* keys, int n_ent,
                                   const int* gid, const int* tree_ent0, const int* top,
                                   const int* own_base_pos) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_ent) return;
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
    if (F.kv_bf16) {
      __nv_bfloat16* K = (__nv_bfloat16*)F.page_k + kslot * F.dkp;
      __nv_bfloat16* V = (__nv_bfloat16*)F.page_v + kslot * F.dvp;
      for (int j = lane; j < F.dim; j += 32) K[j] = __float2bfloat16_rn(kin[j]);
      for (int j = lane; j < F.dim_v; j += 32) V[j] = __float2bfloat16_rn(vin ? vin[j] : 0.f);
    } else {
      float* K = (float*)F.page_k + kslot * F.dkp;
      float* V = (float*)F.page_v + kslot * F.dvp;
      for (int j = lane; j < F.dim; j += 32) K[j] = kin[j];
      for (int j = lane; j < F.dim_v; j += 32) V[j] = vin ? vin[j] : 0.f;
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
  build_levels_kernel<<<(n + 63) / 64, 64, 0, st>>>(F, A, top, occ);
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
  {
    const int D1 = F.dim + 1, PS = D1 | 1;
    size_t sm = sizeof(double) * (NN_BM * PS + NN_BN * (NN_KC + 1));
    ICB_CUDA(cudaFuncSetAttribute(nn_parent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    nn_parent_kernel<<<dim3((P + NN_BM - 1) / NN_BM, n), 256, sm, st>>>(
        F, A, nsq, pts, pts_off, cands, cand_off, cand64, cand_sq, stride, parent_pos);
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
  // total entries (needs host value for sizing)
  int last_base = 0, last_top = 0;
  ICB_CUDA(cudaMemcpyAsync(&last_base, ent_base + (size_t)n * P - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  ICB_CUDA(cudaMemcpyAsync(&last_top, top + (size_t)n * P - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  ICB_CUDA(cudaStreamSynchronize(st));
  const int n_ent = last_base + last_top;
  unsigned long long* keys_in = S.alloc<unsigned long long>(n_ent);
  unsigned long long* keys_out = S.alloc<unsigned long long>(n_ent);
  int* flags = S.alloc<int>(n_ent);
  int* gid = S.alloc<int>(n_ent);
  int* tree_ent0 = S.alloc<int>(n);
  if (!S.ok()) return S.fail();
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
  build_nodes_kernel<<<(n_ent + 255) / 256, 256, 0, st>>>(F, A, keys_out, n_ent, gid, tree_ent0, top,
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
  return S.finish();
}
