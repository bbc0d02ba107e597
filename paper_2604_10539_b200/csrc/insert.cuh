// Dynamic insertion and window rotation on the device (device code; the
// kernels and C ABI are in insert.cu, the fused rotate+append+query kernel in
// search.cu).
//
//   insert_one      DciTree.insert (dci.py:385-431), _grow_top (:433-449),
//                   _place_entry (:368-381); the parent search is the block
//                   search with PARENT_BUDGET (k=1, beam=8, visit_cap=64;
//                   dci.py:78) targeted at level+1.
//   rotate          Engine._rotate_layer (engine.py:516-534): offload the
//                   oldest window page, insert its entries in slot order,
//                   release it, allocate a fresh window page.
//   append          the decode token joins the first non-full window page
//                   (engine.py:426-429).
//   resident pages  sink / window allocation at prefill (engine.py:263-276).
//
// One CTA per tree; inserts of a tree are sequential (each must see the
// previous), trees run in parallel.  Raw fp32 keys of window tokens are
// stashed in the token's (not yet used) lifted row so the insert lifts the
// exact input key even when pages store bf16.
#pragma once
#include "search.cuh"
#include "warp_search.cuh"

namespace icb {


struct InsertArgs {
  const int32_t* trees;
  int n, m;
  const int32_t* tokens;   // [n][m]
  const float* keys;       // [n][m][dim]
  const float* values;     // [n][m][dim_v] or null
  const int32_t* levels;   // [n][m] or null
  int32_t* out_levels;
  int from_window;         // 1: rotate the oldest window page
  int scalar_bytes;
  int64_t* stats;          // [n][2] offload bytes, transactions (may be null)
  unsigned long long* prof;   // optional phase cycles (ICB_PROF): prepare, search, fallback, finish, segments
};

// profiling counters: one copy per translation unit (ICB_PROF diagnostics)
static __device__ unsigned long long g_insert_prof[8];
// per-tree rotation cycles (ICB_PROF): the kernel ends with its slowest tree
static __device__ unsigned long long g_insert_tree_cycles[4096];
static __device__ unsigned g_insert_tree_fallbacks[4096];

__device__ inline int new_node(const ForestView& F, int t, int level, int parent, int owner, int first_member) {
  TreeMeta* m = F.meta + t;
  int id = m->n_nodes;
  if (id >= F.node_cap) { set_err(m, ICB_ERR_CAP_NODES); return -1; }
  m->n_nodes = id + 1;
  size_t x = F.nd(t, id);
  int cap = 4;
  int off = m->member_top;
  if (off + cap > F.member_cap) { set_err(m, ICB_ERR_CAP_MEMBERS); return -1; }
  m->member_top = off + cap;
  F.node_level[x] = level;
  F.node_parent[x] = parent;
  F.node_owner[x] = owner;
  F.node_off[x] = off;
  F.node_size[x] = 1;
  F.node_capm[x] = cap;
  F.node_lastpage[x] = -1;
  F.node_dirs[x] = -1;
  F.node_opos[x] = (owner >= 0 && owner == first_member) ? 0 : -1;
  F.mem(t)[off] = first_member;
  note_node_size(m, level, 1);
  return id;
}

// Keep a node's P-DCI cache (search.cuh pc_ensure) valid across an append of
// member `tok` at position sz (ONE thread): its 8 projections (the same fp64
// chains), then on every ladder its rank by (projection, id) and the shifted
// ranks of the members after it.  Without fresh entries, room and directions
// the cache is left stale (rebuilt by the next block visit).
__device__ inline void pc_append(const ForestView& F, int t, size_t x, const int* mem, int sz, int tok) {
  const int off = F.node_pc[x];
  if (off < 0 || F.node_pcm[x] != sz || F.node_pccap[x] <= sz || F.node_dirs[x] < 0) return;
  const int D1 = F.dim + 1;
  const double* dirs = F.dirs + ((size_t)t * F.dirs_cap + F.node_dirs[x]) * ICB_NPROJ * D1;
  double* proj = F.pc_proj + ((size_t)t * F.pc_cap + off) * ICB_NPROJ;
  int* ord = F.pc_ord + ((size_t)t * F.pc_cap + off) * ICB_NPROJ;
  int* pos = F.pc_pos + ((size_t)t * F.pc_cap + off) * ICB_NPROJ;
  const float* row = F.row(t, tok);
  const float tl = F.tail[F.tk(t, tok)];
  for (int j = 0; j < ICB_NPROJ; ++j) {
    double acc = 0.0;
    for (int u = 0; u < F.dim; ++u) acc = __fma_rn(dirs[j * D1 + u], (double)row[u], acc);
    acc = __fma_rn(dirs[j * D1 + F.dim], (double)tl, acc);
    proj[(size_t)sz * ICB_NPROJ + j] = acc;
    int lo = 0, hi = sz;   // rank: members below (acc, tok)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1, mi = ord[(size_t)mid * ICB_NPROJ + j];
      const double p = proj[(size_t)mi * ICB_NPROJ + j];
      if (p < acc || (p == acc && mem[mi] < tok)) lo = mid + 1;
      else hi = mid;
    }
    for (int r = sz; r > lo; --r) {
      const int mi = ord[(size_t)(r - 1) * ICB_NPROJ + j];
      ord[(size_t)r * ICB_NPROJ + j] = mi;
      pos[(size_t)mi * ICB_NPROJ + j] = r;
    }
    ord[(size_t)lo * ICB_NPROJ + j] = sz;
    pos[(size_t)sz * ICB_NPROJ + j] = lo;
  }
  F.node_pcm[x] = sz + 1;
}

__device__ inline void add_member(const ForestView& F, int t, int node, int tok) {
  TreeMeta* m = F.meta + t;
  size_t x = F.nd(t, node);
  int sz = F.node_size[x], cap = F.node_capm[x], off = F.node_off[x];
  int* mem = F.mem(t);
  if (sz == cap) {
    int ncap = cap < 4 ? 4 : 2 * cap;
    int noff = m->member_top;
    if (noff + ncap > F.member_cap) { set_err(m, ICB_ERR_CAP_MEMBERS); return; }
    m->member_top = noff + ncap;
    for (int i = 0; i < sz; ++i) mem[noff + i] = mem[off + i];
    off = noff;
    F.node_off[x] = off;
    F.node_capm[x] = ncap;
  }
  mem[off + sz] = tok;
  pc_append(F, t, x, mem + off, sz, tok);
  F.node_size[x] = sz + 1;
  note_node_size(m, F.node_level[x], sz + 1);
}

__device__ __forceinline__ void set_own(const ForestView& F, int t, int tok, int lv, int node) {
  F.own_list[(size_t)t * F.own_cap + F.own_base[F.tk(t, tok)] + lv - 1] = node;
  if (lv == 1) F.own1[F.tk(t, tok)] = node;
}

// KV offload: the HBM pool row mirroring page `page` row `slot` when the page
// is resident in the pool (writes go to the host store and to that copy).
__device__ __forceinline__ size_t pool_dst(const ForestView& F, int t, int page, int slot) {
  if (!F.kv_host) return ~(size_t)0;
  const int sl = F.page_slot[F.pg(t, page)];
  return sl < 0 ? ~(size_t)0 : ((size_t)t * F.pool_cap + sl) * F.s + slot;
}

// Copy one entry into a page slot (one warp; lane l owns dims 4l..4l+3).
// K/V come either from fp32 arrays or from another page slot of the same
// forest (window rotation).  Every source element is loaded before any store
// so the copy costs one memory round trip.
__device__ inline void write_slot(const ForestView& F, int t, int page, int slot, const float* kf, const float* vf,
                           long long src_slot) {
  const int lane = threadIdx.x & 31;
  const int j0 = lane * 4;
  const size_t dst = F.pg(t, page) * F.s + slot;
  if (F.kv_bf16) {
    __nv_bfloat16* K = (__nv_bfloat16*)F.page_k;
    __nv_bfloat16* V = (__nv_bfloat16*)F.page_v;
    uint2 kw = make_uint2(0u, 0u), vw = make_uint2(0u, 0u);
    if (src_slot >= 0) {
      if (j0 < F.dkp) kw = *reinterpret_cast<const uint2*>(K + (size_t)src_slot * F.dkp + j0);
      if (j0 < F.dvp) vw = *reinterpret_cast<const uint2*>(V + (size_t)src_slot * F.dvp + j0);
    } else {
      float k[4], v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        k[u] = j0 + u < F.dim ? kf[j0 + u] : 0.f;
        v[u] = (vf && j0 + u < F.dim_v) ? vf[j0 + u] : 0.f;
      }
      __nv_bfloat162 k01 = __floats2bfloat162_rn(k[0], k[1]), k23 = __floats2bfloat162_rn(k[2], k[3]);
      __nv_bfloat162 v01 = __floats2bfloat162_rn(v[0], v[1]), v23 = __floats2bfloat162_rn(v[2], v[3]);
      kw = make_uint2(*reinterpret_cast<unsigned*>(&k01), *reinterpret_cast<unsigned*>(&k23));
      vw = make_uint2(*reinterpret_cast<unsigned*>(&v01), *reinterpret_cast<unsigned*>(&v23));
    }
    if (j0 < F.dkp) *reinterpret_cast<uint2*>(K + dst * F.dkp + j0) = kw;
    if (j0 < F.dvp) *reinterpret_cast<uint2*>(V + dst * F.dvp + j0) = vw;
    const size_t pd = pool_dst(F, t, page, slot);
    if (pd != ~(size_t)0) {
      if (j0 < F.dkp) *reinterpret_cast<uint2*>((__nv_bfloat16*)F.pool_k + pd * F.dkp + j0) = kw;
      if (j0 < F.dvp) *reinterpret_cast<uint2*>((__nv_bfloat16*)F.pool_v + pd * F.dvp + j0) = vw;
    }
  } else {
    float* K = (float*)F.page_k;
    float* V = (float*)F.page_v;
    float4 kw = make_float4(0.f, 0.f, 0.f, 0.f), vw = kw;
    if (src_slot >= 0) {
      if (j0 < F.dkp) kw = *reinterpret_cast<const float4*>(K + (size_t)src_slot * F.dkp + j0);
      if (j0 < F.dvp) vw = *reinterpret_cast<const float4*>(V + (size_t)src_slot * F.dvp + j0);
    } else {
      float k[4], v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        k[u] = j0 + u < F.dim ? kf[j0 + u] : 0.f;
        v[u] = (vf && j0 + u < F.dim_v) ? vf[j0 + u] : 0.f;
      }
      kw = make_float4(k[0], k[1], k[2], k[3]);
      vw = make_float4(v[0], v[1], v[2], v[3]);
    }
    if (j0 < F.dkp) *reinterpret_cast<float4*>(K + dst * F.dkp + j0) = kw;
    if (j0 < F.dvp) *reinterpret_cast<float4*>(V + dst * F.dvp + j0) = vw;
    const size_t pd = pool_dst(F, t, page, slot);
    if (pd != ~(size_t)0) {
      if (j0 < F.dkp) *reinterpret_cast<float4*>((float*)F.pool_k + pd * F.dkp + j0) = kw;
      if (j0 < F.dvp) *reinterpret_cast<float4*>((float*)F.pool_v + pd * F.dvp + j0) = vw;
    }
  }
}

// Inserts run in three stages:
//   prepare   duplicate check, level draw (the tree's level stream, in
//             insertion order), lift (dci.py:225-240) into the token's row and
//             into query slot `qs` of S; returns the level (-1: rejected);
//   place     the node that receives the point at its level (top node /
//             _grow_top / own(parent, level) from the parent search);
//   finish    membership, own-node chain below the level, page placement
//             (dci.py:368-381) and the K/V slot write.
// The level summary (start level, upper list) learns of a point only when it
// is placed, so a point prepared ahead of a pending batched search stays
// invisible to that search.
template <int NT>
__device__ inline int insert_prepare(SearchSmem& S, const ForestView& F, int t, int tok, const float* key, int given_level,
                              int qs) {
  TreeMeta* m = F.meta + t;
  __shared__ int s_level, s_bad;
  __shared__ double s_norm;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_bad = 0;
    if (tok < 0 || tok >= F.tok_cap) { set_err(m, ICB_ERR_CAP_TOKENS); s_bad = 1; }
    else {
      int old = atomicCAS(F.tok2page + F.tk(t, tok), -1, -2);
      if (old != -1) { set_err(m, ICB_ERR_DUP_ID); s_bad = 1; }
    }
    int lv = given_level;
    if (lv <= 0 && !s_bad) {
      Pcg64 g = m->rng;
      lv = icb_draw_level(g, F.r);
      m->rng = g;
    }
    if (lv > 62) lv = 62;
    s_level = lv;
  }
  for (int u = tid; u < F.dim; u += NT) {
    double x = (double)key[u];
    S.q64[u] = __dmul_rn(x, x);
  }
  __syncthreads();
  if (s_bad) return -1;
  if (tid == 0) s_norm = sqrt(pairwise_sum(S.q64, F.dim));
  __syncthreads();
  const double c = m->c, norm = s_norm;
  const bool over = norm > c;
  const double safe = over ? norm : c;
  float* row = F.lift + F.tk(t, tok) * ICB_ROWF;
  // read the raw key before overwriting (it may live in this very row)
  float kv = tid < F.dim ? key[tid] : 0.f;
  __syncthreads();
  for (int u = tid; u < ICB_DPAD; u += NT) {
    float v = u < F.dim ? __double2float_rn(__ddiv_rn((double)kv, safe)) : 0.0f;
    row[u] = v;
    S.q[qs][u] = v;
  }
  if (tid > 0 && tid < ICB_ROWF - ICB_DPAD) row[ICB_DPAD + tid] = 0.0f;
  const int level = s_level;
  if (tid == 0) {
    double ratio = __ddiv_rn(norm, safe);
    double rad = __dsub_rn(1.0, __dmul_rn(ratio, ratio));
    float tl = __double2float_rn(sqrt(rad > 0.0 ? rad : 0.0));
    F.tail[F.tk(t, tok)] = tl;
    if (ICB_ROWF > ICB_DPAD) row[ICB_DPAD] = tl;
    S.qt[qs] = tl;
    if (over) m->scale_clamps += 1;
    F.level[F.tk(t, tok)] = (int8_t)level;
    F.own_base[F.tk(t, tok)] = m->own_top;
    if (m->own_top + level - 1 > F.own_cap) set_err(m, ICB_ERR_CAP_OWN);
    m->own_top += level - 1;
  }
  __syncthreads();
  return level;
}

// Block-wide parent search of query slot qs (the P-DCI-capable path; used
// only when a warp search meets a node the reference visits with P-DCI).
template <int NT>
__device__ __forceinline__ int block_parent_search(SearchSmem& S, GroupSmem* GSA, const RingView& RG,
                                                const ForestView& F, const SearchScratch& SS, int t, int qs,
                                                int target, double* dirs_tmp) {
  __shared__ int s_parent;
  __shared__ float s_swap_t;
  const int tid = threadIdx.x;
  if (qs != 0) {   // tree_search reads slot 0: swap the slots
    for (int u = tid; u < ICB_DPAD; u += NT) { float a = S.q[0][u]; S.q[0][u] = S.q[qs][u]; S.q[qs][u] = a; }
    if (tid == 0) { s_swap_t = S.qt[0]; S.qt[0] = S.qt[qs]; S.qt[qs] = s_swap_t; }
    __syncthreads();
  }
  SearchParams P;
  P.G = 1; P.k = 1; P.beam = 8; P.visit_cap = 64; P.target = target; P.prof = nullptr;
  tree_search<NT, 1>(S, GSA, RG, F, SS, t, P, dirs_tmp);
  const int n = finalize_groups<NT, 1>(S, GSA, F, SS, 1, 1);
  if (tid == 0) s_parent = n > 0 ? key_id(GSA[0].buf[0]) : -1;
  __syncthreads();
  if (qs != 0) {
    for (int u = tid; u < ICB_DPAD; u += NT) { float a = S.q[0][u]; S.q[0][u] = S.q[qs][u]; S.q[qs][u] = a; }
    if (tid == 0) { s_swap_t = S.qt[0]; S.qt[0] = S.qt[qs]; S.qt[qs] = s_swap_t; }
    __syncthreads();
  }
  return s_parent;
}

// Membership, own chain and page placement of one point (ONE thread);
// returns the page (-1 on capacity error) and its slot in *slot.
__device__ inline int finish_book(const ForestView& F, int t, int tok, int level, int container, int chain_from,
                           bool add_to_container, int* slot_out) {
  TreeMeta* m = F.meta + t;
  note_point_level(F, t, tok, level);
  if (add_to_container) add_member(F, t, container, tok);
  int parent_node = container;   // node holding tok at chain_from + 1
  for (int lv = chain_from; lv >= 1; --lv) {
    int nn = new_node(F, t, lv, parent_node, tok, tok);
    set_own(F, t, tok, lv, nn);
    parent_node = nn;
  }
  int leaf = level >= 2 ? F.own(t, tok, 1) : container;
  size_t lx = F.nd(t, leaf);
  int page = F.node_lastpage[lx];
  if (page < 0 || F.page_fill[F.pg(t, page)] >= F.s) {
    page = m->next_page;
    if (page >= F.page_cap) { set_err(m, ICB_ERR_CAP_PAGES); page = -1; }
    else {
      m->next_page = page + 1;
      F.page_fill[F.pg(t, page)] = 0;
      F.page_role[F.pg(t, page)] = ICB_ROLE_INDEXED;
      F.node_lastpage[lx] = page;
    }
  }
  if (page >= 0) {
    int slot = F.page_fill[F.pg(t, page)];
    F.page_tok[F.pg(t, page) * F.s + slot] = tok;
    F.page_fill[F.pg(t, page)] = slot + 1;
    F.tok2page[F.tk(t, tok)] = page;
    *slot_out = slot;
  }
  m->n_points += 1;
  return page;
}

template <int NT>
__device__ inline void insert_finish(SearchSmem& S, const ForestView& F, int t, int tok, int level, int container,
                              int chain_from, bool add_to_container, const float* key, const float* val,
                              long long src_slot) {
  TreeMeta* m = F.meta + t;
  __shared__ int s_leaf;
  const int tid = threadIdx.x;
  if (tid == 0) {
    int slot = 0;
    s_leaf = finish_book(F, t, tok, level, container, chain_from, add_to_container, &slot);
    S.misc[4] = slot;
  }
  __syncthreads();
  if (s_leaf >= 0 && tid < 32) write_slot(F, t, s_leaf, S.misc[4], key, val, src_slot);
  __syncthreads();
  (void)m;
}

struct InsertPoint {
  int tok;
  const float* key;
  const float* val;
  long long src_slot;
  int given_level;
};

// Structure + finish of a prepared point; `parent` is its parent search's
// result when level < the tree height (searched by insert_points).
template <int NT>
__device__ inline void insert_place(SearchSmem& S, const ForestView& F, int t, const InsertPoint& pt, int level,
                             int parent) {
  TreeMeta* m = F.meta + t;
  __shared__ int s_container, s_chain_from, s_add;
  const int tid = threadIdx.x;
  const int tok = pt.tok;
  const int L = m->levels;
  if (L == 0) {
    if (tid == 0) {
      int top = new_node(F, t, level, -1, ICB_ROOT_OWNER, tok);
      m->top_node = top;
      m->levels = level;
      s_container = top;
      s_chain_from = level - 1;
      s_add = 0;
    }
  } else if (level > L) {
    if (tid == 0) {
      int old_top = m->top_node;
      int top = new_node(F, t, level, -1, ICB_ROOT_OWNER, tok);
      m->top_node = top;
      int prev = top;
      for (int lv = level - 1; lv > L; --lv) {
        prev = new_node(F, t, lv, prev, tok, tok);
        set_own(F, t, tok, lv, prev);
      }
      size_t x = F.nd(t, old_top);
      F.node_owner[x] = tok;
      F.node_parent[x] = prev;
      set_own(F, t, tok, L, old_top);
      add_member(F, t, old_top, tok);
      F.node_opos[x] = F.node_size[x] - 1;   // the new owner was appended
      m->levels = level;
      s_container = old_top;   // membership at level L
      s_chain_from = L - 1;
      s_add = 0;
    }
  } else if (level == L) {
    if (tid == 0) { s_container = m->top_node; s_chain_from = level - 1; s_add = 1; }
  } else {
    if (tid == 0) {
      s_container = parent >= 0 ? F.own(t, parent, level) : m->top_node;
      s_chain_from = level - 1;
      s_add = 1;
    }
  }
  __syncthreads();
  insert_finish<NT>(S, F, t, tok, level, s_container, s_chain_from, s_add != 0, pt.key, pt.val, pt.src_slot);
}

// Inserts of one tree in order.  Consecutive level-1 points (tree height >=
// 2) form runs of up to 8 whose parent searches run at once, one warp each:
// a level-1 point's search reads only levels >= 2, which placing level-1
// points never changes, so each parent equals the sequential one.  The point
// that ends a run (level >= 2) has its search (levels >= level + 1 >= 3) on
// the next warp, concurrently.  The run's points are then finished in
// insertion order (membership, pages), then the ending point is placed --
// exactly the sequential result.
template <int NT, typename PointFn>
__device__ inline void insert_points(SearchSmem& S, GroupSmem* GSA, const RingView& RG, const ForestView& F,
                              const SearchScratch& SS, int t, double* dirs_tmp, int n, PointFn point,
                              int32_t* out_levels, unsigned long long* prof) {
  constexpr int NW = NT / 32;
  static_assert(NW <= ICB_MAX_G, "one query slot per warp");
  TreeMeta* m = F.meta + t;
  WarpSearchBuf* WB = reinterpret_cast<WarpSearchBuf*>(RG.ring);   // the ring is idle during inserts
  __shared__ int s_par[NW], s_ok[NW], s_wpage[NW], s_wslot[NW];
  __shared__ int s_rc[NW], s_rsz[NW], s_rcap[NW], s_roff[NW], s_rlv[NW], s_rlp[NW], s_rfill[NW];
  __shared__ unsigned long long s_ev[NW];
  __shared__ InsertPoint s_pt[NW + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  long long tp = clock64();
  auto mark = [&](int k) {
    if (prof && tid == 0) {
      const long long now = clock64();
      atomicAdd(prof + k, (unsigned long long)(now - tp));
      tp = now;
    }
  };
  for (int e = 0; e < n;) {
    int nr = 0, single = -1;
    while (e < n && nr < NW) {
      const InsertPoint pt = point(e);
      const int got = insert_prepare<NT>(S, F, t, pt.tok, pt.key, pt.given_level, nr);
      if (tid == 0 && out_levels) out_levels[e] = got;
      ++e;
      if (got < 0) continue;
      if (tid == 0) s_pt[nr] = pt;
      if (got == 1 && m->levels >= 2) { ++nr; continue; }
      single = got;
      break;
    }
    __syncthreads();
    mark(0);
    if (prof && tid == 0) atomicAdd(prof + 4, 1ull);
    const int L = m->levels;
    const bool single_search = single > 0 && single < L;
    const int nsearch = nr + (single_search ? 1 : 0);
    if (warp < nsearch) {
      int par = -1;
      unsigned long long ev = 0;
      const int target = warp < nr ? 2 : single + 1;
      const bool ok = warp_parent_search(F, t, S.q[warp], S.qt[warp], target, WB[warp], &par, &ev);
      if (lane == 0) { s_par[warp] = par; s_ok[warp] = ok; s_ev[warp] = ev; }
    }
    __syncthreads();
    mark(1);
    if (tid == 0) {
      unsigned long long ev = 0, qc = 0;
      for (int w = 0; w < nsearch; ++w)
        if (s_ok[w]) { ev += s_ev[w]; ++qc; }
      if (qc) { atomicAdd(&m->query_count, qc); atomicAdd(&m->distance_evals, ev); }
    }
    for (int w = 0; w < nsearch; ++w) {
      if (!s_ok[w]) {   // block-uniform; rare (a node the reference visits with P-DCI)
        if (prof && tid == 0 && t < 4096) atomicAdd(&g_insert_tree_fallbacks[t], 1u);
        const int par = block_parent_search<NT>(S, GSA, RG, F, SS, t, w, w < nr ? 2 : single + 1, dirs_tmp);
        if (tid == 0) s_par[w] = par;
        __syncthreads();
      }
    }
    mark(2);
    // The run's bookkeeping in insertion order.  Each point's container and
    // its node / last-page fields are fetched in parallel (one thread per
    // point); one thread then applies the points in order from those copies
    // (updating later points that share a container), so page ids and slots
    // equal the sequential inserts'.  Then the K/V slot writes, one warp per
    // point.
    if (tid < nr) {
      const int par = s_par[tid];
      const int c = par >= 0 ? F.own(t, par, 1) : m->top_node;
      const size_t x = F.nd(t, c);
      const int lp = F.node_lastpage[x];
      s_rc[tid] = c;
      s_rsz[tid] = F.node_size[x];
      s_rcap[tid] = F.node_capm[x];
      s_roff[tid] = F.node_off[x];
      s_rlv[tid] = F.node_level[x];
      s_rlp[tid] = lp;
      s_rfill[tid] = lp >= 0 ? F.page_fill[F.pg(t, lp)] : 0;
    }
    __syncthreads();
    if (tid == 0)
      for (int w = 0; w < nr; ++w) {
        const int tok = s_pt[w].tok, c = s_rc[w];
        const size_t x = F.nd(t, c);
        note_point_level(F, t, tok, 1);
        // add_member (insert.cu:add_member) from the cached node fields
        int sz = s_rsz[w], cap = s_rcap[w], off = s_roff[w];
        int* mem = F.mem(t);
        bool ok = true;
        if (sz == cap) {
          const int ncap = cap < 4 ? 4 : 2 * cap;
          const int noff = m->member_top;
          if (noff + ncap > F.member_cap) { set_err(m, ICB_ERR_CAP_MEMBERS); ok = false; }
          else {
            m->member_top = noff + ncap;
            for (int i = 0; i < sz; ++i) mem[noff + i] = mem[off + i];
            off = noff;
            cap = ncap;
            F.node_off[x] = off;
            F.node_capm[x] = cap;
          }
        }
        if (ok) {
          mem[off + sz] = tok;
          pc_append(F, t, x, mem + off, sz, tok);
          F.node_size[x] = sz + 1;
          note_node_size(m, s_rlv[w], sz + 1);
          ++sz;
        }
        // page placement (dci.py:368-381)
        int page = s_rlp[w], fill = s_rfill[w];
        if (page < 0 || fill >= F.s) {
          page = m->next_page;
          if (page >= F.page_cap) { set_err(m, ICB_ERR_CAP_PAGES); page = -1; }
          else {
            m->next_page = page + 1;
            F.page_fill[F.pg(t, page)] = 0;
            F.page_role[F.pg(t, page)] = ICB_ROLE_INDEXED;
            F.node_lastpage[x] = page;
            fill = 0;
          }
        }
        s_wpage[w] = page;
        s_wslot[w] = fill;
        if (page >= 0) {
          F.page_tok[F.pg(t, page) * F.s + fill] = tok;
          F.page_fill[F.pg(t, page)] = fill + 1;
          F.tok2page[F.tk(t, tok)] = page;
          ++fill;
        }
        m->n_points += 1;
        for (int w2 = w + 1; w2 < nr; ++w2)
          if (s_rc[w2] == c) {
            s_rsz[w2] = sz; s_rcap[w2] = cap; s_roff[w2] = off;
            s_rlp[w2] = page; s_rfill[w2] = fill;
          }
      }
    __syncthreads();
    if (warp < nr && s_wpage[warp] >= 0)
      write_slot(F, t, s_wpage[warp], s_wslot[warp], s_pt[warp].key, s_pt[warp].val, s_pt[warp].src_slot);
    __syncthreads();
    if (single > 0) insert_place<NT>(S, F, t, s_pt[nr], single, single_search ? s_par[nr] : -1);
    mark(3);
  }
}

// Engine._rotate_layer for tree t (engine.py:516-534): insert the oldest window
// page's entries in slot order, release the page, open a fresh window page.
// `stats` points at this tree's [offload bytes, transactions] (or null).
template <int NT>
__device__ void rotate_tree(SearchSmem& S, GroupSmem* GSA, const RingView& RG, const ForestView& F,
                            const SearchScratch& SS, int t, double* dirs_tmp, int64_t* stats, int scalar_bytes,
                            unsigned long long* prof) {
  TreeMeta* m = F.meta + t;
  __shared__ int s_old, s_fill;
  if (threadIdx.x == 0) {
    s_old = m->n_window > 0 ? m->win[0] : -1;
    s_fill = s_old >= 0 ? F.page_fill[F.pg(t, s_old)] : 0;
    if (s_old < 0) set_err(m, ICB_ERR_WINDOW);
    else if (stats) {
      stats[0] += (int64_t)s_fill * (F.dim + F.dim_v) * scalar_bytes;
      stats[1] += 1;
    }
  }
  __syncthreads();
  const int old = s_old;
  if (old < 0) return;
  // the oldest window page's entries in slot order; raw keys were stashed in
  // the tokens' lifted rows, K/V are copied from the page slot
  const long long tt0 = clock64();
  insert_points<NT>(S, GSA, RG, F, SS, t, dirs_tmp, s_fill, [&](int e) {
    InsertPoint p;
    p.tok = F.page_tok[F.pg(t, old) * F.s + e];
    p.key = F.lift + F.tk(t, p.tok) * ICB_ROWF;
    p.val = nullptr;
    p.src_slot = (long long)(F.pg(t, old) * F.s + e);
    p.given_level = 0;
    return p;
  }, (int32_t*)nullptr, prof);
  if (prof && threadIdx.x == 0 && t < 4096) g_insert_tree_cycles[t] += (unsigned long long)(clock64() - tt0);
  if (threadIdx.x == 0) {
    // release (pagestore.py:157-162) then a fresh window page
    F.page_role[F.pg(t, old)] = 0;
    if (F.kv_host) {   // its pool slot, if resident, is free again
      const int sl = F.page_slot[F.pg(t, old)];
      if (sl >= 0) {
        F.slot_page[(size_t)t * F.pool_cap + sl] = -1;
        F.page_slot[F.pg(t, old)] = -1;
      }
    }
    for (int i = 0; i + 1 < m->n_window; ++i) m->win[i] = m->win[i + 1];
    int np = m->next_page;
    if (np >= F.page_cap) { set_err(m, ICB_ERR_CAP_PAGES); }
    else {
      m->next_page = np + 1;
      F.page_fill[F.pg(t, np)] = 0;
      F.page_role[F.pg(t, np)] = ICB_ROLE_WINDOW;
      m->win[m->n_window - 1] = np;
    }
  }
  __syncthreads();
}

// The decode token joins tree t's first non-full window page (engine.py:426-429).
// k: the raw key [dim], v: the value [dim_v].
__device__ inline void append_tree(const ForestView& F, int t, int token, const float* k, const float* v) {
  TreeMeta* m = F.meta + t;
  __shared__ int s_page, s_slot;
  if (threadIdx.x == 0) {
    s_page = -1;
    for (int i = 0; i < m->n_window; ++i) {
      int p = m->win[i];
      if (F.page_fill[F.pg(t, p)] < F.s) { s_page = p; break; }
    }
    if (s_page < 0 || token < 0 || token >= F.tok_cap) set_err(m, ICB_ERR_WINDOW);
    else {
      s_slot = F.page_fill[F.pg(t, s_page)];
      F.page_fill[F.pg(t, s_page)] = s_slot + 1;
      F.page_tok[F.pg(t, s_page) * F.s + s_slot] = token;
    }
  }
  __syncthreads();
  if (s_page < 0 || token < 0 || token >= F.tok_cap) return;
  float* stash = F.lift + F.tk(t, token) * ICB_ROWF;
  for (int j = threadIdx.x; j < F.dim; j += blockDim.x) stash[j] = k[j];
  if (threadIdx.x < 32) write_slot(F, t, s_page, s_slot, k, v, -1);
}

}  // namespace icb
