// Device-side layout of the DCI forest and shared numerics.
//
// One forest holds T independent DCI trees (one per (sequence, layer, kv
// head)).  Everything lives in HBM as flat structure-of-arrays indexed
// [tree][...]; rows of the lifted-key matrix are indexed by TOKEN ID, so a
// 64-bit ranking key (d2 bits << 32 | token id) identifies a candidate and
// its row at once.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "rng.cuh"
#include "../../include/icecache_b200.h"

// Debug builds (-DICB_DEBUG=1, make debug) bounds-check every scratch index
// and trap with a message; release builds compile the checks away.
#ifndef ICB_DEBUG
#define ICB_DEBUG 0
#endif
#if ICB_DEBUG
#include <cstdio>
#define ICB_CHECK(cond, ...)                                                   \
  do {                                                                         \
    if (!(cond)) {                                                             \
      printf("ICB_CHECK %s:%d (%s) ", __FILE__, __LINE__, #cond);              \
      printf(__VA_ARGS__);                                                     \
      printf("\n");                                                            \
      __trap();                                                                \
    }                                                                          \
  } while (0)
#else
#define ICB_CHECK(cond, ...) \
  do {                       \
  } while (0)
#endif

#define ICB_DPAD 128          // key dims held per row; dims >= d are zero
#define ICB_ROWF 128          // row stride in floats: 512 B = exactly four 128-B lines (tail kept in F.tail)
#define ICB_NPROJ 8           // NUM_PROJECTIONS (dci.py:44)
#define ICB_EXHAUSTIVE 64     // EXHAUSTIVE_NODE_LIMIT (dci.py:41)
#define ICB_MAX_WINDOW 8
#define ICB_MAX_SINK 8
#define ICB_MAX_G 8
#define ICB_ROOT_OWNER (-1)
#define ICB_LV_TRACK 16      // levels with tracked point counts / max node sizes (search start level)

// Sticky per-tree error bits (host maps them to the reference's exceptions).
enum {
  ICB_ERR_CAP_NODES = 1 << 0,
  ICB_ERR_CAP_MEMBERS = 1 << 1,
  ICB_ERR_CAP_PAGES = 1 << 2,
  ICB_ERR_CAP_OWN = 1 << 3,
  ICB_ERR_CAP_TOKENS = 1 << 4,
  ICB_ERR_DUP_ID = 1 << 5,
  ICB_ERR_EMPTY_TREE = 1 << 6,
  ICB_ERR_ZERO_QUERY = 1 << 7,
  ICB_ERR_UNMAPPED = 1 << 8,
  ICB_ERR_CAP_SCRATCH = 1 << 9,
  ICB_ERR_PDCI_SIZE = 1 << 10,
  ICB_ERR_WINDOW = 1 << 11,
};

struct TreeMeta {
  int levels;        // number of levels (0 = empty)
  int top_node;
  int n_nodes;
  int next_page;     // TierStore page-id counter (pagestore.py:138-149)
  int member_top;    // bump pointer into the member pool
  int own_top;       // bump pointer into the own list
  int n_points;
  int n_dirs;        // P-DCI direction cache entries used
  int n_window;      // window pages (oldest first in win[])
  int n_sink;
  int win[ICB_MAX_WINDOW];
  int sink[ICB_MAX_SINK];
  int err;
  int n_entropy;
  uint32_t entropy[8];   // SeedSequence run entropy words
  double c;          // KeyScale.c
  Pcg64 rng;         // level stream (spawn_key=(0,)), continues across inserts
  unsigned long long query_count, distance_evals, scale_clamps;
  unsigned long long rows_read;      // lifted rows streamed by the search (union of heads)
  unsigned long long owner_rereads;  // rows re-read because a survivor heads its own child node
  // Level summary for the search start (search.cuh start_level): points per
  // exact top level, the largest node per level, and the list of points with
  // top level >= 2 (unordered).  lv_ovf: a level >= ICB_LV_TRACK exists or the
  // upper list overflowed -- the search then starts at the top node.
  int lvl_count[ICB_LV_TRACK];
  int lvl_maxnode[ICB_LV_TRACK];
  int n_upper;
  int lv_ovf;
  int pc_top;        // P-DCI ladder cache: bump pointer into the tree's arena (entries)
};

struct ForestView {
  int T, dim, dim_v, s, kv_bf16;
  int dkp, dvp;       // page row strides (dim, dim_v rounded up to 4; padding stays zero)
  int tok_cap, node_cap, page_cap, member_cap, own_cap, dirs_cap;
  double r;
  TreeMeta* meta;
  float* lift;        // [T][tok_cap][128]
  float* tail;        // [T][tok_cap]
  int8_t* level;      // [T][tok_cap]  top level (0 = not indexed)
  int* own_base;      // [T][tok_cap]  own(p, lv) = own_list[own_base[p] + lv - 1]
  int* tok2page;      // [T][tok_cap]
  int* own_list;      // [T][own_cap]
  int* own1;          // [T][tok_cap]  own(p, 1) for points of top >= 2 (the search's union fast path)
  int* node_level;    // [T][node_cap]
  int* node_parent;
  int* node_owner;
  int* node_off;      // offset into members
  int* node_size;
  int* node_capm;     // member capacity of the node's block
  int* node_lastpage; // leaves: last page id (-1 none)
  int* node_dirs;     // P-DCI direction cache slot (-1 none)
  int* node_opos;     // position of the owner within the node's members (-1: root node)
  int* members;       // [T][member_cap] token ids
  int* page_fill;     // [T][page_cap]
  int8_t* page_role;  // [T][page_cap] 0 none, 1 sink, 2 window, 3 indexed
  int* page_tok;      // [T][page_cap][s]
  void* page_k;       // [T][page_cap][s][dim]  (fp32 or bf16)
  void* page_v;       // [T][page_cap][s][dim_v]
  double* dirs;       // [T][dirs_cap][8][dim+1]
  uint32_t* prev_sel; // [T][page_cap/32 + 1] residency: previous step's selection
  int* upper;         // [T][upper_cap] points with top level >= 2
  int upper_cap;
  // P-DCI ladder cache (query independent, per node of > 64 members): member
  // projections on the node's 8 directions and, per direction, the members in
  // (projection, id) order and each member's rank.  Valid while the node's
  // size equals node_pcm (members are only ever appended).
  int* node_pc;       // [T][node_cap] arena offset of the node's entries (-1: none)
  int* node_pcm;      // [T][node_cap] member count the entries describe
  int* node_pccap;    // [T][node_cap] entries reserved
  double* pc_proj;    // [T][pc_cap][8] projection of member i on direction j
  int* pc_ord;        // [T][pc_cap][8] entry (off + r, j): member index of rank r on direction j
  int* pc_pos;        // [T][pc_cap][8] entry (off + i, j): rank of member i on direction j
  int pc_cap;
  // KV offload (icb_forest_config.kv_host): page_k / page_v are the pinned,
  // mapped host store; pages a step attends are gathered into a per-tree HBM
  // pool of pool_cap page slots (pagestore.py:169-215 backload / evict)
  int kv_host, pool_cap;
  void* pool_k;       // [T][pool_cap][s][dkp]
  void* pool_v;       // [T][pool_cap][s][dvp]
  int* page_slot;     // [T][page_cap] pool slot of a resident page, -1 if not resident
  int* slot_page;     // [T][pool_cap] page held by a slot, -1 if free
  int* pool_tmp;      // [T][2 * pool_cap] gather scratch (free slots, pages to copy)
  long long* pool_bytes; // [T] bytes gathered host -> pool so far

  __device__ __forceinline__ size_t tk(int t, int tok) const { return (size_t)t * tok_cap + tok; }
  __device__ __forceinline__ size_t nd(int t, int n) const { return (size_t)t * node_cap + n; }
  __device__ __forceinline__ size_t pg(int t, int p) const { return (size_t)t * page_cap + p; }
  __device__ __forceinline__ const float* row(int t, int tok) const {
    return lift + ((size_t)t * tok_cap + tok) * ICB_ROWF;
  }
  __device__ __forceinline__ int own(int t, int p, int lv) const {
    return own_list[(size_t)t * own_cap + own_base[tk(t, p)] + lv - 1];
  }
  __device__ __forceinline__ int* mem(int t) const { return members + (size_t)t * member_cap; }
  __device__ __forceinline__ int* upl(int t) const { return upper + (size_t)t * upper_cap; }
  __device__ __forceinline__ int pwords() const { return page_cap / 32 + 1; }
};

// ---------------------------------------------------------------------------
// numerics

// Squared lifted distance in fp32 with the fixed order the oracle restates
// (oracle/c/oracle_nn.c:oracle_d2_fp32): lane l of a warp owns dims
// 4l..4l+3, d_i = p_i - q_i, s = fma(d3, d3, fma(d2, d2, fma(d1, d1, d0*d0))),
// xor butterfly 16,8,4,2,1 (plain adds), then d2 = fma(dt, dt, s) with
// dt = tail - q_tail.  Every operation is an explicit IEEE op (no contraction).
__device__ __forceinline__ float lane_sq4(float4 p, float4 q) {
  float a = __fsub_rn(p.x, q.x), b = __fsub_rn(p.y, q.y);
  float c = __fsub_rn(p.z, q.z), d = __fsub_rn(p.w, q.w);
  return __fmaf_rn(d, d, __fmaf_rn(c, c, __fmaf_rn(b, b, __fmul_rn(a, a))));
}

// The same lane partial for two heads at once with Blackwell's packed fp32
// (FADD2 / FMUL2 / FFMA2): element-wise IEEE results identical to lane_sq4.
__device__ __forceinline__ unsigned long long pack_f2(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ unsigned long long lane_sq4_x2_packed(float4 p, const unsigned long long (&q2)[4]) {
  unsigned long long d[4], s;
  const float pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long pp = pack_f2(pv[i], pv[i]);
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d[i]) : "l"(pp), "l"(q2[i]));
  }
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(s) : "l"(d[0]));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s) : "l"(d[1]), "l"(s));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s) : "l"(d[2]), "l"(s));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s) : "l"(d[3]), "l"(s));
  return s;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long c;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(c) : "l"(a), "l"(b));
  return c;
}
__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int o) {
  const unsigned lo = __shfl_xor_sync(0xffffffffu, (unsigned)v, o);
  const unsigned hi = __shfl_xor_sync(0xffffffffu, (unsigned)(v >> 32), o);
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ float2 lane_sq4_x2(float4 p, const unsigned long long (&q2)[4]) {
  unsigned long long d[4], s;
  const float pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long pp = pack_f2(pv[i], pv[i]);
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d[i]) : "l"(pp), "l"(q2[i]));
  }
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(s) : "l"(d[0]));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s) : "l"(d[1]), "l"(s));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s) : "l"(d[2]), "l"(s));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s) : "l"(d[3]), "l"(s));
  return make_float2(__uint_as_float((unsigned)s), __uint_as_float((unsigned)(s >> 32)));
}
__device__ __forceinline__ float warp_sum_butterfly(float s) {
  s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 16));
  s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 8));
  s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  return s;
}
__device__ __forceinline__ float d2_finish(float s, float pt, float qt) {
  float dt = __fsub_rn(pt, qt);
  return __fmaf_rn(dt, dt, s);
}

__device__ __forceinline__ unsigned long long make_key(float d2, int id) {
  return ((unsigned long long)__float_as_uint(d2) << 32) | (unsigned)id;
}
__device__ __forceinline__ int key_id(unsigned long long k) { return (int)(unsigned)(k & 0xffffffffu); }

// NumPy pairwise summation (numpy/core/src/umath/loops_utils.h.src) for one
// row held in memory, n <= 256.  Single thread.
__device__ __forceinline__ double pairwise_block(const double* a, int n) {
  if (n < 8) {
    double r = n > 0 ? a[0] : 0.0;
    for (int i = 1; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int lim = n - (n % 8);
  for (int i = 8; i < lim; i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (int i = lim; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}
__device__ __forceinline__ double pairwise_sum(const double* a, int n) {
  if (n <= 128) return pairwise_block(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_block(a, n2), pairwise_block(a + n2, n - n2));
}

// ---------------------------------------------------------------------------
// block helpers

template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int v, int* sm /* >= NT/32+1 */, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NT / 32 ? sm[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) sm[lane] = w;
  }
  __syncthreads();
  int before = (warp > 0 ? sm[warp - 1] : 0) + x - v;
  total = sm[NT / 32 - 1];
  __syncthreads();
  return before;
}

// V independent exclusive scans (one int each per thread) with one pair of
// block barriers; sm holds V * (NT / 32) ints.
template <int NT, int V>
__device__ __forceinline__ void block_scan_multi(const int (&v)[V], int (&ex)[V], int (&tot)[V], int* sm) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    x[k] = v[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x[k], o);
      if (lane >= o) x[k] += y;
    }
  }
  if (lane == 31)
#pragma unroll
    for (int k = 0; k < V; ++k) sm[k * NW + warp] = x[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      int w = lane < NW ? sm[k * NW + lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < NW) sm[k * NW + lane] = w;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < V; ++k) {
    ex[k] = (warp > 0 ? sm[k * NW + warp - 1] : 0) + x[k] - v[k];
    tot[k] = sm[k * NW + NW - 1];
  }
  __syncthreads();
}

__device__ __forceinline__ void set_err(TreeMeta* m, int bit) { atomicOr(&m->err, bit); }

// Level-summary upkeep for inserts (one writer per tree).
__device__ __forceinline__ void note_point_level(const ForestView& F, int t, int tok, int lv) {
  TreeMeta* m = F.meta + t;
  if (lv >= ICB_LV_TRACK) { m->lv_ovf = 1; return; }
  m->lvl_count[lv] += 1;
  if (lv >= 2) {
    if (m->n_upper < F.upper_cap) F.upl(t)[m->n_upper++] = tok;
    else m->lv_ovf = 1;
  }
}
__device__ __forceinline__ void note_node_size(TreeMeta* m, int lv, int sz) {
  if (lv < ICB_LV_TRACK && sz > m->lvl_maxnode[lv]) m->lvl_maxnode[lv] = sz;
}

// ---------------------------------------------------------------------------
// mbarrier + TMA bulk copy (cp.async.bulk) helpers

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// Ampere-style async copies (LDGSTS): 16 bytes per thread, L2-only (.cg).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <typename KT>
__device__ __forceinline__ void store_kv(KT* dst, float v);
template <>
__device__ __forceinline__ void store_kv<float>(float* dst, float v) { *dst = v; }
template <>
__device__ __forceinline__ void store_kv<__nv_bfloat16>(__nv_bfloat16* dst, float v) {
  *dst = __float2bfloat16_rn(v);
}
