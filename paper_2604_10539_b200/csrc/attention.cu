// Decode attention over pages: sparse_attention (attention.py:77-93) over
// sink U window U selected pages in the reference's entry order
// (engine.py:449-475), and dense full_attention for skip layers
// (attention.py:55-74, engine.py:418-422).
//
// Memory-bound: every K/V row is read once with 8/16-byte vector loads (one
// warp per page, lane l owns dims 4l..4l+3), the G query heads of a GQA group
// share each row (G logits per row), softmax is online in fp32, split-K
// partials (m, l, acc) are combined by the last CTA of each tree.
#include "icb.cuh"
#include "internal.h"

namespace icb {

constexpr int kAttnThreads = 256;

// kernels are instantiated for G in {1,2,4,8}; other GQA ratios run padded
inline int padded_g(int G) { return G <= 2 ? G : G <= 4 ? 4 : 8; }

template <typename KT>
__device__ __forceinline__ float4 load4(const KT* p);
template <>
__device__ __forceinline__ float4 load4<float>(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16>(const __nv_bfloat16* p) {
  uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
  float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

struct AttnArgs {
  int n, G, dim, dim_v, splits;
  const int32_t* trees;        // paged mode
  const float* q;              // [n][G][dim]
  const int32_t* pages;        // [n][pages_cap]
  int pages_cap;
  const int32_t* npages;
  // dense mode
  const void* k;
  const void* v;
  long long ld;
  int n_tokens;
  const int32_t* token_dev;    // dense mode: rows [0, *token_dev + 1) when set (CUDA-graph replays)
  float* out;                  // [n][G][dim_v]
  float* part;                 // [n][splits][G][2 + dim_v]
  unsigned* counter;           // [n]
  int64_t* stats;              // [n][5]
  int scalar_bytes;
  float scale_log2;            // log2(e) / sqrt(dim)
};

struct HeadAcc {
  float m, l;
  float4 acc;
};

template <int H, int OFF>
__device__ __forceinline__ float head_sums_rest(const float (&w)[H], int lane) {
  if constexpr (H == 1) {
    float s = w[0];
#pragma unroll
    for (int o = OFF; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
  } else {
    constexpr int H2 = H / 2;
    float x[H2];
    const bool up = lane & OFF;
#pragma unroll
    for (int i = 0; i < H2; ++i) {
      float send = up ? w[i] : w[i + H2];
      x[i] = (up ? w[i + H2] : w[i]) + __shfl_xor_sync(0xffffffffu, send, OFF);
    }
    return head_sums_rest<H2, OFF / 2>(x, lane);
  }
}

// Sum of each head's lane partials transposed across heads: lane l ends with
// head l / (32/G)'s total after G/2 + G/4 + ... + (5 - log2 G) shuffles.
template <int G>
__device__ __forceinline__ float head_sums(const float (&v)[G], int lane) {
  return head_sums_rest<G, 16>(v, lane);
}

// Raw row chunks: 4 dims per lane, loaded for a whole chunk of rows before
// any of them is used (one memory round trip per chunk).
template <typename KT>
struct Raw4;
template <>
struct Raw4<float> {
  using T = float4;
  static __device__ __forceinline__ T load(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ float4 cvt(T r) { return r; }
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
};
template <>
struct Raw4<__nv_bfloat16> {
  using T = uint2;
  static __device__ __forceinline__ T load(const __nv_bfloat16* p) { return __ldg(reinterpret_cast<const uint2*>(p)); }
  static __device__ __forceinline__ float4 cvt(T u) {
    float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
    float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  static __device__ __forceinline__ T zero() { return make_uint2(0u, 0u); }
};

template <typename KT, int G>
__device__ __forceinline__ void attend_vals(HeadAcc (&h)[G], const float4 (&qv)[G], float4 k, float4 v, int lane,
                                            float scale_log2) {
  float s[G];
#pragma unroll
  for (int g = 0; g < G; ++g) s[g] = qv[g].x * k.x + qv[g].y * k.y + qv[g].z * k.z + qv[g].w * k.w;
  if constexpr (G == 1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[0] += __shfl_xor_sync(0xffffffffu, s[0], o);
  } else {
    // transposed reduction (head g's sum lands in lanes g*32/G...), then broadcast
    const float mine = head_sums<G>(s, lane);
#pragma unroll
    for (int g = 0; g < G; ++g) s[g] = __shfl_sync(0xffffffffu, mine, g * (32 / G));
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float x = s[g] * scale_log2;   // identical in every lane: the branch is warp-uniform
    if (x > h[g].m) {                    // rescale only when the running max grows
      const float a = exp2f(h[g].m - x);
      h[g].l *= a;
      h[g].acc.x *= a;
      h[g].acc.y *= a;
      h[g].acc.z *= a;
      h[g].acc.w *= a;
      h[g].m = x;
    }
    const float p = exp2f(x - h[g].m);
    h[g].l += p;
    h[g].acc.x += p * v.x;
    h[g].acc.y += p * v.y;
    h[g].acc.z += p * v.z;
    h[g].acc.w += p * v.w;
  }
}

template <typename KT, int G>
__device__ __forceinline__ void attend_row(HeadAcc (&h)[G], const float4 (&qv)[G], const KT* krow, const KT* vrow,
                                           int lane, int dim, int dim_v, float scale_log2) {
  float4 k = lane * 4 < dim ? load4<KT>(krow + lane * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 v = lane * 4 < dim_v ? load4<KT>(vrow + lane * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  attend_vals<KT, G>(h, qv, k, v, lane, scale_log2);
}

// A chunk of CH rows starting at row index `r0` of a [rows][ld] K/V pair:
// all loads first, then the rows' online-softmax updates in order.
template <typename KT, int G, int CH>
__device__ __forceinline__ void attend_chunk(HeadAcc (&h)[G], const float4 (&qv)[G], const KT* K, const KT* V,
                                             size_t r0, int nrow, int ldk, int ldv, int lane, int dim, int dim_v,
                                             float scale_log2) {
  using R = Raw4<KT>;
  typename R::T kr[CH], vr[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    kr[c] = (c < nrow && lane * 4 < dim) ? R::load(K + (r0 + c) * ldk + lane * 4) : R::zero();
    vr[c] = (c < nrow && lane * 4 < dim_v) ? R::load(V + (r0 + c) * ldv + lane * 4) : R::zero();
  }
#pragma unroll
  for (int c = 0; c < CH; ++c)
    if (c < nrow) attend_vals<KT, G>(h, qv, R::cvt(kr[c]), R::cvt(vr[c]), lane, scale_log2);
}

// G = 4: a chunk of 8 rows at once.  Scores: lane l computes, in slot jj,
// the partial dots of row jj ^ pi(l) (pi = lane bits 4..2) against the two
// head pairs (f32x2), and a transposed reduction (select-free at the row
// levels xor 16/8/4, splitting the pairs at xor 2/1) leaves lane l with the
// score of (row pi(l), head l & 3).  Softmax: one chunk max per head (xor
// 4/8/16), one exp2 per lane, the heads' rescale factors broadcast from lanes
// 0..3; P.V: each lane accumulates its 4 dims of every head from the 32
// broadcast probabilities.  Every lane keeps m and l of its own head.
struct G4State {
  float m, l;          // of head (lane & 3)
  float4 acc[4];       // dims 4l..4l+3 of every head
};

template <typename KT>
__device__ __forceinline__ void attend_chunk8_g4(G4State& st, const unsigned long long (&q2)[2][4], const KT* K,
                                                 const KT* V, size_t r0, int nrow, int ldk, int ldv, int lane,
                                                 int dim, int dim_v, float scale_log2) {
  using R = Raw4<KT>;
  const int pi = (lane >> 2) & 7;
  typename R::T kr[8], vr[8];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int rk = jj ^ pi;
    kr[jj] = (rk < nrow && lane * 4 < dim) ? R::load(K + (r0 + rk) * ldk + lane * 4) : R::zero();
    vr[jj] = (jj < nrow && lane * 4 < dim_v) ? R::load(V + (r0 + jj) * ldv + lane * 4) : R::zero();
  }
  unsigned long long v2[8][2];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const float4 k = R::cvt(kr[jj]);
#pragma unroll
    for (int hp = 0; hp < 2; ++hp) {
      unsigned long long a;
      const unsigned long long kx = pack_f2(k.x, k.x), ky = pack_f2(k.y, k.y);
      const unsigned long long kz = pack_f2(k.z, k.z), kw = pack_f2(k.w, k.w);
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(a) : "l"(kx), "l"(q2[hp][0]));
      asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(ky), "l"(q2[hp][1]));
      asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(kz), "l"(q2[hp][2]));
      asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(kw), "l"(q2[hp][3]));
      v2[jj][hp] = a;
    }
  }
#pragma unroll
  for (int jj = 0; jj < 4; ++jj)
#pragma unroll
    for (int hp = 0; hp < 2; ++hp) v2[jj][hp] = fadd2(v2[jj][hp], shfl_xor_u64(v2[jj + 4][hp], 16));
#pragma unroll
  for (int jj = 0; jj < 2; ++jj)
#pragma unroll
    for (int hp = 0; hp < 2; ++hp) v2[jj][hp] = fadd2(v2[jj][hp], shfl_xor_u64(v2[jj + 2][hp], 8));
#pragma unroll
  for (int hp = 0; hp < 2; ++hp) v2[0][hp] = fadd2(v2[0][hp], shfl_xor_u64(v2[1][hp], 4));
  const bool b1 = lane & 2, b0 = lane & 1;
  const unsigned long long w = fadd2(b1 ? v2[0][1] : v2[0][0], shfl_xor_u64(b1 ? v2[0][0] : v2[0][1], 2));
  const float wl = __uint_as_float((unsigned)w), wh = __uint_as_float((unsigned)(w >> 32));
  const float dot = (b0 ? wh : wl) + __shfl_xor_sync(0xffffffffu, b0 ? wl : wh, 1);
  const float x = pi < nrow ? dot * scale_log2 : -INFINITY;
  // chunk max of this lane's head (lanes sharing lane & 3)
  float cm = x;
  cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 4));
  cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 8));
  cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 16));
  const float mn = fmaxf(st.m, cm);
  const float alpha = exp2f(st.m - mn);   // 0 on the first chunk (m = -inf)
  const float p = exp2f(x - mn);          // 0 for masked rows
  float ps = p;
  ps += __shfl_xor_sync(0xffffffffu, ps, 4);
  ps += __shfl_xor_sync(0xffffffffu, ps, 8);
  ps += __shfl_xor_sync(0xffffffffu, ps, 16);
  st.l = st.l * alpha + ps;
  st.m = mn;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float a = __shfl_sync(0xffffffffu, alpha, h);
    st.acc[h].x *= a; st.acc[h].y *= a; st.acc[h].z *= a; st.acc[h].w *= a;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const float4 v = R::cvt(vr[r]);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float pr = __shfl_sync(0xffffffffu, p, 4 * r + h);
      st.acc[h].x = fmaf(pr, v.x, st.acc[h].x);
      st.acc[h].y = fmaf(pr, v.y, st.acc[h].y);
      st.acc[h].z = fmaf(pr, v.z, st.acc[h].z);
      st.acc[h].w = fmaf(pr, v.w, st.acc[h].w);
    }
  }
}

// Block = (tree b, split sp).  PAGED: rows come from the tree's sink, window
// and selected pages; DENSE: rows [0, n_tokens) of k/v[b].
template <typename KT, int G, bool PAGED>
__global__ void __launch_bounds__(kAttnThreads, 2) attn_kernel(ForestView F, AttnArgs A) {
  const int b = blockIdx.x, sp = blockIdx.y, S = A.splits;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = kAttnThreads / 32;
  __shared__ int s_pages[1024];
  __shared__ int s_np;
  __shared__ float s_red[kAttnThreads / 32][G][2];
  __shared__ float4 s_acc[kAttnThreads / 32][G][32];
  __shared__ bool s_last;
  const int t = PAGED ? A.trees[b] : 0;
  const int GA = A.G;   // actual heads; G is the instantiated (padded) count, extra heads see q = 0
  float4 qv[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float* q = A.q + ((size_t)b * GA + g) * A.dim;
    const int j = lane * 4;
    const bool on = g < GA;
    qv[g] = make_float4(on && j < A.dim ? q[j] : 0.f, on && j + 1 < A.dim ? q[j + 1] : 0.f,
                        on && j + 2 < A.dim ? q[j + 2] : 0.f, on && j + 3 < A.dim ? q[j + 3] : 0.f);
  }
  HeadAcc h[G];
#pragma unroll
  for (int g = 0; g < G; ++g) { h[g].m = -INFINITY; h[g].l = 0.f; h[g].acc = make_float4(0.f, 0.f, 0.f, 0.f); }
  G4State g4;   // G == 4 path (merged into h[] before the warp combine)
  unsigned long long q2[2][4];
  if constexpr (G == 4) {
    g4.m = -INFINITY; g4.l = 0.f;
#pragma unroll
    for (int g = 0; g < 4; ++g) g4.acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int hp = 0; hp < 2; ++hp) {
      q2[hp][0] = pack_f2(qv[2 * hp].x, qv[2 * hp + 1].x);
      q2[hp][1] = pack_f2(qv[2 * hp].y, qv[2 * hp + 1].y);
      q2[hp][2] = pack_f2(qv[2 * hp].z, qv[2 * hp + 1].z);
      q2[hp][3] = pack_f2(qv[2 * hp].w, qv[2 * hp + 1].w);
    }
  }

  if (PAGED) {
    // page list: sink, window, selected (entry order of engine.py:457-461)
    const TreeMeta* m = F.meta + t;
    const int nsel = A.npages[b];
    const int nfix = m->n_sink + m->n_window;
    const int total = nfix + nsel;
    const int p0 = (int)((long long)total * sp / S), p1 = (int)((long long)total * (sp + 1) / S);
    if (threadIdx.x == 0) s_np = min(p1 - p0, 1024);
    for (int i = threadIdx.x; i < p1 - p0 && i < 1024; i += kAttnThreads) {
      int gi = p0 + i;
      int p;
      if (gi < m->n_sink) p = m->sink[gi];
      else if (gi < nfix) p = m->win[gi - m->n_sink];
      else p = A.pages[(size_t)b * A.pages_cap + gi - nfix];
      s_pages[i] = p;
    }
    __syncthreads();
    const KT* K = (const KT*)F.page_k;
    const KT* V = (const KT*)F.page_v;
    // rows per chunk, loaded together (register budget: 2 CTAs / SM)
    constexpr int CH = (sizeof(KT) == 2 ? 16 : 8) / (G >= 4 ? 2 : 1) / (G >= 8 ? 2 : 1);
    for (int i = warp; i < s_np; i += NW) {
      const int p = s_pages[i];
      const int fill = F.page_fill[F.pg(t, p)];
      const size_t base = F.pg(t, p) * F.s;
      if constexpr (G == 4) {
        for (int r0 = 0; r0 < fill; r0 += 8)
          attend_chunk8_g4<KT>(g4, q2, K, V, base + r0, min(8, fill - r0), F.dkp, F.dvp, lane, A.dim, A.dim_v,
                               A.scale_log2);
      } else {
        for (int r0 = 0; r0 < fill; r0 += CH)
          attend_chunk<KT, G, CH>(h, qv, K, V, base + r0, min(CH, fill - r0), F.dkp, F.dvp, lane, A.dim, A.dim_v,
                                  A.scale_log2);
      }
    }
    // residency accounting (pagestore.py:169-215) by split 0
    if (sp == 0 && A.stats) {
      __shared__ int s_fill_sel, s_loaded, s_fill_loaded;
      if (threadIdx.x == 0) { s_fill_sel = 0; s_loaded = 0; s_fill_loaded = 0; }
      __syncthreads();
      uint32_t* bits = F.prev_sel + (size_t)t * F.pwords();
      int fs = 0, ld = 0, fl = 0;
      for (int i = threadIdx.x; i < nsel; i += kAttnThreads) {
        int p = A.pages[(size_t)b * A.pages_cap + i];
        int f = F.page_fill[F.pg(t, p)];
        fs += f;
        if (!((bits[p >> 5] >> (p & 31)) & 1u)) { ld += 1; fl += f; }
      }
      atomicAdd(&s_fill_sel, fs);
      atomicAdd(&s_loaded, ld);
      atomicAdd(&s_fill_loaded, fl);
      __syncthreads();
      for (int w = threadIdx.x; w < F.pwords(); w += kAttnThreads) bits[w] = 0u;
      __syncthreads();
      for (int i = threadIdx.x; i < nsel; i += kAttnThreads) {
        int p = A.pages[(size_t)b * A.pages_cap + i];
        atomicOr(bits + (p >> 5), 1u << (p & 31));
      }
      if (threadIdx.x == 0) {
        int64_t* st = A.stats + (size_t)b * 5;
        st[0] += nsel;
        st[1] += s_fill_sel;
        st[2] += s_loaded;
        st[3] += (int64_t)s_fill_loaded * (A.dim + A.dim_v) * A.scalar_bytes;
        st[4] += s_loaded > 0 ? 1 : 0;
      }
    }
  } else {
    const KT* K = (const KT*)A.k + (size_t)b * A.ld * A.dim;
    const KT* V = (const KT*)A.v + (size_t)b * A.ld * A.dim_v;
    const int ntok = A.token_dev ? *A.token_dev + 1 : A.n_tokens;
    const int r0 = (int)((long long)ntok * sp / S), r1 = (int)((long long)ntok * (sp + 1) / S);
    constexpr int CH = G == 4 ? 8 : (sizeof(KT) == 2 ? 16 : 8) / (G >= 4 ? 2 : 1) / (G >= 8 ? 2 : 1);
    for (int r = r0 + warp * CH; r < r1; r += NW * CH) {
      if constexpr (G == 4)
        attend_chunk8_g4<KT>(g4, q2, K, V, (size_t)r, min(CH, r1 - r), A.dim, A.dim_v, lane, A.dim, A.dim_v,
                             A.scale_log2);
      else
        attend_chunk<KT, G, CH>(h, qv, K, V, (size_t)r, min(CH, r1 - r), A.dim, A.dim_v, lane, A.dim, A.dim_v,
                                A.scale_log2);
    }
  }
  if constexpr (G == 4) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      h[g].m = __shfl_sync(0xffffffffu, g4.m, g);
      h[g].l = __shfl_sync(0xffffffffu, g4.l, g);
      h[g].acc = g4.acc[g];
    }
  }
  // combine warps
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (lane == 0) { s_red[warp][g][0] = h[g].m; s_red[warp][g][1] = h[g].l; }
    s_acc[warp][g][lane] = h[g].acc;
  }
  __syncthreads();
  float* part = A.part + ((size_t)b * S + sp) * G * (2 + A.dim_v);
  for (int x = threadIdx.x; x < G * 32; x += kAttnThreads) {
    int g = x / 32, ln = x % 32;
    float mx = -INFINITY;
    for (int w = 0; w < NW; ++w) mx = fmaxf(mx, s_red[w][g][0]);
    float l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int w = 0; w < NW; ++w) {
      float sc = s_red[w][g][0] == -INFINITY ? 0.f : exp2f(s_red[w][g][0] - mx);
      l += s_red[w][g][1] * sc;
      float4 a = s_acc[w][g][ln];
      acc.x += a.x * sc; acc.y += a.y * sc; acc.z += a.z * sc; acc.w += a.w * sc;
    }
    float* pg = part + (size_t)g * (2 + A.dim_v);
    if (ln == 0) { pg[0] = mx; pg[1] = l; }
    if (ln * 4 < A.dim_v) { pg[2 + ln * 4] = acc.x; pg[3 + ln * 4] = acc.y; pg[4 + ln * 4] = acc.z; pg[5 + ln * 4] = acc.w; }
  }
  // last CTA of this tree combines the splits
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(A.counter + b, 1u);
    s_last = (prev == (unsigned)(S - 1));
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* pb = A.part + (size_t)b * S * G * (2 + A.dim_v);
  for (int x = threadIdx.x; x < GA * A.dim_v; x += kAttnThreads) {
    int g = x / A.dim_v, j = x % A.dim_v;
    float mx = -INFINITY;
    for (int s = 0; s < S; ++s) mx = fmaxf(mx, __ldcg(pb + ((size_t)s * G + g) * (2 + A.dim_v)));
    float l = 0.f, acc = 0.f;
    for (int s = 0; s < S; ++s) {
      const float* pg = pb + ((size_t)s * G + g) * (2 + A.dim_v);
      float ms = __ldcg(pg);
      float sc = ms == -INFINITY ? 0.f : exp2f(ms - mx);
      l += __ldcg(pg + 1) * sc;
      acc += __ldcg(pg + 2 + j) * sc;
    }
    A.out[((size_t)b * GA + g) * A.dim_v + j] = acc / l;
  }
  if (threadIdx.x == 0) A.counter[b] = 0;   // ready for the next launch
}

template <typename KT, bool PAGED>
void launch_attn(int G, dim3 grid, cudaStream_t st, const ForestView& F, const AttnArgs& A) {
  switch (padded_g(G)) {
    case 1: attn_kernel<KT, 1, PAGED><<<grid, kAttnThreads, 0, st>>>(F, A); break;
    case 2: attn_kernel<KT, 2, PAGED><<<grid, kAttnThreads, 0, st>>>(F, A); break;
    case 4: attn_kernel<KT, 4, PAGED><<<grid, kAttnThreads, 0, st>>>(F, A); break;
    case 8: attn_kernel<KT, 8, PAGED><<<grid, kAttnThreads, 0, st>>>(F, A); break;
    default: break;
  }
}

}  // namespace icb

using namespace icb;

static int ensure_attn_scratch(icb_forest* f, size_t part_floats, int n, float** part, unsigned** counter) {
  static thread_local void* dense_buf = nullptr;
  static thread_local size_t dense_bytes = 0;
  void** buf = f ? &f->ascratch : &dense_buf;
  size_t* bytes = f ? &f->ascratch_bytes : &dense_bytes;
  size_t need = part_floats * 4 + 256 + (size_t)n * 4;
  if (need > *bytes) {
    if (*buf) ICB_CUDA(cudaFree(*buf));
    *buf = nullptr;
    *bytes = 0;
    ICB_CUDA(cudaMalloc(buf, need));
    ICB_CUDA(cudaMemset(*buf, 0, need));
    *bytes = need;
  }
  *counter = (unsigned*)*buf;
  *part = (float*)((char*)*buf + (((size_t)n * 4 + 255) & ~(size_t)255));
  return ICB_OK;
}

static bool valid_g(int G) { return G >= 1 && G <= 8; }

int icb_attention_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries,
                       const int32_t* pages, int32_t pages_cap, const int32_t* npages, float* out,
                       int64_t* stats, int32_t scalar_bytes, int32_t splits, cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  if (!valid_g(G)) { icb_set_error(ICB_E_CONFIG, "attention supports 1 <= G <= 8"); return ICB_E_CONFIG; }
  const auto& c = f->cfg;
  // one wave: at most 2 CTAs per SM (the kernel's register budget); each warp
  // keeps a whole row chunk in flight, so one split per tree already streams
  if (splits <= 0) splits = std::max(1, std::min(8, (2 * 148) / n));
  AttnArgs A{};
  A.n = n; A.G = G; A.dim = c.dim; A.dim_v = c.dim_v; A.splits = splits; A.trees = trees; A.q = queries;
  A.pages = pages; A.pages_cap = pages_cap; A.npages = npages; A.out = out; A.stats = stats;
  A.scalar_bytes = scalar_bytes;
  A.scale_log2 = (float)(1.4426950408889634 / sqrt((double)c.dim));
  int rc = ensure_attn_scratch(f, (size_t)n * splits * padded_g(G) * (2 + c.dim_v), n, &A.part, &A.counter);
  if (rc) return rc;
  dim3 grid(n, splits);
  if (c.kv_dtype == ICB_KV_BF16) launch_attn<__nv_bfloat16, true>(G, grid, st, f->view, A);
  else launch_attn<float, true>(G, grid, st, f->view, A);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

int icb_dense_attention_impl(int32_t n, int32_t G, int32_t dim, int32_t dim_v, int32_t kv_dtype, const float* q,
                             const void* k, const void* v, int64_t ld, int32_t n_tokens, const int32_t* token_dev,
                             float* out,
                             int32_t splits, cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  if (!valid_g(G)) { icb_set_error(ICB_E_CONFIG, "attention supports 1 <= G <= 8"); return ICB_E_CONFIG; }
  if (splits <= 0) splits = std::max(1, std::min((n_tokens + 255) / 256, (2 * 148) / n));   // one wave
  AttnArgs A{};
  A.n = n; A.G = G; A.dim = dim; A.dim_v = dim_v; A.splits = splits; A.q = q; A.k = k; A.v = v; A.ld = ld;
  A.n_tokens = n_tokens; A.token_dev = token_dev; A.out = out;
  A.scale_log2 = (float)(1.4426950408889634 / sqrt((double)dim));
  int rc = ensure_attn_scratch(nullptr, (size_t)n * splits * padded_g(G) * (2 + dim_v), n, &A.part, &A.counter);
  if (rc) return rc;
  ForestView F{};
  dim3 grid(n, splits);
  if (kv_dtype == ICB_KV_BF16) launch_attn<__nv_bfloat16, false>(G, grid, st, F, A);
  else launch_attn<float, false>(G, grid, st, F, A);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

namespace icb {
// Append one row to each of n dense K/V planes ([n][ld][dkp] / [n][ld][dvp],
// fp32 or bf16) at the device position *token_dev (the skip layers' cache).
__global__ void dense_append_kernel(int n, int dim, int dim_v, int bf16, const float* k, const float* v, void* dk,
                                    void* dv, long long ld, const int32_t* token_dev) {
  const int b = blockIdx.x;
  const int tok = *token_dev;
  if (tok < 0 || tok >= ld) return;
  const int dkp = (dim + 3) & ~3, dvp = (dim_v + 3) & ~3;
  for (int j = threadIdx.x; j < dkp + dvp; j += blockDim.x) {
    const bool isk = j < dkp;
    const int c = isk ? j : j - dkp;
    const int lim = isk ? dim : dim_v;
    const float x = c < lim ? (isk ? k[(size_t)b * dim + c] : v[(size_t)b * dim_v + c]) : 0.f;
    const size_t o = ((size_t)b * ld + tok) * (isk ? dkp : dvp) + c;
    if (bf16) (isk ? (__nv_bfloat16*)dk : (__nv_bfloat16*)dv)[o] = __float2bfloat16_rn(x);
    else (isk ? (float*)dk : (float*)dv)[o] = x;
  }
}
}  // namespace icb

int icb_dense_append_impl(int32_t n, int32_t dim, int32_t dim_v, int32_t kv_dtype, const float* k, const float* v,
                          void* dense_k, void* dense_v, int64_t ld, const int32_t* token_dev, cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  icb::dense_append_kernel<<<n, 128, 0, st>>>(n, dim, dim_v, kv_dtype == ICB_KV_BF16, k, v, dense_k, dense_v, ld,
                                              token_dev);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}
