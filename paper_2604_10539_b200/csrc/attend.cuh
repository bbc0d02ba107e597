// Decode-attention building blocks shared by the attention kernels
// (attention.cu) and the search kernel's fused epilogue (search.cu).
// full_attention / sparse_attention (attention.py:55-93) in fp32 with an
// online softmax; lane l of a warp owns dims 4l..4l+3 of every row.
#pragma once
#include "icb.cuh"

namespace icb {

constexpr int kAttnThreads = 256;

// kernels are instantiated for G in {1,2,4,8}; other GQA ratios run padded
inline int padded_g(int G) { return G <= 2 ? G : G <= 4 ? 4 : 8; }

// K/V loads: NC = true reads through the non-coherent path (ld.global.nc;
// the pages are read-only for the kernel).  NC = false (the fused decode
// step, whose rotation and window append write pages earlier in the same
// kernel) uses coherent L2 loads (ld.global.cg).
template <bool NC, typename T>
__device__ __forceinline__ T ldkv(const T* p) {
  if constexpr (NC) return __ldg(p);
  else return __ldcg(p);
}
template <typename KT, bool NC = true>
__device__ __forceinline__ float4 load4(const KT* p);
template <>
__device__ __forceinline__ float4 load4<float, true>(const float* p) {
  return ldkv<true>(reinterpret_cast<const float4*>(p));
}
template <>
__device__ __forceinline__ float4 load4<float, false>(const float* p) {
  return ldkv<false>(reinterpret_cast<const float4*>(p));
}
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16, true>(const __nv_bfloat16* p) {
  uint2 u = ldkv<true>(reinterpret_cast<const uint2*>(p));
  float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
  float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16, false>(const __nv_bfloat16* p) {
  uint2 u = ldkv<false>(reinterpret_cast<const uint2*>(p));
  float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
  float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

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
  template <bool NC>
  static __device__ __forceinline__ T load(const float* p) { return ldkv<NC>(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ float4 cvt(T r) { return r; }
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
};
template <>
struct Raw4<__nv_bfloat16> {
  using T = uint2;
  template <bool NC>
  static __device__ __forceinline__ T load(const __nv_bfloat16* p) { return ldkv<NC>(reinterpret_cast<const uint2*>(p)); }
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

template <typename KT, int G, bool NC = true>
__device__ __forceinline__ void attend_row(HeadAcc (&h)[G], const float4 (&qv)[G], const KT* krow, const KT* vrow,
                                           int lane, int dim, int dim_v, float scale_log2) {
  float4 k = lane * 4 < dim ? load4<KT, NC>(krow + lane * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 v = lane * 4 < dim_v ? load4<KT, NC>(vrow + lane * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  attend_vals<KT, G>(h, qv, k, v, lane, scale_log2);
}

// A chunk of CH rows starting at row index `r0` of a [rows][ld] K/V pair:
// all loads first, then the rows' online-softmax updates in order.
template <typename KT, int G, int CH, bool NC = true>
__device__ __forceinline__ void attend_chunk(HeadAcc (&h)[G], const float4 (&qv)[G], const KT* K, const KT* V,
                                             size_t r0, int nrow, int ldk, int ldv, int lane, int dim, int dim_v,
                                             float scale_log2) {
  using R = Raw4<KT>;
  typename R::T kr[CH], vr[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    kr[c] = (c < nrow && lane * 4 < dim) ? R::template load<NC>(K + (r0 + c) * ldk + lane * 4) : R::zero();
    vr[c] = (c < nrow && lane * 4 < dim_v) ? R::template load<NC>(V + (r0 + c) * ldv + lane * 4) : R::zero();
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

template <typename KT, bool NC = true>
__device__ __forceinline__ void attend_chunk8_g4(G4State& st, const unsigned long long (&q2)[2][4], const KT* K,
                                                 const KT* V, size_t r0, int nrow, int ldk, int ldv, int lane,
                                                 int dim, int dim_v, float scale_log2) {
  using R = Raw4<KT>;
  const int pi = (lane >> 2) & 7;
  typename R::T kr[8], vr[8];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int rk = jj ^ pi;
    kr[jj] = (rk < nrow && lane * 4 < dim) ? R::template load<NC>(K + (r0 + rk) * ldk + lane * 4) : R::zero();
    vr[jj] = (jj < nrow && lane * 4 < dim_v) ? R::template load<NC>(V + (r0 + jj) * ldv + lane * 4) : R::zero();
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


// The whole paged attention of one tree by one CTA of NT threads (the search
// kernel's fused epilogue): sparse_attention over sink, window and the
// selected pages in the reference's entry order (engine.py:457-461).  Warps
// take pages round-robin; their online-softmax states are combined in shared
// memory (no split-K).  Residency accounting as attn_kernel's split 0
// (pagestore.py:169-215).  smem: >= NT/32 * G * (2 * 4 + 32 * 16) bytes.
// KV offload (F.kv_host): make tree t's pool hold exactly the pages this step
// attends -- sink, window and the `nsel` selected pages (hot = selected U
// pinned, pagestore.py:169-215).  Resident pages outside that set are evicted,
// missing ones claim the freed slots and their filled rows are copied from the
// pinned host store (mapped; 16-byte loads, 8 in flight per thread, all of the
// tree's pages at once).  rbits: a zeroed page bitmap (page_cap bits) of
// scratch, returned zeroed.  Returns the bytes copied.
template <typename KT, int NT>
__device__ long long gather_pages(const ForestView& F, int t, const int32_t* sel, int nsel, unsigned* rbits) {
  const TreeMeta* m = F.meta + t;
  const int nsink = m->n_sink, nfix = nsink + m->n_window, total = nfix + nsel;
  int* page_slot = F.page_slot + (size_t)t * F.page_cap;
  int* slot_page = F.slot_page + (size_t)t * F.pool_cap;
  int* freel = F.pool_tmp + (size_t)t * 2 * F.pool_cap;
  int* copyl = freel + F.pool_cap;
  __shared__ int s_nfree, s_ncopy;
  auto page_at = [&](int i) { return i < nsink ? m->sink[i] : i < nfix ? m->win[i - nsink] : sel[i - nfix]; };
  for (int i = threadIdx.x; i < total; i += NT) {
    const int p = page_at(i);
    atomicOr(rbits + (p >> 5), 1u << (p & 31));
  }
  if (threadIdx.x == 0) { s_nfree = 0; s_ncopy = 0; }
  __syncthreads();
  for (int s = threadIdx.x; s < F.pool_cap; s += NT) {   // evict, collect free slots
    int p = slot_page[s];
    if (p >= 0 && !((rbits[p >> 5] >> (p & 31)) & 1u)) {
      page_slot[p] = -1;
      slot_page[s] = -1;
      p = -1;
    }
    if (p < 0) freel[atomicAdd(&s_nfree, 1)] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += NT) {        // claim slots for missing pages
    const int p = page_at(i);
    if (page_slot[p] < 0) {
      const int k = atomicAdd(&s_ncopy, 1);
      if (k < s_nfree) {
        const int s = freel[k];
        page_slot[p] = s;
        slot_page[s] = p;
        copyl[k] = p;
      } else {
        set_err(F.meta + t, ICB_ERR_CAP_SCRATCH);   // pool smaller than the step's pages
      }
    }
  }
  __syncthreads();
  // copy the filled rows: items (page, row, 16-byte chunk), K chunks then V
  const int nc = min(s_ncopy, s_nfree);
  const int ck = F.dkp * (int)sizeof(KT) / 16, cv = F.dvp * (int)sizeof(KT) / 16, cr = ck + cv;
  const long long items = (long long)nc * F.s * cr;
  const char* hk = (const char*)F.page_k;
  const char* hv = (const char*)F.page_v;
  char* pk = (char*)F.pool_k;
  char* pv = (char*)F.pool_v;
  long long bytes = 0;
  constexpr int B = 8;
  for (long long x0 = threadIdx.x; x0 < items; x0 += (long long)NT * B) {
    uint4 v[B];
    size_t dst[B];
    bool isk[B], on[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const long long x = x0 + (long long)u * NT;
      on[u] = false;
      if (x < items) {
        const int k = (int)(x / (F.s * cr));
        const int rem = (int)(x - (long long)k * F.s * cr);
        const int r = rem / cr, c = rem - r * cr;
        const int p = copyl[k];
        if (r < F.page_fill[F.pg(t, p)]) {
          isk[u] = c < ck;
          const size_t row_src = F.pg(t, p) * F.s + r;
          const size_t row_dst = ((size_t)t * F.pool_cap + page_slot[p]) * F.s + r;
          const size_t rb = (size_t)(isk[u] ? F.dkp : F.dvp) * sizeof(KT);
          const int cc = isk[u] ? c : c - ck;
          v[u] = *reinterpret_cast<const uint4*>((isk[u] ? hk : hv) + row_src * rb + (size_t)cc * 16);
          dst[u] = row_dst * rb + (size_t)cc * 16;
          on[u] = true;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (on[u]) {
        *reinterpret_cast<uint4*>((isk[u] ? pk : pv) + dst[u]) = v[u];
        bytes += 16;
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += NT) rbits[page_at(i) >> 5] = 0u;
  __syncthreads();
  return bytes;
}

// Residency accounting of one tree's step (TierStore.backload /
// evict_unselected, pagestore.py:169-215): pages of `sel` not selected last
// step are loaded; the previous-selection bitmap becomes `sel`.
template <int NT>
__device__ void tree_residency(const ForestView& F, int t, const int32_t* sel, int nsel, int64_t* stats,
                               int scalar_bytes) {
  if (!stats) return;
  __shared__ int s_fill_sel, s_loaded, s_fill_loaded;
  if (threadIdx.x == 0) { s_fill_sel = 0; s_loaded = 0; s_fill_loaded = 0; }
  __syncthreads();
  uint32_t* bits = F.prev_sel + (size_t)t * F.pwords();
  int fs = 0, ld = 0, fl = 0;
  for (int i = threadIdx.x; i < nsel; i += NT) {
    const int p = sel[i];
    const int f = F.page_fill[F.pg(t, p)];
    fs += f;
    if (!((bits[p >> 5] >> (p & 31)) & 1u)) { ld += 1; fl += f; }
  }
  atomicAdd(&s_fill_sel, fs);
  atomicAdd(&s_loaded, ld);
  atomicAdd(&s_fill_loaded, fl);
  __syncthreads();
  for (int w = threadIdx.x; w < F.pwords(); w += NT) bits[w] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < nsel; i += NT) {
    const int p = sel[i];
    atomicOr(bits + (p >> 5), 1u << (p & 31));
  }
  if (threadIdx.x == 0) {
    stats[0] += nsel;
    stats[1] += s_fill_sel;
    stats[2] += s_loaded;
    stats[3] += (int64_t)s_fill_loaded * (F.dim + F.dim_v) * scalar_bytes;
    stats[4] += s_loaded > 0 ? 1 : 0;
  }
}

template <typename KT, int G, int NT, bool NC = true>
__device__ void attend_tree_paged(const ForestView& F, int t, int GA, const float* q /*[GA][dim]*/,
                                  const int32_t* sel, int nsel, float* out /*[GA][dim_v]*/, int64_t* stats,
                                  int scalar_bytes, float scale_log2, unsigned char* smem) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float (*s_red)[G][2] = reinterpret_cast<float (*)[G][2]>(smem);
  float4 (*s_acc)[G][32] = reinterpret_cast<float4 (*)[G][32]>(smem + (size_t)NW * G * 2 * sizeof(float));
  const TreeMeta* m = F.meta + t;
  float4 qv[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float* qg = q + (size_t)g * F.dim;
    const int j = lane * 4;
    const bool on = g < GA;
    qv[g] = make_float4(on && j < F.dim ? qg[j] : 0.f, on && j + 1 < F.dim ? qg[j + 1] : 0.f,
                        on && j + 2 < F.dim ? qg[j + 2] : 0.f, on && j + 3 < F.dim ? qg[j + 3] : 0.f);
  }
  HeadAcc h[G];
#pragma unroll
  for (int g = 0; g < G; ++g) { h[g].m = -INFINITY; h[g].l = 0.f; h[g].acc = make_float4(0.f, 0.f, 0.f, 0.f); }
  G4State g4;
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
  // pages are read from the HBM pool under KV offload (gathered by the caller)
  const KT* K = (const KT*)(F.kv_host ? F.pool_k : F.page_k);
  const KT* V = (const KT*)(F.kv_host ? F.pool_v : F.page_v);
  const int nsink = m->n_sink, nfix = nsink + m->n_window, total = nfix + nsel;
  constexpr int CH = (sizeof(KT) == 2 ? 16 : 8) / (G >= 4 ? 2 : 1) / (G >= 8 ? 2 : 1);
  for (int i = warp; i < total; i += NW) {
    const int p = i < nsink ? m->sink[i] : i < nfix ? m->win[i - nsink] : sel[i - nfix];
    int slot = 0;
    if (F.kv_host) {
      slot = F.page_slot[F.pg(t, p)];
      if (slot < 0) continue;   // pool overflow (ICB_ERR_CAP_SCRATCH is set): never read outside the pool
    }
    const int fill = F.page_fill[F.pg(t, p)];
    const size_t base = F.kv_host ? ((size_t)t * F.pool_cap + slot) * F.s : F.pg(t, p) * F.s;
    if constexpr (G == 4) {
      for (int r0 = 0; r0 < fill; r0 += 8)
        attend_chunk8_g4<KT, NC>(g4, q2, K, V, base + r0, min(8, fill - r0), F.dkp, F.dvp, lane, F.dim, F.dim_v,
                             scale_log2);
    } else {
      for (int r0 = 0; r0 < fill; r0 += CH)
        attend_chunk<KT, G, CH, NC>(h, qv, K, V, base + r0, min(CH, fill - r0), F.dkp, F.dvp, lane, F.dim, F.dim_v,
                                scale_log2);
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
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (lane == 0) { s_red[warp][g][0] = h[g].m; s_red[warp][g][1] = h[g].l; }
    s_acc[warp][g][lane] = h[g].acc;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < GA * 32; x += NT) {
    const int g = x / 32, ln = x % 32;
    float mx = -INFINITY;
    for (int w = 0; w < NW; ++w) mx = fmaxf(mx, s_red[w][g][0]);
    float l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int w = 0; w < NW; ++w) {
      const float sc = s_red[w][g][0] == -INFINITY ? 0.f : exp2f(s_red[w][g][0] - mx);
      l += s_red[w][g][1] * sc;
      const float4 a = s_acc[w][g][ln];
      acc.x += a.x * sc; acc.y += a.y * sc; acc.z += a.z * sc; acc.w += a.w * sc;
    }
    float* og = out + (size_t)g * F.dim_v;
    const float inv = 1.f / l;
    if (ln * 4 + 0 < F.dim_v) og[ln * 4 + 0] = acc.x * inv;
    if (ln * 4 + 1 < F.dim_v) og[ln * 4 + 1] = acc.y * inv;
    if (ln * 4 + 2 < F.dim_v) og[ln * 4 + 2] = acc.z * inv;
    if (ln * 4 + 3 < F.dim_v) og[ln * 4 + 3] = acc.w * inv;
  }
  tree_residency<NT>(F, t, sel, nsel, stats, scalar_bytes);
}
}  // namespace icb
