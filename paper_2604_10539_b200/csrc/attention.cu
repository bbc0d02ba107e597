// Decode attention over pages: sparse_attention (attention.py:77-93) over
// sink U window U selected pages in the reference's entry order
// (engine.py:449-475), and dense full_attention for skip layers
// (attention.py:55-74, engine.py:418-422).
//
// Memory-bound: every K/V row is read once with 8/16-byte vector loads (one
// warp per page, lane l owns dims 4l..4l+3), the G query heads of a GQA group
// share each row (G logits per row), softmax is online in fp32, split-K
// partials (m, l, acc) are combined by the last CTA of each tree.
#include "attend.cuh"
#include "internal.h"

namespace icb {

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
  int ldk, ldv;                // dense mode row strides: ceil4(dim), ceil4(dim_v)
  int n_tokens;
  const int32_t* token_dev;    // dense mode: rows [0, *token_dev + 1) when set (CUDA-graph replays)
  float* out;                  // [n][G][dim_v]
  float* part;                 // [n][splits][G][2 + dim_v]
  unsigned* counter;           // [n]
  int64_t* stats;              // [n][5]
  int scalar_bytes;
  float scale_log2;            // log2(e) / sqrt(dim)
};

// Block = (tree b, split sp).  PAGED: rows come from the tree's sink, window
// and selected pages; DENSE: rows [0, n_tokens) of k/v[b].
template <typename KT, int G, bool PAGED>
__global__ void __launch_bounds__(kAttnThreads, 2) attn_kernel(ForestView F, AttnArgs A) {
  const int b = blockIdx.x, sp = blockIdx.y, S = A.splits;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = kAttnThreads / 32;
  __shared__ int s_pages[1024];
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
    const KT* K = (const KT*)F.page_k;
    const KT* V = (const KT*)F.page_v;
    // rows per chunk, loaded together (register budget: 2 CTAs / SM)
    constexpr int CH = (sizeof(KT) == 2 ? 16 : 8) / (G >= 4 ? 2 : 1) / (G >= 8 ? 2 : 1);
    // the split's page list is staged 1024 ids at a time
    for (int c0 = p0; c0 < p1; c0 += 1024) {
      const int cn = min(p1 - c0, 1024);
      __syncthreads();   // previous chunk consumed
      for (int i = threadIdx.x; i < cn; i += kAttnThreads) {
        int gi = c0 + i;
        int p;
        if (gi < m->n_sink) p = m->sink[gi];
        else if (gi < nfix) p = m->win[gi - m->n_sink];
        else p = A.pages[(size_t)b * A.pages_cap + gi - nfix];
        s_pages[i] = p;
      }
      __syncthreads();
      for (int i = warp; i < cn; i += NW) {
        const int p = s_pages[i];
        const int fill = F.page_fill[F.pg(t, p)];
        const size_t base = F.pg(t, p) * F.s;
        if constexpr (G == 4) {
          for (int r0 = 0; r0 < fill; r0 += 8)
            attend_chunk8_g4<KT>(g4, q2, K, V, base + r0, min(8, fill - r0), F.dkp, F.dvp, lane, A.dim, A.dim_v,
                                 A.scale_log2);
        } else {
          for (int r0 = 0; r0 < fill; r0 += CH)
            attend_chunk<KT, G, CH>(h, qv, K, V, base + r0, min(CH, fill - r0), F.dkp, F.dvp, lane, A.dim,
                                    A.dim_v, A.scale_log2);
        }
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
    const KT* K = (const KT*)A.k + (size_t)b * A.ld * A.ldk;
    const KT* V = (const KT*)A.v + (size_t)b * A.ld * A.ldv;
    const int ntok = A.token_dev ? *A.token_dev + 1 : A.n_tokens;
    const int r0 = (int)((long long)ntok * sp / S), r1 = (int)((long long)ntok * (sp + 1) / S);
    constexpr int CH = G == 4 ? 8 : (sizeof(KT) == 2 ? 16 : 8) / (G >= 4 ? 2 : 1) / (G >= 8 ? 2 : 1);
    for (int r = r0 + warp * CH; r < r1; r += NW * CH) {
      if constexpr (G == 4)
        attend_chunk8_g4<KT>(g4, q2, K, V, (size_t)r, min(CH, r1 - r), A.ldk, A.ldv, lane, A.dim, A.dim_v,
                             A.scale_log2);
      else
        attend_chunk<KT, G, CH>(h, qv, K, V, (size_t)r, min(CH, r1 - r), A.ldk, A.ldv, lane, A.dim, A.dim_v,
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
    const int j0 = ln * 4;
    if (j0 < A.dim_v) pg[2 + j0] = acc.x;
    if (j0 + 1 < A.dim_v) pg[3 + j0] = acc.y;
    if (j0 + 2 < A.dim_v) pg[4 + j0] = acc.z;
    if (j0 + 3 < A.dim_v) pg[5 + j0] = acc.w;
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
  if (icb_dense_flash_ok(G, dim, dim_v, kv_dtype)) {
    // TMA + tensor-core flash-decoding kernel (dense.cu): two CTAs per SM, one wave
    if (splits <= 0) splits = std::max(1, std::min((n_tokens + 1023) / 1024, (2 * 148) / n));
    float* part;
    unsigned* counter;
    int rc = ensure_attn_scratch(nullptr, (size_t)n * splits * G * (2 + 128), n, &part, &counter);
    if (rc) return rc;
    return icb_dense_flash_impl(n, G, q, k, v, ld, n_tokens, token_dev, out, splits, part, counter, st);
  }
  if (splits <= 0) splits = std::max(1, std::min((n_tokens + 255) / 256, (2 * 148) / n));   // one wave
  AttnArgs A{};
  A.n = n; A.G = G; A.dim = dim; A.dim_v = dim_v; A.splits = splits; A.q = q; A.k = k; A.v = v; A.ld = ld;
  A.n_tokens = n_tokens; A.token_dev = token_dev; A.out = out;
  A.ldk = (dim + 3) & ~3; A.ldv = (dim_v + 3) & ~3;
  // logits / sqrt(q.size) with the unpadded dimension (attention.py:70)
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
