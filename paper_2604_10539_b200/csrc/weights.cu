// Attention weights and exact fp64 attention for the reference-facing API.
//
// The reference's attention returns AttentionOutput(weights: {token: w},
// value_out) (attention.py:26-93) for every query head.  The decode hot path
// needs only value_out (fused into the search kernel, fp32 / bf16); these
// kernels serve the reference-shaped API around it:
//   icb_exact_attention    full_attention of one query over caller rows, all in
//                          fp64 (logits k.q / sqrt(d), max-subtracted softmax,
//                          weights @ V): the drop-in full_attention /
//                          sparse_attention (attention.py:55-93)
//   icb_attention_weights  the softmax weights of a decode step's sparse
//                          attention per tree and query head, over the attended
//                          set in entry order (sink, window, selected pages;
//                          engine.py:454-461), logits in fp64 from the stored K
//   icb_dense_weights      the same for dense planes (skip layers / fallback,
//                          engine.py:418-422)
// They are latency-bound helper launches (one CTA per query head).
#include "internal.h"

namespace icb {

constexpr int kWThreads = 256;

__device__ __forceinline__ double block_reduce(double x, bool is_max, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, x, o);
    x = is_max ? fmax(x, y) : x + y;
  }
  __syncthreads();
  if (lane == 0) sh[warp] = x;
  __syncthreads();
  double r = sh[0];
  for (int w = 1; w < nw; ++w) r = is_max ? fmax(r, sh[w]) : r + sh[w];
  return r;
}

// In-place softmax of w[0, m) (logits -> weights): w -= max; w = exp(w); w /= sum.
__device__ void block_softmax(double* w, int m, double* sh) {
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < m; i += blockDim.x) mx = fmax(mx, w[i]);
  mx = block_reduce(mx, true, sh);
  double sum = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double e = exp(w[i] - mx);
    w[i] = e;
    sum += e;
  }
  sum = block_reduce(sum, false, sh);
  for (int i = threadIdx.x; i < m; i += blockDim.x) w[i] /= sum;
}

template <typename KT>
__device__ __forceinline__ double kv_at(const void* base, size_t i) {
  if constexpr (sizeof(KT) == 2) return (double)__bfloat162float(((const __nv_bfloat16*)base)[i]);
  else return (double)((const float*)base)[i];
}

// full_attention (attention.py:55-74) in fp64 for one query.
__global__ void exact_attention_kernel(int m, int dim, int dim_v, const double* q, const double* k, const double* v,
                                       double* w, double* out) {
  __shared__ double sh[32];
  extern __shared__ double s_part[];   // [nw][dim_v]
  const double sq = sqrt((double)dim);
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double* kr = k + (size_t)i * dim;
    double s = 0.0;
    for (int j = 0; j < dim; ++j) s = fma(kr[j], q[j], s);
    w[i] = s / sq;
  }
  __syncthreads();
  block_softmax(w, m, sh);
  __syncthreads();
  // out = w @ V: warp wp sums rows wp, wp + nw, ...; lanes cover the columns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j0 = 0; j0 < dim_v; j0 += 32) {
    const int j = j0 + lane;
    double acc = 0.0;
    if (j < dim_v)
      for (int i = warp; i < m; i += nw) acc = fma(w[i], v[(size_t)i * dim_v + j], acc);
    if (j < dim_v) s_part[warp * dim_v + j] = acc;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < dim_v; j += blockDim.x) {
    double acc = 0.0;
    for (int p = 0; p < nw; ++p) acc += s_part[p * dim_v + j];
    out[j] = acc;
  }
}

// Per (tree b, head g): attended tokens in entry order and their weights.
template <typename KT>
__global__ void attention_weights_kernel(ForestView F, const int32_t* trees, int G, const float* q,
                                         const int32_t* pages, int pages_cap, const int32_t* npages,
                                         int32_t* out_tokens, double* out_w, int cap, int32_t* out_count) {
  __shared__ double sh[32];
  extern __shared__ int s_off[];   // [total + 1] token offset of each attended page
  const int b = blockIdx.x, g = blockIdx.y;
  const int t = trees[b];
  const TreeMeta* m = F.meta + t;
  const int nsink = m->n_sink, nfix = nsink + m->n_window;
  const int nsel = npages[b];
  const int total = nfix + nsel;
  auto page_at = [&](int i) {
    return i < nsink ? m->sink[i] : i < nfix ? m->win[i - nsink] : pages[(size_t)b * pages_cap + i - nfix];
  };
  if (threadIdx.x == 0) {
    int o = 0;
    for (int i = 0; i < total; ++i) {
      s_off[i] = o;
      o += F.page_fill[F.pg(t, page_at(i))];
    }
    s_off[total] = o;
  }
  __syncthreads();
  const int ntok = min(s_off[total], cap);
  if (g == 0 && threadIdx.x == 0) out_count[b] = s_off[total];
  double* w = out_w + ((size_t)b * G + g) * cap;
  const float* qg = q + ((size_t)b * G + g) * F.dim;
  const double sq = sqrt((double)F.dim);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const KT* K = (const KT*)F.page_k;
  for (int i = warp; i < total; i += nw) {
    const int p = page_at(i);
    const int fill = F.page_fill[F.pg(t, p)];
    const int o = s_off[i];
    if (lane < fill && o + lane < cap) {
      const size_t row = F.pg(t, p) * F.s + lane;
      double s = 0.0;
      for (int j = 0; j < F.dim; ++j) s = fma(kv_at<KT>(K, row * F.dkp + j), (double)qg[j], s);
      w[o + lane] = s / sq;
      if (g == 0) out_tokens[(size_t)b * cap + o + lane] = F.page_tok[F.pg(t, p) * F.s + lane];
    }
  }
  __syncthreads();
  block_softmax(w, ntok, sh);
}

// Dense planes (skip layers / fallback): weights over rows [0, n_tokens).
template <typename KT>
__global__ void dense_weights_kernel(int G, int dim, const float* q, const void* k, long long ld, int n_tokens,
                                     double* out_w) {
  __shared__ double sh[32];
  const int b = blockIdx.x, g = blockIdx.y;
  const int ldk = (dim + 3) & ~3;
  const float* qg = q + ((size_t)b * G + g) * dim;
  double* w = out_w + ((size_t)b * G + g) * n_tokens;
  const double sq = sqrt((double)dim);
  const size_t base = (size_t)b * ld * ldk;
  for (int i = threadIdx.x; i < n_tokens; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < dim; ++j) s = fma(kv_at<KT>(k, base + (size_t)i * ldk + j), (double)qg[j], s);
    w[i] = s / sq;
  }
  __syncthreads();
  block_softmax(w, n_tokens, sh);
}

}  // namespace icb

using namespace icb;

static cudaStream_t S_(void* s) { return (cudaStream_t)s; }

int icb_exact_attention(int32_t n_rows, int32_t dim, int32_t dim_v, const double* q, const double* k,
                        const double* v, double* weights, double* out, void* stream) {
  if (n_rows < 1) { icb_set_error(ICB_E_INPUT, "keys must be a non-empty sequence of vectors"); return ICB_E_INPUT; }
  if (dim < 1 || dim_v < 1) { icb_set_error(ICB_E_INPUT, "dims must be >= 1"); return ICB_E_INPUT; }
  if (!q || !k || !v || !weights || !out) { icb_set_error(ICB_E_INPUT, "null argument"); return ICB_E_INPUT; }
  const int nt = 512;
  const size_t smem = (size_t)(nt / 32) * dim_v * sizeof(double);
  if (smem > 48 * 1024) ICB_CUDA(cudaFuncSetAttribute(exact_attention_kernel,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  exact_attention_kernel<<<1, nt, smem, S_(stream)>>>(n_rows, dim, dim_v, q, k, v, weights, out);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

int icb_attention_weights(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries,
                          const int32_t* pages, int32_t pages_cap, const int32_t* npages, int32_t* out_tokens,
                          double* out_weights, int32_t cap, int32_t* out_count, void* stream) {
  if (!f || n < 0 || G < 1 || cap < 1) { icb_set_error(ICB_E_INPUT, "bad arguments"); return ICB_E_INPUT; }
  if (n == 0) return ICB_OK;
  if (!trees || !queries || !pages || !npages || !out_tokens || !out_weights || !out_count) {
    icb_set_error(ICB_E_INPUT, "null argument");
    return ICB_E_INPUT;
  }
  const size_t smem = (size_t)(ICB_MAX_SINK + ICB_MAX_WINDOW + pages_cap + 1) * sizeof(int);
  dim3 grid(n, G);
  if (f->cfg.kv_dtype == ICB_KV_BF16) {
    if (smem > 48 * 1024) ICB_CUDA(cudaFuncSetAttribute(attention_weights_kernel<__nv_bfloat16>,
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attention_weights_kernel<__nv_bfloat16><<<grid, kWThreads, smem, S_(stream)>>>(
        f->view, trees, G, queries, pages, pages_cap, npages, out_tokens, out_weights, cap, out_count);
  } else {
    if (smem > 48 * 1024) ICB_CUDA(cudaFuncSetAttribute(attention_weights_kernel<float>,
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attention_weights_kernel<float><<<grid, kWThreads, smem, S_(stream)>>>(
        f->view, trees, G, queries, pages, pages_cap, npages, out_tokens, out_weights, cap, out_count);
  }
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

int icb_dense_weights(int32_t n, int32_t G, int32_t dim, int32_t kv_dtype, const float* q, const void* k,
                      int64_t ld, int32_t n_tokens, double* out_weights, void* stream) {
  if (n < 0 || G < 1 || dim < 1 || n_tokens < 1 || n_tokens > ld) {
    icb_set_error(ICB_E_INPUT, "bad arguments");
    return ICB_E_INPUT;
  }
  if (n == 0) return ICB_OK;
  if (!q || !k || !out_weights) { icb_set_error(ICB_E_INPUT, "null argument"); return ICB_E_INPUT; }
  dim3 grid(n, G);
  if (kv_dtype == ICB_KV_BF16)
    dense_weights_kernel<__nv_bfloat16><<<grid, kWThreads, 0, S_(stream)>>>(G, dim, q, k, ld, n_tokens, out_weights);
  else
    dense_weights_kernel<float><<<grid, kWThreads, 0, S_(stream)>>>(G, dim, q, k, ld, n_tokens, out_weights);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}
