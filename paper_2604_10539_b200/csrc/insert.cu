// Dynamic insertion, window rotation and window append: kernels and C ABI
// (the device code is in insert.cuh).
#include "insert.cuh"
#include "internal.h"

namespace icb {

template <int NT>
__global__ void __launch_bounds__(NT, 512 / NT) insert_kernel(ForestView F, InsertArgs A, char* scratch, SlotLayout SL) {
  __shared__ SearchSmem S;
  extern __shared__ __align__(128) unsigned char dsm[];
  GroupSmem* GSA = reinterpret_cast<GroupSmem*>(dsm);
  const RingView RG = ring_view(dsm, 1);
  if (threadIdx.x == 0) S.sortbuf = reinterpret_cast<unsigned long long*>(RG.ring);
  ring_init(RG);
  const int b = blockIdx.x;
  const int t = A.trees[b];
  double* dirs_tmp;
  unsigned* pbits;
  SearchScratch SS = slot_scratch(scratch + (size_t)b * SL.total, SL, F.tok_cap, &dirs_tmp, &pbits);
  if (A.from_window) {
    rotate_tree<NT>(S, GSA, RG, F, SS, t, dirs_tmp, A.stats ? A.stats + (size_t)b * 2 : nullptr, A.scalar_bytes,
                    A.prof);
    return;
  }
  insert_points<NT>(S, GSA, RG, F, SS, t, dirs_tmp, A.m, [&](int e) {
    const size_t x = (size_t)b * A.m + e;
    InsertPoint p;
    p.tok = A.tokens[x];
    p.key = A.keys + x * F.dim;
    p.val = A.values ? A.values + x * F.dim_v : nullptr;
    p.src_slot = -1;
    p.given_level = A.levels ? A.levels[x] : 0;
    return p;
  }, A.out_levels ? A.out_levels + (size_t)b * A.m : (int32_t*)nullptr, A.prof);
}

// Append one decode token to the first non-full window page of each tree.
__global__ void append_window_kernel(ForestView F, const int32_t* trees, int n, int token_host, const int32_t* token_dev,
                                     const float* keys, const float* values) {
  const int token = token_dev ? *token_dev : token_host;   // device position: CUDA-graph replays
  const int b = blockIdx.x;
  const int t = trees[b];
  append_tree(F, t, token, keys + (size_t)b * F.dim, values + (size_t)b * F.dim_v);
}

// Resident (sink/window) pages at prefill.
__global__ void resident_pages_kernel(ForestView F, const int32_t* trees, int n, int role, int count,
                                      int n_tokens, const int32_t* tokens, const float* keys,
                                      const float* values) {
  const int b = blockIdx.x;
  const int t = trees[b];
  TreeMeta* m = F.meta + t;
  __shared__ int s_first;
  if (threadIdx.x == 0) {
    s_first = m->next_page;
    if (s_first + count > F.page_cap) { set_err(m, ICB_ERR_CAP_PAGES); s_first = -1; }
    else {
      m->next_page = s_first + count;
      for (int i = 0; i < count; ++i) {
        int p = s_first + i;
        F.page_role[F.pg(t, p)] = (int8_t)role;
        F.page_fill[F.pg(t, p)] = max(0, min(F.s, n_tokens - i * F.s));
        if (role == ICB_ROLE_SINK && m->n_sink < ICB_MAX_SINK) m->sink[m->n_sink++] = p;
        if (role == ICB_ROLE_WINDOW && m->n_window < ICB_MAX_WINDOW) m->win[m->n_window++] = p;
      }
    }
  }
  __syncthreads();
  if (s_first < 0) return;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = warp; e < n_tokens && e < count * F.s; e += nw) {
    int page = s_first + e / F.s, slot = e % F.s;
    int tok = tokens[(size_t)b * n_tokens + e];
    const float* k = keys + ((size_t)b * n_tokens + e) * F.dim;
    if ((threadIdx.x & 31) == 0) F.page_tok[F.pg(t, page) * F.s + slot] = tok;
    if (tok >= 0 && tok < F.tok_cap) {
      float* stash = F.lift + F.tk(t, tok) * ICB_ROWF;
      for (int j = threadIdx.x & 31; j < F.dim; j += 32) stash[j] = k[j];
    }
    write_slot(F, t, page, slot, k, values + ((size_t)b * n_tokens + e) * F.dim_v, -1);
  }
}

}  // namespace icb

using namespace icb;

int ensure_insert_scratch(icb_forest* f, int n, char** out, SlotLayout* lay) {
  const auto& c = f->cfg;
  SlotLayout L = slot_layout(1, c.tok_cap, c.node_cap, c.page_cap, c.dim);
  size_t need = L.total * (size_t)n;
  if (need > f->iscratch_bytes) {
    if (f->iscratch) ICB_CUDA(cudaFree(f->iscratch));
    f->iscratch = nullptr;
    f->iscratch_bytes = 0;
    ICB_CUDA(cudaMalloc(&f->iscratch, need));
    ICB_CUDA(cudaMemset(f->iscratch, 0, need));
    f->iscratch_bytes = need;
  }
  *out = (char*)f->iscratch;
  *lay = L;
  return ICB_OK;
}

int icb_insert_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t m, const int32_t* tokens,
                    const float* keys, const float* values, const int32_t* levels, int32_t* out_levels,
                    int from_window, int32_t scalar_bytes, int64_t* stats, cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  char* scratch;
  SlotLayout L;
  int rc = ensure_insert_scratch(f, n, &scratch, &L);
  if (rc) return rc;
  InsertArgs A{};
  A.trees = trees; A.n = n; A.m = m; A.tokens = tokens; A.keys = keys; A.values = values;
  A.levels = levels; A.out_levels = out_levels; A.from_window = from_window;
  A.scalar_bytes = scalar_bytes; A.stats = stats;
  A.prof = nullptr;
  if (getenv("ICB_PROF")) ICB_CUDA(cudaGetSymbolAddress((void**)&A.prof, g_insert_prof));
  ICB_CUDA(cudaFuncSetAttribute(insert_kernel<kSearchThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)search_dsm_bytes(1)));
  insert_kernel<kSearchThreads><<<n, kSearchThreads, search_dsm_bytes(1), st>>>(f->view, A, scratch, L);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

int icb_append_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t token, const int32_t* token_dev,
                    const float* keys, const float* values, cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  append_window_kernel<<<n, 128, 0, st>>>(f->view, trees, n, token, token_dev, keys, values);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

int icb_resident_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t role, int32_t count,
                      int32_t n_tokens, const int32_t* tokens, const float* keys, const float* values,
                      cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  resident_pages_kernel<<<n, 256, 0, st>>>(f->view, trees, n, role, count, n_tokens, tokens, keys, values);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

// Insert phase cycle counters (enabled by ICB_PROF=1): prepare, warp
// searches, block fallbacks, finish/place, segments.
extern "C" int icb_insert_tree_profile(unsigned long long* cycles, unsigned* fallbacks, int n) {
  ICB_CUDA(cudaDeviceSynchronize());
  n = n < 4096 ? n : 4096;
  ICB_CUDA(cudaMemcpyFromSymbol(cycles, g_insert_tree_cycles, sizeof(unsigned long long) * n));
  ICB_CUDA(cudaMemcpyFromSymbol(fallbacks, g_insert_tree_fallbacks, sizeof(unsigned) * n));
  return ICB_OK;
}

extern "C" int icb_insert_profile(unsigned long long* out, int reset) {
  ICB_CUDA(cudaDeviceSynchronize());
  ICB_CUDA(cudaMemcpyFromSymbol(out, g_insert_prof, sizeof(unsigned long long) * 8));
  if (reset) {
    unsigned long long z[8] = {};
    ICB_CUDA(cudaMemcpyToSymbol(g_insert_prof, z, sizeof(z)));
  }
  return ICB_OK;
}

extern "C" int icb_pdci_stats(unsigned long long* out, int reset) {
  ICB_CUDA(cudaDeviceSynchronize());
  ICB_CUDA(cudaMemcpyFromSymbol(out, icb::g_pdci_miss, sizeof(unsigned long long) * 4));
  if (reset) {
    unsigned long long z[4] = {};
    ICB_CUDA(cudaMemcpyToSymbol(icb::g_pdci_miss, z, sizeof(z)));
  }
  return ICB_OK;
}
