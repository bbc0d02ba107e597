// Decode-time query: DciTree.query for G heads per tree, find_page_index and
// gqa_union fused into the epilogue (dci.py:318-364, pagestore.py:111-113,
// attention.py:96-103, engine.py:436-447).
#include "search.cuh"
#include "insert.cuh"
#include "attend.cuh"
#include "attend_mma.cuh"
#include "internal.h"

namespace icb {

__device__ unsigned long long g_search_prof[kPhases];
__device__ unsigned long long g_cta_cycles[4096];
__device__ int g_cta_sm[4096];

struct QueryArgs {
  const int32_t* trees;
  int n, G, lifted_input;
  const float* queries;
  SearchParams P;
  int32_t* out_ids;
  int k_out;
  int32_t* out_counts;
  int32_t* out_pages;
  int pages_cap;
  int32_t* out_npages;
  // fused paged attention (icb_query_attend): per tree [G][dim_v] fp32
  float* attn_out;
  int64_t* attn_stats;   // [n][5] or null
  int scalar_bytes;
  float scale_log2;
  int attn_simt;              // 1: CUDA-core attention chunks (ICB_ATTN_SIMT=1, A/B), else tensor cores when possible
  // fused decode-step prologue (icb_step_attend, the STEP kernel variant):
  // rotate the oldest window page into the tree (if rotate), then append the
  // decode token to the window, then search + attend
  int rotate;
  char* rot_scratch;          // insert slot scratch (ensure_insert_scratch)
  SlotLayout rot_SL;
  int64_t* rot_stats;         // [n][2] offload bytes, transactions (or null)
  const int32_t* app_token_dev;
  const float* app_keys;      // [n][dim]
  const float* app_values;    // [n][dim_v]
};

// Lift raw query g (geometry.py:89-98): fp64 norm in pairwise order, fp32 q/|q|.
template <int NT>
__device__ bool lift_query(SearchSmem& S, const ForestView& F, const float* q, int g) {
  for (int u = threadIdx.x; u < F.dim; u += NT) {
    double x = (double)q[u];
    S.q64[u] = __dmul_rn(x, x);
  }
  __syncthreads();
  __shared__ double s_norm;
  if (threadIdx.x == 0) s_norm = sqrt(pairwise_sum(S.q64, F.dim));
  __syncthreads();
  const double nrm = s_norm;
  for (int u = threadIdx.x; u < ICB_DPAD; u += NT)
    S.q[g][u] = (u < F.dim && nrm != 0.0) ? __double2float_rn(__ddiv_rn((double)q[u], nrm)) : 0.0f;
  if (threadIdx.x == 0) S.qt[g] = 0.0f;
  __syncthreads();
  return nrm != 0.0;
}

template <int NT, int GP, bool STEP = false>
__global__ void __launch_bounds__(NT, 512 / NT) query_kernel(ForestView F, QueryArgs A, char* scratch, SlotLayout SL) {
  __shared__ SearchSmem S;
  extern __shared__ __align__(128) unsigned char dsm[];
  GroupSmem* GSA = reinterpret_cast<GroupSmem*>(dsm);
  const int b = blockIdx.x;
  const int t = A.trees[b];
  if constexpr (STEP) {
    // this tree's rotation and window append, in Engine.decode_step order,
    // before its search: the step's slowest rotation no longer gates every
    // tree's search (shared memory is re-initialised for the search below)
    if (A.rotate) {
      const RingView RG1 = ring_view(dsm, 1);
      if (threadIdx.x == 0) S.sortbuf = reinterpret_cast<unsigned long long*>(RG1.ring);
      ring_init(RG1);
      double* dt1;
      unsigned* pb1;
      SearchScratch SS1 = slot_scratch(A.rot_scratch + (size_t)b * A.rot_SL.total, A.rot_SL, F.tok_cap, &dt1, &pb1);
      rotate_tree<NT>(S, GSA, RG1, F, SS1, t, dt1, A.rot_stats ? A.rot_stats + (size_t)b * 2 : nullptr,
                      A.scalar_bytes, nullptr);
    }
    append_tree(F, t, *A.app_token_dev, A.app_keys + (size_t)b * F.dim, A.app_values + (size_t)b * F.dim_v);
    __syncthreads();
  }
  const RingView RG = ring_view(dsm, GP);
  if (threadIdx.x == 0) S.sortbuf = reinterpret_cast<unsigned long long*>(RG.ring);
  ring_init(RG);
  const int G = A.G;
  const long long tk0 = clock64();
  double* dirs_tmp;
  unsigned* pbits;
  SearchScratch SS = slot_scratch(scratch + (size_t)b * SL.total, SL, F.tok_cap, &dirs_tmp, &pbits);
  const int L = F.meta[t].levels;
  if (L == 0) {
    if (threadIdx.x == 0) set_err(F.meta + t, ICB_ERR_EMPTY_TREE);
    for (int g = threadIdx.x; g < G; g += NT) A.out_counts[(size_t)b * G + g] = 0;
    if (threadIdx.x == 0 && A.out_npages) A.out_npages[b] = 0;
    return;
  }
  // queries
  bool ok = true;
  for (int g = 0; g < G; ++g) {
    const float* q = A.queries + ((size_t)b * G + g) * (F.dim + (A.lifted_input ? 1 : 0));
    if (A.lifted_input) {
      for (int u = threadIdx.x; u < ICB_DPAD; u += NT) S.q[g][u] = u < F.dim ? q[u] : 0.0f;
      if (threadIdx.x == 0) S.qt[g] = q[F.dim];
      __syncthreads();
    } else {
      ok = lift_query<NT>(S, F, q, g) && ok;
    }
  }
  if (!ok) {
    if (threadIdx.x == 0) set_err(F.meta + t, ICB_ERR_ZERO_QUERY);
    for (int g = threadIdx.x; g < G; g += NT) A.out_counts[(size_t)b * G + g] = 0;
    if (threadIdx.x == 0 && A.out_npages) A.out_npages[b] = 0;
    return;
  }
  if (A.P.prof && threadIdx.x == 0) atomicAdd(A.P.prof + 3, (unsigned long long)(clock64() - tk0));   // lift
  tree_search<NT, GP>(S, GSA, RG, F, SS, t, A.P, dirs_tmp);
  if (F.meta[t].err & ICB_ERR_CAP_SCRATCH) return;
  // final ranked top-k per head, token -> page bits
  long long tk1 = 0;
  if (A.P.k <= kBuf) {
    constexpr int NTG = NT / GP;
    const int grp = threadIdx.x / NTG, gtid = threadIdx.x % NTG;
    tk1 = clock64();
    const int n = finalize_groups<NT, GP>(S, GSA, F, SS, G, A.P.k);
    if (grp < G) {
      const GroupSmem& GS = GSA[grp];
      const int nw = min(n, A.k_out);
      for (int i = gtid; i < nw; i += NTG) A.out_ids[((size_t)b * G + grp) * A.k_out + i] = key_id(GS.buf[i]);
      if (gtid == 0) A.out_counts[(size_t)b * G + grp] = nw;
      if (A.out_pages) {
        for (int i = gtid; i < n; i += NTG) {
          int id = key_id(GS.buf[i]);
          int p = F.tok2page[F.tk(t, id)];
          if (p < 0 || p >= F.page_cap) set_err(F.meta + t, ICB_ERR_UNMAPPED);
          else atomicOr(pbits + (p >> 5), 1u << (p & 31));
        }
      }
    }
    __syncthreads();
  } else for (int g = 0; g < G; ++g) {
    if (min((long long)S.npool[g], A.P.k) > kSortMax) {
      if (threadIdx.x == 0) set_err(F.meta + t, ICB_ERR_CAP_SCRATCH);
    }
    int n = finalize_head<NT>(S, F, SS, g, A.P.k);
    int nw = min(n, A.k_out);
    for (int i = threadIdx.x; i < nw; i += NT)
      A.out_ids[((size_t)b * G + g) * A.k_out + i] = key_id(S.sortbuf[i]);
    if (threadIdx.x == 0) A.out_counts[(size_t)b * G + g] = nw;
    if (A.out_pages) {
      for (int i = threadIdx.x; i < n; i += NT) {
        int id = key_id(S.sortbuf[i]);
        int p = F.tok2page[F.tk(t, id)];
        if (p < 0 || p >= F.page_cap) set_err(F.meta + t, ICB_ERR_UNMAPPED);
        else atomicOr(pbits + (p >> 5), 1u << (p & 31));
      }
    }
    __syncthreads();
  }
  if (!A.out_pages) return;
  // ascending compaction of the page bitmap (gqa_union + sorted)
  const int nwords = F.page_cap / 32 + 1;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nwords; base += NT) {
    int w = base + threadIdx.x;
    unsigned bits = w < nwords ? pbits[w] : 0u;
    int tot;
    int ex = block_exclusive_scan<NT>(__popc(bits), S.wsum, tot);
    int pos = carry + ex;
    while (bits) {
      int bit = __ffs(bits) - 1;
      bits &= bits - 1;
      if (pos < A.pages_cap) A.out_pages[(size_t)b * A.pages_cap + pos] = w * 32 + bit;
      ++pos;
    }
    if (w < nwords) pbits[w] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) A.out_npages[b] = min(carry, A.pages_cap);
  if (A.P.prof && threadIdx.x == 0 && A.P.k <= kBuf) atomicAdd(A.P.prof + 7, (unsigned long long)(clock64() - tk1));
  if (A.attn_out) {
    // fused sparse attention over this tree's sink, window and selected pages
    // (the row ring is idle: it holds the warps' softmax states)
    __syncthreads();
    const int nsel = min(carry, A.pages_cap);
    const int32_t* sel = A.out_pages + (size_t)b * A.pages_cap;
    unsigned char* sm = reinterpret_cast<unsigned char*>(RG.ring);   // the idle row ring: warps' softmax states
    const float* qb = A.queries + (size_t)b * G * F.dim;
    float* ob = A.attn_out + (size_t)b * G * F.dim_v;
    int64_t* stb = A.attn_stats ? A.attn_stats + (size_t)b * 5 : nullptr;
    const long long ta = clock64();
    if (F.kv_host) {
      // KV offload: gather this step's pages into the tree's HBM pool, then
      // attend from the pool (written by this CTA: coherent loads)
      const long long moved = F.kv_bf16 ? gather_pages<__nv_bfloat16, NT>(F, t, sel, nsel, pbits)
                                        : gather_pages<float, NT>(F, t, sel, nsel, pbits);
      __shared__ unsigned long long s_moved;
      if (threadIdx.x == 0) s_moved = 0;
      __syncthreads();
      atomicAdd(&s_moved, (unsigned long long)moved);
      __syncthreads();
      if (threadIdx.x == 0) F.pool_bytes[t] += (long long)s_moved;
      if (attend_mma_ok(F, G) && !A.attn_simt) {
        attend_tree_mma<NT, false>(F, t, G, qb, sel, nsel, ob, A.scale_log2, sm,
                                   reinterpret_cast<unsigned char*>(&S.q[0][0]));
        tree_residency<NT>(F, t, sel, nsel, stb, A.scalar_bytes);
      } else if (F.kv_bf16)
        attend_tree_paged<__nv_bfloat16, GP, NT, false>(F, t, G, qb, sel, nsel, ob, stb, A.scalar_bytes,
                                                        A.scale_log2, sm);
      else
        attend_tree_paged<float, GP, NT, false>(F, t, G, qb, sel, nsel, ob, stb, A.scalar_bytes, A.scale_log2, sm);
    } else if (attend_mma_ok(F, G) && !A.attn_simt) {
      attend_tree_mma<NT, !STEP>(F, t, G, qb, sel, nsel, ob, A.scale_log2, sm,
                                 reinterpret_cast<unsigned char*>(&S.q[0][0]));
      tree_residency<NT>(F, t, sel, nsel, stb, A.scalar_bytes);
    } else if (F.kv_bf16) {
      attend_tree_paged<__nv_bfloat16, GP, NT, !STEP>(F, t, G, qb, sel, nsel, ob, stb, A.scalar_bytes, A.scale_log2, sm);
    } else {
      attend_tree_paged<float, GP, NT, !STEP>(F, t, G, qb, sel, nsel, ob, stb, A.scalar_bytes, A.scale_log2, sm);
    }
    if (A.P.prof && threadIdx.x == 0) atomicAdd(A.P.prof + 8, (unsigned long long)(clock64() - ta));
  }
  if (A.P.prof && threadIdx.x == 0 && b < 4096) {
    // per-CTA span and SM (profiling: the skew between trees)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_cta_cycles[b] += (unsigned long long)(clock64() - tk0);
    g_cta_sm[b] = (int)smid;
  }
}

}  // namespace icb

using namespace icb;

// Phase cycle counters of the search (enabled by ICB_PROF=1; debug tool, not
// in the public header): out[0..kPhases) = loop, union, scan + row list,
// lift + start, stream, P-DCI + counters, selection, final top-k + pages,
// fused attention; out[kPhases..kPhases + 8) = selection statistics;
// out[kPhases + 8..kPhases + 24) = row-list statistics and sub-phase cycles (g_scan_stats).
extern "C" int icb_search_cta_profile(unsigned long long* cycles, int* sm, int n, int reset) {
  ICB_CUDA(cudaDeviceSynchronize());
  ICB_CUDA(cudaMemcpyFromSymbol(cycles, g_cta_cycles, sizeof(unsigned long long) * n));
  ICB_CUDA(cudaMemcpyFromSymbol(sm, g_cta_sm, sizeof(int) * n));
  if (reset) {
    static unsigned long long z[4096] = {};
    ICB_CUDA(cudaMemcpyToSymbol(g_cta_cycles, z, sizeof(z)));
  }
  return ICB_OK;
}

extern "C" int icb_search_profile(unsigned long long* out, int reset) {
  ICB_CUDA(cudaDeviceSynchronize());
  ICB_CUDA(cudaMemcpyFromSymbol(out, g_search_prof, sizeof(unsigned long long) * kPhases));
  ICB_CUDA(cudaMemcpyFromSymbol(out + kPhases, g_topb_stats, sizeof(unsigned long long) * 8));
  ICB_CUDA(cudaMemcpyFromSymbol(out + kPhases + 8, g_scan_stats, sizeof(unsigned long long) * 16));
  if (reset) {
    unsigned long long z[16] = {};
    ICB_CUDA(cudaMemcpyToSymbol(g_search_prof, z, sizeof(unsigned long long) * kPhases));
    ICB_CUDA(cudaMemcpyToSymbol(g_topb_stats, z, sizeof(unsigned long long) * 8));
    ICB_CUDA(cudaMemcpyToSymbol(g_scan_stats, z, sizeof(unsigned long long) * 16));
  }
  return ICB_OK;
}

// Per-call scratch: one slot per tree in the call (grown and zeroed on demand).
int ensure_query_scratch(icb_forest* f, int n, int G, cudaStream_t st, char** out, SlotLayout* sl) {
  const auto& c = f->cfg;
  SlotLayout L = slot_layout(G, c.tok_cap, c.node_cap, c.page_cap, c.dim);
  size_t need = L.total * (size_t)n;
  if (need > f->qscratch_bytes) {
    if (f->qscratch) ICB_CUDA(cudaFree(f->qscratch));
    f->qscratch = nullptr;
    f->qscratch_bytes = 0;
    ICB_CUDA(cudaMalloc(&f->qscratch, need));
    ICB_CUDA(cudaMemset(f->qscratch, 0, need));   // mark arrays must start zero
    f->qscratch_bytes = need;
    f->qscratch_G = G;
  } else if (f->qscratch_G != G) {
    // the slot layout depends on G: mark arrays move, so re-zero everything
    ICB_CUDA(cudaMemsetAsync(f->qscratch, 0, f->qscratch_bytes, st));
    f->qscratch_G = G;
  }
  *out = (char*)f->qscratch;
  *sl = L;
  (void)st;
  return ICB_OK;
}

int ensure_insert_scratch(icb_forest* f, int n, char** out, SlotLayout* lay);   // insert.cu

int icb_query_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries,
                   int32_t lifted_input, int32_t k, int64_t beam, int64_t visit_cap, int32_t target_level,
                   int32_t* out_ids, int32_t k_out, int32_t* out_counts, int32_t* out_pages,
                   int32_t pages_cap, int32_t* out_npages, cudaStream_t st, float* attn_out,
                   int64_t* attn_stats, int32_t scalar_bytes, const StepOpts* step) {
  if (n <= 0) return ICB_OK;
  if (step && (!attn_out || !step->token_dev || !step->keys || !step->values)) {
    icb_set_error(ICB_E_INPUT, "decode step needs attention outputs, a device token and window K/V");
    return ICB_E_INPUT;
  }
  if (step && f->view.kv_host) {
    // the step's append would write host rows its own gather reads in the same launch
    icb_set_error(ICB_E_CONFIG, "icb_step_attend does not support kv_host forests; use the separate launches");
    return ICB_E_CONFIG;
  }
  if (attn_out && (lifted_input || !out_pages)) {
    icb_set_error(ICB_E_INPUT, "fused attention needs raw queries and page outputs");
    return ICB_E_INPUT;
  }
  if (G < 1 || G > ICB_MAX_G) {
    icb_set_error(ICB_E_CONFIG, "query heads per tree must be in [1, 8]");
    return ICB_E_CONFIG;
  }
  char* scratch;
  SlotLayout SL;
  int rc = ensure_query_scratch(f, n, G, st, &scratch, &SL);
  if (rc) return rc;
  QueryArgs A{};
  A.trees = trees; A.n = n; A.G = G; A.lifted_input = lifted_input; A.queries = queries;
  A.P.G = G; A.P.k = k; A.P.beam = beam; A.P.visit_cap = visit_cap; A.P.target = target_level;
  A.P.prof = nullptr;
  if (getenv("ICB_PROF")) ICB_CUDA(cudaGetSymbolAddress((void**)&A.P.prof, g_search_prof));
  A.out_ids = out_ids; A.k_out = k_out; A.out_counts = out_counts; A.out_pages = out_pages;
  A.pages_cap = pages_cap; A.out_npages = out_npages;
  A.attn_out = attn_out; A.attn_stats = attn_stats; A.scalar_bytes = scalar_bytes;
  A.scale_log2 = (float)(1.4426950408889634 / sqrt((double)f->cfg.dim));
  A.attn_simt = getenv("ICB_ATTN_SIMT") != nullptr;
  if (step) {
    A.rotate = step->rotate;
    if (step->rotate && (rc = ensure_insert_scratch(f, n, &A.rot_scratch, &A.rot_SL))) return rc;
    A.rot_stats = step->rot_stats;
    A.app_token_dev = step->token_dev;
    A.app_keys = step->keys;
    A.app_values = step->values;
  }
  const int GP = G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : 8;
  size_t dsm = search_dsm_bytes(GP);
  switch (GP) {
#define ICB_LAUNCH_Q(gp)                                                                                  \
  case gp:                                                                                                \
    if (step) {                                                                                           \
      ICB_CUDA(cudaFuncSetAttribute(query_kernel<kSearchThreads, gp, true>,                               \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));              \
      query_kernel<kSearchThreads, gp, true><<<n, kSearchThreads, dsm, st>>>(f->view, A, scratch, SL);    \
    } else {                                                                                              \
      ICB_CUDA(cudaFuncSetAttribute(query_kernel<kSearchThreads, gp>,                                     \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));              \
      query_kernel<kSearchThreads, gp><<<n, kSearchThreads, dsm, st>>>(f->view, A, scratch, SL);          \
    }                                                                                                     \
    break;
    ICB_LAUNCH_Q(1)
    ICB_LAUNCH_Q(2)
    ICB_LAUNCH_Q(4)
    ICB_LAUNCH_Q(8)
#undef ICB_LAUNCH_Q
  }
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

namespace icb {
// select_with_reuse for a non-anchor layer (engine.py:331-363): the anchor
// tree's ranked token lists (all G heads) mapped through THIS tree's page
// table, sorted unique (find_page_index, pagestore.py:111-113).  One CTA per
// tree; the page bitmap lives in shared memory.
__global__ void __launch_bounds__(256) pages_from_tokens_kernel(ForestView F, const int32_t* trees,
                                                                 const int32_t* src_rows, const int32_t* src_ids,
                                                                 const int32_t* src_counts, int G, int k_stride,
                                                                 int32_t* out_pages, int pages_cap,
                                                                 int32_t* out_npages) {
  extern __shared__ unsigned pbits_s[];
  __shared__ int wsum[256 / 32 + 1];
  __shared__ int carry;
  const int b = blockIdx.x, t = trees[b], sr = src_rows[b];
  const int nwords = F.page_cap / 32 + 1;
  for (int w = threadIdx.x; w < nwords; w += blockDim.x) pbits_s[w] = 0u;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int g = 0; g < G; ++g) {
    const int cnt = src_counts[(size_t)sr * G + g];
    const int32_t* ids = src_ids + ((size_t)sr * G + g) * k_stride;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const int tok = ids[i];
      const int p = (tok >= 0 && tok < F.tok_cap) ? F.tok2page[F.tk(t, tok)] : -1;
      if (p < 0 || p >= F.page_cap) set_err(F.meta + t, ICB_ERR_UNMAPPED);
      else atomicOr(pbits_s + (p >> 5), 1u << (p & 31));
    }
  }
  __syncthreads();
  for (int base = 0; base < nwords; base += blockDim.x) {
    const int w = base + threadIdx.x;
    unsigned bits = w < nwords ? pbits_s[w] : 0u;
    int tot;
    const int ex = block_exclusive_scan<256>(__popc(bits), wsum, tot);
    int pos = carry + ex;
    while (bits) {
      const int bit = __ffs(bits) - 1;
      bits &= bits - 1;
      if (pos < pages_cap) out_pages[(size_t)b * pages_cap + pos] = w * 32 + bit;
      ++pos;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) out_npages[b] = min(carry, pages_cap);
}
}  // namespace icb

int icb_pages_from_tokens_impl(icb_forest* f, const int32_t* trees, int32_t n, const int32_t* src_rows,
                               const int32_t* src_ids, const int32_t* src_counts, int32_t G, int32_t k_stride,
                               int32_t* out_pages, int32_t pages_cap, int32_t* out_npages, cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  const size_t smem = (size_t)(f->cfg.page_cap / 32 + 1) * 4;
  if (smem > 200 * 1024) { icb_set_error(ICB_E_CONFIG, "page bitmap exceeds shared memory"); return ICB_E_CONFIG; }
  ICB_CUDA(cudaFuncSetAttribute(pages_from_tokens_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  pages_from_tokens_kernel<<<n, 256, smem, st>>>(f->view, trees, src_rows, src_ids, src_counts, G, k_stride,
                                                 out_pages, pages_cap, out_npages);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

namespace icb {
// DciTree.pdci_query (dci.py:282-298, :300-314): the k nearest members of one
// node to a lifted query, ranked by (d2, id) -- all members when the node is
// small or the visit cap covers it, else its P-DCI visit list (visit_cap
// evaluations).  One CTA.
template <int NT>
__global__ void __launch_bounds__(NT) node_query_kernel(ForestView F, int t, int node, const float* q, long long k,
                                                        long long visit_cap, int32_t* out_ids, int32_t* out_count,
                                                        char* scratch, SlotLayout SL) {
  __shared__ SearchSmem S;
  extern __shared__ __align__(128) unsigned char dsm[];
  const RingView RG = ring_view(dsm, 1);
  if (threadIdx.x == 0) S.sortbuf = reinterpret_cast<unsigned long long*>(RG.ring);
  double* dirs_tmp;
  unsigned* pbits;
  SearchScratch SS = slot_scratch(scratch, SL, F.tok_cap, &dirs_tmp, &pbits);
  TreeMeta* m = F.meta + t;
  if (node < 0 || node >= m->n_nodes) {
    if (threadIdx.x == 0) { set_err(m, ICB_ERR_EMPTY_TREE); *out_count = 0; }
    return;
  }
  for (int u = threadIdx.x; u < ICB_DPAD; u += NT) S.q[0][u] = u < F.dim ? q[u] : 0.0f;
  if (threadIdx.x == 0) S.qt[0] = q[F.dim];
  __syncthreads();
  const size_t x = F.nd(t, node);
  const int sz = F.node_size[x];
  const int* list = F.mem(t) + F.node_off[x];
  int cnt = sz;
  if (sz > ICB_EXHAUSTIVE && (long long)sz > visit_cap) {
    cnt = pdci_visit<NT>(S, F, SS, t, node, 0, visit_cap, dirs_tmp);
    list = SS.vis;
  }
  eval_list_one_head<NT>(S, F, t, list, cnt, 0, SS.cand);
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(&m->distance_evals, (unsigned long long)cnt);
  int n = (int)min((long long)cnt, k);
  if (n > kSortMax) { if (threadIdx.x == 0) set_err(m, ICB_ERR_CAP_SCRATCH); n = kSortMax; }
  const int got = block_select<NT>(S, SS.cand, cnt, n, S.sortbuf, nullptr, 0, nullptr);
  block_sort<NT>(S, got);
  for (int i = threadIdx.x; i < got; i += NT) out_ids[i] = key_id(S.sortbuf[i]);
  if (threadIdx.x == 0) *out_count = got;
}
}  // namespace icb

namespace icb {
// Warm the P-DCI caches of freshly built trees (kWarmSplit CTAs per tree, each
// taking every kWarmSplit-th chunk of 2048 nodes): directions
// and ladder entries of every node the decode path visits with P-DCI --
// levels >= 2 above 64 members (insert parent searches, visit cap 64) and
// leaves above the query visit cap -- so no later search pays for them.
template <int NT>
__global__ void __launch_bounds__(NT) pdci_warm_kernel(ForestView F, const int32_t* trees, long long qcap,
                                                       double* tmp_dirs) {
  __shared__ SearchSmem S;
  __shared__ int s_list[512], s_n;
  extern __shared__ __align__(128) unsigned char dsm[];
  const RingView RG = ring_view(dsm, 1);
  if (threadIdx.x == 0) S.sortbuf = reinterpret_cast<unsigned long long*>(RG.ring);
  const int t = trees[blockIdx.x];
  const int nn = F.meta[t].n_nodes;
  double* tmp = tmp_dirs + ((size_t)blockIdx.x * gridDim.y + blockIdx.y) * ICB_NPROJ * (F.dim + 1);
  for (int base = blockIdx.y * 512 * 4; base < nn; base += gridDim.y * 512 * 4) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int node = base + threadIdx.x; node < min(nn, base + 512 * 4); node += NT) {
      const size_t x = F.nd(t, node);
      const int sz = F.node_size[x], lv = F.node_level[x];
      if (sz > ICB_EXHAUSTIVE && sz <= kPdciSort && (lv >= 2 || sz > qcap)) {
        const int at = atomicAdd(&s_n, 1);
        if (at < 512) s_list[at] = node;
      }
    }
    __syncthreads();
    const int cnt = min(s_n, 512);
    for (int i = 0; i < cnt; ++i) {
      const int node = s_list[i];
      const size_t x = F.nd(t, node);
      const double* dirs = pdci_dirs<NT>(F, t, node, tmp);
      if (F.node_dirs[x] < 0) break;   // direction cache full
      pc_ensure<NT>(S, F, t, node, F.node_size[x], F.mem(t) + F.node_off[x], dirs);
    }
    __syncthreads();
  }
}
}  // namespace icb

int icb_pdci_warm_impl(icb_forest* f, const int32_t* trees, int32_t n, int64_t qcap, cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  Scratch S(st);
  constexpr int kWarmSplit = 8;
  double* tmp = S.alloc<double>((size_t)n * kWarmSplit * ICB_NPROJ * (f->view.dim + 1));
  if (!S.ok()) return S.fail();
  const size_t dsm = search_dsm_bytes(1);
  ICB_CUDA(cudaFuncSetAttribute(pdci_warm_kernel<kSearchThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)dsm));
  pdci_warm_kernel<kSearchThreads><<<dim3(n, kWarmSplit), kSearchThreads, dsm, st>>>(f->view, trees, qcap, tmp);
  return S.finish();
}

int icb_node_query_impl(icb_forest* f, int32_t tree, int32_t node, const float* q_lifted, int32_t k,
                        int64_t visit_cap, int32_t* out_ids, int32_t* out_count, cudaStream_t st) {
  char* scratch;
  SlotLayout SL;
  int rc = ensure_query_scratch(f, 1, 1, st, &scratch, &SL);
  if (rc) return rc;
  const size_t dsm = search_dsm_bytes(1);
  ICB_CUDA(cudaFuncSetAttribute(node_query_kernel<kSearchThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)dsm));
  node_query_kernel<kSearchThreads><<<1, kSearchThreads, dsm, st>>>(f->view, tree, node, q_lifted, k, visit_cap,
                                                                    out_ids, out_count, scratch, SL);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}

namespace icb {
// Attended-token masks for evaluation (engine.py:536-566): mask[b][tok] = 1
// for every token of tree trees[b]'s sink, window and selected pages.
__global__ void attended_mask_kernel(ForestView F, const int32_t* trees, const int32_t* pages, int pages_cap,
                                     const int32_t* npages, uint8_t* mask) {
  const int b = blockIdx.x, t = trees[b];
  const TreeMeta* m = F.meta + t;
  uint8_t* mk = mask + (size_t)b * F.tok_cap;
  const int nsink = m->n_sink, nfix = nsink + m->n_window, total = nfix + npages[b];
  for (int i = threadIdx.x / 32; i < total; i += blockDim.x / 32) {
    const int p = i < nsink ? m->sink[i] : i < nfix ? m->win[i - nsink] : pages[(size_t)b * pages_cap + i - nfix];
    const int fill = F.page_fill[F.pg(t, p)];
    for (int r = threadIdx.x & 31; r < fill; r += 32) {
      const int tok = F.page_tok[F.pg(t, p) * F.s + r];
      if (tok >= 0 && tok < F.tok_cap) mk[tok] = 1;
    }
  }
}
}  // namespace icb

int icb_attended_mask_impl(icb_forest* f, const int32_t* trees, int32_t n, const int32_t* pages, int32_t pages_cap,
                           const int32_t* npages, uint8_t* mask, cudaStream_t st) {
  if (n <= 0) return ICB_OK;
  ICB_CUDA(cudaMemsetAsync(mask, 0, (size_t)n * f->cfg.tok_cap, st));
  attended_mask_kernel<<<n, 256, 0, st>>>(f->view, trees, pages, pages_cap, npages, mask);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}
