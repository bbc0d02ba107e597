// Forest arena (HBM) and the C ABI entry points (include/icecache_b200.h).
#include "icb.cuh"
#include "internal.h"
#include <cstring>
#include <mutex>
#include <sys/mman.h>
#include <thread>

static thread_local std::string g_last_error;
static thread_local int g_last_code = 0;

void icb_set_error(int code, const std::string& msg) {
  g_last_code = code;
  g_last_error = msg;
}

namespace icb {

__global__ void zero_nodes_kernel(ForestView F, const int32_t* trees, int n) {
  int b = blockIdx.y;
  int t = trees[b];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < F.node_cap; i += gridDim.x * blockDim.x)
    F.node_size[F.nd(t, i)] = 0;
}

__global__ void seed_kernel(ForestView F, int t, Pcg64 g, int n_words, uint32_t w0, uint32_t w1, uint32_t w2,
                            uint32_t w3, uint32_t w4, uint32_t w5, uint32_t w6, uint32_t w7) {
  TreeMeta* m = F.meta + t;
  m->rng = g;
  m->n_entropy = n_words;
  uint32_t w[8] = {w0, w1, w2, w3, w4, w5, w6, w7};
  for (int i = 0; i < 8; ++i) m->entropy[i] = w[i];
}

}  // namespace icb

using namespace icb;

// Pinned, device-mapped host store of `bytes` (KV offload).  Pinning tens of
// GB is dominated by faulting and locking the pages one range at a time, so
// the range is mmap'ed once and registered in 1 GB chunks from parallel host
// threads.  The chunks' device addresses must continue one another (true
// when registered memory is used at its host address, UVA); otherwise, or if
// anything fails, one cudaHostAlloc does it.  *dev gets the device address.
static int pin_host_store(icb_forest* f, size_t bytes, void** dev) {
  int can_use_host_ptr = 0, d = 0;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&can_use_host_ptr, cudaDevAttrCanUseHostPointerForRegisteredMem, d);
  const size_t chunk = 1ull << 30;
  if (can_use_host_ptr && bytes >= 2 * chunk) {
    void* h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (h != MAP_FAILED) {
      const size_t n = (bytes + chunk - 1) / chunk;
      std::vector<cudaError_t> err(n, cudaSuccess);
      const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
      std::vector<std::thread> pool;
      for (unsigned w = 0; w < nt; ++w)
        pool.emplace_back([&, w]() {
          cudaSetDevice(d);
          for (size_t i = w; i < n; i += nt) {
            const size_t off = i * chunk, len = std::min(chunk, bytes - off);
            err[i] = cudaHostRegister((char*)h + off, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
          }
        });
      for (auto& th : pool) th.join();
      bool ok = true;
      for (size_t i = 0; i < n && ok; ++i) {
        void* dp = nullptr;
        ok = err[i] == cudaSuccess && cudaHostGetDevicePointer(&dp, (char*)h + i * chunk, 0) == cudaSuccess &&
             dp == (char*)h + i * chunk;
      }
      if (ok) {
        f->host_regs.push_back({h, bytes});
        *dev = h;
        return ICB_OK;
      }
      for (size_t i = 0; i < n; ++i)
        if (err[i] == cudaSuccess) cudaHostUnregister((char*)h + i * chunk);
      cudaGetLastError();
      munmap(h, bytes);
    }
  }
  void* h = nullptr;
  cudaError_t e = cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) { icb_set_error(ICB_E_CUDA, cudaGetErrorString(e)); return ICB_E_CUDA; }
  f->host_allocs.push_back(h);
  e = cudaHostGetDevicePointer(dev, h, 0);
  if (e != cudaSuccess) { icb_set_error(ICB_E_CUDA, cudaGetErrorString(e)); return ICB_E_CUDA; }
  return ICB_OK;
}

void zero_node_sizes(icb_forest* f, const int32_t* trees, int n, cudaStream_t st) {
  dim3 grid((f->cfg.node_cap + 255) / 256, n);
  zero_nodes_kernel<<<grid, 256, 0, st>>>(f->view, trees, n);
}

static cudaStream_t S_(void* s) { return (cudaStream_t)s; }

#define ICB_TRY(expr)            \
  do {                           \
    int _rc = (expr);            \
    if (_rc != ICB_OK) return _rc; \
  } while (0)

template <typename T>
static int falloc(icb_forest* f, T** p, size_t n, int fill_byte) {
  void* q = nullptr;
  size_t bytes = std::max<size_t>(n * sizeof(T), 16);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) {
    icb_set_error(ICB_E_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    return ICB_E_CUDA;
  }
  e = cudaMemset(q, fill_byte, bytes);
  if (e != cudaSuccess) {
    icb_set_error(ICB_E_CUDA, cudaGetErrorString(e));
    return ICB_E_CUDA;
  }
  f->allocs.push_back(q);
  *p = (T*)q;
  return ICB_OK;
}

extern "C" {

const char* icb_last_error(void) { return g_last_error.c_str(); }
int icb_version(void) { return 1; }

int icb_forest_create(const icb_forest_config* cfg, icb_forest** out) {
  if (!cfg || !out) { icb_set_error(ICB_E_INPUT, "null argument"); return ICB_E_INPUT; }
  const auto& c = *cfg;
  if (c.n_trees < 1 || c.dim < 1 || c.dim > ICB_DPAD || c.dim_v < 1 || c.dim_v > ICB_DPAD) {
    icb_set_error(ICB_E_CONFIG, "dims must be in [1, 128] and n_trees >= 1");
    return ICB_E_CONFIG;
  }
  if (c.page_size < 2 || c.page_size > 64) { icb_set_error(ICB_E_CONFIG, "page_size must be in [2, 64]"); return ICB_E_CONFIG; }
  if (!(c.promotion_ratio > 0.0 && c.promotion_ratio < 1.0)) {
    icb_set_error(ICB_E_CONFIG, "promotion ratio must lie in (0, 1)");
    return ICB_E_CONFIG;
  }
  if (c.tok_cap < 1 || c.node_cap < 1 || c.page_cap < 1 || c.member_cap < 1 || c.own_cap < 1) {
    icb_set_error(ICB_E_CONFIG, "capacities must be positive");
    return ICB_E_CONFIG;
  }
  icb_forest* f = new icb_forest();
  f->cfg = c;
  ForestView& F = f->view;
  F.T = c.n_trees; F.dim = c.dim; F.dim_v = c.dim_v; F.s = c.page_size; F.kv_bf16 = c.kv_dtype == ICB_KV_BF16;
  F.dkp = (c.dim + 3) & ~3; F.dvp = (c.dim_v + 3) & ~3;
  F.tok_cap = c.tok_cap; F.node_cap = c.node_cap; F.page_cap = c.page_cap; F.member_cap = c.member_cap;
  F.own_cap = c.own_cap; F.dirs_cap = std::max(1, c.dirs_cap); F.r = c.promotion_ratio;
  const size_t T = c.n_trees;
  const size_t kvb = F.kv_bf16 ? 2 : 4;
  int rc = ICB_OK;
#define AL(ptr, n, fb) if (rc == ICB_OK) rc = falloc(f, &ptr, n, fb)
  AL(F.meta, T, 0);
  AL(F.lift, T * c.tok_cap * ICB_ROWF, 0);
  AL(F.tail, T * c.tok_cap, 0);
  AL(F.level, T * c.tok_cap, 0);
  AL(F.own_base, T * c.tok_cap, 0);
  AL(F.tok2page, T * c.tok_cap, 0xff);
  AL(F.own_list, T * c.own_cap, 0);
  AL(F.own1, T * c.tok_cap, 0);
  AL(F.node_level, T * c.node_cap, 0);
  AL(F.node_parent, T * c.node_cap, 0);
  AL(F.node_owner, T * c.node_cap, 0);
  AL(F.node_off, T * c.node_cap, 0);
  AL(F.node_size, T * c.node_cap, 0);
  AL(F.node_capm, T * c.node_cap, 0);
  AL(F.node_lastpage, T * c.node_cap, 0xff);
  AL(F.node_dirs, T * c.node_cap, 0xff);
  AL(F.node_opos, T * c.node_cap, 0xff);
  AL(F.members, T * c.member_cap, 0);
  AL(F.page_fill, T * c.page_cap, 0);
  AL(F.page_role, T * c.page_cap, 0);
  AL(F.page_tok, T * c.page_cap * c.page_size, 0xff);
  AL(F.dirs, T * F.dirs_cap * ICB_NPROJ * (c.dim + 1), 0);
  AL(F.prev_sel, T * (c.page_cap / 32 + 1), 0);
  F.upper_cap = c.tok_cap / 4 + 64;   // ~r = 10% of points expected; overflow only disables the start shortcut
  AL(F.upper, T * F.upper_cap, 0);
  F.pc_cap = std::min(6144, c.tok_cap + 64);
  AL(F.node_pc, T * c.node_cap, 0xff);
  AL(F.node_pcm, T * c.node_cap, 0xff);
  AL(F.node_pccap, T * c.node_cap, 0);
  AL(F.pc_proj, T * F.pc_cap * ICB_NPROJ, 0);
  AL(F.pc_ord, T * F.pc_cap * ICB_NPROJ, 0);
  AL(F.pc_pos, T * F.pc_cap * ICB_NPROJ, 0);
#undef AL
  F.kv_host = c.kv_host != 0;
  F.pool_cap = F.kv_host ? c.pool_pages : 0;
  if (F.kv_host && c.pool_pages < 4) { icb_set_error(ICB_E_CONFIG, "kv_host needs pool_pages >= 4"); rc = ICB_E_CONFIG; }
  if (rc == ICB_OK && !F.kv_host) {
    char* pk = nullptr;
    char* pv = nullptr;
    rc = falloc(f, &pk, T * c.page_cap * c.page_size * F.dkp * kvb, 0);
    if (rc == ICB_OK) rc = falloc(f, &pv, T * c.page_cap * c.page_size * F.dvp * kvb, 0);
    F.page_k = pk;
    F.page_v = pv;
  } else if (rc == ICB_OK) {
    // the host store: pinned, mapped into the device address space
    const size_t nk = T * c.page_cap * c.page_size * F.dkp * kvb, nv = T * c.page_cap * c.page_size * F.dvp * kvb;
    for (int i = 0; i < 2 && rc == ICB_OK; ++i) {
      // no memset: freshly mapped pages are zero, and every row is written at
      // full padded width (build scatter, write_slot) before anything reads it
      void* d = nullptr;
      rc = pin_host_store(f, i ? nv : nk, &d);
      (i ? F.page_v : F.page_k) = d;
    }
    char* qk = nullptr;
    char* qv = nullptr;
    if (rc == ICB_OK) rc = falloc(f, &qk, T * F.pool_cap * c.page_size * F.dkp * kvb, 0);
    if (rc == ICB_OK) rc = falloc(f, &qv, T * F.pool_cap * c.page_size * F.dvp * kvb, 0);
    F.pool_k = qk;
    F.pool_v = qv;
    if (rc == ICB_OK) rc = falloc(f, &F.page_slot, T * c.page_cap, 0xff);
    if (rc == ICB_OK) rc = falloc(f, &F.slot_page, T * F.pool_cap, 0xff);
    if (rc == ICB_OK) rc = falloc(f, &F.pool_tmp, T * 2 * F.pool_cap, 0);
    if (rc == ICB_OK) rc = falloc(f, &F.pool_bytes, T, 0);
  }
  if (rc != ICB_OK) {
    icb_forest_destroy(f);
    return rc;
  }
  *out = f;
  return ICB_OK;
}

int icb_forest_destroy(icb_forest* f) {
  if (!f) return ICB_OK;
  cudaDeviceSynchronize();
  for (void* p : f->allocs) cudaFree(p);
  for (void* p : f->host_allocs) cudaFreeHost(p);
  for (auto& r : f->host_regs) {
    const size_t chunk = 1ull << 30;
    for (size_t off = 0; off < r.second; off += chunk) cudaHostUnregister((char*)r.first + off);
    munmap(r.first, r.second);
  }
  if (f->qscratch) cudaFree(f->qscratch);
  if (f->iscratch) cudaFree(f->iscratch);
  if (f->ascratch) cudaFree(f->ascratch);
  delete f;
  return ICB_OK;
}

int icb_seed_trees(icb_forest* f, const int32_t* trees, int32_t n, const uint32_t* words, int32_t stride,
                   const int32_t* n_words) {
  for (int i = 0; i < n; ++i) {
    int t = trees[i];
    if (t < 0 || t >= f->cfg.n_trees) { icb_set_error(ICB_E_INPUT, "tree index out of range"); return ICB_E_INPUT; }
    int nw = n_words[i];
    if (nw < 1 || nw > 8) { icb_set_error(ICB_E_INPUT, "1..8 entropy words supported"); return ICB_E_INPUT; }
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < nw; ++j) w[j] = words[(size_t)i * stride + j];
    uint32_t spawn0 = 0;
    uint64_t st[4];
    icb_seedseq_u64x4(w, nw, &spawn0, 1, st);
    Pcg64 g = icb_pcg_seed(st);
    seed_kernel<<<1, 1>>>(f->view, t, g, nw, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]);
  }
  ICB_CUDA(cudaGetLastError());
  ICB_CUDA(cudaDeviceSynchronize());
  return ICB_OK;
}

int icb_alloc_resident_pages(icb_forest* f, const int32_t* trees, int32_t n, int32_t role, int32_t count,
                             int32_t n_tokens, const int32_t* tokens, const float* keys, const float* values,
                             void* stream) {
  if (role != ICB_ROLE_SINK && role != ICB_ROLE_WINDOW) {
    icb_set_error(ICB_E_INPUT, "resident pages are sink or window pages");
    return ICB_E_INPUT;
  }
  if (n_tokens > count * f->cfg.page_size) {
    icb_set_error(ICB_E_INPUT, "more tokens than resident page slots");
    return ICB_E_INPUT;
  }
  return icb_resident_impl(f, trees, n, role, count, n_tokens, tokens, keys, values, S_(stream));
}

int icb_build(icb_forest* f, const int32_t* trees, int32_t n, int32_t n_points, const int32_t* tokens,
              const float* keys, const float* values, const double* scales, void* stream) {
  if (n_points < 1) { icb_set_error(ICB_E_INPUT, "cannot index an empty key set"); return ICB_E_INPUT; }
  if ((long long)n_points >= (1ll << 23)) { icb_set_error(ICB_E_CONFIG, "at most 2^23 points per build"); return ICB_E_CONFIG; }
  if (n >= 4096) { icb_set_error(ICB_E_CONFIG, "at most 4095 trees per build call"); return ICB_E_CONFIG; }
  return icb_build_impl(f, trees, n, n_points, tokens, keys, values, scales, S_(stream));
}

int icb_query(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries, int32_t lifted_input,
              int32_t k, int64_t beam, int64_t visit_cap, int32_t target_level, int32_t* out_ids, int32_t k_out,
              int32_t* out_counts, int32_t* out_pages, int32_t pages_cap, int32_t* out_npages, void* stream) {
  if (k < 1) { icb_set_error(ICB_E_INPUT, "k must be >= 1"); return ICB_E_INPUT; }
  if (beam < k || visit_cap < k) { icb_set_error(ICB_E_CONFIG, "beam and visit_cap must be >= k"); return ICB_E_CONFIG; }
  if (target_level != ICB_SENTINEL_LEVEL && target_level < 1) {
    icb_set_error(ICB_E_INPUT, "target level must be -1 or >= 1");
    return ICB_E_INPUT;
  }
  return icb_query_impl(f, trees, n, G, queries, lifted_input, k, beam, visit_cap, target_level, out_ids, k_out,
                        out_counts, out_pages, pages_cap, out_npages, S_(stream));
}

static int check_pool(icb_forest* f, int32_t pages_cap) {
  // KV offload: the pool must hold a step's sink + window + largest selection
  if (f && f->view.kv_host && f->view.pool_cap < pages_cap + 2) {
    icb_set_error(ICB_E_CONFIG, "pool_pages must cover sink + window + pages_cap (the largest selection)");
    return ICB_E_CONFIG;
  }
  return ICB_OK;
}

int icb_query_attend(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries, int32_t k,
                     int64_t beam, int64_t visit_cap, int32_t* out_ids, int32_t k_out, int32_t* out_counts,
                     int32_t* out_pages, int32_t pages_cap, int32_t* out_npages, float* attn_out,
                     int64_t* attn_stats, int32_t scalar_bytes, void* stream) {
  if (k < 1) { icb_set_error(ICB_E_INPUT, "k must be >= 1"); return ICB_E_INPUT; }
  if (beam < k || visit_cap < k) { icb_set_error(ICB_E_CONFIG, "beam and visit_cap must be >= k"); return ICB_E_CONFIG; }
  if (!attn_out || !out_pages || !out_npages) { icb_set_error(ICB_E_INPUT, "null output"); return ICB_E_INPUT; }
  if (int rc = check_pool(f, pages_cap)) return rc;
  return icb_query_impl(f, trees, n, G, queries, 0, k, beam, visit_cap, ICB_SENTINEL_LEVEL, out_ids, k_out,
                        out_counts, out_pages, pages_cap, out_npages, S_(stream), attn_out, attn_stats,
                        scalar_bytes);
}

int icb_step_attend(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries, int32_t k,
                    int64_t beam, int64_t visit_cap, int32_t* out_ids, int32_t k_out, int32_t* out_counts,
                    int32_t* out_pages, int32_t pages_cap, int32_t* out_npages, float* attn_out,
                    int64_t* attn_stats, int32_t scalar_bytes, int32_t rotate, int64_t* rot_stats,
                    const int32_t* token_dev, const float* win_keys, const float* win_values, void* stream) {
  if (k < 1) { icb_set_error(ICB_E_INPUT, "k must be >= 1"); return ICB_E_INPUT; }
  if (beam < k || visit_cap < k) { icb_set_error(ICB_E_CONFIG, "beam and visit_cap must be >= k"); return ICB_E_CONFIG; }
  if (!attn_out || !out_pages || !out_npages) { icb_set_error(ICB_E_INPUT, "null output"); return ICB_E_INPUT; }
  if (int rc = check_pool(f, pages_cap)) return rc;
  StepOpts step{rotate, rot_stats, token_dev, win_keys, win_values};
  return icb_query_impl(f, trees, n, G, queries, 0, k, beam, visit_cap, ICB_SENTINEL_LEVEL, out_ids, k_out,
                        out_counts, out_pages, pages_cap, out_npages, S_(stream), attn_out, attn_stats,
                        scalar_bytes, &step);
}

int icb_insert(icb_forest* f, const int32_t* trees, int32_t n, int32_t m, const int32_t* tokens, const float* keys,
               const float* values, const int32_t* levels, int32_t* out_levels, void* stream) {
  return icb_insert_impl(f, trees, n, m, tokens, keys, values, levels, out_levels, 0, 4, nullptr, S_(stream));
}

int icb_rotate_window(icb_forest* f, const int32_t* trees, int32_t n, int32_t scalar_bytes, int64_t* stats,
                      void* stream) {
  return icb_insert_impl(f, trees, n, 0, nullptr, nullptr, nullptr, nullptr, nullptr, 1, scalar_bytes, stats,
                         S_(stream));
}

int icb_append_window(icb_forest* f, const int32_t* trees, int32_t n, int32_t token, const float* keys,
                      const float* values, void* stream) {
  return icb_append_impl(f, trees, n, token, nullptr, keys, values, S_(stream));
}

int icb_append_window_dev(icb_forest* f, const int32_t* trees, int32_t n, const int32_t* token_dev, const float* keys,
                          const float* values, void* stream) {
  if (!token_dev) { icb_set_error(ICB_E_INPUT, "null device token"); return ICB_E_INPUT; }
  return icb_append_impl(f, trees, n, 0, token_dev, keys, values, S_(stream));
}

int icb_sparse_attention(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries,
                         const int32_t* pages, int32_t pages_cap, const int32_t* npages, float* out, int64_t* stats,
                         int32_t scalar_bytes, int32_t splits, void* stream) {
  int min_splits = (pages_cap + ICB_MAX_SINK + ICB_MAX_WINDOW + 1023) / 1024;
  if (splits > 0 && splits < min_splits) splits = min_splits;
  if (splits <= 0) splits = -min_splits;   // auto, at least min_splits
  if (splits < 0) {
    int auto_s = std::max(1, std::min(8, (2 * 148) / std::max(n, 1)));   // one wave at 2 CTAs / SM
    splits = std::max(auto_s, -splits);
  }
  return icb_attention_impl(f, trees, n, G, queries, pages, pages_cap, npages, out, stats, scalar_bytes, splits,
                            S_(stream));
}

int icb_dense_attention(int32_t n, int32_t G, int32_t dim, int32_t dim_v, int32_t kv_dtype, const float* q,
                        const void* k, const void* v, int64_t ld, int32_t n_tokens, float* out, int32_t splits,
                        void* stream) {
  if (dim < 1 || dim > 128 || dim_v < 1 || dim_v > 128) { icb_set_error(ICB_E_CONFIG, "dense attention supports 1 <= d, d' <= 128"); return ICB_E_CONFIG; }
  if (n_tokens < 1) { icb_set_error(ICB_E_INPUT, "empty key set"); return ICB_E_INPUT; }
  return icb_dense_attention_impl(n, G, dim, dim_v, kv_dtype, q, k, v, ld, n_tokens, nullptr, out, splits,
                                  S_(stream));
}

int icb_dense_attention_dev(int32_t n, int32_t G, int32_t dim, int32_t dim_v, int32_t kv_dtype, const float* q,
                            const void* k, const void* v, int64_t ld, const int32_t* token_dev, float* out,
                            int32_t splits, void* stream) {
  if (dim < 1 || dim > 128 || dim_v < 1 || dim_v > 128) { icb_set_error(ICB_E_CONFIG, "dense attention supports 1 <= d, d' <= 128"); return ICB_E_CONFIG; }
  if (!token_dev || ld < 1) { icb_set_error(ICB_E_INPUT, "null device token / empty capacity"); return ICB_E_INPUT; }
  // splits sized for the full capacity; each CTA clips its rows to *token_dev + 1
  return icb_dense_attention_impl(n, G, dim, dim_v, kv_dtype, q, k, v, ld, (int32_t)ld, token_dev, out, splits,
                                  S_(stream));
}

int icb_attended_mask(icb_forest* f, const int32_t* trees, int32_t n, const int32_t* pages, int32_t pages_cap,
                      const int32_t* npages, uint8_t* mask, void* stream) {
  if (!f || (n > 0 && (!trees || !pages || !npages || !mask))) { icb_set_error(ICB_E_INPUT, "null argument"); return ICB_E_INPUT; }
  return icb_attended_mask_impl(f, trees, n, pages, pages_cap, npages, mask, S_(stream));
}

int icb_node_query(icb_forest* f, int32_t tree, int32_t node, const float* q_lifted, int32_t k, int64_t visit_cap,
                   int32_t* out_ids, int32_t* out_count, void* stream) {
  if (!f || tree < 0 || tree >= f->cfg.n_trees || !q_lifted || !out_ids || !out_count) {
    icb_set_error(ICB_E_INPUT, "bad argument");
    return ICB_E_INPUT;
  }
  if (k < 1 || visit_cap < k) { icb_set_error(ICB_E_CONFIG, "need 1 <= k <= visit_cap"); return ICB_E_CONFIG; }
  return icb_node_query_impl(f, tree, node, q_lifted, k, visit_cap, out_ids, out_count, S_(stream));
}

int icb_pages_from_tokens(icb_forest* f, const int32_t* trees, int32_t n, const int32_t* src_rows,
                          const int32_t* src_ids, const int32_t* src_counts, int32_t G, int32_t k_stride,
                          int32_t* out_pages, int32_t pages_cap, int32_t* out_npages, void* stream) {
  if (!f || (n > 0 && (!trees || !src_rows || !src_ids || !src_counts || !out_pages || !out_npages))) {
    icb_set_error(ICB_E_INPUT, "null argument");
    return ICB_E_INPUT;
  }
  if (G < 1 || G > ICB_MAX_G || k_stride < 1 || pages_cap < 1) {
    icb_set_error(ICB_E_CONFIG, "bad G / k_stride / pages_cap");
    return ICB_E_CONFIG;
  }
  return icb_pages_from_tokens_impl(f, trees, n, src_rows, src_ids, src_counts, G, k_stride, out_pages, pages_cap,
                                    out_npages, S_(stream));
}

int icb_dense_append(int32_t n, int32_t dim, int32_t dim_v, int32_t kv_dtype, const float* k, const float* v,
                     void* dense_k, void* dense_v, int64_t ld, const int32_t* token_dev, void* stream) {
  if (!token_dev || !dense_k || !dense_v) { icb_set_error(ICB_E_INPUT, "null argument"); return ICB_E_INPUT; }
  return icb_dense_append_impl(n, dim, dim_v, kv_dtype, k, v, dense_k, dense_v, ld, token_dev, S_(stream));
}

int icb_tree_info(icb_forest* f, int32_t tree, int64_t* out) {
  if (tree < 0 || tree >= f->cfg.n_trees) { icb_set_error(ICB_E_INPUT, "tree index out of range"); return ICB_E_INPUT; }
  TreeMeta m;
  ICB_CUDA(cudaDeviceSynchronize());
  ICB_CUDA(cudaMemcpy(&m, f->view.meta + tree, sizeof(TreeMeta), cudaMemcpyDeviceToHost));
  int64_t v[16] = {m.levels, m.top_node, m.n_nodes, m.next_page, m.n_points, m.err, m.n_window, m.n_sink,
                   (int64_t)m.query_count, (int64_t)m.distance_evals, (int64_t)m.scale_clamps, m.member_top,
                   m.own_top, m.n_dirs, (int64_t)m.rows_read, (int64_t)m.owner_rereads};
  std::memcpy(out, v, sizeof(v));
  return ICB_OK;
}

int icb_errors(icb_forest* f, int32_t* out, int32_t clear) {
  const int T = f->cfg.n_trees;
  std::vector<TreeMeta> m(T);
  ICB_CUDA(cudaDeviceSynchronize());
  ICB_CUDA(cudaMemcpy(m.data(), f->view.meta, sizeof(TreeMeta) * T, cudaMemcpyDeviceToHost));
  for (int t = 0; t < T; ++t) {
    out[t] = m[t].err;
    if (clear && m[t].err) {
      int zero = 0;
      ICB_CUDA(cudaMemcpy((char*)(f->view.meta + t) + offsetof(TreeMeta, err), &zero, sizeof(int),
                          cudaMemcpyHostToDevice));
    }
  }
  return ICB_OK;
}

int icb_clear_errors(icb_forest* f, int32_t tree) {
  int zero = 0;
  ICB_CUDA(cudaMemcpy((char*)(f->view.meta + tree) + offsetof(TreeMeta, err), &zero, sizeof(int),
                      cudaMemcpyHostToDevice));
  return ICB_OK;
}

int icb_read_meta_c(icb_forest* f, int32_t tree, double* c) {
  ICB_CUDA(cudaMemcpy(c, (char*)(f->view.meta + tree) + offsetof(TreeMeta, c), sizeof(double),
                      cudaMemcpyDeviceToHost));
  return ICB_OK;
}

int icb_set_scale(icb_forest* f, int32_t tree, double c) {
  if (!f || tree < 0 || tree >= f->cfg.n_trees) { icb_set_error(ICB_E_INPUT, "bad tree"); return ICB_E_INPUT; }
  if (!(c > 0.0)) { icb_set_error(ICB_E_CONFIG, "scale must be positive"); return ICB_E_CONFIG; }
  ICB_CUDA(cudaMemcpy((char*)(f->view.meta + tree) + offsetof(TreeMeta, c), &c, sizeof(double),
                      cudaMemcpyHostToDevice));
  return ICB_OK;
}

int icb_export_tree(icb_forest* f, int32_t tree, int32_t* node_level, int32_t* node_parent, int32_t* node_owner,
                    int32_t* node_off, int32_t* node_size, int32_t* node_lastpage, int32_t* members,
                    int32_t* page_fill, int8_t* page_role, int32_t* page_tok, int32_t* tok2page, int8_t* level,
                    int32_t* own_base, int32_t* own_list, float* lift, float* tail, int32_t* win, int32_t* sink) {
  if (tree < 0 || tree >= f->cfg.n_trees) { icb_set_error(ICB_E_INPUT, "tree index out of range"); return ICB_E_INPUT; }
  const ForestView& F = f->view;
  const auto& c = f->cfg;
  ICB_CUDA(cudaDeviceSynchronize());
  size_t t = tree;
#define CP(dst, src, n) \
  if (dst) ICB_CUDA(cudaMemcpy(dst, src, sizeof(*dst) * (size_t)(n), cudaMemcpyDeviceToHost))
  CP(node_level, F.node_level + t * c.node_cap, c.node_cap);
  CP(node_parent, F.node_parent + t * c.node_cap, c.node_cap);
  CP(node_owner, F.node_owner + t * c.node_cap, c.node_cap);
  CP(node_off, F.node_off + t * c.node_cap, c.node_cap);
  CP(node_size, F.node_size + t * c.node_cap, c.node_cap);
  CP(node_lastpage, F.node_lastpage + t * c.node_cap, c.node_cap);
  CP(members, F.members + t * c.member_cap, c.member_cap);
  CP(page_fill, F.page_fill + t * c.page_cap, c.page_cap);
  CP(page_role, F.page_role + t * c.page_cap, c.page_cap);
  CP(page_tok, F.page_tok + t * c.page_cap * c.page_size, (size_t)c.page_cap * c.page_size);
  CP(tok2page, F.tok2page + t * c.tok_cap, c.tok_cap);
  CP(level, F.level + t * c.tok_cap, c.tok_cap);
  CP(own_base, F.own_base + t * c.tok_cap, c.tok_cap);
  CP(own_list, F.own_list + t * c.own_cap, c.own_cap);
  CP(lift, F.lift + t * c.tok_cap * ICB_ROWF, (size_t)c.tok_cap * ICB_ROWF);
  CP(tail, F.tail + t * c.tok_cap, c.tok_cap);
#undef CP
  TreeMeta m;
  ICB_CUDA(cudaMemcpy(&m, F.meta + t, sizeof(TreeMeta), cudaMemcpyDeviceToHost));
  if (win) for (int i = 0; i < ICB_MAX_WINDOW; ++i) win[i] = i < m.n_window ? m.win[i] : -1;
  if (sink) for (int i = 0; i < ICB_MAX_SINK; ++i) sink[i] = i < m.n_sink ? m.sink[i] : -1;
  return ICB_OK;
}

int icb_read_pages(icb_forest* f, int32_t tree, const int32_t* pages, int32_t count, float* keys, float* values) {
  const ForestView& F = f->view;
  const auto& c = f->cfg;
  ICB_CUDA(cudaDeviceSynchronize());
  const size_t kvb = F.kv_bf16 ? 2 : 4;
  std::vector<char> kbuf((size_t)c.page_size * F.dkp * kvb), vbuf((size_t)c.page_size * F.dvp * kvb);
  for (int i = 0; i < count; ++i) {
    size_t slot0 = ((size_t)tree * c.page_cap + pages[i]) * c.page_size;
    ICB_CUDA(cudaMemcpy(kbuf.data(), (char*)F.page_k + slot0 * F.dkp * kvb, kbuf.size(), cudaMemcpyDeviceToHost));
    ICB_CUDA(cudaMemcpy(vbuf.data(), (char*)F.page_v + slot0 * F.dvp * kvb, vbuf.size(), cudaMemcpyDeviceToHost));
    for (int r = 0; r < c.page_size; ++r) {
      for (int j = 0; j < c.dim; ++j) {
        float x;
        if (F.kv_bf16) { uint16_t h; std::memcpy(&h, kbuf.data() + ((size_t)r * F.dkp + j) * 2, 2); uint32_t u = (uint32_t)h << 16; std::memcpy(&x, &u, 4); }
        else std::memcpy(&x, kbuf.data() + ((size_t)r * F.dkp + j) * 4, 4);
        keys[((size_t)i * c.page_size + r) * c.dim + j] = x;
      }
      for (int j = 0; j < c.dim_v; ++j) {
        float x;
        if (F.kv_bf16) { uint16_t h; std::memcpy(&h, vbuf.data() + ((size_t)r * F.dvp + j) * 2, 2); uint32_t u = (uint32_t)h << 16; std::memcpy(&x, &u, 4); }
        else std::memcpy(&x, vbuf.data() + ((size_t)r * F.dvp + j) * 4, 4);
        values[((size_t)i * c.page_size + r) * c.dim_v + j] = x;
      }
    }
  }
  return ICB_OK;
}

// Host restatement self-check: PCG64/SeedSequence draws (for CPU tests).
int icb_host_pcg_doubles(const uint32_t* words, int32_t n_words, const uint32_t* spawn, int32_t n_spawn, int32_t n,
                         double* out) {
  uint64_t st[4];
  icb_seedseq_u64x4(words, n_words, spawn, n_spawn, st);
  Pcg64 g = icb_pcg_seed(st);
  for (int i = 0; i < n; ++i) out[i] = icb_pcg_double(g);
  return ICB_OK;
}

int icb_pool_stats(icb_forest* f, int64_t* out) {
  if (!f->view.kv_host) { icb_set_error(ICB_E_CONFIG, "the forest keeps its KV in HBM (kv_host = 0)"); return ICB_E_CONFIG; }
  const int T = f->cfg.n_trees;
  std::vector<int> slot_page((size_t)T * f->view.pool_cap);
  std::vector<long long> bytes(T);
  ICB_CUDA(cudaMemcpy(bytes.data(), f->view.pool_bytes, sizeof(long long) * T, cudaMemcpyDeviceToHost));
  ICB_CUDA(cudaMemcpy(slot_page.data(), f->view.slot_page, sizeof(int) * slot_page.size(), cudaMemcpyDeviceToHost));
  for (int t = 0; t < T; ++t) {
    long long res = 0;
    for (int s = 0; s < f->view.pool_cap; ++s) res += slot_page[(size_t)t * f->view.pool_cap + s] >= 0;
    out[2 * t] = bytes[t];
    out[2 * t + 1] = res;
  }
  return ICB_OK;
}

int icb_host_pcg_jump_doubles(const uint32_t* words, int32_t n_words, const uint32_t* spawn, int32_t n_spawn,
                              int64_t skip, int32_t n, double* out) {
  uint64_t st[4];
  icb_seedseq_u64x4(words, n_words, spawn, n_spawn, st);
  Pcg64 g = icb_pcg_seed(st);
  icb_u128 A, C;
  icb_pcg_jump((unsigned long long)skip, g.inc, A, C);
  g.state = A * g.state + C;
  for (int i = 0; i < n; ++i) out[i] = icb_pcg_double(g);
  return ICB_OK;
}

}  // extern "C"
