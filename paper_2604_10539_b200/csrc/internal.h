// Host-side internals shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include <utility>
#include <algorithm>
#include "icb.cuh"

void icb_set_error(int code, const std::string& msg);

#define ICB_CUDA(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      icb_set_error(ICB_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));    \
      return ICB_E_CUDA;                                                                \
    }                                                                                   \
  } while (0)

struct BuildArgs {
  const int32_t* trees;
  int n, n_points;
  const int32_t* tokens;
  const float* keys;
  const float* values;
  const double* scales;
  int* pos_of;   // [n][tok_cap] token -> input position
};

struct icb_forest {
  icb_forest_config cfg;
  ForestView view;
  std::vector<void*> allocs;
  std::vector<void*> host_allocs;   // pinned, mapped host store (kv_host)
  std::vector<std::pair<void*, size_t>> host_regs;   // the same, mmap'ed + registered in chunks
  // persistent scratch for queries / inserts (grown on demand)
  void* qscratch = nullptr;
  size_t qscratch_bytes = 0;
  int qscratch_G = 0;
  void* iscratch = nullptr;   // insert-path scratch (separate: mark arrays must stay zero)
  size_t iscratch_bytes = 0;
  void* ascratch = nullptr;   // attention split-K partials
  size_t ascratch_bytes = 0;
};

// Stream-ordered scratch allocations released at the end of a call.
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  bool good = true;
  std::string why;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMallocAsync(&p, n * sizeof(T), st);
    if (e != cudaSuccess) {
      good = false;
      why = cudaGetErrorString(e);
      return nullptr;
    }
    ptrs.push_back(p);
    return (T*)p;
  }
  bool ok() const { return good; }
  int fail() {
    icb_set_error(ICB_E_CUDA, "scratch allocation failed: " + why);
    release();
    return ICB_E_CUDA;
  }
  void release() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    ptrs.clear();
  }
  int finish() {
    release();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      icb_set_error(ICB_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
      return ICB_E_CUDA;
    }
    return ICB_OK;
  }
  ~Scratch() { release(); }
};

void zero_node_sizes(icb_forest* f, const int32_t* trees, int n, cudaStream_t st);
int icb_append_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t token, const int32_t* token_dev,
                    const float* keys, const float* values, cudaStream_t st);
int icb_resident_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t role, int32_t count,
                      int32_t n_tokens, const int32_t* tokens, const float* keys, const float* values,
                      cudaStream_t st);

int icb_build_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t n_points, const int32_t* tokens,
                   const float* keys, const float* values, const double* scales, cudaStream_t st);
// Fused decode-step prologue of the query kernel (icb_step_attend).
struct StepOpts {
  int rotate;                  // rotate the oldest window page into the tree first
  int64_t* rot_stats;          // [n][2] or null
  const int32_t* token_dev;    // the decode position (device memory)
  const float* keys;           // [n][dim] window keys of this token
  const float* values;         // [n][dim_v]
};
int icb_query_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries,
                   int32_t lifted_input, int32_t k, int64_t beam, int64_t visit_cap, int32_t target_level,
                   int32_t* out_ids, int32_t k_out, int32_t* out_counts, int32_t* out_pages,
                   int32_t pages_cap, int32_t* out_npages, cudaStream_t st, float* attn_out = nullptr,
                   int64_t* attn_stats = nullptr, int32_t scalar_bytes = 4, const StepOpts* step = nullptr);
int icb_insert_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t m, const int32_t* tokens,
                    const float* keys, const float* values, const int32_t* levels, int32_t* out_levels,
                    int from_window, int32_t scalar_bytes, int64_t* stats, cudaStream_t st);
int icb_attention_impl(icb_forest* f, const int32_t* trees, int32_t n, int32_t G, const float* queries,
                       const int32_t* pages, int32_t pages_cap, const int32_t* npages, float* out,
                       int64_t* stats, int32_t scalar_bytes, int32_t splits, cudaStream_t st);
int icb_attended_mask_impl(icb_forest* f, const int32_t* trees, int32_t n, const int32_t* pages, int32_t pages_cap,
                           const int32_t* npages, uint8_t* mask, cudaStream_t st);
int icb_node_query_impl(icb_forest* f, int32_t tree, int32_t node, const float* q_lifted, int32_t k,
                        int64_t visit_cap, int32_t* out_ids, int32_t* out_count, cudaStream_t st);
int icb_pages_from_tokens_impl(icb_forest* f, const int32_t* trees, int32_t n, const int32_t* src_rows,
                               const int32_t* src_ids, const int32_t* src_counts, int32_t G, int32_t k_stride,
                               int32_t* out_pages, int32_t pages_cap, int32_t* out_npages, cudaStream_t st);
int icb_dense_append_impl(int32_t n, int32_t dim, int32_t dim_v, int32_t kv_dtype, const float* k, const float* v,
                          void* dense_k, void* dense_v, int64_t ld, const int32_t* token_dev, cudaStream_t st);
int icb_dense_attention_impl(int32_t n, int32_t G, int32_t dim, int32_t dim_v, int32_t kv_dtype,
                             const float* q, const void* k, const void* v, int64_t ld, int32_t n_tokens,
                             const int32_t* token_dev, float* out, int32_t splits, cudaStream_t st);
bool icb_dense_flash_ok(int G, int dim, int dim_v, int kv_dtype);
int icb_dense_flash_impl(int32_t n, int32_t G, const float* q, const void* k, const void* v, int64_t ld,
                         int32_t n_tokens, const int32_t* token_dev, float* out, int32_t splits, float* part,
                         unsigned* counter, cudaStream_t st);
int icb_pdci_warm_impl(icb_forest* f, const int32_t* trees, int32_t n, int64_t qcap, cudaStream_t st);
