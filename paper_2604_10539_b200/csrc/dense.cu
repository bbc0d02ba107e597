// Dense decode attention for the skip layers (full_attention, attention.py:
// 55-74; engine.py:418-422) on bf16 K/V planes with d = d' = 128: a
// flash-decoding kernel fed by TMA.
//
// Memory-bound (2 * 256 B per token per plane, 268 MB per C2 step, 1.07 GB
// at 128k).  The previous CUDA-core kernel (attention.cu, still used for
// fp32 / other shapes) spent ~90 warp-instructions per row and held too few
// bytes in flight; here:
//   - a producer warp streams 64-row K and V tiles with 2-D TMA
//     (cp.async.bulk.tensor, 128-byte swizzle: two 64-column boxes per tile)
//     into an NS-stage shared-memory ring, completion counted on mbarriers;
//   - four consumer warps take 16 rows of each tile: S = Q K^T and O += P V
//     on the tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate; the G <= 8
//     query heads of the GQA group are the M rows, padded to 16), K and V
//     fragments read with ldmatrix (V transposed) from the swizzled tiles;
//     q is split q = q_hi + q_lo (two bf16 MMAs) so the logits keep ~16
//     mantissa bits; online softmax in fp32 (exp2, per-head running max);
//   - split-K over the rows; the CTA's warps merge in shared memory and the
//     last CTA of a plane merges the splits (same partial layout as
//     attention.cu).
#include <cuda.h>
#include <cudaTypedefs.h>
#include "internal.h"

namespace icb {

constexpr int kDenseTile = 64;          // rows per TMA tile (16 per consumer warp)
constexpr int kDenseStages = 3;
constexpr int kDenseThreads = 160;      // 4 consumer warps + 1 producer warp
constexpr int kDenseTileBytes = kDenseTile * 128 * 2;   // one of K / V: 16 KB (two 8 KB boxes)

struct DenseArgs {
  int n, G, splits;
  long long ld;              // rows per plane
  int n_tokens;
  const int32_t* token_dev;  // rows [0, *token_dev + 1) when set
  const float* q;            // [n][G][128]
  float* out;                // [n][G][128]
  float* part;               // [n][splits][G][2 + 128]
  unsigned* counter;         // [n]
  float scale_log2;
};

__device__ __forceinline__ unsigned pack_bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<unsigned*>(&v);
}

__device__ __forceinline__ void mma_bf16(float (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                         unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Byte offset of (row, 16-byte chunk c in 0..15) inside a [64 rows][128 bf16]
// tile stored as two 128B-swizzled boxes of 64 columns: chunk j of row r in a
// box sits at (j ^ (r & 7)) * 16.
__device__ __forceinline__ unsigned tile_off(int row, int c) {
  return (unsigned)((c >> 3) * (kDenseTile * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}

template <int NS>
__global__ void __launch_bounds__(kDenseThreads, 1)
    dense_flash_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       DenseArgs A) {
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  unsigned char* dsm = (unsigned char*)(((size_t)dsm_raw + 1023) & ~(size_t)1023);
  unsigned char* ktile = dsm;                                  // [NS][16 KB]
  unsigned char* vtile = dsm + NS * kDenseTileBytes;           // [NS][16 KB]
  __shared__ __align__(8) unsigned long long full_bar[NS], empty_bar[NS];
  __shared__ float s_m[4][8], s_l[4][8];
  __shared__ bool s_last;
  // the warps' final accumulators reuse the (drained) tile ring
  float (*s_o)[8][128] = reinterpret_cast<float (*)[8][128]>(dsm);
  const int b = blockIdx.x, sp = blockIdx.y, S = A.splits;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = A.G;
  const int ntok = A.token_dev ? *A.token_dev + 1 : A.n_tokens;
  const int r0 = (int)((long long)ntok * sp / S), r1 = (int)((long long)ntok * (sp + 1) / S);
  const int ntiles = (r1 - r0 + kDenseTile - 1) / kDenseTile;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 4); }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == 4) {
    // ---- producer: one lane streams the tiles
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
      const long long rbase = (long long)b * A.ld;
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % NS;
        if (i >= NS) mbar_wait(&empty_bar[s], ((i / NS) - 1) & 1);
        mbar_expect_tx(&full_bar[s], 2 * kDenseTileBytes);
        const int row = (int)(rbase + r0 + i * kDenseTile);
        unsigned char* kd = ktile + s * kDenseTileBytes;
        unsigned char* vd = vtile + s * kDenseTileBytes;
        tma_load_2d(kd, &tmK, 0, row, &full_bar[s]);
        tma_load_2d(kd + kDenseTile * 128, &tmK, 64, row, &full_bar[s]);
        tma_load_2d(vd, &tmV, 0, row, &full_bar[s]);
        tma_load_2d(vd + kDenseTile * 128, &tmV, 64, row, &full_bar[s]);
      }
    }
  } else {
    // ---- consumers: warp w owns rows 16w .. 16w + 15 of every tile
    const int g = lane >> 2, t4 = lane & 3;
    const bool head = g < G;
    // Q A-fragments (M = heads, K = dims), hi and lo bf16 halves, per 16-dim step
    unsigned qa[8][2], ql[8][2];
    {
      const float* q = A.q + ((size_t)b * G + (head ? g : 0)) * 128;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 16 * kk + 8 * h + 2 * t4;
          const float x0 = head ? q[c] : 0.f, x1 = head ? q[c + 1] : 0.f;
          const __nv_bfloat162 hi = __floats2bfloat162_rn(x0, x1);
          const float2 hf = __bfloat1622float2(hi);
          qa[kk][h] = *reinterpret_cast<const unsigned*>(&hi);
          ql[kk][h] = pack_bf2(x0 - hf.x, x1 - hf.y);
        }
      }
    }
    float o[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m = -INFINITY, l = 0.f;
    const int wrow = 16 * warp;
    const int mi = lane >> 3, rr = lane & 7;   // ldmatrix: this lane's matrix and row
    for (int i = 0; i < ntiles; ++i) {
      const int s = i % NS;
      mbar_wait(&full_bar[s], (i / NS) & 1);
      const unsigned kb = smem_u32(ktile + s * kDenseTileBytes);
      const unsigned vb = smem_u32(vtile + s * kDenseTileBytes);
      // S = Q K^T for this warp's 16 rows: two n-tiles of 8 rows
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      const int krow = wrow + ((mi >> 1) << 3) + rr;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        unsigned b00, b01, b10, b11;
        ldsm_x4(kb + tile_off(krow, 2 * kk + (mi & 1)), b00, b01, b10, b11);
        mma_bf16(sc[0], qa[kk][0], 0u, qa[kk][1], 0u, b00, b01);
        mma_bf16(sc[1], qa[kk][0], 0u, qa[kk][1], 0u, b10, b11);
        mma_bf16(sc[0], ql[kk][0], 0u, ql[kk][1], 0u, b00, b01);
        mma_bf16(sc[1], ql[kk][0], 0u, ql[kk][1], 0u, b10, b11);
      }
      // online softmax over the 16 rows (rows past this split's end masked)
      const int rb = r0 + i * kDenseTile + wrow;
      float x[4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = rb + nt * 8 + 2 * t4 + e;
          x[nt * 2 + e] = row < r1 ? sc[nt][e] * A.scale_log2 : -INFINITY;
        }
      float mx = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mn = fmaxf(m, mx);
      const float alpha = mn == -INFINITY ? 1.f : exp2f(m - mn);
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) p[e] = mn == -INFINITY ? 0.f : exp2f(x[e] - mn);
      l = l * alpha + (p[0] + p[1]) + (p[2] + p[3]);
      m = mn;
#pragma unroll
      for (int j = 0; j < 16; ++j) { o[j][0] *= alpha; o[j][1] *= alpha; }
      // O += P V: A = P (heads x 16 rows), B = V tile (16 rows x 8 dims) per n-tile
      const unsigned pa0 = pack_bf2(p[0], p[1]), pa2 = pack_bf2(p[2], p[3]);
      const int vrow = wrow + ((mi & 1) << 3) + rr;
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        unsigned v0, v1, v2, v3;
        ldsm_x4_t(vb + tile_off(vrow, j + (mi >> 1)), v0, v1, v2, v3);
        mma_bf16(o[j], pa0, 0u, pa2, 0u, v0, v1);
        mma_bf16(o[j + 1], pa0, 0u, pa2, 0u, v2, v3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
    // per-head l over the 4 lanes of the head, then the warp's state to smem
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    asm volatile("bar.sync 1, 128;" ::: "memory");   // every consumer is done with the ring
    if (head) {
      if (t4 == 0) { s_m[warp][g] = m; s_l[warp][g] = l; }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        s_o[warp][g][8 * j + 2 * t4] = o[j][0];
        s_o[warp][g][8 * j + 2 * t4 + 1] = o[j][1];
      }
    }
  }
  __syncthreads();
  // merge the 4 warps into this split's partial (m, l, acc) per head
  float* part = A.part + ((size_t)b * S + sp) * G * (2 + 128);
  for (int x = threadIdx.x; x < G * 128; x += kDenseThreads) {
    const int hh = x >> 7, c = x & 127;
    float mx = -INFINITY;
    for (int w = 0; w < 4; ++w) mx = fmaxf(mx, s_m[w][hh]);
    float ls = 0.f, acc = 0.f;
    for (int w = 0; w < 4; ++w) {
      const float sc = s_m[w][hh] == -INFINITY ? 0.f : exp2f(s_m[w][hh] - mx);
      ls += s_l[w][hh] * sc;
      acc += s_o[w][hh][c] * sc;
    }
    float* pg = part + (size_t)hh * (2 + 128);
    if (c == 0) { pg[0] = mx; pg[1] = ls; }
    pg[2 + c] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(A.counter + b, 1u) == (unsigned)(S - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* pb = A.part + (size_t)b * S * G * (2 + 128);
  for (int x = threadIdx.x; x < G * 128; x += kDenseThreads) {
    const int hh = x >> 7, c = x & 127;
    float mx = -INFINITY;
    for (int s2 = 0; s2 < S; ++s2) mx = fmaxf(mx, __ldcg(pb + ((size_t)s2 * G + hh) * (2 + 128)));
    float ls = 0.f, acc = 0.f;
    for (int s2 = 0; s2 < S; ++s2) {
      const float* pg = pb + ((size_t)s2 * G + hh) * (2 + 128);
      const float ms = __ldcg(pg);
      const float sc = ms == -INFINITY ? 0.f : exp2f(ms - mx);
      ls += __ldcg(pg + 1) * sc;
      acc += __ldcg(pg + 2 + c) * sc;
    }
    A.out[((size_t)b * G + hh) * 128 + c] = acc / ls;
  }
  if (threadIdx.x == 0) A.counter[b] = 0;
}

}  // namespace icb

using namespace icb;

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// [rows][128] bf16 plane stack viewed as a 2-D tensor; boxes of 64 rows x 64
// columns, 128-byte swizzle (one box row = one 128-byte swizzle row).
static int make_plane_map(CUtensorMap* map, const void* base, long long rows) {
  auto enc = tensor_map_encoder();
  if (!enc) { icb_set_error(ICB_E_CUDA, "cuTensorMapEncodeTiled unavailable"); return ICB_E_CUDA; }
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128 * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)kDenseTile};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { icb_set_error(ICB_E_CUDA, "cuTensorMapEncodeTiled failed"); return ICB_E_CUDA; }
  return ICB_OK;
}

// True when the TMA / tensor-core kernel serves this call (bf16, d = d' = 128, G <= 8).
bool icb_dense_flash_ok(int G, int dim, int dim_v, int kv_dtype) {
  return kv_dtype == ICB_KV_BF16 && dim == 128 && dim_v == 128 && G >= 1 && G <= 8 &&
         !getenv("ICB_DENSE_SIMT");
}

int icb_dense_flash_impl(int32_t n, int32_t G, const float* q, const void* k, const void* v, int64_t ld,
                         int32_t n_tokens, const int32_t* token_dev, float* out, int32_t splits, float* part,
                         unsigned* counter, cudaStream_t st) {
  CUtensorMap mk, mv;
  if (int rc = make_plane_map(&mk, k, (long long)n * ld)) return rc;
  if (int rc = make_plane_map(&mv, v, (long long)n * ld)) return rc;
  DenseArgs A{};
  A.n = n; A.G = G; A.splits = splits; A.ld = ld; A.n_tokens = n_tokens; A.token_dev = token_dev;
  A.q = q; A.out = out; A.part = part; A.counter = counter;
  A.scale_log2 = (float)(1.4426950408889634 / sqrt(128.0));
  constexpr int NS = kDenseStages;
  const size_t smem = (size_t)2 * NS * kDenseTileBytes + 1024;
  static bool attr = false;
  if (!attr) {
    ICB_CUDA(cudaFuncSetAttribute(dense_flash_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dense_flash_kernel<NS><<<dim3(n, splits), kDenseThreads, smem, st>>>(mk, mv, A);
  ICB_CUDA(cudaGetLastError());
  return ICB_OK;
}
