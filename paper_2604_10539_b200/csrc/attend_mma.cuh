// The decode step's sparse attention on the tensor cores: one tree's sink,
// window and selected pages (sparse_attention over the attended set in entry
// order, attention.py:77-93, engine.py:449-475), bf16 page K/V with
// d = d' = 128 and up to 8 query heads, inside the search kernel after the
// search (the CTA's row ring is idle then).
//
// Each warp takes pages round-robin and streams them in 8-row chunks
// (a page of fill <= 8 is one chunk): K and V rows arrive with 16-byte cp.async
// into a two-stage per-warp slot of the ring (XOR-swizzled 16-byte chunks, so
// ldmatrix reads are conflict-free; rows past the page's fill are zero
// filled), the next chunk loading while the current one computes:
//   S = Q K^T   mma.sync m16n8k16 bf16 (the heads are the M rows, padded to
//               16; q as two bf16 halves, ~16 mantissa bits), K by ldmatrix
//   softmax     online, per head over the chunk's 8 rows (4 lanes per head)
//   O += P V    mma.sync m16n8k8 bf16, P straight from the S accumulator,
//               V by ldmatrix.trans
// then the warps' (m, l, O) merge in shared memory.  About 10 instructions
// per row against ~90 for the CUDA-core chunk loop (attend.cuh).
#pragma once
#include "attend.cuh"

namespace icb {

__device__ __forceinline__ unsigned pack_bf2_rn(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<unsigned*>(&v);
}

__device__ __forceinline__ void mma16816(float (&d)[4], unsigned a0, unsigned a2, unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma1688(float (&d)[4], unsigned a0, unsigned b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(b0));
}
__device__ __forceinline__ void ldsm4(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// 16-byte async copy with zero fill beyond src_bytes (0 or 16)
template <bool NC>
__device__ __forceinline__ void cp16z(unsigned dst, const void* src, int src_bytes) {
  if constexpr (NC)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
  else   // written earlier in the same kernel (fused rotation / KV pool gather): L2 path is coherent anyway
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// Byte offset of (row 0..7, 16-byte chunk c 0..15) in an 8-row x 256-byte tile.
__device__ __forceinline__ unsigned sw8(int row, int c) { return (unsigned)(row * 256 + ((c ^ row) << 4)); }

constexpr int kMmaSlot = 8192;   // per warp: 2 stages x (K 2 KB + V 2 KB)

// Usable when the page K/V are bf16 with d = d' = 128 and G <= 8.
__device__ __forceinline__ bool attend_mma_ok(const ForestView& F, int GA) {
  return F.kv_bf16 && F.dim == 128 && F.dim_v == 128 && F.dkp == 128 && F.dvp == 128 && GA <= 8;
}

template <int NT, bool NC>
__device__ void attend_tree_mma(const ForestView& F, int t, int GA, const float* q /*[GA][128]*/,
                                const int32_t* sel, int nsel, float* out /*[GA][128]*/, float scale_log2,
                                unsigned char* smem /* >= NT/32 * kMmaSlot */,
                                unsigned char* qtile /* 4 KB: q hi / lo as bf16 [2][8 heads][128] */) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const bool head = g < GA;
  const TreeMeta* m = F.meta + t;
  const int nsink = m->n_sink, nfix = nsink + m->n_window, total = nfix + nsel;
  const __nv_bfloat16* K = (const __nv_bfloat16*)(F.kv_host ? F.pool_k : F.page_k);
  const __nv_bfloat16* V = (const __nv_bfloat16*)(F.kv_host ? F.pool_v : F.page_v);
  // q as bf16 hi / lo halves in shared memory (8 x 256-byte rows each, the
  // same swizzle as the K tiles); A-fragments are read per chunk with ldmatrix
  const unsigned qs = (unsigned)__cvta_generic_to_shared(qtile);
  for (int x = threadIdx.x; x < 8 * 64; x += NT) {
    const int hh = x >> 6, c2 = (x & 63) * 2;
    const float x0 = hh < GA ? q[(size_t)hh * 128 + c2] : 0.f, x1 = hh < GA ? q[(size_t)hh * 128 + c2 + 1] : 0.f;
    const __nv_bfloat162 hi = __floats2bfloat162_rn(x0, x1);
    const float2 hf = __bfloat1622float2(hi);
    const unsigned off = sw8(hh, c2 >> 3) + (c2 & 7) * 2;
    *reinterpret_cast<__nv_bfloat162*>(qtile + off) = hi;
    *reinterpret_cast<unsigned*>(qtile + 2048 + off) = pack_bf2_rn(x0 - hf.x, x1 - hf.y);
  }
  __syncthreads();
  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float mrun = -INFINITY, lrun = 0.f;
  const unsigned slot = (unsigned)__cvta_generic_to_shared(smem + (size_t)warp * kMmaSlot);
  // this warp's chunk sequence: pages warp, warp + NW, ...; chunks of 8 rows
  auto page_of = [&](int i) { return i < nsink ? m->sink[i] : i < nfix ? m->win[i - nsink] : sel[i - nfix]; };
  int pi = warp, r0 = 0;          // chunk being issued
  int fill_i = -1;
  size_t base_i = 0;
  auto locate = [&](int i, int& fill, size_t& base) {
    const int p = page_of(i);
    if (F.kv_host) {
      const int sl = F.page_slot[F.pg(t, p)];
      if (sl < 0) { fill = 0; base = 0; return; }   // pool overflow (ICB_ERR_CAP_SCRATCH set)
      base = ((size_t)t * F.pool_cap + sl) * F.s;
    } else {
      base = F.pg(t, p) * F.s;
    }
    fill = F.page_fill[F.pg(t, p)];
  };
  // issue chunk (base, r0, nrow) into stage st: lane copies 4 K and 4 V 16-byte chunks
  auto issue = [&](int st, size_t base, int rr0, int nrow) {
    const unsigned dk = slot + st * 4096, dv = dk + 2048;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = lane + 32 * u;       // 0..127: row e / 16, chunk e % 16
      const int row = e >> 4, c = e & 15;
      const bool on = row < nrow;
      const size_t rg = base + rr0 + (on ? row : 0);
      cp16z<NC>(dk + sw8(row, c), K + rg * 128 + c * 8, on ? 16 : 0);
      cp16z<NC>(dv + sw8(row, c), V + rg * 128 + c * 8, on ? 16 : 0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // advance (pi, r0) to the next chunk with rows; returns false at the end
  auto next_chunk = [&](int& i, int& rr0, int& fill, size_t& base) -> bool {
    while (i < total) {
      if (fill < 0) locate(i, fill, base);
      if (rr0 < fill) return true;
      i += NW;
      rr0 = 0;
      fill = -1;
    }
    return false;
  };
  bool have = next_chunk(pi, r0, fill_i, base_i);
  int cur_st = 0;
  int cur_nrow = 0;
  if (have) {
    cur_nrow = min(8, fill_i - r0);
    issue(0, base_i, r0, cur_nrow);
    r0 += 8;
  }
  const int mi = lane >> 3, rr = lane & 7;
  while (have) {
    // prefetch the following chunk into the other stage
    const bool more = next_chunk(pi, r0, fill_i, base_i);
    int nxt_nrow = 0;
    if (more) {
      nxt_nrow = min(8, fill_i - r0);
      issue(cur_st ^ 1, base_i, r0, nxt_nrow);
      r0 += 8;
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const unsigned kb = slot + cur_st * 4096, vb = kb + 2048;
    // S = Q K^T over the chunk's 8 rows
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kp = 0; kp < 4; ++kp) {   // two 16-dim steps per ldmatrix.x4
      unsigned b0, b1, b2, b3, a0, a1, a2, a3, l0, l1, l2, l3;
      ldsm4(kb + sw8(rr, 4 * kp + mi), b0, b1, b2, b3);
      ldsm4(qs + sw8(rr, 4 * kp + mi), a0, a1, a2, a3);          // heads 0..7: (lo, hi) of two k-steps
      ldsm4(qs + 2048 + sw8(rr, 4 * kp + mi), l0, l1, l2, l3);
      mma16816(sc, a0, a1, b0, b1);
      mma16816(sc, l0, l1, b0, b1);
      mma16816(sc, a2, a3, b2, b3);
      mma16816(sc, l2, l3, b2, b3);
    }
    // online softmax: lane holds rows 2 t4, 2 t4 + 1 of head g
    const float x0 = 2 * t4 < cur_nrow ? sc[0] * scale_log2 : -INFINITY;
    const float x1 = 2 * t4 + 1 < cur_nrow ? sc[1] * scale_log2 : -INFINITY;
    float mx = fmaxf(x0, x1);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(mrun, mx);
    const float alpha = mn == -INFINITY ? 1.f : exp2f(mrun - mn);
    const float p0 = mn == -INFINITY ? 0.f : exp2f(x0 - mn), p1 = mn == -INFINITY ? 0.f : exp2f(x1 - mn);
    lrun = lrun * alpha + p0 + p1;
    mrun = mn;
#pragma unroll
    for (int j = 0; j < 16; ++j) { o[j][0] *= alpha; o[j][1] *= alpha; }
    const unsigned pa = pack_bf2_rn(p0, p1);
    // O += P V: per 8-dim n-tile, B = V rows 0..7 (k) x 8 dims, via ldmatrix.trans (4 tiles per x4)
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      unsigned v0, v1, v2, v3;
      ldsm4t(vb + sw8(rr, j + mi), v0, v1, v2, v3);
      mma1688(o[j], pa, v0);
      mma1688(o[j + 1], pa, v1);
      mma1688(o[j + 2], pa, v2);
      mma1688(o[j + 3], pa, v3);
    }
    __syncwarp();
    have = more;
    cur_st ^= 1;
    cur_nrow = nxt_nrow;
  }
  // per-head l over the head's 4 lanes; the warps' states merge in shared memory
  lrun += __shfl_xor_sync(0xffffffffu, lrun, 1);
  lrun += __shfl_xor_sync(0xffffffffu, lrun, 2);
  __syncthreads();   // every warp is done with its slot
  float* s_m = reinterpret_cast<float*>(smem);             // [NW][8]
  float* s_l = s_m + NW * 8;                                // [NW][8]
  float* s_o = s_l + NW * 8;                                // [NW][8][128]
  if (head) {
    if (t4 == 0) { s_m[warp * 8 + g] = mrun; s_l[warp * 8 + g] = lrun; }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      s_o[(warp * 8 + g) * 128 + 8 * j + 2 * t4] = o[j][0];
      s_o[(warp * 8 + g) * 128 + 8 * j + 2 * t4 + 1] = o[j][1];
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < GA * 128; x += NT) {
    const int hh = x >> 7, c = x & 127;
    float mx = -INFINITY;
    for (int w = 0; w < NW; ++w) mx = fmaxf(mx, s_m[w * 8 + hh]);
    float ls = 0.f, acc = 0.f;
    for (int w = 0; w < NW; ++w) {
      const float sw = s_m[w * 8 + hh] == -INFINITY ? 0.f : exp2f(s_m[w * 8 + hh] - mx);
      ls += s_l[w * 8 + hh] * sw;
      acc += s_o[(w * 8 + hh) * 128 + c] * sw;
    }
    out[(size_t)hh * 128 + c] = acc / ls;
  }
  __syncthreads();
}

}  // namespace icb
