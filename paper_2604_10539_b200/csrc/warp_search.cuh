// Warp-synchronous parent search for inserts: DciTree.query with
// PARENT_BUDGET (k = 1, beam = 8, visit_cap = 64; dci.py:78) targeted at
// level + 1 (dci.py:318-364, :385-431), one warp per point and no block
// barriers.  The parent search is tiny (<= 8 nodes of <= 64 members per
// level), so the block search's per-level phases (union, scans, selection
// passes, each ending in a block barrier) dominate its cost; a warp walks
// the levels on its own and the 8 warps of the insert CTA search up to 8
// points at once (insert.cu batches the level-1 points, whose searches read
// only levels >= 2 and so never see each other's inserts).
//
// Same candidate sets and numerics as the block search: level L reads the
// top node, level lv < L the members of own(s, lv) for the survivors s; d2
// is the fixed-order fp32 distance (per lane fma chain, xor butterfly
// 16,8,4,2,1 -- the first three levels transposed across 8 rows, which keeps
// each row's pairing tree); ranking keys (d2 bits, id).  A node that the
// reference would visit with P-DCI (size > 64 = max(EXHAUSTIVE_NODE_LIMIT,
// visit_cap)) makes the search return false: the caller falls back to the
// block search, which implements P-DCI.
#pragma once
#include "icb.cuh"

namespace icb {

constexpr int kWarpBeam = 8;
constexpr int kWarpMaxCand = kWarpBeam * 64;   // 8 nodes x 64 members

struct WarpSearchBuf {   // per warp, shared memory
  int ids[kWarpMaxCand];
  unsigned long long keys[kWarpMaxCand];
};

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned lo = __shfl_xor_sync(0xffffffffu, (unsigned)v, o);
    const unsigned hi = __shfl_xor_sync(0xffffffffu, (unsigned)(v >> 32), o);
    const unsigned long long w = ((unsigned long long)hi << 32) | lo;
    v = w < v ? w : v;
  }
  return v;
}

// q: lifted query (smem, ICB_DPAD floats), qt its tail.  On success returns
// true with *parent (-1 if the floor level had no candidate) and adds the
// distance evaluations to *evals (lane 0's copy is authoritative).
__device__ inline bool warp_parent_search(const ForestView& F, int t, const float* q, float qt, int target,
                                   WarpSearchBuf& W, int* parent, unsigned long long* evals) {
  const int lane = threadIdx.x & 31;
  const TreeMeta& mt = F.meta[t];
  const int L = mt.levels;
  const int floor = min(target, L);
  const int* mem = F.mem(t);
  const float4 qv = reinterpret_cast<const float4*>(q)[lane];
  const int pi = (lane >> 2) & 7;
  int sv = -1;       // survivor id held by lane i < ns
  int ns = 0;
  unsigned long long ev = 0;
  for (int lv = L; lv >= floor; --lv) {
    // the level's nodes: lane i < nn holds node i
    const int nn = lv == L ? 1 : ns;
    int sz = 0, off = 0;
    if (lane < nn) {
      const int nd = lv == L ? mt.top_node : F.own(t, sv, lv);
      sz = F.node_size[F.nd(t, nd)];
      off = F.node_off[F.nd(t, nd)];
    }
    if (__any_sync(0xffffffffu, sz > 64)) return false;   // P-DCI node: block search
    int ex = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ex, o);
      if (lane >= o) ex += y;
    }
    const int M = __shfl_sync(0xffffffffu, ex, 31);
    ex -= sz;
    // candidate ids, node by node (coalesced member copies)
    for (int i = 0; i < nn; ++i) {
      const int e = __shfl_sync(0xffffffffu, ex, i), o = __shfl_sync(0xffffffffu, off, i);
      const int s = __shfl_sync(0xffffffffu, sz, i);
      for (int j = lane; j < s; j += 32) W.ids[e + j] = mem[o + j];
    }
    __syncwarp();
    ev += (unsigned long long)M;
    // distances, two 8-row batches per round trip: in slot jj of a batch lane
    // l scores row jj ^ pi(l); each lane's output-row tail is loaded with the rows
    for (int b0 = 0; b0 < M; b0 += 16) {
      int idm[2];
      float tl[2];
      float4 p[2][8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int bb = b0 + 8 * h;
        const int cm = bb + pi;
        idm[h] = W.ids[cm < M ? cm : b0];
        tl[h] = F.tail[F.tk(t, idm[h])];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int c = bb + (jj ^ pi);
          p[h][jj] = reinterpret_cast<const float4*>(F.row(t, W.ids[c < M ? c : b0]))[lane];
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) v[jj] = lane_sq4(p[h][jj], qv);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) v[jj] = __fadd_rn(v[jj], __shfl_xor_sync(0xffffffffu, v[jj + 4], 16));
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) v[jj] = __fadd_rn(v[jj], __shfl_xor_sync(0xffffffffu, v[jj + 2], 8));
        float f = __fadd_rn(v[0], __shfl_xor_sync(0xffffffffu, v[1], 4));
        f = __fadd_rn(f, __shfl_xor_sync(0xffffffffu, f, 2));
        f = __fadd_rn(f, __shfl_xor_sync(0xffffffffu, f, 1));
        const int cm = b0 + 8 * h + pi;
        if ((lane & 3) == 0 && cm < M) W.keys[cm] = make_key(d2_finish(f, tl[h], qt), idm[h]);
      }
    }
    __syncwarp();
    // top-B by B rounds of warp argmin over the unique keys
    const int B = lv > floor ? min(kWarpBeam, M) : min(1, M);
    unsigned long long last = 0ull;
    int got = 0;
    for (int r = 0; r < B; ++r) {
      unsigned long long best = ~0ull;
      for (int c = lane; c < M; c += 32) {
        const unsigned long long k = W.keys[c];
        if ((r == 0 || k > last) && k < best) best = k;
      }
      best = warp_min_u64(best);
      last = best;
      if (lane == r) sv = key_id(best);
      ++got;
    }
    ns = got;
    __syncwarp();
  }
  *parent = ns > 0 ? __shfl_sync(0xffffffffu, sv, 0) : -1;
  *evals += ev;
  return true;
}

}  // namespace icb
