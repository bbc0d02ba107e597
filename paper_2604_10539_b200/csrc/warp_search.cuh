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
// reference visits with P-DCI (size > 64 = max(EXHAUSTIVE_NODE_LIMIT,
// visit_cap)) contributes its 64-member visit list, computed here from the
// tree's P-DCI cache (member projections and ladder ranks, search.cuh
// pc_ensure) when the node's entries and directions are cached and it has at
// most kWarpPdciMax members; otherwise the search returns false and the
// caller falls back to the block search (which also fills the cache).
#pragma once
#include "icb.cuh"

namespace icb {

constexpr int kWarpBeam = 8;
constexpr int kWarpMaxCand = kWarpBeam * 64;   // 8 nodes x 64 members
constexpr int kWarpPdciMax = 256;              // P-DCI nodes the warp visits itself (8 members per lane)
// warp-search P-DCI misses by reason: too large, no directions, no cache entries, stale entries
static __device__ unsigned long long g_pdci_miss[4];

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

// P-DCI visit list of node x (sz > 64 members at `moff`, cache entries at
// `pco`, directions `dirs`) for the lifted query (q, qt): the 64 members of
// smallest emission key (search.cuh pdci_visit, same keys) into out[0..64).
__device__ inline void warp_pdci_visit(const ForestView& F, int t, const int* mem, int sz, int pco,
                                       const double* dirs, const float* q, float qt, int* out) {
  const int lane = threadIdx.x & 31;
  const int D1 = F.dim + 1;
  const double* proj = F.pc_proj + ((size_t)t * F.pc_cap + pco) * ICB_NPROJ;
  const int* ord = F.pc_ord + ((size_t)t * F.pc_cap + pco) * ICB_NPROJ;
  const int* pos = F.pc_pos + ((size_t)t * F.pc_cap + pco) * ICB_NPROJ;
  // query projection and ladder start of direction `lane` (lanes 0..7), the
  // same sequential fp64 chain as the block visit
  double qp = 0.0;
  int st = 0;
  if (lane < ICB_NPROJ) {
    double acc = 0.0;
    for (int u = 0; u < D1; ++u) acc = __fma_rn(dirs[lane * D1 + u], u < F.dim ? (double)q[u] : (double)qt, acc);
    qp = acc;
    int lo = 0, hi = sz;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (proj[(size_t)ord[(size_t)mid * ICB_NPROJ + lane] * ICB_NPROJ + lane] < qp) lo = mid + 1;
      else hi = mid;
    }
    st = lo;
  }
  double qpj[ICB_NPROJ];
  int stj[ICB_NPROJ];
#pragma unroll
  for (int j = 0; j < ICB_NPROJ; ++j) { qpj[j] = __shfl_sync(0xffffffffu, qp, j); stj[j] = __shfl_sync(0xffffffffu, st, j); }
  constexpr int R = kWarpPdciMax / 32;
  unsigned long long kh[R];
  unsigned kl[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    unsigned long long bh = ~0ull, bl = 0xffffffffull;
    if (i < sz) {
      bh = 0; bl = 0;
#pragma unroll
      for (int j = 0; j < ICB_NPROJ; ++j) {
        const int p = pos[(size_t)i * ICB_NPROJ + j];
        const double gap = fabs(__dsub_rn(proj[(size_t)i * ICB_NPROJ + j], qpj[j]));
        const unsigned long long h = (unsigned long long)__double_as_longlong(gap);
        const unsigned long long sec = p < stj[j] ? (unsigned long long)((1 << 23) - 1 - p)
                                                  : (unsigned long long)((1 << 23) + p);
        const unsigned long long l = ((unsigned long long)j << 24) | sec;
        if (h > bh || (h == bh && l > bl)) { bh = h; bl = l; }
      }
    }
    kh[r] = bh;
    kl[r] = (unsigned)bl;
  }
  // 64 rounds of warp argmin over the (unique) emission keys
  for (int c = 0; c < 64; ++c) {
    unsigned long long mh = ~0ull;
    unsigned ml = 0xffffffffu;
    int mr = -1;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (kh[r] < mh || (kh[r] == mh && kl[r] < ml)) { mh = kh[r]; ml = kl[r]; mr = r; }
    const unsigned long long wh = warp_min_u64(mh);
    const unsigned wl = __reduce_min_sync(0xffffffffu, mh == wh ? ml : 0xffffffffu);
    const bool mine = mh == wh && ml == wl && mr >= 0;
    if (mine) {
      out[c] = mem[lane + 32 * mr];
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r == mr) { kh[r] = ~0ull; kl[r] = 0xffffffffu; }
    }
  }
  __syncwarp();
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
    int sz = 0, off = 0, nd = -1;
    if (lane < nn) {
      nd = lv == L ? mt.top_node : F.own(t, sv, lv);
      sz = F.node_size[F.nd(t, nd)];
      off = F.node_off[F.nd(t, nd)];
    }
    // P-DCI nodes: 64-member visit lists from the cache, else the block search
    const bool big = sz > 64;
    if (__any_sync(0xffffffffu, big)) {
      const bool ready = !big || (sz <= kWarpPdciMax && F.node_pcm[F.nd(t, nd)] == sz &&
                                  F.node_pc[F.nd(t, nd)] >= 0 && F.node_dirs[F.nd(t, nd)] >= 0);
      if (!ready) {   // why the warp cannot visit this P-DCI node (icb_pdci_stats)
        const size_t x = F.nd(t, nd);
        const int why = sz > kWarpPdciMax ? 0 : F.node_dirs[x] < 0 ? 1 : F.node_pc[x] < 0 ? 2 : 3;
        atomicAdd(&g_pdci_miss[why], 1ull);
      }
      if (!__all_sync(0xffffffffu, ready)) return false;
    }
    const int cnt = big ? 64 : sz;
    int ex = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ex, o);
      if (lane >= o) ex += y;
    }
    const int M = __shfl_sync(0xffffffffu, ex, 31);
    ex -= cnt;
    // candidate ids, node by node (coalesced member copies / P-DCI visit lists)
    for (int i = 0; i < nn; ++i) {
      const int e = __shfl_sync(0xffffffffu, ex, i), o = __shfl_sync(0xffffffffu, off, i);
      const int s = __shfl_sync(0xffffffffu, sz, i);
      if (s > 64) {
        const size_t x = F.nd(t, __shfl_sync(0xffffffffu, nd, i));
        const double* dirs = F.dirs + ((size_t)t * F.dirs_cap + F.node_dirs[x]) * ICB_NPROJ * (F.dim + 1);
        warp_pdci_visit(F, t, mem + o, s, F.node_pc[x], dirs, q, qt, W.ids + e);
      } else {
        for (int j = lane; j < s; j += 32) W.ids[e + j] = mem[o + j];
      }
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
