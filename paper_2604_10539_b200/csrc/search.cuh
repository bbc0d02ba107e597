// Block-level DCI tree search: DciTree.query (dci.py:318-364) for G query
// heads of one tree at once, plus P-DCI within-node truncation
// (_node_candidates / _NodeSearch.visit_order, dci.py:91-135, 300-314).
//
// One CTA owns one tree.  Per level it forms the UNION of the nodes the G
// heads' survivors point to, streams each member row of that union once
// (coalesced 512-byte rows, one warp per node), computes the fp32 lifted
// distance to every head that requested the node, and writes 64-bit keys
// (d2 bits << 32 | token id) to per-head candidate lists.  Per head a
// block-wide radix select picks the `beam` survivors and the level's top-k
// (unique keys, so exact); a per-head pool collects the top-k of every level
// (every level for the sentinel target, only the floor otherwise) and the
// final top-k is sorted in shared memory.
#pragma once
#include "icb.cuh"

namespace icb {

constexpr int kSearchThreads = 512;
constexpr int kSortMax = 4096;   // largest k served by the in-smem final sort

struct SearchScratch {
  unsigned long long* cand;   // [G][ccap]
  unsigned long long* pool;   // [G][ccap]
  int* surv;                  // [G][ccap]
  int* ulist;                 // [node_cap]
  int* umask;                 // [node_cap]
  int* uoff;                  // [G][node_cap]
  unsigned* nmask;            // [node_cap]   zero between levels
  unsigned* seen;             // [G][tok_cap/32+1] zero between queries
  int* vis;                   // [tok_cap]  P-DCI visit list
  double* proj;               // [tok_cap][8] P-DCI projections
  unsigned long long* ekey;   // [tok_cap][2] P-DCI emission keys
  int ccap;
};

struct SearchSmem {
  float q[ICB_MAX_G][ICB_DPAD];
  float qt[ICB_MAX_G];
  double q64[ICB_DPAD + 1];
  double dirs_tmp[ICB_NPROJ];
  int hist[256];
  int wsum[kSearchThreads / 32 + 1];
  int U, nbig;
  int M[ICB_MAX_G];
  int nsurv[ICB_MAX_G];
  int npool[ICB_MAX_G];
  int cnt;
  unsigned long long thr;
  int scan_carry[ICB_MAX_G];
  int misc[8];
  unsigned long long sortbuf[kSortMax];
};

// ------------------------------------------------------------------ select
// Select the B smallest of M unique keys in `keys` (global).  Writes the
// selected keys to out_keys (if not null) and/or their ids to out_ids, in
// arbitrary order; returns the count (= min(B, M)) via smem misc[0].
// If `seen` is given (pool mode), keys whose id is already marked are skipped
// at output time and newly output ids are marked.
template <int NT>
__device__ int block_select(SearchSmem& S, const unsigned long long* keys, int M, long long B,
                            unsigned long long* out_keys, int* out_ids, int out_base,
                            unsigned* seen) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long thr;
  if (B >= M) {
    thr = ~0ull;
  } else {
    unsigned long long prefix = 0, pmask = 0;
    long long remaining = B;   // how many still to take at or below the prefix
    thr = ~0ull;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += NT) S.hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < M + (NT - (M % NT)) % NT; i += NT) {
        bool valid = i < M;
        unsigned long long k = valid ? keys[i] : 0;
        valid = valid && ((k & pmask) == prefix);
        int dig = (int)((k >> shift) & 0xff);
        unsigned act = __ballot_sync(0xffffffffu, valid);
        if (valid) {
          unsigned peers = __match_any_sync(act, dig);
          if ((__ffs(peers) - 1) == lane) atomicAdd(&S.hist[dig], __popc(peers));
        }
      }
      __syncthreads();
      if (warp == 0) {
        // find digit where cumulative count reaches `remaining`
        int c[8];
        int local = 0;
        for (int u = 0; u < 8; ++u) { c[u] = S.hist[lane * 8 + u]; local += c[u]; }
        int incl = local;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        int excl = incl - local;
        bool mine = (excl < remaining) && (incl >= remaining);
        unsigned who = __ballot_sync(0xffffffffu, mine);
        int src = __ffs(who) - 1;
        int digit = 0, before = 0, inbucket = 0;
        if (lane == src) {
          int run = excl;
          for (int u = 0; u < 8; ++u) {
            if (run + c[u] >= remaining) { digit = lane * 8 + u; before = run; inbucket = c[u]; break; }
            run += c[u];
          }
        }
        digit = __shfl_sync(0xffffffffu, digit, src);
        before = __shfl_sync(0xffffffffu, before, src);
        inbucket = __shfl_sync(0xffffffffu, inbucket, src);
        if (lane == 0) {
          S.misc[1] = digit;
          S.misc[2] = before;
          S.misc[3] = inbucket;
        }
      }
      __syncthreads();
      int digit = S.misc[1], before = S.misc[2], inbucket = S.misc[3];
      remaining -= before;
      prefix |= (unsigned long long)digit << shift;
      pmask |= 0xffull << shift;
      if (inbucket == remaining || shift == 0) {
        thr = prefix | ~pmask;   // every key under this prefix is taken
        break;
      }
      __syncthreads();
    }
  }
  if (tid == 0) S.misc[0] = 0;
  __syncthreads();
  for (int i = tid; i < M + (NT - (M % NT)) % NT; i += NT) {
    bool take = false;
    unsigned long long k = 0;
    if (i < M) {
      k = keys[i];
      take = k <= thr;
      if (take && seen) {
        int id = key_id(k);
        unsigned bit = 1u << (id & 31);
        unsigned old = atomicOr(seen + (id >> 5), bit);
        take = !(old & bit);
      }
    }
    unsigned bal = __ballot_sync(0xffffffffu, take);
    int base = 0;
    if (lane == 0 && bal) base = atomicAdd(&S.misc[0], __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (take) {
      int pos = out_base + base + __popc(bal & ((1u << lane) - 1));
      if (out_keys) out_keys[pos] = k;
      if (out_ids) out_ids[pos] = key_id(k);
    }
  }
  __syncthreads();
  int r = S.misc[0];
  __syncthreads();
  return r;
}

// bitonic sort of n (<= kSortMax) keys in S.sortbuf, ascending
template <int NT>
__device__ void block_sort(SearchSmem& S, int n) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = n + threadIdx.x; i < P; i += NT) S.sortbuf[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += NT) {
        int ixj = i ^ j;
        if (ixj > i) {
          unsigned long long a = S.sortbuf[i], b = S.sortbuf[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) { S.sortbuf[i] = b; S.sortbuf[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ P-DCI
// Per-node unit directions, generated on the device from the tree's seed
// (SeedSequence(entropy, spawn_key=(1, node_id)), normal, row-normalized with
// NumPy's pairwise norm; dci.py:268-273), cached in the forest.
template <int NT>
__device__ const double* pdci_dirs(const ForestView& F, int t, int node, double* tmp /*global 8*(dim+1)*/) {
  __shared__ int s_slot;
  const int D1 = F.dim + 1;
  if (threadIdx.x == 0) {
    int slot = F.node_dirs[F.nd(t, node)];
    if (slot < 0) {
      int ns = atomicAdd(&F.meta[t].n_dirs, 1);
      slot = ns < F.dirs_cap ? ns : -1;
      double* dst = slot >= 0 ? F.dirs + ((size_t)t * F.dirs_cap + slot) * ICB_NPROJ * D1 : tmp;
      uint32_t spawn[2] = {1u, (uint32_t)node};
      uint64_t st[4];
      icb_seedseq_u64x4(F.meta[t].entropy, F.meta[t].n_entropy, spawn, 2, st);
      Pcg64 g = icb_pcg_seed(st);
      for (int j = 0; j < ICB_NPROJ * D1; ++j) dst[j] = icb_normal(g);
      double sq[ICB_DPAD + 1];
      for (int j = 0; j < ICB_NPROJ; ++j) {
        for (int u = 0; u < D1; ++u) sq[u] = __dmul_rn(dst[j * D1 + u], dst[j * D1 + u]);
        double nrm = sqrt(pairwise_sum(sq, D1));
        for (int u = 0; u < D1; ++u) dst[j * D1 + u] = __ddiv_rn(dst[j * D1 + u], nrm);
      }
      __threadfence();
      if (slot >= 0) F.node_dirs[F.nd(t, node)] = slot;
      s_slot = slot;
    } else {
      s_slot = slot;
    }
  }
  __syncthreads();
  int slot = s_slot;
  return slot >= 0 ? F.dirs + ((size_t)t * F.dirs_cap + slot) * ICB_NPROJ * D1 : tmp;
}

// Visit list of a large node (cap entries, ascending emission order) into
// SS.vis; returns the count.  Emission key of a member = lexicographic max over
// its 8 ladder entries of (gap, j, chain position) -- the pop order of the
// reference's heap merge (see oracle/dci.py:visit_order for the equivalence).
template <int NT>
__device__ int pdci_visit(SearchSmem& S, const ForestView& F, const SearchScratch& SS, int t, int node,
                          int g, long long cap, double* dirs_tmp) {
  const int D1 = F.dim + 1;
  const int off = F.node_off[F.nd(t, node)], m = F.node_size[F.nd(t, node)];
  const int* mem = F.mem(t) + off;
  const double* dirs = pdci_dirs<NT>(F, t, node, dirs_tmp);
  // query lifted vector in fp64 (device fp32 lift, tail qt)
  for (int u = threadIdx.x; u < D1; u += NT) S.q64[u] = u < F.dim ? (double)S.q[g][u] : (double)S.qt[g];
  __syncthreads();
  if (threadIdx.x < ICB_NPROJ) {
    double acc = 0.0;
    for (int u = 0; u < D1; ++u) acc = __fma_rn(dirs[threadIdx.x * D1 + u], S.q64[u], acc);
    S.dirs_tmp[threadIdx.x] = acc;   // query projections
  }
  // member projections
  for (int x = threadIdx.x; x < m * ICB_NPROJ; x += NT) {
    int i = x / ICB_NPROJ, j = x % ICB_NPROJ;
    const float* row = F.row(t, mem[i]);
    double acc = 0.0;
    for (int u = 0; u < F.dim; ++u) acc = __fma_rn(dirs[j * D1 + u], (double)row[u], acc);
    acc = __fma_rn(dirs[j * D1 + F.dim], (double)F.tail[F.tk(t, mem[i])], acc);
    SS.proj[(size_t)i * ICB_NPROJ + j] = acc;
  }
  __syncthreads();
  // emission keys
  for (int i = threadIdx.x; i < m; i += NT) {
    unsigned long long best_hi = 0, best_lo = 0;
    int id_i = mem[i];
    for (int j = 0; j < ICB_NPROJ; ++j) {
      double pj = SS.proj[(size_t)i * ICB_NPROJ + j];
      double qp = S.dirs_tmp[j];
      int pos = 0, start = 0;
      for (int i2 = 0; i2 < m; ++i2) {
        double p2 = SS.proj[(size_t)i2 * ICB_NPROJ + j];
        int id2 = mem[i2];
        pos += (p2 < pj || (p2 == pj && id2 < id_i)) ? 1 : 0;
        start += p2 < qp ? 1 : 0;
      }
      double gap = fabs(__dsub_rn(pj, qp));
      unsigned long long hi = (unsigned long long)__double_as_longlong(gap);
      unsigned long long sec = pos < start ? (unsigned long long)((1 << 23) - 1 - pos)
                                           : (unsigned long long)((1 << 23) + pos);
      unsigned long long lo = ((unsigned long long)j << 24) | sec;
      if (hi > best_hi || (hi == best_hi && lo > best_lo)) { best_hi = hi; best_lo = lo; }
    }
    SS.ekey[2 * (size_t)i] = best_hi;
    SS.ekey[2 * (size_t)i + 1] = best_lo;
  }
  __syncthreads();
  int cnt = (int)min((long long)m, cap);
  for (int i = threadIdx.x; i < m; i += NT) {
    unsigned long long hi = SS.ekey[2 * (size_t)i], lo = SS.ekey[2 * (size_t)i + 1];
    int rank = 0;
    for (int i2 = 0; i2 < m; ++i2) {
      unsigned long long h2 = SS.ekey[2 * (size_t)i2], l2 = SS.ekey[2 * (size_t)i2 + 1];
      rank += (h2 < hi || (h2 == hi && l2 < lo)) ? 1 : 0;
    }
    if (rank < cnt) SS.vis[rank] = mem[i];
  }
  __syncthreads();
  return cnt;
}

// ------------------------------------------------------------------ search
struct SearchParams {
  int G;
  long long k, beam, visit_cap;
  int target;   // -1 sentinel
};

// Evaluate the rows `ids[0..n)` against head g (single head; used by the
// P-DCI path) writing keys to dst.
template <int NT>
__device__ void eval_list_one_head(SearchSmem& S, const ForestView& F, int t, const int* ids, int n, int g,
                                   unsigned long long* dst) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4 qv = reinterpret_cast<const float4*>(S.q[g])[lane];
  for (int i = warp; i < n; i += NT / 32) {
    int id = ids[i];
    float4 p = reinterpret_cast<const float4*>(F.row(t, id))[lane];
    float s = warp_sum_butterfly(lane_sq4(p, qv));
    float d2 = d2_finish(s, F.tail[F.tk(t, id)], S.qt[g]);
    if (lane == 0) dst[i] = make_key(d2, id);
  }
}

// The multi-level search.  On entry S.q/S.qt hold the lifted queries.  On
// exit SS.pool[g][0..S.npool[g]) holds the unique candidate keys eligible for
// the final top-k (sentinel: top-k of every level; else: top-k of the floor).
template <int NT>
__device__ void tree_search(SearchSmem& S, const ForestView& F, const SearchScratch& SS, int t,
                            const SearchParams& P, double* dirs_tmp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = P.G;
  const int L = F.meta[t].levels;
  const bool collect_all = P.target < 0;
  const int floor = collect_all ? 1 : min(P.target, L);
  const unsigned allmask = (1u << G) - 1u;
  const int* mem = F.mem(t);
  if (tid < G) { S.npool[tid] = 0; S.nsurv[tid] = 0; }
  if (tid == 0) atomicAdd(&F.meta[t].query_count, (unsigned long long)G);
  __syncthreads();
  float4 qv[ICB_MAX_G];
  for (int g = 0; g < G; ++g) qv[g] = reinterpret_cast<const float4*>(S.q[g])[lane];

  for (int lv = L; lv >= floor; --lv) {
    // (1) union of the nodes requested by the heads' survivors
    if (lv == L) {
      if (tid == 0) { SS.ulist[0] = F.meta[t].top_node; SS.umask[0] = (int)allmask; S.U = 1; }
      __syncthreads();
    } else {
      if (tid == 0) S.U = 0;
      __syncthreads();
      for (int g = 0; g < G; ++g) {
        const int ns = S.nsurv[g];
        const int* sv = SS.surv + (size_t)g * SS.ccap;
        for (int i = tid; i < ns; i += NT) {
          int node = F.own(t, sv[i], lv);
          unsigned old = atomicOr(SS.nmask + node, 1u << g);
          if (old == 0) SS.ulist[atomicAdd(&S.U, 1)] = node;
        }
      }
      __syncthreads();
      for (int i = tid; i < S.U; i += NT) SS.umask[i] = (int)SS.nmask[SS.ulist[i]];
      __syncthreads();
    }
    const int U = S.U;
    // (2) per-head offsets over the union (normal nodes only)
    if (tid < G) S.scan_carry[tid] = 0;
    if (tid == 0) S.nbig = 0;
    __syncthreads();
    for (int base = 0; base < U; base += NT) {
      int i = base + tid;
      int node = i < U ? SS.ulist[i] : 0;
      int sz = i < U ? F.node_size[F.nd(t, node)] : 0;
      bool big = sz > ICB_EXHAUSTIVE && (long long)sz > P.visit_cap;
      unsigned mk = i < U ? (unsigned)SS.umask[i] : 0u;
      if (i < U && big) atomicAdd(&S.nbig, 1);
      for (int g = 0; g < G; ++g) {
        int v = (i < U && !big && ((mk >> g) & 1)) ? sz : 0;
        int tot;
        int ex = block_exclusive_scan<NT>(v, S.wsum, tot);
        if (i < U) SS.uoff[(size_t)g * F.node_cap + i] = S.scan_carry[g] + ex;
        __syncthreads();
        if (tid == 0) S.scan_carry[g] += tot;
        __syncthreads();
      }
    }
    if (tid < G) S.M[tid] = S.scan_carry[tid];
    __syncthreads();
    for (int g = 0; g < G; ++g)
      if (S.M[g] > SS.ccap) { if (tid == 0) set_err(F.meta + t, ICB_ERR_CAP_SCRATCH); return; }
    // (3) evaluate normal nodes: one warp per node, 4 rows in flight
    if (tid == 0) S.misc[5] = 0;
    __syncthreads();
    for (int i = warp; i < U; i += NT / 32) {
      const int node = SS.ulist[i];
      const unsigned mk = (unsigned)SS.umask[i];
      const size_t x = F.nd(t, node);
      const int sz = F.node_size[x];
      if (sz > ICB_EXHAUSTIVE && (long long)sz > P.visit_cap) continue;
      if (lane == 0) atomicAdd(&S.misc[5], sz);
      const int off = F.node_off[x];
      int ob[ICB_MAX_G];
      for (int g = 0; g < G; ++g) ob[g] = SS.uoff[(size_t)g * F.node_cap + i];
      for (int j0 = 0; j0 < sz; j0 += 4) {
        int myid = (lane < 4 && j0 + lane < sz) ? mem[off + j0 + lane] : 0;
        float mytail = (lane < 4 && j0 + lane < sz) ? F.tail[F.tk(t, myid)] : 0.f;
        int ids[4];
        float tl[4];
        float4 rows[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ids[u] = __shfl_sync(0xffffffffu, myid, u);
          tl[u] = __shfl_sync(0xffffffffu, mytail, u);
          if (j0 + u < sz) rows[u] = __ldg(reinterpret_cast<const float4*>(F.row(t, ids[u])) + lane);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (j0 + u >= sz) break;
          for (int g = 0; g < G; ++g) {
            if (!((mk >> g) & 1)) continue;
            float s = warp_sum_butterfly(lane_sq4(rows[u], qv[g]));
            float d2 = d2_finish(s, tl[u], S.qt[g]);
            if (lane == 0) SS.cand[(size_t)g * SS.ccap + ob[g] + j0 + u] = make_key(d2, ids[u]);
          }
        }
      }
    }
    __syncthreads();
    // (4) P-DCI truncated nodes (rare): block-wide, per node and head
    if (S.nbig > 0) {
      for (int i = 0; i < U; ++i) {
        const int node = SS.ulist[i];
        const int sz = F.node_size[F.nd(t, node)];
        if (!(sz > ICB_EXHAUSTIVE && (long long)sz > P.visit_cap)) continue;
        const unsigned mk = (unsigned)SS.umask[i];
        for (int g = 0; g < G; ++g) {
          if (!((mk >> g) & 1)) continue;
          int cnt = pdci_visit<NT>(S, F, SS, t, node, g, P.visit_cap, dirs_tmp);
          if (S.M[g] + cnt > SS.ccap) { if (tid == 0) set_err(F.meta + t, ICB_ERR_CAP_SCRATCH); return; }
          eval_list_one_head<NT>(S, F, t, SS.vis, cnt, g, SS.cand + (size_t)g * SS.ccap + S.M[g]);
          __syncthreads();
          if (tid == 0) { S.M[g] += cnt; S.misc[5] += cnt; }
          __syncthreads();
        }
      }
    }
    // (5) counters; (6) clear union marks
    if (tid == 0) {
      unsigned long long ev = 0;
      for (int g = 0; g < G; ++g) ev += S.M[g];
      atomicAdd(&F.meta[t].distance_evals, ev);
      atomicAdd(&F.meta[t].rows_read, (unsigned long long)S.misc[5]);
      if (lv < L) atomicAdd(&F.meta[t].owner_rereads, (unsigned long long)U);
    }
    if (lv < L)
      for (int i = tid; i < U; i += NT) SS.nmask[SS.ulist[i]] = 0u;
    __syncthreads();
    // (7) per-head selection
    for (int g = 0; g < G; ++g) {
      unsigned long long* cg = SS.cand + (size_t)g * SS.ccap;
      unsigned long long* pg = SS.pool + (size_t)g * SS.ccap;
      unsigned* sg = SS.seen + (size_t)g * (F.tok_cap / 32 + 1);
      const int M = S.M[g];
      if (lv > floor) {
        int ns = block_select<NT>(S, cg, M, P.beam, nullptr, SS.surv + (size_t)g * SS.ccap, 0, nullptr);
        if (tid == 0) S.nsurv[g] = ns;
        __syncthreads();
        if (collect_all) {
          // top-k of this level = top-k of its survivors (beam >= k)
          // survivors' keys: re-select from candidates with B = k
          int np = block_select<NT>(S, cg, M, P.k, pg, nullptr, S.npool[g], sg);
          if (tid == 0) S.npool[g] += np;
          __syncthreads();
        }
      } else {
        int np = block_select<NT>(S, cg, M, P.k, pg, nullptr, S.npool[g], sg);
        if (tid == 0) S.npool[g] += np;
        __syncthreads();
      }
    }
    (void)warp;
  }
}

// Final ranked top-k of head g from its pool into S.sortbuf[0..n) (sorted).
// Clears the head's seen marks.  Returns n.
template <int NT>
__device__ int finalize_head(SearchSmem& S, const ForestView& F, const SearchScratch& SS, int g, long long k) {
  unsigned long long* pg = SS.pool + (size_t)g * SS.ccap;
  unsigned* sg = SS.seen + (size_t)g * (F.tok_cap / 32 + 1);
  const int np = S.npool[g];
  // clear seen marks of pooled ids
  for (int i = threadIdx.x; i < np; i += NT) {
    int id = key_id(pg[i]);
    atomicAnd(sg + (id >> 5), ~(1u << (id & 31)));
  }
  __syncthreads();
  int n = (int)min((long long)np, k);
  if (n > kSortMax) n = kSortMax;
  // select top-n of the pool (unique ids) into the sort buffer, then sort
  int got = block_select<NT>(S, pg, np, n, S.sortbuf, nullptr, 0, nullptr);
  block_sort<NT>(S, got);
  return got;
}

}  // namespace icb
