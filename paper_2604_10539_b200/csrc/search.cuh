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

#ifndef ICB_SEARCH_THREADS
#define ICB_SEARCH_THREADS 256
#endif
constexpr int kSearchThreads = ICB_SEARCH_THREADS;   // 256: two CTAs (trees) per SM
constexpr int kSortMax = 4096;   // largest k served by the in-smem final sort

struct SearchScratch {
  unsigned long long* cand;   // [G][ccap]
  unsigned long long* pool;   // [G][ccap]
  unsigned long long* surv;   // [G][ccap] survivor keys
  int* ulist;                 // [node_cap]
  int* umask;                 // [node_cap]
  int* uoff;                  // [G][node_cap]
  unsigned* nmask;            // [node_cap]   zero between levels
  unsigned* seen;             // [G][tok_cap/32+1] zero between queries
  int* vis;                   // [tok_cap]  P-DCI visit list
  double* proj;               // [tok_cap][8] P-DCI projections
  unsigned long long* ekey;   // [tok_cap][2] P-DCI emission keys
  int* upre;                  // [node_cap] union prefix of streamed rows
  int* umoff;                 // [node_cap] member offset of each union node (-1: P-DCI node)
  int* rlist;                 // [tok_cap][2] (token, union index) rows of a level
  int ccap;
};

// Per-CTA scratch slot carved from one buffer (same layout for queries and
// inserts; G = heads per tree of the call).
struct SlotLayout {
  size_t cand, pool, surv, ulist, umask, uoff, nmask, seen, vis, proj, ekey, upre, umoff, rlist, pbits, dirs, total;
};

__host__ __device__ inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline SlotLayout slot_layout(int G, int tok_cap, int node_cap, int page_cap, int dim) {
  SlotLayout L{};
  size_t o = 0;
  size_t cc = (size_t)tok_cap;
  L.cand = o; o = al256(o + (size_t)G * cc * 8);
  L.pool = o; o = al256(o + (size_t)G * cc * 8);
  L.surv = o; o = al256(o + (size_t)G * cc * 8);
  L.ulist = o; o = al256(o + (size_t)node_cap * 4);
  L.umask = o; o = al256(o + (size_t)node_cap * 4);
  L.uoff = o; o = al256(o + (size_t)G * node_cap * 4);
  L.nmask = o; o = al256(o + (size_t)node_cap * 4);
  L.seen = o; o = al256(o + (size_t)G * (tok_cap / 32 + 1) * 4);
  L.vis = o; o = al256(o + cc * 4);
  L.proj = o; o = al256(o + cc * ICB_NPROJ * 8);
  L.ekey = o; o = al256(o + cc * 16);
  L.upre = o; o = al256(o + (size_t)node_cap * 4);
  L.umoff = o; o = al256(o + (size_t)node_cap * 4);
  L.rlist = o; o = al256(o + cc * 8);
  L.pbits = o; o = al256(o + (size_t)(page_cap / 32 + 1) * 4);
  L.dirs = o; o = al256(o + (size_t)ICB_NPROJ * (dim + 1) * 8);
  L.total = o;
  return L;
}

__device__ inline SearchScratch slot_scratch(char* base, const SlotLayout& L, int tok_cap, double** dirs,
                                             unsigned** pbits) {
  SearchScratch S;
  S.cand = (unsigned long long*)(base + L.cand);
  S.pool = (unsigned long long*)(base + L.pool);
  S.surv = (unsigned long long*)(base + L.surv);
  S.ulist = (int*)(base + L.ulist);
  S.umask = (int*)(base + L.umask);
  S.uoff = (int*)(base + L.uoff);
  S.nmask = (unsigned*)(base + L.nmask);
  S.seen = (unsigned*)(base + L.seen);
  S.vis = (int*)(base + L.vis);
  S.proj = (double*)(base + L.proj);
  S.ekey = (unsigned long long*)(base + L.ekey);
  S.upre = (int*)(base + L.upre);
  S.umoff = (int*)(base + L.umoff);
  S.rlist = (int*)(base + L.rlist);
  S.ccap = tok_cap;
  *pbits = (unsigned*)(base + L.pbits);
  *dirs = (double*)(base + L.dirs);
  return S;
}

struct __align__(16) SearchSmem {   // q rows are read as float4
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
  int scan_carry[ICB_MAX_G + 1];
  int wsum2[(ICB_MAX_G + 1) * (kSearchThreads / 32)];
  int misc[8];
  int nopool;   // the final top-k is the floor level's top-k (no cross-level pool)
  int oskip;    // owners are not re-read: their keys are the survivors' (no P-DCI node can occur)
  unsigned long long* sortbuf;   // fallback sort buffer (aliases the idle row ring, >= kSortMax keys)
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

// ------------------------------------------------------------------ per-head groups
// With G heads the CTA splits into G warp groups (NT / GP threads each) that
// run the selections of their head concurrently, synchronizing on named
// barrier 1 + group.
constexpr int kBins = 1024;
constexpr int kBuf = 512;
// The row stream uses cp.async rings (a TMA bulk-copy ring measured slower for
// 512-B rows and was removed).
constexpr int kSub = 16;                             // ring slots per warp (2 batches of 8 rows)
constexpr int kRing = (kSearchThreads / 32) * kSub;  // 128 slots x 512 B = 64 KB (+ 2 mbarriers each)

struct GroupSmem {
  int hist[kBins];
  unsigned long long buf[kBuf];
  int wsum[32];
  int misc[8];
  unsigned lo, hi;          // d2-bit range of the head's current candidate list
  unsigned plo, phi;        // d2-bit range of the head's pool
};

// Dynamic shared memory: [GroupSmem x GP][ring kRing x 528 B][full][empty][q]
struct RingView {
  float* ring;
  unsigned long long* full;
  unsigned long long* empty;
  unsigned* qp;     // per consumer warp: running row count (slot = c*kSub + q % kSub, phase = q / kSub)
};

__host__ __device__ inline size_t search_dsm_bytes(int GP) {
  return sizeof(GroupSmem) * GP + (size_t)kRing * ICB_ROWF * 4 + 2 * kRing * 8 + 4 * 32;
}

__device__ inline RingView ring_view(unsigned char* dsm, int GP) {
  RingView R;
  unsigned char* p = dsm + sizeof(GroupSmem) * GP;
  R.ring = reinterpret_cast<float*>(p);
  p += (size_t)kRing * ICB_ROWF * 4;
  R.full = reinterpret_cast<unsigned long long*>(p);
  R.empty = R.full + kRing;
  R.qp = reinterpret_cast<unsigned*>(R.empty + kRing);
  return R;
}

__device__ inline void ring_init(const RingView& R) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(R.full + s, 1);
      mbar_init(R.empty + s, 1);
    }
    for (int c = 0; c < 32; ++c) R.qp[c] = 0;
    mbar_fence_init();
  }
  __syncthreads();
}

__device__ __forceinline__ void gsync(int bar, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(n) : "memory");
}

// exclusive scan of one int per thread within the group
template <int NTG>
__device__ __forceinline__ int group_scan(GroupSmem& GS, int gtid, int bar, int v, int& total) {
  const int lane = gtid & 31, w = gtid >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) GS.wsum[w] = x;
  gsync(bar, NTG);
  if (w == 0) {
    int s = lane < NTG / 32 ? GS.wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NTG / 32) GS.wsum[lane] = s;
  }
  gsync(bar, NTG);
  int before = (w > 0 ? GS.wsum[w - 1] : 0) + x - v;
  total = GS.wsum[NTG / 32 - 1];
  gsync(bar, NTG);
  return before;
}

// One pass over the list emitting every key <= thr: the keys to out_ids
// (from out_ids_base, no dedup) and/or the keys to out_keys (from
// out_keys_base, skipping ids already marked in `seen` and marking new ones;
// the emitted keys' d2 range is folded into plo/phi).  8 independent loads in
// flight per thread.  Returns (ids written, keys written).
template <int NTG>
__device__ int2 group_emit(GroupSmem& GS, int gtid, int bar, const unsigned long long* keys, int M,
                           unsigned long long thr, unsigned long long* out_ids, int out_ids_base,
                           unsigned long long* out_keys,
                           int out_keys_base, unsigned* seen, unsigned* plo, unsigned* phi) {
  constexpr int U = 8;
  const int lane = gtid & 31;
  if (gtid == 0) { GS.misc[0] = 0; GS.misc[1] = 0; }
  gsync(bar, NTG);
  unsigned mn = 0xffffffffu, mx = 0u;
  const int Mpad = (M + U * NTG - 1) / (U * NTG) * (U * NTG);   // warp-uniform trip count
  for (int i0 = gtid; i0 < Mpad; i0 += U * NTG) {
    unsigned long long kk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * NTG;
      kk[u] = i < M ? keys[i] : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned long long k = kk[u];
      const bool sel = (i0 + u * NTG < M) && k <= thr;
      if (out_ids) {
        const unsigned bal = __ballot_sync(0xffffffffu, sel);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&GS.misc[0], __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (sel) out_ids[out_ids_base + base + __popc(bal & ((1u << lane) - 1))] = k;
      }
      if (out_keys) {
        bool take = sel;
        if (take && seen) {
          const int id = key_id(k);
          const unsigned bit = 1u << (id & 31);
          take = !(atomicOr(seen + (id >> 5), bit) & bit);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&GS.misc[1], __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take) {
          out_keys[out_keys_base + base + __popc(bal & ((1u << lane) - 1))] = k;
          const unsigned hb = (unsigned)(k >> 32);
          mn = min(mn, hb);
          mx = max(mx, hb);
        }
      }
    }
  }
  if (plo) {
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0 && mx >= mn) { atomicMin(plo, mn); atomicMax(phi, mx); }
  }
  gsync(bar, NTG);
  const int2 r = make_int2(GS.misc[0], GS.misc[1]);
  gsync(bar, NTG);
  return r;
}

// Exact threshold (the B-th smallest key) by 8-bit MSB radix passes over the
// list; used for lists whose boundary bin is too crowded for the fast path.
template <int NTG>
__device__ unsigned long long group_radix_threshold(GroupSmem& GS, int gtid, int bar, const unsigned long long* keys,
                                                    int M, long long B) {
  const int lane = gtid & 31, w = gtid >> 5;
  unsigned long long prefix = 0, pmask = 0;
  long long remaining = B;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = gtid; i < 256; i += NTG) GS.hist[i] = 0;
    gsync(bar, NTG);
    for (int i = gtid; i < M + (NTG - (M % NTG)) % NTG; i += NTG) {
      bool valid = i < M;
      unsigned long long k = valid ? keys[i] : 0;
      valid = valid && ((k & pmask) == prefix);
      int dig = (int)((k >> shift) & 0xff);
      unsigned act = __ballot_sync(0xffffffffu, valid);
      if (valid) {
        unsigned peers = __match_any_sync(act, dig);
        if ((__ffs(peers) - 1) == lane) atomicAdd(&GS.hist[dig], __popc(peers));
      }
    }
    gsync(bar, NTG);
    if (w == 0) {
      int c[8], local = 0;
      for (int u = 0; u < 8; ++u) { c[u] = GS.hist[lane * 8 + u]; local += c[u]; }
      int incl = local;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int excl = incl - local;
      bool mine = (excl < remaining) && (incl >= remaining);
      unsigned who = __ballot_sync(0xffffffffu, mine);
      int src = __ffs(who) - 1;
      int digit = 0, before = 0, inb = 0;
      if (lane == src) {
        int run = excl;
        for (int u = 0; u < 8; ++u) {
          if (run + c[u] >= remaining) { digit = lane * 8 + u; before = run; inb = c[u]; break; }
          run += c[u];
        }
      }
      if (lane == src) { GS.misc[1] = digit; GS.misc[2] = before; GS.misc[3] = inb; }
    }
    gsync(bar, NTG);
    int digit = GS.misc[1], before = GS.misc[2], inb = GS.misc[3];
    gsync(bar, NTG);
    remaining -= before;
    prefix |= (unsigned long long)digit << shift;
    pmask |= 0xffull << shift;
    if (inb == remaining || shift == 0) return prefix | ~pmask;
  }
  return ~0ull;
}

// bitonic sort of n keys in the smem buffer `buf` (capacity >= the next power
// of two), ascending, group-wide
template <int NTG>
__device__ void group_sort_buf(unsigned long long* buf, int gtid, int bar, int n) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = n + gtid; i < P; i += NTG) buf[i] = ~0ull;
  gsync(bar, NTG);
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = gtid; i < P; i += NTG) {
        int ixj = i ^ j;
        if (ixj > i) {
          unsigned long long a = buf[i], b = buf[ixj];
          bool upw = (i & k) == 0;
          if ((a > b) == upw) { buf[i] = b; buf[ixj] = a; }
        }
      }
      gsync(bar, NTG);
    }
  }
}
template <int NTG>
__device__ void group_sort(GroupSmem& GS, int gtid, int bar, int n) {
  group_sort_buf<NTG>(GS.buf, gtid, bar, n);
}

// Threshold of the B smallest of M unique keys (d2 bits of every key within
// [lo, hi]): the B-th smallest key, so `key <= thr` selects exactly B.  One
// adaptive histogram pass over kBins bins spanning [lo, hi] finds the
// boundary bin, which is resolved exactly (bitonic sort in smem, or radix
// passes if crowded).
template <int NTG>
__device__ unsigned long long group_threshold(GroupSmem& GS, int gtid, int bar, const unsigned long long* keys, int M,
                                              long long B, unsigned lo, unsigned hi) {
  if (B >= M) return ~0ull;
  const unsigned range = hi - lo;
  const int nbits = range ? 32 - __clz(range) : 0;
  constexpr int kBinBits = 10;   // kBins = 1 << kBinBits
  static_assert((1 << kBinBits) == kBins, "bin count");
  const int shift = nbits > kBinBits ? nbits - kBinBits : 0;
  for (int i = gtid; i < kBins; i += NTG) GS.hist[i] = 0;
  gsync(bar, NTG);
  for (int i0 = gtid; i0 < M; i0 += 8 * NTG) {   // 8 independent loads in flight per thread
    unsigned hbs[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * NTG;
      hbs[u] = i < M ? (unsigned)(keys[i] >> 32) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u * NTG >= M) break;
      const unsigned hb = hbs[u];
      ICB_CHECK(hb >= lo && hb <= hi && ((hb - lo) >> shift) < kBins, "hb %u lo %u hi %u shift %d M %d", hb, lo,
                hi, shift, M);
      atomicAdd(&GS.hist[(hb - lo) >> shift], 1);
    }
  }
  gsync(bar, NTG);
  // locate the boundary bin: each thread owns kBins / NTG consecutive bins
  constexpr int PER = kBins / NTG;
  int c[PER], local = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) { c[u] = GS.hist[gtid * PER + u]; local += c[u]; }
  int tot;
  int excl = group_scan<NTG>(GS, gtid, bar, local, tot);
  if (excl < B && excl + local >= B) {
    int run = excl;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      if (run + c[u] >= B) { GS.misc[4] = gtid * PER + u; GS.misc[5] = run; GS.misc[6] = c[u]; break; }
      run += c[u];
    }
  }
  gsync(bar, NTG);
  const int bstar = GS.misc[4], below = GS.misc[5], nb = GS.misc[6];
  const long long need = B - below;
  unsigned long long thr;
  if (nb <= kBuf) {
    // gather the boundary bin and sort it
    if (gtid == 0) GS.misc[7] = 0;
    gsync(bar, NTG);
    for (int i0 = gtid; i0 < M; i0 += 8 * NTG) {
      unsigned long long kk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * NTG;
        kk[u] = i < M ? keys[i] : ~0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned long long k = kk[u];
        if (i0 + u * NTG < M && (int)(((unsigned)(k >> 32) - lo) >> shift) == bstar) {
          const int at = atomicAdd(&GS.misc[7], 1);
          ICB_CHECK(at < nb, "boundary gather %d >= %d", at, nb);
          GS.buf[at] = k;
        }
      }
    }
    gsync(bar, NTG);
    group_sort<NTG>(GS, gtid, bar, nb);
    thr = GS.buf[need - 1];
    gsync(bar, NTG);
  } else {
    thr = group_radix_threshold<NTG>(GS, gtid, bar, keys, M, B);
  }
  return thr;
}

// Top-B of M unique keys (d2 bits within [lo, hi]) written UNORDERED to `out`
// (global or smem) in two passes over the list instead of three: a
// kTopBins-bin histogram over [lo, hi] in the head group's slice of the idle
// row ring, then one pass that emits every key of a bin below the boundary
// bin and gathers the boundary bin into smem; its sorted head completes the
// B.  16 loads in flight per thread.  A crowded boundary bin falls back to the
// radix threshold.  Returns min(M, B).
// selection statistics (per translation unit; the query kernel's are
// reported by icb_search_profile): selections, radix fallbacks, boundary sizes
static __device__ unsigned long long g_topb_stats[8];
// ICB_PROF: level iterations, union nodes, rows, row-list passes, binary-search passes, start levels
static __device__ unsigned long long g_scan_stats[16];
#define ICB_SUB(k)                                                              \
  do {                                                                          \
    if (P.prof && threadIdx.x == 0) {                                           \
      long long n_ = clock64();                                                 \
      atomicAdd(&g_scan_stats[k], (unsigned long long)(n_ - tsub_));            \
      tsub_ = n_;                                                               \
    }                                                                           \
  } while (0)

template <int GP>
struct TopB {
  static constexpr int kBins = GP <= 4 ? 2048 : 1024;
  static constexpr int kBufN = 512;
  static constexpr size_t kBytes = (size_t)kBins * 4 + (size_t)kBufN * 8;   // per head group
};

template <int NTG, int GP>
__device__ int group_topb(GroupSmem& GS, unsigned char* rg, int gtid, int bar, const unsigned long long* keys,
                          int M, long long B, unsigned lo, unsigned hi, unsigned long long* out, bool prof) {
  static_assert(TopB<GP>::kBytes * GP <= (size_t)kRing * ICB_ROWF * 4, "top-B scratch exceeds the row ring");
  constexpr int U = 16;
  constexpr int NB = TopB<GP>::kBins;
  constexpr int NBB = 31 - __builtin_clz(NB);
  const int lane = gtid & 31;
  int* hist = reinterpret_cast<int*>(rg);
  unsigned long long* bb = reinterpret_cast<unsigned long long*>(rg + (size_t)NB * 4);
  const int Mpad = (M + U * NTG - 1) / (U * NTG) * (U * NTG);   // group-uniform trip counts
  if (B >= M) {
    for (int i0 = gtid; i0 < Mpad; i0 += U * NTG) {
      unsigned long long kk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) kk[u] = i0 + u * NTG < M ? keys[i0 + u * NTG] : 0ull;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * NTG < M) out[i0 + u * NTG] = kk[u];
    }
    gsync(bar, NTG);
    return M;
  }
  long long tq0 = clock64();
  const unsigned range = hi - lo;
  const int nbits = range ? 32 - __clz(range) : 0;
  const int shift = nbits > NBB ? nbits - NBB : 0;
  for (int i = gtid; i < NB; i += NTG) hist[i] = 0;
  gsync(bar, NTG);
  // histogram pass: only the keys' high (d2) words, 2U loads in flight
  const unsigned* khi = reinterpret_cast<const unsigned*>(keys) + 1;
  constexpr int U2 = 2 * U;
  const int Mpad2 = (M + U2 * NTG - 1) / (U2 * NTG) * (U2 * NTG);
  for (int i0 = gtid; i0 < Mpad2; i0 += U2 * NTG) {
    unsigned hb[U2];
#pragma unroll
    for (int u = 0; u < U2; ++u) hb[u] = i0 + u * NTG < M ? khi[2 * (size_t)(i0 + u * NTG)] : 0u;
#pragma unroll
    for (int u = 0; u < U2; ++u)
      if (i0 + u * NTG < M) {
        ICB_CHECK(hb[u] >= lo && hb[u] <= hi, "hb %u outside [%u, %u]", hb[u], lo, hi);
        atomicAdd(&hist[(hb[u] - lo) >> shift], 1);
      }
  }
  long long tq1 = clock64();
  gsync(bar, NTG);
  // boundary bin: each thread owns NB / NTG consecutive bins
  constexpr int PER = NB / NTG;
  int local = 0;
#pragma unroll 8
  for (int u = 0; u < PER; ++u) local += hist[gtid * PER + u];
  int tot;
  const int excl = group_scan<NTG>(GS, gtid, bar, local, tot);
  if (excl < B && excl + local >= B) {
    int run = excl;
    for (int u = 0; u < PER; ++u) {
      const int c = hist[gtid * PER + u];
      if (run + c >= B) { GS.misc[4] = gtid * PER + u; GS.misc[5] = run; GS.misc[6] = c; break; }
      run += c;
    }
  }
  if (gtid == 0) { GS.misc[0] = 0; GS.misc[7] = 0; }
  gsync(bar, NTG);
  const int bstar = GS.misc[4], below = GS.misc[5], nb = GS.misc[6];
  if (prof && gtid == 0) { atomicAdd(&g_topb_stats[0], 1ull); atomicAdd(&g_topb_stats[2], (unsigned long long)nb); }
  if (nb > TopB<GP>::kBufN) {
    if (prof && gtid == 0) atomicAdd(&g_topb_stats[1], 1ull);
    const unsigned long long thr = group_radix_threshold<NTG>(GS, gtid, bar, keys, M, B);
    group_emit<NTG>(GS, gtid, bar, keys, M, thr, nullptr, 0, out, 0, nullptr, nullptr, nullptr);
    return (int)B;
  }
  long long tq2 = clock64();
  for (int i0 = gtid; i0 < Mpad; i0 += U * NTG) {
    unsigned long long kk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) kk[u] = i0 + u * NTG < M ? keys[i0 + u * NTG] : ~0ull;
    // classify all U keys, then ONE warp scan + ONE atomic place this
    // thread's low keys contiguously
    unsigned lowm = 0u;
    int nlow = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool valid = i0 + u * NTG < M;
      const int bin = (int)(((unsigned)(kk[u] >> 32) - lo) >> shift);
      const bool low = valid && bin < bstar;
      lowm |= low ? (1u << u) : 0u;
      nlow += low ? 1 : 0;
      if (valid && bin == bstar) bb[atomicAdd(&GS.misc[7], 1)] = kk[u];
    }
    int incl = nlow;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int at = 0;
    if (lane == 31 && incl) at = atomicAdd(&GS.misc[0], incl);
    at = __shfl_sync(0xffffffffu, at, 31) + incl - nlow;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((lowm >> u) & 1u) out[at++] = kk[u];
  }
  gsync(bar, NTG);
  long long tq3 = clock64();
  group_sort_buf<NTG>(bb, gtid, bar, nb);
  const int need = (int)(B - below);
  for (int i = gtid; i < need; i += NTG) out[below + i] = bb[i];
  gsync(bar, NTG);
  if (prof && gtid == 0) {
    long long tq4 = clock64();
    atomicAdd(&g_topb_stats[3], (unsigned long long)(tq1 - tq0));
    atomicAdd(&g_topb_stats[4], (unsigned long long)(tq2 - tq1));
    atomicAdd(&g_topb_stats[5], (unsigned long long)(tq3 - tq2));
    atomicAdd(&g_topb_stats[6], (unsigned long long)(tq4 - tq3));
  }
  return (int)B;
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

// Block bitonic sort of n (a power of two) entries ascending by (k64, k32),
// the payload `pl` travelling along; shared-memory arrays.
template <int NT>
__device__ void bitonic3(unsigned long long* k64, unsigned* k32, int* pl, int n) {
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += NT) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const unsigned long long a = k64[lo], b = k64[hi];
        const unsigned a2 = k32[lo], b2 = k32[hi];
        const bool gt = a > b || (a == b && a2 > b2);
        if (gt == ((lo & size) == 0)) {
          k64[lo] = b; k64[hi] = a;
          k32[lo] = b2; k32[hi] = a2;
          const int t = pl[lo]; pl[lo] = pl[hi]; pl[hi] = t;
        }
      }
      __syncthreads();
    }
}

__device__ __forceinline__ unsigned long long orderable_f64(double x) {
  if (x == 0.0) x = 0.0;   // -0 == +0 (ties then break by id, as the numeric comparison does)
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Visit list of a large node (cap entries, ascending emission order) into
// SS.vis; returns the count.  Emission key of a member = lexicographic max over
// its 8 ladder entries of (gap, j, chain position) -- the pop order of the
// reference's heap merge (see oracle/dci.py:visit_order for the equivalence).
// The chain position of member i on ladder j is its rank in the node sorted by
// (projection_j, id), and the ladder's start is the number of projections
// below the query's.  Everything but the query's projections and gaps is
// query independent: nodes of up to kPdciSort members keep their projections
// and ladder ranks in the tree's P-DCI cache (built here with one bitonic sort
// per ladder in the idle row ring, S.sortbuf, 64 KB; rebuilt when the node
// has grown), and a visit is then O(8m) plus one sort of the emission keys.
// Nodes the cache cannot hold rank by counting (O(m^2)).
constexpr int kPdciSort = 4096;

// Orderable bits of a fp64 projection.
__device__ __forceinline__ unsigned long long proj_key(double x) { return orderable_f64(x); }

// Make (or confirm) node's cache entries; returns their offset or -1.
template <int NT>
__device__ int pc_ensure(SearchSmem& S, const ForestView& F, int t, int node, int m, const int* mem,
                         const double* dirs) {
  __shared__ int s_off;
  const size_t x = F.nd(t, node);
  if (F.node_pcm[x] == m && F.node_pc[x] >= 0) return F.node_pc[x];
  if (m > kPdciSort) return -1;
  if (threadIdx.x == 0) {
    int off = F.node_pc[x];
    if (off < 0 || F.node_pccap[x] < m) {
      const int want = max(m + (m >> 1), 128);
      TreeMeta* mt = F.meta + t;
      // bump allocation that never overshoots the arena (several CTAs may warm
      // one tree's nodes concurrently, pdci_warm_kernel)
      int cur = *(volatile int*)&mt->pc_top;
      off = -1;
      while (cur + want <= F.pc_cap) {
        const int prev = atomicCAS(&mt->pc_top, cur, cur + want);
        if (prev == cur) { off = cur; break; }
        cur = prev;
      }
      if (off >= 0) { F.node_pc[x] = off; F.node_pccap[x] = want; }
    }
    s_off = off;
  }
  __syncthreads();
  const int off = s_off;
  if (off < 0) return -1;
  const int D1 = F.dim + 1;
  double* proj = F.pc_proj + ((size_t)t * F.pc_cap + off) * ICB_NPROJ;
  int* ord = F.pc_ord + ((size_t)t * F.pc_cap + off) * ICB_NPROJ;
  int* pos = F.pc_pos + ((size_t)t * F.pc_cap + off) * ICB_NPROJ;
  for (int xx = threadIdx.x; xx < m * ICB_NPROJ; xx += NT) {
    const int i = xx / ICB_NPROJ, j = xx % ICB_NPROJ;
    const float* row = F.row(t, mem[i]);
    double acc = 0.0;
    for (int u = 0; u < F.dim; ++u) acc = __fma_rn(dirs[j * D1 + u], (double)row[u], acc);
    acc = __fma_rn(dirs[j * D1 + F.dim], (double)F.tail[F.tk(t, mem[i])], acc);
    proj[(size_t)i * ICB_NPROJ + j] = acc;
  }
  __syncthreads();
  int n2 = 1;
  while (n2 < m) n2 <<= 1;
  unsigned long long* k64 = S.sortbuf;                            // [n2]
  unsigned* k32 = reinterpret_cast<unsigned*>(k64 + n2);          // [n2]
  int* pl = reinterpret_cast<int*>(k32 + n2);                     // [n2]
  for (int j = 0; j < ICB_NPROJ; ++j) {
    for (int i = threadIdx.x; i < n2; i += NT) {
      const bool on = i < m;
      k64[i] = on ? proj_key(proj[(size_t)i * ICB_NPROJ + j]) : ~0ull;
      k32[i] = on ? (unsigned)mem[i] : 0xffffffffu;
      pl[i] = on ? i : -1;
    }
    __syncthreads();
    bitonic3<NT>(k64, k32, pl, n2);
    for (int r = threadIdx.x; r < m; r += NT) {
      ord[(size_t)r * ICB_NPROJ + j] = pl[r];
      pos[(size_t)pl[r] * ICB_NPROJ + j] = r;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) F.node_pcm[x] = m;
  __syncthreads();
  return off;
}

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
  __syncthreads();
  const int cnt = (int)min((long long)m, cap);
  const int pco = pc_ensure<NT>(S, F, t, node, m, mem, dirs);
  if (pco >= 0) {
    const double* proj = F.pc_proj + ((size_t)t * F.pc_cap + pco) * ICB_NPROJ;
    const int* ord = F.pc_ord + ((size_t)t * F.pc_cap + pco) * ICB_NPROJ;
    const int* pos = F.pc_pos + ((size_t)t * F.pc_cap + pco) * ICB_NPROJ;
    __shared__ int s_start[ICB_NPROJ];
    if (threadIdx.x < ICB_NPROJ) {   // ladder start: projections strictly below the query's
      const int j = threadIdx.x;
      const double qp = S.dirs_tmp[j];
      int lo = 0, hi = m;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (proj[(size_t)ord[(size_t)mid * ICB_NPROJ + j] * ICB_NPROJ + j] < qp) lo = mid + 1;
        else hi = mid;
      }
      s_start[j] = lo;
    }
    __syncthreads();
    int n2 = 1;
    while (n2 < m) n2 <<= 1;
    unsigned long long* k64 = S.sortbuf;
    unsigned* k32 = reinterpret_cast<unsigned*>(k64 + n2);
    int* pl = reinterpret_cast<int*>(k32 + n2);
    for (int i = threadIdx.x; i < n2; i += NT) {
      unsigned long long bh = ~0ull, bl = 0xffffffffull;
      if (i < m) {
        bh = 0; bl = 0;
        for (int j = 0; j < ICB_NPROJ; ++j) {
          const int p = pos[(size_t)i * ICB_NPROJ + j], st = s_start[j];
          const double gap = fabs(__dsub_rn(proj[(size_t)i * ICB_NPROJ + j], S.dirs_tmp[j]));
          const unsigned long long h = (unsigned long long)__double_as_longlong(gap);
          const unsigned long long sec = p < st ? (unsigned long long)((1 << 23) - 1 - p)
                                                : (unsigned long long)((1 << 23) + p);
          const unsigned long long l = ((unsigned long long)j << 24) | sec;
          if (h > bh || (h == bh && l > bl)) { bh = h; bl = l; }
        }
      }
      k64[i] = bh;
      k32[i] = (unsigned)bl;
      pl[i] = i < m ? mem[i] : -1;
    }
    __syncthreads();
    bitonic3<NT>(k64, k32, pl, n2);
    for (int r = threadIdx.x; r < cnt; r += NT) SS.vis[r] = pl[r];
    __syncthreads();
    return cnt;
  }
  // uncached: member projections, then ranks by counting
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
  unsigned long long* prof;   // optional per-phase cycle counters (kPhases), thread 0 of each CTA adds
};

constexpr int kPhases = 9;   // + fused attention (search.cu)
#define ICB_MARK(k)                                       \
  do {                                                    \
    if (P.prof && threadIdx.x == 0) {                     \
      long long now_ = clock64();                         \
      atomicAdd(P.prof + (k), (unsigned long long)(now_ - tmark_)); \
      tmark_ = now_;                                      \
    }                                                     \
  } while (0)

// Evaluate the rows `ids[0..n)` against head g (single head; used by the
// P-DCI path) writing keys to dst.
template <int NT>
__device__ void eval_list_one_head(SearchSmem& S, const ForestView& F, int t, const int* ids, int n, int g,
                                   unsigned long long* dst, unsigned* lo = nullptr, unsigned* hi = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4 qv = reinterpret_cast<const float4*>(S.q[g])[lane];
  for (int i = warp; i < n; i += NT / 32) {
    int id = ids[i];
    float4 p = reinterpret_cast<const float4*>(F.row(t, id))[lane];
    float s = warp_sum_butterfly(lane_sq4(p, qv));
    float d2 = d2_finish(s, F.tail[F.tk(t, id)], S.qt[g]);
    if (lane == 0) {
      dst[i] = make_key(d2, id);
      if (lo) { atomicMin(lo, __float_as_uint(d2)); atomicMax(hi, __float_as_uint(d2)); }
    }
  }
}

// The multi-level search.  On entry S.q/S.qt hold the lifted queries.  On
// exit SS.pool[g][0..S.npool[g]) holds the unique candidate keys eligible for
// the final top-k (sentinel: top-k of every level; else: top-k of the floor).
// Sum of each head's lane partials with the xor-butterfly pairing of
// warp_sum_butterfly, transposed across heads: at offset 16 the lower half of
// the warp keeps heads [0, G/2) and the upper half [G/2, G), at 8 the halves
// split again, ...; lane l ends with the full sum of head l / (32 / G).
// Every head's sum is the same pairing tree as the plain butterfly, so the
// result is bit-identical (IEEE addition is commutative).
template <int G>
__device__ __forceinline__ float reduce_heads(float (&v)[G], int lane) {
  if constexpr (G == 1) {
    return warp_sum_butterfly(v[0]);
  } else {
    constexpr int H2 = G / 2;
    float w[H2];
    const bool up = lane & 16;
#pragma unroll
    for (int i = 0; i < H2; ++i) {
      float send = up ? v[i] : v[i + H2];
      float keep = up ? v[i + H2] : v[i];
      w[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
    if constexpr (G == 2) {
      float s = w[0];
      s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 8));
      s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
      s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
      return __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    } else {
      constexpr int H4 = G / 4;
      float x[H4];
      const bool up8 = lane & 8;
#pragma unroll
      for (int i = 0; i < H4; ++i) {
        float send = up8 ? w[i] : w[i + H4];
        float keep = up8 ? w[i + H4] : w[i];
        x[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 8));
      }
      float s;
      if constexpr (G == 4) {
        s = x[0];
        s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
      } else {
        const bool up4 = lane & 4;
        float send = up4 ? x[0] : x[1];
        float keep = up4 ? x[1] : x[0];
        s = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 4));
      }
      s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
      return __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    }
  }
}

// GP: padded head count (power of two >= P.G) fixing register arrays.
// XP: the fully transposed G=4 stream reduction (register heavy; the insert
// kernel's small parent searches use the generic path).
template <int NT, int GP, bool XP = true>
__device__ void tree_search(SearchSmem& S, GroupSmem* GSA, const RingView& RG, const ForestView& F,
                            const SearchScratch& SS, int t,
                            const SearchParams& P, double* dirs_tmp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NTG = NT / GP;
  const int grp = tid / NTG, gtid = tid % NTG, gbar = 1 + grp;
  GroupSmem& GS = GSA[grp];
  const int G = P.G;
  const int L = F.meta[t].levels;
  const bool collect_all = P.target < 0;
  const int floor = collect_all ? 1 : min(P.target, L);
  const unsigned allmask = (1u << G) - 1u;
  const int* mem = F.mem(t);
  if (tid < G) { S.npool[tid] = 0; S.nsurv[tid] = 0; }
  if (tid == 0) atomicAdd(&F.meta[t].query_count, (unsigned long long)G);
  __syncthreads();
  float4 qv[GP];
#pragma unroll
  for (int g = 0; g < GP; ++g)
    qv[g] = g < G ? reinterpret_cast<const float4*>(S.q[g])[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  // head pairs packed for the f32x2 path: q2[h][i] = (q_{2h}[4l+i], q_{2h+1}[4l+i])
  unsigned long long q2[GP / 2 > 0 ? GP / 2 : 1][4];
#pragma unroll
  for (int h = 0; h < GP / 2; ++h) {
    q2[h][0] = pack_f2(qv[2 * h].x, qv[2 * h + 1].x);
    q2[h][1] = pack_f2(qv[2 * h].y, qv[2 * h + 1].y);
    q2[h][2] = pack_f2(qv[2 * h].z, qv[2 * h + 1].z);
    q2[h][3] = pack_f2(qv[2 * h].w, qv[2 * h + 1].w);
  }

  // (0) start level.  Every point of top level >= lv is a member of exactly
  //     one node at level lv, so while C(lv) = #points of top >= lv is <= beam
  //     (and no node is P-DCI-truncated) every candidate survives and the next
  //     level's candidates are again all points of top >= lv - 1.  The search
  //     therefore starts at the lowest such level with the candidate set {top
  //     >= start} read from the tree's upper-point list: same survivors, same
  //     pool (the skipped levels' candidates are a subset of the start
  //     level's), same distance_evals (the skipped C(lv) are counted).
  if (tid == 0) {
    const TreeMeta& mt = F.meta[t];
    int start = L;
    S.nopool = 0;
    S.oskip = 0;
    if (!mt.lv_ovf && L < ICB_LV_TRACK) {
      long long C = 0;
      for (int lv = L; lv >= max(floor, 2); --lv) {
        const int mxn = mt.lvl_maxnode[lv];
        if (mxn > ICB_EXHAUSTIVE && (long long)mxn > P.visit_cap) break;
        start = lv;
        C += mt.lvl_count[lv];
        if (C > P.beam) break;
      }
      // No pool needed when every pooled survivor that could rank in the final
      // top-k is also a floor candidate: a survivor x of level lv is a member
      // of its own node at lv - 1, which x itself requests, so x is evaluated
      // there unless that node is P-DCI-truncated; if x then fails to survive,
      // beam >= k better keys are pooled and x cannot rank.  Hence with
      // beam >= k and no truncated node at any level, pool top-k = floor
      // top-k.  (Targeted searches pool only the floor anyway.)
      int notrunc = 1;
      for (int lv = 1; lv <= L; ++lv) {
        const int mxn = mt.lvl_maxnode[lv];
        if (mxn > ICB_EXHAUSTIVE && (long long)mxn > P.visit_cap) notrunc = 0;
      }
      S.nopool = notrunc && P.beam >= P.k && P.k <= kBuf;
      S.oskip = notrunc;
      unsigned long long Cs = 0, skipped = 0;
      for (int lv = L; lv > start; --lv) { Cs += mt.lvl_count[lv]; skipped += Cs; }
      if (skipped) atomicAdd(&F.meta[t].distance_evals, skipped * (unsigned long long)G);
    }
    S.misc[7] = start;
    if (!collect_all) S.nopool = P.k <= kBuf;
  }
  __syncthreads();
  const int start = S.misc[7];
  const bool oskip = S.oskip;

  long long tmark_ = clock64();
  long long tsub_ = 0;
  // union marks: kMarkBits per node (one bit per head) in the row ring, which
  // is idle between the selection and the row list; global marks when the
  // forest's node capacity does not fit
  constexpr unsigned kMarkBits = GP <= 4 ? 4u : 8u;
  constexpr int kMarkPerWord = 32 / (int)kMarkBits;
  constexpr unsigned kMarkMask = (1u << kMarkBits) - 1u;
  unsigned* rmark = reinterpret_cast<unsigned*>(RG.ring);
  const bool smark = (long long)F.node_cap <= (long long)kRing * ICB_ROWF * 4 / 4 * kMarkPerWord;
  for (int lv = start; lv >= floor; --lv) {
    ICB_MARK(0);
    if (P.prof && threadIdx.x == 0) tsub_ = clock64();
    // (1) union of the nodes requested by the heads' survivors
    if (lv == start) {
      if (tid == 0) { SS.ulist[0] = F.meta[t].top_node; SS.umask[0] = (int)allmask; S.U = 1; }
      __syncthreads();
    } else {
      if (tid == 0) S.U = 0;
      if (tid < GP) { GSA[tid].lo = 0xffffffffu; GSA[tid].hi = 0u; }
      if (smark)
        for (int i = tid; i < (F.node_cap + kMarkPerWord - 1) / kMarkPerWord; i += NT) rmark[i] = 0u;
      __syncthreads();
      // every (head, survivor) pair in parallel: independent own() lookups
      int pre[GP + 1];
      pre[0] = 0;
#pragma unroll
      for (int g = 0; g < GP; ++g) pre[g + 1] = pre[g] + (g < G ? S.nsurv[g] : 0);
      // 8 independent (survivor -> own base -> own node) chains per thread
      constexpr int UU = 8;
      const int* ownl = F.own_list + (size_t)t * F.own_cap;
      unsigned slo[GP], shi[GP];   // survivors' d2 range per head (this thread)
#pragma unroll
      for (int h = 0; h < GP; ++h) { slo[h] = 0xffffffffu; shi[h] = 0u; }
      for (int fb = 0; fb < pre[GP]; fb += NT * UU) {   // block-uniform trip count (ballots below)
        const int f0 = fb + tid;
        int gg[UU], x[UU];
#pragma unroll
        for (int u = 0; u < UU; ++u) {
          const int fl = f0 + u * NT;
          int g = 0;
#pragma unroll
          for (int h = 1; h < GP; ++h) g += fl >= pre[h] ? 1 : 0;
          gg[u] = fl < pre[GP] ? g : -1;
          x[u] = 0;
          if (gg[u] >= 0) {
            const unsigned long long sk = SS.surv[(size_t)g * SS.ccap + fl - pre[g]];
            x[u] = key_id(sk);
            if (oskip) {
              // the survivor owns exactly the node it requests here: its key for
              // head g opens g's candidate list (one entry per requested node)
              SS.cand[(size_t)g * SS.ccap + fl - pre[g]] = sk;
              const unsigned hb = (unsigned)(sk >> 32);
#pragma unroll
              for (int h = 0; h < GP; ++h)
                if (h == g) { slo[h] = min(slo[h], hb); shi[h] = max(shi[h], hb); }
            }
          }
        }
#pragma unroll
        if (lv == 1) {   // one lookup: own(p, 1) is kept per token
#pragma unroll
          for (int u = 0; u < UU; ++u) x[u] = gg[u] >= 0 ? F.own1[F.tk(t, x[u])] : 0;
        } else {
#pragma unroll
          for (int u = 0; u < UU; ++u) x[u] = gg[u] >= 0 ? F.own_base[F.tk(t, x[u])] : 0;
#pragma unroll
          for (int u = 0; u < UU; ++u) x[u] = gg[u] >= 0 ? ownl[x[u] + lv - 1] : 0;
        }
        // all UU mark atomics in flight before any result is used
        unsigned prev[UU];
#pragma unroll
        for (int u = 0; u < UU; ++u) {
          ICB_CHECK(gg[u] < 0 || (x[u] >= 0 && x[u] < F.node_cap), "own(.., %d) = %d", lv, x[u]);
          if (smark) {
            const unsigned sh = (unsigned)(x[u] % kMarkPerWord) * kMarkBits;
            prev[u] = gg[u] >= 0 ? (atomicOr(rmark + x[u] / kMarkPerWord, (1u << gg[u]) << sh) >> sh) & kMarkMask : 1u;
          } else {
            prev[u] = gg[u] >= 0 ? atomicOr(SS.nmask + x[u], 1u << gg[u]) : 1u;
          }
        }
#pragma unroll
        for (int u = 0; u < UU; ++u) {
          const bool fresh = prev[u] == 0u;
          // one smem atomic per warp for the new nodes' list slots
          const unsigned bal = __ballot_sync(0xffffffffu, fresh);
          int at = 0;
          if (lane == 0 && bal) at = atomicAdd(&S.U, __popc(bal));
          at = __shfl_sync(0xffffffffu, at, 0);
          if (fresh) SS.ulist[at + __popc(bal & ((1u << lane) - 1))] = x[u];
        }
      }
      ICB_SUB(8);
      if (oskip) {   // one shared atomic per head per warp (redux over the warp first)
#pragma unroll
        for (int h = 0; h < GP; ++h) {
          const unsigned lo_w = __reduce_min_sync(0xffffffffu, slo[h]);
          const unsigned hi_w = __reduce_max_sync(0xffffffffu, shi[h]);
          if (lane == 0 && h < G && hi_w >= lo_w) { atomicMin(&GSA[h].lo, lo_w); atomicMax(&GSA[h].hi, hi_w); }
        }
      }
      __syncthreads();
      ICB_SUB(9);
      for (int i = tid; i < S.U; i += NT) {
        const int x = SS.ulist[i];
        SS.umask[i] = smark ? (int)((rmark[x / kMarkPerWord] >> ((x % kMarkPerWord) * kMarkBits)) & kMarkMask)
                            : (int)SS.nmask[x];
      }
      __syncthreads();
      ICB_SUB(10);
    }
    const int U = S.U;
    ICB_MARK(1);
    // (2) union prefix (rows to stream) and per-head output offsets over the
    //     union (normal nodes only)
    //     (all heads + the union in one multi-value block scan) and (3a) the
    //     flattened row list (token, union index) written by the node's thread
    const bool skip_owner = oskip && lv < start;   // rows exclude owners; survivors prefix each head's list
    if (tid <= GP) S.scan_carry[tid] = (skip_owner && tid < G) ? S.nsurv[tid] : 0;
    if (tid == 0) S.nbig = 0;
    if (lv == start && tid < GP) { GSA[tid].lo = 0xffffffffu; GSA[tid].hi = 0u; }
    __syncthreads();
    constexpr int NPT = 8;   // consecutive union nodes per thread per pass (loads in parallel)
    int* stage_up = reinterpret_cast<int*>(RG.ring);   // [NT * NPT] (the ring is idle outside the stream)
    int* stage_off = stage_up + NT * NPT;
    int* stage_opos = stage_off + NT * NPT;
    int* row_node = stage_opos + NT * NPT;   // row -> node of the pass (direct lookup when it fits)
    constexpr int kRowNodeCap = (kRing * ICB_ROWF * 4) / 4 - 3 * NT * NPT;
    // start level 2: the upper list is exactly the row set (every entry has
    // top >= 2); the stream reads tokens from it directly (no row list)
    const bool rows_from_upper = lv == start && start == 2 && start < L;
    if (rows_from_upper) {
      if (tid == 0) S.scan_carry[GP] = F.meta[t].n_upper;
      __syncthreads();
      if (tid < G) { S.scan_carry[tid] = S.scan_carry[GP]; SS.uoff[(size_t)tid * F.node_cap] = 0; }
      if (tid == 0) SS.upre[0] = 0;
    } else if (lv == start && start < L) {
      // rows of the start level: the upper points of top >= start, as one
      // virtual union entry 0 requested by every head
      const int nu = F.meta[t].n_upper;
      const int* up = F.upl(t);
      for (int base = 0; base < nu; base += NT * NPT) {
        int tk[NPT], v[1] = {0}, ex[1], tot[1];
#pragma unroll
        for (int u = 0; u < NPT; ++u) {
          const int i = base + tid * NPT + u;
          tk[u] = -1;
          if (i < nu) {
            const int tok = up[i];
            if (start == 2 || F.level[F.tk(t, tok)] >= start) tk[u] = tok;
          }
          v[0] += tk[u] >= 0 ? 1 : 0;
        }
        block_scan_multi<NT, 1>(v, ex, tot, S.wsum2);
        int run = S.scan_carry[GP] + ex[0];
#pragma unroll
        for (int u = 0; u < NPT; ++u)
          if (tk[u] >= 0) {
            SS.rlist[2 * (size_t)run] = tk[u];
            SS.rlist[2 * (size_t)run + 1] = 0;
            ++run;
          }
        __syncthreads();
        if (tid == 0) S.scan_carry[GP] += tot[0];
        __syncthreads();
      }
      if (tid < G) { S.scan_carry[tid] = S.scan_carry[GP]; SS.uoff[(size_t)tid * F.node_cap] = 0; }
      if (tid == 0) SS.upre[0] = 0;
    }
    for (int base = 0; base < U && !(lv == start && start < L); base += NT * NPT) {
      const int i0 = base + tid * NPT;
      int sz[NPT], off[NPT], op[NPT];
      unsigned mk[NPT];
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        sz[u] = 0; off[u] = 0; mk[u] = 0u; op[u] = -1;
        if (i0 + u < U) {
          const size_t x = F.nd(t, SS.ulist[i0 + u]);
          sz[u] = F.node_size[x];
          off[u] = F.node_off[x];
          if (skip_owner) op[u] = F.node_opos[x];
          mk[u] = (unsigned)SS.umask[i0 + u];
        }
      }
      int v[GP + 1], ex[GP + 1], tot[GP + 1];
#pragma unroll
      for (int g = 0; g <= GP; ++g) v[g] = 0;
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        const bool big = sz[u] > ICB_EXHAUSTIVE && (long long)sz[u] > P.visit_cap;
        if (big) { atomicAdd(&S.nbig, 1); sz[u] = -sz[u]; continue; }   // negative marks P-DCI nodes
        if (skip_owner && i0 + u < U) {   // the owner's row is not streamed (rows = members - owner)
          ICB_CHECK(op[u] >= 0 && op[u] < sz[u], "owner position %d size %d", op[u], sz[u]);
          sz[u] -= 1;
        }
#pragma unroll
        for (int g = 0; g < GP; ++g) v[g] += ((mk[u] >> g) & 1) ? sz[u] : 0;
        v[GP] += sz[u];
      }
      block_scan_multi<NT, GP + 1>(v, ex, tot, S.wsum2);
      const int r0p = S.scan_carry[GP];          // rows before this pass
      const bool direct = tot[GP] <= kRowNodeCap;
      if (P.prof && tid == 0) { atomicAdd(&g_scan_stats[3], 1ull); if (!direct) atomicAdd(&g_scan_stats[4], 1ull); }
      int run[GP + 1];
#pragma unroll
      for (int g = 0; g <= GP; ++g) run[g] = S.scan_carry[g] + ex[g];
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        const int i = i0 + u;
        if (i >= U) break;
        const int s = sz[u] > 0 ? sz[u] : 0;
#pragma unroll
        for (int g = 0; g < GP; ++g) {
          if (g < G) SS.uoff[(size_t)g * F.node_cap + i] = run[g];
          run[g] += ((mk[u] >> g) & 1) ? s : 0;
        }
        SS.upre[i] = run[GP];
        stage_up[i - base] = run[GP];     // row prefix / member offset of the pass's nodes (idle ring smem)
        stage_off[i - base] = off[u];
        stage_opos[i - base] = skip_owner ? op[u] : 0x7fffffff;
        if (direct)
          for (int j = 0; j < s; ++j) row_node[run[GP] - r0p + j] = i - base;
        run[GP] += s;
      }
      __syncthreads();
      ICB_SUB(11);
      // the pass's rows in parallel: row r belongs to the last node whose
      // prefix is <= r (binary search over the staged prefixes; nodes without
      // rows share their successor's prefix and are never chosen)
      {
        const int r0 = S.scan_carry[GP], r1 = r0 + tot[GP];
        const int nn = min(U - base, NT * NPT);
        for (int rb = r0 + tid; rb < r1; rb += NT * 8) {
          int src[8], ix[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = rb + u * NT;
            if (direct) {
              ix[u] = r < r1 ? row_node[r - r0] : 0;
            } else {
              int lo = 0, hi = nn;   // first index with prefix > r, minus one
              while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (stage_up[mid] <= r) lo = mid + 1; else hi = mid;
              }
              ix[u] = lo - 1;
            }
            if (r < r1) {
              const int j = r - stage_up[ix[u]];   // member index with the owner skipped
              src[u] = stage_off[ix[u]] + j + (j >= stage_opos[ix[u]] ? 1 : 0);
            } else {
              src[u] = -1;
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) src[u] = src[u] >= 0 ? mem[src[u]] : -1;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = rb + u * NT;
            if (r < r1) {
              SS.rlist[2 * (size_t)r] = src[u];
              SS.rlist[2 * (size_t)r + 1] = base + ix[u];
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0)
#pragma unroll
        for (int g = 0; g <= GP; ++g) S.scan_carry[g] += tot[g];
      __syncthreads();
    }
    if (tid < G) S.M[tid] = S.scan_carry[tid];
    if (tid == 0) S.misc[6] = S.scan_carry[GP];
    __syncthreads();
    for (int g = 0; g < G; ++g)
      if (S.M[g] > SS.ccap) { if (tid == 0) set_err(F.meta + t, ICB_ERR_CAP_SCRATCH); return; }
    ICB_SUB(12);
    ICB_MARK(2);
    const int R = S.misc[6];
    if (P.prof && tid == 0) {
      atomicAdd(&g_scan_stats[0], 1ull);
      atomicAdd(&g_scan_stats[1], (unsigned long long)U);
      atomicAdd(&g_scan_stats[2], (unsigned long long)R);
      if (lv == start) atomicAdd(&g_scan_stats[5], 1ull);
    }
    // (3b) stream the rows through shared memory.  Every warp owns a private
    //      kSub-slot ring (two batches of 8 rows): it issues the async copies
    //      (cp.async, one 512-byte row per instruction) of its batch after
    //      next while it scores the current batch from smem against all heads
    //      (packed f32x2 lane partials, head-transposed butterfly with the
    //      pairing tree of warp_sum_butterfly).  Batches go to warps
    //      round-robin.  (A TMA cp.async.bulk + mbarrier ring was measured to
    //      be no faster for 512-byte rows.)
    {
      constexpr int NW = NT / 32;
      constexpr int LPG = 32 / GP;              // lanes holding one head's sum
      constexpr int SLOTS = (8 + LPG - 1) / LPG;
      const int myh = lane / LPG;
      const float qt_my = S.qt[(GP == 4 && XP) ? (lane & 3) : myh];
      const unsigned qb = RG.qp[warp];
      float* wring = RG.ring + (size_t)warp * kSub * ICB_ROWF;
      unsigned long long* wfull = RG.full + warp * kSub;
      const int nb = (R + 7) / 8;
      // Row metadata pipeline, lanes 0..7 holding one row each:
      //   stage A, three batches ahead: token and union index (row list);
      //   stage B, two batches ahead: lifted tail, requesting-head mask and
      //   the row's output slot per head (gathers that depend on stage A).
      struct RowTok {
        int tok, ix;
      };
      // raw gathered values only: every use is deferred to the batch's own
      // iteration, two batches later, so the loads stay in flight meanwhile
      struct RowMeta {
        int tok;
        float tail;
        int mask;
        int upre;
        int uo[GP];
      };
      const int* upl_t = F.upl(t);
      auto load_a = [&](int kb) {
        RowTok a{0, -1};
        const int j = warp + kb * NW;
        if (j < nb && lane < 8 && 8 * j + lane < R) {
          if (rows_from_upper) {
            a.tok = upl_t[8 * j + lane];
            a.ix = 0;
          } else {
            a.tok = SS.rlist[2 * (size_t)(8 * j + lane)];
            a.ix = SS.rlist[2 * (size_t)(8 * j + lane) + 1];
          }
        }
        return a;
      };
      auto load_b = [&](int kb, const RowTok& a) {
        RowMeta m;
        m.tok = a.tok;
        m.tail = 0.f;
        m.mask = 0;
        m.upre = 0;
#pragma unroll
        for (int g = 0; g < GP; ++g) m.uo[g] = 0;
        if (a.ix >= 0) {
          m.tail = F.tail[F.tk(t, a.tok)];
          m.mask = SS.umask[a.ix];
          m.upre = SS.upre[a.ix];
#pragma unroll
          for (int g = 0; g < GP; ++g) m.uo[g] = g < G ? SS.uoff[(size_t)g * F.node_cap + a.ix] : 0;
        }
        (void)kb;
        return m;
      };
      // LDGSTS: the warp copies each 512-byte row with one instruction (16 B
      // per lane, four full 128-B lines), one commit group per batch
      auto issue = [&](int kb, int tk) {
        const int j = warp + kb * NW;
        if (j < nb) {
          const int sb = (kb & 1) * 8;
          const int nr = min(8, R - 8 * j);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int tu = __shfl_sync(0xffffffffu, tk, u);
            if (u < nr) cp_async16(wring + (size_t)(sb + u) * ICB_ROWF + lane * 4, F.row(t, tu) + lane * 4);
          }
        }
        cp_async_commit();
      };
      RowTok a2 = load_a(2);
      RowMeta m0 = load_b(0, load_a(0));
      RowMeta m1 = load_b(1, load_a(1));
      issue(0, m0.tok);
      issue(1, m1.tok);
      unsigned mn = 0xffffffffu, mx = 0u;
      int kb = 0;
      for (int j = warp; j < nb; j += NW, ++kb) {
        const int base = 8 * j;
        const int nrow = min(8, R - base);
        const RowTok a3 = load_a(kb + 3);       // stage A for the batch three ahead
        const RowMeta m2 = load_b(kb + 2, a2);  // stage B for the batch two ahead
        const int sbase = (kb & 1) * 8;
        cp_async_wait<1>();   // this batch's group has landed (the next one may be in flight)
        __syncwarp();         // ...and every lane's part of it is visible to the warp
        if constexpr (GP == 4 && XP) {
          // Fully transposed reduction of the batch's 8 rows x 4 heads: in
          // slot jj lane l scores smem row jj ^ pi(l), pi(l) = lane bits 4..2,
          // so at the row levels (xor 16, 8, 4) every lane keeps its low slots
          // and sends its high ones with no selects, on packed head pairs
          // (FADD2); the head levels (xor 2, 1) split the pairs.  Every sum is
          // still the 16,8,4,2,1 pairing tree of warp_sum_butterfly, and lane l
          // ends with (row pi(l), head l & 3).
          const int pi = (lane >> 2) & 7;
          unsigned long long v[8][2];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const float4 p = reinterpret_cast<const float4*>(wring + (size_t)(sbase + (jj ^ pi)) * ICB_ROWF)[lane];
            v[jj][0] = lane_sq4_x2_packed(p, q2[0]);
            v[jj][1] = lane_sq4_x2_packed(p, q2[1]);
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int h = 0; h < 2; ++h) v[jj][h] = fadd2(v[jj][h], shfl_xor_u64(v[jj + 4][h], 16));
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int h = 0; h < 2; ++h) v[jj][h] = fadd2(v[jj][h], shfl_xor_u64(v[jj + 2][h], 8));
#pragma unroll
          for (int h = 0; h < 2; ++h) v[0][h] = fadd2(v[0][h], shfl_xor_u64(v[1][h], 4));
          const bool b1 = lane & 2, b0 = lane & 1;
          const unsigned long long w = fadd2(b1 ? v[0][1] : v[0][0], shfl_xor_u64(b1 ? v[0][0] : v[0][1], 2));
          const float wl = __uint_as_float((unsigned)w), wh = __uint_as_float((unsigned)(w >> 32));
          const float f = __fadd_rn(b0 ? wh : wl, __shfl_xor_sync(0xffffffffu, b0 ? wl : wh, 1));
          const float d2 = d2_finish(f, __shfl_sync(0xffffffffu, m0.tail, pi), qt_my);
          // every lane's smem reads of this batch have retired: its slots take
          // the batch after next
          __syncwarp();
          issue(kb + 2, a2.tok);
          const int h = lane & 3;
          const int tok = __shfl_sync(0xffffffffu, m0.tok, pi);
          const int msk = __shfl_sync(0xffffffffu, m0.mask, pi);
          const int upr = __shfl_sync(0xffffffffu, m0.upre, pi);
          int pos = 0;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int pg = __shfl_sync(0xffffffffu, m0.uo[g], pi);
            if (g == h) pos = pg;
          }
          pos += base + pi - upr;
          if (pi < nrow && h < G && ((msk >> h) & 1)) {
            ICB_CHECK(pos >= 0 && pos < S.M[h], "cand pos %d M %d", pos, S.M[h]);
            SS.cand[(size_t)h * SS.ccap + pos] = make_key(d2, tok);
            const unsigned hb = __float_as_uint(d2);
            mn = min(mn, hb);
            mx = max(mx, hb);
          }
        } else {
          float keep[SLOTS];
          // branch-free over the 8 rows (rows >= nrow score stale smem and are
          // never stored) so the 8 independent reduction chains interleave
  #pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float* srow = wring + (size_t)(sbase + u) * ICB_ROWF;
            const float4 p = reinterpret_cast<const float4*>(srow)[lane];
            const float tl = __shfl_sync(0xffffffffu, m0.tail, u);
            float v[GP];
            if constexpr (GP == 1) {
              v[0] = lane_sq4(p, qv[0]);
            } else {
  #pragma unroll
              for (int h = 0; h < GP / 2; ++h) {
                const float2 r2 = lane_sq4_x2(p, q2[h]);
                v[2 * h] = r2.x;
                v[2 * h + 1] = r2.y;
              }
            }
            float f = reduce_heads<GP>(v, lane);
            float d2 = d2_finish(f, tl, qt_my);
            if ((u % LPG) == (lane % LPG)) keep[u / LPG] = d2;
          }
          // every lane's smem reads of this batch have retired (the butterflies
          // consumed them): its slots take the batch after next
          __syncwarp();
          issue(kb + 2, a2.tok);
  #pragma unroll
          for (int sl = 0; sl < SLOTS; ++sl) {
            const int u = sl * LPG + (lane % LPG);
            const int src = u < 8 ? u : 0;
            const int tok = __shfl_sync(0xffffffffu, m0.tok, src);
            const int msk = __shfl_sync(0xffffffffu, m0.mask, src);
            const int upr = __shfl_sync(0xffffffffu, m0.upre, src);
            int pos = 0;
  #pragma unroll
            for (int g = 0; g < GP; ++g) {
              const int pg = __shfl_sync(0xffffffffu, m0.uo[g], src);
              if (g == myh) pos = pg;
            }
            pos += base + u - upr;   // row index within its node
            if (u < nrow && myh < G && ((msk >> myh) & 1)) {
              ICB_CHECK(pos >= 0 && pos < S.M[myh], "cand pos %d M %d", pos, S.M[myh]);
              SS.cand[(size_t)myh * SS.ccap + pos] = make_key(keep[sl], tok);
              const unsigned hb = __float_as_uint(keep[sl]);
              mn = min(mn, hb);
              mx = max(mx, hb);
            }
          }

        }
        m0 = m1;
        m1 = m2;
        a2 = a3;
      }
      // per-head d2 range of this level's candidates (feeds the selection bins)
      if constexpr (GP == 4 && XP) {   // head = lane & 3
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane < G && lane < 4 && mx >= mn) {
          atomicMin(&GSA[lane].lo, mn);
          atomicMax(&GSA[lane].hi, mx);
        }
      } else {
#pragma unroll
        for (int o = 1; o < LPG; o <<= 1) {
          mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if ((lane % LPG) == 0 && myh < G && mx >= mn) {
          atomicMin(&GSA[myh].lo, mn);
          atomicMax(&GSA[myh].hi, mx);
        }
      }
      __syncwarp();
      if (lane == 0) RG.qp[warp] = qb + (unsigned)kb;   // batches this warp consumed
    }
    if (tid == 0) S.misc[5] = R;
    __syncthreads();
    ICB_MARK(4);
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
          eval_list_one_head<NT>(S, F, t, SS.vis, cnt, g, SS.cand + (size_t)g * SS.ccap + S.M[g], &GSA[g].lo,
                                 &GSA[g].hi);
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
      if (lv < start && !oskip) atomicAdd(&F.meta[t].owner_rereads, (unsigned long long)U);
    }
    if (lv < start && !smark)
      for (int i = tid; i < U; i += NT) SS.nmask[SS.ulist[i]] = 0u;
    __syncthreads();
    ICB_MARK(5);
    // (7) per-head selection, heads in parallel (one warp group per head).
    //     Survivors = top-beam (dci.py:359-361).  The pool collects, without
    //     duplicates, every survivor (a superset of the level's top-k since
    //     beam >= k) and the floor level's top-k (dci.py:355-358).
    if (grp < G) {
      const int g = grp;
      unsigned long long* cg = SS.cand + (size_t)g * SS.ccap;
      unsigned long long* pg = SS.pool + (size_t)g * SS.ccap;
      unsigned* sg = SS.seen + (size_t)g * (F.tok_cap / 32 + 1);
      const int M = S.M[g];
      if (lv == start && gtid == 0) { GS.plo = 0xffffffffu; GS.phi = 0u; }
      gsync(gbar, NTG);
      const bool nopool = S.nopool;
      unsigned char* rg = reinterpret_cast<unsigned char*>(RG.ring) + (size_t)grp * TopB<GP>::kBytes;
      if (nopool && lv > floor) {
        const int n = group_topb<NTG, GP>(GS, rg, gtid, gbar, cg, M, P.beam, GS.lo, GS.hi,
                                                  SS.surv + (size_t)g * SS.ccap, P.prof != nullptr);
        if (gtid == 0) S.nsurv[g] = n;
      } else if (lv > floor) {
        unsigned long long thr = group_threshold<NTG>(GS, gtid, gbar, cg, M, P.beam, GS.lo, GS.hi);
        const int2 r = group_emit<NTG>(GS, gtid, gbar, cg, M, thr, SS.surv + (size_t)g * SS.ccap, 0,
                                       collect_all && !nopool ? pg : nullptr, S.npool[g], sg, &GS.plo, &GS.phi);
        if (gtid == 0) {
          S.nsurv[g] = r.x;
          S.npool[g] += r.y;
        }
      } else if (nopool) {
        // the floor's top-k is the answer: straight into the group's buffer, sorted
        const int n = group_topb<NTG, GP>(GS, rg, gtid, gbar, cg, M, P.k, GS.lo, GS.hi, GS.buf, P.prof != nullptr);
        group_sort<NTG>(GS, gtid, gbar, n);
        if (gtid == 0) S.npool[g] = n;
      } else {
        unsigned long long thr = group_threshold<NTG>(GS, gtid, gbar, cg, M, P.k, GS.lo, GS.hi);
        const int2 r = group_emit<NTG>(GS, gtid, gbar, cg, M, thr, nullptr, 0, pg, S.npool[g], sg, &GS.plo,
                                       &GS.phi);
        if (gtid == 0) S.npool[g] += r.y;
      }
    }
    __syncthreads();
    ICB_MARK(6);
  }
}

// Final ranked top-k (k <= kBuf) of every head, in parallel: the pool's
// top-k lands sorted in GSA[g].buf[0..n); seen marks are cleared.  Returns n
// for the calling thread's head (all threads must call).
template <int NT, int GP>
__device__ int finalize_groups(SearchSmem& S, GroupSmem* GSA, const ForestView& F, const SearchScratch& SS, int G,
                               long long k) {
  constexpr int NTG = NT / GP;
  const int tid = threadIdx.x, grp = tid / NTG, gtid = tid % NTG, gbar = 1 + grp;
  int n = 0;
  if (S.nopool) {   // tree_search left the sorted floor top-k in GS.buf
    __syncthreads();
    return grp < G ? S.npool[grp] : 0;
  }
  if (grp < G) {
    GroupSmem& GS = GSA[grp];
    unsigned long long* pg = SS.pool + (size_t)grp * SS.ccap;
    unsigned* sg = SS.seen + (size_t)grp * (F.tok_cap / 32 + 1);
    const int np = S.npool[grp];
    for (int i = gtid; i < np; i += NTG) {
      int id = key_id(pg[i]);
      atomicAnd(sg + (id >> 5), ~(1u << (id & 31)));
    }
    gsync(gbar, NTG);
    const long long want = min((long long)np, k);
    unsigned long long thr = group_threshold<NTG>(GS, gtid, gbar, pg, np, want, GS.plo, GS.phi);
    // emit into a scratch region (the threshold pass may have used buf)
    n = group_emit<NTG>(GS, gtid, gbar, pg, np, thr, nullptr, 0, GS.buf, 0, nullptr, nullptr, nullptr).y;
    group_sort<NTG>(GS, gtid, gbar, n);
  }
  __syncthreads();
  return n;
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
