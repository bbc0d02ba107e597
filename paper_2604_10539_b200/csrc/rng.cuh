// Host+device restatement of the reference's random streams.
//
// The reference draws DCI levels from `np.random.default_rng(SeedSequence(
// entropy, spawn_key=(0,)))` (dci.py:180-183, assign_level dci.py:81-88) and
// P-DCI projection directions from `default_rng(SeedSequence(entropy,
// spawn_key=(1, node_id))).normal(size=(8, d+1))` (dci.py:268-273).  This
// header restates NumPy's SeedSequence hashing, PCG64 (XSL-RR 128/64), the
// 53-bit double draw and the 256-layer ziggurat normal, so the device draws
// the same bits (validated against NumPy in tests/test_native_cpu.py).
#pragma once
#include <stdint.h>
#include <math.h>

#ifdef __CUDACC__
#define ICB_HD __host__ __device__ __forceinline__
#else
#define ICB_HD inline
#endif

typedef unsigned __int128 icb_u128;

struct Pcg64 {
  icb_u128 state;
  icb_u128 inc;
};

// SeedSequence(entropy words, spawn_key).generate_state(4, uint64)
// (numpy/random/bit_generator.pyx: _get_assembled_entropy, mix_entropy,
// generate_state).  `ent` are the run-entropy uint32 words (little-endian
// split of each integer), `spawn` the spawn-key words.
ICB_HD void icb_seedseq_u64x4(const uint32_t* ent, int n_ent, const uint32_t* spawn, int n_spawn,
                              uint64_t out[4]) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  const uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t buf[24];
  int n = 0;
  for (int i = 0; i < n_ent && n < 20; ++i) buf[n++] = ent[i];
  if (n_spawn > 0)
    while (n < 4) buf[n++] = 0u;
  for (int i = 0; i < n_spawn && n < 24; ++i) buf[n++] = spawn[i];
  uint32_t hc = INIT_A;
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) {
    uint32_t v = i < n ? buf[i] : 0u;
    v ^= hc; hc *= MULT_A; v *= hc; v ^= v >> 16;
    pool[i] = v;
  }
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) {
        uint32_t v = pool[s];
        v ^= hc; hc *= MULT_A; v *= hc; v ^= v >> 16;
        uint32_t r = MIX_L * pool[d] - MIX_R * v;
        r ^= r >> 16;
        pool[d] = r;
      }
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) {
      uint32_t v = buf[s];
      v ^= hc; hc *= MULT_A; v *= hc; v ^= v >> 16;
      uint32_t r = MIX_L * pool[d] - MIX_R * v;
      r ^= r >> 16;
      pool[d] = r;
    }
  uint32_t hb = INIT_B;
  uint32_t st[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb; hb *= MULT_B; v *= hb; v ^= v >> 16;
    st[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
}

ICB_HD icb_u128 icb_pcg_mult() {
  return ((icb_u128)0x2360ED051FC65DA4ULL << 64) | (icb_u128)0x4385DF649FCCF645ULL;
}

// pcg64_set_seed -> pcg_setseq_128_srandom_r
ICB_HD Pcg64 icb_pcg_seed(const uint64_t v[4]) {
  Pcg64 g;
  icb_u128 initstate = ((icb_u128)v[0] << 64) | v[1];
  icb_u128 initseq = ((icb_u128)v[2] << 64) | v[3];
  g.state = 0;
  g.inc = (initseq << 1) | 1u;
  g.state = g.state * icb_pcg_mult() + g.inc;
  g.state += initstate;
  g.state = g.state * icb_pcg_mult() + g.inc;
  return g;
}

ICB_HD uint64_t icb_pcg_next64(Pcg64& g) {
  g.state = g.state * icb_pcg_mult() + g.inc;
  uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

ICB_HD double icb_pcg_double(Pcg64& g) {
  return (double)(icb_pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// LCG jump: the state after `delta` steps is A * state + C (the standard
// O(log delta) power-of-the-affine-map construction).
ICB_HD void icb_pcg_jump(unsigned long long delta, icb_u128 inc, icb_u128& A, icb_u128& C) {
  icb_u128 am = 1, ap = 0, cm = icb_pcg_mult(), cp = inc;
  while (delta) {
    if (delta & 1ull) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  A = am;
  C = ap;
}

ICB_HD uint64_t icb_pcg_output(icb_u128 state) {
  uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// assign_level (dci.py:81-88): 1 + number of consecutive uniforms below r.
ICB_HD int icb_draw_level(Pcg64& g, double r) {
  int level = 1;
  while (icb_pcg_double(g) < r) ++level;
  return level;
}

#ifdef __CUDACC__
#define ICB_ZIG_TABLE(T, name) __device__ __constant__ const T name[256]
#else
#define ICB_ZIG_TABLE(T, name) static const T name[256]
#endif
#include "ziggurat_tables.inc"

// NumPy random_standard_normal (distributions.c), ziggurat with 256 layers.
// Device-only (tables live in device constant memory).
#ifdef __CUDACC__
__device__ __forceinline__ double icb_normal(Pcg64& g) {
  const double ZR = 3.6541528853610087963519472518;
  const double ZINV = 0.27366123732975827203338247596;
  for (;;) {
    uint64_t r = icb_pcg_next64(g);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 0x1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * icb_zig_wi[idx];
    if (sign & 0x1) x = -x;
    if (rabs < icb_zig_ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -ZINV * log1p(-icb_pcg_double(g));
        double yy = -log1p(-icb_pcg_double(g));
        if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(ZR + xx) : ZR + xx;
      }
    } else {
      // explicit roundings: NumPy's C build does not contract this to an FMA
      double lhs = __dadd_rn(__dmul_rn(__dsub_rn(icb_zig_fi[idx - 1], icb_zig_fi[idx]),
                                       icb_pcg_double(g)),
                             icb_zig_fi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) return x;
    }
  }
}
#endif
