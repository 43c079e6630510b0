// exact_add.cuh -- exact aggregation of repeated IEEE binary64 additions.
//
// The timeline advances a device clock x by one
// rounded addition per op: x <- RN(x + a_j).  A pipeline task repeats the
// same short op sequence (a GPT-2 block, a pair of MLP layers) many times,
// so a stage's clock is a long serial chain of adds.  This header evaluates
// that chain EXACTLY -- bit-identical to performing every addition -- in
// O(1) per repetition run instead of O(ops):
//
//   Let x > 0 be a normal double in binade E (2^E <= x < 2^(E+1)) and
//   u = 2^(E-52) its ulp, so x = M*u with M an integer in [2^52, 2^53).
//   For a >= 0 the exact sum x + a lies on the same binade's grid (spacing u)
//   as long as x + a < 2^(E+1); then RN(x + a) = (M + RNI(a/u)) * u, where
//   RNI rounds to the nearest integer -- unambiguous unless a/u is exactly
//   half an odd integer (a tie, broken by the parity of the running total).
//   Hence, for an op sequence a_1..a_N with no tie at binade E and
//   r_j = RNI(a_j/u), applying it n times from x yields exactly
//   (M + n*sum_j r_j) * u provided M + n*sum_j r_j <= 2^53 - 1 (every
//   intermediate exact sum then stays below 2^(E+1)).  Otherwise one
//   repetition is performed op by op (it crosses into the next binade, or
//   contains a tie), the cache is recomputed for the new binade, and the
//   remaining repetitions continue.  a/u is exact (power-of-two scaling);
//   all integer-valued doubles involved stay below 2^53.
//
// The kernels only ever call add_reps; the fallback path is the plain
// sequence of __dadd_rn, so the aggregation can never change a result.
#pragma once
#include <cstdint>

#ifndef DISTIR_HD
#ifdef __CUDACC__
#define DISTIR_HD __host__ __device__ __forceinline__
#else
#define DISTIR_HD inline
#endif
#endif

namespace distir {

#ifdef __CUDA_ARCH__
DISTIR_HD double xadd(double a, double b) { return __dadd_rn(a, b); }
DISTIR_HD double xmul(double a, double b) { return __dmul_rn(a, b); }
DISTIR_HD int64_t d2bits(double x) { return __double_as_longlong(x); }
DISTIR_HD double bits2d(int64_t b) { return __longlong_as_double(b); }
DISTIR_HD double xfloor(double x) { return floor(x); }
DISTIR_HD double xrint(double x) { return rint(x); }
#else
DISTIR_HD double xadd(double a, double b) { return a + b; }
DISTIR_HD double xmul(double a, double b) { return a * b; }
DISTIR_HD int64_t d2bits(double x) {
  int64_t b;
  __builtin_memcpy(&b, &x, 8);
  return b;
}
DISTIR_HD double bits2d(int64_t b) {
  double x;
  __builtin_memcpy(&x, &b, 8);
  return x;
}
DISTIR_HD double xfloor(double x) { return __builtin_floor(x); }
DISTIR_HD double xrint(double x) { return __builtin_rint(x); }
#endif

constexpr double kTwo53m1 = 9007199254740991.0;  // 2^53 - 1

// Per-sequence cache: binade exponent field, sum of per-op ulp increments,
// and whether any op is a tie at that binade.
struct SeqCache {
  int32_t ef;      // biased exponent field of the cached binade (-1 = none)
  bool tie;
  double R;        // sum_j RNI(a_j / u), an integer < 2^53 (or >= 2^53: never fits)
};

DISTIR_HD SeqCache seq_cache_empty() { return SeqCache{-1, false, 0.0}; }

// x's biased exponent field; usable binades need 53 <= ef <= 2046 - 53 so
// that u and 1/u are normal powers of two.
DISTIR_HD int32_t exp_field(double x) { return (int32_t)((d2bits(x) >> 52) & 0x7FF); }

template <int N>
DISTIR_HD void seq_plain(double& x, const double (&a)[N]) {
#pragma unroll
  for (int j = 0; j < N; j++) x = xadd(x, a[j]);
}

template <int N>
DISTIR_HD void seq_refresh(SeqCache& c, int32_t ef, const double (&a)[N]) {
  // 1/u = 2^(52 - E) = 2^(1075 - ef); its biased field = 1075 - ef + 1023.
  const double inv_u = bits2d((int64_t)(2098 - ef) << 52);
  double R = 0.0;
  bool tie = false;
#pragma unroll
  for (int j = 0; j < N; j++) {
    const double q = xmul(a[j], inv_u);          // exact: power-of-two scale
    const double fl = xfloor(q);
    tie |= (xadd(q, -fl) == 0.5);
    R = xadd(R, xrint(q));                       // exact while R < 2^53
  }
  c.ef = ef;
  c.tie = tie;
  c.R = R;
}

// x <- N*reps successive RN additions of a[0..N), computed exactly.
template <int N>
DISTIR_HD void add_reps(double& x, const double (&a)[N], int64_t reps, SeqCache& c) {
  while (reps > 0) {
    const int32_t ef = exp_field(x);
    if (x <= 0.0 || ef < 53 || ef > 1993) {      // zero / tiny / huge: plain
      seq_plain(x, a);
      reps--;
      continue;
    }
    if (ef != c.ef) seq_refresh(c, ef, a);
    if (!c.tie) {
      const double inv_u = bits2d((int64_t)(2098 - ef) << 52);
      const double u = bits2d((int64_t)(ef - 52) << 52);
      const double M = xmul(x, inv_u);           // integer in [2^52, 2^53)
      const double avail = xadd(kTwo53m1, -M);   // exact
      int64_t fit = reps;
      if (c.R > 0.0) {
        const double f = xfloor(avail / c.R);
        if (f < (double)reps) fit = (int64_t)f;
        while (fit > 0 && xmul((double)fit, c.R) > avail) fit--;
      }
      if (fit > 0) {
        x = xadd(x, xmul(xmul((double)fit, c.R), u));   // exact: lands on the grid
        reps -= fit;
      }
    }
    if (reps > 0) {                              // crossing (or tie): op by op
      seq_plain(x, a);
      reps--;
    }
  }
}

// ------------------------------------------------------------------ memory --
// A live-memory profile of an op sequence (C.7): the highest point reached
// relative to the start (allocations are counted before frees, so it is the
// max over ops of prefix_net + alloc) and the net change.  Composition and
// repetition are exact integer identities.
struct MemProf {
  int64_t mp, net;
};

DISTIR_HD MemProf mem_id() { return MemProf{INT64_MIN / 4, 0}; }
DISTIR_HD MemProf mem_op(int64_t alloc, int64_t free_) { return MemProf{alloc, alloc - free_}; }
DISTIR_HD MemProf mem_then(MemProf a, MemProf b) {
  const int64_t m2 = a.net + b.mp;
  return MemProf{a.mp > m2 ? a.mp : m2, a.net + b.net};
}
DISTIR_HD MemProf mem_rep(MemProf a, int64_t n) {
  if (n <= 0) return mem_id();
  const int64_t extra = a.net > 0 ? (n - 1) * a.net : 0;
  return MemProf{a.mp + extra, n * a.net};
}
DISTIR_HD void mem_apply(int64_t& live, int64_t& peak, MemProf p) {
  const int64_t hi = live + p.mp;
  peak = peak > hi ? peak : hi;
  live += p.net;
}

}  // namespace distir
