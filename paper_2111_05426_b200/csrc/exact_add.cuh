// exact_add.cuh -- exact aggregation of repeated IEEE binary64 additions.
//
// The timeline advances a device clock x by one
// rounded addition per op: x <- RN(x + a_j).  A pipeline task repeats the
// same short op sequence (a GPT-2 block, a pair of MLP layers) many times,
// so a stage's clock is a long serial chain of adds.  This header evaluates
// that chain EXACTLY -- bit-identical to performing every addition -- in
// O(1) per task instead of O(ops):
//
//   Let x > 0 be a normal double in binade E (2^E <= x < 2^(E+1)) and
//   u = 2^(E-52) its ulp, so x = M*u with M its 53-bit significand
//   (2^52 <= M < 2^53).  For a >= 0 the exact sum x + a lies on the same
//   binade's grid (spacing u) as long as x + a < 2^(E+1); then
//   RN(x + a) = (M + i)*u where i rounds a/u to the nearest integer -- and
//   when a/u is exactly m + 1/2 (a tie), to the i in {m, m+1} that makes
//   M + i even.  So one pass of a sequence a_1..a_N adds an integer number of
//   ulps that depends only on the binade and on the parity of M (R0 / R1),
//   and n passes add a closed-form total S (the parity sequence has period
//   <= 2), provided M + S <= 2^53 - 1: every intermediate exact sum then stays
//   below 2^(E+1).  That condition is checked by computing y = x + S*u: the
//   exact value (M + S)*u is representable iff M + S < 2^53, so y keeps x's
//   exponent exactly when the aggregation is valid (and is then exact).
//   Passes that would cross into the next binade are performed op by op; the
//   cache is then recomputed for the new binade.
//
// The fallback path is the plain sequence of __dadd_rn, so aggregation can
// never change a result (host check: tests/native/exact_add_check.cpp).
#pragma once
#include <cstdint>

#ifndef DISTIR_COLD_NOINLINE
#define DISTIR_COLD_NOINLINE 0
#endif
#ifndef DISTIR_PLAIN_AFTER
#define DISTIR_PLAIN_AFTER 0   // crossings after which a task is walked op by op (0: never)
#endif
#ifndef DISTIR_UNROLL_SEG
#define DISTIR_UNROLL_SEG 0
#endif
#ifndef DISTIR_HD
#ifdef __CUDACC__
#define DISTIR_HD __host__ __device__ __forceinline__
#if DISTIR_COLD_NOINLINE
#define DISTIR_HD_COLD __host__ __device__ __noinline__
#else
#define DISTIR_HD_COLD __host__ __device__ __forceinline__
#endif
#else
#define DISTIR_HD inline
#define DISTIR_HD_COLD inline
#endif
#endif

#ifndef DISTIR_COUNT
#define DISTIR_COUNT(i)
#endif
#ifndef DISTIR_CLK_ADD
#define DISTIR_CLK_ADD(i, t0) ((void)(t0))   // instrumentation: cycles since t0 into counter i
#define DISTIR_CLK_NOW() 0ll
#endif

namespace distir {

#ifdef __CUDA_ARCH__
DISTIR_HD double xadd(double a, double b) { return __dadd_rn(a, b); }
DISTIR_HD int64_t d2bits(double x) { return __double_as_longlong(x); }
DISTIR_HD double bits2d(int64_t b) { return __longlong_as_double(b); }
#else
DISTIR_HD double xadd(double a, double b) { return a + b; }
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
#endif

constexpr int64_t kMant = (int64_t(1) << 52) - 1;
constexpr int64_t kHidden = int64_t(1) << 52;
constexpr int64_t kTwo53 = int64_t(1) << 53;
constexpr double kTwo53d = 9007199254740992.0;
constexpr double kNever = 1.152921504606846976e18;   // 2^60: never fits a binade
DISTIR_HD double kInf() { return bits2d(0x7FF0000000000000ll); }

#ifdef __CUDA_ARCH__
DISTIR_HD double xmul(double a, double b) { return __dmul_rn(a, b); }
DISTIR_HD double xfloor(double x) { return floor(x); }
DISTIR_HD double xrint(double x) { return rint(x); }
#else
DISTIR_HD double xmul(double a, double b) { return a * b; }
DISTIR_HD double xfloor(double x) { return __builtin_floor(x); }
DISTIR_HD double xrint(double x) { return __builtin_rint(x); }
#endif

// x's biased exponent field.
DISTIR_HD int32_t exp_field(double x) { return (int32_t)((d2bits(x) >> 52) & 0x7FF); }

DISTIR_HD int odd(double integral) { return (int)((int64_t)integral & 1); }

constexpr int kSegMax = 14;   // longest op sequence of a segment (GPT-2 block)

#ifdef __CUDA_ARCH__
DISTIR_HD float fdiv_approx(float a, float b) { return __fdividef(a, b); }
#else
DISTIR_HD float fdiv_approx(float a, float b) { return a / b; }
#endif

DISTIR_HD void seq_plain(double& x, const double* a, int n) {
#if DISTIR_UNROLL_SEG
#pragma unroll
  for (int j = 0; j < kSegMax; j++)
    if (j < n) x = xadd(x, a[j]);
#else
  for (int j = 0; j < n; j++) x = xadd(x, a[j]);
#endif
}

// Ulps added by one pass of a[0..n) at binade field ef, from an even (R0) and
// an odd (R1) significand.  Returns false when the pass can never fit the
// binade (an op of at least 2^52 ulps).  Exact: a*2^k is exact, floor/rint of
// such a double are exact, and sums of integers below 2^53 are exact.
DISTIR_HD bool seg_pass_d(const double* a, int n, int32_t ef, double& R0, double& R1) {
  const double inv_u = bits2d((int64_t)(2098 - ef) << 52);    // 2^(52-E)
  // the ops are independent: two partial sums halve the dependent chain (the
  // integers add exactly while below 2^53; a total >= 2^53 fails below
  // either way, rounding being monotone)
  double Ra = 0.0, Rb = 0.0;
  bool tie = false, never = false;
#pragma unroll
  for (int j = 0; j < kSegMax; j++) {
    if (j < n) {
      const double q = xmul(a[j], inv_u);
      never |= !(q < kTwo53d);
      tie |= (xadd(q, -xfloor(q)) == 0.5);
      if (j & 1) Rb = xadd(Rb, xrint(q));
      else Ra = xadd(Ra, xrint(q));
    }
  }
  if (never) return false;
  const double R = xadd(Ra, Rb);
  R0 = R1 = R;
  if (tie) {                      // resolve ties by the running parity
    R0 = R1 = 0.0;
    int p0 = 0, p1 = 1;
    for (int j = 0; j < kSegMax; j++) {
      if (j >= n) break;
      const double q = xmul(a[j], inv_u);
      const double fl = xfloor(q);
      const double fr = xadd(q, -fl);
      double i0 = fr > 0.5 ? xadd(fl, 1.0) : fl, i1 = i0;
      if (fr == 0.5) {
        const int of = odd(fl);
        i0 = (p0 ^ of) ? xadd(fl, 1.0) : fl;
        i1 = (p1 ^ of) ? xadd(fl, 1.0) : fl;
      }
      p0 ^= odd(i0);
      p1 ^= odd(i1);
      R0 = xadd(R0, i0);
      R1 = xadd(R1, i1);
    }
  }
  return R0 < kTwo53d && R1 < kTwo53d;
}

// The per-pass increments as integers (exact: they are integers < 2^53);
// kNeverI marks a pass that never fits a binade.
constexpr int64_t kNeverI = int64_t(1) << 60;
DISTIR_HD bool seg_pass(const double* a, int n, int32_t ef, int64_t& R0, int64_t& R1) {
  double r0, r1;
  if (!seg_pass_d(a, n, ef, r0, r1)) { R0 = R1 = kNeverI; return false; }
  R0 = (int64_t)r0;
  R1 = (int64_t)r1;
  return true;
}

// Total ulps of n passes from significand parity p (the parity sequence has
// period <= 2); kNeverI when it cannot fit a binade.  Integer arithmetic:
// R < 2^53 and n <= 2^10 (passes per segment <= layers per stage <= 1024),
// so no product overflows.
DISTIR_HD int64_t reps_total(int64_t R0, int64_t R1, int p, int64_t n) {
  const int64_t Ra = p ? R1 : R0, Rb = p ? R0 : R1;
  if (n == 1) return Ra;
  int64_t s;
  if (!(Ra & 1)) s = n * Ra;                                    // parity stays
  else if (!(Rb & 1)) s = Ra + (n - 1) * Rb;                    // flips once
  else s = (n - (n >> 1)) * Ra + (n >> 1) * Rb;                 // alternates
  return s < kTwo53 ? s : kNeverI;                              // monotone rounding
}

// A task is a list of segments: `reps` passes over the op costs a[0..n).
struct Seg {
  const double* a;
  int n;
  int64_t reps;
};

// Per-task cache for one binade: the x increment of the whole task from an
// even / odd significand (+inf: the task never fits this binade), the
// binade's bounds [2^E, 2^(E+1)) as high words of their bit patterns
// (lo = INT32_MAX: no binade cached), and each segment's per-pass ulp
// increments (R[2i], R[2i+1]; kNever if a pass never fits) in
// caller-provided per-lane storage.
struct TaskCache {
  int32_t ef;
  int32_t lo, hi;
  double Su0, Su1;
  int64_t* R;
};

#ifdef __CUDA_ARCH__
DISTIR_HD int32_t hiword(double x) { return __double2hiint(x); }
DISTIR_HD int32_t loword(double x) { return __double2loint(x); }
#else
DISTIR_HD int32_t hiword(double x) { return (int32_t)(d2bits(x) >> 32); }
DISTIR_HD int32_t loword(double x) { return (int32_t)d2bits(x); }
#endif

// Per-pass increments of a configuration's nu distinct segment op lists for
// the binades [e0, e0 + nb), filled cooperatively by the configuration's
// lanes before its walk (binade b, list u at tab[(b * nu + u) * 2]); a task
// cache reads its segments through a map (segment i -> list map[i]).
// nb = 0 disables the table.
struct BinTab {
  int64_t* tab;
  int32_t e0, nb, nu;
};

DISTIR_HD TaskCache task_cache_make(int64_t* store) {
  return TaskCache{-1, 0x7FFFFFFF, 0, kInf(), kInf(), store};
}

// Fill binades e0 + first, e0 + first + stride, ... of a table of the NU
// distinct op lists (reps are ignored).
template <int NU>
DISTIR_HD void bintab_fill(const BinTab& t, const Seg (&u)[NU], int first, int stride) {
  for (int b = first; b < t.nb; b += stride) {
    const int32_t ef = t.e0 + b;
#pragma unroll
    for (int i = 0; i < NU; i++) {
      int64_t R0 = kNeverI, R1 = kNeverI;
      if (!(ef >= 53 && ef <= 1993) || !seg_pass(u[i].a, u[i].n, ef, R0, R1)) R0 = R1 = kNeverI;
      t.tab[((int64_t)b * NU + i) * 2] = R0;
      t.tab[((int64_t)b * NU + i) * 2 + 1] = R1;
    }
  }
}

// Identity segment map (segment i is distinct op list i).
template <int NS>
struct IdMap {
  int v[NS];
  DISTIR_HD constexpr IdMap() : v() {
    for (int i = 0; i < NS; i++) v[i] = i;
  }
};

// Move the cache to binade field ef: per-pass increments copied from the
// table when it covers ef, else computed; then the task's total increments
// from each parity (closed forms of reps_total).
template <int NS>
DISTIR_HD void task_refresh(TaskCache& c, int32_t ef, const Seg (&sg)[NS], const BinTab& t,
                            const int (&map)[NS]) {
  DISTIR_COUNT(2);
  if (ef - t.e0 >= 0 && ef - t.e0 < t.nb) {
    const int64_t* row = t.tab + (int64_t)(ef - t.e0) * t.nu * 2;
#pragma unroll
    for (int i = 0; i < NS; i++) {
      c.R[2 * i] = row[2 * map[i]];
      c.R[2 * i + 1] = row[2 * map[i] + 1];
    }
  } else {
#pragma unroll
    for (int i = 0; i < NS; i++) {
      int64_t R0 = kNeverI, R1 = kNeverI;
      if (sg[i].reps > 0) seg_pass(sg[i].a, sg[i].n, ef, R0, R1);
      c.R[2 * i] = R0;
      c.R[2 * i + 1] = R1;
    }
  }
  int64_t T[2] = {0, 0};
  bool ok = true;
#pragma unroll
  for (int i = 0; i < NS; i++) {
    if (sg[i].reps <= 0) continue;
    const int64_t R0 = c.R[2 * i], R1 = c.R[2 * i + 1];
    if (R0 >= kNeverI) { ok = false; continue; }
#pragma unroll
    for (int p = 0; p < 2; p++) {
      const int pe = p ^ (int)(T[p] & 1);           // parity entering segment i
      const int64_t s = reps_total(R0, R1, pe, sg[i].reps);
      T[p] = s < kNeverI ? T[p] + s : kNeverI;      // (< 2^60: no overflow)
    }
  }
  const double u = bits2d((int64_t)(ef - 52) << 52);
  c.ef = ef;
  c.lo = ef << 20;                // high word of 2^E
  c.hi = (ef + 1) << 20;          // high word of 2^(E+1)
  c.Su0 = (ok && T[0] < kTwo53) ? xmul((double)T[0], u) : kInf();     // exact
  c.Su1 = (ok && T[1] < kTwo53) ? xmul((double)T[1], u) : kInf();
}
template <int NS>
DISTIR_HD void task_refresh(TaskCache& c, int32_t ef, const Seg (&sg)[NS]) {
  constexpr IdMap<NS> id;
  task_refresh(c, ef, sg, BinTab{nullptr, 0, 0, 0}, id.v);
}

// Fast path of a task: when x lies in the cached binade and the whole task
// stays inside it, x <- x + Su (exact) and true; otherwise x is untouched
// and false.  x >= 2^E and x + Su < 2^(E+1) is exactly "x in binade E and
// the rounded sum keeps x's exponent" (Su >= 0; +inf never fits); for
// non-negative doubles both are 32-bit compares of the high words.
// Branch-free (the caller branches once, warp-uniformly, on the rare misses).
DISTIR_HD bool task_fast(double& x, const TaskCache& c) {
  const double Su = (loword(x) & 1) ? c.Su1 : c.Su0;
  const double y = xadd(x, Su);
  const bool ok = hiword(x) >= c.lo && hiword(y) < c.hi;
  x = ok ? y : x;
  return ok;
}
// The same, for a lane that runs the task only when `act`: evaluated
// unconditionally (no divergent branch), applied under `act`; true when the
// task still has to be performed (act and not fast).
#ifndef DISTIR_FAST_LO
#define DISTIR_FAST_LO 0
#endif
DISTIR_HD bool task_fast_or_slow(double& x, const TaskCache& c, bool act) {
  const double Su = (loword(x) & 1) ? c.Su1 : c.Su0;
  const double y = xadd(x, Su);
  // (clocks never decrease and the cache is only ever set for the binade x
  // is in, so with DISTIR_FAST_LO=0 the lower bound is implied)
  const bool ok = act && (!DISTIR_FAST_LO || hiword(x) >= c.lo) && hiword(y) < c.hi;
  x = ok ? y : x;
  return act && !ok;
}

// The common slow case in straight-line code: the task crosses exactly one
// binade boundary (E -> E+1), no segment has ties in E or E+1, and the table
// covers E+1.  Segment j holding the crossing is found from the prefix sums
// of reps * R(E); its whole passes that still fit are added in closed form,
// the crossing pass op by op, and the rest of the task in closed form in
// E+1; the cache then moves to E+1 (its increments from the table).  On any
// other case x is left untouched and false is returned (add_task handles it).
// Cheap pre-check of task_cross1's preconditions (x in the cached binade,
// the table covering the next one).
DISTIR_HD bool cross1_eligible(double x, const TaskCache& c, const BinTab& t) {
  const int32_t ef = exp_field(x);
  return x > 0.0 && ef == c.ef && ef + 1 - t.e0 >= 0 && ef + 1 - t.e0 < t.nb && ef + 1 <= 1993;
}

template <int NS>
DISTIR_HD bool task_cross1(double& x, const Seg (&sg)[NS], TaskCache& c, const BinTab& t,
                           const int (&map)[NS]) {
  const int64_t xb = d2bits(x);
  const int32_t ef = (int32_t)((xb >> 52) & 0x7FF);
  if (!(x > 0.0) || ef != c.ef || ef + 1 > 1993) return false;
  const int32_t b1 = ef + 1 - t.e0;
  if (b1 < 0 || b1 >= t.nb) return false;
  const int64_t* row1 = t.tab + (int64_t)b1 * t.nu * 2;
  const int64_t M = (xb & kMant) | kHidden;
  const int64_t avail = kTwo53 - 1 - M;
  // segment j where the task leaves binade E; C = ulps of the segments before
  int j = -1;
  int64_t C = 0;
  bool ok = true;
#pragma unroll
  for (int i = 0; i < NS; i++) {
    const int64_t r = c.R[2 * i], rb = c.R[2 * i + 1];
    const int64_t r1 = row1[2 * map[i]], r1b = row1[2 * map[i] + 1];
    if (sg[i].reps > 0) {
      ok = ok && r < kNeverI && r == rb && r1 < kNeverI && r1 == r1b;
      if (j < 0) {
        int64_t need = sg[i].reps * r;                // < 2^63 (reps <= 2^10)
        need = need < kTwo53 ? need : kTwo53;         // (C + need cannot overflow)
        if (C + need > avail) j = i; else C += need;
      }
    }
  }
  if (!ok || j < 0) return false;
  // whole passes of segment j that still fit, then the crossing pass
  int64_t rj = 0, nj = 0;
  const double* aj = nullptr;
  int naj = 0;
#pragma unroll
  for (int i = 0; i < NS; i++)
    if (i == j) { rj = c.R[2 * i]; nj = sg[i].reps; aj = sg[i].a; naj = sg[i].n; }
  const int64_t room = avail - C;                     // >= 0, < nj * rj
  int64_t fit = (int64_t)fdiv_approx((float)room, (float)rj);
  if (fit > nj - 1) fit = nj - 1;
  if (fit < 0) fit = 0;
  while (fit > 0 && fit * rj > room) fit--;
  while (fit + 1 < nj && (fit + 1) * rj <= room) fit++;
  double y = bits2d(((int64_t)ef << 52) | ((M + C + fit * rj) & kMant));   // exact, in E
  seq_plain(y, aj, naj);
  const int64_t yb = d2bits(y);
  if ((int32_t)((yb >> 52) & 0x7FF) != ef + 1) { DISTIR_COUNT(25); return false; }
  // the rest of the task in E+1
  int64_t rest = 0, T1 = 0;                           // both capped at 2^53
  auto cap_add = [](int64_t a, int64_t b) { return (a >= kTwo53 || b >= kTwo53) ? kTwo53 : a + b; };
#pragma unroll
  for (int i = 0; i < NS; i++) {
    if (sg[i].reps <= 0) continue;
    const int64_t r1 = row1[2 * map[i]];
    T1 = cap_add(T1, sg[i].reps * r1);
    if (i == j) rest = cap_add(rest, (nj - fit - 1) * r1);
    else if (i > j) rest = cap_add(rest, sg[i].reps * r1);
  }
  const int64_t M1 = (yb & kMant) | kHidden;
  if (M1 + rest > kTwo53 - 1) { DISTIR_COUNT(26); return false; }
  x = bits2d(((int64_t)(ef + 1) << 52) | ((M1 + rest) & kMant));
  // the cache follows x into E+1 (no ties: the total does not depend on parity)
#pragma unroll
  for (int i = 0; i < NS; i++) {
    c.R[2 * i] = row1[2 * map[i]];
    c.R[2 * i + 1] = row1[2 * map[i] + 1];
  }
  bool all = true;
#pragma unroll
  for (int i = 0; i < NS; i++) all = all && (sg[i].reps <= 0 || c.R[2 * i] < kNeverI);
  const double u = bits2d((int64_t)(ef + 1 - 52) << 52);
  c.ef = ef + 1;
  c.lo = (ef + 1) << 20;
  c.hi = (ef + 2) << 20;
  c.Su0 = c.Su1 = (all && T1 < kTwo53) ? xmul((double)T1, u) : kInf();
  return true;
}

// Slow path of a three-segment task p x A + n x B + e x C
// (p, e in {0, 1}; A, B, C the first three lists of the binade table, B the
// repeated one -- a GPT-2 stage: prologue, blocks, epilogue), when the table
// covers x's binade E (and E + 1):
//   (i)  a stale cache -- x moved into E between tasks (a Send) and the whole
//        task fits E: x <- x + its ulps;
//   (ii) one crossing: the passes that fit E in closed form, the pass that
//        leaves E op by op, the rest of the task in closed form in E + 1,
//        which must hold it.
// Ties are handled exactly: a pass adds R0 ulps from an even significand and
// R1 from an odd one, so n passes add the closed form of reps_total and the
// parity after them is the start parity xor the total's low bit.
// Returns false with x untouched in every other case (add_task handles it).
// The cache follows x into its new binade, per-segment increments included
// (segment i is table list i: the identity map).
DISTIR_HD int64_t task3_total(const int64_t* r, int64_t p, int64_t n, int64_t e, int par) {
  // r = {A0, A1, B0, B1, C0, C1} (even / odd start) of one binade; capped at 2^53
  int64_t t = 0;
  if (p) {
    const int64_t a = par ? r[1] : r[0];
    t = a;
    par ^= (int)(a & 1);
  }
  if (n > 0) {
    const int64_t b = reps_total(r[2], r[3], par, n);
    if (b >= kTwo53) return kTwo53;
    t += b;
    par ^= (int)(b & 1);
  }
  if (e) t += par ? r[5] : r[4];
  return t < kTwo53 ? t : kTwo53;
}

#if defined(DISTIR_TIES) && DISTIR_TIES == 2 && defined(__CUDACC__)
__host__ __device__ __noinline__
#else
DISTIR_HD
#endif
bool task3_quick_ties(double& x, const Seg (&sg)[3], TaskCache& c, const BinTab& t) {
  const int64_t xb = d2bits(x);
  const int32_t ef = (int32_t)((xb >> 52) & 0x7FF);
  const int32_t b = ef - t.e0;
  if (!(x > 0.0) || b < 0 || b >= t.nb || ef > 1992) { DISTIR_COUNT(29); return false; }
  const int64_t* r0 = t.tab + (int64_t)b * 6;
  const int64_t p = sg[0].reps, n = sg[1].reps, e = sg[2].reps;
  int64_t q0[6];
#pragma unroll
  for (int i = 0; i < 6; i++) q0[i] = r0[i];
  if (q0[2] >= kNeverI || (p && q0[0] >= kNeverI) || (e && q0[4] >= kNeverI)) {
    DISTIR_COUNT(29);
    return false;
  }
  const int64_t M = (xb & kMant) | kHidden, avail = kTwo53 - 1 - M;
  const int par0 = (int)(M & 1);
  const int64_t tot = task3_total(q0, p, n, e, par0);
  if (tot <= avail) {                                   // (i) the task fits E
    x = bits2d(((int64_t)ef << 52) | ((M + tot) & kMant));
    const double u = bits2d((int64_t)(ef - 52) << 52);
    const int64_t T0 = par0 ? task3_total(q0, p, n, e, 0) : tot;
    const int64_t T1 = par0 ? tot : task3_total(q0, p, n, e, 1);
#pragma unroll
    for (int i = 0; i < 6; i++) c.R[i] = q0[i];
    c.ef = ef;
    c.lo = ef << 20;
    c.hi = (ef + 1) << 20;
    c.Su0 = T0 < kTwo53 ? xmul((double)T0, u) : kInf();
    c.Su1 = T1 < kTwo53 ? xmul((double)T1, u) : kInf();
    return true;
  }
  if (b + 1 >= t.nb) { DISTIR_COUNT(29); return false; }
  const int64_t* r1 = r0 + 6;
  int64_t q1[6];
#pragma unroll
  for (int i = 0; i < 6; i++) q1[i] = r1[i];
  if (q1[2] >= kNeverI || (p && q1[0] >= kNeverI) || (e && q1[4] >= kNeverI)) {
    DISTIR_COUNT(29);
    return false;
  }
  // (ii) the segment that leaves E: A (from x), B (the passes that still fit,
  // then one) or C (after A and every B pass); that pass is walked op by op
  // from the exact value where it starts, the rest of the task (B passes
  // left, C) is added in E + 1 from the parity the walk ends on
  int par = par0;
  int64_t Cp = 0;
  if (p) {
    Cp = par ? q0[1] : q0[0];
    par ^= (int)(Cp & 1);
  }
  int64_t pre, nrest, erest;
  const double* a;
  int na;
  if (Cp > avail) {                                           // crossing in A
    pre = 0; a = sg[0].a; na = sg[0].n;
    nrest = n; erest = e;
  } else {
    const int64_t room = avail - Cp;
    const int64_t CB = reps_total(q0[2], q0[3], par, n);     // capped (kNeverI)
    if (CB > room) {                                          // crossing in B
      // passes add Ra, then (Ra odd) Rb, ...: cum(j) below; fit = the most
      // whole passes (< n) with cum(fit) <= room
      const int64_t Ra = par ? q0[3] : q0[2], Rb = par ? q0[2] : q0[3];
      const int kind = !(Ra & 1) ? 0 : (!(Rb & 1) ? 1 : 2);
      auto cum = [&](int64_t j) -> int64_t {                  // j <= 2^10: no overflow
        if (j <= 0) return 0;
        if (kind == 0) return j * Ra;
        if (kind == 1) return Ra + (j - 1) * Rb;
        return ((j + 1) >> 1) * Ra + (j >> 1) * Rb;
      };
      const float avg = kind == 0 ? (float)Ra : kind == 1 ? (float)Rb : 0.5f * ((float)Ra + (float)Rb);
      int64_t fit = avg > 0.0f ? (int64_t)fdiv_approx((float)room, avg) : n - 1;
      fit = fit < 0 ? 0 : (fit > n - 1 ? n - 1 : fit);
      while (fit > 0 && cum(fit) > room) fit--;
      while (fit + 1 < n && cum(fit + 1) <= room) fit++;
      pre = Cp + cum(fit); a = sg[1].a; na = sg[1].n;
      nrest = n - fit - 1; erest = e;
    } else {                                                  // crossing in C
      pre = Cp + CB; a = sg[2].a; na = sg[2].n;
      nrest = 0; erest = 0;
    }
  }
  double y = bits2d(((int64_t)ef << 52) | ((M + pre) & kMant));   // exact, in E
  {
    double v[kSegMax];
#pragma unroll
    for (int j = 0; j < kSegMax; j++) v[j] = j < na ? a[j] : 0.0;   // loads first
#pragma unroll
    for (int j = 0; j < kSegMax; j++)
      if (j < na) y = xadd(y, v[j]);
  }
  const int64_t yb = d2bits(y);
  if ((int32_t)((yb >> 52) & 0x7FF) != ef + 1) { DISTIR_COUNT(29); return false; }
  const int64_t M1 = (yb & kMant) | kHidden;
  const int64_t rest = task3_total(q1, 0, nrest, erest, (int)(M1 & 1));
  if (M1 + rest > kTwo53 - 1) { DISTIR_COUNT(29); return false; }
  x = bits2d(((int64_t)(ef + 1) << 52) | ((M1 + rest) & kMant));
  const double u1 = bits2d((int64_t)(ef + 1 - 52) << 52);
  const int64_t T0 = task3_total(q1, p, n, e, 0), T1 = task3_total(q1, p, n, e, 1);
#pragma unroll
  for (int i = 0; i < 6; i++) c.R[i] = q1[i];
  c.ef = ef + 1;
  c.lo = (ef + 1) << 20;
  c.hi = (ef + 2) << 20;
  c.Su0 = T0 < kTwo53 ? xmul((double)T0, u1) : kInf();
  c.Su1 = T1 < kTwo53 ? xmul((double)T1, u1) : kInf();
  return true;
}

// The no-tie case in straight-line code: 1 when done, 2 when a list has a tie
// in E (or, crossing, in E + 1) -- task3_quick_ties then applies -- and 0
// otherwise (x untouched in both).
DISTIR_HD int task3_quick(double& x, const Seg (&sg)[3], TaskCache& c, const BinTab& t) {
  const int64_t xb = d2bits(x);
  const int32_t ef = (int32_t)((xb >> 52) & 0x7FF);
  const int32_t b = ef - t.e0;
  if (!(x > 0.0) || b < 0 || b >= t.nb || ef > 1992) { DISTIR_COUNT(21); return 0; }
  const int64_t* r0 = t.tab + (int64_t)b * 6;
  const int64_t A0 = r0[0], A0b = r0[1], B0 = r0[2], B0b = r0[3], C0 = r0[4], C0b = r0[5];
  const int64_t p = sg[0].reps, n = sg[1].reps, e = sg[2].reps;
  if (!(B0 == B0b && B0 < kNeverI && (!p || (A0 == A0b && A0 < kNeverI)) &&
        (!e || (C0 == C0b && C0 < kNeverI)))) {
    DISTIR_COUNT(22);
    return 2;
  }
  // (products saturate at 2^53: n <= 2^10 and increments < 2^53, so n * B
  // fits int64 and saturated sums cannot overflow)
  auto sat = [](int64_t v) { return v > kTwo53 ? kTwo53 : v; };
  const int64_t M = (xb & kMant) | kHidden, avail = kTwo53 - 1 - M;
  const int64_t Cp = p * A0, CpB = Cp + sat(n * B0);
  const int64_t tot = CpB + e * C0;
  if (tot <= avail) {                                   // (i) the task fits E
    x = bits2d(((int64_t)ef << 52) | ((M + tot) & kMant));
    c.R[0] = A0; c.R[1] = A0b; c.R[2] = B0; c.R[3] = B0b; c.R[4] = C0; c.R[5] = C0b;
    c.ef = ef;
    c.lo = ef << 20;
    c.hi = (ef + 1) << 20;
    c.Su0 = c.Su1 = xmul((double)tot, bits2d((int64_t)(ef - 52) << 52));
    return 1;
  }
  if (b + 1 >= t.nb) { DISTIR_COUNT(23); return 0; }
  const int64_t* r1 = r0 + 6;
  const int64_t A1 = r1[0], A1b = r1[1], B1 = r1[2], B1b = r1[3], C1 = r1[4], C1b = r1[5];
  if (!(B1 == B1b && B1 < kNeverI && (!p || (A1 == A1b && A1 < kNeverI)) &&
        (!e || (C1 == C1b && C1 < kNeverI)))) {
    DISTIR_COUNT(24);
    return 2;
  }
  // (ii) the segment that leaves E: A (whole task from x), B (the passes that
  // still fit, then one), or C (after A and every B pass); that pass is walked
  // op by op from the exact value where it starts, the rest of the task is
  // added in E + 1
  int64_t pre, rest;
  const double* a;
  int na;
  if (Cp > avail) {                                           // crossing in A
    pre = 0; a = sg[0].a; na = sg[0].n;
    rest = sat(n * B1) + e * C1;
  } else if (CpB > avail) {                                   // crossing in B
    // fit = floor(room / B0) < n: estimate (relative error ~2^-21, fit <
    // 2^10), corrected exactly
    const int64_t room = avail - Cp;
    int64_t fit = (int64_t)fdiv_approx((float)room, (float)B0);
    fit = fit < 0 ? 0 : (fit > n - 1 ? n - 1 : fit);
    if (fit * B0 > room) fit--;
    if (fit + 1 < n && (fit + 1) * B0 <= room) fit++;
    pre = Cp + fit * B0; a = sg[1].a; na = sg[1].n;
    rest = sat((n - fit - 1) * B1) + e * C1;
  } else {                                                    // crossing in C
    pre = CpB; a = sg[2].a; na = sg[2].n;
    rest = 0;
  }
  double y = bits2d(((int64_t)ef << 52) | ((M + pre) & kMant));   // exact, in E
  {
    double v[kSegMax];
#pragma unroll
    for (int j = 0; j < kSegMax; j++) v[j] = j < na ? a[j] : 0.0;   // loads first
#pragma unroll
    for (int j = 0; j < kSegMax; j++)
      if (j < na) y = xadd(y, v[j]);
  }
  const int64_t yb = d2bits(y);
  if ((int32_t)((yb >> 52) & 0x7FF) != ef + 1) { DISTIR_COUNT(25); return 0; }
  const int64_t M1 = (yb & kMant) | kHidden;
  if (M1 + rest > kTwo53 - 1) { DISTIR_COUNT(26); return 0; }
  x = bits2d(((int64_t)(ef + 1) << 52) | ((M1 + rest) & kMant));
  const int64_t tot1 = p * A1 + sat(n * B1) + e * C1;
  c.R[0] = A1; c.R[1] = A1b; c.R[2] = B1; c.R[3] = B1b; c.R[4] = C1; c.R[5] = C1b;
  c.ef = ef + 1;
  c.lo = (ef + 1) << 20;
  c.hi = (ef + 2) << 20;
  c.Su0 = c.Su1 = tot1 < kTwo53 ? xmul((double)tot1, bits2d((int64_t)(ef + 1 - 52) << 52)) : kInf();
  return 1;
}

// Point a three-segment task cache at x's binade from the table (no add):
// after a task walked op by op, so the next task takes the fast path.  The
// cache is left as it was (stale: the next task re-enters the slow path) when
// the table does not cover the binade or a list has ties there.
DISTIR_HD void task3_cache_to(double x, const Seg (&sg)[3], TaskCache& c, const BinTab& t) {
  const int32_t ef = exp_field(x);
  const int32_t b = ef - t.e0;
  if (!(x > 0.0) || b < 0 || b >= t.nb || ef > 1992) return;
  const int64_t* r0 = t.tab + (int64_t)b * 6;
  const int64_t A0 = r0[0], A0b = r0[1], B0 = r0[2], B0b = r0[3], C0 = r0[4], C0b = r0[5];
  const int64_t p = sg[0].reps, n = sg[1].reps, e = sg[2].reps;
  if (!(B0 == B0b && B0 < kNeverI && (!p || (A0 == A0b && A0 < kNeverI)) &&
        (!e || (C0 == C0b && C0 < kNeverI))))
    return;
  auto sat = [](int64_t v) { return v > kTwo53 ? kTwo53 : v; };
  const int64_t tot = p * A0 + sat(n * B0) + e * C0;
  c.R[0] = A0; c.R[1] = A0b; c.R[2] = B0; c.R[3] = B0b; c.R[4] = C0; c.R[5] = C0b;
  c.ef = ef;
  c.lo = ef << 20;
  c.hi = (ef + 1) << 20;
  c.Su0 = c.Su1 = tot < kTwo53 ? xmul((double)tot, bits2d((int64_t)(ef - 52) << 52)) : kInf();
}

// The same straight-line slow path for a task of NS segments read through a
// segment map (the MLP kernels' forward / backward tasks): (i) a stale cache
// -- the whole task fits x's binade E; (ii) one crossing -- the segments and
// passes that fit E in closed form, the pass that leaves E op by op, the rest
// of the task in closed form in E + 1.  No ties in the lists it uses (else
// 2, add_task handles them), the table covering E (and E + 1); 0 in every
// other case; x untouched unless 1.
template <int NS>
DISTIR_HD int taskN_quick(double& x, const Seg (&sg)[NS], TaskCache& c, const BinTab& t,
                          const int (&map)[NS]) {
  const int64_t xb = d2bits(x);
  const int32_t ef = (int32_t)((xb >> 52) & 0x7FF);
  const int32_t b = ef - t.e0;
  if (!(x > 0.0) || b < 0 || b >= t.nb || ef > 1992) return 0;
  const int64_t* r0 = t.tab + (int64_t)b * t.nu * 2;
  auto sat = [](int64_t v) { return v > kTwo53 ? kTwo53 : v; };
  int64_t R[NS];
  int64_t tot = 0;
  bool tie = false;
#pragma unroll
  for (int i = 0; i < NS; i++) {
    const int64_t a0 = r0[2 * map[i]], a1 = r0[2 * map[i] + 1];
    R[i] = a0;
    if (sg[i].reps > 0) {
      tie |= a0 != a1 || a0 >= kNeverI;
      tot = sat(tot + sat(sg[i].reps * (a0 < kNeverI ? a0 : kTwo53)));
    }
  }
  if (tie) return 2;
  const int64_t M = (xb & kMant) | kHidden, avail = kTwo53 - 1 - M;
  if (tot <= avail) {                                   // (i) the task fits E
    x = bits2d(((int64_t)ef << 52) | ((M + tot) & kMant));
#pragma unroll
    for (int i = 0; i < NS; i++) { c.R[2 * i] = R[i]; c.R[2 * i + 1] = R[i]; }
    c.ef = ef;
    c.lo = ef << 20;
    c.hi = (ef + 1) << 20;
    c.Su0 = c.Su1 = xmul((double)tot, bits2d((int64_t)(ef - 52) << 52));
    return 1;
  }
  if (b + 1 >= t.nb) return 0;
  const int64_t* r1 = r0 + t.nu * 2;
  int64_t R1[NS];
  int64_t tot1 = 0;
#pragma unroll
  for (int i = 0; i < NS; i++) {
    const int64_t a0 = r1[2 * map[i]], a1 = r1[2 * map[i] + 1];
    R1[i] = a0;
    if (sg[i].reps > 0) {
      tie |= a0 != a1 || a0 >= kNeverI;
      tot1 = sat(tot1 + sat(sg[i].reps * (a0 < kNeverI ? a0 : kTwo53)));
    }
  }
  if (tie) return 2;
  // the segment j that leaves E, the passes of it that still fit
  int64_t pre = 0, rest = 0, fitj = 0;
  int j = -1;
  const double* aj = nullptr;
  int naj = 0;
#pragma unroll
  for (int i = 0; i < NS; i++) {
    if (sg[i].reps <= 0) continue;
    if (j < 0) {
      const int64_t need = sat(sg[i].reps * R[i]);
      if (pre + need <= avail) { pre += need; continue; }
      const int64_t room = avail - pre;
      int64_t fit = R[i] > 0 ? (int64_t)fdiv_approx((float)room, (float)R[i]) : sg[i].reps - 1;
      fit = fit < 0 ? 0 : (fit > sg[i].reps - 1 ? sg[i].reps - 1 : fit);
      if (fit * R[i] > room) fit--;
      if (fit + 1 < sg[i].reps && (fit + 1) * R[i] <= room) fit++;
      j = i;
      fitj = fit;
      pre += fit * R[i];
      aj = sg[i].a;
      naj = sg[i].n;
      rest = sat((sg[i].reps - fit - 1) * R1[i]);
    } else {
      rest = sat(rest + sat(sg[i].reps * R1[i]));
    }
  }
  (void)fitj;
  if (j < 0) return 0;
  double y = bits2d(((int64_t)ef << 52) | ((M + pre) & kMant));   // exact, in E
  {
    double v[kSegMax];
#pragma unroll
    for (int q = 0; q < kSegMax; q++) v[q] = q < naj ? aj[q] : 0.0;
#pragma unroll
    for (int q = 0; q < kSegMax; q++)
      if (q < naj) y = xadd(y, v[q]);
  }
  const int64_t yb = d2bits(y);
  if ((int32_t)((yb >> 52) & 0x7FF) != ef + 1) return 0;
  const int64_t M1 = (yb & kMant) | kHidden;
  if (M1 + rest > kTwo53 - 1) return 0;
  x = bits2d(((int64_t)(ef + 1) << 52) | ((M1 + rest) & kMant));
#pragma unroll
  for (int i = 0; i < NS; i++) { c.R[2 * i] = R1[i]; c.R[2 * i + 1] = R1[i]; }
  c.ef = ef + 1;
  c.lo = (ef + 1) << 20;
  c.hi = (ef + 2) << 20;
  c.Su0 = c.Su1 = tot1 < kTwo53 ? xmul((double)tot1, bits2d((int64_t)(ef + 1 - 52) << 52)) : kInf();
  return 1;
}

// Any task walked op by op (short tasks: cheaper than any table lookup).
template <int NS>
DISTIR_HD void taskN_plain(double& x, const Seg (&sg)[NS]) {
#pragma unroll
  for (int i = 0; i < NS; i++)
    for (int64_t r = 0; r < sg[i].reps; r++) seq_plain(x, sg[i].a, sg[i].n);
}

// A three-segment task (as task3_quick) walked op by op -- for a clock at
// zero (stage 0's first task), where the sum climbs through many binades:
// the repeated segment's costs are held in registers.
DISTIR_HD void task3_plain(double& x, const Seg (&sg)[3]) {
  for (int64_t r = 0; r < sg[0].reps; r++) seq_plain(x, sg[0].a, sg[0].n);
  double v[kSegMax];
#pragma unroll
  for (int j = 0; j < kSegMax; j++) v[j] = j < sg[1].n ? sg[1].a[j] : 0.0;
  for (int64_t r = 0; r < sg[1].reps; r++) {
#pragma unroll
    for (int j = 0; j < kSegMax; j++)
      if (j < sg[1].n) x = xadd(x, v[j]);
  }
  for (int64_t r = 0; r < sg[2].reps; r++) seq_plain(x, sg[2].a, sg[2].n);
}

// x <- every addition of the task, in order, computed exactly: the cache is
// moved to x's binade and the fast path retried; otherwise each segment
// advances by whole passes while they fit (closed form, or a short parity
// walk when the binade has ties), the pass that leaves the binade is done op
// by op, and the cache follows x into the new binade.
template <int NS>
DISTIR_HD_COLD void add_task(double& x, const Seg (&sg)[NS], TaskCache& c, const BinTab& t,
                             const int (&map)[NS], int plain_after = DISTIR_PLAIN_AFTER) {
  DISTIR_COUNT(0);
  const long long t_all = DISTIR_CLK_NOW();
  // a task that spans several binades (a clock starting at zero, a
  // single-stage configuration's tasks) is cheaper op by op than binade by
  // binade: from a zero clock or after `plain_after` crossings (0: never),
  // walk it plainly
  if (plain_after > 0 && x == 0.0) {
#pragma unroll
    for (int i = 0; i < NS; i++)
      for (int64_t r = 0; r < sg[i].reps; r++) seq_plain(x, sg[i].a, sg[i].n);
    DISTIR_CLK_ADD(15, t_all);
    return;
  }
  int crossings = 0;
  {
    const int32_t ef = exp_field(x);
    if (x > 0.0 && ef >= 53 && ef <= 1993) {
      if (ef != c.ef) {
        const long long t0 = DISTIR_CLK_NOW();
        task_refresh(c, ef, sg, t, map);
        DISTIR_CLK_ADD(12, t0);
      }
      if (task_fast(x, c)) { DISTIR_COUNT(1); DISTIR_CLK_ADD(15, t_all); return; }
    }
  }
#pragma unroll
  for (int i = 0; i < NS; i++) {
    int64_t reps = sg[i].reps;
    if (plain_after > 0 && crossings >= plain_after) {
      for (; reps > 0; reps--) seq_plain(x, sg[i].a, sg[i].n);
      continue;
    }
    while (reps > 0) {
      const int64_t xb = d2bits(x);
      const int32_t ef = (int32_t)((xb >> 52) & 0x7FF);
      if (x > 0.0 && ef >= 53 && ef <= 1993) {
        if (ef != c.ef) {
          const long long t0 = DISTIR_CLK_NOW();
          task_refresh(c, ef, sg, t, map);
          DISTIR_CLK_ADD(12, t0);
        }
        const int64_t r0 = c.R[2 * i], r1 = c.R[2 * i + 1];
        if (r0 < kNeverI) {
          int64_t M = (xb & kMant) | kHidden;
          const int64_t before = reps;
          if (r0 == r1) {                            // no tie: closed form
            const int64_t avail = kTwo53 - 1 - M;
            int64_t fit = reps;                      // min(reps, avail / r0)
            if (r0 > 0 && reps * r0 > avail) {       // (reps <= 2^10, r0 < 2^53)
              // estimate (relative error ~2^-21, fit < reps <= 2^10), corrected below
              fit = (int64_t)fdiv_approx((float)avail, (float)r0);
              if (fit > reps) fit = reps;
              if (fit < 0) fit = 0;
            }
            while (fit > 0 && fit * r0 > avail) fit--;
            while (fit < reps && (fit + 1) * r0 <= avail) fit++;
            M += fit * r0;
            reps -= fit;
          } else {                                   // ties: walk the parity
            int p = (int)(M & 1);
            while (reps > 0) {
              const int64_t r = p ? r1 : r0;
              if (M + r > kTwo53 - 1) break;
              M += r;
              p ^= (int)(r & 1);
              reps--;
            }
          }
          if (reps != before) x = bits2d(((int64_t)ef << 52) | (M & kMant));   // exact
        }
      }
      if (reps > 0) {                                // the crossing pass
        DISTIR_COUNT(3);
        const long long t0 = DISTIR_CLK_NOW();
        seq_plain(x, sg[i].a, sg[i].n);
        DISTIR_CLK_ADD(13, t0);
        reps--;
        if (plain_after > 0 && ++crossings >= plain_after)
          for (; reps > 0; reps--) seq_plain(x, sg[i].a, sg[i].n);
      }
    }
  }
  DISTIR_CLK_ADD(15, t_all);
}

template <int NS>
DISTIR_HD_COLD void add_task(double& x, const Seg (&sg)[NS], TaskCache& c) {
  constexpr IdMap<NS> id;
  add_task(x, sg, c, BinTab{nullptr, 0, 0, 0}, id.v);
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
