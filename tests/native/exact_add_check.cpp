// Host check of the product's exact aggregation (paper_2111_05426_b200/csrc/
// exact_add.cuh): add_reps(x, a, n) must equal n*N plain IEEE additions bit
// for bit, and MemProf composition must equal the op-by-op live/peak walk.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include "../../paper_2111_05426_b200/csrc/exact_add.cuh"

using namespace distir;

template <int N>
static long check(std::mt19937_64& g, int trials, int mode) {
  long bad = 0;
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (int t = 0; t < trials; t++) {
    double a[N];
    for (int j = 0; j < N; j++) {
      if (mode == 0) a[j] = std::ldexp(U(g), -(int)(g() % 40));          // messy costs
      else if (mode == 1) a[j] = (double)(g() % 64) * std::ldexp(1.0, -20 - (int)(g() % 12));  // dyadic: ties
      else a[j] = (g() % 4 == 0) ? 0.0 : std::ldexp(1.0 + (double)(g() % 8) / 8, -(int)(g() % 30));
    }
    double x0 = (g() % 5 == 0) ? 0.0 : std::ldexp(U(g), -(int)(g() % 30));
    const long reps = 1 + (long)(g() % 3000);
    double x = x0;
    for (long r = 0; r < reps; r++)
      for (int j = 0; j < N; j++) x = x + a[j];
    double y = x0;
    SeqCache c = seq_cache_empty();
    long left = reps;
    while (left > 0) {            // split into uneven chunks sharing one cache
      long chunk = 1 + (long)(g() % (left + 1));
      if (chunk > left) chunk = left;
      add_reps(y, a, chunk, c);
      left -= chunk;
    }
    if (std::memcmp(&x, &y, 8) != 0) {
      if (bad < 5) std::printf("mismatch N=%d mode=%d x0=%a reps=%ld plain=%a agg=%a\n", N, mode, x0, reps, x, y);
      bad++;
    }
  }
  return bad;
}

static long check_mem(std::mt19937_64& g, int trials) {
  long bad = 0;
  for (int t = 0; t < trials; t++) {
    const int n = 1 + (int)(g() % 12);
    int64_t al[12], fr[12];
    for (int j = 0; j < n; j++) { al[j] = (int64_t)(g() % 1000); fr[j] = (int64_t)(g() % 1000); }
    const int64_t reps = (int64_t)(g() % 50);
    int64_t live = 5000 + (int64_t)(g() % 1000), peak = live;
    int64_t l2 = live, p2 = peak;
    for (int64_t r = 0; r < reps; r++)
      for (int j = 0; j < n; j++) { live += al[j]; peak = peak > live ? peak : live; live -= fr[j]; }
    MemProf p = mem_id();
    for (int j = 0; j < n; j++) p = mem_then(p, mem_op(al[j], fr[j]));
    mem_apply(l2, p2, mem_rep(p, reps));
    if (live != l2 || peak != p2) bad++;
  }
  return bad;
}

int main(int argc, char** argv) {
  const int trials = argc > 1 ? std::atoi(argv[1]) : 2000;
  std::mt19937_64 g(20211105426ull);
  long bad = 0;
  for (int mode = 0; mode < 3; mode++) {
    bad += check<1>(g, trials, mode);
    bad += check<2>(g, trials, mode);
    bad += check<3>(g, trials, mode);
    bad += check<6>(g, trials, mode);
    bad += check<14>(g, trials, mode);
  }
  bad += check_mem(g, trials * 5);
  std::printf("bad=%ld\n", bad);
  return bad ? 1 : 0;
}
