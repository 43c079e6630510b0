// Host check of the product's exact aggregation (paper_2111_05426_b200/csrc/
// exact_add.cuh): add_task(x, segments) must equal every plain IEEE addition
// of the task, in order, bit for bit -- over random, tie-heavy dyadic and
// zero costs, clocks starting at zero or anywhere, binade crossings, a
// cache reused across tasks, with and without a precomputed binade table,
// including the GPT-2 kernels' quick / plain slow paths -- and MemProf composition must equal the
// op-by-op live/peak walk.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
static long g_cnt[32];
static long g_quickN_ok = 0;
#define DISTIR_COUNT(i) (g_cnt[i]++)
#include "../../paper_2111_05426_b200/csrc/exact_add.cuh"

using namespace distir;

static double draw_cost(std::mt19937_64& g, int mode) {
  std::uniform_real_distribution<double> U(0.0, 1.0);
  if (mode == 0) return std::ldexp(U(g), -(int)(g() % 40));                       // messy
  if (mode == 1) return (double)(g() % 64) * std::ldexp(1.0, -20 - (int)(g() % 12));  // ties
  return (g() % 4 == 0) ? 0.0 : std::ldexp(1.0 + (double)(g() % 8) / 8, -(int)(g() % 30));
}

template <int NS>
static long check(std::mt19937_64& g, int trials, int mode) {
  long bad = 0;
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (int t = 0; t < trials; t++) {
    double store[NS][14];
    Seg sg[NS];
    for (int i = 0; i < NS; i++) {
      const int n = 1 + (int)(g() % 14);
      for (int j = 0; j < n; j++) store[i][j] = draw_cost(g, mode);
      sg[i] = Seg{store[i], n, (g() % 5 == 0) ? 0 : 1 + (int64_t)(g() % ((g() & 7) ? 200 : 1024))};
    }
    double x = (g() % 5 == 0) ? 0.0 : std::ldexp(U(g), -(int)(g() % 30));
    double y = x;
    int64_t cstore[2 * NS];
    TaskCache c = task_cache_make(cstore);
    // half of the trials use a binade table (BinTab) covering a random range
    // around the clocks; binades outside it fall back to the lane's storage
    // (the table holds the segments' op lists in reverse order, read back
    // through a segment map)
    static int64_t tstore[64 * 2 * NS];
    BinTab tb{tstore, 0, 0, NS};
    int map[NS];
    Seg rev[NS];
    for (int i = 0; i < NS; i++) { map[i] = NS - 1 - i; rev[NS - 1 - i] = sg[i]; }
    if (g() & 1) {
      tb.e0 = 1023 - 45 + (int)(g() % 40);
      tb.nb = 1 + (int)(g() % 64);
      bintab_fill(tb, rev, 0, 1);
    }
    const int tasks = 1 + (int)(g() % 40);
    for (int k = 0; k < tasks; k++) {
      for (int i = 0; i < NS; i++)
        for (int64_t r = 0; r < sg[i].reps; r++)
          for (int j = 0; j < sg[i].n; j++) x = x + sg[i].a[j];
      // as the kernels do: fast path, else the straight-line quick path
      // (or the single-crossing path), else add_task
      if ((g() & 1) || !task_fast(y, c)) {
        if (g() & 1) {
          if (taskN_quick(y, sg, c, tb, map) == 1) g_quickN_ok++;
          else add_task(y, sg, c, tb, map, (int)(g() % 3));
        } else if (!(g() & 3) || !task_cross1(y, sg, c, tb, map)) {
          add_task(y, sg, c, tb, map, (int)(g() % 3));
        }
      }
      if (std::memcmp(&x, &y, 8) != 0) {
        if (bad < 5) std::printf("mismatch NS=%d mode=%d task=%d plain=%a agg=%a\n", NS, mode, k, x, y);
        bad++;
        break;
      }
    }
  }
  return bad;
}

// The GPT-2 kernels' slow-path order (simulate.cuh run_gpt2): a task of
// prologue (0/1 pass) + blocks (n passes) + epilogue (0/1 pass) with an
// identity-map binade table; fast path, else op by op from a zero clock,
// else task3_quick, else op by op (short tasks) or add_task.
static long g_quick_ok = 0, g_ties_ok = 0;
static long check_gpt2(std::mt19937_64& g, int trials, int mode) {
  long bad = 0;
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (int t = 0; t < trials; t++) {
    double store[3][14];
    Seg sg[3];
    const int ns[3] = {2, 14, 3};
    for (int i = 0; i < 3; i++) {
      for (int j = 0; j < ns[i]; j++) store[i][j] = draw_cost(g, mode);
      sg[i] = Seg{store[i], ns[i], i == 1 ? 1 + (int64_t)(g() % ((g() & 3) ? 48 : 1024))
                                          : (int64_t)(g() & 1)};
    }
    double x = (g() % 5 == 0) ? 0.0 : std::ldexp(U(g), -(int)(g() % 30));
    double y = x;
    int64_t cstore[6];
    TaskCache c = task_cache_make(cstore);
    static int64_t tstore[64 * 6];
    BinTab tb{tstore, 0, 0, 3};
    const int map[3] = {0, 1, 2};
    if (g() % 8) {
      tb.e0 = 1023 - 45 + (int)(g() % 40);
      tb.nb = 1 + (int)(g() % 24);
      bintab_fill(tb, sg, 0, 1);
    }
    const int tasks = 1 + (int)(g() % 60);
    for (int k = 0; k < tasks; k++) {
      for (int i = 0; i < 3; i++)
        for (int64_t r = 0; r < sg[i].reps; r++)
          for (int j = 0; j < sg[i].n; j++) x = x + sg[i].a[j];
      if (task_fast_or_slow(y, c, true)) {
        int r;
        if (y == 0.0) task3_plain(y, sg);
        else if (!(g() & 3) && task3_quick_ties(y, sg, c, tb)) g_ties_ok++;   // also without ties
        else if ((r = task3_quick(y, sg, c, tb)) == 1) g_quick_ok++;
        else if (r == 2 && task3_quick_ties(y, sg, c, tb)) g_ties_ok++;
        else if (g() & 1) task3_plain(y, sg);
        else add_task(y, sg, c, tb, map);
      }
      if (std::memcmp(&x, &y, 8) != 0) {
        if (bad < 5) std::printf("gpt2 mismatch mode=%d task=%d plain=%a agg=%a\n", mode, k, x, y);
        bad++;
        break;
      }
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
    bad += check<4>(g, trials, mode);
    bad += check_gpt2(g, 2 * trials, mode);
  }
  bad += check_mem(g, trials * 5);
  std::printf("task3_quick_ties: %ld taken, taskN_quick: %ld taken\n", g_ties_ok, g_quickN_ok);
  std::printf("task3_quick: %ld taken; misses: outside table %ld, never-fitting lists %ld / %ld, "
              "crossing beyond E+1 %ld, rest beyond E+1 %ld\n", g_quick_ok, g_cnt[21], g_cnt[22],
              g_cnt[24], g_cnt[25], g_cnt[26]);
  std::printf("bad=%ld\n", bad);
  return bad ? 1 : 0;
}
