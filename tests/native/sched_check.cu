// Host-side check of the cost-balanced stream-K schedule (Sched in
// paper_2203_08263_b200/csrc/nbody_common.cuh), run by tests/test_schedule.py on
// the CPU: for many (units, grid, i-blocks, groups) it verifies that start() is
// monotone and covers [0, units) exactly, that every CTA owns >= 1 unit when the
// grid is capped to cost/kg (as launch_step does), that cta_of() inverts
// start(), that the per-CTA cost stays within one unit of the fair share, and
// that lg == kg reproduces the equal-units split c*units/grid.
#include <cstdio>
#include <cstdlib>

#include "nbody_common.cuh"

void nb::count_launch(int) {}

static int fail(const char* what, long long a, long long b, long long c) {
  std::printf("FAIL %s (%lld %lld %lld)\n", what, a, b, c);
  return 1;
}

int main() {
  long long checked = 0;
  for (int64_t nib = 1; nib <= 40; nib += (nib < 12 ? 1 : 7)) {
    for (int64_t nt : {1, 2, 3, 7, 16, 64, 1024, 8192}) {
      for (int kg = 1; kg <= 3; ++kg) {
        for (int lg = 1; lg <= kg; ++lg) {
          for (int64_t grid0 : {1, 2, 5, 11, 37, 148, 296, 1000}) {
            const int64_t units = nib * nt;
            nb::Sched S = nb::Sched::make(units, 1, nt, nib, kg, lg);
            int64_t grid = grid0 < S.cost / kg ? grid0 : S.cost / kg;
            if (grid < 1) grid = 1;
            S = nb::Sched::make(units, grid, nt, nib, kg, lg);
            if (S.start(0) != 0) return fail("start(0)", units, grid, 0);
            if (S.start(grid) != units) return fail("start(grid)", units, grid, S.start(grid));
            const double fair = (double)S.cost / grid;
            for (int64_t c = 0; c < grid; ++c) {
              const int64_t a = S.start(c), b = S.start(c + 1);
              if (b <= a) return fail("empty CTA", units, grid, c);
              const int64_t cost = S.pos(b) - S.pos(a);
              if (cost > fair + kg || cost < fair - kg) return fail("unbalanced", units, grid, c);
              for (int64_t u = a; u < b; u += (b - a > 64 ? (b - a) / 16 : 1))
                if (S.cta_of(u) != c) return fail("cta_of", units, grid, u);
              if (S.cta_of(b - 1) != c) return fail("cta_of(last)", units, grid, c);
              if (lg == kg && a != c * units / grid) return fail("equal split", units, grid, c);
            }
            ++checked;
          }
        }
      }
    }
  }
  std::printf("ok %lld schedules\n", checked);
  return 0;
}
