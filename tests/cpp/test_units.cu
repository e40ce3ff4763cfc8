// Host-side checks of the exact kernel's work partition (bl_kernel.cuh
// __host__ __device__ helpers), compiled with nvcc and run on the CPU by
// tests/test_host_logic.py (no GPU needed):
//  * bl_geom: the dirty slots [d_lo, d_hi) cover exactly the float4 slots of
//    the owned sources k_lo .. k_lo+owned-1, clean4 = last4 - (d_hi - d_lo);
//  * bl_units: ntt tiles of 32 T targets cover bt; ntt * 32 T * nsub fits red
//    when nsub > 1; nsub <= nsub_max; one dirty sub-range iff dirty;
//  * bl_guided_start: starts are non-decreasing, start(0) = 0, start(nc) = L
//    (the clean sub-ranges tile [0, L) exactly), sizes non-increasing for the
//    linear and quadratic profiles, equal (+-1) for the uniform one.
#include <cstdio>
#include <cstdlib>

#include "bl_kernel.cuh"

static int fails = 0;
#define CHECK(c, ...)                          \
  do {                                         \
    if (!(c)) {                                \
      ++fails;                                 \
      if (fails < 20) {                        \
        std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
        std::printf(__VA_ARGS__);              \
        std::printf("\n");                     \
      }                                        \
    }                                          \
  } while (0)

int main() {
  const int Gs[] = {148, 132, 7};
  const int ns[] = {1, 2, 3, 1000, 6000, 11000, 32768, 262144, 1048576};
  for (int G : Gs)
    for (int n : ns)
      for (int c = 0; c < G; c += (G > 20 ? 13 : 1)) {
        const int m_c = c < n ? (n - 1 - c) / G + 1 : 0;
        for (int k_lo = 0; k_lo < m_c; k_lo += (m_c > 50 ? m_c / 7 + 1 : 1))
          for (int owned : {0, 1, 2, 7, 64}) {
            if (owned > 0 && k_lo + owned > m_c) continue;
            const BLGeom g = bl_geom(c, G, n, k_lo, owned);
            CHECK(g.full4 == m_c / 2 && g.last4 == (m_c + 1) / 2, "geom n=%d c=%d", n, c);
            if (owned == 0) {
              CHECK(g.d_lo == g.d_hi && g.clean4 == g.last4, "no dirty n=%d", n);
            } else {
              CHECK(g.d_lo == k_lo / 2 && g.d_hi == (k_lo + owned - 1) / 2 + 1,
                    "dirty slots n=%d c=%d k=%d o=%d: [%d,%d)", n, c, k_lo, owned, g.d_lo, g.d_hi);
              CHECK(g.clean4 == g.last4 - (g.d_hi - g.d_lo), "clean4");
            }
          }
      }
  for (int T : {2, 4, 6, 8, 16})
    for (int bt : {1, 31, 32, 255, 256, 257, 1000, 1024, 2048})
      for (int clean4 : {0, 1, 15, 16, 100, 886, 3543})
        for (int dirty = 0; dirty < 2; ++dirty)
          for (int red_cap : {4096, 6144, 12288, 16384})
            for (int nmax : {2, 6, 32}) {
              // precondition of a dirty context (both one-barrier drivers check
              // it on the host): red holds two sub-ranges of every tile
              const int tiles = (bt + 32 * T - 1) / (32 * T);
              if (dirty && red_cap / (tiles * 32 * T) < 2) continue;
              const BLUnits u = bl_units(bt, T, clean4, dirty, red_cap, nmax);
              CHECK(u.ntt * 32 * T >= bt && (u.ntt - 1) * 32 * T < bt, "tiles");
              CHECK(u.nc >= 1 && u.nsub >= 1, "counts");
              if (dirty) CHECK(u.nsub >= 2, "the dirty range has its own sub-range");
              if (u.nsub > 1) {
                CHECK((long long)u.ntt * 32 * T * u.nsub <= red_cap, "red fits T=%d bt=%d", T, bt);
                CHECK(u.nsub <= nmax, "nsub cap");
                CHECK(u.nsub == u.nc + dirty, "dirty sub-range");
              }
            }
  for (int profile = 0; profile <= 2; ++profile)
    for (int nc : {1, 2, 3, 5, 7, 15, 31})
      for (int L : {0, 1, 16, 100, 886, 3543}) {
        int prev = 0, prev_size = 1 << 30;
        CHECK(bl_guided_start(0, nc, L, profile) == 0, "start 0");
        CHECK(bl_guided_start(nc, nc, L, profile) == L, "end L p=%d nc=%d L=%d", profile, nc, L);
        for (int k = 1; k <= nc; ++k) {
          const int s = bl_guided_start(k, nc, L, profile);
          CHECK(s >= prev, "monotone");
          const int size = s - prev;
          if (profile > 0 && L >= 16 * nc) CHECK(size <= prev_size + 1, "decreasing p=%d", profile);
          if (profile == 0) CHECK(size >= L / nc && size <= L / nc + 1, "uniform");
          prev = s;
          prev_size = size;
        }
      }
  std::printf("%s (%d failures)\n", fails ? "FAILED" : "OK", fails);
  return fails ? 1 : 0;
}
