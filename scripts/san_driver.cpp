// san_driver.cpp -- a torch-free host program for compute-sanitizer runs
// (memcheck / racecheck / synccheck) of libbl's layout kernels.
//
//   san_driver <graph> <n-ish> <batch> <iters>
//     graph: grid (side x side+3 grid), tri (side x side+10 triangulated
//     mesh, C3 shape), rand (n vertices, ~4 n random undirected edges,
//     skewed towards low ids like the R-MAT configs); a 5th argument "bh"
//     selects BatchLayoutBH
//
// Inputs are seeded (xorshift) and synthetic; the program only calls the
// public C-ABI (bl_create / bl_layout / bl_energy) and checks that the
// result is finite.  The kernel and driver are chosen by the library's own
// rules and the BL_* environment overrides (BL_ASYNC, BL_PIPELINE,
// BL_CLUSTER), so one binary covers every driver.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <utility>
#include <vector>

#include "../include/bl.h"

static unsigned long long g_s = 88172645463325252ull;
static unsigned long long xs() {
  g_s ^= g_s << 13;
  g_s ^= g_s >> 7;
  g_s ^= g_s << 17;
  return g_s;
}
static double u01() { return (xs() >> 11) * (1.0 / 9007199254740992.0); }

int main(int argc, char **argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s grid|tri|rand size batch iters [bh]\n", argv[0]);
    return 2;
  }
  const char *kind = argv[1];
  const int size = std::atoi(argv[2]), batch = std::atoi(argv[3]), iters = std::atoi(argv[4]);
  std::set<std::pair<int, int>> E;
  int n = 0;
  auto add = [&](int a, int b) {
    if (a != b) {
      E.insert({a, b});
      E.insert({b, a});
    }
  };
  if (!std::strcmp(kind, "grid") || !std::strcmp(kind, "tri")) {
    const int R = size, Cc = size + (kind[0] == 'g' ? 3 : 10);
    n = R * Cc;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < Cc; ++c) {
        const int v = r * Cc + c;
        if (c + 1 < Cc) add(v, v + 1);
        if (r + 1 < R) add(v, v + Cc);
        if (kind[0] == 't' && c + 1 < Cc && r + 1 < R) add(v, v + Cc + 1);
      }
  } else {
    n = size;
    for (long long e = 0; e < 4LL * n; ++e) {
      const double a = u01(), b = u01();
      add((int)(a * a * n), (int)(b * b * b * n));  // hubs at low ids
    }
  }
  std::vector<int> rowptr(n + 1, 0), colidx;
  for (auto &e : E) rowptr[e.first + 1]++;
  for (int i = 0; i < n; ++i) rowptr[i + 1] += rowptr[i];
  for (auto &e : E) colidx.push_back(e.second);  // set order: rows ascending
  std::vector<float> xy(2 * (size_t)n);
  for (auto &v : xy) v = (float)u01();

  bl_ctx *h = nullptr;
  bl_status s = bl_create(n, rowptr.data(), colidx.data(), &h);
  if (s != BL_OK) {
    std::fprintf(stderr, "bl_create: %s %s\n", bl_status_string(s), bl_last_error(nullptr));
    return 1;
  }
  bl_params p;
  bl_params_default(&p);
  p.iters = iters;
  p.batch = batch;
  if (argc > 5 && !std::strcmp(argv[5], "bh")) p.algo = BL_ALGO_BH;
  int done = 0;
  s = bl_layout(h, xy.data(), &p, &done);
  if (s != BL_OK) {
    std::fprintf(stderr, "bl_layout: %s %s\n", bl_status_string(s), bl_last_error(h));
    return 1;
  }
  double e = 0;
  s = bl_energy(h, &e, nullptr, 0, nullptr, nullptr);
  for (float v : xy)
    if (!std::isfinite(v)) {
      std::fprintf(stderr, "non-finite coordinate\n");
      return 1;
    }
  std::printf("%s n=%d nnz=%zu b=%d iters=%d done=%d kernel=%s driver=%s E=%.9e\n", kind, n,
              colidx.size(), batch, iters, done, bl_kernel_name(h), bl_driver_name(h), e);
  bl_destroy(h);
  return s == BL_OK ? 0 : 1;
}
