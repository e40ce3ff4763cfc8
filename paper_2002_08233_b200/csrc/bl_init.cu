// bl_init.cu -- greedy initialisation of the layout (host, native C++).
//
// Alg. 3 "Greedy Initialization" (§3.6): a DFS
// with an explicit stack from V0 at (0, 0) that puts each popped vertex's
// not-yet-placed neighbours on the unit circle around it, at angles stepping
// by 360/deg(U) degrees, PI = 3.1416 as the paper states.  O(n + m),
// inherently sequential (the DFS order decides every position), so it runs
// on the host once per layout, not on the GPU.  Readings G1-G4:
// caller-chosen root; full degree in d; components other than V0's restart
// from their smallest id at origins on a square grid.
#include <cmath>
#include <cstdint>
#include <algorithm>
#include <vector>

#include "../../include/bl.h"

namespace {
constexpr double kPaperPi = 3.1416;  // "PI is a constant whose value is 3.1416"
}

extern "C" bl_status bl_greedy_init(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                                    int32_t root, float *xy_out) {
  if (n < 1 || !rowptr || !xy_out || root < 0 || root >= n) return BL_EINVAL;
  if (rowptr[0] != 0) return BL_EINVAL;
  for (int32_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) return BL_EINVAL;
  if (rowptr[n] > 0 && !colidx) return BL_EINVAL;
  for (int32_t k = 0; k < rowptr[n]; ++k)
    if (colidx[k] < 0 || colidx[k] >= n) return BL_EINVAL;

  // components (BFS), ranked: V0's first, then by smallest vertex id (G3)
  std::vector<int32_t> comp(n, -1), queue;
  queue.reserve(n);
  int32_t ncomp = 0;
  size_t largest = 0;
  auto label = [&](int32_t s) {
    queue.clear();
    queue.push_back(s);
    comp[s] = ncomp;
    for (size_t h = 0; h < queue.size(); ++h) {
      const int32_t u = queue[h];
      for (int32_t k = rowptr[u]; k < rowptr[u + 1]; ++k) {
        const int32_t w = colidx[k];
        if (comp[w] < 0) {
          comp[w] = ncomp;
          queue.push_back(w);
        }
      }
    }
    largest = std::max(largest, queue.size());
    ++ncomp;
  };
  label(root);
  for (int32_t v = 0; v < n; ++v)
    if (comp[v] < 0) label(v);
  // grid of g x g origins (smallest g with g^2 >= #components), spacing
  // 2 ceil(sqrt(largest component size))
  int32_t g = 1, side = 1;
  while ((int64_t)g * g < ncomp) ++g;
  while ((int64_t)side * side < (int64_t)largest) ++side;
  const double spacing = 2.0 * side;

  // Alg. 3 per component, fp64 positions
  std::vector<double> V(2 * (size_t)n, 0.0);
  std::vector<char> visited(n, 0);
  std::vector<int32_t> stack;
  stack.reserve(n);
  auto place_from = [&](int32_t v0) {
    const int32_t k = comp[v0];
    V[2 * v0] = (double)(k % g) * spacing;  // V0 = (0, 0) for the first component
    V[2 * v0 + 1] = (double)(k / g) * spacing;
    visited[v0] = 1;
    stack.push_back(v0);
    while (!stack.empty()) {
      const int32_t U = stack.back();
      stack.pop_back();
      const int32_t deg = rowptr[U + 1] - rowptr[U];
      if (deg == 0) continue;  // G4
      const double d = 360.0 / deg;
      double D = 0.0;
      for (int32_t e = rowptr[U]; e < rowptr[U + 1]; ++e) {
        const int32_t u = colidx[e];
        if (visited[u]) continue;
        V[2 * u] = V[2 * U] + std::cos(kPaperPi * D / 180.0);
        V[2 * u + 1] = V[2 * U + 1] + std::sin(kPaperPi * D / 180.0);
        visited[u] = 1;
        stack.push_back(u);
        D += d;
      }
    }
  };
  place_from(root);
  for (int32_t v = 0; v < n; ++v)
    if (!visited[v]) place_from(v);
  for (size_t i = 0; i < V.size(); ++i) xy_out[i] = (float)V[i];
  return BL_OK;
}
