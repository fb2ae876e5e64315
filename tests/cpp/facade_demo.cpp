// tests/cpp/facade_demo.cpp -- reference-style host code compiled against the
// drop-in facade (include/lamg_b200/lamg.hpp). Only the include line differs
// from code written for the reference's own lamg/*.hpp headers.
#include <cstdio>
#include <vector>

#include "lamg_b200/lamg.hpp"

// 5-point N x N grid, node (i,j) -> i*N+j (generators.cpp:19-41)
static lamg::SparseLaplacian grid(int N) {
  lamg::SparseLaplacian a;
  a.n = N * N;
  a.row_ptr.push_back(0);
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      const int nb[4][2] = {{i - 1, j}, {i, j - 1}, {i, j + 1}, {i + 1, j}};
      double d = 0.0;
      for (auto& p : nb) {
        if (p[0] < 0 || p[1] < 0 || p[0] >= N || p[1] >= N) continue;
        a.col.push_back(p[0] * N + p[1]);
        a.val.push_back(-1.0);
        d += 1.0;
      }
      a.diag.push_back(d);
      a.row_ptr.push_back((lamg::EntryCount)a.col.size());
    }
  a.m = (lamg::EntryCount)a.col.size() / 2;
  return a;
}

int main() {
  lamg::SparseLaplacian a = grid(64);
  lamg::Hierarchy h = lamg::setup(a, {.rng_seed = 1});
  lamg::Vector b(a.n, 0.0), x0(a.n, 0.0);
  b[0] = 1.0;
  b[a.n - 1] = -1.0;
  auto [x, stats] = lamg::solve(h, b, x0);
  lamg::HierarchyStats hs = lamg::hierarchy_stats(h);
  std::printf("levels %zu cycles %d converged %d acf %.6f edge_ratio %.4f\n", h.levels.size(), stats.cycles,
              (int)stats.converged, stats.acf, hs.edge_ratio);
  try {
    lamg::Vector bad(a.n, 1.0);
    lamg::solve(h, bad, x0);
    std::printf("no error\n");
  } catch (const lamg::IncompatibleRhsError& e) {
    std::printf("IncompatibleRhsError: %s\n", e.what());
  }
  // whole-problem driver on a disconnected graph with an isolated node
  lamg::SparseLaplacian d;
  d.n = 7;
  d.row_ptr = {0, 1, 3, 4, 6, 8, 10, 10};
  d.col = {1, 0, 2, 1, 4, 5, 3, 5, 3, 4};
  d.val = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
  d.diag = {1, 2, 1, 2, 2, 2, 0};
  d.m = 5;
  lamg::Prepared p = lamg::prepare(d);
  lamg::SolveReport r = lamg::solve_prepared(p, std::vector<double>{1.0, 0.0, -1.0, 0.5, -0.25, -0.25, 0.0});
  std::printf("components %zu converged %d x6 %.1f\n", p.components.size(), (int)r.converged, r.x[6]);
  // Matrix Market round trip (host only) and a parse error with the reference's text
  const char* path = "/tmp/lamg_b200_facade_demo.mtx";
  lamg::write_matrix_market_file(path, a);
  lamg::LoadedLaplacian back = lamg::load_matrix_market_file(path);
  std::printf("mm n %d m %lld same %d laplacian %d\n", back.a.n, (long long)back.a.m,
              (int)(back.a.col == a.col && back.a.val == a.val && back.a.diag == a.diag), (int)back.was_laplacian);
  try {
    lamg::load_matrix_market_file("/nonexistent/x.mtx");
  } catch (const lamg::IoError& e) {
    std::printf("IoError: %s\n", e.what());
  }
  return 0;
}
