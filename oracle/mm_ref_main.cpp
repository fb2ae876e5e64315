// oracle/mm_ref_main.cpp -- TEST INFRASTRUCTURE ONLY (the parity checker).
//
// Runs the UNMODIFIED reference Matrix Market reader (read_matrix_market_file
// + assemble_problem, matrix_market.cpp:37-193) on a file and dumps the result
// for tests/test_mmio.py. A separate process: the reference's iostreams and
// the statically linked C++ runtime of oracle/_ref do not mix with the
// Python process's own.
//
//   mm_ref <in.mtx> <kind 0|1|2> <absolute_policy 0|1> <out.bin>
// out.bin: int32 status; status != 0: the message; else int32 n, int64 m,
// int32 was_laplacian, int32 warnings, each warning (int32 len + bytes), then
// row_ptr, col, val, diag.
#include <cstdint>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "lamg/errors.hpp"
#include "lamg/matrix_market.hpp"

int main(int argc, char** argv) {
  if (argc != 5) {
    std::fprintf(stderr, "usage: mm_ref in.mtx kind policy out.bin\n");
    return 2;
  }
  FILE* f = std::fopen(argv[4], "wb");
  if (!f) return 3;
  auto put = [&](const void* p, size_t n) { std::fwrite(p, 1, n, f); };
  try {
    lamg::MatrixMarketOptions o;
    const int kind = std::atoi(argv[2]);
    o.kind = kind == 1 ? lamg::MatrixKind::Adjacency : kind == 2 ? lamg::MatrixKind::Laplacian : lamg::MatrixKind::Auto;
    o.absolute_weight_policy = std::atoi(argv[3]) != 0;
    auto prob = lamg::read_matrix_market_file(argv[1], o);
    std::vector<std::string> w;
    auto a = lamg::assemble_problem(prob, o, &w);
    int32_t st = 0, n = a.n, lap = prob.was_laplacian, nw = (int32_t)w.size();
    int64_t m = a.m;
    put(&st, 4), put(&n, 4), put(&m, 8), put(&lap, 4), put(&nw, 4);
    for (auto& s : w) {
      int32_t len = (int32_t)s.size();
      put(&len, 4), put(s.data(), s.size());
    }
    put(a.row_ptr.data(), 8 * a.row_ptr.size());
    put(a.col.data(), 4 * a.col.size());
    put(a.val.data(), 8 * a.val.size());
    put(a.diag.data(), 8 * a.diag.size());
  } catch (const std::exception& e) {
    int32_t st = 1;
    std::string msg = e.what();
    put(&st, 4), put(msg.data(), msg.size());
  }
  std::fclose(f);
  return 0;
}
