// mmio.cuh -- Matrix Market input/output (mmio.cu), host code.
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

namespace lamgb {

struct MMEdge {
  int32_t u, v;  // u < v
  double w;
};
// lamg::LoadedProblem (matrix_market.hpp:28-32) after read_matrix_market
struct MMProblem {
  int32_t n = 0;
  std::vector<MMEdge> edges;  // canonical: u < v, sorted, unique
  bool was_laplacian = false;
  bool absolute_policy = false;  // assemble_problem's WeightPolicy
  std::vector<std::string> warnings;
};

// kind: 0 auto, 1 adjacency, 2 laplacian (lamg::MatrixKind)
MMProblem read_matrix_market_file(const std::string& path, int kind, bool absolute_weight_policy);
// assemble_problem: the CSR Laplacian (warnings appended to p.warnings)
void assemble_problem(MMProblem& p, std::vector<int64_t>& rp, std::vector<int32_t>& col, std::vector<double>& val,
                      std::vector<double>& diag);
void write_matrix_market_file(const std::string& path, int32_t n, int64_t m, const int64_t* rp, const int32_t* col,
                              const double* val, const double* diag, bool as_laplacian);

}  // namespace lamgb
