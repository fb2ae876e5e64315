// part.cuh -- fine-level node-block partition with halo exchange (part.cu).
#pragma once
#include <memory>
#include <vector>

#include "hier.cuh"

namespace lamgb {

// one part of a contiguous row-block partition of a symmetric CSR (host)
struct PartPlan {
  int32_t nparts = 0, part = 0, lo = 0, hi = 0, nloc = 0, nghost = 0;
  std::vector<int64_t> rp;         // [nloc+1] local rows
  std::vector<int32_t> col;        // owned column g -> g - lo; ghost -> nloc + ghost index
  std::vector<double> val, diag;
  std::vector<int32_t> ghost_gid;  // [nghost] ascending global ids
  std::vector<int32_t> recv_ptr;   // [nparts+1] ghost range owned by each part
  std::vector<int32_t> send_ptr;   // [nparts+1] ranges of send_idx per peer
  std::vector<int32_t> send_idx;   // owned local rows each peer needs (ascending)
};

// row bounds balancing rows + entries
void part_bounds(int32_t n, const int64_t* rp, int32_t nparts, std::vector<int32_t>& bounds);
PartPlan build_part_plan(int32_t n, const int64_t* rp, const int32_t* col, const double* val, const double* diag,
                         const std::vector<int32_t>& bounds, int32_t part);

// NCCL communicator (one rank per GPU)
struct Comm {
  int32_t nranks = 0, rank = 0;
  void* handle = nullptr;  // ncclComm_t
  Comm(int32_t nranks, int32_t rank, const char id[128]);
  ~Comm();
};
void comm_unique_id(char out[128]);

// the parts of one level owned by this process: all of them (in-process
// transport, comm == nullptr) or exactly this rank's (NCCL)
struct PartLevel {
  struct Part;
  Ctx& c;
  std::vector<int32_t> bounds;
  Comm* comm;
  int32_t ncolors = 0;
  int group = 1;
  bool use_tasks = false;  // residual by tasks (the level has long rows)
  int task_group = 1;
  std::vector<std::unique_ptr<Part>> parts;

  PartLevel(Ctx& c, const CSRv& full_dev, const std::vector<int64_t>& rp_h, const std::vector<int32_t>& col_h,
            const std::vector<double>& val_h, const std::vector<double>& diag_h, const std::vector<int32_t>& bounds,
            int32_t first_part, int32_t nown, Comm* comm);
  ~PartLevel();
  int32_t nparts() const;
  Part& local(int32_t part);
  void exchange();                 // ghost values of every owned part
  void sweep(int sweeps);          // coloured GS, an exchange after every colour
  void residual();                 // r = b - A x on every owned part (ghosts current)
  void load(const double* b_global_dev, const double* x_global_dev);  // owned slices (+ exchange)
  void store(double* x_global_dev, double* r_global_dev);            // owned slices back
  // every rank's owned slices into a full-size vector on every rank (x or r)
  void allgather(bool residual, double* full_dev);
  // x_local += xc[aggregate_of[global row]] for owned rows (add_interpolated), then exchange
  void interpolate(const int32_t* aggregate_of_full, const double* xc);
};

// lamg::solve (cycle.cpp:221-273) with the first smoothing level partitioned
// (part_level_of): its sweeps and residuals run on the parts (halo exchange),
// its residual is allgathered so every rank restricts it and runs the coarse
// levels exactly as one device does (replicated, deterministic); a
// relaxation-coarsest level (coarse_solver.cpp:82-93) relaxes on the parts.
// THROUGHPUT, flat cycle. With an aggregation child the result is
// bit-identical to solve_device with exact_levels = 0; the relaxation form is
// bit-identical across part counts.
struct SolveResult;
struct CycleCfg;
struct DHier;
// the level lamg_part_solve partitions: the finest level that smooths (0, or 1
// when the finest level is reduced by elimination first)
int part_level_of(const DHier& h);
int solve_partitioned(Ctx& c, const DHier& h, PartLevel& pl, const double* b, const double* x0, const CycleCfg& cfg,
                      double* x, SolveResult& res);

}  // namespace lamgb
