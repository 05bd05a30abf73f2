// K3 entry sampler / K4 direct sum (see sample.cu).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

extern "C" {
#include "midbf_b200.h"
}

namespace midbf::dev {

// Device copy of one kernel description (point sets / low-rank factors and
// per-point phase coefficients), reused across the sweeps of a factorization.
class EntrySampler {
 public:
  explicit EntrySampler(const midbf_kernel_desc& kd);
  ~EntrySampler();
  EntrySampler(const EntrySampler&) = delete;
  EntrySampler& operator=(const EntrySampler&) = delete;

  // tasks: ntasks x 5 (row_off, nr, col_off, nc, out_off); host in/out.
  void sample(int64_t ntasks, const int64_t* tasks, const int64_t* row_ids, int64_t n_row_ids,
              const int64_t* col_ids, int64_t n_col_ids, double* out, int64_t out_len);
  // Same, each task's block written to its own destination outs[t].
  void sample_blocks(int64_t ntasks, const int64_t* tasks, const int64_t* row_ids, int64_t n_row_ids,
                     const int64_t* col_ids, int64_t n_col_ids, double* const* outs);
  // K3 + K5: sample each task's block into a device workspace and compute
  // its interpolative decomposition there (column ID of the block, or with
  // `rowid` a row ID = column ID of its transpose).  Per task: rank (-1: not
  // computed on the device, recompute on the host), skeleton positions and
  // the interpolation matrix (V: rank x n, ld rank; W: n x rank, ld n) at
  // vals + ooff[t].  kcap = skeleton stride.
  struct IdBatch {
    std::vector<int> rank, skel;
    std::vector<int64_t> ooff;
    int kcap = 0;
    const double* vals = nullptr;  // pinned, process-wide: valid until the next sample_ids call
  };
  // on_part(t0, t1), when given, runs on the calling thread as soon as tasks
  // [t0, t1) are complete on the host side of `out` (values, ranks,
  // skeletons), while the device still works on later tasks.
  void sample_ids(int64_t ntasks, const int64_t* tasks, const int64_t* row_ids, int64_t n_row_ids,
                  const int64_t* col_ids, int64_t n_col_ids, bool rowid, int64_t k_max, double eps, IdBatch& out,
                  const std::function<void(int64_t, int64_t)>& on_part = {});
  // Phi(rows, cols) (real, column-major nr x nc; rows / cols null: 0..n-1)
  // for the kernels with a phase (FIO 2D/3D, low-rank, x.xi).
  void phase_block(int64_t nr, const int64_t* rows, int64_t nc, const int64_t* cols, double* out);
  void direct_sum(const double* f, const int64_t* rows, int64_t nsel, double* g);
  int64_t entries_evaluated() const;
  // Device time of this sampler's kernel launches (CUDA events).
  struct KernelTimes {
    int64_t k3_launches = 0, k3_entries = 0, k5_launches = 0;
    double k3_seconds = 0, k5_seconds = 0;
  };
  KernelTimes kernel_times() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

double& last_direct_sum_seconds();  // device time of the thread's last direct sum (K4)

}  // namespace midbf::dev
