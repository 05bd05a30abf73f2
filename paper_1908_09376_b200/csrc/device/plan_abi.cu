// MIDBF001 container -> device plan, device checks, and the plan C ABI
// (include/midbf_b200.h "plan" section).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <fstream>
#include <mutex>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "flow.cuh"
#include "plan.hpp"
#include "pool.hpp"

namespace midbf::dev {

// ------------------------------------------------------------- MIDBF001 I/O
// Container layout: reference include/midbf/butterfly_io.hpp:2-15; checks as
// src/butterfly_io.cpp:103-167.
std::unique_ptr<Plan> load_plan(const std::string& path, unsigned directions) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for reading: " + path);
  const auto need = [&](bool ok, const char* what) {
    if (!ok) throw std::runtime_error(std::string(what) + " in " + path);
  };
  const auto raw = [&]() {
    int64_t v = 0;
    f.read(reinterpret_cast<char*>(&v), 8);
    need(bool(f), "truncated container");
    return v;
  };
  const int64_t big = int64_t{1} << 40;
  const auto count = [&](const char* what, int64_t mx) {
    const int64_t v = raw();
    need(v >= 0 && v <= mx, what);
    return v;
  };
  char magic[8];
  f.read(magic, 8);
  need(bool(f), "truncated container");
  need(std::memcmp(magic, "MIDBF001", 8) == 0, "unrecognized container magic");
  PlanTables T;
  T.nrows = count("bad row count", big);
  T.ncols = count("bad column count", big);
  count("bad level count", 64);
  count("bad stop level", 64);
  count("bad leaf size", big);
  count("bad rank cap", big);
  count("bad sampling oversize", big);
  raw();
  raw();
  raw();
  T.nfactors = count("bad factor count", 4096);
  std::vector<int64_t> rp(static_cast<size_t>(T.nrows)), cp(static_cast<size_t>(T.ncols));
  for (auto& v : rp) {
    v = count("bad row permutation entry", big);
    need(v < T.nrows, "row permutation out of range");
  }
  for (auto& v : cp) {
    v = count("bad column permutation entry", big);
    need(v < T.ncols, "column permutation out of range");
  }
  std::vector<std::vector<int64_t>> blocks(static_cast<size_t>(T.nfactors)), groups(static_cast<size_t>(T.nfactors));
  T.factors.resize(static_cast<size_t>(T.nfactors));
  for (int64_t i = 0; i < T.nfactors; ++i) {
    FactorView& F = T.factors[static_cast<size_t>(i)];
    F.rows = count("bad factor rows", big);
    F.cols = count("bad factor cols", big);
    const int64_t nb = count("bad block count", big), ng = count("bad group count", big);
    auto& bl = blocks[static_cast<size_t>(i)];
    auto& gr = groups[static_cast<size_t>(i)];
    bl.resize(static_cast<size_t>(4 * nb));
    gr.resize(static_cast<size_t>(2 * ng));
    for (int64_t b = 0; b < nb; ++b) {
      for (int q = 0; q < 4; ++q) bl[4 * b + q] = count(q == 0   ? "bad block row offset"
                                                        : q == 1 ? "bad block column offset"
                                                        : q == 2 ? "bad block height"
                                                                 : "bad block width",
                                                        big);
      need(bl[4 * b] + bl[4 * b + 2] <= F.rows && bl[4 * b + 1] + bl[4 * b + 3] <= F.cols,
           "block outside its factor");
    }
    for (int64_t g = 0; g < ng; ++g) {
      gr[2 * g] = count("bad group begin", big);
      gr[2 * g + 1] = count("bad group end", big);
      need(gr[2 * g] <= gr[2 * g + 1] && gr[2 * g + 1] <= nb, "group outside block table");
    }
    F.nblocks = nb;
    F.ngroups = ng;
  }
  int64_t total = 0, nblocks_all = 0;
  for (int64_t i = 0; i < T.nfactors; ++i)
    for (int64_t b = 0; b < T.factors[i].nblocks; ++b) {
      total += blocks[i][4 * b + 2] * blocks[i][4 * b + 3];
      ++nblocks_all;
    }
  // payload: contiguous in block order = the plan's raw layout; stream it
  // through the pinned staging pool straight into device memory
  double2* d_raw = nullptr;
  cuda_check(cudaMalloc(&d_raw, std::max<int64_t>(total, 1) * sizeof(double2)), "cudaMalloc raw payload");
  try {
    PinnedPool& P = pinned_pool();
    std::lock_guard<std::mutex> lock(P.mu);
    P.ensure();
    const int64_t cap = static_cast<int64_t>(PinnedPool::kBytes / sizeof(double2));
    int buf = 0, used = 0;
    for (int64_t at = 0; at < total; at += cap) {
      const int64_t n = std::min(cap, total - at);
      if (used >= 2) cuda_check(cudaEventSynchronize(P.ev[buf]), "payload buffer reuse");
      f.read(P.h[buf], static_cast<std::streamsize>(16 * n));
      need(bool(f), "truncated payload");
      cuda_check(cudaMemcpyAsync(d_raw + at, P.h[buf], n * sizeof(double2), cudaMemcpyHostToDevice, nullptr),
                 "payload H2D");
      cuda_check(cudaEventRecord(P.ev[buf], nullptr), "event");
      buf ^= 1;
      ++used;
    }
    cuda_check(cudaDeviceSynchronize(), "payload upload");
    f.peek();
    need(f.eof(), "trailing bytes after payload");
  } catch (...) {
    cudaDeviceSynchronize();
    cudaFree(d_raw);
    throw;
  }
  for (int64_t i = 0; i < T.nfactors; ++i) {
    FactorView& F = T.factors[static_cast<size_t>(i)];
    F.blocks = blocks[i].data();
    F.groups = groups[i].data();
  }
  T.row_perm = rp.data();
  T.col_perm = cp.data();
  T.total_nnz = total;
  T.total_blocks = nblocks_all;
  return std::make_unique<Plan>(T, directions, d_raw);
}

int require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw detail::CudaFailure("no CUDA device visible: the MIDBF B200 path has no CPU fallback");
  }
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  cudaDeviceProp prop;
  cuda_check(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
  if (prop.major != 10)
    throw detail::CudaFailure("device " + std::string(prop.name) + " is not sm_100 (this build targets sm_100a)");
  return dev;
}

}  // namespace midbf::dev

// ------------------------------------------------------------------ C ABI
using midbf::detail::guard;
using midbf::dev::Plan;

struct midbf_plan_s {
  std::unique_ptr<Plan> p;
};

namespace {

// Shared body of midbf_plan_create / midbf_plan_create_blocks: payload(i, b)
// returns block b of factor i (column-major complex, rows x cols).
template <typename PayloadAt>
midbf_plan_t create_plan(int64_t nrows, int64_t ncols, const int64_t* row_perm, const int64_t* col_perm,
                         int64_t nfactors, const int64_t* factor_shape, const int64_t* blocks,
                         const int64_t* groups, PayloadAt payload, unsigned directions) {
  midbf::dev::PlanTables T;
  T.nrows = nrows;
  T.ncols = ncols;
  T.row_perm = row_perm;
  T.col_perm = col_perm;
  T.nfactors = nfactors;
  T.factors.resize(static_cast<size_t>(nfactors));
  std::vector<std::vector<const double*>> ptrs(static_cast<size_t>(nfactors));
  const int64_t* bp = blocks;
  const int64_t* gp = groups;
  int64_t flat = 0;
  for (int64_t i = 0; i < nfactors; ++i) {
    auto& F = T.factors[static_cast<size_t>(i)];
    F.rows = factor_shape[4 * i];
    F.cols = factor_shape[4 * i + 1];
    F.nblocks = factor_shape[4 * i + 2];
    F.ngroups = factor_shape[4 * i + 3];
    F.blocks = bp;
    F.groups = gp;
    for (int64_t b = 0; b < F.nblocks; ++b, ++flat) {
      const int64_t m = bp[4 * b + 2], n = bp[4 * b + 3];
      if (m < 0 || n < 0 || bp[4 * b] < 0 || bp[4 * b + 1] < 0 || bp[4 * b] + m > F.rows ||
          bp[4 * b + 1] + n > F.cols)
        throw std::invalid_argument("block outside its factor");
      const double* pb = payload(flat, m * n);
      if (!pb && m * n > 0) throw std::invalid_argument("null block payload");
      ptrs[i].push_back(pb);
      T.total_nnz += m * n;
      ++T.total_blocks;
    }
    for (int64_t g = 0; g < F.ngroups; ++g)
      if (gp[2 * g] < 0 || gp[2 * g] > gp[2 * g + 1] || gp[2 * g + 1] > F.nblocks)
        throw std::invalid_argument("group outside block table");
    F.payload = ptrs[i].data();
    bp += 4 * F.nblocks;
    gp += 2 * F.ngroups;
  }
  return new midbf_plan_s{std::make_unique<Plan>(T, directions)};
}

}  // namespace

extern "C" int midbf_plan_create(midbf_plan_t* out, int64_t nrows, int64_t ncols, const int64_t* row_perm,
                                 const int64_t* col_perm, int64_t nfactors, const int64_t* factor_shape,
                                 const int64_t* blocks, const int64_t* groups, const double* payload,
                                 unsigned directions) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output handle");
    const double* pp = payload;
    *out = create_plan(nrows, ncols, row_perm, col_perm, nfactors, factor_shape, blocks, groups,
                       [&pp](int64_t, int64_t mn) {
                         const double* p = pp;
                         pp += 2 * mn;
                         return p;
                       },
                       directions);
  });
}

extern "C" int midbf_plan_create_blocks(midbf_plan_t* out, int64_t nrows, int64_t ncols, const int64_t* row_perm,
                                        const int64_t* col_perm, int64_t nfactors, const int64_t* factor_shape,
                                        const int64_t* blocks, const int64_t* groups,
                                        const double* const* block_payloads, unsigned directions) {
  return guard([&] {
    if (!out || !block_payloads) throw std::invalid_argument("null argument");
    *out = create_plan(nrows, ncols, row_perm, col_perm, nfactors, factor_shape, blocks, groups,
                       [block_payloads](int64_t flat, int64_t) { return block_payloads[flat]; }, directions);
  });
}

extern "C" int midbf_plan_load(midbf_plan_t* out, const char* path, unsigned directions) {
  return guard([&] { *out = new midbf_plan_s{midbf::dev::load_plan(path, directions)}; });
}

extern "C" int midbf_plan_destroy(midbf_plan_t plan) {
  return guard([&] { delete plan; });
}

extern "C" int midbf_plan_info(midbf_plan_t plan, int64_t* out) {
  return guard([&] {
    const Plan& p = *plan->p;
    out[0] = p.nrows;
    out[1] = p.ncols;
    out[2] = p.nfactors;
    out[3] = p.total_nnz;
    int64_t bytes = 0, tasks = 0;
    unsigned dirs = 0;
    for (int d = 0; d < 2; ++d)
      if (p.dir[d].built) {
        bytes += p.dir[d].arena_elems * 16;
        tasks += p.dir[d].nstrips;
        dirs |= 1u << d;
      }
    out[4] = bytes;
    out[5] = tasks;
    out[6] = dirs;
    out[7] = p.max_len;
  });
}

extern "C" int midbf_apply(midbf_plan_t plan, const double* f, double* g, int64_t nrhs, int transpose, void* stream) {
  return guard([&] {
    if (!plan || !f || !g) throw std::invalid_argument("null argument");
    plan->p->apply(f, g, nrhs, transpose != 0, static_cast<cudaStream_t>(stream));
  });
}

extern "C" int midbf_apply_async(midbf_plan_t plan, const double* f, double* g, int64_t nrhs, int transpose,
                                 void* stream) {
  return guard([&] {
    if (!plan || !f || !g) throw std::invalid_argument("null argument");
    plan->p->apply_async(f, g, nrhs, transpose != 0, static_cast<cudaStream_t>(stream));
  });
}

// Stage table for benchmarks / roofline accounting:
// out[s*4 + 0..3] = strips, payload bytes, in_len, out_len of stage s.
extern "C" int midbf_plan_stages(midbf_plan_t plan, int transpose, int64_t* out, int64_t cap) {
  return guard([&] {
    const auto& D = plan->p->dir[transpose ? 1 : 0];
    int64_t s = 0;
    for (const auto& st : D.stages) {
      if (s >= cap) break;
      out[4 * s] = st.nstrips;
      out[4 * s + 1] = st.payload_bytes;
      out[4 * s + 2] = st.in_len;
      out[4 * s + 3] = st.out_len;
      ++s;
    }
  });
}

// Panel bytes k1_flow streams per stage (identity-compressed unless flag bit
// 9 is set or the plan runs the dense-only k1_flow, Plan::flow_lite): out[s],
// application order.
extern "C" int midbf_plan_flow_bytes(midbf_plan_t plan, int transpose, int64_t* out, int64_t cap) {
  return guard([&] {
    const Plan& p = *plan->p;
    const auto& D = p.dir[transpose ? 1 : 0];
    const bool dense = p.flow_dense(transpose ? 1 : 0);
    int64_t s = 0;
    for (const auto& st : D.stages) {
      if (s >= cap) break;
      out[s++] = dense ? st.payload_bytes : st.flow_bytes;
    }
  });
}

// Panel entries x 16 bytes the multi-RHS DMMA kernel multiplies per apply on
// 32- / 64-wide tiles (identity-compressed V-type strips unless flag bit 9).
extern "C" int midbf_plan_k2_bytes(midbf_plan_t plan, int transpose, int64_t* out) {
  return guard([&] {
    const Plan& p = *plan->p;
    const auto& D = p.dir[transpose ? 1 : 0];
    int64_t dense = 0;
    for (const auto& st : D.stages) dense += st.payload_bytes;
    *out = (D.d_k2strips && !(p.flags & 512u)) ? 16 * D.k2_elems : dense;
  });
}

// Tuning switches (bench / profiling): bit0 PDL, bit1 L2 bulk prefetch
// (stage kernels), bit2 CUDA graphs, bit3 persistent dataflow kernel.
extern "C" int midbf_plan_set_flags(midbf_plan_t plan, unsigned flags) {
  return guard([&] {
    std::lock_guard<std::recursive_mutex> lock(plan->p->mu);
    Plan& p = *plan->p;
    p.flags = flags;
    if ((flags & 4096u) && !p.d_prof)  // phase-timer buffer, allocated outside any capture
      midbf::dev::cuda_check(
          cudaMalloc(&p.d_prof, (midbf::dev::kProfStripBase + 3 * size_t(midbf::dev::kProfStrips)) * sizeof(long long)),
          "prof buffer");
  });
}

extern "C" int midbf_plan_get_flags(midbf_plan_t plan, unsigned* out) {
  return guard([&] {
    std::lock_guard<std::recursive_mutex> lock(plan->p->mu);
    *out = plan->p->flags;
  });
}

// Kernel launches of one apply (evidence for bench.py's gpu_launches).
extern "C" int midbf_plan_launches(midbf_plan_t plan, int transpose, int64_t nrhs, int64_t* out) {
  return guard([&] { *out = plan->p->launches_per_apply(transpose ? 1 : 0, nrhs); });
}

// Phase timers of the last k1_flow launch made with flag bit 12: per warp
// 16 counters (cycles); out must hold grid * 2 * warps_per_cta * 16 values.
extern "C" int midbf_plan_flow_profile(midbf_plan_t plan, int64_t* out, int64_t n) {
  return guard([&] {
    Plan& p = *plan->p;
    if (!p.d_prof) throw std::logic_error("no profiled k1_flow launch");
    midbf::dev::cuda_check(cudaDeviceSynchronize(), "sync");
    const size_t bytes =
        std::min<size_t>(static_cast<size_t>(n), midbf::dev::kProfStripBase + 3 * size_t(midbf::dev::kProfStrips)) *
        sizeof(long long);
    midbf::dev::cuda_check(cudaMemcpy(out, p.d_prof, bytes, cudaMemcpyDeviceToHost), "prof D2H");
  });
}
