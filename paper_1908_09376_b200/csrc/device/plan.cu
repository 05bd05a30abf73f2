// K1 — MIDBF apply on sm_100a: device plan (one contiguous factor arena) and
// the apply kernels.
//
// Replaces bf::apply_impl / apply_factor (reference src/butterfly.cpp:624-667):
//   v = f[col_perm];  for factor V^1 .. U^1: v = F_i v;  g[row_perm] = v.
// The reference keeps every block as a separately allocated Eigen matrix and
// runs one OpenMP-parallel Eigen GEMV per group.  Here each applied factor (a
// "stage") becomes a list of output *strips* of <= 32 rows; a strip owns the
// ordered list of block panels that write its rows (the reference's fixed
// in-group block order), so exactly one warp writes every output entry: no
// atomics, no float reductions across warps, results bitwise reproducible.
//
// Arena: panel of (strip, block) = the strip's rows of that block, h x n
// column-major, panels appended in strip order and strips in application
// order, so one apply streams the arena once, front to back.
//
// k1_flow (single RHS, default; flow.cuh): ONE persistent launch for all
//   stages.  1 CTA per SM, 4 (or 8 for plans > 512 MB) consumer / producer
//   / x-stager warp triples; strips are dealt round-robin to the consumer
//   warps stage by stage (static deal, no counters); each producer streams
//   its consumer's panels into a ring of shared-memory slots with
//   cp.async.bulk (TMA bulk copy, mbarrier complete_tx); a strip's x window
//   is gathered by the stager (stage 0 of the 4-pair layout: straight from f
//   through col_perm), which polls the previous stage's output until
//   no entry carries the sentinel (the data is its own ready signal: relaxed
//   GPU-scope stores and loads, no flags) — there is no stage-wide barrier,
//   so HBM streaming continues across stage boundaries; each lane owns one
//   output row; the last stage scatters through row_perm.  Consecutive
//   applies on one stream are chained by programmatic dependent launch
//   (flag bit 17).
// k1_coop (single RHS, plans below kCoopBytes; coop.cuh): a CTA per strip,
//   its 8 warps splitting the columns, panels of the next strips prefetched.
// k1_stage (multi-RHS fallback and A/B reference): one launch per stage,
//   warp per strip, streaming 128-bit loads; chained with programmatic
//   dependent launch inside a CUDA graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "plan.hpp"
#include "pool.hpp"
#include "flow.cuh"
#include "k2.cuh"
#include "k2flow.cuh"
#include "coop.cuh"

namespace midbf::dev {

namespace {


// ---------------------------------------------------------------- helpers
__device__ __forceinline__ void cmac(double& ar, double& ai, double2 m, double2 x) {
  ar = fma(m.x, x.x, ar);
  ar = fma(-m.y, x.y, ar);
  ai = fma(m.x, x.y, ai);
  ai = fma(m.y, x.x, ai);
}

__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// ------------------------------------------------------------ k1_stage
constexpr int kWarps = 4;
constexpr int kXChunk = 256;

template <bool kPrefetch>
__global__ void __launch_bounds__(kWarps * 32) k1_stage(const Strip* __restrict__ strips, int nstrips,
                                                        const Seg* __restrict__ segs,
                                                        const double2* __restrict__ arena,
                                                        const double2* __restrict__ x, int64_t xld,
                                                        const int* __restrict__ xperm, double2* __restrict__ y,
                                                        int64_t yld, const int* __restrict__ yperm) {
  __shared__ __align__(16) double2 xs[kWarps][kXChunk];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int t = blockIdx.x * kWarps + wid;
  Strip st = {0, 0, 0, 0, 0, 0, 0, 0};
  if (t < nstrips) st = strips[t];
  if (kPrefetch && t < nstrips && lane < st.nseg) {
    const Seg s = segs[st.seg0 + lane];
    bulk_prefetch_l2(arena + s.off, static_cast<uint32_t>(s.n) * static_cast<uint32_t>(st.h) * 16u);
  }
  pdl_wait();
  pdl_launch_dependents();
  if (t >= nstrips) return;
  x += blockIdx.y * xld;
  y += blockIdx.y * yld;
  const int h = st.h;
  const bool live = lane < h;
  double ar0 = 0, ai0 = 0, ar1 = 0, ai1 = 0;
  double2* xw = xs[wid];
  for (int si = 0; si < st.nseg; ++si) {
    const Seg s = segs[st.seg0 + si];
    const double2* P = arena + s.off + lane;
    for (int cb = 0; cb < s.n; cb += kXChunk) {
      const int cn = min(kXChunk, s.n - cb);
      __syncwarp();
      for (int j = lane; j < cn; j += 32) {
        int idx = s.x0 + cb + j;
        if (xperm) idx = xperm[idx];
        xw[j] = x[idx];
      }
      __syncwarp();
      if (live) {
        int c = 0;
        for (; c + 8 <= cn; c += 8) {
          double2 m[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) m[u] = ld_stream(P + (int64_t)(cb + c + u) * h);
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            cmac(ar0, ai0, m[u], xw[c + u]);
            cmac(ar1, ai1, m[u + 1], xw[c + u + 1]);
          }
        }
        for (; c < cn; ++c) cmac(ar0, ai0, ld_stream(P + (int64_t)(cb + c) * h), xw[c]);
      }
    }
  }
  if (live) {
    int idx = st.y0 + lane;
    if (yperm) idx = yperm[idx];
    y[idx] = make_double2(ar0 + ar1, ai0 + ai1);
  }
}

struct EffBlock {
  int64_t yoff, xoff, m, n;  // as applied in this direction
  int64_t raw;               // offset of the column-major block payload in the raw upload (complex)
  int64_t ld;                // original row count
  bool tr;                   // panel(i,c) = block(c, i) when transposed
  int64_t order;
};

template <int FW, int FS, int SLOT>
int flow_setup(int num_sms) {
  const size_t smem = FlowCfg<FW, FS, SLOT>::kSmem;
  cuda_check(cudaFuncSetAttribute(k1_flow<FW, FS, SLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)),
             "flow smem attribute");
  cuda_check(cudaFuncSetAttribute(k1_flow<FW, FS, SLOT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)),
             "flow smem attribute");
  cuda_check(cudaFuncSetAttribute(k1_flow<FW, FS, SLOT, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)),
             "flow smem attribute");
  int per_sm = 0;
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1_flow<FW, FS, SLOT>, flow_threads<FW>(), smem),
             "occupancy");
  if (per_sm < 1) throw detail::CudaFailure("k1_flow does not fit on an SM");
  return std::min(per_sm * num_sms, kMaxFlowCtas);
}

template <int NCB>
int k2flow_setup(int num_sms) {
  const size_t smem = K2FCfg<NCB>::kSmem;
  constexpr bool kG3 = NCB >= 2;  // (32- / 64-wide tiles: Gauss's three DMMAs by default, see launch_k2flow)
  cuda_check(cudaFuncSetAttribute(k2_flow<NCB, kG3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)),
             "k2_flow smem attribute");
  cuda_check(cudaFuncSetAttribute(k2_flow<NCB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)),
             "k2_flow smem attribute");
  int per_sm = 0, per_sm4 = 0;
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_flow<NCB, kG3>, kK2FThreads, smem), "occupancy");
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm4, k2_flow<NCB, false>, kK2FThreads, smem),
             "occupancy");
  return std::min(std::min(per_sm, per_sm4) * num_sms, kMaxFlowCtas);  // 0: unavailable
}

template <int FW, int FS, int SLOT>
void flow_launch(FlowParams& P, int grid, cudaStream_t stream, bool lite) {
  P.nwarps = grid * FW;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid), 1, 1);
  cfg.blockDim = dim3(flow_threads<FW>(), 1, 1);
  cfg.dynamicSmemBytes = FlowCfg<FW, FS, SLOT>::kSmem;
  cfg.stream = stream;
  // chained applies (flow.cuh P.pdl): programmatic dependent launch and no
  // cooperative guarantee (1 CTA per SM fits only once the previous grid
  // left); else a cooperative launch (all CTAs co-resident: they wait on each
  // other).  One attribute each way (fewer attributes, cheaper launch).
  cudaLaunchAttribute attr[1];
  if (P.pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
  } else {
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (P.prof)
    cuda_check(cudaLaunchKernelEx(&cfg, k1_flow<FW, FS, SLOT, true>, P), "k1_flow launch");
  else if (lite)
    cuda_check(cudaLaunchKernelEx(&cfg, k1_flow<FW, FS, SLOT, false, false>, P), "k1_flow launch");
  else
    cuda_check(cudaLaunchKernelEx(&cfg, k1_flow<FW, FS, SLOT>, P), "k1_flow launch");
}

}  // namespace

// One panel of the device arena cut out of the raw block payload: panel(i, c)
// = block(r0 + i, c), or block(c, r0 + i) for the transpose direction.
struct PanelJob {
  int64_t dst;  // arena offset (complex)
  int64_t src;  // raw offset of the block (complex, column-major, leading dim ld)
  int32_t h, n, ld, r0, tr, pad_;
};

// K0: one warp per panel, lanes over rows, columns in order (coalesced
// stores; the transposed gathers read rows of the block from L2).
__global__ void __launch_bounds__(256) k0_repack(const PanelJob* __restrict__ jobs, int64_t njobs,
                                                 const double2* __restrict__ raw, double2* __restrict__ arena) {
  const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= njobs) return;
  const PanelJob J = jobs[j];
  for (int c = 0; c < J.n; ++c)
    for (int i = lane; i < J.h; i += 32) {
      const int64_t r = J.r0 + i;
      arena[J.dst + static_cast<int64_t>(c) * J.h + i] =
          raw[J.src + (J.tr ? c + r * J.ld : r + static_cast<int64_t>(c) * J.ld)];
    }
}

// K0 identity detection, one warp per strip (k1_flow-eligible strips only),
// panel by panel: urow[seg*32 + r] = the column of row r's single nonzero in
// this panel when it is an exact 1 (a unit row), else -1; cinfo[column] over
// the panel's other rows = -2 (all zero), r >= 0 (a single exact 1 at row r,
// the first such column of row r in this panel), else -1 (kept).  Exact
// comparisons: the ID's identity parts are exact ones and zeros (reference
// src/linalg.cpp:278-290).
__global__ void __launch_bounds__(256) k0_units(const Strip* __restrict__ strips, int64_t nstrips,
                                                const Seg* __restrict__ segs, const double2* __restrict__ arena,
                                                int* __restrict__ urow, int8_t* __restrict__ cinfo) {
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nstrips) return;
  const Strip st = strips[t];
  if (st.nseg > kMaxSeg) return;
  const int h = st.h;
  const bool in = lane < h;
  for (int j = 0; j < st.nseg; ++j) {
    const Seg g = segs[st.seg0 + j];
    int cnt = 0, one = -1;
    if (in)
      for (int c = 0; c < g.n; ++c) {
        const double2 v = arena[g.off + static_cast<int64_t>(c) * h + lane];
        if (v.x != 0.0 || v.y != 0.0) {
          ++cnt;
          if (v.x == 1.0 && v.y == 0.0) one = c;
        }
      }
    const bool unit = in && cnt == 1 && one >= 0;
    urow[static_cast<int64_t>(st.seg0 + j) * 32 + lane] = unit ? one : -1;
    unsigned used = 0;  // rows that already have a unit column in this panel
    for (int c = 0; c < g.n; ++c) {
      double2 v = make_double2(0.0, 0.0);
      if (in && !unit) v = arena[g.off + static_cast<int64_t>(c) * h + lane];
      const unsigned nz = __ballot_sync(0xffffffffu, v.x != 0.0 || v.y != 0.0);
      const unsigned ones = __ballot_sync(0xffffffffu, v.x == 1.0 && v.y == 0.0);
      int8_t info = -1;
      if (nz == 0) {
        info = -2;
      } else if (__popc(nz) == 1 && ones == nz && !(used & nz)) {
        info = static_cast<int8_t>(__ffs(nz) - 1);
        used |= nz;
      }
      if (lane == 0) cinfo[g.pad_[0] + c] = info;
    }
  }
}

// One compressed panel: the kept columns (kcols) of the non-unit rows.
struct PackJob {
  int64_t src, dst;  // dense / compressed arena offsets (complex)
  int32_t h, hc;
  int32_t nkept, k0;  // kept columns kcols[k0, k0 + nkept)
  uint32_t urows;
  int32_t pad_;
};

__global__ void __launch_bounds__(256) k0_pack(const PackJob* __restrict__ jobs, int64_t njobs,
                                               const int* __restrict__ kcols, double2* __restrict__ arena) {
  const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= njobs) return;
  const PackJob J = jobs[j];
  if (lane >= J.h || ((J.urows >> lane) & 1u)) return;
  const int prow = __popc(~J.urows & ((1u << lane) - 1u));
  for (int q = 0; q < J.nkept; ++q)
    arena[J.dst + static_cast<int64_t>(q) * J.hc + prow] = arena[J.src + static_cast<int64_t>(kcols[J.k0 + q]) * J.h + lane];
}

// Every block's payload, factor by factor, packed back to back on the device
// (chunks of whole blocks copied in parallel into pinned memory while the
// previous chunk uploads).  offs[f][b] = complex offset of block b of factor f.
double2* upload_raw(const PlanTables& T, std::vector<std::vector<int64_t>>& offs) {
  offs.assign(T.factors.size(), {});
  struct Blk {
    const double* src;
    int64_t off, n;  // complex entries
  };
  std::vector<Blk> blks;
  int64_t total = 0;
  for (size_t f = 0; f < T.factors.size(); ++f) {
    const FactorView& F = T.factors[f];
    offs[f].resize(static_cast<size_t>(F.nblocks), 0);
    for (int64_t b = 0; b < F.nblocks; ++b) {
      const int64_t n = F.blocks[4 * b + 2] * F.blocks[4 * b + 3];
      offs[f][static_cast<size_t>(b)] = total;
      if (n > 0) blks.push_back({F.payload[static_cast<size_t>(b)], total, n});
      total += n;
    }
  }
  double2* d_raw = nullptr;
  cuda_check(cudaMalloc(&d_raw, std::max<int64_t>(total, 1) * sizeof(double2)), "cudaMalloc raw payload");
  PinnedPool& P = pinned_pool();
  std::lock_guard<std::mutex> lock(P.mu);
  P.ensure();
  cudaStream_t stream;
  cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
  const int64_t cap = static_cast<int64_t>(PinnedPool::kBytes / sizeof(double2));
  size_t i = 0;
  int buf = 0, used = 0;
  try {
    while (i < blks.size()) {
      // chunk = whole blocks up to the buffer size (a larger block goes alone, in pieces)
      size_t e = i;
      int64_t n = 0;
      while (e < blks.size() && (e == i || n + blks[e].n <= cap) && n < cap) n += blks[e++].n;
      if (used >= 2) cuda_check(cudaEventSynchronize(P.ev[buf]), "upload buffer reuse");
      const int64_t base = blks[i].off;
      if (n <= cap) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t q = static_cast<int64_t>(i); q < static_cast<int64_t>(e); ++q)
          std::memcpy(P.h[buf] + (blks[q].off - base) * sizeof(double2), blks[q].src, blks[q].n * sizeof(double2));
        cuda_check(cudaMemcpyAsync(d_raw + base, P.h[buf], n * sizeof(double2), cudaMemcpyHostToDevice, stream),
                   "raw payload H2D");
        cuda_check(cudaEventRecord(P.ev[buf], stream), "event");
        buf ^= 1;
        ++used;
      } else {  // one block larger than the buffer: synchronous pieces
        cuda_check(cudaStreamSynchronize(stream), "raw payload");
        cuda_check(cudaMemcpy(d_raw + base, blks[i].src, n * sizeof(double2), cudaMemcpyHostToDevice),
                   "raw payload H2D");
      }
      i = e;
    }
    cuda_check(cudaStreamSynchronize(stream), "raw payload upload");
  } catch (...) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
    cudaFree(d_raw);
    throw;
  }
  cudaStreamDestroy(stream);
  return d_raw;
}

// k1_flow strip records: one self-contained StripCtx per strip, dealt in
// stage order and, within a stage, by the last previous-stage strip read
// (any order inside a stage keeps the deadlock-freedom argument: every
// dependency lies in an earlier stage).  Two sets: dense (the panels as
// stored) and identity-compressed (flow.cuh, StripCtx); the compressed panels
// are appended to the arena behind the dense ones.
void Plan::build_flow_records(Direction& D, const std::vector<Strip>& strips, const std::vector<Seg>& segs) {
  const size_t ns = strips.size();
  std::vector<size_t> order(ns);
  for (size_t t = 0; t < ns; ++t) order[t] = t;
  // (measured within noise of the natural order: cfg1 64.1 vs 64.2 us,
  // cfg2 270.7 vs 272.0 us)
  auto maxdep = [&](size_t t) {
    int32_t m = 0;
    for (int j = 0; j < strips[t].nseg; ++j) m = std::max(m, segs[static_cast<size_t>(strips[t].seg0 + j)].dep1);
    return m;
  };
  for (const Stage& stg : D.stages) {
    auto b = order.begin() + stg.strip0, e = b + stg.nstrips;
    std::stable_sort(b, e, [&](size_t x, size_t y) { return maxdep(x) < maxdep(y); });
  }
  std::vector<StripCtx> dense(ns);
  for (size_t t = 0; t < ns; ++t) {
    StripCtx& c = dense[t];
    std::memset(static_cast<void*>(&c), 0, sizeof(c));
    const Strip& st = strips[order[t]];
    c.s = st;
    c.s.seg0 = static_cast<int32_t>(order[t]);
    for (int j = 0; j < st.nseg; ++j) {
      const Seg& g = segs[static_cast<size_t>(st.seg0 + j)];
      c.g[j] = FlowSeg{g.off, g.x0, g.n, 0u, 0u, st.h, 0};
    }
  }
  auto up = [](void** dptr, const void* src, size_t bytes, const char* what) {
    cuda_check(cudaMalloc(dptr, std::max<size_t>(bytes, 16)), what);
    if (bytes) cuda_check(cudaMemcpy(*dptr, src, bytes, cudaMemcpyHostToDevice), what);
  };
  up(&D.d_ctx, dense.data(), ns * sizeof(StripCtx), "upload strip records");
  for (Stage& stg : D.stages) stg.flow_bytes = stg.payload_bytes;
  D.farena_elems = 0;
  D.k2_elems = 0;
  for (const Strip& st : strips) D.k2_elems += static_cast<int64_t>(st.h) * st.xcols;
  if (ns == 0 || D.ncols_total > INT32_MAX) return;

  // identity detection on the dense panels
  const size_t nsg = segs.size();
  int* d_urow = nullptr;
  int8_t* d_cinfo = nullptr;
  cuda_check(cudaMalloc(&d_urow, std::max<size_t>(nsg, 1) * 32 * sizeof(int)), "cudaMalloc unit rows");
  cuda_check(cudaMalloc(&d_cinfo, std::max<int64_t>(D.ncols_total, 1)), "cudaMalloc unit columns");
  std::vector<int> urow(nsg * 32);
  std::vector<int8_t> cinfo(static_cast<size_t>(D.ncols_total));
  cudaError_t err = cudaMemset(d_cinfo, -1, std::max<int64_t>(D.ncols_total, 1));
  if (err == cudaSuccess) err = cudaMemset(d_urow, 0xff, std::max<size_t>(nsg, 1) * 32 * sizeof(int));
  if (err == cudaSuccess) {
    k0_units<<<static_cast<unsigned>((ns * 32 + 255) / 256), 256>>>(D.d_strips, static_cast<int64_t>(ns), D.d_segs,
                                                                     D.d_arena, d_urow, d_cinfo);
    err = cudaGetLastError();
  }
  if (err == cudaSuccess && nsg) err = cudaMemcpy(urow.data(), d_urow, nsg * 32 * sizeof(int), cudaMemcpyDeviceToHost);
  if (err == cudaSuccess && D.ncols_total)
    err = cudaMemcpy(cinfo.data(), d_cinfo, static_cast<size_t>(D.ncols_total), cudaMemcpyDeviceToHost);
  cudaFree(d_urow);
  cudaFree(d_cinfo);
  cuda_check(err, "k0_units");

  // compressed records (same deal order), panels appended behind the dense arena
  std::vector<StripCtx> comp(dense);
  std::vector<PackJob> jobs;
  std::vector<int> kcols;
  std::vector<int> wmap;  // wide compressed strips: kept columns, then add columns (per strip at wbase)
  int64_t at = D.arena_elems;  // next compressed panel (complex offset)
  auto align = [](int64_t v) { return (v + 7) & ~int64_t(7); };
  for (Stage& stg : D.stages) stg.flow_bytes = 0;
  std::vector<int> kpos;  // staged position of each dense column of the strip (-1: dropped)
  bool any = false;       // some strip compressed (possibly to no panel at all: permutation blocks)
  for (size_t t = 0; t < ns; ++t) {
    const size_t o = order[t];
    const Strip& st = strips[o];
    const int h = st.h;
    Stage& stg = D.stages[static_cast<size_t>(st.stage)];
    const int64_t dense_elems = static_cast<int64_t>(h) * st.xcols;
    if (st.nseg > kMaxSeg) {
      stg.flow_bytes += 16 * dense_elems;
      continue;
    }
    if (st.xcols > kXWin) {  // wide strip: x windows over the kept columns (wmap), adds read from x itself
      StripCtx c = dense[t];
      const size_t wb = wmap.size();
      int nkept = 0;
      for (int j = 0; j < st.nseg; ++j) {
        const Seg& g = segs[static_cast<size_t>(st.seg0 + j)];
        int nk = 0;
        for (int q = 0; q < g.n; ++q)
          if (cinfo[static_cast<size_t>(g.pad_[0] + q)] == -1) {
            wmap.push_back(q);
            ++nk;
          }
        c.g[j].n = nk;
        nkept += nk;
      }
      std::vector<int> addcols;
      int64_t comp_elems = 0;
      for (int j = 0; j < st.nseg; ++j) {
        const Seg& g = segs[static_cast<size_t>(st.seg0 + j)];
        int ucol[32];
        for (int r = 0; r < 32; ++r) ucol[r] = -1;
        for (int q = 0; q < g.n; ++q) {
          const int8_t ci = cinfo[static_cast<size_t>(g.pad_[0] + q)];
          if (ci >= 0) ucol[ci] = q;
        }
        uint32_t um = 0, am = 0;
        c.g[j].aoff = static_cast<int32_t>(addcols.size());
        for (int r = 0; r < h; ++r) {
          const int q = urow[static_cast<size_t>(st.seg0 + j) * 32 + static_cast<size_t>(r)];
          if (q >= 0) um |= 1u << r;
          const int col = q >= 0 ? q : ucol[r];
          if (col >= 0) {
            am |= 1u << r;
            addcols.push_back(col);
          }
        }
        c.g[j].hc = h - __builtin_popcount(um);
        c.g[j].urows = um;
        c.g[j].adds = am;
        if (c.g[j].hc == 0) c.g[j].n = 0;  // (every column dropped: no rows left)
        comp_elems += static_cast<int64_t>(c.g[j].hc) * c.g[j].n;
      }
      if (comp_elems >= dense_elems) {  // nothing saved: stays dense
        wmap.resize(wb);
        stg.flow_bytes += 16 * dense_elems;
        continue;
      }
      wmap.insert(wmap.end(), addcols.begin(), addcols.end());
      c.mapped = 2;
      c.wbase = static_cast<int32_t>(wb);
      c.nkept = nkept;  // (s.xcols stays > kXWin: the consumer keeps the windowed path)
      size_t k0 = wb;
      for (int j = 0; j < st.nseg; ++j) {
        const Seg& g = segs[static_cast<size_t>(st.seg0 + j)];
        const int nk = c.g[j].n, hc = c.g[j].hc;
        at = align(at);
        c.g[j].off = at;
        if (hc > 0 && nk > 0) {
          jobs.push_back({g.off, at, h, hc, nk, static_cast<int32_t>(kcols.size()), c.g[j].urows, 0});
          kcols.insert(kcols.end(), wmap.begin() + static_cast<int64_t>(k0), wmap.begin() + static_cast<int64_t>(k0) + nk);
          at += static_cast<int64_t>(hc) * nk;
        }
        k0 += static_cast<size_t>(nk);
      }
      comp[t] = c;
      any = true;
      stg.flow_bytes += 16 * comp_elems;
      continue;
    }
    StripCtx c = dense[t];
    kpos.assign(static_cast<size_t>(st.xcols), -1);
    // kept columns, panel by panel
    int nkept = 0, cb = 0;
    for (int j = 0; j < st.nseg; ++j) {
      const Seg& g = segs[static_cast<size_t>(st.seg0 + j)];
      int nk = 0;
      for (int q = 0; q < g.n; ++q)
        if (cinfo[static_cast<size_t>(g.pad_[0] + q)] == -1) {
          kpos[static_cast<size_t>(cb + q)] = nkept;
          c.cmap[nkept++] = static_cast<uint8_t>(q);
          ++nk;
        }
      c.g[j].n = nk;
      cb += g.n;
    }
    // adds: unit rows (reuse the kept column's staged entry when there is one)
    // and unit columns (an extra staged entry)
    std::vector<uint16_t> ext;
    std::vector<uint8_t> addpos;
    bool ok = true;
    int64_t comp_elems = 0;
    cb = 0;
    auto extra = [&](int j, int q) {
      const uint16_t key = static_cast<uint16_t>(j << 8 | q);
      for (size_t e = 0; e < ext.size(); ++e)
        if (ext[e] == key) return static_cast<int>(e);
      ext.push_back(key);
      return static_cast<int>(ext.size()) - 1;
    };
    std::vector<std::pair<int, int>> rowadd;  // (row, staged position)
    for (int j = 0; j < st.nseg && ok; ++j) {
      const Seg& g = segs[static_cast<size_t>(st.seg0 + j)];
      uint32_t um = 0;
      int ucol[32];
      for (int r = 0; r < 32; ++r) ucol[r] = -1;
      for (int q = 0; q < g.n; ++q) {
        const int8_t ci = cinfo[static_cast<size_t>(g.pad_[0] + q)];
        if (ci >= 0) ucol[ci] = q;
      }
      rowadd.clear();
      for (int r = 0; r < h; ++r) {
        const int q = urow[static_cast<size_t>(st.seg0 + j) * 32 + static_cast<size_t>(r)];
        if (q >= 0) {
          um |= 1u << r;
          const int kp = kpos[static_cast<size_t>(cb + q)];
          rowadd.push_back({r, kp >= 0 ? kp : nkept + extra(j, q)});
        } else if (ucol[r] >= 0) {
          rowadd.push_back({r, nkept + extra(j, ucol[r])});
        }
      }
      const int hc = h - __builtin_popcount(um);
      c.g[j].hc = hc;
      c.g[j].urows = um;
      c.g[j].adds = 0;
      c.g[j].aoff = static_cast<int32_t>(addpos.size());
      for (const auto& ra : rowadd) {
        c.g[j].adds |= 1u << ra.first;
        addpos.push_back(static_cast<uint8_t>(std::min(ra.second, 255)));
      }
      comp_elems += static_cast<int64_t>(hc) * c.g[j].n;
      cb += g.n;
      ok = addpos.size() <= 64 && ext.size() <= 32;
    }
    ok = ok && nkept + static_cast<int>(ext.size()) <= kXWin && comp_elems < dense_elems;
    if (!ok) {  // stays dense
      stg.flow_bytes += 16 * dense_elems;
      continue;
    }
    c.nkept = nkept;
    c.next = static_cast<int32_t>(ext.size());
    c.mapped = 1;
    c.s.xcols = nkept + c.next;
    for (size_t e = 0; e < ext.size(); ++e) c.xext[e] = ext[e];
    for (size_t e = 0; e < addpos.size(); ++e) c.addpos[e] = addpos[e];
    // compressed panels
    size_t k0 = 0;
    for (int j = 0; j < st.nseg; ++j) {
      const Seg& g = segs[static_cast<size_t>(st.seg0 + j)];
      const int nk = c.g[j].n, hc = c.g[j].hc;
      at = align(at);
      c.g[j].off = at;
      if (hc > 0 && nk > 0) {
        jobs.push_back({g.off, at, h, hc, nk, static_cast<int32_t>(kcols.size()), c.g[j].urows, 0});
        for (int q = 0; q < nk; ++q) kcols.push_back(c.cmap[k0 + static_cast<size_t>(q)]);
        at += static_cast<int64_t>(hc) * nk;
      }
      k0 += static_cast<size_t>(nk);  // (hc == 0: every column is dropped, nk == 0)
    }
    comp[t] = c;
    any = true;
    stg.flow_bytes += 16 * comp_elems;
  }
  D.farena_elems = at - D.arena_elems;
  if (any) build_k2_records(D, strips, segs, order, comp);
  if (!any) {  // nothing to compress: the dense records serve both
    for (Stage& stg : D.stages) stg.flow_bytes = stg.payload_bytes;
    D.d_fctx = nullptr;
    return;
  }
  if (!wmap.empty()) up(reinterpret_cast<void**>(&D.d_wmap), wmap.data(), wmap.size() * sizeof(int), "upload wide maps");
  if (jobs.empty()) {  // compressed strips stream no panel at all (permutation blocks)
    up(&D.d_fctx, comp.data(), ns * sizeof(StripCtx), "upload compressed strip records");
    return;
  }
  // arena = [dense panels | compressed panels]
  double2* arena = nullptr;
  cuda_check(cudaMalloc(&arena, std::max<int64_t>(at, 1) * sizeof(double2)), "cudaMalloc flow arena");
  PackJob* d_jobs = nullptr;
  int* d_kcols = nullptr;
  err = cudaMemcpy(arena, D.d_arena, D.arena_elems * sizeof(double2), cudaMemcpyDeviceToDevice);
  if (err == cudaSuccess) err = cudaMalloc(&d_jobs, jobs.size() * sizeof(PackJob));
  if (err == cudaSuccess) err = cudaMalloc(&d_kcols, std::max<size_t>(kcols.size(), 1) * sizeof(int));
  if (err == cudaSuccess) err = cudaMemcpy(d_jobs, jobs.data(), jobs.size() * sizeof(PackJob), cudaMemcpyHostToDevice);
  if (err == cudaSuccess) err = cudaMemcpy(d_kcols, kcols.data(), kcols.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (err == cudaSuccess) {
    const int64_t nj = static_cast<int64_t>(jobs.size());
    k0_pack<<<static_cast<unsigned>((nj * 32 + 255) / 256), 256>>>(d_jobs, nj, d_kcols, arena);
    err = cudaGetLastError();
  }
  if (err == cudaSuccess) err = cudaDeviceSynchronize();
  cudaFree(d_jobs);
  cudaFree(d_kcols);
  if (err != cudaSuccess) {
    cudaFree(arena);
    cuda_check(err, "k0_pack");
  }
  cudaFree(D.d_arena);
  D.d_arena = arena;
  up(&D.d_fctx, comp.data(), ns * sizeof(StripCtx), "upload compressed strip records");
}

// k2_flow records for the identity-compressed panels.  The DMMA tiles are 32
// rows, so unit rows save no tensor-core work; unit / zero columns shorten K.
// A strip qualifies when its compressed record has no unit rows and at most
// one identity add per row (the V-type ID strips): its panels are the
// compressed ones (h x n' per panel), its kept columns' input rows go to
// xmap, and each row's added input row to addx.  Other strips stay dense.
void Plan::build_k2_records(Direction& D, const std::vector<Strip>& strips, const std::vector<Seg>& segs,
                            const std::vector<size_t>& order, const std::vector<StripCtx>& comp) {
  const size_t ns = strips.size();
  std::vector<size_t> pos(ns);
  for (size_t t = 0; t < ns; ++t) pos[order[t]] = t;
  std::vector<Strip> ks(strips);
  std::vector<Seg> kg;
  std::vector<int> xmap, addx;
  bool any = false;
  for (size_t o = 0; o < ns; ++o) {
    const StripCtx& c = comp[pos[o]];
    const Strip& st = strips[o];
    bool ok = c.mapped == 1;
    int rowadds[32] = {0};
    for (int j = 0; ok && j < st.nseg; ++j) {
      ok = c.g[j].urows == 0;
      for (int r = 0; r < 32; ++r) rowadds[r] += (c.g[j].adds >> r) & 1u;
    }
    for (int r = 0; ok && r < 32; ++r) ok = rowadds[r] <= 1;
    if (!ok) continue;
    Strip& k = ks[o];
    k.seg0 = static_cast<int32_t>(segs.size() + kg.size());  // after the dense segs (one array)
    k.xcols = c.nkept;
    k.pad_[0] = static_cast<int32_t>(xmap.size());
    k.pad_[1] = static_cast<int32_t>(addx.size());
    int kk = 0;
    for (int j = 0; j < st.nseg; ++j) {
      Seg g = segs[static_cast<size_t>(st.seg0 + j)];
      g.off = c.g[j].off;
      g.n = c.g[j].n;
      kg.push_back(g);
      for (int q = 0; q < c.g[j].n; ++q) xmap.push_back(g.x0 + c.cmap[kk++]);
    }
    int add[32];
    for (int r = 0; r < 32; ++r) add[r] = -1;
    for (int j = 0; j < st.nseg; ++j)
      for (int r = 0; r < 32; ++r)
        if ((c.g[j].adds >> r) & 1u) {
          const int p = c.addpos[c.g[j].aoff + __builtin_popcount(c.g[j].adds & ((1u << r) - 1u))];
          const int e = p - c.nkept;  // (no unit rows: every add is an extra entry)
          const unsigned key = c.xext[e];
          add[r] = c.g[key >> 8].x0 + static_cast<int>(key & 0xffu);
        }
    addx.insert(addx.end(), add, add + 32);
    any = true;
  }
  D.k2_elems = 0;  // panel entries k2_flow multiplies (64-wide / 32-wide tiles)
  for (size_t o = 0; o < ns; ++o) D.k2_elems += static_cast<int64_t>(strips[o].h) * (any ? ks[o].xcols : strips[o].xcols);
  if (!any) return;
  std::vector<Seg> allsegs(segs);
  allsegs.insert(allsegs.end(), kg.begin(), kg.end());
  auto up = [](void** dptr, const void* src, size_t bytes, const char* what) {
    cuda_check(cudaMalloc(dptr, std::max<size_t>(bytes, 16)), what);
    if (bytes) cuda_check(cudaMemcpy(*dptr, src, bytes, cudaMemcpyHostToDevice), what);
  };
  up(reinterpret_cast<void**>(&D.d_k2strips), ks.data(), ks.size() * sizeof(Strip), "upload k2 strips");
  up(reinterpret_cast<void**>(&D.d_k2segs), allsegs.data(), allsegs.size() * sizeof(Seg), "upload k2 segs");
  up(reinterpret_cast<void**>(&D.d_k2xmap), xmap.data(), xmap.size() * sizeof(int), "upload k2 column map");
  up(reinterpret_cast<void**>(&D.d_k2addx), addx.data(), addx.size() * sizeof(int), "upload k2 adds");
}

// Build one direction (forward or transpose) of the plan on the host and
// upload it.  Strip construction is general (ragged, overlapping and
// uncovered rows): breakpoints at every block edge, active blocks in the
// reference's serial order (groups in order, blocks in group order).
void Plan::build_direction(int d, const PlanTables& T, const double2* d_raw,
                           const std::vector<std::vector<int64_t>>& raw_off) {
  Direction& D = dir[d];
  const auto t_begin = std::chrono::steady_clock::now();
  const int64_t nf = T.nfactors;
  if (nf > kMaxStages) throw std::invalid_argument("too many factors for one device plan");
  D.stages.clear();
  if (nf == 0) {  // no factors: the reference's apply_impl is the two permutations (k0_permute)
    D.in_len = d == 0 ? T.ncols : T.nrows;
    D.built = true;
    return;
  }
  D.ncols_total = 0;
  std::vector<Strip> strips;
  std::vector<Seg> segs;
  std::vector<PanelJob> jobs;
  int64_t arena_len = 0;  // complex entries
  // stage buffer layout: [permuted input of stage 0 | output of stage 0 | ...]
  D.in_len = d == 0 ? T.factors[static_cast<size_t>(nf - 1)].cols : T.factors[0].rows;
  int64_t bufoff = std::max<int64_t>(D.in_len, 1);

  for (int64_t s = 0; s < nf; ++s) {
    const int64_t fi = d == 0 ? nf - 1 - s : s;
    const FactorView& F = T.factors[static_cast<size_t>(fi)];
    Stage stg;
    stg.out_len = d == 0 ? F.rows : F.cols;
    stg.in_len = d == 0 ? F.cols : F.rows;
    stg.strip0 = static_cast<int32_t>(strips.size());
    stg.arena0 = arena_len;
    stg.buf_off = bufoff;
    if (s + 1 < nf) bufoff += std::max<int64_t>(stg.out_len, 1);
    if (s > 0 && stg.in_len != D.stages.back().out_len)
      throw std::invalid_argument("consecutive factors have mismatched inner dimensions");
    std::vector<EffBlock> eb;
    int64_t ord = 0;
    for (int64_t g = 0; g < F.ngroups; ++g) {
      for (int64_t b = F.groups[2 * g]; b < F.groups[2 * g + 1]; ++b) {
        const int64_t* bd = F.blocks + 4 * b;
        if (bd[2] == 0 || bd[3] == 0) continue;
        EffBlock e;
        e.ld = bd[2];
        e.raw = raw_off[static_cast<size_t>(fi)][static_cast<size_t>(b)];
        e.order = ord++;
        e.tr = d != 0;
        e.yoff = d == 0 ? bd[0] : bd[1];
        e.xoff = d == 0 ? bd[1] : bd[0];
        e.m = d == 0 ? bd[2] : bd[3];
        e.n = d == 0 ? bd[3] : bd[2];
        eb.push_back(e);
      }
    }
    std::vector<int64_t> bp{0, stg.out_len};
    for (const auto& e : eb) {
      bp.push_back(e.yoff);
      bp.push_back(e.yoff + e.m);
    }
    std::sort(bp.begin(), bp.end());
    bp.erase(std::unique(bp.begin(), bp.end()), bp.end());
    std::vector<int64_t> by_start(eb.size());
    for (size_t i = 0; i < eb.size(); ++i) by_start[i] = static_cast<int64_t>(i);
    std::sort(by_start.begin(), by_start.end(), [&](int64_t a, int64_t b) { return eb[a].yoff < eb[b].yoff; });
    std::set<std::pair<int64_t, int64_t>> active;  // (order, index)
    size_t next = 0;
    // producers of the previous stage, for dependency ranges
    const int32_t prev0 = s > 0 ? D.stages.back().strip0 : 0;
    const int32_t prev1 = s > 0 ? D.stages.back().strip0 + D.stages.back().nstrips : 0;
    auto deps = [&](int64_t x0, int64_t n, int32_t& d0, int32_t& d1) {
      if (s == 0) {
        d0 = d1 = 0;
        return;
      }
      // first strip with y0 + h > x0, one past the last strip with y0 < x0 + n
      int32_t lo = prev0, hi = prev1;
      while (lo < hi) {
        const int32_t mid = (lo + hi) / 2;
        if (strips[mid].y0 + strips[mid].h > x0) hi = mid; else lo = mid + 1;
      }
      d0 = lo;
      hi = prev1;
      while (lo < hi) {
        const int32_t mid = (lo + hi) / 2;
        if (strips[mid].y0 < x0 + n) lo = mid + 1; else hi = mid;
      }
      d1 = lo;
    };
    for (size_t q = 0; q + 1 < bp.size(); ++q) {
      const int64_t a = bp[q], b = bp[q + 1];
      if (a >= stg.out_len) break;
      while (next < by_start.size() && eb[by_start[next]].yoff <= a) {
        const int64_t i = by_start[next++];
        active.insert({eb[i].order, i});
      }
      for (auto it = active.begin(); it != active.end();) {
        if (eb[it->second].yoff + eb[it->second].m <= a)
          it = active.erase(it);
        else
          ++it;
      }
      for (int64_t y = a; y < b; y += strip_rows) {
        const int h = static_cast<int>(std::min<int64_t>(strip_rows, b - y));
        Strip st{};
        st.pad_[0] = st.pad_[1] = -1;  // k2_flow: dense strip (no identity maps)
        st.y0 = static_cast<int32_t>(y);
        st.h = h;
        st.seg0 = static_cast<int32_t>(segs.size());
        st.stage = static_cast<int32_t>(s);
        for (const auto& pr : active) {
          const EffBlock& e = eb[pr.second];
          Seg sg{};
          // 128-byte aligned panels: every full TMA chunk (h x 32 columns)
          // then starts on a cache-line boundary (unaligned bulk copies
          // stream at a fraction of the rate, tools/bw_probe.cu)
          arena_len = (arena_len + 7) & ~int64_t(7);
          sg.off = arena_len;
          sg.x0 = static_cast<int32_t>(e.xoff);
          sg.n = static_cast<int32_t>(e.n);
          sg.pad_[0] = static_cast<int32_t>(std::min<int64_t>(D.ncols_total, INT32_MAX));  // column base (k0_units)
          D.ncols_total += e.n;
          deps(e.xoff, e.n, sg.dep0, sg.dep1);
          jobs.push_back({arena_len, e.raw, h, static_cast<int32_t>(e.n), static_cast<int32_t>(e.ld),
                          static_cast<int32_t>(y - e.yoff), e.tr ? 1 : 0, 0});
          arena_len += static_cast<int64_t>(h) * e.n;
          segs.push_back(sg);
          ++st.nseg;
          st.xcols += sg.n;
        }
        D.max_seg = std::max(D.max_seg, static_cast<int>(st.nseg));
        D.max_xcols = std::max(D.max_xcols, static_cast<int>(st.xcols));
        D.max_strip_bytes = std::max<int64_t>(D.max_strip_bytes, int64_t{16} * st.h * st.xcols);
        strips.push_back(st);
      }
    }
    stg.nstrips = static_cast<int32_t>(strips.size()) - stg.strip0;
    stg.payload_bytes = 16 * (arena_len - stg.arena0);
    D.stages.push_back(stg);
  }
  if (strips.size() > 0x7ffffff0 || segs.size() > 0x7ffffff0)
    throw std::invalid_argument("factorization too large for one device plan");
  const auto t_meta = std::chrono::steady_clock::now();
  D.nstrips = static_cast<int64_t>(strips.size());
  D.nsegs = static_cast<int64_t>(segs.size());
  D.arena_elems = arena_len;
  D.stagebuf_elems = std::max<int64_t>(bufoff, 1);
  auto up = [](void** dptr, const void* src, size_t bytes, const char* what) {
    cuda_check(cudaMalloc(dptr, std::max<size_t>(bytes, 16)), what);
    if (bytes) cuda_check(cudaMemcpy(*dptr, src, bytes, cudaMemcpyHostToDevice), what);
  };
  up(reinterpret_cast<void**>(&D.d_strips), strips.data(), strips.size() * sizeof(Strip), "upload strips");
  up(reinterpret_cast<void**>(&D.d_segs), segs.data(), segs.size() * sizeof(Seg), "upload segs");
  // panels cut out of the raw payload on the device (K0)
  cuda_check(cudaMalloc(&D.d_arena, std::max<int64_t>(arena_len, 1) * sizeof(double2)), "cudaMalloc arena");
  if (!jobs.empty()) {
    PanelJob* d_jobs = nullptr;
    up(reinterpret_cast<void**>(&d_jobs), jobs.data(), jobs.size() * sizeof(PanelJob), "upload panel jobs");
    const int64_t nj = static_cast<int64_t>(jobs.size());
    k0_repack<<<static_cast<unsigned>((nj * 32 + 255) / 256), 256>>>(d_jobs, nj, d_raw, D.d_arena);
    const cudaError_t e = cudaGetLastError();
    const cudaError_t e2 = e == cudaSuccess ? cudaDeviceSynchronize() : e;
    cudaFree(d_jobs);
    cuda_check(e2, "k0_repack");
  }
  // two parity sets, armed with the all-ones sentinel (k1_flow's ready signal)
  cuda_check(cudaMalloc(&D.d_stagebuf, 2 * D.stagebuf_elems * sizeof(double2)), "cudaMalloc stage buffer");
  cuda_check(cudaMemset(D.d_stagebuf, 0xff, 2 * D.stagebuf_elems * sizeof(double2)), "arm stage buffers");
  cuda_check(cudaMalloc(&D.d_sync, kMaxFlowCtas * sizeof(unsigned)), "cudaMalloc sync");
  cuda_check(cudaMemset(D.d_sync, 0, kMaxFlowCtas * sizeof(unsigned)), "memset sync");
  if (D.max_seg <= kMaxSeg) build_flow_records(D, strips, segs);
  D.built = true;
  if (std::getenv("MIDBF_PLAN_TIMING"))
    std::fprintf(stderr, "[plan] dir %d: metadata %.1f ms, repack+uploads %.1f ms (%lld strips, %lld segs)\n", d,
                 1e3 * std::chrono::duration<double>(t_meta - t_begin).count(),
                 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t_meta).count(),
                 static_cast<long long>(D.nstrips), static_cast<long long>(D.nsegs));
}

// Table checks the reference's apply relies on (src/butterfly.cpp:642-667):
// permutation entries index the outer spaces (they drive device gathers and
// scatters), the outermost factors match the outer dimensions, and a
// factor-free plan is square (apply_impl then only permutes).
static void check_tables(const PlanTables& T) {
  auto perm_ok = [](const int64_t* p, int64_t n, const char* what) {
    std::vector<char> seen(static_cast<size_t>(std::max<int64_t>(n, 0)), 0);
    for (int64_t i = 0; i < n; ++i) {
      if (p[i] < 0 || p[i] >= n) throw std::invalid_argument(std::string(what) + " permutation entry out of range");
      if (seen[static_cast<size_t>(p[i])]++) throw std::invalid_argument(std::string(what) + " permutation repeats an index");
    }
  };
  if (T.nrows < 0 || T.ncols < 0 || T.nfactors < 0) throw std::invalid_argument("negative plan dimension");
  perm_ok(T.row_perm, T.nrows, "row");
  perm_ok(T.col_perm, T.ncols, "column");
  if (T.nfactors == 0) {
    if (T.nrows != T.ncols) throw std::invalid_argument("a factorization without factors must be square");
    return;
  }
  if (T.factors.front().rows != T.nrows) throw std::invalid_argument("first factor rows do not match nrows");
  if (T.factors.back().cols != T.ncols) throw std::invalid_argument("last factor columns do not match ncols");
  for (size_t f = 0; f + 1 < T.factors.size(); ++f)
    if (T.factors[f].cols != T.factors[f + 1].rows) throw std::invalid_argument("adjacent factor shapes do not chain");
}

// Factor-free plans: out[out_perm[p]] = in[in_perm[p]] per column.
__global__ void __launch_bounds__(256) k0_permute(const double2* __restrict__ in, double2* __restrict__ out,
                                                  const int* __restrict__ in_perm, const int* __restrict__ out_perm,
                                                  int64_t n, int64_t nrhs) {
  const int64_t total = n * nrhs;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = i / n, p = i - c * n;
    out[c * n + out_perm[p]] = in[c * n + in_perm[p]];
  }
}

Plan::Plan(const PlanTables& T, unsigned directions, double2* d_raw_in) {
  check_tables(T);
  device = require_device();
  if (const char* e = std::getenv("MIDBF_STRIP_ROWS")) {  // experiments: strip height 1..32
    const int v = std::atoi(e);
    if (v >= 1 && v <= 32) strip_rows = v;
  }
  cuda_check(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device), "SM count");
  nrows = T.nrows;
  ncols = T.ncols;
  nfactors = T.nfactors;
  total_nnz = T.total_nnz;
  if (nrows > 0x7fffffff || ncols > 0x7fffffff) throw std::invalid_argument("dimension exceeds int32 range");
  max_len = std::max(nrows, ncols);
  for (const auto& F : T.factors) max_len = std::max({max_len, F.rows, F.cols});
  std::vector<int> rp(T.row_perm, T.row_perm + nrows), cp(T.col_perm, T.col_perm + ncols);
  cuda_check(cudaMalloc(&d_row_perm, std::max<int64_t>(1, nrows) * sizeof(int)), "cudaMalloc perm");
  cuda_check(cudaMalloc(&d_col_perm, std::max<int64_t>(1, ncols) * sizeof(int)), "cudaMalloc perm");
  cuda_check(cudaMemcpy(d_row_perm, rp.data(), rp.size() * sizeof(int), cudaMemcpyHostToDevice), "upload perm");
  cuda_check(cudaMemcpy(d_col_perm, cp.data(), cp.size() * sizeof(int), cudaMemcpyHostToDevice), "upload perm");
  static const bool timing = std::getenv("MIDBF_PLAN_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return 1e3 * std::chrono::duration<double>(b - a).count(); };
  const auto t0 = now();
  std::vector<std::vector<int64_t>> raw_off;
  double2* d_raw = nullptr;
  if (d_raw_in) {  // payload already on the device, blocks back to back in table order
    d_raw = d_raw_in;
    int64_t at = 0;
    raw_off.resize(T.factors.size());
    for (size_t f = 0; f < T.factors.size(); ++f)
      for (int64_t b = 0; b < T.factors[f].nblocks; ++b) {
        raw_off[f].push_back(at);
        at += T.factors[f].blocks[4 * b + 2] * T.factors[f].blocks[4 * b + 3];
      }
  } else {
    d_raw = upload_raw(T, raw_off);
  }
  const auto t1 = now();
  try {
    for (int d = 0; d < 2; ++d)
      if (directions & (1u << d)) build_direction(d, T, d_raw, raw_off);
  } catch (...) {
    cudaFree(d_raw);
    throw;
  }
  cudaFree(d_raw);
  const auto t2 = now();
  if (timing) std::fprintf(stderr, "[plan] raw upload %.1f ms, directions %.1f ms\n", ms(t0, t1), ms(t1, t2));
  flow_grid[0] = flow_setup<4, 3, 16384>(num_sms);
  flow_grid[1] = flow_setup<8, 2, 8192>(num_sms);
  flow_grid[2] = flow_grid[1];  // variant 2 (6 pairs x 3 x 8 KB) retired: it deadlocked at cfg3
  flow_grid[3] = flow_grid[0];  // unused: variant 3 resolves per direction (flow_variant)
  {
    cuda_check(cudaFuncSetAttribute(k1_coop<kCoopWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kCoopSmem)),
               "coop smem attribute");
    int per_sm = 0;
    cuda_check(
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1_coop<kCoopWarps>, kCoopWarps * 32, kCoopSmem),
        "occupancy");
    coop_grid = std::min(per_sm * num_sms, kMaxFlowCtas);
  }
  cuda_check(cudaFuncSetAttribute(k2_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kK2Smem)),
             "k2 smem attribute");
  k2flow_grid[0] = k2flow_setup<1>(num_sms);  // 16-wide tiles
  k2flow_grid[1] = k2flow_setup<2>(num_sms);  // 32
  k2flow_grid[2] = k2flow_setup<4>(num_sms);  // 64
  // one grid for every width: the per-CTA launch epochs (k2flow.cuh) assume
  // every launch runs the same set of CTAs
  const int g = std::min({k2flow_grid[0], k2flow_grid[1], k2flow_grid[2]});
  for (int& v : k2flow_grid) v = g;
  cuda_check(cudaEventCreateWithFlags(&ev_last, cudaEventDisableTiming), "event");
}

Plan::~Plan() {
  for (auto& D : dir) {
    cudaFree(D.d_strips);
    cudaFree(D.d_segs);
    cudaFree(D.d_arena);
    cudaFree(D.d_ctx);
    cudaFree(D.d_fctx);
    cudaFree(D.d_wmap);
    cudaFree(D.d_k2strips);
    cudaFree(D.d_k2segs);
    cudaFree(D.d_k2xmap);
    cudaFree(D.d_k2addx);
    cudaFree(D.d_k2buf);
    cudaFree(D.d_k2done);
    cudaFree(D.d_k2epoch);
    cudaFree(D.d_stagebuf);
    cudaFree(D.d_stageio);
    cudaFree(D.d_sync);
  }
  for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
  if (ev_last) cudaEventDestroy(ev_last);
  cudaFree(d_inflag);
  if (s_h2d) {
    cudaStreamSynchronize(s_d2h);
    for (auto& a : aslots) {
      cudaFree(a.d_in);
      cudaFree(a.d_out);
      cudaEventDestroy(a.in_ready);
      cudaEventDestroy(a.applied);
      cudaEventDestroy(a.done);
    }
    cudaEventDestroy(ev_user);
    cudaStreamDestroy(s_h2d);
    cudaStreamDestroy(s_comp);
    cudaStreamDestroy(s_d2h);
  }
  cudaFree(d_prof);
  cudaFree(d_row_perm);
  cudaFree(d_col_perm);
  cudaFree(d_buf[0]);
  cudaFree(d_buf[1]);
  cudaFree(d_io[0]);
  cudaFree(d_io[1]);
}

// k1_flow variant: flags bits 4-5 (0: 4 pairs x 3 x 16 KB, 1: 8 x 2 x 8 KB,
// 2: retired -- 6 x 3 x 8 KB never won and hung at cfg3 -- runs 1), 3 = by size: measured at cfg1 (358 MB of panels) variant
// 0 is fastest (66.5 vs 74.7 us), at cfg3 / cfg2 (872 / 1726 MB) variant 1
// (135.7 vs 140.6, 275.1 vs 287.2 us) -- more warps pay off once every
// warp streams enough panels to amortise its pipeline start and stage waits.
int Plan::flow_variant(int d) const {
  const int v = static_cast<int>((flags >> 4) & 3u);
  if (v != 3) return v;
  int64_t bytes = 0;
  const bool dense = flow_dense(d);
  for (const auto& st : dir[d].stages) bytes += dense ? st.payload_bytes : st.flow_bytes;
  return bytes > (int64_t{512} << 20) ? 1 : 0;
}

// Dense-only k1_flow (no identity-compression code on the strips' critical
// path) for small plans (< 200 MB of panels), or with flag bit 10 (bit 16:
// never): the extra per-strip work of
// the compressed kernel costs more than the bytes it saves when each warp pair
// owns at most a strip or two per stage (measured).
bool Plan::flow_lite(int d) const {
  if (flags & 65536u) return false;  // bit 16: always the compressed kernel
  if (flags & 1024u) return true;
  int64_t bytes = 0;
  for (const auto& st : dir[d].stages) bytes += st.payload_bytes;
  // measured (round 1, tools/flow_ab.py; us per apply, default | dense-only |
  // compressed): cfg0 7.6 MB 17.0 | 16.9 | 19.2, cfg1_unitxi 145 MB
  // 37.0 (dense-only) vs 40.2, cfg1 358 MB 62.5 (dense-only) vs 55.2
  return bytes < (int64_t{200} << 20);
}

// k1_coop for small plans (coop.cuh): dense strip records, x windows of at
// most kCoopX entries.  Default below kCoopBytes of panels (measured, DESIGN.md
// "small plans"); flag bit 18 forces it, bit 19 forbids it.
// cfg0 (7.6 MB, L2-resident): k1_flow 14.5 us, k1_coop 9.4 us; at cfg1_unitxi
// (145 MB) k1_coop streams far below k1_flow (115 vs 33.6 us): it has one
// strip in flight per SM and no warp specialisation.
constexpr int64_t kCoopBytes = int64_t{32} << 20;
bool Plan::coop(int d) const {
  if (flags & kFlagNoCoop) return false;
  if (dir[d].max_xcols > kCoopX || dir[d].max_strip_bytes > kCoopSlotBytes || coop_grid <= 0 || !dir[d].d_ctx)
    return false;
  if (flags & kFlagCoop) return true;
  // by size only on the fully default path: an explicit k1_flow layout
  // (variant bits), dense-only (bit 10) or compressed (bit 16) choice wins
  if (((flags >> 4) & 3u) != 3u || (flags & (1024u | 65536u))) return false;
  int64_t bytes = 0;
  for (const auto& st : dir[d].stages) bytes += st.payload_bytes;
  return bytes < kCoopBytes;
}

bool Plan::flow_dense(int d) const { return !dir[d].d_fctx || (flags & 512u) || flow_lite(d); }

// Up to kFlowColumns right-hand sides run k1_flow once per column: at cfg1 a
// column costs ~66 us, the narrowest DMMA slice (16 wide) ~155 us.
bool Plan::flow_ok(int d, int64_t nrhs) const {
  return nrhs >= 1 && nrhs <= kFlowColumns && (flags & 8u) && dir[d].max_seg <= kMaxSeg;
}

int64_t Plan::launches_per_apply(int d, int64_t nrhs) const {
  if (dir[d].stages.empty()) return nrows * nrhs > 0 ? 1 : 0;  // k0_permute
  if (flow_ok(d, nrhs)) return nrhs;
  if (k2flow_ok(d, nrhs)) return (nrhs + kK2Rhs - 1) / kK2Rhs;
  if (k2_ok(d, nrhs)) {
    int64_t n = 0;
    for (const auto& st : dir[d].stages) n += st.nstrips > 0;
    return n;
  }
  return static_cast<int64_t>(dir[d].stages.size());
}

void Plan::ensure_buffers(int64_t nrhs) {
  const int64_t need = std::max<int64_t>(1, max_len) * nrhs;
  if (need > buf_elems) {
    cudaFree(d_buf[0]);
    cudaFree(d_buf[1]);
    d_buf[0] = d_buf[1] = nullptr;
    cuda_check(cudaMalloc(&d_buf[0], need * sizeof(double2)), "cudaMalloc work vector");
    cuda_check(cudaMalloc(&d_buf[1], need * sizeof(double2)), "cudaMalloc work vector");
    buf_elems = need;
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
}

// The k1_flow / k1_coop stage table (FlowParams::st) on the device, once per
// direction, outside any stream capture.
void Plan::ensure_stageio(int d) {
  Direction& D = dir[d];
  if (!D.d_stageio) {
    const int ns = static_cast<int>(D.stages.size());
    std::vector<StageIO> st(static_cast<size_t>(ns));
    for (int s = 0; s < ns; ++s) {
      StageIO& io = st[static_cast<size_t>(s)];
      io.x = s == 0 ? D.d_stagebuf : D.d_stagebuf + D.stages[s - 1].buf_off;  // stage 0: permuted input
      io.y = s == ns - 1 ? nullptr : D.d_stagebuf + D.stages[s].buf_off;   // last stage: FlowParams::out
      io.xperm = nullptr;
      io.yperm = s == ns - 1 ? (d == 0 ? d_row_perm : d_col_perm) : nullptr;
      io.x_par = 1;
      io.y_par = s == ns - 1 ? 0 : 1;
    }
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(16, st.size() * sizeof(StageIO))), "cudaMalloc stage table");
    cuda_check(cudaMemcpy(p, st.data(), st.size() * sizeof(StageIO), cudaMemcpyHostToDevice), "upload stage table");
    D.d_stageio = static_cast<StageIO*>(p);
  }
}

void Plan::launch_flow(int d, const double2* in, double2* out, cudaStream_t stream) {
  Direction& D = dir[d];
  const int variant = flow_variant(d);
  FlowParams P{};
  // bit 9: dense panels (identity compression off, A/B experiments)
  const bool lite = flow_lite(d);
  P.ctxs = static_cast<const StripCtx*>(flow_dense(d) ? D.d_ctx : D.d_fctx);
  P.strips = D.d_strips;
  P.segs = D.d_segs;
  P.arena = D.d_arena;
  P.wmap = D.d_wmap;
  P.epoch = D.d_sync;
  P.stagebuf = D.d_stagebuf;
  P.par_elems = D.stagebuf_elems;
  P.nstrips = static_cast<int>(D.nstrips);
  P.nodeps = static_cast<int>((flags >> 6) & 7u);  // bits 6-8: timing experiments
  if ((flags & 4096u) && d_prof) P.prof = d_prof;  // bit 12: phase timers (experiments)
  P.st = D.d_stageio;
  P.nstages = static_cast<int>(D.stages.size());
  P.out = out;
  P.in = in;
  P.in_flag = next_in_flag;
  P.in_seq = next_in_seq;
  P.in_perm = d == 0 ? d_col_perm : d_row_perm;
  P.in_len = D.in_len;
  P.arena_len = D.arena_elems + D.farena_elems;
  P.out_len = d == 0 ? nrows : ncols;
  P.pdl = (flags & kFlagChain) ? 1 : 0;
  P.l2_first = (flags & kFlagL2Normal) ? 0 : 1;
  // Stage 0 gathers the user input through the permutation itself (no
  // stage -1 prologue), its permutation indices loaded before the chained
  // wait; 4-pair layout only (separate stager warps): measured cfg1 51.7 ->
  // 50.1 us, cfg1_unitxi 36.4 -> 35.1; with the 8-pair layout's in-warp
  // stager cfg2 got slower (242 -> 245 us).  Flag bit 24 keeps the prologue.
  P.direct0 = (variant == 0 && !(flags & kFlagPrologue)) ? 1 : 0;
  if (coop(d)) {
    P.ctxs = static_cast<const StripCtx*>(D.d_ctx);  // dense records
    P.nwarps = coop_grid;
    P.direct0 = (flags & kFlagPrologue) ? 0 : 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(coop_grid), 1, 1);
    cfg.blockDim = dim3(kCoopWarps * 32, 1, 1);
    cfg.dynamicSmemBytes = kCoopSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];  // as flow_launch
    if (P.pdl) {
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
    } else {
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, k1_coop<kCoopWarps>, P), "k1_coop launch");
    return;
  }
  switch (variant) {
    case 1:
    case 2:  // retired variant: runs variant 1
      flow_launch<8, 2, 8192>(P, flow_grid[1], stream, lite);
      break;
    default:
      flow_launch<4, 3, 16384>(P, flow_grid[0], stream, lite);
  }
}

void Plan::launch_stages(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream) {
  const Direction& D = dir[d];
  const int ns = static_cast<int>(D.stages.size());
  const int* in_perm = d == 0 ? d_col_perm : d_row_perm;
  const int* out_perm = d == 0 ? d_row_perm : d_col_perm;
  for (int s = 0; s < ns; ++s) {
    const Stage& st = D.stages[s];
    const double2* x = s == 0 ? in : d_buf[(s - 1) & 1];
    double2* y = s == ns - 1 ? out : d_buf[s & 1];
    const int64_t xld = s == 0 ? (d == 0 ? ncols : nrows) : max_len;
    const int64_t yld = s == ns - 1 ? (d == 0 ? nrows : ncols) : max_len;
    const int* xp = s == 0 ? in_perm : nullptr;
    const int* yp = s == ns - 1 ? out_perm : nullptr;
    const int nblk = std::max(1, (st.nstrips + kWarps - 1) / kWarps);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(nblk), static_cast<unsigned>(nrhs), 1);
    cfg.blockDim = dim3(kWarps * 32, 1, 1);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (flags & 1u) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const Strip* sp = D.d_strips + st.strip0;
    if (flags & 2u)
      cuda_check(cudaLaunchKernelEx(&cfg, k1_stage<true>, sp, st.nstrips, (const Seg*)D.d_segs,
                                    (const double2*)D.d_arena, x, xld, xp, y, yld, yp),
                 "k1_stage launch");
    else
      cuda_check(cudaLaunchKernelEx(&cfg, k1_stage<false>, sp, st.nstrips, (const Seg*)D.d_segs,
                                    (const double2*)D.d_arena, x, xld, xp, y, yld, yp),
                 "k1_stage launch");
  }
}

// K2: one DMMA launch per stage, chained with programmatic dependent launch.
void Plan::launch_k2(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream) {
  const Direction& D = dir[d];
  const int ns = static_cast<int>(D.stages.size());
  const int* in_perm = d == 0 ? d_col_perm : d_row_perm;
  const int* out_perm = d == 0 ? d_row_perm : d_col_perm;
  for (int s = 0; s < ns; ++s) {
    const Stage& st = D.stages[s];
    if (st.nstrips == 0) continue;
    const double2* x = s == 0 ? in : d_buf[(s - 1) & 1];
    double2* y = s == ns - 1 ? out : d_buf[s & 1];
    const int64_t xld = s == 0 ? (d == 0 ? ncols : nrows) : max_len;
    const int64_t yld = s == ns - 1 ? (d == 0 ? nrows : ncols) : max_len;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(st.nstrips), static_cast<unsigned>((nrhs + kK2Rhs - 1) / kK2Rhs), 1);
    cfg.blockDim = dim3(kK2Threads, 1, 1);
    cfg.dynamicSmemBytes = kK2Smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, k2_stage, (const Strip*)(D.d_strips + st.strip0), (const Seg*)D.d_segs,
                                  (const double2*)D.d_arena, x, xld, s == 0 ? in_perm : nullptr, y, yld,
                                  s == ns - 1 ? out_perm : nullptr, static_cast<int>(nrhs)),
               "k2_stage launch");
  }
}

bool Plan::k2flow_ok(int d, int64_t nrhs) const {
  return k2_ok(d, nrhs) && !(flags & 8192u) && k2flow_grid[0] > 0 && k2flow_grid[1] > 0 && k2flow_grid[2] > 0;
}

void Plan::ensure_k2flow(int d) {
  Direction& D = dir[d];
  if (D.d_k2done) return;
  int64_t rows = 0;
  for (size_t s = 0; s + 1 < D.stages.size(); ++s) rows += D.stages[s].out_len;
  cuda_check(cudaMalloc(&D.d_k2buf, std::max<int64_t>(rows, 1) * kK2Xs * sizeof(double2)), "cudaMalloc k2 stages");
  cuda_check(cudaMalloc(&D.d_k2done, std::max<int64_t>(D.nstrips, 1) * sizeof(unsigned)), "cudaMalloc k2 counters");
  cuda_check(cudaMalloc(&D.d_k2epoch, kMaxFlowCtas * sizeof(unsigned)), "cudaMalloc k2 epochs");
  cuda_check(cudaMemset(D.d_k2done, 0, std::max<int64_t>(D.nstrips, 1) * sizeof(unsigned)), "reset k2 counters");
  cuda_check(cudaMemset(D.d_k2epoch, 0, kMaxFlowCtas * sizeof(unsigned)), "reset k2 epochs");
}

// K2-flow: one cooperative dataflow launch per 64-RHS slice (k2flow.cuh).
void Plan::launch_k2flow(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream) {
  const Direction& D = dir[d];
  const int ns = static_cast<int>(D.stages.size());
  const int64_t in_ld = d == 0 ? ncols : nrows, out_ld = d == 0 ? nrows : ncols;
  K2FParams P{};
  // identity-compressed V panels (flag bit 9: dense) on 32- and 64-wide tiles;
  // the 16-wide tiles are latency-bound and lose more to the end-of-strip
  // identity adds and the split input-row copies than the shorter K saves
  // (cfg1: 16 RHS 171.6 vs 162.4 us; 24 / 48 / 64 RHS 204 / 357 / 377 vs
  // 217 / 402 / 392 us)
  const bool comp = D.d_k2strips && !(flags & 512u);
  P.xmap = D.d_k2xmap;
  P.addx = D.d_k2addx;
  P.arena_len = D.arena_elems + D.farena_elems;
  P.arena = D.d_arena;
  P.done = D.d_k2done;
  P.epoch = D.d_k2epoch;
  P.nstrips = static_cast<int>(D.nstrips);
  P.nstages = ns;
  P.mode = static_cast<int>((flags >> 14) & 3u);
  P.l2_first = (flags & kFlagK2L2Normal) ? 0 : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kK2FThreads, 1, 1);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // CTAs wait on each other's strips
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int64_t c0 = 0; c0 < nrhs; c0 += kK2Rhs) {
    P.ncv = static_cast<int>(std::min<int64_t>(kK2Rhs, nrhs - c0));
    const int wi = P.ncv <= 16 ? 0 : (P.ncv <= 32 ? 1 : 2);  // narrowest tile covering the slice
    P.strips = comp && wi > 0 ? D.d_k2strips : D.d_strips;
    P.segs = comp && wi > 0 ? D.d_k2segs : D.d_segs;
    const int64_t xs = (16 << wi) + 2;                      // its X / stage-row stride
    cfg.gridDim = dim3(static_cast<unsigned>(k2flow_grid[wi]), 1, 1);
    int64_t off = 0;
    for (int s = 0; s < ns; ++s) {
      K2FStage& io = P.st[s];
      const int64_t len = D.stages[static_cast<size_t>(s)].out_len;
      if (s == 0) {
        io.x = in + c0 * in_ld;
        io.xld = in_ld;
        io.xperm = d == 0 ? d_col_perm : d_row_perm;
      } else {
        io.x = P.st[s - 1].y;
        io.xld = P.st[s - 1].yld;
        io.xperm = nullptr;
      }
      if (s == ns - 1) {
        io.y = out + c0 * out_ld;
        io.yld = out_ld;
        io.yperm = d == 0 ? d_row_perm : d_col_perm;
      } else {
        io.y = D.d_k2buf + off * xs;
        io.yld = xs;  // row-major, RHS fastest, rows padded to the smem slot stride
        io.yperm = nullptr;
        off += len;
      }
    }
    // Gauss's three real DMMAs per complex product on 32- and 64-wide tiles
    // (cfg4, 64 RHS: 377 -> 366 us; 32 RHS 209 -> 194 us, 24 RHS 204 -> 189
    // us); the 16-wide tiles measured slower with it (162 -> 166 us at 16
    // RHS, 158 -> 161 at 8), so they keep four.  Flag bit 26 forces four
    // everywhere (A/B).
    const bool mul4 = (flags & kFlagK2Mul4) != 0;
    switch (wi) {
      case 0:
        cfg.dynamicSmemBytes = K2FCfg<1>::kSmem;
        cuda_check(cudaLaunchKernelEx(&cfg, k2_flow<1, false>, P), "k2_flow launch");
        break;
      case 1:
        cfg.dynamicSmemBytes = K2FCfg<2>::kSmem;
        cuda_check(cudaLaunchKernelEx(&cfg, mul4 ? k2_flow<2, false> : k2_flow<2, true>, P), "k2_flow launch");
        break;
      default:
        cfg.dynamicSmemBytes = K2FCfg<4>::kSmem;
        cuda_check(cudaLaunchKernelEx(&cfg, mul4 ? k2_flow<4, false> : k2_flow<4, true>, P), "k2_flow launch");
    }
  }
}

bool Plan::k2_ok(int d, int64_t nrhs) const {
  return nrhs > 1 && !(flags & 2048u) && dir[d].max_seg <= kK2MaxSeg;
}

void Plan::launch(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream) {
  if (flow_ok(d, nrhs)) {
    const int64_t in_ld = d == 0 ? ncols : nrows, out_ld = d == 0 ? nrows : ncols;
    for (int64_t c = 0; c < nrhs; ++c) launch_flow(d, in + c * in_ld, out + c * out_ld, stream);
  } else if (k2flow_ok(d, nrhs))
    launch_k2flow(d, in, out, nrhs, stream);
  else if (k2_ok(d, nrhs))
    launch_k2(d, in, out, nrhs, stream);
  else
    launch_stages(d, in, out, nrhs, stream);
}

// Device-operand apply; the launch sequence is captured once per operand set
// into a CUDA graph.
// k1_flow keeps per-CTA apply epochs (parity of the stage-buffer set) that
// assume one grid size; a variant switch re-initialises them, outside any
// stream capture and after all earlier work.
void Plan::prepare_flow(int d) {
  const int grid = coop(d) ? (coop_grid | (1 << 20)) : flow_grid[flow_variant(d)];
  if (last_grid[d] == grid) return;
  Direction& D = dir[d];
  cuda_check(cudaDeviceSynchronize(), "flow reset sync");
  cuda_check(cudaMemset(D.d_sync, 0, kMaxFlowCtas * sizeof(unsigned)), "reset flow epochs");
  cuda_check(cudaMemset(D.d_stagebuf, 0xff, 2 * D.stagebuf_elems * sizeof(double2)), "arm stage buffers");
  last_grid[d] = grid;
}

// Process-wide order of chained (non-cooperative, persistent) k1_flow grids,
// per device: the event of the last one and the stream it ran on (compared
// only, never used for API calls).
struct ChainOrder {
  std::mutex mu;
  cudaEvent_t ev = nullptr;
  cudaStream_t last = nullptr;
  bool used = false;
};
static ChainOrder& chain_order(int device) {
  static ChainOrder orders[64];
  static std::once_flag once[64];
  ChainOrder& co = orders[device & 63];
  std::call_once(once[device & 63], [&co] {
    cuda_check(cudaEventCreateWithFlags(&co.ev, cudaEventDisableTiming), "chain event");
  });
  return co;
}

void Plan::apply_device(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream) {
  std::lock_guard<std::recursive_mutex> lock(mu);
  if (!dir[d].built) throw std::logic_error("plan was built without this apply direction");
  if (dir[d].stages.empty()) {  // no factors (square, check_tables): the permutations alone
    const int64_t n = nrows, total = n * nrhs;
    if (total == 0) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(stream, &cs), "capture status");
    if (cs == cudaStreamCaptureStatusNone) cuda_check(cudaStreamWaitEvent(stream, ev_last, 0), "order applies");
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, int64_t(num_sms) * 8));
    k0_permute<<<blocks, 256, 0, stream>>>(in, out, d == 0 ? d_col_perm : d_row_perm, d == 0 ? d_row_perm : d_col_perm,
                                           n, nrhs);
    cuda_check(cudaGetLastError(), "k0_permute");
    if (cs == cudaStreamCaptureStatusNone) cuda_check(cudaEventRecord(ev_last, stream), "event");
    return;
  }
  ensure_buffers(nrhs);
  if (flow_ok(d, nrhs)) {
    prepare_flow(d);
    ensure_stageio(d);
  }
  if (k2flow_ok(d, nrhs)) ensure_k2flow(d);
  // after the previous apply on this plan, whichever stream it ran on
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(stream, &cs), "capture status");
  const bool ordered = cs == cudaStreamCaptureStatusNone;
  // chained single-RHS applies (bit 17): plain launches with programmatic
  // dependent launch, so consecutive applies on one stream overlap launch and
  // panel prefetch; stream order already orders them, the event wait (which
  // would serialise the two grids) is only needed across streams
  const bool chain = ordered && (flags & kFlagChain) && flow_ok(d, nrhs) && nrhs == 1;
  if (ordered && !(chain && stream == last_stream)) cuda_check(cudaStreamWaitEvent(stream, ev_last, 0), "order applies");
  if (ordered) last_stream = stream;
  // Chained grids launch without the cooperative guarantee (it would wait for
  // the whole GPU and forbid the overlap), so two of them must never share
  // the SMs: process-wide, a chained k1_flow on another stream than the
  // previous one waits for it.  On one stream they follow each other.
  std::unique_lock<std::mutex> chain_lock;
  ChainOrder* co = nullptr;
  if (chain) {
    co = &chain_order(device);
    chain_lock = std::unique_lock<std::mutex>(co->mu);
    if (co->last != stream && co->used) cuda_check(cudaStreamWaitEvent(stream, co->ev, 0), "order chained grids");
  }
  struct ChainDone {
    ChainOrder* co;
    cudaStream_t s;
    ~ChainDone() {
      if (co) {
        cudaEventRecord(co->ev, s);
        co->last = s;
        co->used = true;
      }
    }
  } chain_done{co, stream};
  struct Done {
    Plan* p;
    cudaStream_t s;
    bool on;
    ~Done() {
      if (on) cudaEventRecord(p->ev_last, s);
    }
  } done{this, stream, ordered};
  if (!(flags & 4u) || chain) {
    launch(d, in, out, nrhs, stream);
    cuda_check(cudaGetLastError(), "apply");
    return;
  }
  for (auto& g : graphs)
    if (g.d == d && g.in == in && g.out == out && g.nrhs == nrhs && g.flags == flags) {
      cuda_check(cudaGraphLaunch(g.exec, stream), "cudaGraphLaunch");
      return;
    }
  cudaStream_t cap;
  cuda_check(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "stream create");
  cudaGraph_t graph;
  cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
  launch(d, in, out, nrhs, cap);
  cuda_check(cudaStreamEndCapture(cap, &graph), "end capture");
  cudaGraphExec_t exec;
  cuda_check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cap);
  if (graphs.size() >= 8) {
    cudaGraphExecDestroy(graphs.front().exec);
    graphs.erase(graphs.begin());
  }
  graphs.push_back({d, in, out, nrhs, flags, exec});
  cuda_check(cudaGraphLaunch(exec, stream), "cudaGraphLaunch");
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

namespace {
// Makes the plan's device current for a call and restores the caller's.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
}  // namespace

void Plan::apply(const double* f, double* g, int64_t nrhs, bool transpose, cudaStream_t stream) {
  std::lock_guard<std::recursive_mutex> lock(mu);
  if (nrhs < 1) throw std::invalid_argument("nrhs must be >= 1");
  const DeviceScope on_device(device);
  const int d = transpose ? 1 : 0;
  const int64_t nin = transpose ? nrows : ncols, nout = transpose ? ncols : nrows;
  const bool din = is_device_ptr(f), dout = is_device_ptr(g);
  const double2* in = reinterpret_cast<const double2*>(f);
  double2* out = reinterpret_cast<double2*>(g);
  if (!din || !dout) {
    const int64_t need = std::max<int64_t>(1, std::max(nrows, ncols)) * nrhs;
    if (need > io_elems) {
      cudaFree(d_io[0]);
      cudaFree(d_io[1]);
      d_io[0] = d_io[1] = nullptr;
      cuda_check(cudaMalloc(&d_io[0], need * sizeof(double2)), "cudaMalloc staging");
      cuda_check(cudaMalloc(&d_io[1], need * sizeof(double2)), "cudaMalloc staging");
      io_elems = need;
      for (auto& gr : graphs) cudaGraphExecDestroy(gr.exec);
      graphs.clear();
    }
  }
  if (!din) {
    // d_io[0] is shared by every host-input apply of this plan: the previous
    // one (possibly host-in / device-out on another stream, which returns
    // without a sync) may still be reading it, so the copy waits for it.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(stream, &cs), "capture status");
    if (cs == cudaStreamCaptureStatusNone) cuda_check(cudaStreamWaitEvent(stream, ev_last, 0), "order staging");
    cuda_check(cudaMemcpyAsync(d_io[0], f, nin * nrhs * sizeof(double2), cudaMemcpyHostToDevice, stream), "H2D");
    in = d_io[0];
  }
  double2* dst = dout ? out : d_io[1];
  apply_device(d, in, dst, nrhs, stream);
  if (!dout) {
    cuda_check(cudaMemcpyAsync(g, dst, nout * nrhs * sizeof(double2), cudaMemcpyDeviceToHost, stream), "D2H");
    cuda_check(cudaStreamSynchronize(stream), "apply sync");
  }
}

// Pipelined apply on host operands: H2D on one stream, the apply on another,
// D2H on a third, rotating through kAsyncSlots device staging slots, so the
// copies of consecutive calls overlap the previous apply.  Returns after
// enqueueing; `user` waits for this call's D2H.  f is read asynchronously
// (host-written input: it is not ordered after work on `user`), so it must
// not change until `user` is synchronized.
void Plan::apply_async(const double* f, double* g, int64_t nrhs, bool transpose, cudaStream_t user) {
  std::lock_guard<std::recursive_mutex> lock(mu);
  if (nrhs < 1) throw std::invalid_argument("nrhs must be >= 1");
  const DeviceScope on_device(device);
  const int d = transpose ? 1 : 0;
  if (!dir[d].built) throw std::logic_error("plan was built without this apply direction");
  const int64_t nin = transpose ? nrows : ncols, nout = transpose ? ncols : nrows;
  const int64_t need = std::max<int64_t>(1, std::max(nrows, ncols)) * nrhs;
  if (!s_h2d) {
    cuda_check(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreateWithFlags(&ev_user, cudaEventDisableTiming), "event");
    for (auto& a : aslots) {
      cuda_check(cudaEventCreateWithFlags(&a.in_ready, cudaEventDisableTiming), "event");
      cuda_check(cudaEventCreateWithFlags(&a.applied, cudaEventDisableTiming), "event");
      cuda_check(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming), "event");
    }
  }
  AsyncSlot& S = aslots[acount++ % kAsyncSlots];
  if (S.used) cuda_check(cudaStreamWaitEvent(s_h2d, S.done, 0), "slot reuse");
  if (need > S.elems) {
    cuda_check(cudaStreamSynchronize(s_d2h), "slot resize");
    cudaFree(S.d_in);
    cudaFree(S.d_out);
    S.d_in = S.d_out = nullptr;
    cuda_check(cudaMalloc(&S.d_in, need * sizeof(double2)), "cudaMalloc async staging");
    cuda_check(cudaMalloc(&S.d_out, need * sizeof(double2)), "cudaMalloc async staging");
    S.elems = need;
  }
  cuda_check(cudaMemcpyAsync(S.d_in, f, nin * nrhs * sizeof(double2), cudaMemcpyHostToDevice, s_h2d), "H2D");
  // A chained single-RHS apply waits for its input inside the kernel (a flag
  // byte written after the copy on the copy stream) rather than through a
  // cross-stream event, which would break the programmatic chain on s_comp.
  const bool in_kernel_wait = (flags & kFlagChain) && flow_ok(d, nrhs) && nrhs == 1 && !dir[d].stages.empty();
  if (in_kernel_wait) {
    if (!d_inflag) {
      cuda_check(cudaMalloc(&d_inflag, 64), "cudaMalloc input flags");
      cuda_check(cudaMemset(d_inflag, 0, 64), "input flags");
    }
    const int si = static_cast<int>(&S - aslots);
    S.flag_seq = static_cast<unsigned char>(S.flag_seq + 1 == 0 ? 1 : S.flag_seq + 1);
    cuda_check(cudaMemsetAsync(d_inflag + si, S.flag_seq, 1, s_h2d), "input flag");
    next_in_flag = d_inflag + si;
    next_in_seq = S.flag_seq;
  } else {
    cuda_check(cudaEventRecord(S.in_ready, s_h2d), "event");
    cuda_check(cudaStreamWaitEvent(s_comp, S.in_ready, 0), "wait H2D");
  }
  struct ClearFlag {
    Plan* p;
    ~ClearFlag() { p->next_in_flag = nullptr; }
  } clear_flag{this};
  apply_device(d, S.d_in, S.d_out, nrhs, s_comp);
  cuda_check(cudaEventRecord(S.applied, s_comp), "event");
  cuda_check(cudaStreamWaitEvent(s_d2h, S.applied, 0), "wait apply");
  cuda_check(cudaMemcpyAsync(g, S.d_out, nout * nrhs * sizeof(double2), cudaMemcpyDeviceToHost, s_d2h), "D2H");
  cuda_check(cudaEventRecord(S.done, s_d2h), "event");
  cuda_check(cudaStreamWaitEvent(user, S.done, 0), "signal user");
  S.used = true;
}

}  // namespace midbf::dev
