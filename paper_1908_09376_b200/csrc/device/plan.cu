// K1 — MIDBF apply on sm_100a: device plan (level-contiguous factor arena) and
// the per-stage streaming ZGEMV kernel.
//
// Replaces bf::apply_impl / apply_factor (reference src/butterfly.cpp:624-667):
//   v = f[col_perm];  for factor V^1 .. U^1: v = F_i v;  g[row_perm] = v.
// In the reference every block is a separately heap-allocated Eigen matrix and
// each group is an Eigen GEMV under OpenMP.  Here each applied factor (a
// "stage") becomes a list of row *strips* of <= 32 output rows.  A strip owns
// the ordered list of block panels that write those rows (the reference's
// fixed in-group order), so no two warps ever write the same output and no
// float atomics are used: results are run-to-run bitwise stable.
//
// Arena layout (the whole factorization is one device allocation):
//   strip panels in stage order, each panel = the strip's rows of one block,
//   stored as column PAIRS: pair p holds (M(i,2p), M(i,2p+1)) for i = 0..h-1,
//   so lane i of a warp fetches its row's two columns with one 256-bit
//   LDG (LDG.E.256, sm_100), and a warp streams h*32 contiguous bytes per
//   instruction.  An odd last column is stored as h plain complex values.
//   Panels are padded to 32-byte multiples (<= 16 B each).
// Perms are fused: stage 0 gathers f through col_perm while staging x into
// shared memory, the last stage scatters through row_perm.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "plan.hpp"

namespace midbf::dev {

namespace {

constexpr int kWarps = 4;    // warps per CTA (one strip per warp)
constexpr int kXChunk = 256; // x entries staged per warp per chunk (4 KB)
constexpr int kStripRows = 32;

__device__ __forceinline__ double4 ld_stream4(const double2* p) {
  double4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void cmac(double& ar, double& ai, double mr, double mi, double xr, double xi) {
  ar = fma(mr, xr, ar);
  ar = fma(-mi, xi, ar);
  ai = fma(mr, xi, ai);
  ai = fma(mi, xr, ai);
}

// One warp per strip.  blockIdx.y selects the right-hand side (v1 multi-RHS:
// the payload is re-streamed per column).
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
  Strip st = {0, 0, 0, 0};
  if (t < nstrips) st = strips[t];
  if (kPrefetch && t < nstrips && lane < st.nseg) {
    // Factor payload does not depend on the previous stage: pull this
    // strip's panels toward L2 before waiting on the dependency.
    const Seg s = segs[st.seg0 + lane];
    bulk_prefetch_l2(arena + s.off, static_cast<uint32_t>(s.elems) * 16u);
  }
  pdl_wait();
  pdl_launch_dependents();
  if (t >= nstrips) return;
  x += blockIdx.y * xld;
  y += blockIdx.y * yld;

  const int h = st.h;
  const bool row_live = lane < h;
  double ar0 = 0, ai0 = 0, ar1 = 0, ai1 = 0;
  double2* xw = xs[wid];
  for (int si = 0; si < st.nseg; ++si) {
    const Seg s = segs[st.seg0 + si];
    const double2* P = arena + s.off;
    const int n = s.n;
    const int npair = n >> 1;
    for (int cb = 0; cb < n; cb += kXChunk) {
      const int cn = min(kXChunk, n - cb);
      __syncwarp();
      for (int j = lane; j < cn; j += 32) {
        int idx = s.x0 + cb + j;
        if (xperm) idx = xperm[idx];
        xw[j] = x[idx];
      }
      __syncwarp();
      // column pairs fully inside this chunk (cb is even: kXChunk is even)
      const int p0 = cb >> 1;
      const int p1 = min(npair, (cb + cn) >> 1);
      int p = p0;
      constexpr int U = 4;  // 4 x 256-bit loads in flight per lane per batch
      for (; p + U <= p1; p += U) {
        double4 m[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          m[u] = row_live ? ld_stream4(P + 2 * ((int64_t)(p + u) * h + lane)) : make_double4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double2 xa = xw[2 * (p + u) - cb];
          const double2 xb = xw[2 * (p + u) + 1 - cb];
          cmac(ar0, ai0, m[u].x, m[u].y, xa.x, xa.y);
          cmac(ar1, ai1, m[u].z, m[u].w, xb.x, xb.y);
        }
      }
      for (; p < p1; ++p) {
        const double4 m = row_live ? ld_stream4(P + 2 * ((int64_t)p * h + lane)) : make_double4(0, 0, 0, 0);
        const double2 xa = xw[2 * p - cb];
        const double2 xb = xw[2 * p + 1 - cb];
        cmac(ar0, ai0, m.x, m.y, xa.x, xa.y);
        cmac(ar1, ai1, m.z, m.w, xb.x, xb.y);
      }
      if ((n & 1) && cb + cn == n) {  // odd tail column, stored as h complex
        const double2 m = row_live ? ld_stream2(P + 2 * (int64_t)npair * h + lane) : make_double2(0, 0);
        const double2 xa = xw[n - 1 - cb];
        cmac(ar0, ai0, m.x, m.y, xa.x, xa.y);
      }
    }
  }
  if (row_live) {
    int idx = st.y0 + lane;
    if (yperm) idx = yperm[idx];
    y[idx] = make_double2(ar0 + ar1, ai0 + ai1);
  }
}

struct EffBlock {
  int64_t yoff, xoff, m, n;  // as applied in this direction
  const double* data;        // original column-major block payload (complex)
  int64_t ld;                // original row count
  bool tr;                   // panel(i,c) = data[c + i*ld] when transposed
  int64_t order;
};

inline void get_entry(const EffBlock& b, int64_t i, int64_t c, double* dst) {
  const double* src = b.tr ? b.data + 2 * (c + i * b.ld) : b.data + 2 * (i + c * b.ld);
  dst[0] = src[0];
  dst[1] = src[1];
}

}  // namespace

// Build one direction (forward or transpose) of the plan on the host and
// upload it.  Task construction is general (ragged, overlapping, uncovered
// rows): breakpoints at every block edge, active blocks in reference order.
void Plan::build_direction(int d, const PlanTables& T) {
  Direction& D = dir[d];
  const int64_t nf = T.nfactors;
  D.stages.clear();
  std::vector<Strip> strips;
  std::vector<Seg> segs;
  std::vector<double> arena;  // interleaved complex, grown per panel
  arena.reserve(static_cast<size_t>(2 * T.total_nnz + 64 * T.total_blocks));

  for (int64_t s = 0; s < nf; ++s) {
    const int64_t fi = d == 0 ? nf - 1 - s : s;
    const FactorView& F = T.factors[static_cast<size_t>(fi)];
    Stage stg;
    stg.out_len = d == 0 ? F.rows : F.cols;
    stg.in_len = d == 0 ? F.cols : F.rows;
    stg.strip0 = static_cast<int32_t>(strips.size());
    stg.arena0 = static_cast<int64_t>(arena.size() / 2);
    // effective blocks in the reference's serial order: groups, then blocks
    std::vector<EffBlock> eb;
    int64_t ord = 0;
    for (int64_t g = 0; g < F.ngroups; ++g) {
      for (int64_t b = F.groups[2 * g]; b < F.groups[2 * g + 1]; ++b) {
        const int64_t* bd = F.blocks + 4 * b;
        EffBlock e;
        e.ld = bd[2];
        e.data = F.payload[static_cast<size_t>(b)];
        e.order = ord++;
        if (bd[2] == 0 || bd[3] == 0) continue;
        if (d == 0) {
          e.yoff = bd[0];
          e.xoff = bd[1];
          e.m = bd[2];
          e.n = bd[3];
          e.tr = false;
        } else {
          e.yoff = bd[1];
          e.xoff = bd[0];
          e.m = bd[3];
          e.n = bd[2];
          e.tr = true;
        }
        eb.push_back(e);
      }
    }
    // breakpoints
    std::vector<int64_t> bp{0, stg.out_len};
    for (const auto& e : eb) {
      bp.push_back(e.yoff);
      bp.push_back(e.yoff + e.m);
    }
    std::sort(bp.begin(), bp.end());
    bp.erase(std::unique(bp.begin(), bp.end()), bp.end());
    // blocks sorted by start for the active-set sweep
    std::vector<int64_t> by_start(eb.size());
    for (size_t i = 0; i < eb.size(); ++i) by_start[i] = static_cast<int64_t>(i);
    std::sort(by_start.begin(), by_start.end(), [&](int64_t a, int64_t b) { return eb[a].yoff < eb[b].yoff; });
    std::set<std::pair<int64_t, int64_t>> active;  // (order, index)
    size_t next = 0;
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
      for (int64_t y = a; y < b; y += kStripRows) {
        const int h = static_cast<int>(std::min<int64_t>(kStripRows, b - y));
        Strip st;
        st.y0 = static_cast<int32_t>(y);
        st.h = h;
        st.seg0 = static_cast<int32_t>(segs.size());
        st.nseg = 0;
        for (const auto& pr : active) {
          const EffBlock& e = eb[pr.second];
          Seg sg;
          sg.off = static_cast<int64_t>(arena.size() / 2);
          sg.x0 = static_cast<int32_t>(e.xoff);
          sg.n = static_cast<int32_t>(e.n);
          const int64_t r0 = y - e.yoff;
          const int64_t npair = e.n / 2;
          size_t base = arena.size();
          int64_t elems = h * e.n;
          if (elems & 1) ++elems;  // pad to 32 bytes
          arena.resize(base + static_cast<size_t>(2 * elems), 0.0);
          double* dst = arena.data() + base;
          for (int64_t p = 0; p < npair; ++p)
            for (int i = 0; i < h; ++i) {
              get_entry(e, r0 + i, 2 * p, dst + 4 * (p * h + i));
              get_entry(e, r0 + i, 2 * p + 1, dst + 4 * (p * h + i) + 2);
            }
          if (e.n & 1)
            for (int i = 0; i < h; ++i) get_entry(e, r0 + i, e.n - 1, dst + 2 * (2 * npair * h + i));
          sg.elems = static_cast<int32_t>(elems);
          segs.push_back(sg);
          ++st.nseg;
        }
        strips.push_back(st);
      }
    }
    stg.nstrips = static_cast<int32_t>(strips.size()) - stg.strip0;
    stg.payload_bytes = 16 * (static_cast<int64_t>(arena.size() / 2) - stg.arena0);
    D.stages.push_back(stg);
  }
  if (strips.size() > 0x7fffffff || segs.size() > 0x7fffffff)
    throw std::invalid_argument("factorization too large for one device plan");
  D.nstrips = static_cast<int64_t>(strips.size());
  D.nsegs = static_cast<int64_t>(segs.size());
  D.arena_elems = static_cast<int64_t>(arena.size() / 2);
  cuda_check(cudaMalloc(&D.d_strips, std::max<size_t>(1, strips.size()) * sizeof(Strip)), "cudaMalloc strips");
  cuda_check(cudaMalloc(&D.d_segs, std::max<size_t>(1, segs.size()) * sizeof(Seg)), "cudaMalloc segs");
  cuda_check(cudaMalloc(&D.d_arena, std::max<size_t>(1, arena.size() / 2) * sizeof(double2)), "cudaMalloc arena");
  cuda_check(cudaMemcpy(D.d_strips, strips.data(), strips.size() * sizeof(Strip), cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(D.d_segs, segs.data(), segs.size() * sizeof(Seg), cudaMemcpyHostToDevice), "upload");
  cuda_check(cudaMemcpy(D.d_arena, arena.data(), arena.size() * sizeof(double), cudaMemcpyHostToDevice), "upload");
  D.built = true;
}

Plan::Plan(const PlanTables& T, unsigned directions) {
  device = require_device();
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
  for (int d = 0; d < 2; ++d)
    if (directions & (1u << d)) build_direction(d, T);
}

Plan::~Plan() {
  for (auto& D : dir) {
    cudaFree(D.d_strips);
    cudaFree(D.d_segs);
    cudaFree(D.d_arena);
  }
  for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
  cudaFree(d_row_perm);
  cudaFree(d_col_perm);
  cudaFree(d_buf[0]);
  cudaFree(d_buf[1]);
  cudaFree(d_io[0]);
  cudaFree(d_io[1]);
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
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = use_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const Strip* sp = D.d_strips + st.strip0;
    if (use_prefetch)
      cuda_check(cudaLaunchKernelEx(&cfg, k1_stage<true>, sp, st.nstrips, (const Seg*)D.d_segs,
                                    (const double2*)D.d_arena, x, xld, xp, y, yld, yp),
                 "k1_stage launch");
    else
      cuda_check(cudaLaunchKernelEx(&cfg, k1_stage<false>, sp, st.nstrips, (const Seg*)D.d_segs,
                                    (const double2*)D.d_arena, x, xld, xp, y, yld, yp),
                 "k1_stage launch");
  }
}

// Device-operand apply; the stage chain is captured once per operand set into
// a CUDA graph (7 launches at cfg1 become one graph launch).
void Plan::apply_device(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream) {
  if (!dir[d].built) throw std::logic_error("plan was built without this apply direction");
  ensure_buffers(nrhs);
  if (dir[d].stages.empty()) return;
  if (!use_graph) {
    launch_stages(d, in, out, nrhs, stream);
    cuda_check(cudaGetLastError(), "apply");
    return;
  }
  for (auto& g : graphs)
    if (g.d == d && g.in == in && g.out == out && g.nrhs == nrhs) {
      cuda_check(cudaGraphLaunch(g.exec, stream), "cudaGraphLaunch");
      return;
    }
  cudaStream_t cap;
  cuda_check(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "stream create");
  cudaGraph_t graph;
  cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
  launch_stages(d, in, out, nrhs, cap);
  cuda_check(cudaStreamEndCapture(cap, &graph), "end capture");
  cudaGraphExec_t exec;
  cuda_check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cap);
  if (graphs.size() >= 8) {
    cudaGraphExecDestroy(graphs.front().exec);
    graphs.erase(graphs.begin());
  }
  graphs.push_back({d, in, out, nrhs, exec});
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

void Plan::apply(const double* f, double* g, int64_t nrhs, bool transpose, cudaStream_t stream) {
  if (nrhs < 1) throw std::invalid_argument("nrhs must be >= 1");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
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
  std::vector<double> payload(static_cast<size_t>(2 * total));
  f.read(reinterpret_cast<char*>(payload.data()), static_cast<std::streamsize>(16 * total));
  need(bool(f), "truncated payload");
  f.peek();
  need(f.eof(), "trailing bytes after payload");
  const double* p = payload.data();
  std::vector<std::vector<const double*>> ptrs(static_cast<size_t>(T.nfactors));
  for (int64_t i = 0; i < T.nfactors; ++i) {
    FactorView& F = T.factors[static_cast<size_t>(i)];
    F.blocks = blocks[i].data();
    F.groups = groups[i].data();
    for (int64_t b = 0; b < F.nblocks; ++b) {
      ptrs[i].push_back(p);
      p += 2 * blocks[i][4 * b + 2] * blocks[i][4 * b + 3];
    }
    F.payload = ptrs[i].data();
  }
  T.row_perm = rp.data();
  T.col_perm = cp.data();
  T.total_nnz = total;
  T.total_blocks = nblocks_all;
  return std::make_unique<Plan>(T, directions);
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

extern "C" int midbf_plan_create(midbf_plan_t* out, int64_t nrows, int64_t ncols, const int64_t* row_perm,
                                 const int64_t* col_perm, int64_t nfactors, const int64_t* factor_shape,
                                 const int64_t* blocks, const int64_t* groups, const double* payload,
                                 unsigned directions) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output handle");
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
    const double* pp = payload;
    for (int64_t i = 0; i < nfactors; ++i) {
      auto& F = T.factors[static_cast<size_t>(i)];
      F.rows = factor_shape[4 * i];
      F.cols = factor_shape[4 * i + 1];
      F.nblocks = factor_shape[4 * i + 2];
      F.ngroups = factor_shape[4 * i + 3];
      F.blocks = bp;
      F.groups = gp;
      for (int64_t b = 0; b < F.nblocks; ++b) {
        const int64_t m = bp[4 * b + 2], n = bp[4 * b + 3];
        if (m < 0 || n < 0 || bp[4 * b] < 0 || bp[4 * b + 1] < 0 || bp[4 * b] + m > F.rows ||
            bp[4 * b + 1] + n > F.cols)
          throw std::invalid_argument("block outside its factor");
        ptrs[i].push_back(pp);
        pp += 2 * m * n;
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
    *out = new midbf_plan_s{std::make_unique<Plan>(T, directions)};
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

// Tuning switches (bench / profiling): bit0 PDL, bit1 L2 bulk prefetch, bit2 graphs.
extern "C" int midbf_plan_set_flags(midbf_plan_t plan, unsigned flags) {
  return guard([&] {
    Plan& p = *plan->p;
    p.use_pdl = flags & 1u;
    p.use_prefetch = flags & 2u;
    p.use_graph = flags & 4u;
    for (auto& g : p.graphs) cudaGraphExecDestroy(g.exec);
    p.graphs.clear();
  });
}
