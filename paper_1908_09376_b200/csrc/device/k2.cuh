// K2 — multi-RHS MIDBF apply on the FP64 tensor cores (DMMA), sm_100a.
//
// Replaces apply_factor's Eigen GEMM path for x.cols() > 1
// (reference src/butterfly.cpp:633-637 with bf::apply(F, MatXc),
// :779): per stage, Y(strip rows, :) = sum over the strip's panels
// P (h x n) * X(x0 .. x0+n, :), complex, fixed panel order.
//
// tcgen05 has no f64 kind (CUDA 12.9 tcgen05.mma: f16/tf32/f8f6f4/i8/mx*),
// so the FP64 tensor path is the warp-level mma.sync.m8n8k4.f64 (DMMA),
// measured at 36.8 TFLOP/s on this B200 (tools/fp64_probe.cu).
//
// CTA = one strip x 64 right-hand sides, 8 warps (8 rows x 32 RHS each).
// A complex MAC is four real DMMAs (re*re, -im*im, re*im, im*re) into
// separate re/im accumulators.  The strip's panels are walked as ONE
// concatenated K dimension (sum of panel widths, panel order kept) in
// 16-column chunks through a 4-deep cp.async ring with one barrier per
// chunk; panel chunks (plan constants) are prefetched before the PDL wait
// on the previous stage.  Shared layouts are padded so every fragment load
// is bank-conflict free: panel column stride 34 complex, X row stride 66
// complex (stride/16B == 2 mod 8 puts the 8 lanes of a quarter-warp phase
// on distinct bank groups).  Up to kK2MaxSeg panel records per strip are
// held one per lane.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "plan.hpp"

namespace midbf::dev {

constexpr int kK2Rhs = 64;    // right-hand sides per CTA tile
constexpr int kK2Kc = 16;     // K (panel columns) per staged chunk
constexpr int kK2Stages = 4;  // cp.async ring depth
constexpr int kK2MaxSeg = 32; // panel records per strip (one per lane)
constexpr int kK2Ps = 34;     // padded panel column stride (complex)
constexpr int kK2Xs = 66;     // padded X row stride (complex)
constexpr int kK2PBuf = kK2Kc * kK2Ps;   // complex per panel buffer
constexpr int kK2XBuf = kK2Kc * kK2Xs;   // complex per X buffer
constexpr size_t kK2Smem = size_t(kK2Stages) * (kK2PBuf + kK2XBuf) * 16;

namespace k2dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// pure register op: not volatile, so ptxas schedules it freely
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

}  // namespace k2dev

// One stage.  x/y: column-major (len x nrhs, leading dims xld/yld); stage 0
// gathers rows through xperm, the last stage scatters through yperm.
// 8 warps: warp w owns rows 8*(w&3) .. +8 and RHS 32*(w>>2) .. +32 (4 column
// blocks of 8) of the CTA's 32 x 64 output tile.
constexpr int kK2Threads = 256;
__global__ void __launch_bounds__(kK2Threads, 2) k2_stage(const Strip* __restrict__ strips, const Seg* __restrict__ segs,
                                                       const double2* __restrict__ arena,
                                                       const double2* __restrict__ x, int64_t xld,
                                                       const int* __restrict__ xperm, double2* __restrict__ y,
                                                       int64_t yld, const int* __restrict__ yperm, int nrhs) {
  using namespace k2dev;
  extern __shared__ __align__(16) double2 k2smem[];
  double2* const Pb = k2smem;                        // kK2Stages panel buffers
  double2* const Xb = k2smem + kK2Stages * kK2PBuf;  // kK2Stages X buffers
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int rb = w & 3, ch = w >> 2;  // row block, RHS half
  const Strip st = strips[blockIdx.x];
  const int h = st.h;
  const int c0 = blockIdx.y * kK2Rhs;      // first RHS of this tile
  const int ncv = min(kK2Rhs, nrhs - c0);  // valid RHS in the tile
  const int K = st.xcols;
  const int nq = (K + kK2Kc - 1) / kK2Kc;  // chunks

  // lane l holds panel l: arena offset, first input entry, start in K
  int64_t s_off = 0;
  int s_x0 = 0, s_n = 0;
  if (lane < st.nseg) {
    const Seg sg = segs[st.seg0 + lane];
    s_off = sg.off;
    s_x0 = sg.x0;
    s_n = sg.n;
  }
  int s_k0 = s_n;  // inclusive -> exclusive prefix of the panel widths
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, s_k0, o);
    if (lane >= o) s_k0 += v;
  }
  s_k0 -= s_n;

  // K column kg -> (panel, column within it); every lane resolves column
  // q*16 + (lane & 15).
  auto locate = [&](int q, int& seg, int& cc) {
    const int kg = q * kK2Kc + (lane & (kK2Kc - 1));
    int sidx = 0;
    for (int l = 1; l < st.nseg; ++l) sidx += __shfl_sync(0xffffffffu, s_k0, l) <= kg;
    seg = sidx;
    cc = kg - __shfl_sync(0xffffffffu, s_k0, sidx);
    return kg < K;
  };
  // panel chunk q -> buffer b: warp w copies columns 2w, 2w+1 (lane = row)
  auto issue_p = [&](int q, int b) {
    int seg, cc;
    const bool ok = locate(q, seg, cc);
    const int64_t src = __shfl_sync(0xffffffffu, s_off, seg) + static_cast<int64_t>(cc) * h;
    double2* pd = Pb + b * kK2PBuf;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int col = 2 * w + i;
      const int64_t cs = __shfl_sync(0xffffffffu, src, col);
      const bool cok = __shfl_sync(0xffffffffu, ok, col);
      if (cok) {
        if (lane < h) cp_async16(pd + col * kK2Ps + lane, arena + cs + lane);
      } else {
        pd[col * kK2Ps + lane] = make_double2(0, 0);  // K tail
      }
    }
  };
  // X chunk q -> buffer b: lane&15 = k, RHS = 16*it + 2w + (lane >> 4)
  auto issue_x = [&](int q, int b) {
    int seg, cc;
    const bool ok = locate(q, seg, cc);
    int xi = __shfl_sync(0xffffffffu, s_x0, seg) + cc;
    if (ok && xperm) xi = __ldg(xperm + xi);
    double2* xd = Xb + b * kK2XBuf + (lane & (kK2Kc - 1)) * kK2Xs;
#pragma unroll
    for (int it = 0; it < kK2Rhs / 16; ++it) {
      const int rhs = 16 * it + 2 * w + (lane >> 4);
      if (ok) {
        if (rhs < ncv) cp_async16(xd + rhs, x + static_cast<int64_t>(c0 + rhs) * xld + xi);
      } else {
        xd[rhs] = make_double2(0, 0);  // K tail
      }
    }
  };

  // prologue: panel chunks need no predecessor; X chunks wait for it.
  // Rows >= h and RHS >= ncv of the buffers are never written: they only
  // feed output rows / RHS that are not stored.
  for (int q = 0; q < kK2Stages - 1; ++q)
    if (q < nq) issue_p(q, q);
  cp_async_commit();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // previous stage's output
  asm volatile("griddepcontrol.launch_dependents;" :::);
  for (int q = 0; q < kK2Stages - 1; ++q) {
    if (q < nq) issue_x(q, q);
    cp_async_commit();
  }

  double acc[4][2][2];  // [col block][re, im][2 entries]
#pragma unroll
  for (int cb = 0; cb < 4; ++cb)
#pragma unroll
    for (int r = 0; r < 2; ++r) acc[cb][r][0] = acc[cb][r][1] = 0.0;

  for (int q = 0; q < nq; ++q) {
    cp_async_wait<kK2Stages - 2>();  // chunk q landed (this thread's copies)
    __syncthreads();                 // ... everyone's; buffer (q-1) is free
    const int qn = q + kK2Stages - 1;
    if (qn < nq) {
      issue_p(qn, qn % kK2Stages);
      issue_x(qn, qn % kK2Stages);
    }
    cp_async_commit();
    const int b = q % kK2Stages;
    const double2* Ps = Pb + b * kK2PBuf;
    const double2* Xs = Xb + b * kK2XBuf + ch * 32;
    const int kend = q + 1 < nq ? kK2Kc : ((K - q * kK2Kc + 3) & ~3);
#pragma unroll 4
    for (int kk = 0; kk < kend; kk += 4) {
      const double2 a = Ps[(kk + t) * kK2Ps + 8 * rb + g];
      const double naim = -a.y;
      double2 bv[4];
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) bv[cb] = Xs[(kk + t) * kK2Xs + cb * 8 + g];
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        dmma(acc[cb][0][0], acc[cb][0][1], a.x, bv[cb].x);
        dmma(acc[cb][1][0], acc[cb][1][1], a.x, bv[cb].y);
      }
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        dmma(acc[cb][0][0], acc[cb][0][1], naim, bv[cb].y);
        dmma(acc[cb][1][0], acc[cb][1][1], a.y, bv[cb].x);
      }
    }
  }
  // D fragment: row 8*rb + g, RHS 32*ch + cb*8 + 2t + {0,1}
  const int row = 8 * rb + g;
  if (row < h) {
    int idx = st.y0 + row;
    if (yperm) idx = yperm[idx];
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int rhs = 32 * ch + cb * 8 + 2 * t + i;
        if (rhs < ncv) y[static_cast<int64_t>(c0 + rhs) * yld + idx] = make_double2(acc[cb][0][i], acc[cb][1][i]);
      }
  }
}

}  // namespace midbf::dev
