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
// A complex MAC is four real
// DMMAs (re*re, -im*im, re*im, im*re) into separate re/im accumulators.
// Operands move global -> shared with cp.async (16 B per complex entry) in
// 32-column K chunks, double-buffered; the shared layouts are padded so
// every fragment load is bank-conflict free: panel column stride 34
// complex, X row stride 66 complex (stride/16B == 2 mod 8 puts the 8 lanes
// of a quarter-warp phase on distinct bank groups).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "plan.hpp"

namespace midbf::dev {

constexpr int kK2Rhs = 64;    // right-hand sides per CTA tile
constexpr int kK2Kc = 32;     // K (panel columns) per staged chunk
constexpr int kK2Ps = 34;     // padded panel column stride (complex)
constexpr int kK2Xs = 66;     // padded X row stride (complex)
constexpr int kK2PBuf = kK2Kc * kK2Ps;   // complex per panel buffer
constexpr int kK2XBuf = kK2Kc * kK2Xs;   // complex per X buffer
constexpr size_t kK2Smem = size_t(2) * (kK2PBuf + kK2XBuf) * 16;

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
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
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
  double2* const Pb = k2smem;                // 2 panel buffers
  double2* const Xb = k2smem + 2 * kK2PBuf;  // 2 X buffers
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int rb = w & 3, ch = w >> 2;  // row block, RHS half
  const Strip st = strips[blockIdx.x];
  const int h = st.h;
  const int c0 = blockIdx.y * kK2Rhs;      // first RHS of this tile
  const int ncv = min(kK2Rhs, nrhs - c0);  // valid RHS in the tile
  asm volatile("griddepcontrol.wait;" ::: "memory");  // previous stage's output
  asm volatile("griddepcontrol.launch_dependents;" :::);

  double acc[4][2][2];  // [col block][re, im][2 entries]
#pragma unroll
  for (int cb = 0; cb < 4; ++cb)
#pragma unroll
    for (int r = 0; r < 2; ++r) acc[cb][r][0] = acc[cb][r][1] = 0.0;

  // Zero both buffers once: rows >= h, RHS >= ncv and K tails of short
  // chunks stay zero (tails are re-zeroed per chunk below), so the inner
  // loop needs no masking.
  for (int i = tid; i < 2 * (kK2PBuf + kK2XBuf); i += kK2Threads) k2smem[i] = make_double2(0, 0);
  __syncthreads();

  // chunk enumeration over the strip's panels: (seg j, column c)
  int j = 0, c = 0;
  auto stage = [&](int jj, int cc, int buf) {
    const Seg s = segs[st.seg0 + jj];
    const int kc = min(kK2Kc, s.n - cc);
    const double2* P = arena + s.off + static_cast<int64_t>(cc) * h;
    double2* pd = Pb + buf * kK2PBuf;
    double2* xd = Xb + buf * kK2XBuf;
    for (int col = w; col < kK2Kc; col += kK2Threads / 32) {  // panel columns (lane = row)
      if (lane < h) {
        if (col < kc)
          cp_async16(pd + col * kK2Ps + lane, P + col * h + lane);
        else
          pd[col * kK2Ps + lane] = make_double2(0, 0);
      }
    }
    for (int rhs = w; rhs < ncv; rhs += kK2Threads / 32) {  // X rows x0+cc .. (lane = k)
      const double2* xc = x + static_cast<int64_t>(c0 + rhs) * xld;
      const int k = lane;
      if (k < kc) {
        int idx = s.x0 + cc + k;
        if (xperm) idx = __ldg(xperm + idx);
        cp_async16(xd + k * kK2Xs + rhs, xc + idx);
      } else {
        xd[k * kK2Xs + rhs] = make_double2(0, 0);
      }
    }
    cp_async_commit();
    return kc;
  };
  if (st.nseg > 0) {
    int kc_cur = stage(0, 0, 0);
    int buf = 0;
    while (true) {
      int jn = j, cn = c + kc_cur;
      if (cn >= segs[st.seg0 + jn].n) {
        ++jn;
        cn = 0;
      }
      const bool more = jn < st.nseg;
      int kc_next = 0;
      if (more) kc_next = stage(jn, cn, buf ^ 1);
      if (more)
        cp_async_wait<1>();
      else
        cp_async_wait<0>();
      __syncthreads();
      const double2* Ps = Pb + buf * kK2PBuf;
      const double2* Xs = Xb + buf * kK2XBuf + ch * 32;
      const int kend = (kc_cur + 3) & ~3;
      for (int kk = 0; kk < kend; kk += 4) {
        const double2 a = Ps[(kk + t) * kK2Ps + 8 * rb + g];
        const double naim = -a.y;
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
          const double2 b = Xs[(kk + t) * kK2Xs + cb * 8 + g];
          dmma(acc[cb][0][0], acc[cb][0][1], a.x, b.x);
          dmma(acc[cb][0][0], acc[cb][0][1], naim, b.y);
          dmma(acc[cb][1][0], acc[cb][1][1], a.x, b.y);
          dmma(acc[cb][1][0], acc[cb][1][1], a.y, b.x);
        }
      }
      __syncthreads();
      if (!more) break;
      j = jn;
      c = cn;
      kc_cur = kc_next;
      buf ^= 1;
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
