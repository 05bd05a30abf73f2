// K3 — fused batched kernel-entry sampler and K4 — direct O(N^2) sum, sm_100a.
//
// K3 replaces the EntryFn fills of shared_sweep (reference
// src/butterfly.cpp:462-464, 512-514, 598-600) that call
// polar(1, 2*pi*Phi(x_i, xi_j)) per entry (src/kernels.cpp:18-24, 242-245;
// low-rank form src/metrics.cpp:18-24).  One launch fills every block of a
// sweep pass: task t writes the nr x nc column-major block K(rows_t, cols_t).
// Nothing N x N is materialised; entries are formed from the point sets (or
// the low-rank factors A, B) on the fly.
//
// K4 replaces the direct summation of metrics::eps_b_of (src/metrics.cpp:40-45)
// and tests/test_butterfly.cpp:29-37: g(i) = sum_j K(i,j) f(j) for selected
// rows, column range split across CTAs, partial sums reduced in a fixed order.
//
// Arithmetic follows the reference expression by expression with
// non-contracted multiplies/adds (__dmul_rn/__dadd_rn), so the phase Phi is
// bitwise the x86 value; only the final sincos (CUDA libdevice vs glibc) may
// differ in the last ulp.  The per-point coefficients c_k(x) are evaluated on
// the host with glibc exactly as the reference does.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "common.cuh"
#include "k5_id.cuh"
#include "pool.hpp"
#include "sample.hpp"

namespace midbf::dev {

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

struct DevK {
  int kind, dim, rank;
  const double* X;     // nrows x dim
  const double* Om;    // ncols x dim
  const double* coef;  // nrows x 3, c_k(x) of the FIO phases
  const double* A;     // nrows x rank
  const double* B;     // ncols x rank
  const double2* u;
  const double2* v;
  double cre, cim;
};

// sin and cos of one argument, FP64-pipe lean: Cody-Waite reduction by
// pi/2 in three FMA steps (pi/2 split as fdlibm's pio2_1/2/3; the first part
// has 33 bits, so q * P1 is exact for |q| < 2^20) and fdlibm's
// __kernel_sin / __kernel_cos minimax polynomials on [-pi/4, pi/4].  Max
// abs error 1.2e-16 against long-double sin/cos and 1.1e-16 against glibc
// over 2e7 arguments of the BASELINE phase range (|x| < 2200).  About 22 FP64
// operations and no table or local-memory path; |x| >= 1e6, inf and NaN take
// CUDA's sincos.  CUDA's own sincos spends ~90 further integer / uniform-move
// instructions per call on its general reduction (ncu, r1_k3 source page).
// Coefficients live in the constant bank: DFMA takes them as c[][] operands
// directly, where literal double constants cost two uniform moves each per
// use (28 UMOV per entry in the r1_k3 SASS with literals).
__constant__ double kSC[18] = {
    6.36619772367581382433e-01,  6755399441055744.0,          // 2/pi, 1.5 * 2^52
    1.57079632673412561417e+00,  6.07710050630396597660e-11,  2.02226624871116645580e-21,  // pi/2 = P1+P2+P3
    -1.66666666666666324348e-01, 8.33333333332248946124e-03,  -1.98412698298579493134e-04,  // S1..S6
    2.75573137070700676789e-06,  -2.50507602534068634195e-08, 1.58969099521155010221e-10,
    4.16666666666666019037e-02,  -1.38888888888741095749e-03, 2.48015872894767294178e-05,  // C1..C6
    -2.75573143513906633035e-07, 2.08757232129817482790e-09,  -1.13596475577881948265e-11,
    6.283185307179586476925286766559};  // 2 pi (the reference's product 2*pi*Phi)

__device__ __forceinline__ void sincos_fast(double x, double* sn, double* cs) {  // |x| < 1e6
  const double kInvPio2 = kSC[0], kMagic = kSC[1], P1 = kSC[2], P2 = kSC[3], P3 = kSC[4];
  const double S1 = kSC[5], S2 = kSC[6], S3 = kSC[7], S4 = kSC[8], S5 = kSC[9], S6 = kSC[10];
  const double C1 = kSC[11], C2 = kSC[12], C3 = kSC[13], C4 = kSC[14], C5 = kSC[15], C6 = kSC[16];
  const double t = __fma_rn(x, kInvPio2, kMagic);
  const double q = __dsub_rn(t, kMagic);  // nearest integer to x * 2/pi
  const int n = __double2loint(t) & 3;    // quadrant
  double r = __fma_rn(-q, P1, x);
  r = __fma_rn(-q, P2, r);
  r = __fma_rn(-q, P3, r);
  const double z = __dmul_rn(r, r), v = __dmul_rn(z, r);
  const double ps = __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, S6, S5), S4), S3), S2);
  const double s = __fma_rn(v, __fma_rn(z, ps, S1), r);
  const double pc =
      __dmul_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, __fma_rn(z, C6, C5), C4), C3), C2), C1));
  const double hz = __dmul_rn(0.5, z), w = __dsub_rn(1.0, hz);
  const double c = __dadd_rn(w, __dadd_rn(__dsub_rn(__dsub_rn(1.0, w), hz), __dmul_rn(z, pc)));
  const double so = (n & 1) ? c : s, co = (n & 1) ? s : c;
  *sn = (n & 2) ? -so : so;
  *cs = ((n + 1) & 2) ? -co : co;
}

__device__ __forceinline__ void sincos_lean(double x, double* sn, double* cs) {
  if (fabs(x) < 1.0e6)
    sincos_fast(x, sn, cs);
  else
    sincos(x, sn, cs);
}

// Two independent arguments in one straight-line block, so that the two
// Horner chains interleave (the single-entry loop stalled on DFMA latency:
// "wait" 49% of the warp samples in r1_k3).
__device__ __forceinline__ void polar1x2(double phi0, double phi1, double2* e0, double2* e1) {
  const double x0 = __dmul_rn(kSC[17], phi0), x1 = __dmul_rn(kSC[17], phi1);
  double s0, c0, s1, c1;
  if (fabs(x0) < 1.0e6 && fabs(x1) < 1.0e6) {
    sincos_fast(x0, &s0, &c0);
    sincos_fast(x1, &s1, &c1);
  } else {
    sincos_lean(x0, &s0, &c0);
    sincos_lean(x1, &s1, &c1);
  }
  *e0 = make_double2(c0, s0);
  *e1 = make_double2(c1, s1);
}

// Four independent arguments (K4: more Horner chains in flight per warp,
// dependent DFMA latency 17 cycles measured, tools/lat_probe.cu).
__device__ __forceinline__ void polar1x4(const double (&phi)[4], double2 (&e)[4]) {
  double x[4], s[4], c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = __dmul_rn(kSC[17], phi[i]);
  if (fabs(x[0]) < 1.0e6 && fabs(x[1]) < 1.0e6 && fabs(x[2]) < 1.0e6 && fabs(x[3]) < 1.0e6) {
#pragma unroll
    for (int i = 0; i < 4; ++i) sincos_fast(x[i], &s[i], &c[i]);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) sincos_lean(x[i], &s[i], &c[i]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) e[i] = make_double2(c[i], s[i]);
}

__device__ __forceinline__ double2 polar1(double phi) {
  double s, c;
  sincos_lean(__dmul_rn(kSC[17], phi), &s, &c);
  return make_double2(c, s);
}

// Phi(x_i, xi_j) of the kernels that have one (FIO 2D/3D, low-rank A.B^T,
// x.xi), reference operation order, non-contracted.
__device__ __forceinline__ double phase_of(const DevK& k, int64_t i, int64_t j) {
  switch (k.kind) {
    case MIDBF_KERNEL_FIO2D: {
      const double x0 = k.X[2 * i], x1 = k.X[2 * i + 1];
      const double c1 = k.coef[3 * i], c2 = k.coef[3 * i + 1];
      const double w0 = k.Om[2 * j], w1 = k.Om[2 * j + 1];
      const double lin = __dadd_rn(__dmul_rn(x0, w0), __dmul_rn(x1, w1));
      const double q = __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(c1, c1), w0), w0),
                                 __dmul_rn(__dmul_rn(__dmul_rn(c2, c2), w1), w1));
      return __dadd_rn(lin, __dsqrt_rn(q));
    }
    case MIDBF_KERNEL_FIO3D: {
      const double* x = k.X + 3 * i;
      const double* w = k.Om + 3 * j;
      const double* a = k.coef + 3 * i;
      const double lin = __dadd_rn(__dadd_rn(__dmul_rn(x[0], w[0]), __dmul_rn(x[1], w[1])), __dmul_rn(x[2], w[2]));
      const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(a[0], a[0]), w[0]), w[0]),
                                           __dmul_rn(__dmul_rn(__dmul_rn(a[1], a[1]), w[1]), w[1])),
                                 __dmul_rn(__dmul_rn(__dmul_rn(a[2], a[2]), w[2]), w[2]));
      return __dadd_rn(lin, __dsqrt_rn(q));
    }
    case MIDBF_KERNEL_LOWRANK: {
      double s = 0.0;
      for (int q = 0; q < k.rank; ++q) s = __dadd_rn(s, __dmul_rn(k.A[i * k.rank + q], k.B[j * k.rank + q]));
      return s;
    }
    default: {  // NUFFT: x . xi
      double s = 0.0;
      for (int q = 0; q < k.dim; ++q) s = __dadd_rn(s, __dmul_rn(k.X[i * k.dim + q], k.Om[j * k.dim + q]));
      return s;
    }
  }
}

__device__ __forceinline__ double2 entry(const DevK& k, int64_t i, int64_t j) {
  switch (k.kind) {
    case MIDBF_KERNEL_CONST:
      return make_double2(k.cre, k.cim);
    case MIDBF_KERNEL_RANK1: {
      const double2 a = k.u[i], b = k.v[j];
      return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                          __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    }
    default:
      return polar1(phase_of(k, i, j));
  }
}

// Phi(rows, cols) block, column-major (rid / cid null: 0..n-1).
__global__ void __launch_bounds__(256) k3_phase(DevK k, const int* __restrict__ rid, int nr,
                                                const int* __restrict__ cid, int nc, double* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(nr) * nc;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e / nr), r = static_cast<int>(e - static_cast<int64_t>(c) * nr);
    out[e] = phase_of(k, rid ? rid[r] : r, cid ? cid[c] : c);
  }
}

// tasks: ntasks x 5 (row_off, nr, col_off, nc, out_off) as int32, out_off
// relative to this chunk's output base.  One CTA per task, threads stride
// the task's entries in output (column-major) order: coalesced stores.
__global__ void __launch_bounds__(256) k3_sample(DevK k, const int* __restrict__ tasks,
                                                 const int* __restrict__ rid, const int* __restrict__ cid,
                                                 double2* __restrict__ out) {
  const int* tk = tasks + 5 * blockIdx.x;
  const int ro = tk[0], nr = tk[1], co = tk[2], nc = tk[3], oo = tk[4];
  const int total = nr * nc;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int c = e / nr, r = e - c * nr;
    out[oo + e] = entry(k, rid[ro + r], cid[co + c]);
  }
}

// K3 into the K5 workspace: task t's block B (m x n column-major at
// ws + off): B = K(rows, cols) (m = nr, n = nc), or with TRANS its transpose
// (m = nc, n = nr) for a row ID.  rc = {row_off, nr, col_off, nc}.
template <bool TRANS>
__global__ void __launch_bounds__(256) k3_sample_ws(DevK k, const int4* __restrict__ rc,
                                                    const IdTask* __restrict__ tasks, const int* __restrict__ rid,
                                                    const int* __restrict__ cid, double2* __restrict__ ws) {
  const int4 q = rc[blockIdx.x];
  const IdTask tk = tasks[blockIdx.x];
  const int m = tk.m, total = tk.m * tk.n;
  double2* B = ws + tk.off;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int c = e / m, r = e - c * m;
    B[e] = TRANS ? entry(k, rid[q.x + c], cid[q.z + r]) : entry(k, rid[q.x + r], cid[q.z + c]);
  }
}

// ---- staged sampling (K3 / K4) ---------------------------------------------
// Every phase kernel is a function of per-row operands R (depending on x_i
// only) and per-column operands C (depending on xi_j only).  A block's
// operands are staged once in shared memory (structure of arrays, stride
// `rs` / `cs` between operand q and q+1), so the entry loop issues no
// dependent global loads: it is the FP64 arithmetic of Phi plus sincos.
// Staged values are the reference's own intermediate values (c_k*c_k is the
// first multiply of c_k*c_k*xi*xi, src/kernels.cpp:22), so results stay
// bitwise those of phase_of().
template <int KIND>
struct Ops;

template <>
struct Ops<MIDBF_KERNEL_FIO2D> {
  __device__ static int rw(const DevK&) { return 4; }
  __device__ static int cw(const DevK&) { return 2; }
  __device__ static void row(const DevK& k, int64_t i, double* o, int s) {
    const double c1 = k.coef[3 * i], c2 = k.coef[3 * i + 1];
    o[0] = k.X[2 * i];
    o[s] = k.X[2 * i + 1];
    o[2 * s] = __dmul_rn(c1, c1);
    o[3 * s] = __dmul_rn(c2, c2);
  }
  __device__ static void col(const DevK& k, int64_t j, double* o, int s) {
    o[0] = k.Om[2 * j];
    o[s] = k.Om[2 * j + 1];
  }
  __device__ static double phase(const DevK&, const double* R, int rs, const double* C, int cs) {
    const double w0 = C[0], w1 = C[cs];
    const double lin = __dadd_rn(__dmul_rn(R[0], w0), __dmul_rn(R[rs], w1));
    const double q = __dadd_rn(__dmul_rn(__dmul_rn(R[2 * rs], w0), w0), __dmul_rn(__dmul_rn(R[3 * rs], w1), w1));
    return __dadd_rn(lin, __dsqrt_rn(q));
  }
};

template <>
struct Ops<MIDBF_KERNEL_FIO3D> {
  __device__ static int rw(const DevK&) { return 6; }
  __device__ static int cw(const DevK&) { return 3; }
  __device__ static void row(const DevK& k, int64_t i, double* o, int s) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double a = k.coef[3 * i + q];
      o[q * s] = k.X[3 * i + q];
      o[(3 + q) * s] = __dmul_rn(a, a);
    }
  }
  __device__ static void col(const DevK& k, int64_t j, double* o, int s) {
#pragma unroll
    for (int q = 0; q < 3; ++q) o[q * s] = k.Om[3 * j + q];
  }
  __device__ static double phase(const DevK&, const double* R, int rs, const double* C, int cs) {
    const double w0 = C[0], w1 = C[cs], w2 = C[2 * cs];
    const double lin =
        __dadd_rn(__dadd_rn(__dmul_rn(R[0], w0), __dmul_rn(R[rs], w1)), __dmul_rn(R[2 * rs], w2));
    const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(R[3 * rs], w0), w0),
                                         __dmul_rn(__dmul_rn(R[4 * rs], w1), w1)),
                               __dmul_rn(__dmul_rn(R[5 * rs], w2), w2));
    return __dadd_rn(lin, __dsqrt_rn(q));
  }
};

template <>
struct Ops<MIDBF_KERNEL_LOWRANK> {
  __device__ static int rw(const DevK& k) { return k.rank; }
  __device__ static int cw(const DevK& k) { return k.rank; }
  __device__ static void row(const DevK& k, int64_t i, double* o, int s) {
    for (int q = 0; q < k.rank; ++q) o[q * s] = k.A[i * k.rank + q];
  }
  __device__ static void col(const DevK& k, int64_t j, double* o, int s) {
    for (int q = 0; q < k.rank; ++q) o[q * s] = k.B[j * k.rank + q];
  }
  __device__ static double phase(const DevK& k, const double* R, int rs, const double* C, int cs) {
    double s = 0.0;
    if (k.rank == 8) {  // BASELINE cfg2's rank, unrolled
#pragma unroll
      for (int q = 0; q < 8; ++q) s = __dadd_rn(s, __dmul_rn(R[q * rs], C[q * cs]));
    } else {
      for (int q = 0; q < k.rank; ++q) s = __dadd_rn(s, __dmul_rn(R[q * rs], C[q * cs]));
    }
    return s;
  }
};

template <>
struct Ops<MIDBF_KERNEL_NUFFT> {
  __device__ static int rw(const DevK& k) { return k.dim; }
  __device__ static int cw(const DevK& k) { return k.dim; }
  __device__ static void row(const DevK& k, int64_t i, double* o, int s) {
    for (int q = 0; q < k.dim; ++q) o[q * s] = k.X[i * k.dim + q];
  }
  __device__ static void col(const DevK& k, int64_t j, double* o, int s) {
    for (int q = 0; q < k.dim; ++q) o[q * s] = k.Om[j * k.dim + q];
  }
  __device__ static double phase(const DevK& k, const double* R, int rs, const double* C, int cs) {
    double s = 0.0;
    for (int q = 0; q < k.dim; ++q) s = __dadd_rn(s, __dmul_rn(R[q * rs], C[q * cs]));
    return s;
  }
};

// Staging capacities: m-side (fast, contiguous output index) operands for up
// to kMCap points, n-side operands in tiles of kNTile points.  Operand
// width <= kMaxW doubles per point (FIO 3D: 6; low-rank / x.xi: r, dim).
constexpr int kMCap = 512, kNTile = 128, kMaxW = 8;
constexpr int64_t kTaskEntries = 8192;  // entries per CTA of k3_sample (sample_blocks sub-tasks)
// Staging width per kind (max of row / column operands): shared memory per
// CTA 20 KB for FIO 2D, 30 KB for 3D, 40 KB otherwise -- small enough for 8
// CTAs (all 64 warps) per SM with the FIO kernels.
template <int KIND>
__host__ __device__ constexpr int stage_w() {
  return KIND == MIDBF_KERNEL_FIO2D ? 4 : KIND == MIDBF_KERNEL_FIO3D ? 6 : kMaxW;
}
template <int KIND>
constexpr size_t stage_smem() {
  return static_cast<size_t>(kMCap + kNTile) * stage_w<KIND>() * sizeof(double);
}

__host__ __device__ inline bool stageable(int kind, int rank, int dim) {
  switch (kind) {
    case MIDBF_KERNEL_FIO2D:
    case MIDBF_KERNEL_FIO3D:
      return true;
    case MIDBF_KERNEL_LOWRANK:
      return rank >= 1 && rank <= kMaxW;
    case MIDBF_KERNEL_NUFFT:
      return dim >= 1 && dim <= kMaxW;
    default:
      return false;
  }
}

// One block B (m x n, column-major, ld m) of K(rid[ro..ro+nr), cid[co..co+nc)),
// or with TRANS of its transpose (m = nc, n = nr).  Requires m <= kMCap.
template <int KIND, bool TRANS>
__device__ __forceinline__ void fill_staged(const DevK& k, const int* __restrict__ rid, const int* __restrict__ cid,
                                            int ro, int nr, int co, int nc, double2* __restrict__ B, double* sm) {
  using O = Ops<KIND>;
  const int m = TRANS ? nc : nr, n = TRANS ? nr : nc;
  double* sM = sm;                 // m-side operands, stride kMCap
  double* sN = sm + kMCap * stage_w<KIND>();  // n-side operands, stride kNTile
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    if (TRANS)
      O::col(k, cid[co + r], sM + r, kMCap);
    else
      O::row(k, rid[ro + r], sM + r, kMCap);
  }
  const int sr = static_cast<int>(blockDim.x) % m, sc = static_cast<int>(blockDim.x) / m;
  for (int c0 = 0; c0 < n; c0 += kNTile) {
    const int nt = min(kNTile, n - c0);
    __syncthreads();  // previous tile consumed (and, first time, m-side staged)
    for (int c = threadIdx.x; c < nt; c += blockDim.x) {
      if (TRANS)
        O::row(k, rid[ro + c0 + c], sN + c, kNTile);
      else
        O::col(k, cid[co + c0 + c], sN + c, kNTile);
    }
    __syncthreads();
    double2* out = B + static_cast<int64_t>(c0) * m;
    int r = threadIdx.x % m, c = threadIdx.x / m;
    auto step = [&]() {
      r += sr;
      c += sc;
      if (r >= m) {
        r -= m;
        ++c;
      }
    };
    int e = threadIdx.x;
    // four of this thread's entries per iteration: four independent sincos
    // Horner chains (dependent DFMA latency 17 cycles, tools/lat_probe.cu)
    for (;;) {
      int rr[4], cc[4];
      bool ok = true;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        rr[i] = r;
        cc[i] = c;
        ok = ok && c < nt;
        step();
      }
      if (!ok) {  // fewer than four left: back to the first of them, one at a time
        r = rr[0];
        c = cc[0];
        break;
      }
      double ph[4];
      double2 v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        ph[i] = TRANS ? O::phase(k, sN + cc[i], kNTile, sM + rr[i], kMCap)
                      : O::phase(k, sM + rr[i], kMCap, sN + cc[i], kNTile);
      polar1x4(ph, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) out[e + i * static_cast<int>(blockDim.x)] = v[i];
      e += 4 * static_cast<int>(blockDim.x);
    }
    for (; c < nt; e += blockDim.x) {
      const double phi = TRANS ? O::phase(k, sN + c, kNTile, sM + r, kMCap) : O::phase(k, sM + r, kMCap, sN + c, kNTile);
      out[e] = polar1(phi);
      step();
    }
  }
}

// Generic (unstaged) fill: kernels without a phase, or blocks taller than
// the staging capacity.
template <bool TRANS>
__device__ __forceinline__ void fill_generic(const DevK& k, const int* __restrict__ rid, const int* __restrict__ cid,
                                             int ro, int nr, int co, int nc, double2* __restrict__ B) {
  const int m = TRANS ? nc : nr;
  const int total = nr * nc;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int c = e / m, r = e - c * m;
    B[e] = TRANS ? entry(k, rid[ro + c], cid[co + r]) : entry(k, rid[ro + r], cid[co + c]);
  }
}

template <int KIND, bool TRANS>
__device__ __forceinline__ void fill_block(const DevK& k, const int* __restrict__ rid, const int* __restrict__ cid,
                                           int ro, int nr, int co, int nc, double2* __restrict__ B, double* sm) {
  if ((TRANS ? nc : nr) <= kMCap)
    fill_staged<KIND, TRANS>(k, rid, cid, ro, nr, co, nc, B, sm);
  else
    fill_generic<TRANS>(k, rid, cid, ro, nr, co, nc, B);
}

template <int KIND>
__global__ void __launch_bounds__(256) k3_sample_s(DevK k, const int* __restrict__ tasks, const int* __restrict__ rid,
                                                   const int* __restrict__ cid, double2* __restrict__ out) {
  extern __shared__ double sm[];
  const int* tk = tasks + 5 * blockIdx.x;
  fill_block<KIND, false>(k, rid, cid, tk[0], tk[1], tk[2], tk[3], out + tk[4], sm);
}

template <int KIND, bool TRANS>
__global__ void __launch_bounds__(256) k3_sample_ws_s(DevK k, const int4* __restrict__ rc,
                                                      const IdTask* __restrict__ tasks, const int* __restrict__ rid,
                                                      const int* __restrict__ cid, double2* __restrict__ ws) {
  extern __shared__ double sm[];
  const int4 q = rc[blockIdx.x];
  fill_block<KIND, TRANS>(k, rid, cid, q.x, q.y, q.z, q.w, ws + tasks[blockIdx.x].off, sm);
}

// Direct sum, staged: the CTA's 256 rows and each 256-column tile of
// operands (plus f) in shared memory.
template <int KIND>
__global__ void __launch_bounds__(256) k4_direct_s(DevK k, const int* __restrict__ rows, int nsel,
                                                   const double2* __restrict__ f, int64_t ncols, int64_t cps,
                                                   double2* __restrict__ partial) {
  using O = Ops<KIND>;
  constexpr int kT = 256;
  __shared__ double sR[kMaxW * kT];
  __shared__ double sC[kMaxW * kT];
  __shared__ double2 fs[kT];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c0 = blockIdx.y * cps, c1 = min(ncols, c0 + cps);
  O::row(k, r < nsel ? rows[r] : rows[0], sR + threadIdx.x, kT);
  double ar = 0.0, ai = 0.0;
  for (int64_t cb = c0; cb < c1; cb += kT) {
    const int cn = static_cast<int>(c1 - cb < kT ? c1 - cb : kT);
    __syncthreads();
    if (threadIdx.x < cn) {
      fs[threadIdx.x] = f[cb + threadIdx.x];
      O::col(k, cb + threadIdx.x, sC + threadIdx.x, kT);
    }
    __syncthreads();
    if (r < nsel) {
      auto mac = [&](double2 e, double2 x) {  // acc += K * f, std::complex's product (no fma)
        ar = __dadd_rn(ar, __dsub_rn(__dmul_rn(e.x, x.x), __dmul_rn(e.y, x.y)));
        ai = __dadd_rn(ai, __dadd_rn(__dmul_rn(e.x, x.y), __dmul_rn(e.y, x.x)));
      };
      int q = 0;
      for (; q + 3 < cn; q += 4) {  // four entries' sincos interleaved, accumulated in column order
        double ph[4];
        double2 e[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) ph[i] = O::phase(k, sR + threadIdx.x, kT, sC + q + i, kT);
        polar1x4(ph, e);
#pragma unroll
        for (int i = 0; i < 4; ++i) mac(e[i], fs[q + i]);
      }
      for (; q + 1 < cn; q += 2) {  // two entries' sincos interleaved
        double2 e0, e1;
        polar1x2(O::phase(k, sR + threadIdx.x, kT, sC + q, kT), O::phase(k, sR + threadIdx.x, kT, sC + q + 1, kT),
                 &e0, &e1);
        mac(e0, fs[q]);
        mac(e1, fs[q + 1]);
      }
      if (q < cn) mac(polar1(O::phase(k, sR + threadIdx.x, kT, sC + q, kT)), fs[q]);
    }
  }
  if (r < nsel) partial[static_cast<int64_t>(blockIdx.y) * nsel + r] = make_double2(ar, ai);
}

// Direct sum: blockIdx.x covers 256 selected rows (one per thread),
// blockIdx.y a contiguous column split.  Column data staged in shared memory.
constexpr int kTile = 256;
__global__ void __launch_bounds__(256) k4_direct(DevK k, const int* __restrict__ rows, int nsel,
                                                 const double2* __restrict__ f, int64_t ncols, int64_t cps,
                                                 double2* __restrict__ partial) {
  __shared__ double2 fs[kTile];
  __shared__ int js[kTile];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c0 = blockIdx.y * cps, c1 = min(ncols, c0 + cps);
  const int64_t i = r < nsel ? rows[r] : 0;
  double ar = 0.0, ai = 0.0;
  for (int64_t cb = c0; cb < c1; cb += kTile) {
    const int cn = static_cast<int>(c1 - cb < kTile ? c1 - cb : kTile);
    __syncthreads();
    if (threadIdx.x < cn) {
      fs[threadIdx.x] = f[cb + threadIdx.x];
      js[threadIdx.x] = static_cast<int>(cb + threadIdx.x);
    }
    __syncthreads();
    if (r < nsel) {
      for (int q = 0; q < cn; ++q) {
        const double2 e = entry(k, i, js[q]);
        const double2 x = fs[q];
        // acc += K * f, the same complex product as std::complex (no fma)
        ar = __dadd_rn(ar, __dsub_rn(__dmul_rn(e.x, x.x), __dmul_rn(e.y, x.y)));
        ai = __dadd_rn(ai, __dadd_rn(__dmul_rn(e.x, x.y), __dmul_rn(e.y, x.x)));
      }
    }
  }
  if (r < nsel) partial[static_cast<int64_t>(blockIdx.y) * nsel + r] = make_double2(ar, ai);
}

__global__ void k4_reduce(const double2* __restrict__ partial, int nsel, int nsplit, double2* __restrict__ g) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nsel) return;
  double ar = 0.0, ai = 0.0;
  for (int s = 0; s < nsplit; ++s) {
    const double2 p = partial[static_cast<int64_t>(s) * nsel + r];
    ar += p.x;
    ai += p.y;
  }
  g[r] = make_double2(ar, ai);
}

// Launchers: the staged kernels for kernels with a phase (and operands that
// fit the staging width), the generic ones otherwise.
void launch_k3(const DevK& k, unsigned grid, cudaStream_t st, const int* tasks, const int* rid, const int* cid,
               double2* out) {
  if (!stageable(k.kind, k.rank, k.dim)) {
    k3_sample<<<grid, 256, 0, st>>>(k, tasks, rid, cid, out);
    return;
  }
  switch (k.kind) {
    case MIDBF_KERNEL_FIO2D:
      k3_sample_s<MIDBF_KERNEL_FIO2D><<<grid, 256, stage_smem<MIDBF_KERNEL_FIO2D>(), st>>>(k, tasks, rid, cid, out);
      break;
    case MIDBF_KERNEL_FIO3D:
      k3_sample_s<MIDBF_KERNEL_FIO3D><<<grid, 256, stage_smem<MIDBF_KERNEL_FIO3D>(), st>>>(k, tasks, rid, cid, out);
      break;
    case MIDBF_KERNEL_LOWRANK:
      k3_sample_s<MIDBF_KERNEL_LOWRANK><<<grid, 256, stage_smem<MIDBF_KERNEL_LOWRANK>(), st>>>(k, tasks, rid, cid, out);
      break;
    default:
      k3_sample_s<MIDBF_KERNEL_NUFFT><<<grid, 256, stage_smem<MIDBF_KERNEL_NUFFT>(), st>>>(k, tasks, rid, cid, out);
      break;
  }
}

template <bool TRANS>
void launch_k3_ws(const DevK& k, unsigned grid, cudaStream_t st, const int4* rc, const IdTask* tk, const int* rid,
                  const int* cid, double2* ws) {
  if (!stageable(k.kind, k.rank, k.dim)) {
    k3_sample_ws<TRANS><<<grid, 256, 0, st>>>(k, rc, tk, rid, cid, ws);
    return;
  }
  switch (k.kind) {
    case MIDBF_KERNEL_FIO2D:
      k3_sample_ws_s<MIDBF_KERNEL_FIO2D, TRANS><<<grid, 256, stage_smem<MIDBF_KERNEL_FIO2D>(), st>>>(k, rc, tk, rid, cid, ws);
      break;
    case MIDBF_KERNEL_FIO3D:
      k3_sample_ws_s<MIDBF_KERNEL_FIO3D, TRANS><<<grid, 256, stage_smem<MIDBF_KERNEL_FIO3D>(), st>>>(k, rc, tk, rid, cid, ws);
      break;
    case MIDBF_KERNEL_LOWRANK:
      k3_sample_ws_s<MIDBF_KERNEL_LOWRANK, TRANS><<<grid, 256, stage_smem<MIDBF_KERNEL_LOWRANK>(), st>>>(k, rc, tk, rid, cid, ws);
      break;
    default:
      k3_sample_ws_s<MIDBF_KERNEL_NUFFT, TRANS><<<grid, 256, stage_smem<MIDBF_KERNEL_NUFFT>(), st>>>(k, rc, tk, rid, cid, ws);
      break;
  }
}

void launch_k4(const DevK& k, dim3 grid, cudaStream_t st, const int* rows, int nsel, const double2* f, int64_t ncols,
               int64_t cps, double2* part) {
  if (!stageable(k.kind, k.rank, k.dim)) {
    k4_direct<<<grid, 256, 0, st>>>(k, rows, nsel, f, ncols, cps, part);
    return;
  }
  switch (k.kind) {
    case MIDBF_KERNEL_FIO2D:
      k4_direct_s<MIDBF_KERNEL_FIO2D><<<grid, 256, 0, st>>>(k, rows, nsel, f, ncols, cps, part);
      break;
    case MIDBF_KERNEL_FIO3D:
      k4_direct_s<MIDBF_KERNEL_FIO3D><<<grid, 256, 0, st>>>(k, rows, nsel, f, ncols, cps, part);
      break;
    case MIDBF_KERNEL_LOWRANK:
      k4_direct_s<MIDBF_KERNEL_LOWRANK><<<grid, 256, 0, st>>>(k, rows, nsel, f, ncols, cps, part);
      break;
    default:
      k4_direct_s<MIDBF_KERNEL_NUFFT><<<grid, 256, 0, st>>>(k, rows, nsel, f, ncols, cps, part);
      break;
  }
}

// K5 with the register capacity the tallest block needs (taller blocks
// return rank -1 from the kernel and are recomputed on the host).
void launch_k5(int64_t max_m, unsigned grid, cudaStream_t st, double2* ws, const IdTask* tk, int ntasks, int kmax,
               double eps, int rowid, double2* vals, int* rank, int* skel, int kcap) {
  // Warps per block, measured (round 1, K5 device ms per
  // factorization): 2D cfg1 8 warps 12.8 vs 4 warps 15.9 ms; 3D cfg3 (k5_id<16>,
  // 254 registers) 4 warps 73.3 vs 8 warps 76.3 ms.  Capping resident blocks
  // per SM so the in-flight blocks fit L2 was slower (cfg1 19.6-21.3 ms).
  auto go = [&](auto kern, size_t smem, int nthreads) {
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "k5 smem attribute");
    kern<<<grid, nthreads, smem, st>>>(ws, tk, ntasks, kmax, eps, rowid, vals, rank, skel, kcap);
  };
  // register slots sized to the tallest block (fewer registers, more
  // resident blocks): 2D k = 30 blocks are 150 x {64, 120} (t k = 150
  // samples), 3D k = 64 blocks 320 x {64, 512}
  if (max_m <= 160)
    go(k5_id<5, 8>, id_smem<5, 8>(id_r11(kmax)), 256);
  else if (max_m <= 256)
    go(k5_id<8, 8>, id_smem<8, 8>(id_r11(kmax)), 256);
  else if (max_m <= 320)
    go(k5_id<10, 4>, id_smem<10, 4>(id_r11(kmax)), 128);
  else
    go(k5_id<16, 4>, id_smem<16, 4>(id_r11(kmax)), 128);
}

template <class T>
T* upload(const T* h, size_t n, const char* what) {
  if (!h || n == 0) return nullptr;
  T* d = nullptr;
  cuda_check(cudaMalloc(&d, n * sizeof(T)), what);
  cuda_check(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice), what);
  return d;
}

}  // namespace

// K5 workspace, process-wide and grow-only (a factorization builds its own
// sampler; reallocating ~0.5 GB of device and pinned memory per call cost
// more than the IDs themselves).  Held under `mu` for a whole ID batch.
struct IdPool {
  std::mutex mu;
  double2* d_ws = nullptr;
  double2* d_vals = nullptr;
  double2* h_vals = nullptr;
  int* h_rank = nullptr;  // pinned: per-part D2H without a host-blocking staged copy
  int* h_skel = nullptr;
  int* d_rank = nullptr;
  int* d_skel = nullptr;
  int64_t ws_cap = 0, vals_cap = 0, hvals_cap = 0, rank_cap = 0, skel_cap = 0, hrank_cap = 0, hskel_cap = 0;
  template <typename T>
  static void grow(T*& p, int64_t& cap, int64_t need, bool pinned, const char* what) {
    if (need <= cap) return;
    const int64_t n = std::max<int64_t>(need, cap + cap / 2);
    if (pinned) {
      cudaFreeHost(p);
      p = nullptr;
      cuda_check(cudaMallocHost(&p, n * sizeof(T)), what);
    } else {
      cudaFree(p);
      p = nullptr;
      cuda_check(cudaMalloc(&p, n * sizeof(T)), what);
    }
    cap = n;
  }
};
IdPool& id_pool() {
  static IdPool* p = new IdPool;  // never destroyed: may outlive the CUDA context teardown order
  return *p;
}

// Double-buffered device output of sample_blocks (process-wide, allocated on
// first use); the pinned side is the shared staging pool (pool.hpp).
struct ChunkPool {
  static constexpr int64_t kChunk = static_cast<int64_t>(PinnedPool::kBytes / sizeof(double2));  // 4M entries
  double2* d_out[2] = {nullptr, nullptr};
  void ensure() {
    if (d_out[0]) return;
    for (int b = 0; b < 2; ++b) cuda_check(cudaMalloc(&d_out[b], kChunk * sizeof(double2)), "cudaMalloc sample buffer");
  }
};
ChunkPool& chunk_pool() {
  static ChunkPool* p = new ChunkPool;
  return *p;
}

struct EntrySampler::Impl {
  DevK k{};
  std::vector<void*> owned;
  int64_t nrows = 0, ncols = 0;
  int64_t launched_entries = 0;
  // Device time of the K3 / K5 launches (CUDA events on the sampler's
  // stream), collected at the synchronisation points of each call.
  struct Timed {
    cudaEvent_t a, b;
    int kind;  // 3: K3, 5: K5
    int64_t entries;
  };
  std::vector<Timed> pend;
  KernelTimes times;
  void begin(int kind, int64_t entries) {
    Timed t{nullptr, nullptr, kind, entries};
    cuda_check(cudaEventCreate(&t.a), "event");
    cuda_check(cudaEventCreate(&t.b), "event");
    cuda_check(cudaEventRecord(t.a, stream), "event record");
    pend.push_back(t);
  }
  void end() { cuda_check(cudaEventRecord(pend.back().b, stream), "event record"); }
  void collect() {  // after the stream has been synchronised
    for (Timed& t : pend) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
        if (t.kind == 3) {
          times.k3_seconds += 1e-3 * ms;
          times.k3_launches += 1;
          times.k3_entries += t.entries;
        } else {
          times.k5_seconds += 1e-3 * ms;
          times.k5_launches += 1;
        }
      }
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    pend.clear();
  }
  static constexpr int64_t kChunk = ChunkPool::kChunk;
  cudaStream_t stream = nullptr;
  cudaStream_t cstream = nullptr;  // ID batches: downloads overlapping the next part's kernels
  void ensure_stream() {
    if (!stream) cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    if (!cstream) cuda_check(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking), "stream");
  }
  ~Impl() {
    if (stream) cudaStreamDestroy(stream);
    if (cstream) cudaStreamDestroy(cstream);
  }
};

EntrySampler::EntrySampler(const midbf_kernel_desc& kd) : impl_(new Impl) {
  require_device();
  Impl& I = *impl_;
  I.nrows = kd.nrows;
  I.ncols = kd.ncols;
  if (kd.nrows < 0 || kd.ncols < 0 || kd.nrows > 0x7fffffff || kd.ncols > 0x7fffffff)
    throw std::invalid_argument("kernel point counts out of range");
  DevK& k = I.k;
  k.kind = kd.kind;
  k.dim = kd.dim;
  k.rank = kd.rank;
  k.cre = kd.cre;
  k.cim = kd.cim;
  auto own = [&](void* p) {
    if (p) I.owned.push_back(p);
    return p;
  };
  switch (kd.kind) {
    case MIDBF_KERNEL_FIO2D:
    case MIDBF_KERNEL_FIO3D: {
      const int dim = kd.kind == MIDBF_KERNEL_FIO2D ? 2 : 3;
      if (kd.dim != dim || !kd.X || !kd.Omega) throw std::invalid_argument("FIO kernel needs X and Omega of matching dim");
      std::vector<double> coef(static_cast<size_t>(3 * kd.nrows), 0.0);
#pragma omp parallel for schedule(static) if (kd.nrows > 4096)  // (4 host sincos per point: 5 ms at N = 65536 serially)
      for (int64_t i = 0; i < kd.nrows; ++i) {
        const double* x = kd.X + dim * i;
        if (dim == 2) {  // src/kernels.cpp:20-21
          coef[3 * i] = (2.0 + std::sin(kTwoPi * x[0]) * std::sin(kTwoPi * x[1])) / 16.0;
          coef[3 * i + 1] = (2.0 + std::cos(kTwoPi * x[0]) * std::cos(kTwoPi * x[1])) / 16.0;
        } else {  // BASELINE.json configs[3]
          const double s0 = std::sin(kTwoPi * x[0]), s1 = std::sin(kTwoPi * x[1]), s2 = std::sin(kTwoPi * x[2]);
          const double c0 = std::cos(kTwoPi * x[0]), c1 = std::cos(kTwoPi * x[1]), c2 = std::cos(kTwoPi * x[2]);
          coef[3 * i] = (2.0 + s0 * s1 * s2) / 16.0;
          coef[3 * i + 1] = (2.0 + c0 * c1 * c2) / 16.0;
          coef[3 * i + 2] = (2.0 + s0 * c1 * s2) / 16.0;
        }
      }
      k.X = static_cast<double*>(own(upload(kd.X, static_cast<size_t>(dim * kd.nrows), "upload X")));
      k.Om = static_cast<double*>(own(upload(kd.Omega, static_cast<size_t>(dim * kd.ncols), "upload Omega")));
      k.coef = static_cast<double*>(own(upload(coef.data(), coef.size(), "upload coef")));
      break;
    }
    case MIDBF_KERNEL_NUFFT:
      if (kd.dim < 1 || !kd.X || !kd.Omega) throw std::invalid_argument("x.xi kernel needs X and Omega");
      k.X = static_cast<double*>(own(upload(kd.X, static_cast<size_t>(kd.dim * kd.nrows), "upload X")));
      k.Om = static_cast<double*>(own(upload(kd.Omega, static_cast<size_t>(kd.dim * kd.ncols), "upload Omega")));
      break;
    case MIDBF_KERNEL_LOWRANK:
      if (kd.rank < 1 || !kd.A || !kd.B) throw std::invalid_argument("low-rank kernel needs A and B");
      k.A = static_cast<double*>(own(upload(kd.A, static_cast<size_t>(kd.rank * kd.nrows), "upload A")));
      k.B = static_cast<double*>(own(upload(kd.B, static_cast<size_t>(kd.rank * kd.ncols), "upload B")));
      break;
    case MIDBF_KERNEL_CONST:
      break;
    case MIDBF_KERNEL_RANK1:
      if (!kd.u || !kd.v) throw std::invalid_argument("rank-one kernel needs u and v");
      k.u = static_cast<double2*>(own(upload(reinterpret_cast<const double2*>(kd.u), kd.nrows, "upload u")));
      k.v = static_cast<double2*>(own(upload(reinterpret_cast<const double2*>(kd.v), kd.ncols, "upload v")));
      break;
    default:
      throw std::invalid_argument("unknown kernel kind");
  }
}

EntrySampler::~EntrySampler() {
  for (void* p : impl_->owned) cudaFree(p);
}

int64_t EntrySampler::entries_evaluated() const { return impl_->launched_entries; }
EntrySampler::KernelTimes EntrySampler::kernel_times() const { return impl_->times; }

void EntrySampler::sample(int64_t ntasks, const int64_t* tasks, const int64_t* row_ids, int64_t n_row_ids,
                          const int64_t* col_ids, int64_t n_col_ids, double* out, int64_t out_len) {
  std::vector<double*> outs(static_cast<size_t>(ntasks));
  for (int64_t t = 0; t < ntasks; ++t) {
    const int64_t* tk = tasks + 5 * t;
    if (tk[4] < 0 || tk[1] < 0 || tk[3] < 0 || tk[4] + tk[1] * tk[3] > out_len)
      throw std::invalid_argument("sample task outside its output");
    outs[static_cast<size_t>(t)] = out + 2 * tk[4];
  }
  sample_blocks(ntasks, tasks, row_ids, n_row_ids, col_ids, n_col_ids, outs.data());
}

// Pipeline: chunk i's kernel and D2H copy run on the sampler's stream while
// the host scatters chunk i-1 from pinned memory into the destination blocks
// (OpenMP over tasks).
void EntrySampler::sample_blocks(int64_t ntasks, const int64_t* tasks, const int64_t* row_ids, int64_t n_row_ids,
                                 const int64_t* col_ids, int64_t n_col_ids, double* const* outs) {
  Impl& I = *impl_;
  if (ntasks <= 0) return;
  if (n_row_ids > 0x7fffffff || n_col_ids > 0x7fffffff) throw std::invalid_argument("too many sample ids");
  std::vector<int> rid(static_cast<size_t>(n_row_ids)), cid(static_cast<size_t>(n_col_ids));
  for (int64_t q = 0; q < n_row_ids; ++q) {
    if (row_ids[q] < 0 || row_ids[q] >= I.nrows) throw std::invalid_argument("row id out of range");
    rid[q] = static_cast<int>(row_ids[q]);
  }
  for (int64_t q = 0; q < n_col_ids; ++q) {
    if (col_ids[q] < 0 || col_ids[q] >= I.ncols) throw std::invalid_argument("column id out of range");
    cid[q] = static_cast<int>(col_ids[q]);
  }
  // Sub-tasks: a block larger than kTaskEntries is split into column ranges;
  // chunks = consecutive sub-tasks with <= kChunk entries.
  struct Sub {
    int ro, nr, co, nc;
    double* dst;
  };
  std::vector<Sub> subs;
  subs.reserve(static_cast<size_t>(ntasks));
  for (int64_t t = 0; t < ntasks; ++t) {
    const int64_t* tk = tasks + 5 * t;
    if (tk[1] < 0 || tk[3] < 0 || tk[0] < 0 || tk[2] < 0 || tk[0] + tk[1] > n_row_ids || tk[2] + tk[3] > n_col_ids)
      throw std::invalid_argument("sample task outside its id lists");
    if (tk[1] == 0 || tk[3] == 0) continue;
    // sub-tasks of <= kTaskEntries entries (one CTA each): a few large
    // blocks (3D S blocks, 512 x 512) must still fill all 148 SMs
    const int64_t cols_per = std::max<int64_t>(1, std::min(Impl::kChunk, kTaskEntries) / tk[1]);
    if (tk[1] > Impl::kChunk) throw std::invalid_argument("sample block taller than the sampler chunk");
    for (int64_t c0 = 0; c0 < tk[3]; c0 += cols_per)
      subs.push_back({static_cast<int>(tk[0]), static_cast<int>(tk[1]), static_cast<int>(tk[2] + c0),
                      static_cast<int>(std::min<int64_t>(cols_per, tk[3] - c0)), outs[t] + 2 * c0 * tk[1]});
  }
  const int64_t nsub = static_cast<int64_t>(subs.size());
  if (nsub == 0) return;
  std::vector<int> dt(static_cast<size_t>(5 * nsub));
  std::vector<int64_t> chunk_begin{0}, chunk_entries;
  int64_t acc = 0;
  for (int64_t t = 0; t < nsub; ++t) {
    const Sub& u = subs[static_cast<size_t>(t)];
    const int64_t n = static_cast<int64_t>(u.nr) * u.nc;
    if (acc + n > Impl::kChunk) {
      chunk_entries.push_back(acc);
      chunk_begin.push_back(t);
      acc = 0;
    }
    int* d = &dt[static_cast<size_t>(5 * t)];
    d[0] = u.ro;
    d[1] = u.nr;
    d[2] = u.co;
    d[3] = u.nc;
    d[4] = static_cast<int>(acc);
    acc += n;
  }
  chunk_entries.push_back(acc);
  chunk_begin.push_back(nsub);
  I.ensure_stream();
  ChunkPool& CP = chunk_pool();
  PinnedPool& PP = pinned_pool();
  std::lock_guard<std::mutex> lock(PP.mu);
  PP.ensure();
  CP.ensure();
  int* d_rid = upload(rid.data(), rid.size(), "upload row ids");
  int* d_cid = upload(cid.data(), cid.size(), "upload col ids");
  int* d_tasks = upload(dt.data(), dt.size(), "upload tasks");
  const int64_t nchunks = static_cast<int64_t>(chunk_entries.size());
  auto scatter = [&](int64_t c) {
    const int b = static_cast<int>(c & 1);
    cuda_check(cudaEventSynchronize(PP.ev[b]), "sample chunk");
    const double2* src = reinterpret_cast<double2*>(PP.h[b]);
    const int64_t t0 = chunk_begin[static_cast<size_t>(c)], t1 = chunk_begin[static_cast<size_t>(c + 1)];
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = t0; t < t1; ++t) {
      const Sub& u = subs[static_cast<size_t>(t)];
      std::memcpy(u.dst, src + dt[static_cast<size_t>(5 * t + 4)], static_cast<size_t>(16) * u.nr * u.nc);
    }
  };
  try {
    for (int64_t c = 0; c < nchunks; ++c) {
      const int b = static_cast<int>(c & 1);
      if (c >= 2) cuda_check(cudaEventSynchronize(PP.ev[b]), "sample buffer reuse");
      const int64_t t0 = chunk_begin[static_cast<size_t>(c)], t1 = chunk_begin[static_cast<size_t>(c + 1)];
      if (chunk_entries[static_cast<size_t>(c)] > 0) {
        I.begin(3, chunk_entries[static_cast<size_t>(c)]);
        launch_k3(I.k, static_cast<unsigned>(t1 - t0), I.stream, d_tasks + 5 * t0, d_rid, d_cid, CP.d_out[b]);
        cuda_check(cudaGetLastError(), "k3_sample launch");
        I.end();
        cuda_check(cudaMemcpyAsync(reinterpret_cast<double2*>(PP.h[b]), CP.d_out[b], chunk_entries[static_cast<size_t>(c)] * sizeof(double2),
                                   cudaMemcpyDeviceToHost, I.stream),
                   "sample D2H");
      }
      cuda_check(cudaEventRecord(PP.ev[b], I.stream), "event record");
      if (c >= 1) scatter(c - 1);
      I.launched_entries += chunk_entries[static_cast<size_t>(c)];
    }
    scatter(nchunks - 1);
    cuda_check(cudaStreamSynchronize(I.stream), "sampler");
    I.collect();
  } catch (...) {
    cudaStreamSynchronize(I.stream);
    I.collect();
    cudaFree(d_rid);
    cudaFree(d_cid);
    cudaFree(d_tasks);
    throw;
  }
  cudaFree(d_rid);
  cudaFree(d_cid);
  cudaFree(d_tasks);
}

void EntrySampler::sample_ids(int64_t ntasks, const int64_t* tasks, const int64_t* row_ids, int64_t n_row_ids,
                              const int64_t* col_ids, int64_t n_col_ids, bool rowid, int64_t k_max, double eps,
                              IdBatch& out, const std::function<void(int64_t, int64_t)>& on_part) {
  Impl& I = *impl_;
  static const bool timing = std::getenv("MIDBF_ID_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t_start = now();
  out.rank.assign(static_cast<size_t>(ntasks), 0);
  out.ooff.assign(static_cast<size_t>(ntasks), 0);
  out.kcap = 0;
  out.vals = nullptr;
  if (ntasks <= 0) return;
  if (ntasks > 0x7fffffff || n_row_ids > 0x7fffffff || n_col_ids > 0x7fffffff)
    throw std::invalid_argument("too many ID tasks");
  std::vector<int> rid(static_cast<size_t>(n_row_ids)), cid(static_cast<size_t>(n_col_ids));
  for (int64_t q = 0; q < n_row_ids; ++q) {
    if (row_ids[q] < 0 || row_ids[q] >= I.nrows) throw std::invalid_argument("row id out of range");
    rid[q] = static_cast<int>(row_ids[q]);
  }
  for (int64_t q = 0; q < n_col_ids; ++q) {
    if (col_ids[q] < 0 || col_ids[q] >= I.ncols) throw std::invalid_argument("column id out of range");
    cid[q] = static_cast<int>(col_ids[q]);
  }
  std::vector<int4> rc(static_cast<size_t>(ntasks));
  std::vector<IdTask> tk(static_cast<size_t>(ntasks));
  int64_t ws = 0, vals = 0;
  int kcap = 1;
  int64_t max_m = 0;
  for (int64_t t = 0; t < ntasks; ++t) {
    const int64_t* q = tasks + 5 * t;
    if (q[1] <= 0 || q[3] <= 0 || q[0] < 0 || q[2] < 0 || q[0] + q[1] > n_row_ids || q[2] + q[3] > n_col_ids)
      throw std::invalid_argument("ID task outside its id lists (or empty)");
    const int64_t m = rowid ? q[3] : q[1], n = rowid ? q[1] : q[3];
    if (m * n > 0x7fffffff) throw std::invalid_argument("ID block too large");
    const int64_t full = std::min(m, n), cap = k_max > 0 ? std::min(full, k_max) : full;
    rc[t] = make_int4(static_cast<int>(q[0]), static_cast<int>(q[1]), static_cast<int>(q[2]), static_cast<int>(q[3]));
    tk[t] = IdTask{ws, vals, static_cast<int32_t>(m), static_cast<int32_t>(n)};
    out.ooff[t] = 2 * vals;  // in doubles
    ws += m * n;
    vals += cap * n;
    kcap = std::max<int>(kcap, static_cast<int>(cap));
    max_m = std::max(max_m, m);
  }
  out.kcap = kcap;
  out.skel.assign(static_cast<size_t>(ntasks * kcap), 0);
  const auto t_prep = now();
  I.ensure_stream();
  IdPool& P = id_pool();
  std::lock_guard<std::mutex> lock(P.mu);
  IdPool::grow(P.d_ws, P.ws_cap, ws, false, "cudaMalloc ID workspace");
  IdPool::grow(P.d_vals, P.vals_cap, vals, false, "cudaMalloc ID values");
  IdPool::grow(P.h_vals, P.hvals_cap, vals, true, "cudaMallocHost ID values");
  IdPool::grow(P.d_rank, P.rank_cap, ntasks, false, "cudaMalloc ranks");
  IdPool::grow(P.d_skel, P.skel_cap, ntasks * kcap, false, "cudaMalloc skeletons");
  IdPool::grow(P.h_rank, P.hrank_cap, ntasks, true, "cudaMallocHost ranks");
  IdPool::grow(P.h_skel, P.hskel_cap, ntasks * kcap, true, "cudaMallocHost skeletons");
  int* d_rid = upload(rid.data(), rid.size(), "upload row ids");
  int* d_cid = upload(cid.data(), cid.size(), "upload col ids");
  int4* d_rc = upload(rc.data(), rc.size(), "upload ID tasks");
  IdTask* d_tk = upload(tk.data(), tk.size(), "upload ID tasks");
  const auto t_up = now();
  auto cleanup = [&] {
    cudaFree(d_rid);
    cudaFree(d_cid);
    cudaFree(d_rc);
    cudaFree(d_tk);
  };
  try {
    // Pipelined in parts: part p's V/W values download on a second stream
    // (and are copied out on the host, on_part) while part p+1 is
    // decomposed (K5) -- the values are contiguous per part (task order).  At least 256 tasks per part (about one K5 wave): smaller parts
    // leave the tall 3D blocks' K5 in partial waves (cfg3 4 parts of 128:
    // K5 68 -> 109 ms).  Measured (tools/fact_timing.py): cfg1 1024-task
    // batches 7 -> 3.6 ms, factorize 55 -> 44-46 ms with 4 parts (2: 48,
    // 8: 49-62); cfg3 512-task batches, 2 parts: 145 -> 134 ms.
    const int parts = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4, ntasks / 256)));
    std::vector<cudaEvent_t> evs;
    std::vector<cudaEvent_t> done(static_cast<size_t>(parts), nullptr);  // part's results on the host
    auto drop_events = [&] {
      for (cudaEvent_t e : evs) cudaEventDestroy(e);
      evs.clear();
      for (cudaEvent_t& e : done)
        if (e) cudaEventDestroy(e), e = nullptr;
    };
    out.vals = reinterpret_cast<const double*>(P.h_vals);
    // MIDBF_ID_TIMING: device timeline of the parts (kernels done / values on host)
    std::vector<cudaEvent_t> tev;
    auto tmark = [&](cudaStream_t st) {
      if (!timing) return;
      cudaEvent_t e = nullptr;
      if (cudaEventCreate(&e) == cudaSuccess && cudaEventRecord(e, st) == cudaSuccess) tev.push_back(e);
    };
    tmark(I.stream);
    try {
      // K3 samples every block of the batch in one launch (a CTA per task:
      // a part's 256 CTAs would leave the SMs half empty), then K5 runs per part
      I.begin(3, ws);
      if (rowid)
        launch_k3_ws<true>(I.k, static_cast<unsigned>(ntasks), I.stream, d_rc, d_tk, d_rid, d_cid, P.d_ws);
      else
        launch_k3_ws<false>(I.k, static_cast<unsigned>(ntasks), I.stream, d_rc, d_tk, d_rid, d_cid, P.d_ws);
      cuda_check(cudaGetLastError(), "k3_sample_ws launch");
      I.end();
      for (int part = 0; part < parts; ++part) {
        const int64_t t0 = ntasks * part / parts, t1 = ntasks * (part + 1) / parts;
        if (t1 <= t0) continue;
        const unsigned nt = static_cast<unsigned>(t1 - t0);
        I.begin(5, 0);
        launch_k5(max_m, nt, I.stream, P.d_ws, d_tk + t0, static_cast<int>(nt),
                  static_cast<int>(std::max<int64_t>(k_max, 0)), eps, rowid ? 1 : 0, P.d_vals, P.d_rank + t0,
                  P.d_skel + t0 * kcap, kcap);
        cuda_check(cudaGetLastError(), "k5_id launch");
        I.end();
        tmark(I.stream);
        cudaEvent_t ev = nullptr;
        cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        evs.push_back(ev);
        cuda_check(cudaEventRecord(ev, I.stream), "event record");
        cuda_check(cudaStreamWaitEvent(I.cstream, ev, 0), "event wait");
        const int64_t v0 = tk[static_cast<size_t>(t0)].ooff, v1 = t1 < ntasks ? tk[static_cast<size_t>(t1)].ooff : vals;
        if (v1 > v0)
          cuda_check(cudaMemcpyAsync(P.h_vals + v0, P.d_vals + v0, (v1 - v0) * sizeof(double2),
                                     cudaMemcpyDeviceToHost, I.cstream),
                     "ID values D2H");
        // (pinned staging: a D2H into pageable memory would block the host
        // until the part is done, serialising the issue of the later parts)
        cuda_check(cudaMemcpyAsync(P.h_rank + t0, P.d_rank + t0, (t1 - t0) * sizeof(int), cudaMemcpyDeviceToHost,
                                   I.cstream),
                   "ID ranks D2H");
        cuda_check(cudaMemcpyAsync(P.h_skel + t0 * kcap, P.d_skel + t0 * kcap, (t1 - t0) * kcap * sizeof(int),
                                   cudaMemcpyDeviceToHost, I.cstream),
                   "ID skeletons D2H");
        cuda_check(cudaEventCreateWithFlags(&done[static_cast<size_t>(part)], cudaEventDisableTiming), "event");
        cuda_check(cudaEventRecord(done[static_cast<size_t>(part)], I.cstream), "event record");
        tmark(I.cstream);
      }
      if (timing)
        std::fprintf(stderr, "[id]   issued at %.2f ms\n", 1e3 * std::chrono::duration<double>(now() - t_up).count());
      // hand finished parts to the caller (host copy-out) while later parts compute
      for (int part = 0; part < parts; ++part) {
        const int64_t t0 = ntasks * part / parts, t1 = ntasks * (part + 1) / parts;
        if (t1 <= t0) continue;
        cuda_check(cudaEventSynchronize(done[static_cast<size_t>(part)]), "ID part");
        std::memcpy(out.rank.data() + t0, P.h_rank + t0, static_cast<size_t>(t1 - t0) * sizeof(int));
        std::memcpy(out.skel.data() + t0 * kcap, P.h_skel + t0 * kcap, static_cast<size_t>((t1 - t0) * kcap) * sizeof(int));
        const auto t_ready = now();
        if (on_part) on_part(t0, t1);
        if (timing)
          std::fprintf(stderr, "[id]   part %d: results on host at %.2f ms, copied out at %.2f ms\n", part,
                       1e3 * std::chrono::duration<double>(t_ready - t_up).count(),
                       1e3 * std::chrono::duration<double>(now() - t_up).count());
      }
    } catch (...) {
      cudaStreamSynchronize(I.stream);
      cudaStreamSynchronize(I.cstream);
      drop_events();
      throw;
    }
    if (timing) cuda_check(cudaStreamSynchronize(I.stream), "ID kernels");
    const auto t_k = now();
    if (timing)
      std::fprintf(stderr, "[id] tasks %lld prep %.2f ms upload+alloc %.2f ms kernels %.2f ms\n",
                   static_cast<long long>(ntasks), 1e3 * std::chrono::duration<double>(t_prep - t_start).count(),
                   1e3 * std::chrono::duration<double>(t_up - t_prep).count(),
                   1e3 * std::chrono::duration<double>(t_k - t_up).count());
    cuda_check(cudaStreamSynchronize(I.stream), "ID batch");
    const cudaError_t ce = cudaStreamSynchronize(I.cstream);
    if (timing && ce == cudaSuccess) {
      std::string line = "[id]   device timeline (ms, kernels done | values on host):";
      for (size_t q = 1; q < tev.size(); ++q) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[0], tev[q]);
        char b[32];
        std::snprintf(b, sizeof b, " %.2f", ms);
        line += b;
      }
      std::fprintf(stderr, "%s\n", line.c_str());
    }
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
    drop_events();
    cuda_check(ce, "ID values D2H");
    I.collect();
    if (timing)
      std::fprintf(stderr, "[id] D2H %.2f ms (%lld MB)\n", 1e3 * std::chrono::duration<double>(now() - t_k).count(),
                   static_cast<long long>(vals * 16 >> 20));
  } catch (...) {
    cudaStreamSynchronize(I.stream);
    cudaStreamSynchronize(I.cstream);
    I.collect();
    cleanup();
    throw;
  }
  cleanup();
  I.launched_entries += ws;
}

void EntrySampler::phase_block(int64_t nr, const int64_t* rows, int64_t nc, const int64_t* cols, double* out) {
  Impl& I = *impl_;
  const int kind = I.k.kind;
  if (kind != MIDBF_KERNEL_FIO2D && kind != MIDBF_KERNEL_FIO3D && kind != MIDBF_KERNEL_LOWRANK &&
      kind != MIDBF_KERNEL_NUFFT)
    throw std::invalid_argument("this kernel has no phase");
  if (nr <= 0 || nc <= 0) return;
  if (nr > 0x7fffffff || nc > 0x7fffffff) throw std::invalid_argument("phase block too large");
  auto ids = [](const int64_t* v, int64_t n, int64_t lim, const char* what) {
    std::vector<int> o;
    if (!v) return o;
    o.resize(static_cast<size_t>(n));
    for (int64_t q = 0; q < n; ++q) {
      if (v[q] < 0 || v[q] >= lim) throw std::invalid_argument(what);
      o[q] = static_cast<int>(v[q]);
    }
    return o;
  };
  if (!rows && nr > I.nrows) throw std::invalid_argument("phase rows out of range");
  if (!cols && nc > I.ncols) throw std::invalid_argument("phase columns out of range");
  const std::vector<int> r = ids(rows, nr, I.nrows, "phase row out of range");
  const std::vector<int> c = ids(cols, nc, I.ncols, "phase column out of range");
  I.ensure_stream();
  int* d_r = rows ? upload(r.data(), r.size(), "upload phase rows") : nullptr;
  int* d_c = cols ? upload(c.data(), c.size(), "upload phase cols") : nullptr;
  double* d_out = nullptr;
  const cudaError_t e0 = cudaMalloc(&d_out, nr * nc * sizeof(double));
  if (e0 == cudaSuccess) {
    const int64_t blocks = std::min<int64_t>((nr * nc + 255) / 256, 148 * 16);
    k3_phase<<<static_cast<unsigned>(blocks), 256, 0, I.stream>>>(I.k, d_r, static_cast<int>(nr), d_c,
                                                                   static_cast<int>(nc), d_out);
  }
  cudaError_t e = e0 != cudaSuccess ? e0 : cudaGetLastError();
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, d_out, nr * nc * sizeof(double), cudaMemcpyDeviceToHost, I.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(I.stream);
  cudaFree(d_out);
  cudaFree(d_r);
  cudaFree(d_c);
  cuda_check(e, "phase block");
}

// Device time of the calling thread's last direct sum (K4 + its fixed-order
// reduction, CUDA events), for throughput reporting.
double& last_direct_sum_seconds() {
  thread_local double s = 0.0;
  return s;
}

void EntrySampler::direct_sum(const double* f, const int64_t* rows, int64_t nsel, double* g) {
  Impl& I = *impl_;
  if (nsel == 0) return;
  std::vector<int> r(static_cast<size_t>(nsel));
  for (int64_t q = 0; q < nsel; ++q) {
    const int64_t v = rows ? rows[q] : q;
    if (v < 0 || v >= I.nrows) throw std::invalid_argument("direct-sum row out of range");
    r[q] = static_cast<int>(v);
  }
  if (nsel > 0x7fffffff) throw std::invalid_argument("too many rows");
  int* d_rows = upload(r.data(), r.size(), "upload rows");
  double2* d_f = upload(reinterpret_cast<const double2*>(f), static_cast<size_t>(I.ncols), "upload f");
  const int rb = static_cast<int>((nsel + 255) / 256);
  // ~16 CTAs per SM; column ranges down to 64 columns, so that a 256-row
  // eps_b sum (one row block) still fills the GPU
  const int64_t target = 148 * 16;
  int64_t nsplit = std::max<int64_t>(1, std::min<int64_t>((I.ncols + 63) / 64, (target + rb - 1) / rb));
  nsplit = std::min<int64_t>(nsplit, 65535);
  const int64_t cps = (I.ncols + nsplit - 1) / nsplit;
  double2 *d_part = nullptr, *d_g = nullptr;
  cuda_check(cudaMalloc(&d_part, nsplit * nsel * sizeof(double2)), "cudaMalloc partial");
  cuda_check(cudaMalloc(&d_g, nsel * sizeof(double2)), "cudaMalloc g");
  cudaEvent_t e0, e1;
  cuda_check(cudaEventCreate(&e0), "event");
  cuda_check(cudaEventCreate(&e1), "event");
  cuda_check(cudaEventRecord(e0, 0), "event");
  launch_k4(I.k, dim3(rb, static_cast<unsigned>(nsplit)), 0, d_rows, static_cast<int>(nsel), d_f, I.ncols, cps, d_part);
  cuda_check(cudaGetLastError(), "k4_direct launch");
  k4_reduce<<<rb, 256>>>(d_part, static_cast<int>(nsel), static_cast<int>(nsplit), d_g);
  cuda_check(cudaGetLastError(), "k4_reduce launch");
  cuda_check(cudaEventRecord(e1, 0), "event");
  cuda_check(cudaEventSynchronize(e1), "event");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  last_direct_sum_seconds() = 1e-3 * ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cuda_check(cudaMemcpy(g, d_g, nsel * sizeof(double2), cudaMemcpyDeviceToHost), "direct sum D2H");
  cudaFree(d_part);
  cudaFree(d_g);
  cudaFree(d_rows);
  cudaFree(d_f);
}

}  // namespace midbf::dev

using midbf::detail::guard;

// Batched column IDs of explicit host blocks (K5 only; midbf_cid_batch).
extern "C" int midbf_cid_batch(const double* blocks, const int64_t* dims, int64_t nblocks, int64_t k_max, double eps,
                               int64_t* ranks, int64_t* skel, int64_t kcap, double* vals) {
  using namespace midbf::dev;
  return guard([&] {
    require_device();
    if (nblocks < 0 || (nblocks > 0 && (!blocks || !dims || !ranks || !skel || !vals)))
      throw std::invalid_argument("null argument");
    if (nblocks == 0) return;
    if (nblocks > 0x7fffffff) throw std::invalid_argument("too many blocks");
    std::vector<IdTask> tk(static_cast<size_t>(nblocks));
    int64_t ws = 0, nv = 0;
    for (int64_t b = 0; b < nblocks; ++b) {
      const int64_t m = dims[2 * b], n = dims[2 * b + 1];
      if (m <= 0 || n <= 0 || m * n > 0x7fffffff) throw std::invalid_argument("ID block dimensions out of range");
      const int64_t full = std::min(m, n), cap = k_max > 0 ? std::min(full, k_max) : full;
      if (cap > kcap) throw std::invalid_argument("kcap smaller than a block's step cap");
      tk[b] = IdTask{ws, nv, static_cast<int32_t>(m), static_cast<int32_t>(n)};
      ws += m * n;
      nv += cap * n;
    }
    IdPool& P = id_pool();
    std::lock_guard<std::mutex> lock(P.mu);
    IdPool::grow(P.d_ws, P.ws_cap, ws, false, "cudaMalloc ID workspace");
    IdPool::grow(P.d_vals, P.vals_cap, nv, false, "cudaMalloc ID values");
    IdPool::grow(P.d_rank, P.rank_cap, nblocks, false, "cudaMalloc ranks");
    IdPool::grow(P.d_skel, P.skel_cap, nblocks * kcap, false, "cudaMalloc skeletons");
    cuda_check(cudaMemcpy(P.d_ws, blocks, ws * sizeof(double2), cudaMemcpyHostToDevice), "ID blocks H2D");
    IdTask* d_tk = upload(tk.data(), tk.size(), "upload ID tasks");
    const unsigned nt = static_cast<unsigned>(nblocks);
    int64_t max_m = 0;
    for (const IdTask& q : tk) max_m = std::max<int64_t>(max_m, q.m);
    launch_k5(max_m, nt, nullptr, P.d_ws, d_tk, static_cast<int>(nblocks), static_cast<int>(std::max<int64_t>(k_max, 0)),
              eps, 0, P.d_vals, P.d_rank, P.d_skel, static_cast<int>(kcap));
    const cudaError_t e = cudaGetLastError();
    std::vector<int> r(static_cast<size_t>(nblocks)), sk(static_cast<size_t>(nblocks * kcap), 0);
    if (e == cudaSuccess) {
      cuda_check(cudaMemcpy(r.data(), P.d_rank, nblocks * sizeof(int), cudaMemcpyDeviceToHost), "ranks D2H");
      cuda_check(cudaMemcpy(sk.data(), P.d_skel, nblocks * kcap * sizeof(int), cudaMemcpyDeviceToHost), "skel D2H");
      cuda_check(cudaMemcpy(vals, P.d_vals, nv * sizeof(double2), cudaMemcpyDeviceToHost), "V D2H");
    }
    cudaFree(d_tk);
    cuda_check(e, "k5_id launch");
    for (int64_t b = 0; b < nblocks; ++b) ranks[b] = r[b];
    for (int64_t q = 0; q < nblocks * kcap; ++q) skel[q] = sk[q];
  });
}


extern "C" int midbf_sample(const midbf_kernel_desc* kernel, int64_t ntasks, const int64_t* tasks,
                            const int64_t* row_ids, int64_t n_row_ids, const int64_t* col_ids, int64_t n_col_ids,
                            double* out, int64_t out_len) {
  return guard([&] {
    if (!kernel) throw std::invalid_argument("null kernel");
    midbf::dev::EntrySampler s(*kernel);
    s.sample(ntasks, tasks, row_ids, n_row_ids, col_ids, n_col_ids, out, out_len);
  });
}

extern "C" int midbf_direct_sum(const midbf_kernel_desc* kernel, const double* f, const int64_t* rows, int64_t nsel,
                                double* g) {
  return guard([&] {
    if (!kernel || !f || !g) throw std::invalid_argument("null argument");
    midbf::dev::EntrySampler s(*kernel);
    s.direct_sum(f, rows, nsel, g);
  });
}

extern "C" int midbf_last_direct_sum_seconds(double* out) {
  return guard([&] { *out = midbf::dev::last_direct_sum_seconds(); });
}

extern "C" int midbf_device_count(int* out) {
  return guard([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    int good = 0;
    for (int d = 0; d < n; ++d) {
      cudaDeviceProp p;
      if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++good;
    }
    *out = good;
  });
}
