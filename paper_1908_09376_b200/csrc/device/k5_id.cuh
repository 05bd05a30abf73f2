// K5 — batched interpolative decompositions on the device, sm_100a
// (SURVEY.md §8(f)1).
//
// Replaces the host IDs of shared_sweep (reference src/butterfly.cpp:466-472,
// 516-519 -> la::rid_from_cols / la::cid_from_rows, src/linalg.cpp:266-295),
// i.e. the truncated pivoted Householder QR pqr_impl (src/linalg.cpp:23-107)
// plus id_rank (:249-264) and V = [I, R11^-1 R12] P^T.  Same step sequence as
// the host restatement (csrc/host/linalg.cpp householder_qr): pivot = largest
// remaining squared norm (lowest index on ties), Householder vector
// v = [1; x(k+1:)/v0] with v0 = a0 + phase(a0) |x|, beta = 2 / (1 + |v|^2),
// trailing update c -= beta v (v^H c), squared-norm downdate with the
// reference's recompute guard (cur < 0 or cur <= 1e-12 ref).  Sums are warp
// butterfly reductions (fixed order: bitwise run to run, not bitwise equal
// to the host's serial sums).  The phase fix of R's rows is skipped: it
// cancels in R11^-1 R12 and leaves |R_ii| unchanged.
//
// One CTA of kIdWarps (8 for m <= 256, 4 above) warps per block: rows distributed over lanes (row i
// -> lane i % 32, register slot i / 32; m <= 32 * kIdRows), squared norms,
// the column permutation and the Householder vector in shared memory
// (n <= kIdCols).  Per step warp 0 picks the pivot and builds the reflector
// (positions are permuted, the columns stay where K3 sampled them: no column
// swaps through L2), then all warps update interleaved trailing columns, two
// per pass (two CTA barriers per step).  Blocks outside those limits,
// and blocks whose first min(m,n,k_max) diagonals hit id_rank's 1e-14 tail
// trim below the full factorization (the host's fallback case), return
// rank -1: the caller recomputes them on the host.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace midbf::dev {

// Register slots per lane ROWS: k5_id<8> takes m <= 256 (2D blocks, e.g.
// 150 x 120 at cfg1), k5_id<16> m <= 512 (3D blocks, 320 x 512 at cfg3).
constexpr int kIdRowsMax = 16;
constexpr int kIdCols = 512;           // n <= 512
// Dynamic shared memory: squared norms (current, reference), |R_ii|, the
// column permutation, the Householder vector and R11 (r11 x r11, the
// epilogue's triangular solves; r11 = k_max when 1 <= k_max <= 64, else 0
// and the epilogue reads R from the workspace).
constexpr int kIdR11Max = 64;
// Plus one column slot per warp: the warp's pivot candidate for the next
// step, kept on chip so the reflector does not re-read it through L2.
template <int ROWS, int WARPS>
constexpr size_t id_smem(int r11 = 0) {
  return size_t(kIdCols) * (8 + 8 + 8 + 4) + size_t(32 * ROWS) * 16 * (1 + WARPS) + size_t(r11) * r11 * 16 + 64;
}
__host__ __device__ inline int id_r11(int kmax) { return kmax >= 1 && kmax <= kIdR11Max ? kmax : 0; }

struct IdTask {
  int64_t off;   // block B (m x n, column-major) in the workspace
  int64_t ooff;  // output slot: cap x n complex
  int32_t m, n;
};

namespace k5dev {

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ double nrm2(double2 z) { return z.x * z.x + z.y * z.y; }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

}  // namespace k5dev

// ranks[t] = k (or -1: recompute on the host); skel[t * kcap + i] = perm[i];
// out + ooff: V (k x n, ld k) for a column ID, W = V^T (n x k, ld n) for a row
// ID (`rowid`: the workspace holds the transposed block).
template <int kIdRows, int kIdWarps>  // register slots per lane, warps cooperating on one block
__global__ void __launch_bounds__(kIdWarps * 32, kIdRows <= 5 ? 2 : 1) k5_id(double2* __restrict__ ws, const IdTask* __restrict__ tasks,
                                                       int ntasks, int kmax, double eps, int rowid,
                                                       double2* __restrict__ out, int* __restrict__ ranks,
                                                       int* __restrict__ skel, int kcap) {
  using namespace k5dev;
  constexpr int kIdMaxRows = 32 * kIdRows;
  extern __shared__ __align__(16) unsigned char k5smem[];
  double* cur = reinterpret_cast<double*>(k5smem);
  double* ref = cur + kIdCols;
  double* dg = ref + kIdCols;                               // |R_ii|
  double2* vsh = reinterpret_cast<double2*>(dg + kIdCols);  // Householder vector (rows)
  double2* R11 = vsh + kIdMaxRows;                          // r11 x r11 (epilogue)
  const int r11 = id_r11(kmax);
  int* perm = reinterpret_cast<int*>(R11 + r11 * r11);
  double2* cbuf = reinterpret_cast<double2*>(perm + kIdCols);  // [kIdWarps][kIdMaxRows] candidate columns
  __shared__ int sh_stop, sh_rank, sh_fb;
  __shared__ double sh_beta;
  __shared__ double cand_v[kIdWarps];  // per-warp pivot candidates of the next step (largest
  __shared__ int cand_p[kIdWarps];     // downdated norm, lowest position), set by the trailing update
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int t = blockIdx.x;
  if (t >= ntasks) return;
  const IdTask tk = tasks[t];
  const int m = tk.m, n = tk.n;
  if (m > kIdMaxRows || n > kIdCols || m <= 0 || n <= 0) {
    if (tid == 0) ranks[t] = -1;
    return;
  }
  double2* B = ws + tk.off;
  const int full = min(m, n);
  const int cap = kmax > 0 ? min(full, kmax) : full;

  // squared column norms (warp w: columns w, w + kIdWarps, ...)
  for (int j = w; j < n; j += kIdWarps) {
    const double2* c = B + static_cast<int64_t>(j) * m;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < kIdRows; ++r) {
      const int i = lane + 32 * r;
      if (i < m) s += nrm2(c[i]);
    }
    s = wsum(s);
    if (lane == 0) cur[j] = ref[j] = s;
  }
  for (int j = tid; j < n; j += kIdWarps * 32) perm[j] = j;
  __syncthreads();

  unsigned lmask = 0;  // slots of this lane that are rows of the block (row < m)
#pragma unroll
  for (int r = 0; r < kIdRows; ++r) lmask |= (lane + 32 * r < m) ? 1u << r : 0u;

  int k = 0;
  for (; k < cap; ++k) {
    if (w == 0) {  // pivot: largest remaining norm, lowest index on ties
      double bv = -1.0;
      int bp = n;
      if (k == 0) {
        for (int j = lane; j < n; j += 32)
          if (cur[j] > bv) bv = cur[j], bp = j;
      } else if (lane < kIdWarps) {  // the update of step k - 1 left one candidate per warp
        bv = cand_v[lane];
        bp = cand_p[lane];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        if (o >= kIdWarps && k > 0) continue;  // candidates sit in lanes 0 .. kIdWarps-1 (uniform branch)
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (ov > bv || (ov == bv && op < bp)) bv = ov, bp = op;
      }
      bp = __shfl_sync(0xffffffffu, bp, 0);
      // Positions are permuted, columns stay where K3 put them: position k
      // is column perm[k] of the workspace (no column swap through L2, and
      // the pivot and the reflector are one warp-0 phase)
      if (lane == 0 && bp != k) {
        const int tp = perm[k];
        perm[k] = perm[bp];
        perm[bp] = tp;
        double tv = cur[k];
        cur[k] = cur[bp];
        cur[bp] = tv;
        tv = ref[k];
        ref[k] = ref[bp];
        ref[bp] = tv;
      }
      __syncwarp();
      // Householder vector from position k's column (rows k..m-1)
      double2* col = B + static_cast<int64_t>(perm[k]) * m;
      // the winning candidate's warp (position bp was dealt to warp (bp - k) mod kIdWarps
      // by the update of step k - 1) left the updated column in its slot
      const double2* src = k == 0 ? col : cbuf + ((bp - k) % kIdWarps) * kIdMaxRows;
      double2 x[kIdRows];
#pragma unroll
      for (int r = 0; r < kIdRows; ++r) {
        const int i = lane + 32 * r;
        x[r] = (i >= k && i < m) ? src[i] : make_double2(0, 0);
      }
      double xs = 0.0;
#pragma unroll
      for (int r = 0; r < kIdRows; ++r) xs += nrm2(x[r]);
      xs = wsum(xs);
      const double xn = sqrt(xs);
      if (xn == 0.0) {
        if (lane == 0) sh_stop = 1;
      } else {
        double2 mine = make_double2(0, 0);  // row k's entry (static register indexing)
#pragma unroll
        for (int r = 0; r < kIdRows; ++r)
          if (r == (k >> 5)) mine = x[r];
        const double2 a0 =
            make_double2(__shfl_sync(0xffffffffu, mine.x, k & 31), __shfl_sync(0xffffffffu, mine.y, k & 31));
        const double aa = sqrt(nrm2(a0));
        const double2 ph = aa == 0.0 ? make_double2(1.0, 0.0) : make_double2(a0.x / aa, a0.y / aa);
        const double2 v0 = make_double2(a0.x + ph.x * xn, a0.y + ph.y * xn);
        const double iv = 1.0 / nrm2(v0);
        const double2 v0i = make_double2(v0.x * iv, -v0.y * iv);  // 1 / v0
        double vs = 0.0;
#pragma unroll
        for (int r = 0; r < kIdRows; ++r) {
          const int i = lane + 32 * r;
          if (i > k && i < m) {
            x[r] = cmul(x[r], v0i);
            vs += nrm2(x[r]);
            col[i] = x[r];
          }
        }
        vs = wsum(vs);
        const double2 rkk = make_double2(-ph.x * xn, -ph.y * xn);
        if (lane == (k & 31)) col[k] = rkk;
#pragma unroll
        for (int r = 0; r < kIdRows; ++r) {
          const int i = lane + 32 * r;
          if (i < m) vsh[i] = i == k ? make_double2(1.0, 0.0) : (i > k ? x[r] : make_double2(0, 0));
        }
        if (lane == 0) {
          dg[k] = sqrt(nrm2(rkk));
          sh_beta = 2.0 / (1.0 + vs);
          sh_stop = 0;
        }
      }
    }
    __syncthreads();
    if (sh_stop) break;
    const double beta = sh_beta;
    double2 v[kIdRows];
#pragma unroll
    for (int r = 0; r < kIdRows; ++r) {
      const int i = lane + 32 * r;
      v[r] = i < m ? vsh[i] : make_double2(0, 0);
    }
    // trailing columns (warp w: k+1+w, k+1+w+kIdWarps, ...): c -= beta v (v^H c),
    // two columns per pass (kIdRows <= 8) so their loads and reduction
    // chains overlap.  Every row below m is loaded (rows above k hold finished
    // R entries and meet v = 0) through a per-lane column pointer with
    // immediate slot offsets, only rows k..m-1 are stored back; explicit fma
    // chains.
    constexpr int kPair = kIdRows <= 8 ? 2 : 1;
    unsigned smask = 0;  // slots this lane stores: k <= row < m
#pragma unroll
    for (int r = 0; r < kIdRows; ++r) {
      const int i = lane + 32 * r;
      smask |= (i >= k && i < m) ? 1u << r : 0u;
    }
    const int kslot = k >> 5;
    double best_v = -1.0;
    int best_p = n;
    double2 cv[kPair][kIdRows];  // slots past row m stay zero (never loaded, v = 0 there)
#pragma unroll
    for (int u = 0; u < kPair; ++u)
#pragma unroll
      for (int r = 0; r < kIdRows; ++r) cv[u][r] = make_double2(0, 0);
    for (int j0 = k + 1 + w; j0 < n; j0 += kPair * kIdWarps) {
      double wr[kPair], wi[kPair];
#pragma unroll
      for (int u = 0; u < kPair; ++u) {
        const int j = j0 + u * kIdWarps;
        const double2* c = B + static_cast<int64_t>(j < n ? perm[j] : 0) * m + lane;
        wr[u] = 0.0;
        wi[u] = 0.0;
#pragma unroll
        for (int r = 0; r < kIdRows; ++r)
          if (lmask >> r & 1u) cv[u][r] = c[32 * r];
      }
#pragma unroll
      for (int u = 0; u < kPair; ++u)
#pragma unroll
        for (int r = 0; r < kIdRows; ++r) {  // w += conj(c) v
          wr[u] = fma(cv[u][r].x, v[r].x, wr[u]);
          wr[u] = fma(cv[u][r].y, v[r].y, wr[u]);
          wi[u] = fma(cv[u][r].x, v[r].y, wi[u]);
          wi[u] = fma(-cv[u][r].y, v[r].x, wi[u]);
        }
      if constexpr (kPair == 2) {
        // The four sums reduce together: the first two rounds halve what
        // each lane carries (6 shuffled doubles instead of 20), then
        // lanes 0 / 8 / 16 / 24 hold wr0 / wi0 / wr1 / wi1 and broadcast them.
        const bool hi = lane & 16, b3 = lane & 8;
        double k0 = hi ? wr[1] : wr[0], k1 = hi ? wi[1] : wi[0];
        k0 += __shfl_xor_sync(0xffffffffu, hi ? wr[0] : wr[1], 16);
        k1 += __shfl_xor_sync(0xffffffffu, hi ? wi[0] : wi[1], 16);
        double t = b3 ? k1 : k0;
        t += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        wr[0] = __shfl_sync(0xffffffffu, t, 0);
        wi[0] = __shfl_sync(0xffffffffu, t, 8);
        wr[1] = __shfl_sync(0xffffffffu, t, 16);
        wi[1] = __shfl_sync(0xffffffffu, t, 24);
      } else {
        static_assert(kPair == 1, "one or two columns per pass");
        // the real and the imaginary sum share the rounds after the first:
        // lanes 0 / 16 end with wr / wi (5 shuffled doubles instead of 10)
        const bool hi = lane & 16;
        double t = hi ? wi[0] : wr[0];
        t += __shfl_xor_sync(0xffffffffu, hi ? wr[0] : wi[0], 16);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        wr[0] = __shfl_sync(0xffffffffu, t, 0);
        wi[0] = __shfl_sync(0xffffffffu, t, 16);
      }
#pragma unroll
      for (int u = 0; u < kPair; ++u) {
        const int j = j0 + u * kIdWarps;
        if (j >= n) break;
        double2* c = B + static_cast<int64_t>(perm[j]) * m + lane;
        const double2 cw = make_double2(beta * wr[u], -beta * wi[u]);  // beta conj(w)
#pragma unroll
        for (int r = 0; r < kIdRows; ++r) {  // c -= v cw
          cv[u][r].x = fma(-v[r].x, cw.x, cv[u][r].x);
          cv[u][r].x = fma(v[r].y, cw.y, cv[u][r].x);
          cv[u][r].y = fma(-v[r].x, cw.y, cv[u][r].y);
          cv[u][r].y = fma(-v[r].y, cw.x, cv[u][r].y);
          if (smask >> r & 1u) c[32 * r] = cv[u][r];
        }
        double2 ek = cv[u][0];  // row k's slot (uniform: slot 0 while k < 32)
        if (kslot != 0) {
#pragma unroll
          for (int r = 1; r < kIdRows; ++r)
            if (r == kslot) ek = cv[u][r];
        }
        double ck = nrm2(ek);
        ck = __shfl_sync(0xffffffffu, ck, k & 31);
        double cj = cur[j] - ck;
        double rj = ref[j];
        if (cj < 0.0 || cj <= 1e-12 * rj) {  // recompute guard (warp-uniform, rare): rows below k
          double rest = 0.0;
#pragma unroll
          for (int r = 0; r < kIdRows; ++r) {
            const int i = lane + 32 * r;
            if (i > k && i < m) rest += nrm2(cv[u][r]);
          }
          const double s = wsum(rest);
          cj = m - k > 1 ? s : 0.0;
          rj = cj;
        }
        if (lane == 0) cur[j] = cj, ref[j] = rj;
        if (cj > best_v) {  // warp-uniform; positions ascend within a warp: lowest on ties
          best_v = cj, best_p = j;
#pragma unroll
          for (int r = 0; r < kIdRows; ++r) cbuf[w * kIdMaxRows + lane + 32 * r] = cv[u][r];
        }
      }
    }
    if (lane == 0) cand_v[w] = best_v, cand_p[w] = best_p;
    __syncthreads();
  }
  const int steps = k;
  __syncthreads();

  // rank (id_rank, src/linalg.cpp:249-264) on |R_ii|, i < steps
  if (tid == 0) {
    int rank = 0;
    bool fallback = false;
    const double d0 = steps > 0 ? dg[0] : 0.0;
    if (steps > 0 && d0 != 0.0) {
      if (steps == cap && cap < full)
        for (int i = 0; i < steps; ++i) fallback = fallback || dg[i] <= 1e-14 * d0;
      int mm = steps;
      while (mm > 0 && dg[mm - 1] <= 1e-14 * d0) --mm;
      rank = mm;
      if (eps > 0.0)
        for (int i = 0; i < mm; ++i)
          if (dg[i] <= eps * d0) {
            rank = i + 1;
            break;
          }
      if (kmax > 0) rank = min(rank, kmax);
    }
    sh_rank = rank;
    sh_fb = fallback ? 1 : 0;
    ranks[t] = fallback ? -1 : rank;
  }
  __syncthreads();
  if (sh_fb) return;
  const int rank = sh_rank;
  for (int i = tid; i < rank; i += kIdWarps * 32) skel[static_cast<int64_t>(t) * kcap + i] = perm[i];

  // V(:, perm[j]) = e_j (j < rank), else R11^-1 R(0:rank, j); thread per column
  double2* V = out + tk.ooff;
  if (r11 >= rank) {  // R11 staged in shared memory, the solution in registers / local memory
    for (int q = tid; q < rank * rank; q += kIdWarps * 32) {
      const int i = q % rank, l = q / rank;
      R11[q] = i <= l ? B[static_cast<int64_t>(perm[l]) * m + i] : make_double2(0, 0);
    }
    __syncthreads();
    for (int j = tid; j < n; j += kIdWarps * 32) {
      const int pj = perm[j];
      auto at = [&](int i) -> double2& {
        return rowid ? V[static_cast<int64_t>(i) * n + pj] : V[static_cast<int64_t>(pj) * rank + i];
      };
      if (j < rank) {
        for (int i = 0; i < rank; ++i) at(i) = make_double2(i == j ? 1.0 : 0.0, 0.0);
        continue;
      }
      const double2* bj = B + static_cast<int64_t>(pj) * m;
      for (int i = rank - 1; i >= 0; --i) {
        double2 s = bj[i];
        for (int l = i + 1; l < rank; ++l) {
          const double2 q = cmul(R11[l * rank + i], at(l));
          s.x -= q.x;
          s.y -= q.y;
        }
        at(i) = cdiv(s, R11[i * rank + i]);
      }
    }
    return;
  }
  for (int j = tid; j < n; j += kIdWarps * 32) {
    const int pj = perm[j];
    auto at = [&](int i) -> double2& {
      return rowid ? V[static_cast<int64_t>(i) * n + pj] : V[static_cast<int64_t>(pj) * rank + i];
    };
    if (j < rank) {
      for (int i = 0; i < rank; ++i) at(i) = make_double2(i == j ? 1.0 : 0.0, 0.0);
      continue;
    }
    for (int i = rank - 1; i >= 0; --i) {
      double2 s = B[static_cast<int64_t>(pj) * m + i];
      for (int l = i + 1; l < rank; ++l) {
        const double2 q = cmul(B[static_cast<int64_t>(perm[l]) * m + i], at(l));
        s.x -= q.x;
        s.y -= q.y;
      }
      at(i) = cdiv(s, B[static_cast<int64_t>(perm[i]) * m + i]);
    }
  }
}

}  // namespace midbf::dev
