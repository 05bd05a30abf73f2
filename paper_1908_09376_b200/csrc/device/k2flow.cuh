// K2-flow — the multi-RHS MIDBF apply as ONE persistent dataflow launch per
// 64-RHS slice, on the FP64 tensor cores (DMMA), sm_100a.
//
// Same arithmetic as k2_stage (k2.cuh) — per strip, Y(rows, 64 RHS) = sum
// over its panels P (h x n) * X(x0 .. x0+n, :), the panels walked as one
// concatenated K dimension in 16-column chunks — with every stage in one
// cooperative launch, which removes the per-stage launch gaps and the
// per-stage wave tails (cfg4: 1024 strips per stage on 296 CTA slots is
// 3.46 waves).  Reference: apply_factor's GEMM path for x.cols() > 1
// (src/butterfly.cpp:633-637 with bf::apply(F, MatXc), :779).
//
// CTA = 8 consumer warps + 1 producer warp + 1 publisher warp, 2 CTAs per SM.
//   * Producer: walks this CTA's strips (global strip list, stage-major,
//     dealt round-robin over the grid), and streams each strip's chunks
//     (panel: 16 columns x h rows; X: 16 rows x 64 RHS) into a 4-slot shared
//     ring with TMA bulk copies (cp.async.bulk, complete_tx on the slot's
//     `full` barrier), into the padded layouts of k2_stage: intermediate
//     stage buffers are row-major with the slot's padded row stride (66), so
//     a run of consecutive input rows is ONE copy; panel columns are one copy
//     per run when the strip height h == 2, 6 (mod 8) (stride h is then
//     conflict-free for the A fragments), else one copy per column (stride 34).
//     Stage 0 gathers its input rows (user operand, column-major) through
//     the column permutation with cp.async (cp.async.mbarrier.arrive.noinc).  Before the
//     first X chunk of a strip it acquires the completion counters of the
//     previous-stage strips that produce its input rows (Seg::dep0/dep1).
//   * Consumers: LDS + DMMA only (8 rows x 32 RHS per warp, as in k2_stage);
//     release the slot on its `empty` barrier; at the end of a strip store
//     the 32 x 64 tile and arrive on the strip's `done` barrier (8-deep ring).
//   * A publisher warp waits on the `done` ring and publishes each completed
//     strip with one gpu-scope release add on its counter (a warp with no
//     loads in flight, so the release fence is cheap); the producer never
//     runs more than 8 strips ahead of the publications.
//   * Per-CTA apply epochs (all CTAs run every launch): a strip of launch e
//     is complete when its counter reaches e.
// Deadlock freedom: CTAs are co-resident (cooperative launch) and each
// walks its strips in increasing global order; the smallest unpublished
// strip has all its inputs published, its CTA's producer has issued it or is
// at it, and publication waits on nothing but this CTA's consumers.
// Stages overlap, so every stage but the last writes its own buffer.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "flow.cuh"
#include "k2.cuh"
#include "plan.hpp"

namespace midbf::dev {

constexpr int kK2FConsumers = 8;                      // consumer warps
constexpr int kK2FThreads = (kK2FConsumers + 3) * 32;  // + panel / input producer warps and a publisher warp
constexpr int kK2FSlots = 4;                           // ring depth
constexpr int kK2FDone = 8;                            // strip-completion barrier ring

// Tile width W = 16 NCB right-hand sides (2 warp halves x NCB column blocks of
// 8); X slot / stage-buffer row stride W + 2 (== 2 mod 8 in 16-byte units:
// conflict-free B fragments).  The host picks the narrowest W covering a slice.
// Narrower tiles have smaller X slots, so the same ~100 KB holds a deeper
// ring (8 / 6 / 4 slots at W = 16 / 32 / 64).
template <int NCB>
struct K2FCfg {
  static constexpr int W = 16 * NCB;
  static constexpr int XS = W + 2;
  static constexpr int XBUF = kK2Kc * XS;
  static constexpr int SLOTS = NCB == 1 ? 8 : (NCB == 2 ? 6 : kK2FSlots);
  static constexpr size_t kSmem = size_t(SLOTS) * (kK2PBuf + XBUF) * 16 + SLOTS * (16 + 16) + kK2FDone * 8;
};

struct K2FStage {
  const double2* x;  // input (stage 0: user operand, gathered through xperm)
  double2* y;        // output (last stage: user operand, scattered through yperm)
  int64_t xld, yld;  // user operands: column-major ld; stage buffers: row-major, row stride W + 2
  const int* xperm;
  const int* yperm;
};

struct K2FParams {
  const Strip* strips;  // all stages, application order; identity-compressed
                        // strips: pad_[0] = base in xmap, pad_[1] = base in addx
  const Seg* segs;
  const int* xmap;      // compressed strips: stage-local input row of each kept column
  const int* addx;      // compressed strips: per output row, the input row added to it (-1: none)
  const double2* arena;
  unsigned* done;   // per strip: completions over all launches
  unsigned* epoch;  // per CTA: launches completed
  int nstrips;
  int nstages;
  int ncv;     // valid RHS of this slice (<= W)
  // timing experiments only (flag bits 14-15), results invalid: 1 skip the
  // dependency waits, 2 stream only (no math), 3 math only (no loads)
  int mode;
  int64_t arena_len;  // complex entries of the arena (checked builds)
  int l2_first;       // panels streamed with an L2 evict_first policy (plan.hpp kFlagK2L2Normal)
  K2FStage st[kMaxStages];
};

namespace k2fdev {

__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(flowdev::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace k2fdev

// G3: complex products with three real DMMAs (Gauss: P1 = a.re c.re,
// P2 = a.im c.im, P3 = (a.re + a.im)(c.re + c.im); re = P1 - P2,
// im = P3 - P1 - P2) instead of four; the kernel is DMMA-bound.
template <int NCB, bool G3 = true, bool RB2 = true>
__global__ void __launch_bounds__(kK2FThreads, 2) k2_flow(const __grid_constant__ K2FParams P) {
  using Cfg = K2FCfg<NCB>;
  constexpr int kW = Cfg::W, kXs = Cfg::XS, kXBuf = Cfg::XBUF, kSlots = Cfg::SLOTS;
  using namespace k2dev;
  using namespace k2fdev;
  using flowdev::mbar_arrive;
  using flowdev::mbar_init;
  using flowdev::mbar_wait;
  extern __shared__ __align__(16) double2 k2smem[];
  double2* const Pb = k2smem;                        // kSlots panel buffers
  double2* const Xb = k2smem + kSlots * kK2PBuf;  // kSlots X buffers
  uint64_t* const full = reinterpret_cast<uint64_t*>(Xb + kSlots * kXBuf);
  uint64_t* const empty = full + kSlots;
  int4* const meta = reinterpret_cast<int4*>(empty + kSlots);  // per slot: {y0, h, stage | A stride, K}
  uint64_t* const done = reinterpret_cast<uint64_t*>(meta + kSlots);
  __shared__ unsigned s_epoch;
  __shared__ int s_pub;  // strips of this CTA published so far
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&full[i], 34);  // panel-producer lane 0 + input-producer lane 0 + its 32 cp.async arrivals
      mbar_init(&empty[i], kK2FConsumers);
    }
    for (int i = 0; i < kK2FDone; ++i) mbar_init(&done[i], kK2FConsumers);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_epoch = P.epoch[blockIdx.x] + 1;
    s_pub = 0;
  }
  __syncthreads();
  const unsigned target = s_epoch;

  if (w == kK2FConsumers || w == kK2FConsumers + 1) {
    // ---------------- producers: panels (no waits) | inputs (dependencies) -------
    const bool xrole = w == kK2FConsumers + 1;
    const uint64_t pol = P.l2_first ? flowdev::l2_evict_first_policy() : 0ull;
    int gc = 0;  // chunks issued
    int started = 0;  // this CTA's strips started
    for (int item = blockIdx.x; item < P.nstrips; item += gridDim.x) {
      while (started - *reinterpret_cast<volatile int*>(&s_pub) >= kK2FDone) __nanosleep(64);  // done-ring slot free
      ++started;
      const Strip st = P.strips[item];
      const K2FStage io = P.st[st.stage];
      int64_t s_off = 0;
      int s_x0 = 0, s_n = 0, s_d0 = 0, s_d1 = 0;
      if (lane < st.nseg) {
        const Seg sg = P.segs[st.seg0 + lane];
        s_off = sg.off, s_x0 = sg.x0, s_n = sg.n, s_d0 = sg.dep0, s_d1 = sg.dep1;
      }
      int s_k0 = s_n;  // exclusive prefix of the panel widths
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, s_k0, o);
        if (lane >= o) s_k0 += v;
      }
      s_k0 -= s_n;
      const int K = st.xcols, h = st.h;
      const int xmb = st.pad_[0];  // >= 0: kept columns' input rows in P.xmap (identity-compressed strip)
      const int nq = K > 0 ? (K + kK2Kc - 1) / kK2Kc : 1;
      bool deps = st.stage == 0 || P.mode != 0;
      for (int q = 0; q < nq; ++q, ++gc) {
        const int slot = gc % kSlots, use = gc / kSlots;
        if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
        // lane resolves K column c = lane & 15 of the chunk
        const int c = lane & (kK2Kc - 1);
        const int kg = q * kK2Kc + c;
        int sidx = 0;
        for (int l = 1; l < st.nseg; ++l) sidx += __shfl_sync(0xffffffffu, s_k0, l) <= kg;
        const int cc = kg - __shfl_sync(0xffffffffu, s_k0, sidx);
        const bool ok = kg < K;
        const int kval = min(kK2Kc, K - q * kK2Kc);  // valid columns (<= 0: none)
        const int64_t psrc = __shfl_sync(0xffffffffu, s_off, sidx) + static_cast<int64_t>(cc) * h;
        int xi = __shfl_sync(0xffffffffu, s_x0, sidx) + cc;
        if (xmb >= 0 && ok) xi = __ldg(P.xmap + xmb + kg);
        const bool gather = io.xperm != nullptr;
        const bool load = P.mode != 3 && kval > 0;
        // panel column stride in the slot: h itself when h == 2, 6 (mod 8)
        // (A fragment loads conflict-free, one copy per column run), else 34
        const bool prun = (h & 3) == 2;
        const int pst = prun ? h : kK2Ps;
        // runs of columns on one panel (consecutive panel columns and input rows)
        const int prev = __shfl_up_sync(0xffffffffu, sidx, 1);
        const int prevx = __shfl_up_sync(0xffffffffu, xi, 1);
        unsigned runs = __ballot_sync(0xffffffffu, ok && lane < kK2Kc && (c == 0 || prev != sidx));
        // input rows: runs also break where the kept columns skip input rows
        unsigned xruns = __ballot_sync(0xffffffffu, ok && lane < kK2Kc && (c == 0 || prev != sidx || prevx + 1 != xi));
        double2* pd = Pb + slot * kK2PBuf;
        double2* xd = Xb + slot * kXBuf;
        if (!xrole) {  // panels: plan constants, never wait on other strips
          if (lane == 0) {
            meta[slot] = make_int4(st.y0, h, st.stage | (pst << 8), K);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                             flowdev::smem_u32(&full[slot])),
                         "r"(load ? kval * 16u * h : 0u)
                         : "memory");
          }
          __syncwarp();
          if (load) {
            if (!prun) {
              MIDBF_DCHECK(!(ok && lane < kK2Kc) || (psrc >= 0 && psrc + h <= P.arena_len), "k2_flow panel column");
              if (ok && lane < kK2Kc) {
                if (P.l2_first)
                  flowdev::bulk_g2s_hint(pd + c * kK2Ps, P.arena + psrc, h * 16u, &full[slot], pol);
                else
                  flowdev::bulk_g2s(pd + c * kK2Ps, P.arena + psrc, h * 16u, &full[slot]);
              }
            } else {
              unsigned r = runs;
              while (r) {
                const int r0 = __ffs(r) - 1;
                r &= r - 1;
                const int r1 = r ? __ffs(r) - 1 : kval;
                const int64_t src = __shfl_sync(0xffffffffu, psrc, r0);
                MIDBF_DCHECK(lane != 0 || (src >= 0 && src + int64_t(r1 - r0) * h <= P.arena_len), "k2_flow panel run");
                if (lane == 0) {
                  if (P.l2_first)
                    flowdev::bulk_g2s_hint(pd + r0 * h, P.arena + src, (r1 - r0) * h * 16u, &full[slot], pol);
                  else
                    flowdev::bulk_g2s(pd + r0 * h, P.arena + src, (r1 - r0) * h * 16u, &full[slot]);
                }
              }
            }
          }
          continue;
        }
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(flowdev::smem_u32(&full[slot])),
                       "r"(load && !gather ? kval * 16u * kXs : 0u)
                       : "memory");
        __syncwarp();
        if (!deps) {
          while (!deps) {  // previous-stage producers of this strip's input rows
            bool ready = true;
            for (int l = 0; l < st.nseg; ++l) {
              const int d0 = __shfl_sync(0xffffffffu, s_d0, l), d1 = __shfl_sync(0xffffffffu, s_d1, l);
              for (int s = d0 + lane; s < d1 && ready; s += 32) ready = ld_acquire(P.done + s) >= target;
            }
            deps = __all_sync(0xffffffffu, ready);
            if (!deps) __nanosleep(64);
          }
          // The input rows were written by other CTAs' generic stores and
          // published by their release adds; every lane's acquire is ordered
          // before lane 0's copies by the warp barrier, and the proxy fence
          // orders them before the TMA engine's (async proxy) reads.
          __syncwarp();
          fence_proxy_async_global();
        }
        if (load) {
          if (gather) {  // stage 0: lane & 15 = k, RHS (lane >> 4) + 2 i
            if (ok) {
              const double2* xs = io.x + __ldg(io.xperm + xi);
              double2* xk = xd + c * kXs;
#pragma unroll 4
              for (int rhs = lane >> 4; rhs < P.ncv; rhs += 2) cp_async16(xk + rhs, xs + rhs * io.xld);
            }
          } else {  // stage buffers: rows padded to the slot stride, one copy per run
            while (xruns) {
              const int r0 = __ffs(xruns) - 1;
              xruns &= xruns - 1;
              const int r1 = xruns ? __ffs(xruns) - 1 : kval;
              const int64_t src = static_cast<int64_t>(__shfl_sync(0xffffffffu, xi, r0)) * kXs;
              if (lane == 0) flowdev::bulk_g2s(xd + r0 * kXs, io.x + src, (r1 - r0) * kXs * 16u, &full[slot]);
            }
          }
        }
        cp_async_arrive_noinc(&full[slot]);
      }
    }
  } else if (w == kK2FConsumers + 2) {
    // ------------------------------ publisher ------------------------------
    int n = 0;
    for (int item = blockIdx.x; item < P.nstrips; item += gridDim.x, ++n) {
      mbar_wait(&done[n % kK2FDone], (n / kK2FDone) & 1);
      if (lane == 0) {
        red_release_add(P.done + item, 1u);
        *reinterpret_cast<volatile int*>(&s_pub) = n + 1;
      }
    }
  } else {
    // ------------------------------ consumers ------------------------------
    // Warp tile: RBW row blocks of 8 rows x CBW column blocks of 8 RHS.
    // RBW = 2 on the 64-wide tiles (16 rows x 16 RHS: per K step 2 A and 2 B
    // fragment loads for 12 DMMAs), else 1 (8 rows x W/2 RHS).
    constexpr int RBW = (NCB == 4 && RB2) ? 2 : 1;
    constexpr int CBW = NCB / RBW;
    const int g = lane >> 2, t = lane & 3;
    const int rb0 = RBW == 2 ? 2 * (w & 1) : (w & 3);  // first row block
    const int ch = RBW == 2 ? (w >> 1) : (w >> 2);     // RHS group of CBW * 8
    int gc = 0, nit = 0;
    for (int item = blockIdx.x; item < P.nstrips; item += gridDim.x) {
      constexpr int NA = G3 ? 3 : 2;  // accumulators per D fragment: re, im (or P1, P2, P3)
      double acc[RBW][CBW][NA][2];
#pragma unroll
      for (int rr = 0; rr < RBW; ++rr)
#pragma unroll
        for (int cb = 0; cb < CBW; ++cb)
#pragma unroll
          for (int r = 0; r < NA; ++r) acc[rr][cb][r][0] = acc[rr][cb][r][1] = 0.0;
      int4 m = make_int4(0, 0, 0, 0);
      int nq = 1;
      for (int q = 0; q < nq; ++q, ++gc) {
        const int slot = gc % kSlots;
        mbar_wait(&full[slot], (gc / kSlots) & 1);
        if (q == 0) {
          m = meta[slot];
          nq = m.w > 0 ? (m.w + kK2Kc - 1) / kK2Kc : 1;
        }
        const int krem = min(kK2Kc, m.w - q * kK2Kc);
        const int kfull = krem & ~3;
        const int pst = m.z >> 8;
        const double2* Ps = Pb + slot * kK2PBuf + 8 * rb0 + g;
        const double2* Xs = Xb + slot * kXBuf + t * kXs + ch * (CBW * 8) + g;
        auto step = [&](int kk, bool live) {
          double2 a[RBW], bv[CBW];
#pragma unroll
          for (int rr = 0; rr < RBW; ++rr) a[rr] = Ps[(kk + t) * pst + 8 * rr];
#pragma unroll
          for (int cb = 0; cb < CBW; ++cb) bv[cb] = Xs[kk * kXs + cb * 8];
          if (!live) {  // K tail: stale slot contents must not reach the sums
#pragma unroll
            for (int rr = 0; rr < RBW; ++rr) a[rr] = make_double2(0, 0);
#pragma unroll
            for (int cb = 0; cb < CBW; ++cb) bv[cb] = make_double2(0, 0);
          }
#pragma unroll
          for (int rr = 0; rr < RBW; ++rr) {
            if (G3) {
              const double sa = a[rr].x + a[rr].y;
#pragma unroll
              for (int cb = 0; cb < CBW; ++cb) {
                dmma(acc[rr][cb][0][0], acc[rr][cb][0][1], a[rr].x, bv[cb].x);
                dmma(acc[rr][cb][1][0], acc[rr][cb][1][1], a[rr].y, bv[cb].y);
                dmma(acc[rr][cb][NA - 1][0], acc[rr][cb][NA - 1][1], sa, bv[cb].x + bv[cb].y);
              }
            } else {
              const double naim = -a[rr].y;
#pragma unroll
              for (int cb = 0; cb < CBW; ++cb) {
                dmma(acc[rr][cb][0][0], acc[rr][cb][0][1], a[rr].x, bv[cb].x);
                dmma(acc[rr][cb][1][0], acc[rr][cb][1][1], a[rr].x, bv[cb].y);
              }
#pragma unroll
              for (int cb = 0; cb < CBW; ++cb) {
                dmma(acc[rr][cb][0][0], acc[rr][cb][0][1], naim, bv[cb].y);
                dmma(acc[rr][cb][1][0], acc[rr][cb][1][1], a[rr].y, bv[cb].x);
              }
            }
          }
        };
        if (P.mode == 2) {
        } else if (kfull == kK2Kc) {
#pragma unroll
          for (int kk = 0; kk < kK2Kc; kk += 4) step(kk, true);
        } else {
          for (int kk = 0; kk < kfull; kk += 4) step(kk, true);
          if (kfull < krem) step(kfull, t < krem - kfull);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
      if (G3) {  // (P1, P2, P3) -> (re, im) in acc[..][0], acc[..][1]
#pragma unroll
        for (int rr = 0; rr < RBW; ++rr)
#pragma unroll
          for (int cb = 0; cb < CBW; ++cb)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const double p1 = acc[rr][cb][0][i], p2 = acc[rr][cb][1][i];
              acc[rr][cb][0][i] = p1 - p2;
              acc[rr][cb][1][i] = acc[rr][cb][NA - 1][i] - p1 - p2;
            }
      }
      // D fragment: row 8*(rb0 + rr) + g, RHS (CBW*8)*ch + cb*8 + 2t + {0,1}
      const int stage = m.z & 255;
      const K2FStage io = P.st[stage];
      const bool last = stage + 1 == P.nstages;
      const int ab = P.strips[item].pad_[1];
#pragma unroll
      for (int rr = 0; rr < RBW; ++rr) {
        const int row = 8 * (rb0 + rr) + g;
        if (ab >= 0 && row < m.y) {  // identity columns: Y(row, :) += X(input row, :)
          const int xa = __ldg(P.addx + ab + row);
          if (xa >= 0) {
            const K2FStage xin = P.st[stage];
            const double2* xr = xin.xperm ? xin.x + __ldg(xin.xperm + xa) : xin.x + static_cast<int64_t>(xa) * xin.xld;
            const int64_t rs = xin.xperm ? xin.xld : 1;  // user operand: column-major; stage buffers: row-major
#pragma unroll
            for (int cb = 0; cb < CBW; ++cb)
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int rhs = (CBW * 8) * ch + cb * 8 + 2 * t + i;
                if (rhs < P.ncv) {
                  const double2 v = xin.xperm ? __ldg(xr + rhs * rs) : flowdev::ld_cg(xr + rhs);
                  acc[rr][cb][0][i] += v.x;
                  acc[rr][cb][1][i] += v.y;
                }
              }
          }
        }
        if (row < m.y) {
          int idx = m.x + row;
          if (io.yperm) idx = __ldg(io.yperm + idx);
#pragma unroll
          for (int cb = 0; cb < CBW; ++cb)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int rhs = (CBW * 8) * ch + cb * 8 + 2 * t + i;
              if (rhs < P.ncv) io.y[last ? rhs * io.yld + idx : idx * io.yld + rhs] =
                  make_double2(acc[rr][cb][0][i], acc[rr][cb][1][i]);
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[nit % kK2FDone]);
      ++nit;
    }
  }
  __syncthreads();
  if (tid == 0) P.epoch[blockIdx.x] = s_epoch;
}

}  // namespace midbf::dev
