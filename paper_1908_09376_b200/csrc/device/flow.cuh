// k1_flow — the single-RHS MIDBF apply as ONE persistent dataflow launch.
//
// Work unit: a strip (<= 32 output rows of one stage, see plan.cu).  Strips
// are numbered stage by stage and dealt round-robin: warp w of NW owns
// strips w, w+NW, w+2NW, ... and processes them in increasing order.  A strip
// only waits on strips with smaller ids, and the smallest unfinished strip's
// owner has finished everything before it, so progress is guaranteed once all
// CTAs are co-resident (cooperative launch).  There are no atomics: a global
// claim counter serialises ~8K same-address atomics per apply at one L2 slice
// (measured ~118 us at cfg1), the static deal costs nothing.
//
// Per warp (FW warps per CTA, one CTA per SM):
//   producer (lane 0): copies the claimed strips' panels, chunk by chunk, into
//     the warp's ring of FS shared-memory slots with cp.async.bulk (TMA bulk
//     engine, mbarrier complete_tx); chunk = a column range of one panel,
//     derived arithmetically from the strip's cached metadata;
//   consumer (32 lanes, lane = output row): waits on the slot's mbarrier,
//     multiplies the panel columns with the staged x entries (fp64 FMA), and
//     after the last panel writes its row and publishes the strip's flag.
// Dependencies: a strip reads x[x0, x0+n) of each panel; the previous
// stage's strips producing that range are [dep0, dep1).  Lane 0 polls their
// flags (relaxed loads of the apply epoch) and issues one acquire fence; x
// is then gathered asynchronously with cp.async into a double-buffered
// window, one strip ahead when the next strip's producers are already done.
// Strip metadata (strip + up to kMaxSeg panels) is loaded once per claim into
// a per-warp shared-memory context ring, so the hot loop issues no
// dependent global loads besides x.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "plan.hpp"

namespace midbf::dev {

constexpr int kMaxSeg = 8;  // panels per strip supported by k1_flow
constexpr int kQN = 4;      // claimed-strip context ring per warp
constexpr int kXWin = 128;  // staged x entries per buffer (two per warp)

struct StageIO {
  const double2* x;
  double2* y;
  const int* xperm;
  const int* yperm;
};

struct StripCtx;
struct FlowParams {
  const StripCtx* ctxs;  // per strip: metadata record (strip id in s.seg0)
  const Strip* strips;
  const Seg* segs;
  const double2* arena;
  unsigned* flags;   // per strip: epoch of its last completion
  unsigned* epoch;   // per CTA: applies completed (all CTAs run every apply)
  int nstrips;
  int nwarps;
  // Timing experiments only (results invalid): 1 skip dependency waits,
  // 2 stream the payload only, 3 compute on resident slots without
  // streaming, 4 everything but the FMA loop.
  int nodeps;
  int pubmode;  // 0 publish after the x prefetch, 1 before it, 2 no fence (timing only)
  StageIO st[kMaxStages];
};

struct StripCtx {
  Strip s;
  Seg g[kMaxSeg];
};

namespace flowdev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Blocking wait.  The suspend-time hint lets the hardware park the thread
// until the phase completes instead of re-polling: with 8 waiting warps per
// SM, back-to-back polls otherwise contend with the TMA complete_tx updates.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cmac(double& ar, double& ai, double2 m, double2 x) {
  ar = fma(m.x, x.x, ar);
  ar = fma(-m.y, x.y, ar);
  ai = fma(m.x, x.y, ai);
  ai = fma(m.y, x.x, ai);
}

// Warp-wide dependency check: every producer flag of the strip is loaded in
// parallel (lane-strided per panel, no early exit, so all loads are in flight
// together) and voted; the caller issues one acquire fence on success.
__device__ __forceinline__ bool deps_done(const FlowParams& P, const StripCtx& c, unsigned e, int lane) {
  if (P.nodeps) return true;
  bool ok = true;
  for (int j = 0; j < c.s.nseg; ++j)
    for (int p = c.g[j].dep0 + lane; p < c.g[j].dep1; p += 32) ok &= ld_relaxed(P.flags + p) >= e;
  return __all_sync(0xffffffffu, ok);
}

// Gather a strip's x entries (sum of panel widths <= kXWin) with cp.async.
__device__ __forceinline__ void issue_x(const FlowParams& P, const StripCtx& c, double2* dst, int lane) {
  const StageIO io = P.st[c.s.stage];
  int cb = 0;
  for (int j = 0; j < c.s.nseg; ++j) {
    const int n = c.g[j].n, x0 = c.g[j].x0;
    for (int k = lane; k < n; k += 32) {
      int idx = x0 + k;
      if (io.xperm) idx = __ldg(io.xperm + idx);
      cp_async16(dst + cb + k, io.x + idx);
    }
    cb += n;
  }
  cp_async_commit();
}

__host__ __device__ constexpr int chunk_cols_for(int h, int slot_bytes) {
  int c = 64;
  while (c > 1 && h * c * 16 > slot_bytes) c >>= 1;
  return c;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

}  // namespace flowdev

// Shared-memory layout of one CTA: FW (producer, consumer) warp pairs.
template <int FW, int FS, int SLOT>
struct FlowCfg {
  static constexpr size_t kSlotArea = size_t(FW) * FS * SLOT;
  static constexpr size_t kXArea = size_t(FW) * 2 * kXWin * 16;
  static constexpr size_t kCtxArea = size_t(FW) * kQN * sizeof(StripCtx);
  // per pair: full[FS], empty[FS], ctx_full[kQN], ctx_empty[kQN]
  static constexpr size_t kBarArea = size_t(FW) * (2 * FS + 2 * kQN) * 8;
  static constexpr size_t kSmem = kSlotArea + kXArea + kCtxArea + kBarArea;
};

// Warps [0, FW) consume, warps [FW, 2*FW) produce: producer warp FW+c feeds
// consumer warp c.  The producer's lane 0 walks the consumer's strips (warp
// gw of NW owns strips gw, gw+NW, ...): it waits for a free context entry,
// writes the strip metadata, then for every chunk waits for a free slot and
// issues one cp.async.bulk into it.  It never waits on the consumer's
// dependency polls, x gathers or completion fences, so the slot ring stays
// full and HBM keeps streaming while the consumer is stalled.
template <int FW, int FS, int SLOT>
__global__ void __launch_bounds__(2 * FW * 32, 1) k1_flow(const __grid_constant__ FlowParams P) {
  using namespace flowdev;
  using Cfg = FlowCfg<FW, FS, SLOT>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool producer = warp >= FW;
  const int c = producer ? warp - FW : warp;  // pair index
  unsigned char* slots = smem + size_t(c) * FS * SLOT;
  double2* xb = reinterpret_cast<double2*>(smem + Cfg::kSlotArea) + c * 2 * kXWin;
  StripCtx* ctx = reinterpret_cast<StripCtx*>(smem + Cfg::kSlotArea + Cfg::kXArea) + c * kQN;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSlotArea + Cfg::kXArea + Cfg::kCtxArea) +
                   c * (2 * FS + 2 * kQN);
  uint64_t* full = bars;
  uint64_t* empty = bars + FS;
  uint64_t* cfull = bars + 2 * FS;
  uint64_t* cempty = bars + 2 * FS + kQN;
  if (producer && lane == 0) {
    for (int s = 0; s < 2 * FS + 2 * kQN; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const unsigned e = *reinterpret_cast<volatile unsigned*>(P.epoch + blockIdx.x) + 1u;
  const int gw = blockIdx.x * FW + c;

  if (producer) {
    if (lane == 0) {
      // Strips owned by this pair: gw, gw + NW, ...; context k == nmine is
      // the terminator.  Contexts are prefetched with bulk copies as soon as
      // their ring entry is released, so reading a strip's metadata never
      // waits on a plain global load.
      const int nmine = gw < P.nstrips ? (P.nstrips - 1 - gw) / P.nwarps + 1 : 0;
      int kf = 0;  // next context to request
      auto prefetch = [&](bool block) {
        while (kf <= nmine) {
          const int sc = kf % kQN;
          const unsigned par = ((kf / kQN) & 1) ^ 1;
          if (block) {
            mbar_wait(&cempty[sc], par);
            block = false;
          } else if (!mbar_test(&cempty[sc], par)) {
            break;
          }
          if (kf == nmine) {
            ctx[sc].s.y0 = -1;
            mbar_arrive(&cfull[sc]);
          } else {
            fence_proxy_async();
            mbar_expect_tx(&cfull[sc], sizeof(StripCtx));
            bulk_g2s(&ctx[sc], P.ctxs + gw + static_cast<int64_t>(kf) * P.nwarps, sizeof(StripCtx), &cfull[sc]);
          }
          ++kf;
        }
      };
      unsigned q = 0;
      for (int k = 0; k < nmine; ++k) {
        prefetch(kf <= k);
        const int sc = k % kQN;
        mbar_wait(&cfull[sc], (k / kQN) & 1);
        const StripCtx& C = ctx[sc];
        const int nseg = C.s.nseg, h = C.s.h;
        const int cpc = chunk_cols_for(h, SLOT);
        for (int j = 0; j < nseg; ++j) {
          const int n = C.g[j].n;
          const double2* src = P.arena + C.g[j].off;
          for (int col = 0; col < n; col += cpc, ++q) {
            const int ncol = min(cpc, n - col);
            const unsigned slot = q % FS;
            if (P.nodeps == 3 && q >= FS) continue;  // timing experiment: compute on resident data
            mbar_wait(&empty[slot], ((q / FS) & 1) ^ 1);
            fence_proxy_async();
            const unsigned bytes = static_cast<unsigned>(h * ncol * 16);
            mbar_expect_tx(&full[slot], bytes);
            bulk_g2s(slots + size_t(slot) * SLOT, src + static_cast<int64_t>(col) * h, bytes, &full[slot]);
            prefetch(false);
          }
        }
      }
      while (kf <= nmine) prefetch(true);
    }
    __syncwarp();
  } else {
    unsigned q = 0;
    int xsel = 0;
    bool have_x = false;
    int pending = -1;  // finished strip whose flag is not yet published
    // Release: the strip's row stores (all lanes, ordered by the warp
    // barrier) before its flag.  Deferred by one strip so the fence finds the
    // stores already drained instead of waiting for them.
    auto publish = [&]() {
      if (pending >= 0) {
        if (lane == 0) {
          if (P.pubmode != 2) fence_acq_rel();
          st_relaxed(P.flags + pending, e);
        }
        pending = -1;
      }
    };
    for (int k = 0;; ++k) {
      const int sc = k % kQN;
      mbar_wait(&cfull[sc], (k / kQN) & 1);
      const StripCtx& C = ctx[sc];
      if (C.s.y0 < 0) break;
      if (P.nodeps == 2) {  // timing experiment: stream the payload only
        const int cpc = chunk_cols_for(C.s.h, SLOT);
        for (int j = 0; j < C.s.nseg; ++j)
          for (int col0 = 0; col0 < C.g[j].n; col0 += cpc, ++q) {
            mbar_wait(&full[q % FS], (q / FS) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[q % FS]);
          }
        if (lane == 0) mbar_arrive(&cempty[sc]);
        continue;
      }
      const int t = C.s.seg0;
      const int h = C.s.h, nseg = C.s.nseg, y0 = C.s.y0;
      const StageIO io = P.st[C.s.stage];
      const bool fast = C.s.xcols <= kXWin;
      double2* xcur = xb + xsel * kXWin;
      if (P.pubmode == 1) publish();
      if (fast && !have_x) {
        publish();  // before any blocking dependency wait (deadlock freedom)
        while (!deps_done(P, C, e, lane)) {
        }
        if (lane == 0) fence_acq_rel();
        __syncwarp();
        issue_x(P, C, xcur, lane);
      }
      // x of the next strip, if its metadata is in and its producers are done
      bool pref = false;
      {
        const int sn = (k + 1) % kQN;
        if (mbar_test(&cfull[sn], ((k + 1) / kQN) & 1)) {
          const StripCtx& Cn = ctx[sn];
          if (Cn.s.y0 >= 0 && Cn.s.xcols <= kXWin && deps_done(P, Cn, e, lane)) {
            if (lane == 0) fence_acq_rel();
            __syncwarp();
            issue_x(P, Cn, xb + (xsel ^ 1) * kXWin, lane);
            pref = true;
          }
        }
      }
      publish();
      if (fast) {
        if (pref)
          cp_async_wait<1>();
        else
          cp_async_wait<0>();
        __syncwarp();
      }
      const bool live = lane < h;
      const int cpc = chunk_cols_for(h, SLOT);
      double ar0 = 0, ai0 = 0, ar1 = 0, ai1 = 0;
      int cb = 0;
      for (int j = 0; j < nseg; ++j) {
        const int n = C.g[j].n;
        int win = -1;
        if (!fast) {
          if (lane == 0) {
            for (int p = C.g[j].dep0; p < C.g[j].dep1 && !P.nodeps; ++p)
              while (ld_relaxed(P.flags + p) < e) {
              }
            fence_acq_rel();
          }
          __syncwarp();
        }
        for (int col0 = 0; col0 < n; col0 += cpc, ++q) {
          const int ncol = min(cpc, n - col0);
          const double2* xv;
          if (fast) {
            xv = xcur + cb + col0;
          } else {  // wide strip: synchronous windows of kXWin columns
            const int w0 = col0 / kXWin;
            if (w0 != win) {
              __syncwarp();
              const int cnt = min(kXWin, n - w0 * kXWin);
              for (int kk = lane; kk < cnt; kk += 32) {
                int idx = C.g[j].x0 + w0 * kXWin + kk;
                if (io.xperm) idx = __ldg(io.xperm + idx);
                xcur[kk] = __ldcg(io.x + idx);
              }
              __syncwarp();
              win = w0;
            }
            xv = xcur + (col0 - w0 * kXWin);
          }
          const unsigned slot = q % FS;
          if (P.nodeps != 3 || q < FS) mbar_wait(&full[slot], (q / FS) & 1);
          const double2* M = reinterpret_cast<const double2*>(slots + size_t(slot) * SLOT);
          if (live && P.nodeps != 4) {
            int cc = 0;
            for (; cc + 4 <= ncol; cc += 4) {
              const double2 m0 = M[(cc + 0) * h + lane], m1 = M[(cc + 1) * h + lane];
              const double2 m2 = M[(cc + 2) * h + lane], m3 = M[(cc + 3) * h + lane];
              cmac(ar0, ai0, m0, xv[cc + 0]);
              cmac(ar1, ai1, m1, xv[cc + 1]);
              cmac(ar0, ai0, m2, xv[cc + 2]);
              cmac(ar1, ai1, m3, xv[cc + 3]);
            }
            for (; cc < ncol; ++cc) cmac(ar0, ai0, M[cc * h + lane], xv[cc]);
          }
          __syncwarp();
          if (lane == 0 && P.nodeps != 3) mbar_arrive(&empty[slot]);  // slot back to the producer
        }
        cb += n;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty[sc]);  // context no longer read
      if (live) {
        int idx = y0 + lane;
        if (io.yperm) idx = io.yperm[idx];
        io.y[idx] = make_double2(ar0 + ar1, ai0 + ai1);
      }
      __syncwarp();
      pending = t;  // flag published at the next strip, once the stores drained
      if (pref) xsel ^= 1;
      have_x = pref;
    }
    publish();
    cp_async_wait<0>();
  }
  __syncthreads();
  if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned*>(P.epoch + blockIdx.x) = e;
}

}  // namespace midbf::dev
