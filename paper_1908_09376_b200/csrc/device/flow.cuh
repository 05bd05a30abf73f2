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
//     after the last panel writes its row (the row value is the ready signal).
// Dependencies: a strip reads x[x0, x0+n) of each panel from the previous
// stage's output buffer (stage 0 of the 4-pair layout: from the user's f
// through in_perm, FlowParams::direct0), which is armed with a sentinel bit
// pattern before the apply; an x stager polls exactly the entries a strip
// needs until none is a sentinel (the data is its own ready signal: no flags, no fences) and stages
// them in shared memory up to two strips ahead of the consumer (x_full /
// x_empty mbarriers).  The stager is a dedicated warp per pair when the
// register file allows (<= 4 pairs), else the producer warp's lanes 1..31.
// Strip metadata (strip + up to kMaxSeg panels) is loaded once per claim into
// a per-warp shared-memory context ring, so the hot loop issues no
// dependent global loads besides x.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "plan.hpp"

namespace midbf::dev {

constexpr int kMaxSeg = 8;  // panels per strip supported by k1_flow
constexpr int kQN = 4;      // claimed-strip context ring per warp
constexpr int kXWin = 128;  // staged x entries per buffer (two per warp)
// PROF builds: per-warp phase timers in the first kProfStripBase entries of
// FlowParams::prof, then 3 timestamps per strip (up to kProfStrips strips)
constexpr int64_t kProfStripBase = int64_t(1024) * 64 * 16;
constexpr int kProfStrips = 1 << 18;

struct StageIO {
  const double2* x;  // parity-0 address for stage buffers
  double2* y;
  const int* xperm;
  const int* yperm;
  int x_par, y_par;  // 1: stage buffer, add FlowParams::par_elems on odd applies
};

struct StripCtx;
struct FlowParams {
  const StripCtx* ctxs;  // per strip: metadata record (strip id in s.seg0)
  const Strip* strips;
  const Seg* segs;
  const double2* arena;
  unsigned* epoch;   // per CTA: applies completed (all CTAs run every apply)
  double2* stagebuf;  // both parity sets of intermediate stage buffers
  int64_t par_elems;  // complex entries per parity set
  const double2* in;  // user input (read once by the permutation prologue)
  // Pipelined host-operand applies (Plan::apply_async): the input is copied
  // on another stream, followed by a one-byte flag write; the prologue waits
  // for flag == in_seq instead of the stream waiting on an event, so the
  // chained launch is not broken by a cross-stream dependency.  Null: none.
  const unsigned char* in_flag;
  unsigned in_seq;
  const int* in_perm;
  int64_t in_len;
  int nstrips;
  int nwarps;
  // Timing experiments only (results invalid): 2 stream the payload only,
  // 3 compute on resident slots without streaming, 4 everything but the
  // FMA loop.
  int nodeps;
  long long* prof;  // phase timers of the PROF instantiation
  const int* wmap;  // wide compressed strips: kept columns, then add columns (StripCtx::wbase)
  int pdl;          // launched as a programmatic dependent of the previous apply (see k1_flow)
  // per-stage inputs / outputs, a device table built with the plan (the
  // launch parameters stay small: they are copied on every launch); the last
  // stage has y == nullptr and writes `out`
  const StageIO* st;
  double2* out;
  int64_t arena_len;  // complex entries of the arena (checked builds)
  int64_t out_len;    // entries of `out` (checked builds)
  int direct0;        // stage 0 gathers the user input through in_perm itself (no stage -1 prologue)
  int nstages;        // entries of st (copied into shared memory at launch)
  int l2_first;       // panels streamed with an L2 evict_first policy (flag bit 27)
};

// A panel as k1_flow streams it.
struct FlowSeg {
  int64_t off;     // complex offset in the arena (dense part, or compressed part)
  int32_t x0;      // first input entry of the block's column range
  int32_t n;       // columns streamed (the kept columns of a compressed panel)
  uint32_t urows;  // bit r: row r is a unit row of this panel (no panel row)
  uint32_t adds;   // bit r: row r adds one staged x entry for this panel
  int32_t hc;      // rows streamed: the strip's rows minus this panel's unit rows
  int32_t aoff;    // this panel's first entry in StripCtx::addpos
};

// Identity compression (plan.cu, build_flow_records).  The factors' ID blocks
// hold exact identity parts (src/linalg.cpp:278-290 writes MatXc::Identity
// into every column ID; a row ID is its transpose), so within one panel
//   a unit row    (its only nonzero is an exact 1 at column c) contributes
//                 y_r += x[c] and is not streamed;
//   a unit column (over the remaining rows, a single exact 1 at row r)
//                 contributes y_r += x[c] and is not streamed;
//   a zero column (over the remaining rows) is dropped.
// A compressed strip streams hc x n' per panel; its staged x window holds the
// kept columns (cmap) followed by `next` extra entries (xext) that only the
// adds read; each add is a staged position (addpos), summed after the panels.
struct StripCtx {
  Strip s;              // s.h rows, s.xcols staged x entries, s.seg0 = strip id
  FlowSeg g[kMaxSeg];
  int32_t nkept;        // staged kept columns (sum of g[j].n)
  int32_t next;         // extra staged entries after them
  int32_t mapped;       // 1: compressed record (cmap / xext / adds valid); 2: wide compressed
                        //    strip (kept / add columns in FlowParams::wmap at wbase)
  int32_t wbase;
  uint8_t cmap[kXWin];  // kept column (within its block) of staged entry kk
  uint16_t xext[32];    // extra staged entry e: segment << 8 | column
  uint8_t addpos[64];   // per panel, per add row (row order): staged position
};
static_assert(sizeof(StripCtx) % 16 == 0, "StripCtx is copied with cp.async.bulk");

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
// Blocking wait: try_wait suspends the thread for an implementation-defined
// time per attempt.  An explicit suspend-time hint of 1e6 ns (round 1) was
// measured slightly slower than the default (second session, same-box A/B:
// cfg1 50.8 -> 50.5 us, cfg2 224.3 -> 223.2 us, cfg4 unchanged);
// -DMIDBF_MBAR_HINT=<ns> restores a hint.
#ifndef MIDBF_MBAR_HINT
#define MIDBF_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
#if MIDBF_MBAR_HINT == 0
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(MIDBF_MBAR_HINT)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// The same copy with an L2 eviction-priority policy (createpolicy).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cmac(double& ar, double& ai, double2 m, double2 x) {
  ar = fma(m.x, x.x, ar);
  ar = fma(-m.y, x.y, ar);
  ai = fma(m.x, x.y, ai);
  ai = fma(m.y, x.x, ai);
}

// ---- data-as-signal dependencies -------------------------------------------
// Intermediate stage buffers are armed with an all-ones bit pattern before an
// apply uses them; a consumer polls the entries it reads (L2, .cg) until none
// carries the sentinel.  An entry is written exactly once per apply by the
// warp owning its strip, and 8-byte aligned stores are single-copy atomic,
// so "re and im both differ from the sentinel" means the final value is
// visible: no flags, no fences on the critical path.
constexpr int kXPerLane = kXWin / 32;
__device__ __forceinline__ bool is_sentinel(const double2& v) {
  return __double_as_longlong(v.x) == -1ll || __double_as_longlong(v.y) == -1ll;
}
__device__ __forceinline__ double unsentinel(double v) {
  return __double_as_longlong(v) == -1ll ? __longlong_as_double(0x7ff8000000000000ll) : v;
}
// Spin on one entry until it is not the sentinel (loop in PTX, strong loads).
__device__ __forceinline__ double2 poll_cg(const double2* p) {
  unsigned long long a, b;
  asm volatile(
      "{\n .reg .pred s0, s1;\n"
      "POLL_CG_AGAIN:\n"
      " ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];\n"
      " setp.eq.s64 s0, %0, -1;\n"
      " setp.eq.or.s64 s1, %1, -1, s0;\n"
      " @s1 bra POLL_CG_AGAIN;\n}"
      : "=l"(a), "=l"(b)
      : "l"(p)
      : "memory");
  return make_double2(__longlong_as_double(static_cast<long long>(a)), __longlong_as_double(static_cast<long long>(b)));
}
// The matching strong store: every value another CTA polls is written with a
// relaxed GPU-scope store, so each (store, poll) pair is a pair of morally
// strong accesses and the protocol has no data race under the PTX memory
// model (a weak st.global raced by ld.relaxed would be one; each 8-byte half
// is single-copy atomic, which is all the sentinel test needs).
__device__ __forceinline__ void st_signal(double2* p, double2 v) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// Wait for the input-ready flag of a pipelined host-operand apply (see
// FlowParams::in_flag); bounded: a flag that never arrives traps instead of
// hanging the GPU.
__device__ __forceinline__ void wait_in_flag(const unsigned char* f, unsigned seq) {
  if (!f) return;
  for (long long it = 0;; ++it) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u8 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if ((v & 0xffu) == (seq & 0xffu)) return;
    if (it > (1ll << 26)) __trap();
    __nanosleep(128);
  }
}
__device__ __forceinline__ double2 ld_cg(const double2* p) {
  double2 v;
  // A strong (relaxed, GPU-scope) load: the polls re-read it until another
  // CTA's store lands.  With a weak ld.global.cg the compiler may treat a
  // retry as redundant: ptxas reduced the wide strips' identity-add poll to
  // a single load and a sentinel leaked into y (nufft3d transpose, variant 0).
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
// Gather cnt entries from x0 (stage 0 through xperm, never polled: user f),
// polling intermediate buffers until every loaded entry is valid.
__device__ __forceinline__ void gather_range(const double2* x, const int* xperm, int x0, int cnt, double2* dst,
                                             int lane) {
  for (int base = 0; base < cnt; base += 32 * 4) {
    double2 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = base + lane + 32 * i;
      if (kk < cnt) v[i] = xperm ? __ldg(x + __ldg(xperm + x0 + kk)) : ld_cg(x + x0 + kk);
    }
    if (!xperm) {
      bool ok;
      do {
        ok = true;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int kk = base + lane + 32 * i;
          if (kk < cnt && is_sentinel(v[i])) {
            v[i] = ld_cg(x + x0 + kk);
            ok = false;
          }
        }
      } while (!ok);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = base + lane + 32 * i;
      if (kk < cnt) dst[kk] = v[i];
    }
  }
}
// Wide compressed strips: gather cnt kept columns x[x0 + map[kk]], polling.
__device__ __forceinline__ void gather_mapped(const double2* x, const int* xperm, int x0, const int* map, int cnt,
                                              double2* dst, int lane) {
  for (int base = 0; base < cnt; base += 32 * 4) {
    double2 v[4];
    int idx[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = base + lane + 32 * i;
      idx[i] = kk < cnt ? x0 + __ldg(map + kk) : -1;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (idx[i] >= 0) v[i] = xperm ? __ldg(x + __ldg(xperm + idx[i])) : ld_cg(x + idx[i]);
    bool ok = xperm != nullptr;  // the user input is never polled
    if (!ok) do {
      ok = true;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (idx[i] >= 0 && is_sentinel(v[i])) {
          v[i] = ld_cg(x + idx[i]);
          ok = false;
        }
    } while (!ok);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (idx[i] >= 0) dst[base + lane + 32 * i] = v[i];
  }
}
__device__ __forceinline__ void gather_x(const StripCtx& c, const double2* x, const int* xperm, double2* dst,
                                         int lane) {
  int cb = 0;
  for (int j = 0; j < c.s.nseg; ++j) {
    gather_range(x, xperm, c.g[j].x0, c.g[j].n, dst + cb, lane);
    cb += c.g[j].n;
  }
  __syncwarp();
}
__device__ __forceinline__ void load_x_regs(const StripCtx& c, const double2* x, const int* xperm, double2* v,
                                            int lane) {
  // input index of each of this lane's staged columns, one pass over the panels
  int idx[kXPerLane];
#pragma unroll
  for (int i = 0; i < kXPerLane; ++i) idx[i] = -1;
  int cb = 0;
  for (int j = 0; j < c.s.nseg; ++j) {
    const int n = c.g[j].n, x0 = c.g[j].x0;
#pragma unroll
    for (int i = 0; i < kXPerLane; ++i) {
      const int kk = lane + 32 * i - cb;
      if (kk >= 0 && kk < n) idx[i] = x0 + kk;
    }
    cb += n;
  }
#pragma unroll
  for (int i = 0; i < kXPerLane; ++i)
    if (idx[i] >= 0) v[i] = xperm ? __ldg(x + __ldg(xperm + idx[i])) : ld_cg(x + idx[i]);
}
__device__ __forceinline__ bool x_regs_ready(const StripCtx& c, const double2* v, int lane) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < kXPerLane; ++i)
    if (lane + 32 * i < c.s.xcols && is_sentinel(v[i])) ok = false;
  return __all_sync(0xffffffffu, ok);
}
__device__ __forceinline__ void store_x_regs(const StripCtx& c, const double2* v, double2* dst, int lane) {
#pragma unroll
  for (int i = 0; i < kXPerLane; ++i)
    if (lane + 32 * i < c.s.xcols) dst[lane + 32 * i] = v[i];
}

// A strip's x window is staged into shared memory by a stager: a dedicated
// warp per pair (flow_sep) or the producer warp's lanes 1..31.  Each lane
// gathers its entries (lane-strided over the flattened panel columns) and
// polls until none is a sentinel; no warp-collective ops inside, so the
// producer's lane 0 can run the TMA issue loop concurrently.
template <int NS, bool CMP, bool PF = false>  // stager lanes, identity-compressed records possible, prefetch only
__device__ __forceinline__ void stage_x(const StripCtx& c, const double2* x, const int* xperm, double2* dst, int sl,
                                        const double2* xbase_lo = nullptr, const double2* xbase_hi = nullptr) {
  constexpr int kPer = (kXWin + NS - 1) / NS;
  int idx[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) idx[i] = -1;
  int cb = 0;
  const bool mapped = CMP && c.mapped != 0;
  for (int j = 0; j < c.s.nseg; ++j) {
    const int n = c.g[j].n, x0 = c.g[j].x0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int kk = sl + NS * i - cb;
      if (kk >= 0 && kk < n) idx[i] = x0 + (mapped ? static_cast<int>(c.cmap[sl + NS * i]) : kk);
    }
    cb += n;
  }
  if (mapped) {  // extra entries: x of unit columns / dropped columns read by adds
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = sl + NS * i - cb;
      if (e >= 0 && e < c.next) {
        const unsigned t = c.xext[e];
        idx[i] = c.g[t >> 8].x0 + static_cast<int>(t & 0xffu);
      }
    }
  }
  if (PF) {  // touch the permutation entries (plan constants) so the gather after the dependency wait hits L1
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (idx[i] >= 0 && xperm) {
        unsigned t;
        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(t) : "l"(xperm + idx[i]));
      }
    return;
  }
  double2 v[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i)
    MIDBF_DCHECK(idx[i] < 0 || (xbase_lo <= x + idx[i] && x + idx[i] < xbase_hi), "k1_flow x gather outside the stage buffers");
#pragma unroll
  for (int i = 0; i < kPer; ++i)
    if (idx[i] >= 0) v[i] = xperm ? __ldg(x + __ldg(xperm + idx[i])) : ld_cg(x + idx[i]);
  if (!xperm) {
    bool ok;
    bool first = true;
    do {
      // The in-warp stager (NS < 32) shares its warp with the TMA-issuing
      // lane 0: back off between polls so that spinning lanes never starve
      // it (variant 2 deadlocked at cfg3 without this).
      if (NS < 32 && !first) __nanosleep(64);
      first = false;
      ok = true;
#pragma unroll
      for (int i = 0; i < kPer; ++i)
        if (idx[i] >= 0 && is_sentinel(v[i])) {
          v[i] = ld_cg(x + idx[i]);
          ok = false;
        }
    } while (!ok);
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i)
    if (idx[i] >= 0) dst[sl + NS * i] = v[i];
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

// Up to 4 pairs per CTA a dedicated x-stager warp per pair fits the register
// file (3 x 4 x 32 threads x 160 registers); with more pairs the producer
// warp's idle lanes 1..31 stage x instead.
template <int FW>
__host__ __device__ constexpr bool flow_sep() {
  return FW <= 4;
}
template <int FW>
__host__ __device__ constexpr int flow_threads() {
  return (flow_sep<FW>() ? 3 : 2) * FW * 32;
}

// Shared-memory layout of one CTA: FW (producer, consumer) warp pairs.
template <int FW, int FS, int SLOT>
struct FlowCfg {
  static constexpr size_t kSlotArea = size_t(FW) * FS * SLOT;
  static constexpr size_t kXArea = size_t(FW) * 2 * kXWin * 16;
  static constexpr size_t kAddArea = size_t(FW) * 2 * 32 * 16;  // per-row identity sums (stager -> consumer)
  static constexpr size_t kCtxArea = size_t(FW) * kQN * sizeof(StripCtx);
  // per pair: full[FS], empty[FS], ctx_full[kQN], ctx_empty[kQN], x_full[2], x_empty[2], a_full[2]
  static constexpr size_t kBarArea = size_t(FW) * (2 * FS + 2 * kQN + 6) * 8;
  static constexpr size_t kStageArea = size_t(kMaxStages) * sizeof(StageIO);  // the stage table, per CTA
  static constexpr size_t kSmem = kSlotArea + kXArea + kAddArea + kCtxArea + kBarArea + kStageArea;
  static_assert(kSmem <= 232448, "k1_flow exceeds the 227 KB dynamic shared memory of a CTA");
};

// Warps [0, FW) consume, warps [FW, 2*FW) produce: producer warp FW+c feeds
// consumer warp c.  The producer's lane 0 walks the consumer's strips (warp
// gw of NW owns strips gw, gw+NW, ...): it waits for a free context entry,
// writes the strip metadata, then for every chunk waits for a free slot and
// issues one cp.async.bulk into it.  It never waits on the consumer's
// dependency polls, x gathers or completion fences, so the slot ring stays
// full and HBM keeps streaming while the consumer is stalled.
// PROF: per-warp clock64 phase timers (experiment builds only), written to
// P.prof[(blockIdx.x * 2*FW + warp) * 16 + phase].
// CMP = false: dense strip records only (no identity-compression code on the
// strips' critical path; small, latency-bound plans, see plan.cu flow_lite).
template <int FW, int FS, int SLOT, bool PROF = false, bool CMP = true>
__global__ void __launch_bounds__(flow_threads<FW>(), 1) k1_flow(const __grid_constant__ FlowParams P) {
  using namespace flowdev;
  using Cfg = FlowCfg<FW, FS, SLOT>;
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned long long g_entry = PROF ? globaltimer_ns() : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr bool kSep = flow_sep<FW>();
  const bool producer = warp >= FW && warp < 2 * FW;
  const bool stager_warp = kSep && warp >= 2 * FW;
  const int c = warp % FW;  // pair index
  unsigned char* slots = smem + size_t(c) * FS * SLOT;
  double2* xb = reinterpret_cast<double2*>(smem + Cfg::kSlotArea) + c * 2 * kXWin;
  double2* asum = reinterpret_cast<double2*>(smem + Cfg::kSlotArea + Cfg::kXArea) + c * 2 * 32;
  StripCtx* ctx = reinterpret_cast<StripCtx*>(smem + Cfg::kSlotArea + Cfg::kXArea + Cfg::kAddArea) + c * kQN;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem + Cfg::kSlotArea + Cfg::kXArea + Cfg::kAddArea + Cfg::kCtxArea) +
      c * (2 * FS + 2 * kQN + 6);
  uint64_t* full = bars;
  uint64_t* empty = bars + FS;
  uint64_t* cfull = bars + 2 * FS;
  uint64_t* cempty = bars + 2 * FS + kQN;
  uint64_t* xfull = bars + 2 * FS + 2 * kQN;      // x window of strip k staged (buffer k & 1)
  uint64_t* xempty = bars + 2 * FS + 2 * kQN + 2;  // buffer k & 1 released by the consumer
  uint64_t* afull = bars + 2 * FS + 2 * kQN + 4;   // identity sums of strip k in asum[k & 1] (separate stagers)
  // the stage table (plan constants) in shared memory: read at every strip
  StageIO* stsm = reinterpret_cast<StageIO*>(smem + Cfg::kSlotArea + Cfg::kXArea + Cfg::kAddArea + Cfg::kCtxArea +
                                             Cfg::kBarArea);
  for (int i = threadIdx.x; i < P.nstages; i += blockDim.x) stsm[i] = P.st[i];
  if (producer && lane == 0) {
    // xfull: one arrival from a separate stager warp (after its warp
    // barrier), or one per lane of the producer warp's in-warp stager, which
    // must not use warp barriers while lane 0 runs the TMA loop (FW > 4 hung
    // at cfg3 with them)
    for (int s = 0; s < 2 * FS + 2 * kQN + 6; ++s)
      mbar_init(&bars[s], (!kSep && s >= 2 * FS + 2 * kQN && s < 2 * FS + 2 * kQN + 2) ? 31 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // Chained applies (P.pdl, programmatic dependent launch): the next apply's
  // grid may be scheduled as soon as every CTA of this one got here, and its
  // CTAs take SMs as ours exit.  The panel stream (plan constants) may run
  // ahead; everything that touches the previous apply's results (epochs,
  // stage buffers, input, output) waits for its completion and memory flush.
  const bool tma_lane = producer && (kSep || lane == 0);  // streams plan constants only
  // With direct stage-0 gathers the separate x-stager warps run ahead of the
  // dependency wait as far as their first window's permutation indices (plan
  // constants), so that only the input loads follow the wait.
  const bool early = kSep && stager_warp && P.pdl && P.direct0;
  if (P.pdl) {
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (!tma_lane && !early) asm volatile("griddepcontrol.wait;" ::: "memory");
  }

  unsigned e = (tma_lane || early) ? 0u : *reinterpret_cast<volatile unsigned*>(P.epoch + blockIdx.x) + 1u;
  const int gw = blockIdx.x * FW + c;
  int64_t par_off = (e & 1u) ? P.par_elems : 0;  // this apply's set of stage buffers
  if (!producer && kSep && P.direct0) {
    wait_in_flag(P.in_flag, P.in_seq);  // stage 0 reads the input itself
  } else if (!producer) {
    // stage -1: the input permutation, gathered once into the head of this
    // apply's set (sentinel-armed; stage 0 polls it like any other stage) by
    // the consumer / stager warps while the producers start streaming panels
    const int nw = flow_threads<FW>() / 32 - FW;  // non-producer warps per CTA
    const int wl = warp < FW ? warp : warp - FW;   // index among them
    const int64_t i0 = (static_cast<int64_t>(blockIdx.x) * nw + wl) * 32 + lane;
    const int64_t di = static_cast<int64_t>(gridDim.x) * nw * 32;
    double2* x0 = P.stagebuf + par_off;
    wait_in_flag(P.in_flag, P.in_seq);
    for (int64_t i = i0; i < P.in_len; i += di) {
      const double2 v = __ldg(P.in + __ldg(P.in_perm + i));
      st_signal(x0 + i, make_double2(unsentinel(v.x), unsentinel(v.y)));
    }
  }
  // re-arm the other set for the next apply (nobody reads it during this
  // one): done by the x stagers once their last window is staged
  auto rearm = [&](int sl, int ns) {
    long long* other = reinterpret_cast<long long*>(P.stagebuf + ((e & 1u) ? 0 : P.par_elems));
    const int64_t i0 = (static_cast<int64_t>(blockIdx.x) * FW + c) * ns + sl;
    const int64_t di = static_cast<int64_t>(gridDim.x) * FW * ns;
    for (int64_t i = i0; i < 2 * P.par_elems; i += di) other[i] = -1ll;
  };
  long long tm[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) tm[i] = 0;
  long long t_start = PROF ? clock64() : 0;
  const unsigned long long g_prologue = PROF ? globaltimer_ns() : 0;
#define FLOW_T(i, ...)                          \
  do {                                          \
    if (PROF) {                                 \
      const long long t0_ = clock64();          \
      __VA_ARGS__;                              \
      tm[i] += clock64() - t0_;                 \
    } else {                                    \
      __VA_ARGS__;                              \
    }                                           \
  } while (0)

  // x stager: stages the x window of each of the pair's strips, up to two
  // strips ahead of the consumer (double buffer xb[k & 1])
  auto stager = [&](auto ns, int sl, unsigned mask, bool arriver) {
    constexpr int NS = decltype(ns)::value;
    const int nmine = gw < P.nstrips ? (P.nstrips - 1 - gw) / P.nwarps + 1 : 0;
    bool waited = !early;
    auto dep_wait = [&]() {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      e = *reinterpret_cast<volatile unsigned*>(P.epoch + blockIdx.x) + 1u;
      par_off = (e & 1u) ? P.par_elems : 0;
      waited = true;
    };
    for (int k = 0; k < nmine; ++k) {
      const int sc = k % kQN, b = k & 1;
      FLOW_T(3, mbar_wait(&cfull[sc], (k / kQN) & 1));
      const StripCtx& C = ctx[sc];
      if (!waited) {
        if (C.s.stage == 0 && C.s.xcols <= kXWin)
          stage_x<NS, CMP, true>(C, P.in, P.in_perm, xb + b * kXWin, sl);
        dep_wait();
      }
      if (k >= 2) FLOW_T(12, mbar_wait(&xempty[b], ((k >> 1) - 1) & 1));
      if (C.s.xcols <= kXWin && P.nodeps != 2) {
        const StageIO io = stsm[C.s.stage];
        const bool d0 = kSep && P.direct0 && C.s.stage == 0;
        FLOW_T(13, stage_x<NS, CMP>(C, d0 ? P.in : io.x + (io.x_par ? par_off : 0), d0 ? P.in_perm : io.xperm,
                                    xb + b * kXWin, sl, d0 ? P.in : P.stagebuf,
                                    d0 ? P.in + P.in_len : P.stagebuf + 2 * P.par_elems));
      }
      if (kSep) {
        __syncwarp(mask);
        if (arriver) mbar_arrive(&xfull[b]);
      } else {
        mbar_arrive(&xfull[b]);  // each lane's own entries (release)
      }
      if (CMP && kSep) {
        // Per-row sums of the identity entries, off the consumer's critical
        // path: formed after x_full is signalled (the consumer needs them
        // only after its panel sums) and signalled on a_full (separate
        // stager warps only; with the in-warp stager of FW > 4 the
        // consumers sum in place).
        if (C.mapped == 1 && C.s.xcols <= kXWin && P.nodeps != 2) {
          const double2* xs = xb + b * kXWin;
          for (int r = sl; r < C.s.h; r += NS) {
            const unsigned below = (1u << r) - 1u;
            double ar = 0.0, ai = 0.0;
            for (int j = 0; j < C.s.nseg; ++j) {
              const unsigned a = C.g[j].adds;
              if ((a >> r) & 1u) {
                const double2 t = xs[C.addpos[C.g[j].aoff + __popc(a & below)]];
                ar += t.x;
                ai += t.y;
              }
            }
            asum[b * 32 + r] = make_double2(ar, ai);
          }
        }
        __syncwarp(mask);
        if (arriver) mbar_arrive(&afull[b]);
      }
    }
    if (!waited) dep_wait();
    rearm(sl, NS);
  };

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
            MIDBF_DCHECK(gw + static_cast<int64_t>(kf) * P.nwarps < P.nstrips, "k1_flow strip record index");
            bulk_g2s(&ctx[sc], P.ctxs + gw + static_cast<int64_t>(kf) * P.nwarps, sizeof(StripCtx), &cfull[sc]);
          }
          ++kf;
        }
      };
      unsigned q = 0;
      const uint64_t pol = P.l2_first ? l2_evict_first_policy() : 0ull;
      for (int k = 0; k < nmine; ++k) {
        prefetch(kf <= k);
        const int sc = k % kQN;
        FLOW_T(0, mbar_wait(&cfull[sc], (k / kQN) & 1));
        const StripCtx& C = ctx[sc];
        const int nseg = C.s.nseg;
        for (int j = 0; j < nseg; ++j) {
          const int n = C.g[j].n, h = C.g[j].hc;  // panel rows streamed
          const int cpc = chunk_cols_for(h, SLOT);
          const double2* src = P.arena + C.g[j].off;
          for (int col = 0; col < n; col += cpc, ++q) {
            const int ncol = min(cpc, n - col);
            const unsigned slot = q % FS;
            if (P.nodeps == 3 && q >= FS) continue;  // timing experiment: compute on resident data
            FLOW_T(1, mbar_wait(&empty[slot], ((q / FS) & 1) ^ 1));
            fence_proxy_async();
            const unsigned bytes = static_cast<unsigned>(h * ncol * 16);
            MIDBF_DCHECK(bytes <= SLOT, "k1_flow panel chunk exceeds its slot");
            MIDBF_DCHECK(C.g[j].off >= 0 && C.g[j].off + static_cast<int64_t>(col + ncol) * h <= P.arena_len,
                         "k1_flow panel outside the arena");
            mbar_expect_tx(&full[slot], bytes);
            if (P.l2_first)
              bulk_g2s_hint(slots + size_t(slot) * SLOT, src + static_cast<int64_t>(col) * h, bytes, &full[slot], pol);
            else
              bulk_g2s(slots + size_t(slot) * SLOT, src + static_cast<int64_t>(col) * h, bytes, &full[slot]);
            prefetch(false);
          }
        }
      }
      while (kf <= nmine) prefetch(true);
    } else if (!kSep) {
      stager(std::integral_constant<int, 31>{}, lane - 1, 0xfffffffeu, lane == 1);  // lanes 1..31
    }
    __syncwarp();
  } else if (stager_warp) {
    stager(std::integral_constant<int, 32>{}, lane, 0xffffffffu, lane == 0);
  } else {
    unsigned q = 0;
    for (int k = 0;; ++k) {
      const int sc = k % kQN;
      FLOW_T(2, mbar_wait(&cfull[sc], (k / kQN) & 1));
      const StripCtx& C = ctx[sc];
      if (C.s.y0 < 0) break;
      if (P.nodeps == 2) {  // timing experiment: stream the payload only
        mbar_wait(&xfull[k & 1], (k >> 1) & 1);
        for (int j = 0; j < C.s.nseg; ++j)
          for (int col0 = 0, cpc = chunk_cols_for(C.g[j].hc, SLOT); col0 < C.g[j].n; col0 += cpc, ++q) {
            mbar_wait(&full[q % FS], (q / FS) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[q % FS]);
          }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&xempty[k & 1]);
          mbar_arrive(&cempty[sc]);
        }
        continue;
      }
      const long long t_setup = PROF ? clock64() : 0;
      const int h = C.s.h, nseg = C.s.nseg, y0 = C.s.y0;
      const StageIO io = stsm[C.s.stage];
      const bool d0 = kSep && P.direct0 && C.s.stage == 0;  // (4-pair layout only: plan.cu)
      const double2* xin = d0 ? P.in : io.x + (io.x_par ? par_off : 0);
      const int* xperm = d0 ? P.in_perm : io.xperm;
      double2* yout = io.y ? io.y + (io.y_par ? par_off : 0) : P.out;
      const bool fast = C.s.xcols <= kXWin;
      double2* xcur = xb + (k & 1) * kXWin;
      const unsigned long long g_ctx = PROF ? globaltimer_ns() : 0;
      if (PROF) tm[5] += clock64() - t_setup;
      FLOW_T(4, mbar_wait(&xfull[k & 1], (k >> 1) & 1));  // staged by the producer warp's lanes 1..31
      const unsigned long long g_x = PROF ? globaltimer_ns() : 0;
      // Lane mapping: strips of <= 16 rows use both half-warps (row = lane&15,
      // column parity = lane>>4, combined by one shuffle at the end), wider
      // strips one lane per row.
      const bool halves = h <= 16;
      const int row = halves ? (lane & 15) : lane;
      const int cpar = halves ? (lane >> 4) : 0;
      const int cstep = halves ? 2 : 1;
      const unsigned below = (1u << row) - 1u;  // rows before this lane's
      int yidx = y0 + row;  // output permutation looked up now, used after the compute
      if (io.yperm && row < h && cpar == 0) yidx = io.yperm[yidx];
      double ar0 = 0, ai0 = 0, ar1 = 0, ai1 = 0, ar2 = 0, ai2 = 0, ar3 = 0, ai3 = 0;
      int cb = 0;
      for (int j = 0; j < nseg; ++j) {
        const int n = C.g[j].n;
        // compressed panels: hc rows (this panel's non-unit rows, in order)
        const int hc = CMP ? C.g[j].hc : h;
        const unsigned urows = CMP ? C.g[j].urows : 0u;
        const bool live = row < h && !((urows >> row) & 1u);
        const int prow = __popc(~urows & below);  // row within the streamed panel
        const int cpc = chunk_cols_for(hc, SLOT);
        int win = -1;
        for (int col0 = 0; col0 < n; col0 += cpc, ++q) {
          const int ncol = min(cpc, n - col0);
          const double2* xv;
          if (fast) {
            xv = xcur + cb + col0;
          } else {  // wide strip: windows of kXWin columns, polled synchronously
            const int w0 = col0 / kXWin;
            if (w0 != win) {
              __syncwarp();
              const int cnt = min(kXWin, n - w0 * kXWin);
              if (CMP && C.mapped == 2)
                gather_mapped(xin, xperm, C.g[j].x0, P.wmap + C.wbase + cb + w0 * kXWin, cnt, xcur, lane);
              else
                gather_range(xin, xperm, C.g[j].x0 + w0 * kXWin, cnt, xcur, lane);
              __syncwarp();
              win = w0;
            }
            xv = xcur + (col0 - w0 * kXWin);
          }
          const unsigned slot = q % FS;
          if (P.nodeps != 3 || q < FS) FLOW_T(8, mbar_wait(&full[slot], (q / FS) & 1));
          const double2* M = reinterpret_cast<const double2*>(slots + size_t(slot) * SLOT);
          const long long tc0 = PROF ? clock64() : 0;
          if (live && P.nodeps != 4) {
            // one consumer warp per SM sub-partition: 4 independent
            // accumulators keep the DFMA chains short (latency 8 cycles)
            // pointer walk with the column step a compile-time constant
            // (x offsets immediate, panel offsets loop-invariant): one add
            // per panel load instead of the index arithmetic
            auto body = [&](auto cs_) {
              constexpr int CS = decltype(cs_)::value;
              const int ms = CS * hc;  // panel elements between this lane's columns
              const double2* mp = M + cpar * hc + prow;
              const double2* xp = xv + cpar;
              int c = cpar;
              for (; c + 7 * CS < ncol; c += 8 * CS, mp += 8 * ms, xp += 8 * CS) {
                double2 m[8], xr[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  m[i] = mp[i * ms];
                  xr[i] = xp[i * CS];
                }
                cmac(ar0, ai0, m[0], xr[0]);
                cmac(ar1, ai1, m[1], xr[1]);
                cmac(ar2, ai2, m[2], xr[2]);
                cmac(ar3, ai3, m[3], xr[3]);
                cmac(ar0, ai0, m[4], xr[4]);
                cmac(ar1, ai1, m[5], xr[5]);
                cmac(ar2, ai2, m[6], xr[6]);
                cmac(ar3, ai3, m[7], xr[7]);
              }
              return c;
            };
            int cc = halves ? body(std::integral_constant<int, 2>{}) : body(std::integral_constant<int, 1>{});
            if (cc + 3 * cstep < ncol) {  // remainder spread over the 4 chains
              cmac(ar0, ai0, M[cc * hc + prow], xv[cc]);
              cmac(ar1, ai1, M[(cc + cstep) * hc + prow], xv[cc + cstep]);
              cmac(ar2, ai2, M[(cc + 2 * cstep) * hc + prow], xv[cc + 2 * cstep]);
              cmac(ar3, ai3, M[(cc + 3 * cstep) * hc + prow], xv[cc + 3 * cstep]);
              cc += 4 * cstep;
            }
            if (cc + cstep < ncol) {
              cmac(ar0, ai0, M[cc * hc + prow], xv[cc]);
              cmac(ar1, ai1, M[(cc + cstep) * hc + prow], xv[cc + cstep]);
              cc += 2 * cstep;
            }
            if (cc < ncol) cmac(ar2, ai2, M[cc * hc + prow], xv[cc]);
          }
          if (PROF) tm[9] += clock64() - tc0;
          __syncwarp();
          if (lane == 0 && P.nodeps != 3) mbar_arrive(&empty[slot]);  // slot back to the producer
        }
        cb += n;
      }
      const long long t_epi = PROF ? clock64() : 0;
      double yr = (ar0 + ar1) + (ar2 + ar3), yi = (ai0 + ai1) + (ai2 + ai3);
      if (halves) {  // odd-column half-warp adds into the even one (fixed order)
        yr += __shfl_down_sync(0xffffffffu, yr, 16);
        yi += __shfl_down_sync(0xffffffffu, yi, 16);
      }
      if (CMP && kSep) mbar_wait(&afull[k & 1], (k >> 1) & 1);  // (signalled for every strip)
      if (CMP && kSep && C.mapped == 1 && row < h) {  // identity parts: the row's sum, formed by the x stager
        const double2 t = asum[(k & 1) * 32 + row];
        yr += t.x;
        yi += t.y;
      } else if (CMP && C.mapped == 1 && row < h) {  // identity parts: one staged entry per (panel, add row)
        for (int j = 0; j < nseg; ++j) {
          const unsigned a = C.g[j].adds;
          if ((a >> row) & 1u) {
            const double2 t = xcur[C.addpos[C.g[j].aoff + __popc(a & below)]];
            yr += t.x;
            yi += t.y;
          }
        }
      } else if (CMP && C.mapped == 2 && row < h && cpar == 0) {  // wide strips: read (and poll) the entry itself
        for (int j = 0; j < nseg; ++j) {
          const unsigned a = C.g[j].adds;
          if ((a >> row) & 1u) {
            const int xi = C.g[j].x0 + __ldg(P.wmap + C.wbase + C.nkept + C.g[j].aoff + __popc(a & below));
            const double2 t = xperm ? __ldg(xin + __ldg(xperm + xi)) : poll_cg(xin + xi);
            yr += t.x;
            yi += t.y;
          }
        }
      }
      // The stored value is the readiness signal of this row: never let a
      // result alias the "not yet written" sentinel.
      MIDBF_DCHECK(!(row < h && cpar == 0) || (io.y ? (yout + yidx >= P.stagebuf && yout + yidx < P.stagebuf + 2 * P.par_elems)
                                                    : (yidx >= 0 && yidx < P.out_len)),
                   "k1_flow row store outside its buffer");
      if (PROF) tm[6] += clock64() - t_epi;
      FLOW_T(7, if (row < h && cpar == 0) st_signal(yout + yidx, make_double2(unsentinel(yr), unsentinel(yi))));
      if (PROF && lane == 0 && C.s.seg0 < kProfStrips) {  // per-strip timeline (ns): ctx ready, x staged, stored
        long long* ts = P.prof + kProfStripBase + 3 * static_cast<int64_t>(C.s.seg0);
        ts[0] = static_cast<long long>(g_ctx);
        ts[1] = static_cast<long long>(g_x);
        ts[2] = static_cast<long long>(globaltimer_ns());
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&xempty[k & 1]);  // x buffer free for strip k + 2
        mbar_arrive(&cempty[sc]);     // context no longer read
      }
    }
  }
  if (PROF) {
    tm[10] = clock64() - t_start;  // until this warp is done
    tm[11] = static_cast<long long>(globaltimer_ns());  // absolute ns: this warp's end
    tm[14] = static_cast<long long>(g_entry);          // ... kernel entry
    tm[15] = static_cast<long long>(g_prologue);       // ... after the prologue
    long long* out = P.prof + (static_cast<int64_t>(blockIdx.x) * (flow_threads<FW>() / 32) + warp) * 16;
    if (lane == 0)
      for (int i = 0; i < 16; ++i) out[i] = tm[i];
    __syncwarp();
    if (!kSep && producer && lane == 1) {  // the in-warp x stager's timers
      out[3] = tm[3];
      out[12] = tm[12];
      out[13] = tm[13];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned*>(P.epoch + blockIdx.x) = e;
}
#undef FLOW_T

}  // namespace midbf::dev
