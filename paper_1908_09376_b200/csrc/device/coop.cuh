// k1_coop — the single-RHS MIDBF apply for small (L2-resident, latency-bound)
// plans: ONE persistent launch, a whole CTA per strip, every strip's panels
// prefetched.
//
// k1_flow gives each strip to one warp; in a small plan most of its 592 warps
// idle while a stage's few strips run their column loops one warp each, and
// the apply is a chain of per-stage latencies (cfg0: 5 stages of ~3 us, the
// FMA loop most of each).  Here the CTAs take the strips round-robin (CTA b:
// strips b, b+G, ... of the dealt record order k1_flow uses, stage by stage)
// and inside a CTA the W warps split the strip's panel columns (warp w:
// columns w, w+W, ... of the concatenated panels; lane = output row):
//   * thread 0 copies the records and panels of the CTA's next kCoopSlots
//     strips into a shared-memory ring with cp.async.bulk (mbarrier
//     complete_tx) — they are plan constants, so the first ones are in
//     flight before the kernel even waits for the previous apply (chained
//     launch) and never on a stage's critical path;
//   * per strip the CTA gathers the x window into shared memory, polling the
//     previous stage's output for the sentinel (flow.cuh: data as signal,
//     relaxed.gpu loads / stores), multiplies (4 complex accumulators per
//     lane), and warp 0 adds the W per-row partials in warp order (fixed:
//     bitwise run to run) and stores each row with the strong store that
//     signals it (the last stage through row_perm).
// Stage -1 (the input permutation), the parity sets of the stage buffers,
// the per-CTA epochs, the re-arm of the other set and programmatic chaining
// follow k1_flow.  Progress: CTAs walk their strips in increasing order and
// every dependency lies in an earlier stage, so the smallest unfinished
// strip can always run once all CTAs are resident.  Dense strip records
// only; a plan is eligible when every strip's panels fit one slot and its x
// window kCoopX entries (Plan::coop).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "flow.cuh"

namespace midbf::dev {

constexpr int kCoopWarps = 8;
constexpr int kCoopX = 1024;           // staged x entries per strip (16 KB)
constexpr int kCoopSlots = 2;          // strips in flight per CTA
constexpr int kCoopSlotBytes = 65536;  // panels of one strip
constexpr size_t kCoopSmem = size_t(kCoopSlots) * (kCoopSlotBytes + sizeof(StripCtx)) +
                             size_t(kCoopX) * 16 + size_t(kCoopWarps) * 32 * 16 + 64;

template <int W>
__global__ void __launch_bounds__(W * 32) k1_coop(const __grid_constant__ FlowParams P) {
  using namespace flowdev;
  extern __shared__ __align__(128) unsigned char csm[];
  unsigned char* slots = csm;
  StripCtx* ctx = reinterpret_cast<StripCtx*>(csm + size_t(kCoopSlots) * kCoopSlotBytes);
  double2* xs = reinterpret_cast<double2*>(ctx + kCoopSlots);
  double2* red = xs + kCoopX;  // [W][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + W * 32);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NT = W * 32;
  const int G = gridDim.x;
  const int nmine = static_cast<int>(blockIdx.x) < P.nstrips ? (P.nstrips - 1 - static_cast<int>(blockIdx.x)) / G + 1 : 0;
  if (tid == 0) {
    for (int s = 0; s < kCoopSlots; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // thread 0: records + panels of the CTA's i-th strip into slot i % kCoopSlots
  auto fetch = [&](int i) {
    const int s = i % kCoopSlots;
    const StripCtx* src = P.ctxs + blockIdx.x + static_cast<int64_t>(i) * G;
    int64_t bytes = sizeof(StripCtx);
    const int nseg = __ldg(&src->s.nseg), h = __ldg(&src->s.h);
    for (int j = 0; j < nseg; ++j) bytes += int64_t(h) * __ldg(&src->g[j].n) * 16;
    fence_proxy_async();
    mbar_expect_tx(&full[s], static_cast<unsigned>(bytes));
    bulk_g2s(&ctx[s], src, sizeof(StripCtx), &full[s]);
    unsigned char* dst = slots + size_t(s) * kCoopSlotBytes;
    MIDBF_DCHECK(bytes - static_cast<int64_t>(sizeof(StripCtx)) <= kCoopSlotBytes, "k1_coop strip exceeds its slot");
    for (int j = 0; j < nseg; ++j) {
      const unsigned b = static_cast<unsigned>(h * __ldg(&src->g[j].n) * 16);
      MIDBF_DCHECK(__ldg(&src->g[j].off) >= 0 && __ldg(&src->g[j].off) + b / 16 <= P.arena_len,
                   "k1_coop panel outside the arena");
      bulk_g2s(dst, P.arena + __ldg(&src->g[j].off), b, &full[s]);
      dst += b;
    }
  };
  if (tid == 0)
    for (int i = 0; i < kCoopSlots && i < nmine; ++i) fetch(i);  // plan constants: before the wait
  // P.direct0: stage 0 gathers the user input through the permutation itself
  // (no stage -1 hop on the chain); the first strip's permutation indices are
  // plan constants, loaded before the wait.
  constexpr int kPre = kCoopX / NT;
  int pre[kPre];
#pragma unroll
  for (int t = 0; t < kPre; ++t) pre[t] = -1;
  if (P.direct0 && nmine > 0) {
    const StripCtx* c0 = P.ctxs + blockIdx.x;
    if (__ldg(&c0->s.stage) == 0) {
      const int nseg = __ldg(&c0->s.nseg), xcols = __ldg(&c0->s.xcols);
#pragma unroll
      for (int t = 0; t < kPre; ++t) {
        const int kk = tid + t * NT;
        if (kk < xcols) {
          int j = 0, c = kk;
          while (j < nseg - 1 && c >= __ldg(&c0->g[j].n)) c -= __ldg(&c0->g[j].n), ++j;
          pre[t] = __ldg(P.in_perm + __ldg(&c0->g[j].x0) + c);
        }
      }
    }
  }
  if (P.pdl) {
    if (tid == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const unsigned e = *reinterpret_cast<volatile unsigned*>(P.epoch + blockIdx.x) + 1u;
  const int64_t par_off = (e & 1u) ? P.par_elems : 0;
  wait_in_flag(P.in_flag, P.in_seq);
  if (!P.direct0) {  // stage -1: the input permutation into the head of this apply's set
    double2* x0 = P.stagebuf + par_off;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * NT + tid; i < P.in_len; i += static_cast<int64_t>(G) * NT) {
      const double2 v = __ldg(P.in + __ldg(P.in_perm + i));
      st_signal(x0 + i, make_double2(unsentinel(v.x), unsentinel(v.y)));
    }
  }
  for (int i = 0; i < nmine; ++i) {
    const int s = i % kCoopSlots;
    mbar_wait(&full[s], (i / kCoopSlots) & 1);
    const StripCtx& C = ctx[s];
    const double2* M = reinterpret_cast<const double2*>(slots + size_t(s) * kCoopSlotBytes);
    const int h = C.s.h, nseg = C.s.nseg, xcols = C.s.xcols;
    const bool live = lane < h;
    const StageIO io = P.st[C.s.stage];
    const double2* xin = io.x + (io.x_par ? par_off : 0);
    double2* yout = io.y ? io.y + (io.y_par ? par_off : 0) : P.out;
    // x window (polled; stage 0 reads the permuted input the same way, or
    // the user input through the permutation with P.direct0)
    if (P.direct0 && C.s.stage == 0) {
#pragma unroll
      for (int t = 0; t < kPre; ++t) {  // xcols <= kCoopX = kPre * NT
        const int kk = tid + t * NT;
        if (kk >= xcols) break;
        int pi = i == 0 ? pre[t] : -1;
        if (pi < 0) {
          int j = 0, c = kk;
          while (j < nseg - 1 && c >= C.g[j].n) c -= C.g[j].n, ++j;
          pi = __ldg(P.in_perm + C.g[j].x0 + c);
        }
        MIDBF_DCHECK(kk < kCoopX && pi >= 0 && pi < P.in_len, "k1_coop input gather");
        xs[kk] = __ldg(P.in + pi);
      }
    } else for (int kk = tid; kk < xcols; kk += NT) {
      int j = 0, c = kk;
      while (j < nseg - 1 && c >= C.g[j].n) c -= C.g[j].n, ++j;
      const double2* p = xin + C.g[j].x0 + c;
      MIDBF_DCHECK(kk < kCoopX && p >= P.stagebuf && p < P.stagebuf + 2 * P.par_elems, "k1_coop x gather");
      double2 v = ld_cg(p);
      while (is_sentinel(v)) v = ld_cg(p);
      xs[kk] = v;
    }
    __syncthreads();
    // this warp's columns: concatenated panel columns w, w+W, ... (the
    // panels lie back to back in the slot, so column q starts at q * h)
    double ar0 = 0, ai0 = 0, ar1 = 0, ai1 = 0, ar2 = 0, ai2 = 0, ar3 = 0, ai3 = 0;
    if (live) {
      int q = w;
      for (; q + 3 * W < xcols; q += 4 * W) {
        const double2 m0 = M[q * h + lane], m1 = M[(q + W) * h + lane];
        const double2 m2 = M[(q + 2 * W) * h + lane], m3 = M[(q + 3 * W) * h + lane];
        cmac(ar0, ai0, m0, xs[q]);
        cmac(ar1, ai1, m1, xs[q + W]);
        cmac(ar2, ai2, m2, xs[q + 2 * W]);
        cmac(ar3, ai3, m3, xs[q + 3 * W]);
      }
      for (; q < xcols; q += W) cmac(ar0, ai0, M[q * h + lane], xs[q]);
    }
    red[w * 32 + lane] = make_double2((ar0 + ar1) + (ar2 + ar3), (ai0 + ai1) + (ai2 + ai3));
    __syncthreads();
    if (w == 0 && live) {
      double yr = 0.0, yi = 0.0;
#pragma unroll
      for (int ww = 0; ww < W; ++ww) {
        yr += red[ww * 32 + lane].x;
        yi += red[ww * 32 + lane].y;
      }
      int yidx = C.s.y0 + lane;
      if (io.yperm) yidx = io.yperm[yidx];
      MIDBF_DCHECK(io.y ? (yout + yidx >= P.stagebuf && yout + yidx < P.stagebuf + 2 * P.par_elems)
                        : (yidx >= 0 && yidx < P.out_len),
                   "k1_coop row store outside its buffer");
      st_signal(yout + yidx, make_double2(unsentinel(yr), unsentinel(yi)));
    }
    __syncthreads();  // slot s, xs and red are rewritten next
    if (tid == 0 && i + kCoopSlots < nmine) fetch(i + kCoopSlots);
  }
  {  // re-arm the other set for the next apply (nobody reads it during this one)
    long long* other = reinterpret_cast<long long*>(P.stagebuf + ((e & 1u) ? 0 : P.par_elems));
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * NT + tid; i < 2 * P.par_elems; i += static_cast<int64_t>(G) * NT)
      other[i] = -1ll;
  }
  __syncthreads();
  if (tid == 0) *reinterpret_cast<volatile unsigned*>(P.epoch + blockIdx.x) = e;
}

}  // namespace midbf::dev
