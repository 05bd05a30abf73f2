// Device plan of one factorization (K1 apply).  See plan.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace midbf::dev {

struct StripCtx;
struct StageIO;

constexpr int kMaxStages = 64;
// Plan flag bit 17: chain consecutive single-RHS k1_flow applies on one stream
// with programmatic dependent launch (no graph, no same-stream event wait).
constexpr unsigned kFlagChain = 1u << 17;
// bits 18 / 19: force / forbid k1_coop (CTA-per-strip kernel, coop.cuh) for
// single-RHS applies; by default it runs below kCoopBytes of panels.
constexpr unsigned kFlagCoop = 1u << 18;
constexpr unsigned kFlagNoCoop = 1u << 19;
// k1_flow: gather the input permutation in a stage -1 prologue instead of in
// stage 0's x windows (A/B experiments)
constexpr unsigned kFlagPrologue = 1u << 24;
// k2_flow: four real DMMAs per complex product instead of Gauss's three (A/B)
constexpr unsigned kFlagK2Mul4 = 1u << 26;
// k1_flow / k2_flow stream the factor panels with an L2 evict_first policy,
// so the streamed payload (read once per apply) does not displace the
// intermediate stage vectors the dependency polls read from L2; bits 27 / 28
// restore the default policy (A/B).  Same-box A/B, chained applies: cfg1
// 50.2 -> 47.6 us, cfg1_unitxi 33.8 -> 32.4, cfg3 127.2 -> 121.4, cfg2
// 227.7 -> 223.1.
constexpr unsigned kFlagL2Normal = 1u << 27;
constexpr unsigned kFlagK2L2Normal = 1u << 28;
constexpr int kMaxFlowCtas = 1024;  // per-CTA epoch words
constexpr int kFlowColumns = 2;     // nrhs up to this: k1_flow per column (Plan::flow_ok)

// Output strip of <= 32 rows of one stage; one warp computes it.
struct Strip {
  int32_t y0;     // first output row (stage-local)
  int32_t h;      // rows
  int32_t seg0;   // first panel in the segment table
  int32_t nseg;   // panels accumulated in the reference's block order
  int32_t stage;  // application stage
  int32_t xcols;  // sum of the panel widths (staged x entries)
  int32_t pad_[2];
};

// One block panel feeding a strip: h x n complex, column-major, at arena+off.
struct Seg {
  int64_t off;   // complex-element offset in the arena
  int32_t x0;    // first input entry read (stage-local)
  int32_t n;     // columns
  int32_t dep0;  // producer strips [dep0, dep1) of the previous stage (global ids)
  int32_t dep1;
  int32_t pad_[2];
};

// Host-side view of one factor in MIDBF001 table form.
struct FactorView {
  int64_t rows = 0, cols = 0, nblocks = 0, ngroups = 0;
  const int64_t* blocks = nullptr;         // nblocks x 4
  const int64_t* groups = nullptr;         // ngroups x 2
  const double* const* payload = nullptr;  // per block, column-major complex
};

struct PlanTables {
  int64_t nrows = 0, ncols = 0, nfactors = 0, total_nnz = 0, total_blocks = 0;
  const int64_t* row_perm = nullptr;
  const int64_t* col_perm = nullptr;
  std::vector<FactorView> factors;  // product order [U^1..U^T, S, V^T..V^1]
};

struct Stage {
  int64_t in_len = 0, out_len = 0;
  int32_t strip0 = 0, nstrips = 0;
  int64_t arena0 = 0, payload_bytes = 0;
  int64_t buf_off = 0;  // offset of this stage's output in the stage buffer
  int64_t flow_bytes = 0;  // panel bytes k1_flow streams (identity-compressed)
};

struct Direction {
  bool built = false;
  std::vector<Stage> stages;  // application order
  Strip* d_strips = nullptr;
  Seg* d_segs = nullptr;
  double2* d_arena = nullptr;
  void* d_ctx = nullptr;          // k1_flow strip records (StripCtx, flow.cuh), dense panels
  void* d_fctx = nullptr;         // ... identity-compressed panels (null: nothing to compress)
  int* d_wmap = nullptr;          // wide compressed strips: kept / add columns (StripCtx::wbase)
  // k2_flow on identity-compressed V-type strips (build_k2_records); null: all dense
  Strip* d_k2strips = nullptr;
  Seg* d_k2segs = nullptr;  // the dense segs followed by the compressed strips' segs
  int* d_k2xmap = nullptr;
  int* d_k2addx = nullptr;
  int64_t k2_elems = 0;  // panel entries k2_flow multiplies on 32 / 64-wide tiles
  int64_t farena_elems = 0;       // compressed panels, stored behind the dense ones in d_arena
  int64_t ncols_total = 0;        // panel columns over all segments (plan build)
  double2* d_stagebuf = nullptr;  // outputs of every stage but the last, two parity sets
  StageIO* d_stageio = nullptr;   // k1_flow / k1_coop stage table (built on the first launch)
  unsigned* d_sync = nullptr;     // per-CTA apply epochs (kMaxFlowCtas)
  int64_t nstrips = 0, nsegs = 0, arena_elems = 0, stagebuf_elems = 0;
  int max_seg = 0;  // most panels feeding one strip (k1_flow needs <= kMaxSeg)
  int max_xcols = 0;  // widest x window of a strip (k1_coop needs <= kCoopX)
  int64_t max_strip_bytes = 0;  // largest panel payload of one strip (k1_coop: <= one slot)
  int64_t in_len = 0;  // input length of the first stage (head of the stage buffers)
  // k2_flow (multi-RHS dataflow): per-stage outputs for one 64-RHS slice,
  // per-strip completion counters, per-CTA launch epochs; allocated on first use
  double2* d_k2buf = nullptr;
  unsigned* d_k2done = nullptr;
  unsigned* d_k2epoch = nullptr;
};

struct AsyncSlot {  // device staging of one in-flight host-operand apply
  double2* d_in = nullptr;
  double2* d_out = nullptr;
  int64_t elems = 0;
  bool used = false;
  cudaEvent_t in_ready = nullptr, applied = nullptr, done = nullptr;
  unsigned char flag_seq = 0;  // value of this slot's input-ready flag byte for its latest use
};

struct GraphEntry {
  int d;
  const double2* in;
  double2* out;
  int64_t nrhs;
  unsigned flags;
  cudaGraphExec_t exec;
};

class Plan {
 public:
  // d_raw: optional device copy of every block's payload back to back in
  // table order (taken over and freed); else uploaded from T's payload pointers.
  Plan(const PlanTables& T, unsigned directions, double2* d_raw = nullptr);
  ~Plan();
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  // f, g: host or device, column-major N x nrhs complex.
  void apply(const double* f, double* g, int64_t nrhs, bool transpose, cudaStream_t stream);
  void apply_device(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream);
  // host f/g, enqueue only; `stream` waits for completion (midbf_apply_async)
  void apply_async(const double* f, double* g, int64_t nrhs, bool transpose, cudaStream_t stream);

  int device = 0;
  int num_sms = 0;
  int64_t nrows = 0, ncols = 0, nfactors = 0, total_nnz = 0, max_len = 0;
  Direction dir[2];
  // bit0 PDL + bit1 L2 prefetch (stage kernels), bit2 CUDA graphs,
  // bit3 persistent dataflow kernel for single-RHS applies,
  // bits4-5 k1_flow variant (warps per CTA / ring slots / slot size),
  // bits6-8 timing experiments (flow.cuh), bit9 dense k1_flow panels (identity
  // compression off), bit11 disable K2 (DMMA multi-RHS),
  // bit13 per-stage K2 launches instead of the k2_flow dataflow kernel,
  // bits14-15 k2_flow timing experiments (k2flow.cuh, results invalid).
  // default: k1_flow variant chosen by size (flow_variant), graphs, PDL,
  // prefetch, consecutive single-RHS applies chained (kFlagChain)
  unsigned flags = 0x3F | kFlagChain;
  std::vector<GraphEntry> graphs;
  int flow_grid[4] = {0, 0, 0, 0};
  int coop_grid = 0;  // persistent CTAs of k1_coop (small plans, coop.cuh)
  bool coop(int d) const;
  void ensure_stageio(int d);
  int strip_rows = 32;  // output rows per strip (one warp's lanes)
  long long* d_prof = nullptr;  // k1_flow phase timers (flag bit 12)
  int64_t launches_per_apply(int d, int64_t nrhs) const;
  bool flow_ok(int d, int64_t nrhs) const;
  int flow_variant(int d) const;
  bool flow_lite(int d) const;   // k1_flow without identity-compression code (dense records)
  bool flow_dense(int d) const;  // k1_flow streams the dense panels
  bool k2_ok(int d, int64_t nrhs) const;
  bool k2flow_ok(int d, int64_t nrhs) const;
  int k2flow_grid[3] = {0, 0, 0};  // persistent CTAs of k2_flow<1 | 2 | 4> (16 / 32 / 64-wide tiles)
  int last_grid[2] = {-1, -1};
  void prepare_flow(int d);

 private:
  void build_direction(int d, const PlanTables& T, const double2* d_raw,
                       const std::vector<std::vector<int64_t>>& raw_off);
  void build_flow_records(Direction& D, const std::vector<Strip>& strips, const std::vector<Seg>& segs);
  void build_k2_records(Direction& D, const std::vector<Strip>& strips, const std::vector<Seg>& segs,
                        const std::vector<size_t>& order, const std::vector<StripCtx>& comp);
  void ensure_buffers(int64_t nrhs);
  void launch(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream);
  void launch_stages(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream);
  void launch_flow(int d, const double2* in, double2* out, cudaStream_t stream);
  void launch_k2(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream);
  void launch_k2flow(int d, const double2* in, double2* out, int64_t nrhs, cudaStream_t stream);
  void ensure_k2flow(int d);
  int* d_row_perm = nullptr;
  int* d_col_perm = nullptr;
  double2* d_buf[2] = {nullptr, nullptr};
  int64_t buf_elems = 0;
  double2* d_io[2] = {nullptr, nullptr};
  int64_t io_elems = 0;
  static constexpr int kAsyncSlots = 3;
  AsyncSlot aslots[kAsyncSlots];
  int64_t acount = 0;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_user = nullptr;

 public:
  // One apply at a time per plan (the stage buffers, launch epochs and
  // counters are per plan): `mu` serialises the host side (graph cache,
  // staging, flags), `ev_last` orders the device work of consecutive applies
  // across callers' streams.
  std::recursive_mutex mu;

 private:
  cudaEvent_t ev_last = nullptr;
  cudaStream_t last_stream = nullptr;
  // input-ready flags of the pipelined host-operand path (one byte per async
  // slot) and the flag the next single-RHS flow launch waits on (apply_async)
  unsigned char* d_inflag = nullptr;
  const unsigned char* next_in_flag = nullptr;
  unsigned next_in_seq = 0;  // stream of the previous ordered apply (chain mode skips same-stream waits)
};

std::unique_ptr<Plan> load_plan(const std::string& path, unsigned directions);

}  // namespace midbf::dev
