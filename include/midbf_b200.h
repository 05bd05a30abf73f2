/*
 * midbf_b200.h — C ABI of the B200-native MIDBF hot path.
 *
 * The reference (arxiv/paper_1908_09376, /root/reference/proj) is a C++20
 * library with no FFI; its hot-path interface is the C++ API in
 * proj/include/midbf/butterfly.hpp and butterfly_io.hpp.  Each entry point
 * below replaces one piece of that interface (cited per function) and is
 * what a maintainer would bind from another language (INTEGRATION.md shows
 * the ctypes binding used by this repo's Python package and tests).
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / Eigen / STL types;
 *   - complex numbers are interleaved double (re, im) = std::complex<double>;
 *   - vectors and blocks are column-major; a multi-RHS operand is N x nrhs;
 *   - point sets are row-major N x dim doubles;
 *   - every function returns MIDBF_OK (0) or a negative status, and the
 *     message of the last failure on the calling thread is available from
 *     midbf_last_error().  The C++ wrapper rethrows MIDBF_EINVAL as
 *     std::invalid_argument, MIDBF_ELOGIC as std::logic_error and the rest
 *     as std::runtime_error — the reference's error classes
 *     (src/butterfly.cpp:297-304,425-430,645; src/butterfly_io.cpp:33-35).
 *   - there is no CPU fallback: without a usable sm_100 device the device
 *     entry points fail with MIDBF_ECUDA.
 */
#ifndef MIDBF_B200_H
#define MIDBF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MIDBF_OK 0
#define MIDBF_EINVAL (-1)   /* std::invalid_argument */
#define MIDBF_ELOGIC (-2)   /* std::logic_error */
#define MIDBF_ERUNTIME (-3) /* std::runtime_error (I/O, container) */
#define MIDBF_ECUDA (-4)    /* CUDA error or no sm_100 device */

/* Kernel kinds (see include/midbf/kernels.hpp). */
#define MIDBF_KERNEL_FIO2D 0
#define MIDBF_KERNEL_FIO3D 1
#define MIDBF_KERNEL_LOWRANK 2
#define MIDBF_KERNEL_NUFFT 3
#define MIDBF_KERNEL_CONST 4
#define MIDBF_KERNEL_RANK1 5

/* Typed replacement for the reference's per-entry `EntryFn`
 * (proj/include/midbf/butterfly.hpp:24) so the GPU can evaluate entries.
 * All arrays are host memory. */
typedef struct midbf_kernel_desc {
  int32_t kind;
  int32_t dim;          /* 2 or 3 for point kernels */
  int32_t rank;         /* r for MIDBF_KERNEL_LOWRANK */
  int64_t nrows, ncols; /* |X|, |Omega| */
  const double* X;      /* nrows x dim, row-major */
  const double* Omega;  /* ncols x dim, row-major */
  const double* A;      /* nrows x rank, row-major (low-rank phase) */
  const double* B;      /* ncols x rank, row-major */
  const double* u;      /* nrows complex (rank-one test kernel) */
  const double* v;      /* ncols complex */
  double cre, cim;      /* constant test kernel */
} midbf_kernel_desc;

typedef struct midbf_plan_s* midbf_plan_t; /* device arena of one factorization */
typedef struct midbf_fact_s* midbf_fact_t; /* host factorization (bf::Factorization) */

const char* midbf_last_error(void);
/* Number of visible sm_100 devices (0 when none). */
int midbf_device_count(int* out);

/* ---------------------------------------------------------------- plan
 * Upload a factorization given by MIDBF001-style tables into a device plan.
 * Replaces the first half of bf::apply (src/butterfly.cpp:642-667), whose
 * factors live in separately heap-allocated Eigen blocks.
 *   factor_shape: nfactors x 4 (rows, cols, nblocks, ngroups), product order
 *                 [U^1..U^T, S, V^T..V^1] as bf::Factorization::factors;
 *   blocks:       sum(nblocks) x 4 (row_off, col_off, m, n);
 *   groups:       sum(ngroups) x 2 ([begin, end) into the factor's blocks);
 *   payload:      every block, factor by factor, column-major complex
 *                 (exactly the MIDBF001 payload, butterfly_io.hpp:14);
 *   directions:   bit 0 = forward apply, bit 1 = transpose apply. */
int midbf_plan_create(midbf_plan_t* out, int64_t nrows, int64_t ncols, const int64_t* row_perm,
                      const int64_t* col_perm, int64_t nfactors, const int64_t* factor_shape,
                      const int64_t* blocks, const int64_t* groups, const double* payload,
                      unsigned directions);
/* Same, with one payload pointer per block (block b of factor i at
 * block_payloads[sum of earlier factors' block counts + b], column-major
 * complex rows x cols): a factorization whose blocks live in separate
 * allocations (the reference's FactorBlock matrices) needs no host packing. */
int midbf_plan_create_blocks(midbf_plan_t* out, int64_t nrows, int64_t ncols, const int64_t* row_perm,
                             const int64_t* col_perm, int64_t nfactors, const int64_t* factor_shape,
                             const int64_t* blocks, const int64_t* groups, const double* const* block_payloads,
                             unsigned directions);
/* MIDBF001 container straight into a device plan
 * (replaces bf::load_factorization, src/butterfly_io.cpp:103-167). */
int midbf_plan_load(midbf_plan_t* out, const char* path, unsigned directions);
int midbf_plan_destroy(midbf_plan_t plan);
/* out[0..7]: nrows, ncols, nfactors, total_nnz, arena_bytes, ntasks, directions, max_len */
int midbf_plan_info(midbf_plan_t plan, int64_t* out);

/* g = F f (transpose = 0) or f = F^T g (transpose = 1); the plain transpose,
 * not the adjoint (src/butterfly.cpp:636-637).  f / g are N x nrhs
 * column-major complex, each either device memory or host memory (pinned or
 * pageable; host operands are staged through the plan's device buffers).
 * `stream` is a cudaStream_t (NULL = legacy default).  Replaces bf::apply /
 * bf::apply_transpose (include/midbf/butterfly.hpp:123-126). */
int midbf_apply(midbf_plan_t plan, const double* f, double* g, int64_t nrhs, int transpose, void* stream);
/* Pipelined variant for host operands (serving): enqueues H2D, apply and D2H
 * on internal streams with rotating device staging, and returns at once;
 * `stream` waits for this call's result (synchronize it before reading g or
 * reusing f; f is read asynchronously and is not ordered after earlier
 * work on `stream`).  Consecutive calls overlap their copies with the
 * previous apply.  Pinned host memory is needed for real overlap.  A
 * chained single-RHS apply waits for its staged f inside the kernel (a
 * one-byte flag the copy stream sets after the H2D copy), so its launch
 * stays chained to the previous apply. */
int midbf_apply_async(midbf_plan_t plan, const double* f, double* g, int64_t nrhs, int transpose, void* stream);

/* ------------------------------------------------------- entry sampling
 * Batched K(rows, cols) blocks (replaces the EntryFn fills of shared_sweep,
 * src/butterfly.cpp:462-464, 512-514, 598-600).  Task t fills an
 * nr x nc column-major block at out + 2*out_off (complex):
 *   tasks: ntasks x 5 (row_off, nr, col_off, nc, out_off) with row ids
 *   row_ids[row_off .. row_off+nr) and column ids col_ids[col_off .. +nc).
 * All pointers are host memory; the call returns when `out` is filled. */
int midbf_sample(const midbf_kernel_desc* kernel, int64_t ntasks, const int64_t* tasks, const int64_t* row_ids,
                 int64_t n_row_ids, const int64_t* col_ids, int64_t n_col_ids, double* out, int64_t out_len);

/* Direct O(N^2) sum g(r) = sum_j K(rows[r], j) f(j) for the listed rows
 * (rows == NULL: all rows).  Replaces the direct-summation loops of
 * metrics::eps_b_of (src/metrics.cpp:40-45) and the test oracle
 * dense_matvec (tests/test_butterfly.cpp:29-37).  Host pointers. */
int midbf_direct_sum(const midbf_kernel_desc* kernel, const double* f, const int64_t* rows, int64_t nsel,
                     double* g);
/* Device seconds (CUDA events around K4 and its fixed-order reduction) of the
 * calling thread's last midbf_direct_sum. */
int midbf_last_direct_sum_seconds(double* out);

/* ----------------------------------------- batched interpolative decompositions
 * Column IDs of explicit blocks on the GPU (K5): la::cid_from_rows
 * (src/linalg.cpp:266-286) = truncated pivoted QR pqr_impl (:23-107) +
 * id_rank (:249-264) + V = [I, R11^-1 R12] P^T.  Block b is m_b x n_b complex
 * column-major (dims[2b], dims[2b+1]), blocks packed back to back in
 * `blocks`.  Out: ranks[b] (-1: not computed on the device -- m > 256,
 * n > 512, or the rank rule needs the full QR, the host's fallback case;
 * recompute with the host ID), skel[b*kcap + i] for i < rank (kcap >=
 * min(m_b, n_b, k_max) for every b), V (rank x n_b, ld rank) at
 * vals + 2*voff_b with voff_b = sum over earlier blocks of
 * min(m, n, k_max) * n.  Host pointers; returns when done. */
int midbf_cid_batch(const double* blocks, const int64_t* dims, int64_t nblocks, int64_t k_max, double eps,
                    int64_t* ranks, int64_t* skel, int64_t kcap, double* vals);

/* ------------------------------------------- low-rank phase
 * la::thin_q / la::pinv / la::rsvd (src/linalg.cpp:109-219) on dense host
 * matrices (column-major; complex interleaved when is_complex), the
 * explicit-phase low_rank_phase_factorization (src/phase_md.cpp:184-224,
 * recovery = identity for closed-form phases; rows / columns of Phi
 * evaluated on the GPU) and metrics::eps_K (src/metrics.cpp:55-86, entries
 * sampled on the GPU).  thin_q: Q is m x min(m,n).  pinv: P is n x m, cond =
 * sigma_max / sigma_min.  rsvd_dense: U m x r, S r, V n x r (zero-padded past
 * the returned rank); rng = std::mt19937_64(seed) draws the enlargement
 * sets; info = {rank, rows evaluated, cols evaluated, ill conditioned}.
 * lowrank_phase: rng = std::mt19937_64(seed) draws R, C then rsvd's sets;
 * U nrows x r, V ncols x r (V scaled by S); info = {rank, rows, cols}. */
int midbf_thin_q(const double* A, int64_t m, int64_t n, int is_complex, double* Q);
int midbf_pinv(const double* A, int64_t m, int64_t n, int is_complex, double rel_cutoff, double* P, double* cond);
int midbf_rsvd_dense(const double* A, int64_t m, int64_t n, int is_complex, const int64_t* R0, const int64_t* C0,
                     int64_t s, int64_t r, uint64_t seed, double* U, double* S, double* V, int64_t* info);
int midbf_lowrank_phase(const midbf_kernel_desc* kernel, int64_t r, int64_t q, uint64_t seed, double* U, double* V,
                        int64_t* info);
int midbf_eps_K(const midbf_kernel_desc* kernel, const double* U, const double* V, int64_t r, int64_t nsamp,
                uint64_t seed, double* out);

/* ------------------------------------------- host factorization object
 * bf::idbf_factorize (src/butterfly.cpp:708-769) with trees built the way
 * the reference tests and experiment do (both sides at a common depth,
 * src/experiment.cpp:140-144).  sampler = 0: entries sampled on the GPU (K3),
 * IDs on the host; 1: host evaluation of the same descriptor, host IDs;
 * 2: entries AND interpolative decompositions on the GPU (K3 + K5, replacing
 * la::rid_from_cols / la::cid_from_rows, src/linalg.cpp:266-295; blocks the
 * device hands back are recomputed on the host).  exec = 0 serial, 1 OpenMP.*/
int midbf_factorize(midbf_fact_t* out, const midbf_kernel_desc* kernel, int64_t n0, int64_t k_max, double eps,
                    int64_t t, uint64_t seed, int exec, int sampler);
int midbf_fact_load(midbf_fact_t* out, const char* path);       /* bf::load_factorization */
int midbf_fact_save(midbf_fact_t fact, const char* path);       /* bf::save_factorization */
int midbf_fact_destroy(midbf_fact_t fact);
/* out[0..11]: nrows ncols L h n0 nfactors total_nnz max_factor_nnz k_max t seed exec */
int midbf_fact_info(midbf_fact_t fact, int64_t* out, double* eps);
/* out[0..3]: rows cols nblocks ngroups of factor i */
int midbf_fact_factor(midbf_fact_t fact, int64_t i, int64_t* out);
int midbf_fact_tables(midbf_fact_t fact, int64_t i, int64_t* blocks4, int64_t* groups2);
int midbf_fact_block(midbf_fact_t fact, int64_t i, int64_t b, double* out);
int midbf_fact_perms(midbf_fact_t fact, int64_t* row_perm, int64_t* col_perm);
/* Device plan owned by the factorization (built on first use, both
 * directions, so the handle stays valid until midbf_fact_destroy).
 * Applies through the factorization or its plan may come from several
 * threads / streams at once: a plan runs one apply at a time, in call order. */
int midbf_fact_plan(midbf_fact_t fact, unsigned directions, midbf_plan_t* out);
/* bf::apply on the factorization's cached device plan (host or device operands). */
int midbf_fact_apply(midbf_fact_t fact, const double* f, double* g, int64_t nrhs, int transpose, void* stream);

/* Statistics of a device-sampled factorize: out[0] entries, out[1] sampler calls,
 * out[2] nanoseconds spent in the device sampler (kernel + copies). */
int midbf_fact_stats(midbf_fact_t fact, int64_t* out);
/* out[0] IDs computed on the GPU (K5), out[1] IDs handed back to the host,
 * out[2] nanoseconds in the device ID batches (K3 + K5 + copies), out[3]
 * nanoseconds for the whole factorize (sampler 0 / 2). */
int midbf_fact_id_stats(midbf_fact_t fact, int64_t* out);
/* Device time of the factorize's kernels, CUDA events on the sampler stream:
 * out[0] K3 entry-sampling launches, out[1] entries they evaluated, out[2]
 * their nanoseconds; out[3] K5 ID launches, out[4] their nanoseconds (all 0
 * for host-sampled factorizations).  Not a reference interface: the
 * reference has no device kernels to time. */
int midbf_fact_kernel_stats(midbf_fact_t fact, int64_t* out);

/* Plan introspection / tuning (benchmarks, profiling):
 * stage table out[s*4 + 0..3] = strips, payload bytes, in_len, out_len
 * (application order); flags bit0 = programmatic dependent launch,
 * bit1 = L2 bulk prefetch of the next stage's payload, bit2 = CUDA graphs. */
int midbf_plan_stages(midbf_plan_t plan, int transpose, int64_t* out, int64_t cap);
/* Panel bytes the single-RHS dataflow kernel streams per stage, out[s]
 * (application order): the factors' exact identity parts (unit rows / unit
 * columns of the ID blocks) are gathered from x instead of streamed, unless
 * flag bit 9 (dense panels) is set. */
int midbf_plan_flow_bytes(midbf_plan_t plan, int transpose, int64_t* out, int64_t cap);
/* Panel bytes (16 per entry) the multi-RHS DMMA kernel multiplies per apply on
 * 32- / 64-wide tiles: unit / zero columns of V-type ID strips skipped. */
int midbf_plan_k2_bytes(midbf_plan_t plan, int transpose, int64_t* out);
/* Kernel-path switches (plan.cu): bit0 PDL, bit1 L2 prefetch, bit2 graphs,
 * bit3 k1_flow, bits4-5 k1_flow variant (3 = by size), bits6-8 / 14-15
 * timing experiments (results invalid), bit9 dense panels, bit10 dense-only
 * k1_flow, bit11 no DMMA, bit12 phase timers, bit13 per-stage DMMA, bit16
 * always the compressed k1_flow, bit17 chained single-RHS applies
 * (consecutive k1_flow grids on one stream launch as programmatic dependents,
 * non-cooperatively; process-wide, chained grids on different streams are
 * serialised), bits18 / 19 force / forbid k1_coop, bit24 k1_flow's stage -1
 * input prologue (instead of stage 0 gathering f itself), bit26 four real
 * DMMAs per complex product on k2_flow's 32- / 64-wide tiles (instead of Gauss's
 * three).  A new plan starts at 0x3F | bit17. */
int midbf_plan_set_flags(midbf_plan_t plan, unsigned flags);
int midbf_plan_get_flags(midbf_plan_t plan, unsigned* out);
/* Kernel launches one apply of nrhs columns issues (1 k1_flow launch per
 * column up to 2 RHS, 1 k2_flow launch per 64-RHS slice, else one per stage);
 * the evidence behind bench.py's gpu_launches. */
int midbf_plan_launches(midbf_plan_t plan, int transpose, int64_t nrhs, int64_t* out);
/* Phase timers of the last k1_flow launch made with flag bit 12 (profiling
 * builds/tools only): out holds n int64 counters. */
int midbf_plan_flow_profile(midbf_plan_t plan, int64_t* out, int64_t n);

/* Seeded inputs of the reference experiment (src/experiment.cpp:75-81). */
int midbf_random_coefficients(int64_t n, uint64_t seed, double* out);
uint64_t midbf_chain(uint64_t a, uint64_t b); /* src/butterfly.cpp:20-27 */
/* la::rand_subset with std::mt19937_64(seed) (src/linalg.cpp:390-400); returns the count. */
int64_t midbf_rand_subset(int64_t n, int64_t k, uint64_t seed, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* MIDBF_B200_H */
