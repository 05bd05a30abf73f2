// Interpolative decompositions used by the factorization (drop-in for the ID
// subset of the reference's proj/include/midbf/linalg.hpp:56-108); the
// randomized SVD / pinv / thin_q part of that header is in midbf/lowrank.hpp.
//
// These are the host IDs (bitwise the oracle's arithmetic); the factorization
// runs its IDs on the GPU by default (K5, midbf_cid_batch) and falls back to
// these for blocks the device hands back.  The pivoted QR is truncated after
// k_max steps and never forms Q: rows 0..k_max-1 of R and the first k_max
// pivots are final after step k_max-1, so the skeleton, the rank and the
// interpolation matrix equal the reference's full-QR result
// (src/linalg.cpp:23-107, 266-286).
#pragma once

#include <random>

#include "midbf/types.hpp"

namespace midbf::la {

struct RankSpec {  // include/midbf/linalg.hpp:63-66
  Index k_max = 0;
  double eps = 0.0;
};

struct ColumnID {  // :70-74
  IndexVec skeleton;
  MatXc V;  // k x n, V(:, skeleton) = I
  Index rank = 0;
};

struct RowID {  // :81-85
  IndexVec skeleton;
  MatXc W;  // m x k, W(skeleton, :) = I
  Index rank = 0;
};

// Pivoted-QR result restricted to what the ID needs.
struct PivotedQR {
  MatXc R;        // r x n upper trapezoidal, real non-negative diagonal
  IndexVec perm;  // column pivot order, size n
  Index rank = 0;
};

// Column-pivoted Householder QR (largest remaining column norm, ties to the
// lowest position), stopping after `max_steps` steps (<0: min(m,n)).
PivotedQR pivoted_qr(const MatXc& A, Index max_steps = -1);

Index id_rank(const VecXd& rdiag_abs, const RankSpec& spec);  // :91
ColumnID cid_from_rows(const MatXc& rows_block, const RankSpec& spec);
RowID rid_from_cols(const MatXc& cols_block, const RankSpec& spec);

// Sampling helpers (:96-108).
IndexVec mock_chebyshev_points(const MatXd& points, Index s, std::mt19937_64& rng);
IndexVec rand_subset(Index n, Index k, std::mt19937_64& rng);

}  // namespace midbf::la
