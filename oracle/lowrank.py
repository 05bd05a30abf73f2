"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's low-rank
phase production, the checker for the product's
la::rsvd / pinv / thin_q, explicit-phase low_rank_phase_factorization and
metrics::eps_K (paper_1908_09376_b200/csrc/host/lowrank.cpp).  Only tests/
may import it.

Follows (reference, /root/reference/proj):
  pinv_impl          src/linalg.cpp:112-131  (SVD, rel cutoff, condition number)
  thin_q_impl        src/linalg.cpp:109-111  (any orthonormal basis: numpy QR)
  rsvd_impl          src/linalg.cpp:134-219
  low_rank_phase_factorization  src/phase_md.cpp:184-224 (recovery = identity)
  eps_K              src/metrics.cpp:55-86
The pivoted QR is the oracle's C restatement of pqr_impl (src/linalg.cpp:23-107,
oracle.pivoted_qr); index sets come from std::mt19937_64 through
oracle.rand_subset_seq in the reference's draw order.
"""
import numpy as np

import oracle as O


def pinv(A, rel_cutoff=1e-12):
    """(pseudoinverse, sigma_max / sigma_min) as pinv_impl."""
    U, s, Vh = np.linalg.svd(A, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((A.shape[1], A.shape[0]), dtype=A.dtype), np.inf
    cond = s[0] / max(s[-1], np.finfo(float).tiny)
    inv = np.where(s > rel_cutoff * s[0], 1.0 / np.where(s > 0, s, 1.0), 0.0)
    return (Vh.conj().T * inv) @ U.conj().T, cond


def thin_q(A):
    return np.linalg.qr(A, mode="reduced")[0]


def rsvd(row, col, m, n, R0, C0, r, draw):
    """rsvd_impl.  row(i) / col(j): full row / column; draw(sr, sc) -> the
    enlargement sets (rand_subset(m, sr), rand_subset(n, sc)) from the rng.
    Returns U, S, V, rows_evaluated, cols_evaluated, ill_conditioned."""
    rows, cols = {}, {}

    def get_row(i):
        if i not in rows:
            rows[i] = np.asarray(row(i))
        return rows[i]

    def get_col(j):
        if j not in cols:
            cols[j] = np.asarray(col(j))
        return cols[j]

    s = len(R0)
    rows_slab = np.array([get_row(i) for i in R0])
    _, _, perm_c, k_c = O.pivoted_qr(rows_slab, s)
    sc = min(s, k_c)
    cols_slab = np.array([get_col(j) for j in C0]).T
    _, _, perm_r, k_r = O.pivoted_qr(np.ascontiguousarray(cols_slab.conj().T), s)
    sr = min(s, k_r)
    dt = rows_slab.dtype
    if sc == 0 or sr == 0:
        return np.zeros((m, 0), dt), np.zeros(0), np.zeros((n, 0), dt), len(rows), len(cols), False
    pc, pr = perm_c[:sc], perm_r[:sr]
    Qc = thin_q(np.array([get_col(j) for j in pc]).T)
    Qr = thin_q(np.array([get_row(i) for i in pr]).conj().T)
    I_rand, J_rand = draw(sr, sc)
    I = np.concatenate([pr, I_rand])
    J = np.concatenate([pc, J_rand])
    AIJ = np.array([get_row(i)[J] for i in I])
    Pc, cond_c = pinv(Qc[I])
    Pr, cond_r = pinv(Qr[J].conj().T)
    M = Pc @ AIJ @ Pr
    ill = not (cond_c < 1e8) or not (cond_r < 1e8)
    Um, sm, Vmh = np.linalg.svd(M)
    rr = min(r, len(sm))
    return Qc @ Um[:, :rr], sm[:rr], Qr @ Vmh.conj().T[:, :rr], len(rows), len(cols), ill


def rsvd_dense(A, R0, C0, r, seed):
    """rsvd on a dense matrix; rng = std::mt19937_64(seed) for the draws."""
    m, n = A.shape
    return rsvd(lambda i: A[i, :], lambda j: A[:, j], m, n, R0, C0, r,
                lambda sr, sc: O.rand_subset_seq(seed, [(m, sr), (n, sc)]))


def lowrank_phase(phi_rows, phi_cols, n1, n2, r, q, seed):
    """low_rank_phase_factorization with recovery = identity:
    R = rand_subset(n1, rq), C = rand_subset(n2, rq), rsvd, V <- V diag(S).
    phi_rows(i) / phi_cols(j): rows / columns of the explicit phase."""
    s = r * q
    R, C = O.rand_subset_seq(seed, [(n1, s), (n2, s)])

    def draw(sr, sc):
        return O.rand_subset_seq(seed, [(n1, s), (n2, s), (n1, sr), (n2, sc)])[2:]

    U, S, V, nr, nc, _ = rsvd(phi_rows, phi_cols, n1, n2, R, C, r, draw)
    return U, V * S, nr, nc


def eps_K(entries, U, V, nsamp, seed):
    """Spectral-norm relative error of exp(2 pi i U V^T) against the kernel
    entries(rows, cols) on rand_subset rows / columns (all when nsamp >= n)."""
    nr, nc = U.shape[0], V.shape[0]
    draws = [(n, nsamp) for n in (nr, nc) if nsamp < n]
    got = iter(O.rand_subset_seq(seed, draws) if draws else [])
    S1 = next(got) if nsamp < nr else np.arange(nr)
    S2 = next(got) if nsamp < nc else np.arange(nc)
    rr, cc = np.meshgrid(S1, S2, indexing="ij")
    A = entries(rr.ravel(), cc.ravel()).reshape(len(S1), len(S2))
    B = np.exp(2j * np.pi * (U[S1] @ V[S2].T))
    den = np.linalg.svd(A, compute_uv=False)[0]
    num = np.linalg.svd(A - B, compute_uv=False)[0]
    return num if den == 0.0 else num / den


def fio2d_phase_block(X, Om, rows, cols):
    """Phi(x, xi) = x.xi + sqrt(c1^2 xi1^2 + c2^2 xi2^2) (src/kernels.cpp:18-24)."""
    tw = 2.0 * np.pi
    x = X[rows]
    w = Om[cols]
    c1 = (2.0 + np.sin(tw * x[:, 0]) * np.sin(tw * x[:, 1])) / 16.0
    c2 = (2.0 + np.cos(tw * x[:, 0]) * np.cos(tw * x[:, 1])) / 16.0
    lin = x @ w.T
    return lin + np.sqrt((c1[:, None] * c1[:, None] * w[None, :, 0]) * w[None, :, 0]
                         + (c2[:, None] * c2[:, None] * w[None, :, 1]) * w[None, :, 1])
