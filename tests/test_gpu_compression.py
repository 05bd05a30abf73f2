"""Identity compression against adversarial factor tables (flow.cuh
StripCtx, plan.cu build_flow_records / build_k2_records).  The detection is
structural — it accepts any exact unit row / unit column / zero column, not
just the IDs the factorization writes — so these factors plant every case:
several unit columns on one row of a panel, unit rows in panels that share
their rows with other panels, unit rows whose column is also a unit column of
another row, zero columns, panels that compress to nothing (permutations),
near-misses that must stay dense (2.0, 1 + 1e-15 i, -1), all-zero rows, and
strips wider than the 128-entry x window.  Checked against a dense numpy
product of the same tables, both directions, 1 / 16 / 48 right-hand sides,
every k1_flow layout, compressed and dense panels."""
import numpy as np
import pytest

import paper_1908_09376_b200 as M
from helpers import rel

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _cplx(rng, m, n):
    return rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))


def _unit_cols(rng, B, ncols, rows=None):
    """Make ncols random columns exact unit vectors (distinct rows unless given)."""
    m, n = B.shape
    cols = rng.choice(n, ncols, replace=False)
    rs = rng.choice(m, ncols, replace=ncols > m) if rows is None else rows
    for c, r in zip(cols, rs):
        B[:, c] = 0
        B[r, c] = 1
    return cols


def _unit_rows(rng, B, nrows):
    m, n = B.shape
    rows = rng.choice(m, nrows, replace=False)
    for r in rows:
        B[r, :] = 0
        B[r, rng.integers(n)] = 1
    return rows


def _factor(rows, cols, blocks):
    """blocks: list of (r0, c0, M); one group per block."""
    tab = [(r0, c0, Mb.shape[0], Mb.shape[1]) for r0, c0, Mb in blocks]
    groups = [(i, i + 1) for i in range(len(blocks))]
    return rows, cols, tab, groups, [Mb for _, _, Mb in blocks]


def _dense(f):
    rows, cols, tab, _, mats = f
    D = np.zeros((rows, cols), complex)
    for (r0, c0, m, n), Mb in zip(tab, mats):
        D[r0:r0 + m, c0:c0 + n] += Mb
    return D


@pytest.fixture(scope="module")
def adversarial(gpu):
    rng = np.random.default_rng(77)
    fs = []
    # applied first: 64 x 200 — a wide strip (200 columns: 1 panel) with unit
    # columns and unit rows, and a wide strip of two 100-column panels
    W0 = _cplx(rng, 32, 200)
    _unit_cols(rng, W0, 20)
    _unit_rows(rng, W0, 6)
    W0[:, 7] = 0  # zero column
    W1, W2 = _cplx(rng, 32, 100), _cplx(rng, 32, 100)
    _unit_rows(rng, W1, 9)
    _unit_cols(rng, W2, 12)
    f_wide = _factor(64, 200, [(0, 0, W0), (32, 0, W1), (32, 100, W2)])
    # V-type 48 x 64: unit columns (two on row 3 of the first panel), zero
    # columns, near-misses
    V0 = _cplx(rng, 20, 40)
    _unit_cols(rng, V0, 12)
    V0[:, [1, 2]] = 0
    V0[:, 5] = 0
    V0[3, 5] = 1  # a second unit column on row 3 (unless 3 already had one: then both cases)
    V0[:, 6] = 0
    V0[4, 6] = 2.0  # not a unit
    V0[:, 8] = 0
    V0[9, 8] = 1 + 1e-15j  # not exactly one
    V1 = _cplx(rng, 28, 64)
    _unit_cols(rng, V1, 28)  # an identity part on every row
    f_v = _factor(48, 64, [(0, 0, V0), (20, 0, V1)])
    # U-type 80 x 48: rows [0, 40) are written by two panels (cols [0, 24) and
    # [24, 48)), each with its own unit rows; unit rows whose column is also a
    # unit column; an all-zero row; a row whose single nonzero is -1
    U0, U1 = _cplx(rng, 40, 24), _cplx(rng, 40, 24)
    _unit_rows(rng, U0, 10)
    _unit_rows(rng, U1, 10)
    U0[:, 3] = 0
    U0[11, 3] = 1
    U0[11, :] = 0
    U0[11, 3] = 1  # unit row 11 and unit column 3 at the same entry
    U1[12, :] = 0  # all-zero row in this panel
    U1[13, :] = 0
    U1[13, 4] = -1
    U2 = _cplx(rng, 40, 48)
    _unit_rows(rng, U2, 25)
    f_u = _factor(80, 48, [(0, 0, U0), (0, 24, U1), (40, 0, U2)])
    # permutation 80 x 80: blocks that compress to no panel at all, one negated
    P0 = np.eye(32)[rng.permutation(32)].astype(complex)
    P1 = -np.eye(32)[rng.permutation(32)].astype(complex)
    P2 = np.eye(16)[rng.permutation(16)].astype(complex)
    f_p = _factor(80, 80, [(0, 0, P0), (32, 32, P1), (64, 64, P2)])
    # dense tail 60 x 80
    f_s = _factor(60, 80, [(0, 0, _cplx(rng, 60, 80))])
    fs = [f_s, f_p, f_u, f_v, f_wide]  # product order (the last is applied first)
    rp, cp = rng.permutation(60), rng.permutation(200)
    plan = M.DevicePlan.from_tables(60, 200, rp, cp, fs, directions=3)
    D = np.eye(60, dtype=complex)
    for f in fs:
        D = D @ _dense(f)
    A = np.zeros((60, 200), complex)
    A[np.ix_(rp, cp)] = D  # g[rp] = D f[cp]
    return plan, A, fs


def test_streams_less_than_stored(adversarial):
    plan, A, fs = adversarial
    plan.set_flags(lite=False)  # the compressed kernel (small plans default to the dense-only one)
    stored = [s[1] for s in plan.stages()]
    fb = plan.flow_bytes()
    assert fb[0] < stored[0] and fb[1] < stored[1] and fb[2] < stored[2]  # wide, V, U
    assert fb[3] < stored[3] // 2  # permutations: only the negated block streams
    assert fb[4] == stored[4]  # dense


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("nrhs", [1, 16, 48])
def test_matches_dense_product(adversarial, variant, nrhs):
    plan, A, _ = adversarial
    rng = np.random.default_rng(nrhs + 10 * variant)
    f = _cplx(rng, 200, nrhs)
    g = _cplx(rng, 60, nrhs)
    try:
        plan.set_flags(variant=variant, lite=False)
        a, b = plan.apply(f), plan.apply(g, transpose=True)
        plan.set_flags(variant=variant, compress=False)
        a0, b0 = plan.apply(f), plan.apply(g, transpose=True)
    finally:
        plan.reset_flags()
    assert rel(a, A @ f) <= TOL and rel(b, A.T @ g) <= TOL
    assert rel(a0, A @ f) <= TOL and rel(b0, A.T @ g) <= TOL
