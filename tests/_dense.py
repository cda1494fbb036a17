"""Independent numpy/scipy assembly of the 7-point operator — used only to PIN the oracle.

Written from the grid definition (periodic longitude, zero-flux latitude and vertical, layout
q = i + nx*(k + nz*j)) without looking at oracle/oracle.c, so a wrong neighbour, sign or index in
either one shows up as a mismatch.
"""
import numpy as np
import scipy.sparse as sp

BAND_OFFSETS = ("E", "W", "N", "S", "U", "D")


def idx(nx, ny, nz, i, j, k):
    return i + nx * (k + nz * j)


def neighbours(nx, ny, nz):
    """yield (q, direction_index, q_nbr) for every present neighbour."""
    for j in range(ny):
        for k in range(nz):
            for i in range(nx):
                q = idx(nx, ny, nz, i, j, k)
                yield q, 0, idx(nx, ny, nz, (i + 1) % nx, j, k)
                yield q, 1, idx(nx, ny, nz, (i - 1) % nx, j, k)
                if j + 1 < ny:
                    yield q, 2, idx(nx, ny, nz, i, j + 1, k)
                if j > 0:
                    yield q, 3, idx(nx, ny, nz, i, j - 1, k)
                if k + 1 < nz:
                    yield q, 4, idx(nx, ny, nz, i, j, k + 1)
                if k > 0:
                    yield q, 5, idx(nx, ny, nz, i, j, k - 1)


def sparse_from_bands(grid, diag, off6):
    """CSR matrix with `diag` on the diagonal and off6[d][q] at (q, nbr_d(q)).
    Duplicate (q, q') pairs (nx == 2 wrap) are summed."""
    nx, ny, nz = grid
    n = nx * ny * nz
    rows, cols, vals = list(range(n)), list(range(n)), list(np.asarray(diag, np.float64))
    for q, d, qn in neighbours(nx, ny, nz):
        rows.append(q)
        cols.append(qn)
        vals.append(off6[d][q])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def dense_Ahat(grid, ahat6):
    n = grid[0] * grid[1] * grid[2]
    return sparse_from_bands(grid, np.ones(n), ahat6).toarray()


def dense_A(grid, bands7):
    return sparse_from_bands(grid, bands7[0], bands7[1:]).toarray()


def transpose_apply(grid, ahat6, y):
    """Ahat^T y by scatter: (Ahat^T y)_{q'} = y_{q'} + sum over q with nbr_d(q) = q' of ahat_d(q) y_q."""
    out = np.array(y, np.float64, copy=True)
    for q, d, qn in neighbours(*grid):
        out[qn] += ahat6[d][q] * y[q]
    return out


def dense_T(grid, ahat6):
    """block-diagonal vertical tridiagonal part T of Ahat (U/D bands + unit diagonal)."""
    nx, ny, nz = grid
    n = nx * ny * nz
    T = np.eye(n)
    for j in range(ny):
        for i in range(nx):
            for k in range(nz):
                q = idx(nx, ny, nz, i, j, k)
                if k + 1 < nz:
                    T[q, idx(nx, ny, nz, i, j, k + 1)] = ahat6[4][q]
                if k > 0:
                    T[q, idx(nx, ny, nz, i, j, k - 1)] = ahat6[5][q]
    return T
