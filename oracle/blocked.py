"""numpy restatement of the reference's blocked CPU path (the numerics of
blockmv/kernels.py, offset.py and multidevice.py, without the Kepler
transaction accounting).  Test infrastructure and the single-core
`reference` CPU arm only.

Operands are plain 2-D numpy arrays (any strides); outputs are fresh
arrays in the operand dtype, accumulated in that dtype in the reference's
fixed thread-block order, so for the same inputs they reproduce
blockmv's y_out (tests/test_oracle.py checks this against golden vectors
made by the real package).
"""

from __future__ import annotations

import numpy as np


def tb_share(total: int, coop: int, slot: int):
    """partition.py:101-114."""
    base, rem = divmod(total, coop)
    return base + (1 if slot < rem else 0), slot * base + min(slot, rem)


def scal(y, beta, dtype):
    """kernels.py:127-146 (beta == 0 writes zeros without reading y)."""
    if beta == 0:
        return np.zeros(len(y), dtype=dtype)
    return (np.asarray(y) * dtype.type(beta)).astype(dtype)


def gemv_accumulate(A, x, alpha, nb: int, coop: int, transposed: bool, conjugate: bool):
    """kernels.py:149-201."""
    m, n = A.shape
    if transposed:
        x_count, total, out_len, inner = -(-n // nb), -(-m // nb), n, m
    else:
        x_count, total, out_len, inner = -(-m // nb), -(-n // nb), m, n
    dtype = A.dtype
    alpha = dtype.type(alpha)
    acc_out = np.zeros(out_len, dtype=dtype)
    for xb in range(x_count):
        o0, o1 = xb * nb, min(out_len, (xb + 1) * nb)
        for slot in range(coop):
            w, s = tb_share(total, coop, slot)
            if w == 0:
                continue
            acc = np.zeros(o1 - o0, dtype=dtype)
            for j in range(s, s + w):
                i0, i1 = j * nb, min(inner, (j + 1) * nb)
                if transposed:
                    blk = A[i0:i1, o0:o1]
                    bt = blk.conj().T if conjugate else blk.T
                    acc += bt @ x[i0:i1]
                else:
                    acc += A[o0:o1, i0:i1] @ x[i0:i1]
            acc_out[o0:o1] += alpha * acc
    return acc_out


def symv_offdiag_accumulate(A, uplo: str, x, alpha, nb: int, coop: int, conjugate: bool):
    """kernels.py:239-284."""
    d = A.shape[0]
    t = -(-d // nb)
    dtype = A.dtype
    alpha = dtype.type(alpha)
    lower = uplo == "l"
    acc_out = np.zeros(d, dtype=dtype)
    for i in range(t):
        c0, c1 = i * nb, min(d, (i + 1) * nb)
        total = (t - i - 1) if lower else i
        for slot in range(coop):
            w, s = tb_share(total, coop, slot)
            if w == 0:
                continue
            vacc = np.zeros(c1 - c0, dtype=dtype)
            for k in range(s, s + w):
                j = (i + 1 + k) if lower else k
                r0, r1 = j * nb, min(d, (j + 1) * nb)
                blk = A[r0:r1, c0:c1]
                acc_out[r0:r1] += alpha * (blk @ x[c0:c1])
                bt = blk.conj().T if conjugate else blk.T
                vacc += bt @ x[r0:r1]
            acc_out[c0:c1] += alpha * vacc
    return acc_out


def _mirror_block(blk, uplo: str, hermitian: bool):
    """kernels.py:344-354."""
    blk = np.array(blk, copy=True)
    if uplo == "l":
        half, mirror = np.tril(blk), np.tril(blk, -1)
    else:
        half, mirror = np.triu(blk), np.triu(blk, 1)
    mirrored = half + (mirror.conj().T if hermitian else mirror.T)
    if hermitian:
        idx = np.arange(blk.shape[0])
        mirrored[idx, idx] = mirrored[idx, idx].real
    return mirrored


def diag_accumulate(A, uplo: str, x, alpha, nb: int, hermitian: bool):
    """kernels.py:316-359."""
    d = A.shape[0]
    t = -(-d // nb)
    dtype = A.dtype
    alpha = dtype.type(alpha)
    out = np.zeros(d, dtype=dtype)
    for k in range(t):
        r0, r1 = k * nb, min(d, (k + 1) * nb)
        out[r0:r1] = alpha * (_mirror_block(A[r0:r1, r0:r1], uplo, hermitian) @ x[r0:r1])
    return out


def gemv(trans: str, alpha, A, x, beta, y, nb: int = 64, coop: int = 1):
    """kernels.py:402-440 (y_out only)."""
    A = np.asarray(A)
    dtype = A.dtype
    trans = trans.lower()
    if trans == "c" and not np.iscomplexobj(A):
        trans = "t"
    x = np.asarray(x, dtype=dtype)
    y = np.asarray(y, dtype=dtype)
    if alpha == 0 and beta == 1:
        return y.copy()
    ys = scal(y, beta, dtype)
    if alpha == 0:
        return ys
    contrib = gemv_accumulate(A, x, alpha, nb, coop, trans != "n", trans == "c")
    return ys + contrib


def symv_hemv(uplo: str, alpha, A, x, beta, y, nb: int = 64, coop: int = 1, hermitian: bool | None = None):
    """kernels.py:443-486 and run_diag_block 362-392 (y_out only)."""
    A = np.asarray(A)
    dtype = A.dtype
    if hermitian is None:
        hermitian = np.iscomplexobj(A)
    x = np.asarray(x, dtype=dtype)
    y = np.asarray(y, dtype=dtype)
    d = A.shape[0]
    if alpha == 0 and beta == 1:
        return y.copy()
    contrib = diag_accumulate(A, uplo, x, alpha, nb, hermitian)
    y_diag = contrib if beta == 0 else dtype.type(beta) * y + contrib
    if alpha == 0:
        return y_diag
    return y_diag + symv_offdiag_accumulate(A, uplo, x, alpha, nb, coop, hermitian)


def _frame_extent(parent_dim: int, off: int, sub: int, nb: int):
    """offset.py:66-71."""
    start = off - off % nb
    lead = off - start
    frame = min(parent_dim - start, -(-(lead + sub) // nb) * nb)
    return start, frame, lead


def gemv_offset(trans, alpha, parent, row_off, col_off, sub_m, sub_n, x, beta, y, nb: int = 64, coop: int = 1):
    """offset.py:83-143 (y_out only)."""
    parent = np.asarray(parent)
    dtype = parent.dtype
    trans = trans.lower()
    if trans == "c" and not np.iscomplexobj(parent):
        trans = "t"
    pm, pn = parent.shape
    sr, fh, lr = _frame_extent(pm, row_off, sub_m, nb)
    sc, fw, lc = _frame_extent(pn, col_off, sub_n, nb)
    F = np.array(parent[sr:sr + fh, sc:sc + fw], copy=True)
    F[:lr, :] = 0
    F[lr + sub_m:, :] = 0
    F[:, :lc] = 0
    F[:, lc + sub_n:] = 0
    x = np.asarray(x, dtype=dtype)
    y = np.asarray(y, dtype=dtype)
    if alpha == 0 and beta == 1:
        return y.copy()
    ys = scal(y, beta, dtype)
    if alpha == 0:
        return ys
    if trans == "n":
        xf = np.zeros(fw, dtype=dtype)
        xf[lc:lc + sub_n] = x
        sub = gemv_accumulate(F, xf, alpha, nb, coop, False, False)[lr:lr + sub_m]
    else:
        xf = np.zeros(fh, dtype=dtype)
        xf[lr:lr + sub_m] = x
        sub = gemv_accumulate(F, xf, alpha, nb, coop, True, trans == "c")[lc:lc + sub_n]
    return ys + sub


def symv_hemv_offset(uplo, alpha, parent, offset, sub_d, x, beta, y, nb: int = 64, coop: int = 1,
                     hermitian: bool | None = None):
    """offset.py:146-208 (y_out only)."""
    parent = np.asarray(parent)
    dtype = parent.dtype
    if hermitian is None:
        hermitian = np.iscomplexobj(parent)
    s, fd, lead = _frame_extent(parent.shape[0], offset, sub_d, nb)
    F = np.array(parent[s:s + fd, s:s + fd], copy=True)
    F[:lead, :] = 0
    F[lead + sub_d:, :] = 0
    F[:, :lead] = 0
    F[:, lead + sub_d:] = 0
    x = np.asarray(x, dtype=dtype)
    y = np.asarray(y, dtype=dtype)
    if alpha == 0 and beta == 1:
        return y.copy()
    xf = np.zeros(fd, dtype=dtype)
    xf[lead:lead + sub_d] = x
    contrib = diag_accumulate(F, uplo, xf, alpha, nb, hermitian)
    if alpha != 0:
        contrib = contrib + symv_offdiag_accumulate(F, uplo, xf, alpha, nb, coop, hermitian)
    sub = contrib[lead:lead + sub_d]
    return sub.astype(dtype) if beta == 0 else dtype.type(beta) * y + sub


def owned_block_cols(n: int, nb: int, G: int, g: int):
    """multidevice.py:33-35."""
    return list(range(g, -(-n // nb), G))


def symv_hemv_mgpu(uplo, alpha, A, x, beta, y, G: int, nb: int = 64, coop: int = 1, hermitian=None):
    """multidevice.py:183-284 (y_out only; the packed local panels are the
    owned block columns of A)."""
    A = np.asarray(A)
    dtype = A.dtype
    if hermitian is None:
        hermitian = np.iscomplexobj(A)
    d = A.shape[0]
    t = -(-d // nb)
    x = np.asarray(x, dtype=dtype)
    y = np.asarray(y, dtype=dtype)
    alpha_t = dtype.type(alpha)
    accum = np.zeros(d, dtype=dtype)
    for g in range(G):
        if alpha == 0:
            continue
        partial = np.zeros(d, dtype=dtype)
        for i in owned_block_cols(d, nb, G, g):
            c0, c1 = i * nb, min(d, (i + 1) * nb)
            partial[c0:c1] += alpha_t * (_mirror_block(A[c0:c1, c0:c1], uplo, hermitian) @ x[c0:c1])
            total = (t - i - 1) if uplo == "l" else i
            for slot in range(coop):
                w, s = tb_share(total, coop, slot)
                if w == 0:
                    continue
                vacc = np.zeros(c1 - c0, dtype=dtype)
                for k in range(s, s + w):
                    j = (i + 1 + k) if uplo == "l" else k
                    r0, r1 = j * nb, min(d, (j + 1) * nb)
                    oblk = A[r0:r1, c0:c1]
                    partial[r0:r1] += alpha_t * (oblk @ x[c0:c1])
                    vacc += (oblk.conj().T if hermitian else oblk.T) @ x[r0:r1]
                partial[c0:c1] += alpha_t * vacc
        if owned_block_cols(d, nb, G, g):
            accum += partial
    beta_part = dtype.type(beta) * y if beta != 0 else np.zeros(d, dtype=dtype)
    return beta_part + accum


def gemv_mgpu(trans, alpha, A, x, beta, y, G: int, nb: int = 64, coop: int = 1):
    """multidevice.py:119-180 (y_out only)."""
    A = np.asarray(A)
    dtype = A.dtype
    trans = trans.lower()
    if trans == "c" and not np.iscomplexobj(A):
        trans = "t"
    m, n = A.shape
    x = np.asarray(x, dtype=dtype)
    y = np.asarray(y, dtype=dtype)
    y_len = m if trans == "n" else n
    accum = np.zeros(y_len, dtype=dtype)
    for g in range(G):
        blocks = owned_block_cols(n, nb, G, g)
        if not blocks or alpha == 0:
            continue
        cols = np.concatenate([np.arange(j * nb, min(n, (j + 1) * nb)) for j in blocks])
        local = np.array(A[:, cols], copy=True)
        if trans == "n":
            accum += gemv_accumulate(local, x[cols], alpha, nb, coop, False, False)
        else:
            accum[cols] = gemv_accumulate(local, x, alpha, nb, coop, True, trans == "c")
    beta_part = dtype.type(beta) * y if beta != 0 else np.zeros(y_len, dtype=dtype)
    return beta_part + accum
