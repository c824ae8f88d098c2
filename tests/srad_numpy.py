"""Tile-level SRAD kernels in numpy — TEST INFRASTRUCTURE (an oracle).

Same operation order as csrc/srad.cu / oracle_srad (float32 arithmetic, no
contraction; fp64 ROI butterfly), acting on the tile buffers of
paper_2107_05681_b200.srad_tiles.SradTiles so the multi-rank exchange logic
can be tested on CPU (gloo) without a GPU.
"""
import numpy as np
import torch


def _roi_layout(roi):
    r1, r2, c1, c2 = roi
    w0 = c1 // 128
    return r1, r2, c1, c2, w0, c2 // 128 - w0 + 1


def roi_partials_rows(img_rows, g_of_row, cols, roi, out):
    """Fill out[(g-r1), w, 0/1] for every given row (img_rows[i] is global row g_of_row[i])."""
    r1, r2, c1, c2, w0, groups = _roi_layout(roi)
    out = out.reshape(r2 - r1 + 1, groups, 2)
    lanes = np.arange(32)
    for row, g in zip(img_rows, g_of_row):
        if g < r1 or g > r2:
            continue
        for w in range(w0, w0 + groups):
            a, b = np.zeros(32), np.zeros(32)
            for k in range(4):   # each lane's 4 columns in order
                j = w * 128 + 4 * lanes + k
                inn = (j < cols) & (j >= c1) & (j <= c2)
                v = np.where(inn, row[np.clip(j, 0, cols - 1)].astype(np.float64), 0.0)
                a, b = a + v, b + v * v
            for o in (16, 8, 4, 2, 1):
                a, b = a + a[lanes ^ o], b + b[lanes ^ o]
            out[g - r1, w - w0, 0] = a[0]
            out[g - r1, w - w0, 1] = b[0]


def q0_from_partials(part, roi):
    r1, r2, c1, c2, w0, groups = _roi_layout(roi)
    s = s2 = 0.0
    p = part.reshape(r2 - r1 + 1, groups, 2)
    for r in range(p.shape[0]):
        for g in range(groups):
            s += float(p[r, g, 0])
            s2 += float(p[r, g, 1])
    npix = float(r2 - r1 + 1) * float(c2 - c1 + 1)
    mean = s / npix
    var = s2 / npix - mean * mean
    return np.float32(var / (mean * mean))


def coeff(jc, n, s, w, e, q0sqr, q0den):
    f = np.float32
    dN, dS, dW, dE = n - jc, s - jc, w - jc, e - jc
    g2 = (((dN * dN + dS * dS) + dW * dW) + dE * dE) / (jc * jc)
    l = (((dN + dS) + dW) + dE) / jc
    num = (f(0.5) * g2) - (f(1.0 / 16.0) * (l * l))
    den = f(1.0) + (f(0.25) * l)
    qsqr = num / (den * den)
    den = (qsqr - q0sqr) / q0den
    c = f(1.0) / (f(1.0) + den)
    return np.where(c < 0, f(0), np.where(c > 1, f(1), c)).astype(np.float32)


class NumpyTileKernels:
    """Drop-in for GpuTileKernels on CPU torch tensors."""

    def roi(self, tile, cols, tile_rows, r0, rows, roi, roi_out):
        t = tile.numpy()[:, :cols]
        out = np.zeros(roi_out.numel(), dtype=np.float64)
        roi_partials_rows([t[i + 1] for i in range(tile_rows)], [r0 + i for i in range(tile_rows)], cols, roi, out)
        roi_out.copy_(torch.from_numpy(out))

    def step(self, tin, tout, cols, tile_rows, r0, rows, lam, roi, roi_in, roi_out, q0, part=0):
        f = np.float32
        if part == 2:   # DARM_SRAD_EDGE_ROWS: rows 0 and n-2, n-1 (own, 0-based); q0 from the interior call
            todo = [0] + list(range(max(1, tile_rows - 2), tile_rows)) if tile_rows > 3 else []
        elif part == 1:   # DARM_SRAD_INTERIOR_ROWS
            todo = list(range(1, tile_rows - 2)) if tile_rows > 3 else list(range(tile_rows))
        else:
            todo = list(range(tile_rows))
        T = tin.numpy()[:, :cols]
        q0sqr = q0_from_partials(roi_in.numpy(), roi)
        q0den = f(q0sqr * (f(1.0) + q0sqr))
        gmax = rows - 1

        def row(g):
            return T[min(max(g, 0), gmax) - r0 + 1]

        jidx = np.arange(cols)
        jw, je = np.clip(jidx - 1, 0, cols - 1), np.clip(jidx + 1, 0, cols - 1)

        def c_of(g):
            jc = row(g)
            return coeff(jc, row(g - 1), row(g + 1), jc[jw], jc[je], q0sqr, q0den)

        lq = f(f(0.25) * f(lam))
        out = roi_out.numpy().copy() if part == 2 else np.zeros(roi_out.numel(), dtype=np.float64)
        newrows = []
        for i in todo:
            g = r0 + i
            jc = row(g)
            c0 = c_of(g)
            c1 = c_of(g + 1) if g + 1 <= gmax else c0
            ce = c0[je]
            dN, dS, dW, dE = row(g - 1) - jc, row(g + 1) - jc, jc[jw] - jc, jc[je] - jc
            d = ((c0 * dN + c1 * dS) + c0 * dW) + ce * dE
            jn = (jc + lq * d).astype(np.float32)
            tout.numpy()[i + 1, :cols] = jn
            newrows.append(jn)
        roi_partials_rows(newrows, [r0 + i for i in todo], cols, roi, out)
        roi_out.copy_(torch.from_numpy(out))
