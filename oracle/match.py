"""oracle.match — fp64 NCC and PCE (a7, a8).  TEST INFRASTRUCTURE ONLY.

The paper names the two statistics but gives no formula: "Normalized
Cross-Correlation (NCC) to correlate", "PCE and NCC methods were used
for comparison. A preset threshold of 60 ... Values higher than this
threshold".  The definitions below are SPEC.md's (S:287, S:296, S:305,
S:328-331) as fixed by DESIGN.md readings R-15..R-19.  numpy's FFT is used as
a library primitive for the circular correlation (pinned in tests against the
direct O(N^4) sum).
"""
from __future__ import annotations

import numpy as np

PCE_CAP = 1e12
PCE_THRESHOLD = 60.0    # P:259, strict ">"


def ncc(a, b) -> float:
    """Aligned Pearson correlation over all pixels (S:287 value at shift (0,0), R-16)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if a.shape != b.shape:
        raise ValueError("dimension mismatch")
    a = a - a.mean()
    b = b - b.mean()
    saa, sbb = float(np.dot(a, a)), float(np.dot(b, b))
    if saa == 0.0 or sbb == 0.0:
        raise ValueError("constant input")  # S:288 ConstantInput
    return float(np.dot(a, b) / np.sqrt(saa * sbb))


def pce_template(K, Iq):
    """Correlation template T = K_hat (.) I_q (S:305 multiplicative model, R-18)."""
    return np.asarray(K, dtype=np.float64) * np.asarray(Iq, dtype=np.float64)


def correlation_surface(R, T):
    """C[dy,dx] = sum_{y,x} R0[y,x] T0[(y-dy) mod H, (x-dx) mod W], with R0, T0
    the mean-removed inputs (R-17).  If R is T circularly shifted by (dy0,dx0)
    the peak is at (dy0,dx0)."""
    R = np.asarray(R, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    R0 = R - R.mean()
    T0 = T - T.mean()
    return np.real(np.fft.ifft2(np.fft.fft2(R0) * np.conj(np.fft.fft2(T0))))


def pce_from_surface(C, exclusion_half: int = 5, peak=None):
    """peak = argmax|C| (ties -> smallest row-major index, R-17);
    pce = sign(C[p]) C[p]^2 / mean(C[s]^2 over s outside the circular
    (2e+1)^2 neighbourhood of p); zero background -> cap 1e12."""
    C = np.asarray(C, dtype=np.float64)
    H, W = C.shape
    if peak is None:
        flat = int(np.argmax(np.abs(C).ravel()))   # numpy returns the first maximal index
        py, px = divmod(flat, W)
    else:
        py, px = peak
    e = exclusion_half
    ys = [(py + k) % H for k in range(-e, e + 1)]
    xs = [(px + k) % W for k in range(-e, e + 1)]
    ys = sorted(set(ys))
    xs = sorted(set(xs))
    E = C * C
    excl = float(E[np.ix_(ys, xs)].sum())
    n_out = H * W - len(ys) * len(xs)
    v = float(C[py, px])
    if n_out <= 0:
        return PCE_CAP * np.sign(v), (py, px), v
    bg = (float(E.sum()) - excl) / n_out
    if bg <= 0.0:
        return (PCE_CAP if v >= 0 else -PCE_CAP), (py, px), v
    return float(np.sign(v) * v * v / bg), (py, px), v


def pce(R, T, exclusion_half: int = 5, aligned: bool = False):
    """Returns (pce, (dy, dx), peak_value).  aligned=True fixes the peak at (0,0)."""
    C = correlation_surface(R, T)
    return pce_from_surface(C, exclusion_half, peak=(0, 0) if aligned else None)


def block_grid(H: int, W: int, block: int = 500):
    """S:275-278 BlockGrid: disjoint block x block tiles covering the frame in
    row-major order; edge tiles are smaller and kept (never empty).
    Returns [(y, x, h, w)]."""
    if block < 1:
        raise ValueError("block must be >= 1")
    return [(y, x, min(block, H - y), min(block, W - x)) for y in range(0, H, block) for x in range(0, W, block)]


def blockwise_match(R, T, block: int = 500, exclusion_half: int = 5):
    """S:311-314 ("500x500 disjoint blocks"): one aligned
    correlation per tile (no shift search): PCE with the peak fixed at (0,0) of
    the tile's own circular correlation surface, and the aligned NCC of the
    tile.  Returns [(y, x, h, w, pce, ncc)] in row-major tile order."""
    R = np.asarray(R, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    out = []
    for (y, x, h, w) in block_grid(R.shape[0], R.shape[1], block):
        r, t = R[y:y + h, x:x + w], T[y:y + h, x:x + w]
        p, _, _ = pce(r, t, exclusion_half, aligned=True)
        out.append((y, x, h, w, p, ncc(r, t)))
    return out


def wiener_dft(K, windows=(3, 5, 7, 9)):
    """f2 (S:151 option; reading R-23): Wiener filtering of a zero-mean fingerprint
    in the DFT domain, written out step by step:
      F = DFT2(K); A = |F| / sqrt(HW); s2 = mean(K^2);
      m = min over w of the w x w box mean of A^2 with mirror (half-sample
          symmetric) extension (the denoiser's window rule, R-7);
      K' = real(IDFT2(F * s2 / max(m, s2)))
    (the mirror windows make the gain not exactly symmetric under k -> -k; the
    real part keeps its Hermitian part, as any real-to-real implementation must).
    numpy's FFT and scipy's mirror box mean ('reflect', pinned equal to the e_N
    windows in tests) are library primitives."""
    from scipy.ndimage import uniform_filter
    K = np.asarray(K, dtype=np.float64)
    H, W = K.shape
    F = np.fft.fft2(K)
    A2 = (np.abs(F) ** 2) / (H * W)
    s2 = float(np.mean(K * K))
    if s2 == 0.0:
        return np.zeros_like(K)
    m = np.full(K.shape, np.inf)
    for w in windows:
        m = np.minimum(m, uniform_filter(A2, size=w, mode="reflect"))
    return np.real(np.fft.ifft2(F * (s2 / np.maximum(m, s2))))
