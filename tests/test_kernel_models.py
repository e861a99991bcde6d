"""CPU models of two kernel decompositions (no GPU, no oracle arithmetic reused by the product):

* the 28-tile m8n8k4 cover of a node's 12^3 spread taps (dmma3.cuh, spread3_t28_ksteps /
  spread3_t28_update): with the kernel's own row / column / accumulator index formulas, every
  (tx, ty, tz) is produced exactly once, by exactly one warp of the pair, and each tile's A x B
  operand product equals w phi_x[tx] phi_y[ty] phi_z[tz];
* the d = 2 box/band-pruned FFT convolution (fftconv2.cu): radix-2 Stockham autosort, rows over
  the box rows only, band columns x D, Hermitian row inverse == rfft2 -> band multiply -> irfft2
  (cuFFT's unnormalised D2Z / Z2D semantics), with the kernel's index conventions.
"""
import numpy as np
import pytest

W = 12


def _t28_tiles():
    """(warp h, acc slot, A(g, node), B(node, g), out(g, c) -> (tx, ty, tz) or None) per tile,
    transcribed from spread3_t28_ksteps / spread3_t28_update."""
    tiles = []
    for h in (0, 1):
        for j in range(9):   # F1: rows tx = g, columns flat (ty, tz) = 8 (9 h + j) + c
            def out(g, c, h=h, j=j):
                f = 8 * (9 * h + j) + c
                return (g, f // W, f % W)

            def a(g, p):
                return ("wx", g)

            def b(c, h=h, j=j):
                f = 8 * (9 * h + j) + c
                return ("y", f // W), ("z", f % W)
            tiles.append((h, j, a, b, out))
    for p in range(5):       # F2, warp 0: rows (tx, ty) = (8 + g%4, 2p + g/4), columns tz = c
        tiles.append((0, 9 + p, lambda g, _, p=p: ("wx", 8 + (g & 3), "y", 2 * p + (g >> 2)),
                      lambda c: (("z", c),), lambda g, c, p=p: (8 + (g & 3), 2 * p + (g >> 2), c)))
    tiles.append((1, 9, lambda g, _: ("wx", 8 + (g & 3), "y", 10 + (g >> 2)),   # F2 p = 5
                  lambda c: (("z", c),), lambda g, c: (8 + (g & 3), 10 + (g >> 2), c)))
    for t in range(2):       # F3: rows ty = g, columns (tx, tz) = (8 + 2t + c/4, 8 + c%4)
        tiles.append((1, 10 + t, lambda g, _: ("y", g),
                      lambda c, t=t: (("wx", 8 + 2 * t + (c >> 2)), ("z", 8 + (c & 3))),
                      lambda g, c, t=t: (8 + 2 * t + (c >> 2), g, 8 + (c & 3))))
    for p in range(2):       # F4: rows as F2 with pairs 4, 5; columns tz = 8 + c for c < 4
        tiles.append((1, 12 + p, lambda g, _, p=p: ("wx", 8 + (g & 3), "y", 8 + 2 * p + (g >> 2)),
                      lambda c: (("z", 8 + c),) if c < 4 else None,
                      lambda g, c, p=p: (8 + (g & 3), 8 + 2 * p + (g >> 2), 8 + c) if c < 4 else None))
    return tiles


def test_t28_cover_is_an_exact_partition():
    tiles = _t28_tiles()
    assert len(tiles) == 28
    assert sorted((h, s) for h, s, *_ in tiles) == [(h, s) for h in (0, 1) for s in range(14)]
    seen = {}
    for h, slot, _, _, out in tiles:
        for g in range(8):
            for c in range(8):
                o = out(g, c)
                if o is None:
                    continue
                assert all(0 <= v < W for v in o)
                assert o not in seen, (o, seen[o], (h, slot))
                seen[o] = (h, slot)
    assert len(seen) == W ** 3   # 1728 = 28 x 64 - 64 (the half-empty F4 pair)


def test_t28_tile_products_are_the_spread_contribution():
    """A[g][node] * B[node][c] of every tile equals w phi_x[tx] phi_y[ty] phi_z[tz] at its
    output (tx, ty, tz): each of w, phi_x, phi_y, phi_z enters exactly once."""
    rng = np.random.default_rng(3)
    w = rng.random()
    phi = {"x": rng.random(W), "y": rng.random(W), "z": rng.random(W)}

    def val(fs):
        v = 1.0
        i = 0
        while i < len(fs):
            k, t = fs[i], fs[i + 1]
            v *= w * phi["x"][t] if k == "wx" else phi[k][t]
            i += 2
        return v
    for _, _, a, b, out in _t28_tiles():
        for g in range(8):
            for c in range(8):
                o = out(g, c)
                bf = b(c)
                if o is None:
                    assert bf is None
                    continue
                got = val(a(g, 0)) * np.prod([val(f) for f in bf])
                assert np.isclose(got, w * phi["x"][o[0]] * phi["y"][o[1]] * phi["z"][o[2]], rtol=1e-15, atol=0)


def _stockham(x, inverse=False):
    """fftconv2.cu fft_stockham: radix-2 autosort, twiddles e^{-2 pi i k / n}, k < n/2."""
    n = len(x)
    x = x.astype(complex).copy()
    tw = np.exp(-2j * np.pi * np.arange(n // 2) / n)
    if inverse:
        tw = np.conj(tw)
    ns = 1
    while ns < n:
        y = np.empty_like(x)
        for j in range(n // 2):
            k = j & (ns - 1)
            a, b = x[j], x[j + n // 2] * tw[k * (n // (2 * ns))]
            o = ((j - k) << 1) + k
            y[o], y[o + ns] = a + b, a - b
        x, ns = y, ns * 2
    return x


@pytest.mark.parametrize("n,N,box", [(64, 24, (10, 30, 5, 40)), (32, 16, (0, 32, 0, 32)), (64, 62, (3, 7, 50, 14))])
def test_fftconv2_pruned_passes_equal_full_transform(n, N, box):
    rng = np.random.default_rng(n + N)
    h = N // 2
    lo0, bn0, lo1, bn1 = box
    g = np.zeros((n, n))
    g[lo0:lo0 + bn0, lo1:lo1 + bn1] = rng.normal(size=(bn0, bn1))
    D = rng.normal(size=(N + 1, h + 1))   # D[k0 + h][kl], as multiply_kernel / fc2_cols_kernel
    S = np.fft.rfft2(g)
    M = np.zeros_like(S)
    for i in range(n):
        k0 = i if i <= n // 2 else i - n
        if abs(k0) <= h:
            M[i, :h + 1] = S[i, :h + 1] * D[k0 + h]
    ref = np.fft.irfft2(M, s=(n, n)) * n * n   # cuFFT Z2D is unnormalised
    S1 = np.zeros((n, h + 1), complex)
    for i in range(lo0, lo0 + bn0):            # K1: box rows, kl <= N/2
        S1[i] = _stockham(g[i])[:h + 1]
    for kl in range(h + 1):                    # K2: band columns, x D, inverse, box rows back
        c = np.zeros(n, complex)
        c[lo0:lo0 + bn0] = S1[lo0:lo0 + bn0, kl]
        X = _stockham(c)
        for i in range(n):
            k0 = i if i <= n // 2 else i - n
            X[i] = X[i] * D[k0 + h, kl] if abs(k0) <= h else 0
        S1[lo0:lo0 + bn0, kl] = _stockham(X, inverse=True)[lo0:lo0 + bn0]
    for i in range(lo0, lo0 + bn0):            # K3: Hermitian extension, inverse, real part
        F = np.zeros(n, complex)
        F[:h + 1] = S1[i]
        F[n - np.arange(1, h + 1)] = np.conj(S1[i, 1:h + 1])
        out = _stockham(F, inverse=True).real
        assert np.abs(out - ref[i]).max() <= 1e-12 * np.abs(ref).max()
