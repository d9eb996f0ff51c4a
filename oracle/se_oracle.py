"""CPU ORACLE for the Spectral Ewald hot path -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference algorithm
(`/root/reference/pkg/src/pmewald`, package `pmewald`).  It exists so that
the CUDA product path can be checked on the GPU box, where the reference
itself is not present.  It is pinned against golden vectors produced by the
unmodified reference (`tests/golden/make_golden.py` -> `tests/golden/*.npz`,
checked by `tests/test_oracle_golden.py`), so parity is PINNED.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
leg and `--impl reference`) may import this file, and only as the checker /
CPU baseline.  The product package `paper_1712_04732_b200` never imports it.

Every function cites the reference file:line whose behaviour it restates.
Third-party numerics used by the reference and here: numpy.fft (pocketfft),
scipy.special erfc / i0 / j0 / j1 (cephes) -- same libraries, unpinned
versions (pyproject.toml:10-13); container numpy 2.3.5, scipy 1.18.1.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import erf as _erf, erfc as _erfc, erfcx as _erfcx, i0 as _i0, j0 as _j0, j1 as _j1

FOUR_PI = 4.0 * math.pi


# --------------------------------------------------------------- integer plan

def is_7smooth(m: int) -> bool:
    for p in (2, 3, 5, 7):
        while m % p == 0:
            m //= p
    return m == 1


def next_even_smooth(n: int) -> int:
    """aft.py:68-73 -- smallest even 7-smooth integer >= max(2, n)."""
    m = max(2, int(n))
    while (m & 1) or not is_7smooth(m):
        m += 1
    return m


def padded_size(s: float, n: int) -> int:
    """aft.py:76-84 -- ceil(s*n - 1e-9) rounded up to even 7-smooth, or n."""
    if s < 1.0:
        raise ValueError("upsampling factor must be >= 1")
    want = int(np.ceil(s * n - 1e-9))
    return n if want <= n else next_even_smooth(want)


def signed_modes(n: int) -> np.ndarray:
    """aft.py:56-58 -- 0..n/2-1, -n/2..-1 (FFT order)."""
    j = np.arange(n)
    return np.where(j < (n + 1) // 2, j, j - n)


def wavenumbers(n: int, h: float) -> np.ndarray:
    """sekspace.py:100-102 -- 2*pi*fftfreq(n, d=h)."""
    return 2.0 * np.pi * np.fft.fftfreq(n, d=h)


def geometry(L, D, M, P, s0=1.0, s=1.0, R=0.0):
    """sekspace.py:53-70 -- Grid.build and its derived shape / offsets."""
    h = L / M
    Mt = M + P
    g = dict(L=L, D=D, M=M, P=P, h=h, Mt=Mt, Lt=L + P * h,
             R=(R if D < 3 else 0.0),
             g0=(padded_size(s0, Mt) if D < 3 else M),
             gs=(padded_size(s, Mt) if D in (1, 2) else Mt))
    g["shape"] = tuple(M if a < D else Mt for a in range(3))
    g["offsets"] = np.array([0.0 if a < D else 0.5 * P * h for a in range(3)])
    return g


def mode_partition(M, D, nI):
    """aft.py:102-117 -- max-norm split into zero / I / J rows (argwhere order)."""
    n = np.abs(signed_modes(M))
    mu = np.maximum(n[:, None], n[None, :]) if D == 2 else n
    I_idx = np.argwhere((mu >= 1) & (mu <= nI))
    J_idx = np.argwhere(mu > nI)
    return I_idx, J_idx


# --------------------------------------------------------------------- windows

def window_eval(kind, shape, w, x):
    """windows.py:74-84 (gaussian), 106-112 (kb), 148-154 (bm)."""
    x = np.asarray(x, dtype=float)
    inside = np.abs(x) <= w
    if kind == "gaussian":
        v = (shape / (w * math.sqrt(2.0 * math.pi))) * np.exp(-(shape * shape) * (x * x) / (2.0 * w * w))
    else:
        t = np.clip(1.0 - (x / w) ** 2, 0.0, None)
        if kind == "kb":
            v = _i0(shape * np.sqrt(t)) / _i0(shape)
        elif kind == "bm":
            v = np.exp(shape * (np.sqrt(t) - 1.0))
        else:
            raise ValueError(kind)
    return np.where(inside, v, 0.0)


_GL = {}


def _gauss_legendre_ld(n):
    """windows.py:184-199 -- Gauss-Legendre rule polished in long double."""
    if n in _GL:
        return _GL[n]
    x = np.polynomial.legendre.leggauss(n)[0].astype(np.longdouble)

    def legendre(xv):
        a, b = np.ones_like(xv), xv.copy()
        for j in range(2, n + 1):
            a, b = b, ((2 * j - 1) * xv * b - (j - 1) * a) / j
        return b, n * (xv * b - a) / (xv * xv - 1.0)

    for _ in range(2):
        p, dp = legendre(x)
        x = x - p / dp
    _, dp = legendre(x)
    _GL[n] = (x, 2.0 / ((1.0 - x * x) * dp * dp))
    return _GL[n]


def _bm_hat(w, beta, k, nodes):
    """windows.py:202-211 -- 2w int_0^{pi/2} e^{b(cos t-1)} cos(kw sin t) cos t dt."""
    x, wt = _gauss_legendre_ld(nodes)
    th = np.longdouble(0.25 * math.pi) * (x + 1.0)
    f = np.exp(beta * (np.cos(th) - 1.0)) * np.cos(th) * (wt * np.longdouble(0.25 * math.pi))
    ph = np.outer(np.asarray(k, dtype=np.longdouble) * np.longdouble(w), np.sin(th))
    return (2.0 * w * (np.cos(ph) @ f)).astype(float)


def window_fourier(kind, shape, w, k):
    """windows.py:87-91 (gaussian), 115-145 (kb), 214-239 (bm quadrature)."""
    k = np.asarray(k, dtype=float)
    if kind == "gaussian":
        return np.exp(-(w * k) ** 2 / (2.0 * shape * shape))
    if kind == "kb":
        rho2 = shape * shape - (k * w) ** 2
        out = np.empty_like(rho2)
        sm = np.abs(rho2) < 1e-6
        po = rho2 >= 1e-6
        ne = rho2 <= -1e-6
        r = rho2[sm]
        out[sm] = 1.0 + r / 6.0 + r * r / 120.0 + r ** 3 / 5040.0
        out[po] = np.sinh(np.sqrt(rho2[po])) / np.sqrt(rho2[po])
        out[ne] = np.sin(np.sqrt(-rho2[ne])) / np.sqrt(-rho2[ne])
        return 2.0 * w * out / _i0(shape)
    kmax = float(np.max(np.abs(k))) if k.size else 0.0
    nodes = max(64, int(0.75 * (kmax * w + shape)) + 32)
    # the reference keeps the 2x-node evaluation after its convergence check
    return _bm_hat(w, shape, k, 2 * nodes)


def window_fourier_checked(kind, shape, w, k):
    """sekspace.py:181-185 -- transform table with the underflow guard."""
    v = window_fourier(kind, shape, w, k)
    if np.min(np.abs(v)) < 1e-30:
        raise AssertionError("window transform underflow")
    return v


# ---------------------------------------------------------------------- greens

def greens_zero_block(D, R, kappa):
    """greens.py:48-85 -- truncated free-space kernel on the zero periodic block
    (including the D=2 sign convention of the reference, greens.py:75-82)."""
    kappa = np.abs(np.asarray(kappa, dtype=float))
    t = R * kappa
    small = t < 1e-2
    out = np.empty_like(kappa)
    z = t[small] ** 2
    tl = t[~small]
    if D == 0:
        out[small] = R * R * (0.5 - z / 24.0 + z ** 2 / 720.0 - z ** 3 / 40320.0 + z ** 4 / 3628800.0)
        out[~small] = R * R * (1.0 - np.cos(tl)) / tl ** 2
    elif D == 1:
        lr = math.log(R)
        out[small] = R * R * ((0.25 - 0.5 * lr) - z * (1.0 / 64.0 - lr / 16.0)
                              + z ** 2 * (1.0 / 2304.0 - lr / 384.0)
                              - z ** 3 * (1.0 / 147456.0 - lr / 18432.0)
                              + z ** 4 * (1.0 / 14745600.0 - lr / 1474560.0))
        kl = kappa[~small]
        out[~small] = (1.0 - _j0(tl)) / kl ** 2 - (R * lr) * _j1(tl) / kl
    elif D == 2:
        out[small] = R * R * (-0.5 + z / 8.0 - z ** 2 / 144.0 + z ** 3 / 5760.0 - z ** 4 / 403200.0)
        out[~small] = R * R * (1.0 - np.cos(tl) - tl * np.sin(tl)) / tl ** 2
    else:
        raise ValueError("zero block kernel needs D < 3")
    return out


# --------------------------------------------------------------- spread/gather

def stencils(pos, g, kind, shape):
    """sekspace.py:105-121 -- per-axis P-point index sets and window weights."""
    P, h = g["P"], g["h"]
    w = 0.5 * P * h
    t = np.arange(P)
    idx, wts = [], []
    for a in range(3):
        u = pos[:, a] + g["offsets"][a]
        first = np.floor(u / h - 0.5 * P).astype(np.int64) + 1
        ia = first[:, None] + t[None, :]
        d = ia * h - u[:, None]
        if a < g["D"]:
            ia = np.mod(ia, g["M"])
        idx.append(ia)
        wts.append(window_eval(kind, shape, w, d))
    return idx, wts


def spread(pos, q, g, kind, shape, chunk=2048):
    """sekspace.py:130-156 -- H = sum_n q_n wx (x) wy (x) wz, wrapped on periodic axes."""
    if g["P"] > g["M"]:
        raise ValueError("window support P must not exceed M")
    H = np.zeros(g["shape"])
    for s in range(0, len(q), chunk):
        sl = slice(s, s + chunk)
        (ix, iy, iz), (wx, wy, wz) = stencils(pos[sl], g, kind, shape)
        vals = q[sl, None, None, None] * wx[:, :, None, None] * wy[:, None, :, None] * wz[:, None, None, :]
        np.add.at(H, (ix[:, :, None, None], iy[:, None, :, None], iz[:, None, None, :]), vals)
    return H


def gather(H, pos, g, kind, shape, chunk=2048):
    """sekspace.py:159-178 -- phi_m = h^3 sum H~ wx wy wz (adjoint of spread)."""
    out = np.empty(len(pos))
    for s in range(0, len(pos), chunk):
        sl = slice(s, s + chunk)
        (ix, iy, iz), (wx, wy, wz) = stencils(pos[sl], g, kind, shape)
        v = H[ix[:, :, None, None], iy[:, None, :, None], iz[:, None, None, :]]
        out[sl] = np.einsum("npqr,np,nq,nr->n", v, wx, wy, wz)
    return out * g["h"] ** 3


# ---------------------------------------------------------------- k-space stage

def _mollify(k2, xi):
    """sekspace.py:188-189."""
    return np.exp(-k2 / (4.0 * xi * xi))


def kspace_d3(H, g, xi, kind, shape):
    """aft.py:203-206 + sekspace.py:198-206 + aft.py:237-238."""
    w = 0.5 * g["P"] * g["h"]
    k = wavenumbers(g["M"], g["h"])
    wh = window_fourier_checked(kind, shape, w, k)
    k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    inv = np.zeros_like(k2)
    nz = k2 > 0
    inv[nz] = 1.0 / k2[nz]
    W = wh[:, None, None] * wh[None, :, None] * wh[None, None, :]
    F = np.fft.fftn(H.astype(complex)) * (FOUR_PI * _mollify(k2, xi) * inv / W ** 2)
    out = np.fft.ifftn(F)
    _check_real(out)
    return out.real


def _check_real(out):
    """sekspace.py:377-378 -- inverse transform must be real."""
    ref = np.max(np.abs(out.real)) + 1e-300
    if np.max(np.abs(out.imag)) >= 1e-10 * ref:
        raise AssertionError("inverse transform must be real")


def kspace_d0_full(H, g, xi, kind, shape):
    """aft.py:207-211 + sekspace.py:208-215 + aft.py:239-241 (use_kernel=False)."""
    w = 0.5 * g["P"] * g["h"]
    g0, Mt = g["g0"], g["Mt"]
    k = wavenumbers(g0, g["h"])
    wh = window_fourier_checked(kind, shape, w, k)
    k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    G = greens_zero_block(0, g["R"], np.sqrt(k2))
    W = wh[:, None, None] * wh[None, :, None] * wh[None, None, :]
    Hp = np.zeros((g0, g0, g0), dtype=complex)
    Hp[:Mt, :Mt, :Mt] = H
    F = np.fft.fftn(Hp) * (FOUR_PI * _mollify(k2, xi) * G / W ** 2)
    out = np.fft.ifftn(F)[:Mt, :Mt, :Mt]
    _check_real(out)
    return out.real


def d0_kernel_geometry(L, M, P, s0, rc):
    """sekspace.py:266-279 -- nconv, R, bumped s0 and fine grid g0 of the D=0 kernel."""
    if s0 < 1.0 + math.sqrt(3.0) - 1e-12:
        raise ValueError("free-space precompute requires s0 >= 1 + sqrt(3)")
    h = L / M
    Mt = M + P
    Lt = L + P * h
    margin = max(P * h, min(rc, L) if rc is not None else 0.0)
    nhalf = int(np.ceil((L + margin) / h - 0.5))
    nconv = next_even_smooth(max(2 * nhalf, 2 * Mt))
    R = math.sqrt(3.0) * L + margin
    s0b = max(s0, ((nconv // 2) * h + R) / Lt)
    return dict(h=h, Mt=Mt, nconv=nconv, R=R, g0=padded_size(s0b, Mt))


def d0_kernel_table(L, M, P, s0, rc):
    """sekspace.py:257-298 -- real half-spectrum table of the truncated kernel."""
    kg = d0_kernel_geometry(L, M, P, s0, rc)
    h, g0, nconv = kg["h"], kg["g0"], kg["nconv"]
    k = wavenumbers(g0, h)
    k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    fine = np.fft.ifftn(greens_zero_block(0, kg["R"], np.sqrt(k2))) / h ** 3
    del k2
    half = nconv // 2
    sel = np.r_[0:half, g0 - half:g0]
    cube = fine.real[np.ix_(sel, sel, sel)]
    tab = h ** 3 * np.fft.rfftn(cube, s=(nconv,) * 3, axes=(0, 1, 2))
    return np.ascontiguousarray(tab.real), kg


def kspace_d0_kernel(H, g, xi, kind, shape, table, nconv):
    """sekspace.py:301-337 -- 2x padded real-FFT convolution with the table."""
    w = 0.5 * g["P"] * g["h"]
    Mt = g["Mt"]
    F = np.fft.rfft(H, n=nconv, axis=2)
    F = np.fft.fft(F, n=nconv, axis=1)
    F = np.fft.fft(F, n=nconv, axis=0)
    kf = wavenumbers(nconv, g["h"])
    kh = 2.0 * np.pi * np.fft.rfftfreq(nconv, d=g["h"])
    af = _mollify(kf ** 2, xi) / window_fourier_checked(kind, shape, w, kf) ** 2
    ah = _mollify(kh ** 2, xi) / window_fourier_checked(kind, shape, w, kh) ** 2
    F *= table
    F *= FOUR_PI * af[:, None, None]
    F *= af[None, :, None]
    F *= ah[None, None, :]
    out = np.fft.ifft(F, axis=0)[:Mt]
    out = np.fft.ifft(out, axis=1)[:, :Mt]
    return np.fft.irfft(out, n=nconv, axis=2)[:, :, :Mt]


def _zero_pad_axes(a, n, axes):
    shp = list(a.shape)
    for ax in axes:
        shp[ax] = n
    out = np.zeros(shp, dtype=complex)
    out[tuple(slice(0, a.shape[i]) for i in range(a.ndim))] = a
    return out


def kspace_mixed(H, g, xi, kind, shape, nI):
    """D in {1,2}: aft.py:168-190 (forward), sekspace.py:217-254 (scale),
    aft.py:243-265 (inverse)."""
    D, M, Mt, h, g0, gs = g["D"], g["M"], g["Mt"], g["h"], g["g0"], g["gs"]
    if Mt % 2:
        raise ValueError("free-axis grid size must be even")
    w = 0.5 * g["P"] * h
    nfree = 3 - D
    faxes = tuple(range(1, 1 + nfree))
    I_idx, J_idx = mode_partition(M, D, nI)
    kp = wavenumbers(M, h)
    wp = window_fourier_checked(kind, shape, w, kp)

    Hk = np.fft.fftn(H.astype(complex), axes=tuple(range(D)))

    def rows(idx):
        return Hk[idx[:, 0], idx[:, 1]] if D == 2 else Hk[idx[:, 0]]

    # zero block
    zrow = Hk[(0,) * D]
    Z = np.fft.fftn(_zero_pad_axes(zrow[None], g0, faxes), axes=faxes)[0]
    k0 = wavenumbers(g0, h)
    w0 = window_fourier_checked(kind, shape, w, k0)
    if nfree == 1:
        kap2, wfree = k0 ** 2, w0
    else:
        kap2 = k0[:, None] ** 2 + k0[None, :] ** 2
        wfree = w0[:, None] * w0[None, :]
    Z *= FOUR_PI * _mollify(kap2, xi) * greens_zero_block(D, g["R"], np.sqrt(kap2)) / ((wp[0] ** D) * wfree) ** 2

    def block(idx, glen, pad):
        B = rows(idx)
        if pad:
            B = _zero_pad_axes(B, glen, faxes)
        B = np.fft.fftn(B, axes=faxes)
        if len(idx) == 0:
            return B
        kf = wavenumbers(glen, h)
        wf = window_fourier_checked(kind, shape, w, kf)
        if D == 2:
            kr2 = kp[idx[:, 0]] ** 2 + kp[idx[:, 1]] ** 2
            wr = wp[idx[:, 0]] * wp[idx[:, 1]]
        else:
            kr2 = kp[idx[:, 0]] ** 2
            wr = wp[idx[:, 0]]
        if nfree == 1:
            k2 = kr2[:, None] + kf[None, :] ** 2
            W = wr[:, None] * wf[None, :]
        else:
            k2 = kr2[:, None, None] + kf[None, :, None] ** 2 + kf[None, None, :] ** 2
            W = wr[:, None, None] * (wf[:, None] * wf[None, :])[None]
        return B * (FOUR_PI * _mollify(k2, xi) / (k2 * W ** 2))

    Ib = block(I_idx, gs, gs != Mt)
    Jb = block(J_idx, Mt, False)

    cut = (slice(None),) + (slice(0, Mt),) * nfree
    out = np.zeros((M,) * D + (Mt,) * nfree, dtype=complex)
    out[(0,) * D] = np.fft.ifftn(Z[None], axes=faxes)[cut][0]
    Ii = np.fft.ifftn(Ib, axes=faxes)[cut]
    Ji = np.fft.ifftn(Jb, axes=faxes)[cut]
    if D == 2:
        out[I_idx[:, 0], I_idx[:, 1]] = Ii
        out[J_idx[:, 0], J_idx[:, 1]] = Ji
    else:
        out[I_idx[:, 0]] = Ii
        out[J_idx[:, 0]] = Ji
    res = np.fft.ifftn(out, axes=tuple(range(D)))
    _check_real(res)
    return res.real


def se_kspace(pos, q, L, D, prm, use_kernel=None):
    """sekspace.py:340-389 -- spread, k-space stage, gather.

    prm: dict with xi, rc, M, P, window, shape, s0, s, nI, R.
    """
    g = geometry(L, D, prm["M"], prm["P"], prm.get("s0", 1.0), prm.get("s", 1.0), prm.get("R", 0.0))
    kind, shape, xi = prm["window"], prm["shape"], prm["xi"]
    H = spread(pos, q, g, kind, shape)
    if D == 3:
        Ht = kspace_d3(H, g, xi, kind, shape)
    elif D == 0 and (use_kernel or use_kernel is None):
        tab, kg = d0_kernel_table(L, prm["M"], prm["P"], prm["s0"], prm["rc"])
        Ht = kspace_d0_kernel(H, g, xi, kind, shape, tab, kg["nconv"])
    elif D == 0:
        Ht = kspace_d0_full(H, g, xi, kind, shape)
    else:
        Ht = kspace_mixed(H, g, xi, kind, shape, prm["nI"])
    return gather(Ht, pos, g, kind, shape)


# ------------------------------------------------------------------ real space

def _pair_block(xt, xs, qs, xi, rc, same_mask=None):
    d = xt[:, None, :] - xs[None, :, :]
    r = np.sqrt(np.sum(d * d, axis=2))
    zero = r < 1e-14
    if same_mask is not None:
        if np.any(zero & ~same_mask):
            raise SingularConfigurationError_("coincident distinct particles")
    elif np.any(zero):
        raise SingularConfigurationError_("particle coincides with an image")
    use = (r < rc) & ~zero
    rs = np.where(use, r, 1.0)
    return np.where(use, _erfc(xi * rs) / rs, 0.0) @ qs


class SingularConfigurationError_(ValueError):
    """Mirror of core.py:23-24 for the oracle (kept local: no product import)."""


def realspace(pos, q, L, D, xi, rc, targets=None):
    """realspace.py:168-180 -- erfc(xi r)/r pair sum within rc.

    Cell path (realspace.py:43-135) when rc <= L/2 on periodic axes: every
    (source, image shift in {-1,0,1}^D) within rc, i.e. the minimum image,
    restated here with rc-edge cells and a minimum-image displacement.
    Image path (realspace.py:138-165) when D >= 1 and rc > L/2.
    `targets` restricts the evaluation to a subset (for bounded CPU samples).
    """
    if xi <= 0 or rc <= 0:
        raise ValueError("xi and rc must be positive")
    N = len(q)
    tsel = np.arange(N) if targets is None else np.asarray(targets)
    per = np.array([a < D for a in range(3)])
    if D >= 1 and rc > L / 2 + 1e-12:
        layers = int(np.floor((rc + L / 2) / L)) + 1
        rng = [np.arange(-layers, layers + 1) if per[a] else np.array([0]) for a in range(3)]
        out = np.zeros(len(tsel))
        for a in rng[0]:
            for b in rng[1]:
                for c in rng[2]:
                    sh = np.array([a, b, c], float) * L
                    if a == 0 and b == 0 and c == 0:
                        same = tsel[:, None] == np.arange(N)[None, :]
                        out += _pair_block(pos[tsel], pos, q, xi, rc, same)
                    else:
                        out += _pair_block(pos[tsel], pos - sh, q, xi, rc)
        return out
    n = max(1, int(np.floor(L / rc)))
    edge = L / n
    cell = np.minimum((pos / edge).astype(int), n - 1)
    flat = (cell[:, 0] * n + cell[:, 1]) * n + cell[:, 2]
    order = np.argsort(flat, kind="stable")
    starts = np.searchsorted(flat[order], np.arange(n ** 3 + 1))
    out = np.zeros(len(tsel))
    tflat = flat[tsel]
    for hc in np.unique(tflat):
        tpos_i = np.nonzero(tflat == hc)[0]
        ti = tsel[tpos_i]
        hx, hy, hz = hc // (n * n), (hc // n) % n, hc % n
        cand = set()
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    c = [hx + dx, hy + dy, hz + dz]
                    ok = True
                    for a in range(3):
                        if per[a]:
                            c[a] %= n
                        elif not 0 <= c[a] < n:
                            ok = False
                    if ok:
                        cand.add((c[0] * n + c[1]) * n + c[2])
        src = np.concatenate([order[starts[c]:starts[c + 1]] for c in sorted(cand)])
        # bounded dense blocks (clustered inputs hold ~2.4e4 particles per cell)
        step = max(1, int(4_000_000 // max(len(src), 1)))
        for b in range(0, len(ti), step):
            tb, ob = ti[b:b + step], tpos_i[b:b + step]
            d = pos[tb][:, None, :] - pos[src][None, :, :]
            for a in range(3):
                if per[a]:
                    d[:, :, a] -= L * np.round(d[:, :, a] / L)
            r = np.sqrt(np.sum(d * d, axis=2))
            zero = r < 1e-14
            same = tb[:, None] == src[None, :]
            if np.any(zero & ~same):
                raise SingularConfigurationError_("coincident distinct particles")
            use = (r < rc) & ~zero
            rs = np.where(use, r, 1.0)
            out[ob] = np.where(use, _erfc(xi * rs) / rs, 0.0) @ q[src]
    return out


def self_term(q, xi):
    """realspace.py:183-185."""
    return -2.0 * xi * np.asarray(q, dtype=float) / math.sqrt(math.pi)


def total_potential(pos, q, L, D, prm, use_kernel=None):
    """core.py:194-216 -- phi = phi_real + phi_fourier + phi_self."""
    return (realspace(pos, q, L, D, prm["xi"], prm["rc"])
            + se_kspace(pos, q, L, D, prm, use_kernel)
            + self_term(q, prm["xi"]))


# --------------------------------------------------------------- direct sums

def direct_kspace_3p(pos, q, L, xi, kmax, targets=None):
    """Ewald Fourier sum over integer modes |n_a| <= kmax, n != 0 (oracle.py:109-118):
    (4 pi / L^3) sum_k e^{-k^2/4xi^2}/k^2 Re(e^{i k.x_m} S_k), S_k = sum_n q_n e^{-i k.x_n}.
    Separable per-axis phases; modes in slabs of n1 to bound memory."""
    pos = np.asarray(pos, float)
    tg = np.arange(len(pos)) if targets is None else np.asarray(targets)
    n = np.arange(-kmax, kmax + 1)
    c = 2.0 * np.pi / L
    ex, ey, ez = (np.exp(-1j * c * np.outer(pos[:, a], n)) for a in range(3))  # (N, 2kmax+1)
    out = np.zeros(len(tg))
    for i1, n1 in enumerate(n):
        # S[n2, n3] = sum_n q ex[n, n1] ey[n, n2] ez[n, n3]
        S = np.einsum("n,nb,nc->bc", q * ex[:, i1], ey, ez)
        k2 = c * c * (n1 * n1 + n[:, None] ** 2 + n[None, :] ** 2)
        with np.errstate(divide="ignore", invalid="ignore"):
            coef = np.where(k2 > 0, np.exp(-k2 / (4.0 * xi * xi)) / k2, 0.0)
        E = np.einsum("t,tb,tc->tbc", np.conj(ex[tg, i1]), np.conj(ey[tg]), np.conj(ez[tg]))
        out += np.einsum("tbc,bc->t", E, coef * S).real
    return (4.0 * np.pi / L ** 3) * out


def direct_kspace_2p(pos, q, L, xi, kmax, targets=None):
    """Closed-form doubly periodic Fourier sum (oracle.py:120-153): per mode
    k = 2 pi (n1, n2)/L != 0, (pi/L^2) sum_n q_n e^{i k.d} B(k, z)/k with
    B = e^{kz} erfc(k/2xi + xi z) + e^{-kz} erfc(k/2xi - xi z) (erfcx form where
    the argument is >= 0), minus (2 sqrt(pi)/L^2) sum_n q_n [e^{-xi^2 z^2}/xi +
    sqrt(pi) z erf(xi z)]; modes over the half plane with weight 2."""
    pos = np.asarray(pos, float)
    tg = np.arange(len(pos)) if targets is None else np.asarray(targets)
    d = pos[tg, None, :] - pos[None, :, :]
    z = d[..., 2]
    out = np.zeros(len(tg))
    for n1 in range(0, kmax + 1):
        for n2 in range(-kmax, kmax + 1):
            if n1 == 0 and n2 <= 0:
                continue
            kx, ky = 2 * np.pi * n1 / L, 2 * np.pi * n2 / L
            k = math.hypot(kx, ky)
            guard = -(k * k / (4 * xi * xi) + (xi * z) ** 2)
            b = np.zeros_like(z)
            for sgn in (1.0, -1.0):
                u = k / (2 * xi) + sgn * xi * z
                pos_u = u >= 0
                b += np.where(pos_u, _erfcx(np.where(pos_u, u, 0.0)) * np.exp(guard),
                              np.exp(sgn * k * np.where(pos_u, 0.0, z)) * _erfc(u))
            out += 2.0 * (np.cos(kx * d[..., 0] + ky * d[..., 1]) * b / k) @ q
    zero = (np.exp(-(xi * z) ** 2) / xi + math.sqrt(math.pi) * z * _erf(xi * z)) @ q
    return (np.pi / L ** 2) * out - (2 * math.sqrt(math.pi) / L ** 2) * zero


def direct_kspace_0p(pos, q, xi, targets=None):
    """sum_{n != m} q_n erf(xi r)/r + q_m 2 xi / sqrt(pi) (oracle.py:181-192)."""
    pos = np.asarray(pos, float)
    tg = np.arange(len(pos)) if targets is None else np.asarray(targets)
    d = pos[tg, None, :] - pos[None, :, :]
    r = np.sqrt(np.sum(d * d, axis=2))
    same = tg[:, None] == np.arange(len(pos))[None, :]
    if np.any((r < 1e-14) & ~same):
        raise ValueError("coincident distinct particles")
    with np.errstate(divide="ignore", invalid="ignore"):
        kern = np.where(same, 0.0, _erf(xi * r) / r)
    return kern @ q + q[tg] * (2.0 * xi / math.sqrt(math.pi))


def relative_rms(phi, ref):
    """core.py:156-165."""
    phi = np.asarray(phi, dtype=complex)
    ref = np.asarray(ref, dtype=complex)
    return float(np.sqrt(np.mean(np.abs(phi - ref) ** 2)) / np.sqrt(np.mean(np.abs(ref) ** 2)))


# ------------------------------------------------------------ field (forces)
# Beyond the reference, which stops at potentials (SURVEY 8f
# item 4).  Pinned by central differences of the reference's own
# real_space_sum (realspace.py:168-180) and oracle.kspace_direct_3p
# (oracle.py:109-118): tests/golden/make_golden.py -> field.npz.

def realspace_field(pos, q, L, D, xi, rc, targets=None):
    """E_R(x_t) = sum q_s (erfc(xi r)/r + 2 xi/sqrt(pi) e^{-xi^2 r^2}) d / r^2,
    d = x_t - x_s over the same pair set as realspace(): minimum image when
    rc <= L/2 on the periodic axes, explicit images otherwise.  Brute force
    over all sources (test sizes)."""
    N = len(q)
    tsel = np.arange(N) if targets is None else np.asarray(targets)
    per = np.array([a < D for a in range(3)])
    c = 2.0 * xi / math.sqrt(math.pi)

    def block(xt, xs, same=None):
        d = xt[:, None, :] - xs[None, :, :]
        r = np.sqrt(np.sum(d * d, axis=2))
        zero = r < 1e-14
        if same is not None and np.any(zero & ~same):
            raise SingularConfigurationError_("coincident distinct particles")
        use = (r < rc) & ~zero
        rs = np.where(use, r, 1.0)
        g = np.where(use, (_erfc(xi * rs) / rs + c * np.exp(-(xi * rs) ** 2)) / rs ** 2, 0.0) * q[None, :]
        return np.einsum("ts,tsa->ta", g, d)

    out = np.zeros((len(tsel), 3))
    for i0 in range(0, len(tsel), 256):
        ti = tsel[i0:i0 + 256]
        same = ti[:, None] == np.arange(N)[None, :]
        if D >= 1 and rc > L / 2 + 1e-12:
            layers = int(np.floor((rc + L / 2) / L)) + 1
            rng = [np.arange(-layers, layers + 1) if per[a] else np.array([0]) for a in range(3)]
            for a in rng[0]:
                for b in rng[1]:
                    for cc in rng[2]:
                        sh = np.array([a, b, cc], float) * L
                        out[i0:i0 + 256] += block(pos[ti], pos - sh, same if (a == b == cc == 0) else None)
        else:
            d = pos[ti][:, None, :] - pos[None, :, :]
            d -= per[None, None, :] * L * np.rint(d / L)
            out[i0:i0 + 256] += _field_from_disp(d, q, xi, rc, c, same)
    return out


def _field_from_disp(d, q, xi, rc, c, same):
    r = np.sqrt(np.sum(d * d, axis=2))
    zero = r < 1e-14
    if np.any(zero & ~same):
        raise SingularConfigurationError_("coincident distinct particles")
    use = (r < rc) & ~zero
    rs = np.where(use, r, 1.0)
    g = np.where(use, (_erfc(xi * rs) / rs + c * np.exp(-(xi * rs) ** 2)) / rs ** 2, 0.0) * q[None, :]
    return np.einsum("ts,tsa->ta", g, d)


def kspace_field_d3(pos, q, L, prm, targets=None):
    """E_F = gather(IFFT(-i k_a Phi)), Phi the scaled spectrum of kspace_d3
    (aft.py:203-206 + sekspace.py:198-206); the Nyquist index of the
    differentiated axis is zeroed (real output)."""
    g = geometry(L, 3, prm["M"], prm["P"])
    kind, shape, xi = prm["window"], prm["shape"], prm["xi"]
    H = spread(pos, q, g, kind, shape)
    M, w = g["M"], 0.5 * g["P"] * g["h"]
    k = wavenumbers(M, g["h"])
    wh = window_fourier_checked(kind, shape, w, k)
    k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    inv = np.zeros_like(k2)
    inv[k2 > 0] = 1.0 / k2[k2 > 0]
    W = wh[:, None, None] * wh[None, :, None] * wh[None, None, :]
    F = np.fft.fftn(H) * (FOUR_PI * _mollify(k2, xi) * inv / W ** 2)
    kd = k.copy()
    kd[M // 2] = 0.0
    tpos = pos if targets is None else pos[np.asarray(targets)]
    out = np.zeros((len(tpos), 3))
    for a in range(3):
        shp = [1, 1, 1]
        shp[a] = M
        Ea = np.fft.ifftn(-1j * kd.reshape(shp) * F).real
        out[:, a] = gather(Ea, tpos, g, kind, shape)
    return out


def window_deriv(kind, shape, w, x):
    """d/dx of window_eval (windows.py:74-84, 106-112): Gaussian
    -m^2 x / w^2 w(x); Kaiser-Bessel -beta I1(beta s) r / (w s I0(beta)),
    s = sqrt(1 - r^2), r = x / w (finite at the edge).  Not for the ES
    window (singular derivative at the support edge)."""
    from scipy.special import i1 as _i1

    x = np.asarray(x, dtype=float)
    inside = np.abs(x) <= w
    if kind == "gaussian":
        v = -(shape * shape) * x / (w * w) * window_eval(kind, shape, w, x)
    elif kind == "kb":
        r = x / w
        sq = np.sqrt(np.clip(1.0 - r * r, 0.0, None))
        i1s = np.where(sq > 1e-8, _i1(shape * sq) / np.where(sq > 1e-8, sq, 1.0), 0.5 * shape)
        v = -shape * i1s * r / w / _i0(shape)
    else:
        raise ValueError("the window-gradient field needs the Gaussian or Kaiser-Bessel window")
    return np.where(inside, v, 0.0)


def kspace_field_grad(pos, q, L, D, prm, targets=None, use_kernel=None):
    """E_F = -grad phi_F for any D by the gradient of the gather: the filtered
    grid H~ of se_kspace (sekspace.py:340-381) and
    E_a(x) = h^3 sum_g H~[g] w'(delta_a) prod_{b != a} w(delta_b),
    delta = g h - (x + offset) (the derivative of gather, sekspace.py:159-178,
    with respect to the particle position)."""
    g = geometry(L, D, prm["M"], prm["P"], prm.get("s0", 1.0), prm.get("s", 1.0), prm.get("R", 0.0))
    kind, shape, xi = prm["window"], prm["shape"], prm["xi"]
    H = spread(pos, q, g, kind, shape)
    if D == 3:
        Ht = kspace_d3(H, g, xi, kind, shape)
    elif D == 0 and (use_kernel or use_kernel is None):
        tab, kg = d0_kernel_table(L, prm["M"], prm["P"], prm["s0"], prm["rc"])
        Ht = kspace_d0_kernel(H, g, xi, kind, shape, tab, kg["nconv"])
    else:
        Ht = kspace_mixed(H, g, xi, kind, shape, prm["nI"])
    tpos = pos if targets is None else pos[np.asarray(targets)]
    P, h = g["P"], g["h"]
    w = 0.5 * P * h
    t = np.arange(P)
    idx, wv, dv = [], [], []
    for a in range(3):
        u = tpos[:, a] + g["offsets"][a]
        first = np.floor(u / h - 0.5 * P).astype(np.int64) + 1
        ia = first[:, None] + t[None, :]
        d = ia * h - u[:, None]
        if a < D:
            ia = np.mod(ia, g["M"])
        idx.append(ia)
        wv.append(window_eval(kind, shape, w, d))
        dv.append(window_deriv(kind, shape, w, d))
    v = Ht[idx[0][:, :, None, None], idx[1][:, None, :, None], idx[2][:, None, None, :]]
    ex = np.einsum("npqr,np,nq,nr->n", v, dv[0], wv[1], wv[2])
    ey = np.einsum("npqr,np,nq,nr->n", v, wv[0], dv[1], wv[2])
    ez = np.einsum("npqr,np,nq,nr->n", v, wv[0], wv[1], dv[2])
    return np.stack([ex, ey, ez], axis=1) * h ** 3


def total_field(pos, q, L, prm):
    """E = E_R + E_F (D = 3)."""
    return realspace_field(pos, q, L, 3, prm["xi"], prm["rc"]) + kspace_field_d3(pos, q, L, prm)


def direct_field_3p(pos, q, L, xi, kmax, targets=None):
    """-grad of direct_kspace_3p at the targets: (4 pi / L^3) sum_k
    e^{-k^2/4xi^2}/k^2 k Im(e^{i k.x_m} S_k)."""
    pos = np.asarray(pos, float)
    tg = np.arange(len(pos)) if targets is None else np.asarray(targets)
    n = np.arange(-kmax, kmax + 1)
    c = 2.0 * np.pi / L
    ex, ey, ez = (np.exp(-1j * c * np.outer(pos[:, a], n)) for a in range(3))
    out = np.zeros((len(tg), 3))
    for i1, n1 in enumerate(n):
        S = np.einsum("n,nb,nc->bc", q * ex[:, i1], ey, ez)
        k2 = c * c * (n1 * n1 + n[:, None] ** 2 + n[None, :] ** 2)
        with np.errstate(divide="ignore", invalid="ignore"):
            coef = np.where(k2 > 0, np.exp(-k2 / (4.0 * xi * xi)) / k2, 0.0)
        E = np.einsum("t,tb,tc->tbc", np.conj(ex[tg, i1]), np.conj(ey[tg]), np.conj(ez[tg]))
        im = np.imag(E * S[None]) * coef[None]
        out[:, 0] += c * n1 * im.sum(axis=(1, 2))
        out[:, 1] += c * np.einsum("tbc,b->t", im, n.astype(float))
        out[:, 2] += c * np.einsum("tbc,c->t", im, n.astype(float))
    return out * (FOUR_PI / L ** 3)
