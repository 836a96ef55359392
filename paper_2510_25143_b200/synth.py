"""Seeded synthetic stand-ins for the five BASELINE.json configurations.

The paper's datasets (SCF/CFVKV/HCBA/FS) are not
available; SURVEY.md §8(d) specifies generators with the same shapes, sizes
and value distributions.  Conventions:
  * float64 generation, cast to float32; dx = dy = dt = 1;
  * numpy.random.default_rng(seed = config index), draws in listed order;
  * x = column j (u), y = row i (v); "N x M grid" is W x H.

Each generator returns (H, W, T, u, v) with u, v float32 of length H*W*T in
the reference's VID(t,i,j) = t*H*W + i*W + j order (field.py:4-5).
`scale_down` shrinks a config for parity tests (same generator, smaller
grid/frames).
"""

from __future__ import annotations

import numpy as np

# (H, W, T, eps_rel list) per BASELINE.json configs[0..4]
CONFIGS = {
    1: dict(H=128, W=128, T=32, eps=(1e-2,)),
    2: dict(H=512, W=512, T=100, eps=(1e-3,)),
    3: dict(H=256, W=1024, T=200, eps=(1e-2, 1e-3)),
    4: dict(H=2400, W=3600, T=24, eps=(1e-3,)),
    5: dict(H=8192, W=8192, T=16, eps=(1e-2, 1e-3, 1e-4)),
}


def _vortices(H, W, T, rng):
    """Config 1: 4 Gaussian vortices drifting over background (0.2, 0.1)."""
    nv = 4
    cx = rng.uniform(0.0, W, nv)
    cy = rng.uniform(0.0, H, nv)
    R = rng.uniform(6.0, 12.0, nv)
    G = rng.uniform(0.5, 1.5, nv) * rng.choice((-1.0, 1.0), nv)
    drift = rng.uniform(-0.5, 0.5, (nv, 2))
    jj, ii = np.meshgrid(np.arange(W, dtype=np.float64),
                         np.arange(H, dtype=np.float64))
    u = np.empty((T, H, W), np.float32)
    v = np.empty((T, H, W), np.float32)
    for t in range(T):
        uu = np.full((H, W), 0.2)
        vv = np.full((H, W), 0.1)
        for k in range(nv):
            x0 = cx[k] + drift[k, 0] * t
            y0 = cy[k] + drift[k, 1] * t
            dxk = jj - x0
            dyk = ii - y0
            g = (G[k] / R[k]) * np.exp(0.5 * (1.0 - (dxk * dxk + dyk * dyk)
                                             / (R[k] * R[k])))
            uu += g * (-dyk)
            vv += g * dxk
        uu += rng.normal(0.0, 1e-3, (H, W))
        vv += rng.normal(0.0, 1e-3, (H, W))
        u[t] = uu
        v[t] = vv
    return u, v


def _spectral(H, W, T, rng, U=(0.7, 0.3), kmax=64, drift=0.02):
    """Configs 2 and 5: k^-3 random-phase stream function, frozen turbulence
    advected by the mean flow with a slow phase drift."""
    ky = np.fft.fftfreq(H, 1.0 / H)[:, None]          # integer wavenumbers
    kx = np.fft.rfftfreq(W, 1.0 / W)[None, :]
    kk = np.sqrt(kx * kx + ky * ky)
    band = (kk >= 1.0) & (kk <= kmax)
    phase = rng.uniform(0.0, 2.0 * np.pi, kk.shape)
    amp = np.zeros(kk.shape)
    amp[band] = kk[band] ** -3.0
    psi0 = amp * np.exp(1j * phase)
    # restrict work to the band (the spectrum is zero elsewhere)
    rows = np.flatnonzero(band.any(axis=1))
    cols = np.flatnonzero(band.any(axis=0))
    sub = np.ix_(rows, cols)
    psi_b = psi0[sub]
    kx_b = np.broadcast_to(kx, kk.shape)[sub]
    ky_b = np.broadcast_to(ky, kk.shape)[sub]
    u = np.empty((T, H, W), np.float32)
    v = np.empty((T, H, W), np.float32)
    scale = None
    for t in range(T):
        ph = np.exp(-2j * np.pi * (kx_b * U[0] * t / W + ky_b * U[1] * t / H)
                    + 1j * drift * t)
        spec = np.zeros(kk.shape, np.complex128)
        spec[sub] = psi_b * ph
        # u' = d psi / dy (y = row), v' = -d psi / dx
        du = np.fft.irfft2(spec * (2j * np.pi * ky / H), s=(H, W))
        dv = -np.fft.irfft2(spec * (2j * np.pi * kx / W), s=(H, W))
        if scale is None:
            rms = np.sqrt(np.mean(du * du + dv * dv))
            scale = 1.0 / rms if rms > 0 else 1.0
        u[t] = U[0] + scale * du
        v[t] = U[1] + scale * dv
    return u, v


def _wake(H, W, T, rng):
    """Config 3: parabolic inflow + alternating Rankine vortex street."""
    jj, ii = np.meshgrid(np.arange(W, dtype=np.float64),
                         np.arange(H, dtype=np.float64))
    yp = ii / (H - 1)
    base_u = 4.0 * yp * (1.0 - yp)
    a = 8.0
    u = np.empty((T, H, W), np.float32)
    v = np.empty((T, H, W), np.float32)
    for t in range(T):
        uu = base_u.copy()
        vv = np.zeros((H, W))
        # vortex k sits at x_k(t) = 64 + 0.8 t - 48 k and is present while
        # 64 <= x_k <= W + 24; k <= 0 is the street already shed at t = 0
        k_hi = int(np.floor(0.8 * t / 48.0))
        k_lo = int(np.ceil((64.0 + 0.8 * t - (W + 24.0)) / 48.0))
        for k in range(k_lo, k_hi + 1):
            xk = 64.0 + 0.8 * t - 48.0 * k
            if not (64.0 <= xk <= W + 24.0):
                continue
            s = 1.0 if k % 2 == 0 else -1.0
            yk = (H - 1) / 2.0 + s * 0.15 * H
            dx = jj - xk
            dy = ii - yk
            r = np.sqrt(dx * dx + dy * dy)
            vt = np.where(r < a, r / a, a / np.maximum(r, 1e-300))
            inv = np.where(r > 0, 1.0 / np.maximum(r, 1e-300), 0.0)
            uu += s * vt * (-dy) * inv
            vv += s * vt * dx * inv
        uu += rng.normal(0.0, 1e-4, (H, W))
        vv += rng.normal(0.0, 1e-4, (H, W))
        u[t] = uu
        v[t] = vv
    return u, v


def _eddies(H, W, T, rng, n_eddy=2000):
    """Config 4: Gaussian eddies with random-walking centres."""
    cx = rng.uniform(0.0, W, n_eddy)
    cy = rng.uniform(0.0, H, n_eddy)
    R = rng.uniform(5.0, 40.0, n_eddy)
    A = rng.uniform(0.05, 1.0, n_eddy) * rng.choice((-1.0, 1.0), n_eddy)
    u = np.empty((T, H, W), np.float32)
    v = np.empty((T, H, W), np.float32)
    for t in range(T):
        uu = np.zeros((H, W))
        vv = np.zeros((H, W))
        for k in range(n_eddy):
            r4 = 4.0 * R[k]
            i0 = max(0, int(np.floor(cy[k] - r4)))
            i1 = min(H, int(np.ceil(cy[k] + r4)) + 1)
            j0 = max(0, int(np.floor(cx[k] - r4)))
            j1 = min(W, int(np.ceil(cx[k] + r4)) + 1)
            if i0 >= i1 or j0 >= j1:
                continue
            ii = np.arange(i0, i1, dtype=np.float64)[:, None] - cy[k]
            jj = np.arange(j0, j1, dtype=np.float64)[None, :] - cx[k]
            g = (A[k] / R[k]) * np.exp(0.5 * (1.0 - (ii * ii + jj * jj)
                                             / (R[k] * R[k])))
            uu[i0:i1, j0:j1] += g * (-ii)
            vv[i0:i1, j0:j1] += g * jj
        u[t] = uu
        v[t] = vv
        cx += rng.normal(0.0, 0.5, n_eddy)
        cy += rng.normal(0.0, 0.5, n_eddy)
    return u, v


def generate(cfg: int, H: int | None = None, W: int | None = None,
             T: int | None = None, n_eddy: int | None = None):
    """Field of config `cfg` (1..5), optionally at a reduced size.

    Returns (H, W, T, u, v) with flat float32 u, v."""
    spec = CONFIGS[cfg]
    H = spec["H"] if H is None else H
    W = spec["W"] if W is None else W
    T = spec["T"] if T is None else T
    rng = np.random.default_rng(cfg)
    if cfg == 1:
        u, v = _vortices(H, W, T, rng)
    elif cfg == 2:
        u, v = _spectral(H, W, T, rng, U=(0.7, 0.3))
    elif cfg == 3:
        u, v = _wake(H, W, T, rng)
    elif cfg == 4:
        if n_eddy is None:
            # keep eddy density of the full config when reduced
            n_eddy = max(8, int(round(2000 * (H * W) / (2400 * 3600))))
        u, v = _eddies(H, W, T, rng, n_eddy)
    elif cfg == 5:
        u, v = _spectral(H, W, T, rng, U=(1.3, -0.6))
    else:
        raise ValueError(f"unknown config {cfg}")
    return H, W, T, u.reshape(-1), v.reshape(-1)
