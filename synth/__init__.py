"""Seeded synthetic inputs shaped like the paper's wide-field workloads.

This module is the ONLY code shared by the CUDA path's callers (bench.py, the
GPU tests) and by the fp64 oracle's callers (tests, cpu_baseline).  It holds
none of the method's arithmetic: no blur operator H / H^T, no regulariser, no
consensus.  It produces the *inputs* of deblur_create():

  * a PSF grid h_k (P x P, odd P, unit sum in fp64, stored fp32)  -- PAPER.md:106-107
  * first-order (bilinear-hat) interpolation weights wy[G_y][N_y], wx[G_x][N_x]
    whose products are the omega_k of PAPER.md:107 (ramp in [0,1] between
    adjacent equidistant grid points, partition of unity)
  * an observed image y (M x M, M = N - P + 1, PAPER.md:61 footnote) and the
    diagonal data weights W = 1/sigma^2
  * the solver parameters of BASELINE.json configs[0..4].

The paper measures on photographs that are not in this container
(PAPER.md:268, :270, :376).  Per BASELINE.json the stand-ins are seeded star
fields.  The observed image is rendered *analytically*: a Gaussian source of
width s seen through a PSF whose Gaussian-equivalent width at that field
position is p is a Gaussian of width sqrt(s^2 + p^2) (exact for Gaussian
PSFs, a stand-in for Moffat wings).  No blur operator is applied, so y never
depends on either implementation under test.  The recipe is in DESIGN.md §3.

Seeds: numpy PCG64 with SeedSequence(1000*k).spawn(4) -> [sources, galaxies,
PSF jitter, noise] for config k.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional

import numpy as np

__all__ = ["Problem", "CONFIGS", "make_config", "make_problem", "per_node", "hat_weights",
           "psf_grid", "render_observed", "render_scene", "input_hash"]


@dataclasses.dataclass
class Problem:
    name: str
    ny: int
    nx: int
    P: int
    gy: int
    gx: int
    psfs: np.ndarray          # [gy*gx, P, P] float32, k = p*gx + q
    wy: np.ndarray            # [gy, ny] float32
    wx: np.ndarray            # [gx, nx] float32
    y: np.ndarray             # [my, mx] float32
    noise_w: Optional[np.ndarray]   # [my, mx] float32 or None
    noise_w_scalar: float
    lam: float = 0.01
    eps: float = 1e-3
    gamma: float = 4000.0
    rho: float = 1.0
    reg_kind: int = 0
    tv_boundary: int = 0
    inner_steps: int = 1
    fy: int = 1
    fx: int = 1
    overlap: int = 0
    iters: int = 20
    x0: Optional[np.ndarray] = None
    operator_mode: int = 0    # 0: interpolated H restricted to facets; 1: per-node PSFs
    independent: int = 0      # 1: the paper's independent baseline (no consensus, alpha = 0)
    local_solver: int = 0     # 0: projected gradient (inner_steps); 1: VMLM-B (budget inner_steps + k inner_increment)
    inner_increment: int = 0

    @property
    def my(self) -> int:
        return self.ny - self.P + 1

    @property
    def mx(self) -> int:
        return self.nx - self.P + 1

    def w_array(self) -> np.ndarray:
        if self.noise_w is not None:
            return self.noise_w
        return np.full((self.my, self.mx), self.noise_w_scalar, np.float32)


# BASELINE.json configs[0..4] (c1..c5).  n = scene/estimate side.
CONFIGS = {
    1: dict(n=256, P=15, G=2, psf="gauss_axis", sources=200, galaxies=0,
            noise=("gauss", 0.01), facets=(1, 1), overlap=0, iters=20),
    2: dict(n=1024, P=31, G=4, psf="gauss_radial", sources=2000, galaxies=0,
            noise=("gauss", 0.01), facets=(2, 2), overlap=64, iters=100),
    3: dict(n=4096, P=63, G=8, psf="gauss_moffat", sources=30000, galaxies=2000,
            noise=("poisson_gauss", 0.005), facets=(2, 4), overlap=128, iters=100),
    4: dict(n=16384, P=63, G=16, psf="moffat_radial", sources=500000, galaxies=0,
            noise=("gauss", 0.005), facets=(4, 2), overlap=128, iters=50),
    5: dict(n=32768, P=127, G=32, psf="moffat_elliptic", sources=2000000, galaxies=0,
            noise=("gauss", 0.005), facets=(8, 8), overlap=192, iters=20),
    # c6: the paper's shift-variant experiment shape (SURVEY §8d
    # "optional paper-shaped config", NEXT-4): 1151 x 1407 at 6000 photons/pixel, sigma^2 =
    # 400, 9 x 9 Gaussian PSFs of 201 x 201, Huber delta = 100, lambda = 0.002, gamma =
    # 0.4 W = 0.001, 25 iterations; a star field stands in for the photograph.
    6: dict(n=1151, nx=1407, P=201, G=9, psf="paper_gauss", sources=3000, galaxies=300,
            noise=("gauss", 20.0), scale=6000.0, facets=(3, 3), overlap=64, iters=25,
            reg_kind=1, eps=100.0, lam=0.002),
}

GAIN_E = 1000.0     # Poisson gain for the mixed-noise config
READ_SIGMA = 0.005  # read-noise sigma


def hat_weights(n: int, G: int) -> np.ndarray:
    """First-order interpolation hats on n pixels for G equidistant grid points.

    Grid points at cell centres C_p = (p + 0.5) n / G; the hat of
    point p is a ramp in [0, 1] to its neighbours (Fig. 1 caption
    PAPER.md:239), clamped to 1 beyond the outermost points, so
    the hats form a partition of unity.  Returns float64 [G, n].
    """
    t = np.arange(n, dtype=np.float64)
    if G == 1:
        return np.ones((1, n))
    L = n / G
    C = (np.arange(G) + 0.5) * L
    w = np.maximum(0.0, 1.0 - np.abs(t[None, :] - C[:, None]) / L)
    w[0, t <= C[0]] = 1.0
    w[G - 1, t >= C[G - 1]] = 1.0
    return w


def _rhat(G: int) -> np.ndarray:
    """Radius of each PSF-cell centre from the field centre / corner-cell radius."""
    c = (np.arange(G) + 0.5) / G - 0.5
    r = np.sqrt(c[:, None] ** 2 + c[None, :] ** 2)
    rmax = r.max()
    return r / rmax if rmax > 0 else np.zeros_like(r)


def _angle(G: int) -> np.ndarray:
    c = (np.arange(G) + 0.5) / G - 0.5
    return np.arctan2(c[:, None] * np.ones((1, G)), np.ones((G, 1)) * c[None, :])


def _moffat_alpha(fwhm: float, beta: float) -> float:
    return fwhm / (2.0 * math.sqrt(2.0 ** (1.0 / beta) - 1.0))


def psf_grid(kind: str, G: int, P: int, rng: np.random.Generator):
    """Returns (psfs fp64 [G*G, P, P] normalised to unit sum, sigma_eq [G, G]).

    sigma_eq is the Gaussian-equivalent width (FWHM / 2.3548) used only by the
    analytic renderer of the observed image.
    """
    c = (P - 1) // 2
    a = np.arange(P, dtype=np.float64) - c
    Y, X = np.meshgrid(a, a, indexing="ij")
    rh = _rhat(G)
    ang = _angle(G)
    out = np.zeros((G * G, P, P))
    sig = np.zeros((G, G))
    for p in range(G):
        for q in range(G):
            if kind == "gauss_axis":     # c1: sigma in [1.0, 2.5], axis aligned
                sx = 1.0 + 1.5 * q / max(G - 1, 1)
                sy = 1.0 + 1.5 * p / max(G - 1, 1)
                h = np.exp(-0.5 * ((X / sx) ** 2 + (Y / sy) ** 2))
                s_eq = math.sqrt(sx * sy)
            elif kind == "gauss_radial":  # c2: elongated along the radius
                r = rh[p, q]
                smaj = 1.5 + 1.0 * r
                smin = smaj * (1.0 - 0.4 * r)
                th = ang[p, q]
                u = X * math.cos(th) + Y * math.sin(th)
                v = -X * math.sin(th) + Y * math.cos(th)
                h = np.exp(-0.5 * ((u / smaj) ** 2 + (v / smin) ** 2))
                s_eq = math.sqrt(smaj * smin)
            elif kind == "gauss_moffat":  # c3: Gaussian core + Moffat wings
                r = rh[p, q]
                sc = 1.2 + 0.8 * r
                beta = 3.0
                al = 2.0 * sc
                g = np.exp(-0.5 * (X ** 2 + Y ** 2) / sc ** 2)
                g /= g.sum()
                m = (1.0 + (X ** 2 + Y ** 2) / al ** 2) ** (-beta)
                m /= m.sum()
                h = 0.8 * g + 0.2 * m
                s_eq = sc * 1.15
            elif kind == "moffat_radial":  # c4: FWHM grows 2x radially
                r = rh[p, q]
                beta = 3.0
                fwhm = 3.0 * (1.0 + r)
                al = _moffat_alpha(fwhm, beta)
                h = (1.0 + (X ** 2 + Y ** 2) / al ** 2) ** (-beta)
                s_eq = fwhm / 2.3548
            elif kind == "moffat_elliptic":  # c5
                r = rh[p, q]
                beta = 3.0
                fwhm = 4.0 * (1.0 + 0.5 * r)
                e = 0.3 * r
                th = ang[p, q] + math.radians(10.0) * rng.standard_normal()
                al = _moffat_alpha(fwhm, beta)
                u = X * math.cos(th) + Y * math.sin(th)
                v = -X * math.sin(th) + Y * math.cos(th)
                h = (1.0 + (u / al) ** 2 + (v / (al * (1.0 - e))) ** 2) ** (-beta)
                s_eq = fwhm * math.sqrt(1.0 - e) / 2.3548
            elif kind == "paper_gauss":  # c6: FWHM 3.5 x 3.5 at the centre, growing
                r = rh[p, q]               # linearly with the radius to 16.5 x 10.5 at the corners (coma-like)
                fmaj, fmin = 3.5 + 13.0 * r, 3.5 + 7.0 * r
                smaj, smin = fmaj / 2.3548, fmin / 2.3548
                th = ang[p, q]
                u = X * math.cos(th) + Y * math.sin(th)
                v = -X * math.sin(th) + Y * math.cos(th)
                h = np.exp(-0.5 * ((u / smaj) ** 2 + (v / smin) ** 2))
                s_eq = math.sqrt(smaj * smin)
            else:
                raise ValueError(kind)
            out[p * G + q] = h / h.sum()
            sig[p, q] = s_eq
    return out, sig


def _splat(img: np.ndarray, rows: np.ndarray, cols: np.ndarray, amp: np.ndarray,
           s2: np.ndarray, R: int, band: int = 512, chunk: int = 20000):
    """Accumulate isotropic Gaussians amp*exp(-d^2/(2 s2)) into img (in place),
    stamps of radius R, using per-row-band bincount (no Python per-source loop)."""
    H, W = img.shape
    order = np.argsort(rows, kind="stable")
    rows, cols, amp, s2 = rows[order], cols[order], amp[order], s2[order]
    off = np.arange(-R, R + 1)
    bh = band + 2 * R + 2
    for b0 in range(0, H, band):
        lo = np.searchsorted(rows, b0 - 0.5)
        hi = np.searchsorted(rows, b0 + band - 0.5)
        if hi <= lo:
            continue
        buf = np.zeros(bh * W)
        for s in range(lo, hi, chunk):
            e = min(hi, s + chunk)
            r, c_, A, v = rows[s:e], cols[s:e], amp[s:e], s2[s:e]
            ri = np.floor(r).astype(np.int64)
            ci = np.floor(c_).astype(np.int64)
            pr = ri[:, None] + off[None, :]            # (n, S)
            pc = ci[:, None] + off[None, :]
            dr = (pr - r[:, None]) ** 2
            dc = (pc - c_[:, None]) ** 2
            val = A[:, None, None] * np.exp(-(dr[:, :, None] + dc[:, None, :]) / (2 * v[:, None, None]))
            br = pr - (b0 - R - 1)                     # row in buffer
            ok = (pc[:, None, :] >= 0) & (pc[:, None, :] < W) & (pr[:, :, None] >= 0) & (pr[:, :, None] < H)
            idx = br[:, :, None] * W + pc[:, None, :]
            buf += np.bincount(idx[ok], weights=val[ok], minlength=bh * W)
        buf = buf.reshape(bh, W)
        r0 = b0 - R - 1
        a0, a1 = max(0, r0), min(H, r0 + bh)
        img[a0:a1] += buf[a0 - r0:a1 - r0]


def _local_sigma(sig: np.ndarray, wy: np.ndarray, wx: np.ndarray, r: np.ndarray, c: np.ndarray):
    """Gaussian-equivalent PSF width at estimate positions (r, c), interpolated
    with the same hats (renderer only)."""
    ri = np.clip(np.round(r).astype(np.int64), 0, wy.shape[1] - 1)
    ci = np.clip(np.round(c).astype(np.int64), 0, wx.shape[1] - 1)
    return np.einsum("pn,pq,qn->n", wy[:, ri], sig, wx[:, ci])


def render_observed(n: int, P: int, sig: np.ndarray, wy: np.ndarray, wx: np.ndarray,
                    n_src: int, n_gal: int, rng_src, rng_gal, nx: Optional[int] = None) -> np.ndarray:
    """Noiseless observed image (M_y x M_x, fp64) of a star field (+ galaxies) seen
    through the PSF grid, rendered analytically (see module docstring).  The scene
    is n x nx (nx = n if not given)."""
    ny = n
    nx = n if nx is None else nx
    c = (P - 1) // 2
    My, Mx = ny - P + 1, nx - P + 1
    img = np.zeros((My, Mx))
    # smooth background 0.05 + 0.02*(c1 u + c2 v + c3 uv + c4 u^2 + c5 v^2), clipped >= 0
    cc = rng_src.uniform(-1, 1, 5)
    U = np.linspace(-1, 1, nx)[c:c + Mx][None, :]
    V = np.linspace(-1, 1, ny)[c:c + My][:, None]
    img += np.maximum(0.0, 0.05 + 0.02 * (cc[0] * U + cc[1] * V + cc[2] * U * V + cc[3] * U ** 2 + cc[4] * V ** 2))
    # point sources: position U[0,n)^2 (estimate coords), peak U(0.2,1), sigma U(0.5,1.5)
    pr = rng_src.uniform(0, ny, n_src)
    pc = rng_src.uniform(0, nx, n_src)
    amp = rng_src.uniform(0.2, 1.0, n_src)
    ss = rng_src.uniform(0.5, 1.5, n_src)
    sp = _local_sigma(sig, wy, wx, pr, pc)
    s2 = ss ** 2 + sp ** 2
    A = amp * ss ** 2 / s2                       # flux-conserving peak after blur
    R = int(math.ceil(4.0 * math.sqrt(s2.max())))
    _splat(img, pr - c, pc - c, A, s2, R)
    # extended elliptical galaxies (c3): sigma_major U(2,12), ratio U(0.3,1), angle U(0,pi), peak U(0.02,0.3)
    for _ in range(n_gal):
        gr, gc = rng_gal.uniform(0, ny), rng_gal.uniform(0, nx)
        smaj = rng_gal.uniform(2, 12)
        smin = smaj * rng_gal.uniform(0.3, 1.0)
        th = rng_gal.uniform(0, math.pi)
        pk = rng_gal.uniform(0.02, 0.3)
        spv = float(_local_sigma(sig, wy, wx, np.array([gr]), np.array([gc]))[0])
        cth, sth = math.cos(th), math.sin(th)
        Sg = np.array([[cth, -sth], [sth, cth]]) @ np.diag([smaj ** 2, smin ** 2]) @ np.array([[cth, sth], [-sth, cth]])
        St = Sg + spv ** 2 * np.eye(2)
        peak = pk * math.sqrt(np.linalg.det(Sg) / np.linalg.det(St))
        Si = np.linalg.inv(St)
        Rg = int(math.ceil(4.0 * math.sqrt(max(np.linalg.eigvalsh(St)))))
        r0, c0 = gr - c, gc - c
        i0, i1 = max(0, int(r0) - Rg), min(My, int(r0) + Rg + 1)
        j0, j1 = max(0, int(c0) - Rg), min(Mx, int(c0) + Rg + 1)
        if i0 >= i1 or j0 >= j1:
            continue
        dy = np.arange(i0, i1)[:, None] - r0
        dx = np.arange(j0, j1)[None, :] - c0
        q = Si[0, 0] * dy * dy + 2 * Si[0, 1] * dy * dx + Si[1, 1] * dx * dx
        img[i0:i1, j0:j1] += peak * np.exp(-0.5 * q)
    return img


def render_scene(n: int, n_src: int, seed: int) -> np.ndarray:
    """Unblurred non-negative star-field scene (N x N, fp64) for pins that need a
    ground truth x* (tests only)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    img = np.full((n, n), 0.05)
    pr = rng.uniform(0, n, n_src)
    pc = rng.uniform(0, n, n_src)
    amp = rng.uniform(0.2, 1.0, n_src)
    ss = rng.uniform(0.5, 1.5, n_src)
    _splat(img, pr, pc, amp, ss ** 2, int(math.ceil(4 * 1.5)))
    return img


def make_problem(name: str, n: int, P: int, G: int, psf: str, sources: int, galaxies: int,
                 noise, facets, overlap: int, iters: int, seed: int, nx: Optional[int] = None,
                 lam: float = 0.01, eps: float = 1e-3, rho: float = 1.0, inner_steps: int = 1,
                 reg_kind: int = 0, tv_boundary: int = 0, gamma: Optional[float] = None,
                 Gx: Optional[int] = None, scale: float = 1.0) -> Problem:
    ny = n
    nx = n if nx is None else nx
    Gy = G
    Gx = G if Gx is None else Gx
    ss = np.random.SeedSequence(seed)
    rng_src, rng_gal, rng_psf, rng_noise = [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(4)]
    psfs64, sig = psf_grid(psf, max(Gy, Gx), P, rng_psf)
    if Gy != Gx:   # rectangular grids: take the leading Gy x Gx block of a square grid
        Gm = max(Gy, Gx)
        idx = [p * Gm + q for p in range(Gy) for q in range(Gx)]
        psfs64 = psfs64[idx]
        sig = sig[:Gy, :Gx]
    wy64 = hat_weights(ny, Gy)
    wx64 = hat_weights(nx, Gx)
    # scale: photons per unit of the star-field intensity (the paper's 6000-photon images)
    clean = scale * render_observed(n, P, sig, wy64, wx64, sources, galaxies, rng_src, rng_gal, nx=nx)
    kind, sigma = noise
    if kind == "gauss":
        y = clean + sigma * rng_noise.standard_normal(clean.shape)
        noise_w = None
        w_scalar = 1.0 / sigma ** 2
        med_w = w_scalar
    elif kind == "poisson_gauss":
        y = rng_noise.poisson(GAIN_E * np.maximum(clean, 0.0)) / GAIN_E
        y = y + READ_SIGMA * rng_noise.standard_normal(clean.shape)
        noise_w = (1.0 / (READ_SIGMA ** 2 + np.maximum(y, 0.0) / GAIN_E)).astype(np.float32)
        w_scalar = 0.0
        med_w = float(np.median(noise_w))
    else:
        raise ValueError(kind)
    if gamma is None:
        gamma = 0.4 * med_w     # keep the paper's gamma/W ratio (0.001 / (1/400))
    return Problem(name=name, ny=ny, nx=nx, P=P, gy=Gy, gx=Gx,
                   psfs=psfs64.astype(np.float32), wy=wy64.astype(np.float32),
                   wx=wx64.astype(np.float32), y=y.astype(np.float32), noise_w=noise_w,
                   noise_w_scalar=float(w_scalar), lam=lam, eps=eps, gamma=float(gamma), rho=rho,
                   reg_kind=reg_kind, tv_boundary=tv_boundary, inner_steps=inner_steps,
                   fy=facets[0], fx=facets[1], overlap=overlap, iters=iters)


def make_config(k: int, n: Optional[int] = None, **over) -> Problem:
    """BASELINE.json configs[k-1] (k = 1..5).  `n` shrinks the image (sources
    scale with area) for parity tests at oracle-friendly sizes."""
    cfg = dict(CONFIGS[k])
    full_n = cfg["n"]
    if n is not None and n != full_n:
        scale = (n / full_n) ** 2
        cfg["sources"] = max(1, int(round(cfg["sources"] * scale)))
        cfg["galaxies"] = int(round(cfg["galaxies"] * scale))
        if "nx" in cfg:                  # keep the aspect ratio
            cfg["nx"] = int(round(cfg["nx"] * n / full_n))
        cfg["n"] = n
    cfg.update(over)
    return make_problem(name=f"c{k}" + ("" if n in (None, full_n) else f"@{n}"), seed=1000 * k, **cfg)


def per_node(pb: Problem, overlap: Optional[int] = None) -> Problem:
    """The paper's node geometry for a problem: one facet per
    PSF grid point (F = G), each facet deblurred with its own PSF only and
    consensus weights = its interpolation weights (operator_mode 1).  The default
    overlap is the largest the facet planner admits (every estimate pixel in at
    most two facets per axis: O <= floor(M/F) - (P - 1), even), so each block
    spans about three grid points as in PAPER.md:255."""
    if overlap is None:
        core = min(pb.my // pb.gy, pb.mx // pb.gx)
        overlap = max(0, core - (pb.P - 1))
        overlap -= overlap % 2
    return dataclasses.replace(pb, fy=pb.gy, fx=pb.gx, overlap=int(overlap), operator_mode=1,
                               name=pb.name + "-node")


def input_hash(pb: Problem) -> str:
    """sha256 of the exact bytes deblur_create / the oracle consume (PSFs, weights,
    y, W and the scalar parameters), so stored golden values can be tied to the
    inputs they were computed from."""
    h = hashlib.sha256()
    for a in (pb.psfs, pb.wy, pb.wx, pb.y, pb.noise_w, pb.x0):
        if a is None:
            h.update(b"none")
        else:
            a = np.ascontiguousarray(a)
            h.update(str((a.dtype.str, a.shape)).encode())
            h.update(a.tobytes())
    h.update(repr((pb.ny, pb.nx, pb.P, pb.gy, pb.gx, float(pb.noise_w_scalar), pb.lam, pb.eps, pb.gamma,
                   pb.rho, pb.reg_kind, pb.tv_boundary, pb.inner_steps, pb.fy, pb.fx, pb.overlap,
                   pb.operator_mode, pb.independent, pb.local_solver, pb.inner_increment)).encode())
    return h.hexdigest()
