"""synth — seeded synthetic inputs shaped like the paper's workloads.

Shared by the oracle tests and the GPU path (the only module both sides use).
It renders frames from the sensor model of Eq. (1), P:75-80,

    I = I0 + I0 K + psi,   stored as u8 = rint(clip(I0 (1+K) + N(0, sigma_n^2), 0, 255)),

and holds none of the method's arithmetic (no averaging, filtering,
estimation or matching).  The paper's datasets (VISION, NYUAD-MMD; P:259,
P:430) are not available; these recipes stand in for their shapes (Full-HD
video at 30 fps of about 1200-1800 frames P:382/P:468, multi-megapixel stills,
720p camera batches).  The recipes are the configs of BASELINE.json as
restated in SURVEY.md §8(d) and DESIGN.md §"Inputs".

Every draw comes from a ``torch.Generator`` seeded from (config, seed, stream),
so a given (recipe, seed, device) always yields the same bytes.  The bytes
differ between CPU and CUDA generators; every comparison feeds the SAME bytes
to both sides (frames generated on the device are copied to the host for the
oracle).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

TWO_PI = 2.0 * math.pi


def _gen(device, cfg: int, seed: int, stream: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((cfg * 1_000_003 + seed * 7_919 + stream * 104_729) & 0x7FFF_FFFF_FFFF)
    return g


def camera_K(H: int, W: int, sigma_k: float, cfg: int, seed: int, camera: int = 0, device="cpu"):
    """True PRNU K ~ N(0, sigma_k^2) i.i.d. per pixel, fixed per camera (BASELINE configs)."""
    g = _gen(device, cfg, seed, 10_000 + camera)
    return torch.randn((H, W), generator=g, device=device, dtype=torch.float32) * sigma_k


@dataclass
class SceneParams:
    fx: torch.Tensor      # [C] integer x frequencies (cycles per frame width)
    fy: torch.Tensor      # [C] integer y frequencies
    amp: torch.Tensor     # [C] amplitudes U(0.5, 1)
    phase: torch.Tensor   # [C] phases U(0, 2 pi)
    omega: torch.Tensor   # [C] phase drift per frame (rad/frame)


def _scene_params(n: int, fmax: int, drift: float, g: torch.Generator, device) -> SceneParams:
    fx = torch.randint(0, fmax + 1, (n,), generator=g, device=device)
    fy = torch.randint(-fmax, fmax + 1, (n,), generator=g, device=device)
    zero = (fx == 0) & (fy == 0)
    fx = torch.where(zero, torch.ones_like(fx), fx)          # (fx, fy) != (0, 0)
    amp = 0.5 + 0.5 * torch.rand((n,), generator=g, device=device, dtype=torch.float64)
    phase = TWO_PI * torch.rand((n,), generator=g, device=device, dtype=torch.float64)
    omega = (2 * torch.rand((n,), generator=g, device=device, dtype=torch.float64) - 1) * drift
    return SceneParams(fx.double(), fy.double(), amp, phase, omega)


def _render_sinusoids(p: SceneParams, H: int, W: int, t: torch.Tensor, ty: torch.Tensor, tx: torch.Tensor):
    """s_t(y,x) = sum_c A_c sin(2 pi (fx_c (x - tx_t)/W + fy_c (y - ty_t)/H) + phi_c + omega_c t)
    for a batch of frame indices t, as one batched [H,2C]x[2C,W] product
    (sin(a+b) = sin a cos b + cos a sin b).  Integer frequencies make the scene
    periodic, so integer translations are exact circular shifts.  fp64."""
    dev = t.device
    y = torch.arange(H, device=dev, dtype=torch.float64)
    x = torch.arange(W, device=dev, dtype=torch.float64)
    # alpha[b, c, x], beta[b, c, y]
    alpha = TWO_PI * p.fx[None, :, None] * (x[None, None, :] - tx[:, None, None]) / W
    beta = (TWO_PI * p.fy[None, :, None] * (y[None, None, :] - ty[:, None, None]) / H
            + p.phase[None, :, None] + p.omega[None, :, None] * t[:, None, None].double())
    A = p.amp[None, :, None]
    Ycat = torch.cat([A * torch.cos(beta), A * torch.sin(beta)], dim=1).transpose(1, 2)  # [b, H, 2C]
    Xcat = torch.cat([torch.sin(alpha), torch.cos(alpha)], dim=1)                       # [b, 2C, W]
    return torch.bmm(Ycat, Xcat)  # [b, H, W]


def _quantise(I0K: torch.Tensor, sigma_n: float, g: torch.Generator) -> torch.Tensor:
    """u8 = rint(clip(I0 (1+K) + N(0, sigma_n^2), 0, 255)), round half to even."""
    noise = torch.randn(I0K.shape, generator=g, device=I0K.device, dtype=torch.float32) * sigma_n
    return torch.round(torch.clamp(I0K + noise, 0.0, 255.0)).to(torch.uint8)


@dataclass
class Video:
    frames: torch.Tensor   # u8 [m, H, W]
    K: torch.Tensor        # fp32 [H, W] true PRNU of this camera
    K_other: torch.Tensor  # fp32 [H, W] a second, independent camera's PRNU
    recipe: str


def video(recipe: str, m: int, H: int, W: int, seed: int = 0, device="cpu", camera: int = 0,
          sigma_k: float | None = None, sigma_n: float | None = None, chunk: int = 32,
          out: torch.Tensor | None = None) -> Video:
    """Render an m-frame u8 video.

    recipe "shift" (configs 1 and 5): I0 = 8 sinusoids, |f| <= 4, min-max scaled
        to [40, 215]; each frame is I0 circularly shifted by a random integer
        (dy, dx); K ~ N(0, 0.02^2); sigma_n = 2.
    recipe "drift" (configs 2 and 4): 16 sinusoids, |f| <= 8, phases drifting by
        omega_c t (omega_c ~ U(-0.05, 0.05) rad/frame) plus a global circular
        translation round(v t), |v| <= 0.5 px/frame; scaled 127.5 + 87.5 s/sum A
        into [40, 215]; K ~ N(0, 0.01^2); sigma_n = 4 ("heavy compression").
    """
    cfg = {"shift": 1, "drift": 2}[recipe]
    sk = sigma_k if sigma_k is not None else (0.02 if recipe == "shift" else 0.01)
    sn = sigma_n if sigma_n is not None else (2.0 if recipe == "shift" else 4.0)
    K = camera_K(H, W, sk, cfg, seed, camera, device)
    K_other = camera_K(H, W, sk, cfg, seed, camera + 5_000, device)
    gs = _gen(device, cfg, seed, 20_000 + camera)   # scene parameters
    gn = _gen(device, cfg, seed, 30_000 + camera)   # per-frame noise
    frames = out if out is not None else torch.empty((m, H, W), dtype=torch.uint8, device=device)
    assert frames.shape == (m, H, W) and frames.dtype == torch.uint8
    if recipe == "shift":
        p = _scene_params(8, 4, 0.0, gs, device)
        zero = torch.zeros(1, device=device, dtype=torch.float64)
        base = _render_sinusoids(p, H, W, zero, zero, zero)[0]
        lo, hi = base.min(), base.max()
        scale = 175.0 / (hi - lo) if float(hi - lo) > 0 else torch.zeros_like(hi)
        I0 = (40.0 + (base - lo) * scale).float()
        dy = torch.randint(0, H, (m,), generator=gs, device=device)
        dx = torch.randint(0, W, (m,), generator=gs, device=device)
        for s in range(0, m, chunk):
            e = min(m, s + chunk)
            for j in range(s, e):
                I0t = torch.roll(I0, shifts=(int(dy[j]), int(dx[j])), dims=(0, 1))
                frames[j] = _quantise((I0t * (1.0 + K))[None], sn, gn)[0]
    else:
        p = _scene_params(16, 8, 0.05, gs, device)
        v = (2 * torch.rand((2,), generator=gs, device=device, dtype=torch.float64) - 1) * 0.5
        sumA = p.amp.sum()
        for s in range(0, m, chunk):
            e = min(m, s + chunk)
            t = torch.arange(s, e, device=device, dtype=torch.float64)
            ty, tx = torch.round(v[0] * t), torch.round(v[1] * t)
            sc = _render_sinusoids(p, H, W, t, ty, tx)
            I0 = (127.5 + 87.5 * sc / sumA).float()
            frames[s:e] = _quantise(I0 * (1.0 + K)[None], sn, gn)
    return Video(frames, K, K_other, recipe)


def stills(n: int, H: int, W: int, seed: int = 0, device="cpu", sigma_k: float = 0.015, sigma_n: float = 2.0,
           texture_std: float = 20.0, blur_sigma: float = 1.5):
    """Config 3: n independent RGB scenes (16 sinusoids scaled to [40, 215] plus a
    band-limited texture: white N(0,1) -> Gaussian blur sigma=1.5 px -> std 20),
    per-channel gain U(0.85, 1.15), per-channel K_c ~ N(0, 0.015^2), sigma_n = 2,
    then BT.601 luma Y = rint(0.299 R + 0.587 G + 0.114 B) as u8 (R-21; the luma
    conversion is input preparation).  Returns (Y u8 [n,H,W], K_luma fp32)."""
    cfg = 3
    Ks = [camera_K(H, W, sigma_k, cfg, seed, c, device) for c in range(3)]
    K_luma = 0.299 * Ks[0] + 0.587 * Ks[1] + 0.114 * Ks[2]
    gs = _gen(device, cfg, seed, 20_000)
    gn = _gen(device, cfg, seed, 30_000)
    r = int(math.ceil(3 * blur_sigma))
    k1 = torch.exp(-0.5 * (torch.arange(-r, r + 1, device=device, dtype=torch.float32) / blur_sigma) ** 2)
    k1 = k1 / k1.sum()
    Y = torch.empty((n, H, W), dtype=torch.uint8, device=device)
    for i in range(n):
        p = _scene_params(16, 8, 0.0, gs, device)
        zero = torch.zeros(1, device=device, dtype=torch.float64)
        s = _render_sinusoids(p, H, W, zero, zero, zero)[0]
        s = (40.0 + (s - s.min()) * (175.0 / (s.max() - s.min()))).float()
        tex = torch.randn((1, 1, H, W), generator=gs, device=device, dtype=torch.float32)
        tex = torch.nn.functional.conv2d(torch.nn.functional.pad(tex, (r, r, 0, 0), mode="circular"),
                                         k1.view(1, 1, 1, -1))
        tex = torch.nn.functional.conv2d(torch.nn.functional.pad(tex, (0, 0, r, r), mode="circular"),
                                         k1.view(1, 1, -1, 1))[0, 0]
        tex = tex * (texture_std / tex.std())
        gains = 0.85 + 0.3 * torch.rand((3,), generator=gs, device=device)
        acc = torch.zeros((H, W), dtype=torch.float32, device=device)
        for c, wgt in enumerate((0.299, 0.587, 0.114)):
            I0 = torch.clamp((s + tex) * gains[c], 0.0, 255.0)
            ch = _quantise(I0 * (1.0 + Ks[c]), sigma_n, gn).float()
            acc += wgt * ch
        Y[i] = torch.round(acc).clamp(0, 255).to(torch.uint8)
    return Y, K_luma


# BASELINE.json configs, as (recipe, m, H, W, depths).  H = rows, W = columns.
CONFIGS = {
    1: dict(recipe="shift", m=16, H=64, W=64, depths=(4, 1)),
    2: dict(recipe="drift", m=1800, H=1080, W=1920, depths=(1, 50)),
    3: dict(recipe="stills", m=200, H=3000, W=4000, depths=(1, 5, 10, 20, 50)),
    4: dict(recipe="drift", m=300, H=720, W=1280, depths=(30,), cameras=64),
    5: dict(recipe="shift", m=3600, H=1080, W=1920, depths=(1, 2, 5, 10, 25, 50, 100, 300, 3600)),
}
