"""Seeded synthetic inputs for the stochastic spatial-domain CSC hot path.

This module is shared by the oracle-side tests and the CUDA-side tests/bench.
It holds NONE of the method's arithmetic (no convolution, no mask, no prox):
only the input recipe of DESIGN.md §"Input recipe".

The paper's workloads are datasets that are not in this container (fruit/city,
10 images 100x100; 1000 ImageNet 100x100 patches,
PAPER.md:432-433; 10 test images 256x256).  These generators
stand in for them with the same shapes: K=100 filters 11x11,
K=400 over-complete, lambda=1, the p set
{1, .5, .2, .1, .05}.  Contrast normalisation
 is replaced by a 1/f^2 field minus its sigma=2 Gaussian
blur, scaled to unit std (BASELINE.json configs).  No dataset item is
reproduced.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Sequence

import numpy as np

ROOT_SEED = 190900145  # arxiv id, fixed once


@dataclasses.dataclass(frozen=True)
class CSCConfig:
    """One BASELINE.json config.  Codes are K x (H+s-1) x (W+s-1) per image."""

    index: int          # 1-based BASELINE.json configs[index-1]
    name: str
    K: int
    s: int
    N: int              # images (batch) or mini-batch size (online)
    H: int
    W: int
    lam: float
    p: float
    iters: int
    online: bool = False
    n_inner: int = 1    # code steps per filter step (online: 10)

    @property
    def Hc(self) -> int:
        return self.H + self.s - 1

    @property
    def Wc(self) -> int:
        return self.W + self.s - 1

    def with_(self, **kw) -> "CSCConfig":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    "tiny": CSCConfig(1, "tiny", K=8, s=5, N=4, H=32, W=32, lam=1.0, p=0.5, iters=50),
    "batch": CSCConfig(2, "batch", K=100, s=11, N=10, H=100, W=100, lam=1.0, p=0.1, iters=100),
    "sweep": CSCConfig(3, "sweep", K=100, s=11, N=40, H=256, W=256, lam=1.0, p=0.1, iters=100),
    "online": CSCConfig(4, "online", K=400, s=11, N=8, H=100, W=100, lam=1.0, p=0.1,
                        iters=2000, online=True, n_inner=10),
    "large": CSCConfig(5, "large", K=1024, s=11, N=64, H=512, W=512, lam=1.0, p=0.1, iters=50),
}

SWEEP_P = (0.05, 0.1, 0.2, 0.5, 1.0)


def _highpass_field(rng: np.random.Generator, H: int, W: int, sigma: float = 2.0) -> np.ndarray:
    """1/f^2-PSD Gaussian random field minus its sigma-px Gaussian blur, unit std (fp64)."""
    w = rng.standard_normal((H, W))
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.fftfreq(W)[None, :]
    f = np.sqrt(fx * fx + fy * fy)
    amp = np.zeros_like(f)
    nz = f > 0
    amp[nz] = 1.0 / f[nz]
    highpass = 1.0 - np.exp(-2.0 * np.pi ** 2 * sigma ** 2 * f * f)
    x = np.real(np.fft.ifft2(np.fft.fft2(w) * amp * highpass))
    x = x - x.mean()
    sd = x.std()  # population std (ddof=0)
    if sd > 0:
        x = x / sd
    return x


def make_image(cfg: CSCConfig, n: int) -> np.ndarray:
    rng = np.random.default_rng(np.random.SeedSequence([ROOT_SEED, cfg.index, 1, n]))
    return _highpass_field(rng, cfg.H, cfg.W).astype(np.float32)


def make_images(cfg: CSCConfig, n0: int = 0, count: Optional[int] = None) -> np.ndarray:
    """Images n0 .. n0+count-1 as float32 [count, H, W] (count defaults to cfg.N)."""
    count = cfg.N if count is None else count
    out = np.empty((count, cfg.H, cfg.W), dtype=np.float32)
    for i in range(count):
        out[i] = make_image(cfg, n0 + i)
    return out


def make_filters(cfg: CSCConfig) -> np.ndarray:
    """N(0,1) filters, per-filter zero mean, unit L2 norm, float32 [K, s, s]."""
    rng = np.random.default_rng(np.random.SeedSequence([ROOT_SEED, cfg.index, 2]))
    d = rng.standard_normal((cfg.K, cfg.s, cfg.s))
    d = d - d.mean(axis=(1, 2), keepdims=True)
    nrm = np.sqrt((d * d).sum(axis=(1, 2), keepdims=True))
    d = d / np.where(nrm > 0, nrm, 1.0)
    return d.astype(np.float32)


def make_codes(cfg: CSCConfig, count: Optional[int] = None) -> np.ndarray:
    count = cfg.N if count is None else count
    return np.zeros((count, cfg.K, cfg.Hc, cfg.Wc), dtype=np.float32)


def mask_seed(cfg: CSCConfig) -> int:
    return int(np.random.SeedSequence([ROOT_SEED, cfg.index, 3]).generate_state(1, np.uint64)[0])


def online_image_index(step: int, member: int, batch: int = 8) -> int:
    """Config 4 stream: image for step t, member j is n = batch*t + j."""
    return batch * step + member


def random_problem(seed: int, N: int, K: int, s: int, H: int, W: int,
                   code_density: float = 1.0, dtype=np.float32):
    """Small generic random (x, d, z) for tests: seeded, no structure beyond shapes."""
    rng = np.random.default_rng(np.random.SeedSequence([ROOT_SEED, 99, seed]))
    x = rng.standard_normal((N, H, W))
    d = rng.standard_normal((K, s, s))
    d = d / np.sqrt((d * d).sum(axis=(1, 2), keepdims=True))
    z = rng.standard_normal((N, K, H + s - 1, W + s - 1))
    if code_density < 1.0:
        z = z * (rng.random(z.shape) < code_density)
    return x.astype(dtype), d.astype(dtype), z.astype(dtype)


def config_by_name(name: str, p: Optional[float] = None) -> CSCConfig:
    cfg = CONFIGS[name]
    if p is not None:
        cfg = cfg.with_(p=float(p))
    return cfg


__all__: Sequence[str] = [
    "CSCConfig", "CONFIGS", "SWEEP_P", "make_image", "make_images", "make_filters",
    "make_codes", "mask_seed", "online_image_index", "random_problem", "config_by_name",
]
