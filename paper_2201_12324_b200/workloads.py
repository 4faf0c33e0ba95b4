"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference publishes no dataset for this path, so every
config is a seeded numpy draw with the shapes and distributions that
BASELINE.json's ``configs`` list names.  Draws are made in float64 with
``np.random.default_rng(seed)`` and rounded to float32; the CUDA path gets
those float32 values and the CPU oracle gets the same values upcast to
float64.  Draw order is fixed: x, then y, then a, then b (cfg3: per problem
mu_k, x_k, y_k).  Weights are normalised in float64 and passed as float64.

Every generator takes optional ``n``/``m`` overrides so tests can draw the
same distributions at sizes the CPU oracle finishes in seconds.
"""

from __future__ import annotations

import dataclasses

import numpy as np

SUBSAMPLE = 4096  # epsilon estimate subsample edge for cfg2 / cfg4 (BASELINE.json configs[1,3])


@dataclasses.dataclass
class Workload:
    name: str
    x: np.ndarray            # float32 [n, d]   (cfg3: [B, n, d])
    y: np.ndarray            # float32 [m, d]   (cfg3: [B, m, d])
    a: np.ndarray | None     # float64 [n] or None (uniform)
    b: np.ndarray | None
    eps: float | np.ndarray  # float64 scalar (cfg3: [B])
    threshold: float
    max_iters: int
    inner_iters: int = 10
    materialised: bool = False
    eps_scale: float = 0.05              # eps = eps_scale x mean cost ...
    eps_subsample_seed: int | None = None  # ... over a seeded SUBSAMPLE x SUBSAMPLE block (else exact)

    @property
    def shape(self):
        return (self.x.shape[-2], self.y.shape[-2])

    @property
    def d(self):
        return self.x.shape[-1]


def exact_mean_sqeucl(x: np.ndarray, y: np.ndarray) -> float:
    """mean_ij |x_i - y_j|^2 = mean|x|^2 + mean|y|^2 - 2 xbar.ybar, in float64."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return float(np.einsum("id,id->", x, x) / x.shape[0]
                 + np.einsum("jd,jd->", y, y) / y.shape[0]
                 - 2.0 * x.mean(axis=0) @ y.mean(axis=0))


def subsample_rows(n: int, m: int, seed: int, edge: int = SUBSAMPLE):
    """The seeded subsample rows of the eps estimate (drawn without replacement)."""
    rng = np.random.default_rng(seed + 1000)
    ix = rng.choice(n, size=min(edge, n), replace=False)
    iy = rng.choice(m, size=min(edge, m), replace=False)
    return ix, iy


def subsample_mean_sqeucl(x: np.ndarray, y: np.ndarray, seed: int, edge: int = SUBSAMPLE) -> float:
    """Exact mean cost over a seeded edge x edge subsample (rows drawn without replacement)."""
    ix, iy = subsample_rows(x.shape[0], y.shape[0], seed, edge)
    return exact_mean_sqeucl(x[ix], y[iy])


def estimate_eps_device(wl: Workload, xd, yd) -> float:
    """The workload's eps rule evaluated on device-resident points (torch, float64):
    the time-to-tolerance measurement includes it.  Same
    formula and subsample as the host value, so it agrees to float64 rounding."""
    import torch
    if wl.eps_subsample_seed is not None:
        ix, iy = subsample_rows(xd.shape[0], yd.shape[0], wl.eps_subsample_seed)
        xd = xd[torch.as_tensor(ix, device=xd.device)]
        yd = yd[torch.as_tensor(iy, device=yd.device)]
    x = xd.double()
    y = yd.double()
    mean = ((x * x).sum() / x.shape[0] + (y * y).sum() / y.shape[0]
            - 2.0 * torch.dot(x.mean(dim=0), y.mean(dim=0)))
    return wl.eps_scale * float(mean.item())


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def cfg1(n: int = 2048, m: int = 2048, d: int = 3, seed: int = 0) -> Workload:
    """configs[0]: x~N(0,I), y~N(0.5*1,I), uniform weights, eps = 0.05 * exact mean(C)."""
    rng = np.random.default_rng(seed)
    x = _f32(rng.standard_normal((n, d)))
    y = _f32(rng.standard_normal((m, d)) + 0.5)
    eps = 0.05 * exact_mean_sqeucl(x, y)
    return Workload("cfg1_pointcloud_2048_d3", x, y, None, None, eps, 1e-3, 2000)


def cfg2(n: int = 65536, m: int = 65536, d: int = 64, seed: int = 2) -> Workload:
    """configs[1]: x~N(0,I), y=1.5*N(0,I), uniform, eps = 0.05 * mean on a 4096^2 subsample."""
    rng = np.random.default_rng(seed)
    x = _f32(rng.standard_normal((n, d)))
    y = _f32(1.5 * rng.standard_normal((m, d)))
    eps = 0.05 * subsample_mean_sqeucl(x, y, seed)
    return Workload("cfg2_online_65536_d64", x, y, None, None, eps, 1e-3, 1000,
                    eps_subsample_seed=seed)


def cfg3(batch: int = 512, n: int = 512, m: int = 512, d: int = 16, seed: int = 3) -> Workload:
    """configs[2]: B problems, y_k ~ N(mu_k, I), mu_k ~ U[-1,1]^d, materialised cost,
    eps_k = 0.05 * exact mean(C_k)."""
    rng = np.random.default_rng(seed)
    xs = np.empty((batch, n, d), np.float32)
    ys = np.empty((batch, m, d), np.float32)
    eps = np.empty(batch)
    for k in range(batch):
        mu = rng.uniform(-1.0, 1.0, size=d)
        xs[k] = rng.standard_normal((n, d))
        ys[k] = rng.standard_normal((m, d)) + mu
        eps[k] = 0.05 * exact_mean_sqeucl(xs[k], ys[k])
    return Workload("cfg3_batched_512x512x512_d16", xs, ys, None, None, eps, 1e-3, 500,
                    materialised=True)


def cfg4(n: int = 262144, m: int = 131072, d: int = 128, seed: int = 4) -> Workload:
    """configs[3]: x~N(0,I); y an equal-weight mixture of 0.5*N(0,I) and N(0.3*1, I)
    (component label drawn per point); a, b ~ U(0.5,1.5) normalised;
    eps = 0.05 * subsample mean."""
    rng = np.random.default_rng(seed)
    x = _f32(rng.standard_normal((n, d)))
    comp = rng.random(m) < 0.5
    z = rng.standard_normal((m, d))
    y = _f32(np.where(comp[:, None], 0.5 * z, z + 0.3))
    a = rng.uniform(0.5, 1.5, size=n)
    a /= a.sum()
    b = rng.uniform(0.5, 1.5, size=m)
    b /= b.sum()
    eps = 0.05 * subsample_mean_sqeucl(x, y, seed)
    return Workload("cfg4_unbalanced_262144x131072_d128", x, y, a, b, eps, 1e-3, 1000,
                    eps_subsample_seed=seed)


def cfg5(n: int = 32768, m: int = 32768, d: int = 1024, seed: int = 5) -> Workload:
    """configs[4]: rows N(0,I) L2-normalised to the unit sphere; eps = 0.01 * exact mean;
    tolerance 1e-4, max 3000."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y = rng.standard_normal((m, d))
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    x, y = _f32(x), _f32(y)
    eps = 0.01 * exact_mean_sqeucl(x, y)
    return Workload("cfg5_highdim_32768_d1024", x, y, None, None, eps, 1e-4, 3000, eps_scale=0.01)


CONFIGS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5}


def make(k: int, **kw) -> Workload:
    return CONFIGS[k](**kw)
