"""Seeded synthetic cost volumes shared by the oracle side and the CUDA side.

This module is the ONLY code both sides use.  It holds no max-flow / min-cut
arithmetic: it only produces int32 cost volumes c[x][y][z] (z fastest) in
0..255 that stand in for the paper's seismic volumes (§3.4,
Table 1 -- the real volumes are not available), with the shapes of
BASELINE.json `configs` C1..C5 and the recipe of SURVEY.md §8(d).

Bit-reproducibility.  Every value is computed from a counter-based hash
(splitmix64 of seed ^ stream<<56 ^ index) and float64 operations that IEEE-754
rounds correctly (+ - * /, sqrt, floor, ceil, fmod).  No libm transcendental is
called: sin/cos are a fixed Taylor polynomial evaluated here, and the noise is
Irwin-Hall(4) (sum of four 16-bit uniforms, rescaled to unit variance) instead
of Box-Muller, so the bytes are identical on every x86/ARM host.  The sha256 of
each config's bytes is pinned in `MANIFEST` and checked by the tests.

Recipe:
    I(x,y,z) = sum_k A_k(x,y) * [z >= ceil(z_k(x,y))] + sigma * N(x,y,z)
    g(z) = I(z) - I(z-1) (g(0) = 0);  q = min(255, floor(|g| + 0.5));  c = 255 - q
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)

STREAM_NOISE = 0
STREAM_PARAMS = 2
STREAM_SALT = 3
STREAM_TINY = 4

PI = 3.141592653589793
TWO_PI = 6.283185307179586


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrap-around arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + _GOLD
    z = (z ^ (z >> np.uint64(30))) * _MIX1
    z = (z ^ (z >> np.uint64(27))) * _MIX2
    return z ^ (z >> np.uint64(31))


def hash_stream(seed: int, stream: int, index: np.ndarray) -> np.ndarray:
    key = np.uint64((seed ^ (stream << 56)) & 0xFFFFFFFFFFFFFFFF)
    return splitmix64(np.asarray(index, dtype=np.uint64) ^ key)


def uniform01(seed: int, stream: int, index) -> np.ndarray:
    """Uniform in (0, 1] from the top 53 bits."""
    h = hash_stream(seed, stream, np.atleast_1d(np.asarray(index, dtype=np.uint64)))
    return ((h >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)


def noise(seed: int, index: np.ndarray) -> np.ndarray:
    """Zero-mean unit-variance Irwin-Hall(4) noise (range +-2*sqrt(3))."""
    h = hash_stream(seed, STREAM_NOISE, index)
    s = np.zeros(h.shape, dtype=np.float64)
    for j in range(4):
        s += ((h >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.float64)
    # each term is (k + 0.5) / 65536 in (0, 1); the sum has mean 2 and variance 1/3
    s = (s + 2.0) / 65536.0 - 2.0
    return s * np.sqrt(3.0)


def dsin(t) -> np.ndarray:
    """sin(t) by range reduction to [-pi, pi] and a degree-27 Taylor polynomial."""
    t = np.asarray(t, dtype=np.float64)
    r = t - TWO_PI * np.round(t / TWO_PI)
    r2 = r * r
    acc = np.zeros_like(r)
    for k in range(13, -1, -1):  # terms r^(2k+1)/(2k+1)!, Horner in r^2
        coef = 1.0
        for j in range(1, 2 * k + 2):
            coef /= j
        acc = acc * r2 + ((-1.0) ** k) * coef
    return acc * r


def dcos(t) -> np.ndarray:
    return dsin(np.asarray(t, dtype=np.float64) + PI / 2.0)


@dataclass
class VolumeSpec:
    name: str
    X: int
    Y: int
    Z: int
    delta: int
    seed: int
    sigma: float
    kind: str  # "sinus", "planes", "fault", "salt", "ampfield", "tiny"
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.X * self.Y * self.Z


# BASELINE.json configs C1..C5 (shapes, Delta, horizons, sigma); SURVEY.md §8(d) table.
CONFIGS = {
    "C1": VolumeSpec("C1", 16, 16, 32, 2, 1, 20.0, "sinus"),
    "C2": VolumeSpec("C2", 128, 128, 128, 3, 2, 25.0, "planes",
                     {"depths": [32.0, 64.0, 96.0], "amps": [200.0, 150.0, 100.0], "slope": 0.1}),
    "C3": VolumeSpec("C3", 256, 256, 256, 2, 3, 25.0, "fault",
                     {"depths": [64.0, 128.0, 192.0], "amps": [200.0, 150.0, 100.0], "slope": 0.1,
                      "throw": 12}),
    "C4": VolumeSpec("C4", 512, 512, 256, 4, 4, 30.0, "salt",
                     {"depths": [256.0 * (k + 1) / 6.0 for k in range(5)],
                      "amps": [200.0 - 30.0 * k for k in range(5)], "slope": 0.1, "salt": 0.01}),
    "C5": VolumeSpec("C5", 1024, 1024, 96, 1, 5, 20.0, "ampfield",
                     {"depths": [32.0, 64.0], "slope": 0.05}),
}

# sha256 of c.astype('<i4').tobytes() for each config (written by
# scripts/make_manifest.py, which calls only this module).
MANIFEST = {
    "C1": "7fa573b57eeb7dd458e207c4cebdd5df8103611296895e84e28e67af35176113",
    "C2": "17f64f64e27ab42869d3065dcb026806fdcb7c97edbcb65655779ced7b5218b7",
    "C3": "3e52bfea6a3c7f29c04541f649a954e149e47787f6b0b4c4bb09edd4b7c590eb",
    "C4": "bd1977cddcccd80091599e1067fc00a26b22c30a6b1eb8328bd7e90d7271a3dd",
    "C5": "6556f30956c38278266f68a5b7cb8314f76229b1c98b06215b64c6ca6b2d24dd",
}


def _plane_params(spec: VolumeSpec):
    """Random slopes (sx, sy) per horizon, U[-slope, slope], stream PARAMS."""
    depths = spec.extra["depths"]
    sl = spec.extra["slope"]
    out = []
    for k in range(len(depths)):
        u = uniform01(spec.seed, STREAM_PARAMS, [2 * k, 2 * k + 1])
        out.append((sl * (2.0 * u[0] - 1.0), sl * (2.0 * u[1] - 1.0)))
    return out


def _structure(spec: VolumeSpec, xs: np.ndarray, ys: np.ndarray, zs: np.ndarray) -> np.ndarray:
    """Noise-free intensity for a block of columns; xs (bx,1,1), ys (1,Y,1), zs (1,1,Z) float64."""
    if spec.kind == "sinus":
        z0 = 16.0 + 4.0 * dsin(TWO_PI * xs / 16.0) * dcos(TWO_PI * ys / 16.0)
        return 200.0 * (zs >= np.ceil(z0))
    depths = spec.extra["depths"]
    cx, cy = spec.X / 2.0, spec.Y / 2.0
    acc = np.zeros(np.broadcast_shapes(xs.shape, ys.shape, zs.shape), dtype=np.float64)
    for k, (sx, sy) in enumerate(_plane_params(spec)):
        zk = depths[k] + sx * (xs - cx) + sy * (ys - cy)
        if spec.kind == "ampfield":
            amp = 200.0 * (0.6 + 0.4 * dsin(TWO_PI * xs / spec.X) * dsin(TWO_PI * ys / spec.Y))
        else:
            amp = spec.extra["amps"][k]
        acc = acc + amp * (zs >= np.ceil(zk))
    return acc


def _fault_params(spec: VolumeSpec):
    u = uniform01(spec.seed, STREAM_PARAMS, [100, 101, 102, 103, 104])
    px = spec.X / 4.0 + u[0] * spec.X / 2.0
    py = spec.Y / 4.0 + u[1] * spec.Y / 2.0
    pz = spec.Z / 4.0 + u[2] * spec.Z / 2.0
    theta = u[3] * PI                      # strike in [0, pi)
    phi = (30.0 + 30.0 * u[4]) * PI / 180.0  # dip in [30, 60] degrees
    nx = float(dsin(phi)) * -float(dsin(theta))
    ny = float(dsin(phi)) * float(dcos(theta))
    nz = float(dcos(phi))
    return (px, py, pz), (nx, ny, nz)


def generate(spec: VolumeSpec | str, x_chunk: int = 64, x_range: tuple | None = None) -> np.ndarray:
    """int32 cost volume c[x][y][z] in 0..255 for a config (z fastest); x_range=(x0, x1)
    generates only that x-slab (identical bytes to the same slice of the full volume)."""
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    X, Y, Z = spec.X, spec.Y, spec.Z
    xa, xb = x_range if x_range is not None else (0, X)
    out = np.empty((xb - xa, Y, Z), dtype=np.int32)
    ys = np.arange(Y, dtype=np.float64).reshape(1, Y, 1)
    zs = np.arange(Z, dtype=np.float64).reshape(1, 1, Z)
    if spec.kind == "fault":
        (px, py, pz), (nx, ny, nz) = _fault_params(spec)
        throw = float(spec.extra["throw"])
    for x0 in range(xa, xb, x_chunk):
        x1 = min(xb, x0 + x_chunk)
        xs = np.arange(x0, x1, dtype=np.float64).reshape(-1, 1, 1)
        base = _structure(spec, xs, ys, zs)
        if spec.kind == "fault":
            shifted = _structure(spec, xs, ys, zs - throw)
            side = (nx * (xs - px) + ny * (ys - py) + nz * (zs - pz)) > 0.0
            base = np.where(side, shifted, base)
        idx = (np.arange(x0 * Y * Z, x1 * Y * Z, dtype=np.uint64)).reshape(x1 - x0, Y, Z)
        inten = base + spec.sigma * noise(spec.seed, idx)
        if spec.kind == "salt":
            u = uniform01(spec.seed, STREAM_SALT, idx.ravel()).reshape(idx.shape)
            inten = np.where(u < spec.extra["salt"], 255.0, inten)
        g = np.zeros_like(inten)
        g[:, :, 1:] = inten[:, :, 1:] - inten[:, :, :-1]
        q = np.minimum(255.0, np.floor(np.abs(g) + 0.5))
        out[x0 - xa:x1 - xa] = (255.0 - q).astype(np.int32)
    return out


def tiny(seed: int, X: int, Y: int, Z: int, cmax: int) -> np.ndarray:
    """Uniform integer costs in 0..cmax for the random tiny sweeps (seeds 1000..)."""
    idx = np.arange(X * Y * Z, dtype=np.uint64)
    h = hash_stream(seed, STREAM_TINY, idx)
    return ((h >> np.uint64(11)) % np.uint64(cmax + 1)).astype(np.int32).reshape(X, Y, Z)


def tiny_case(seed: int):
    """A random tiny instance (X, Y <= 5, Z <= 12, Delta in 0..4, cost ranges {3, 9, 255})."""
    u = uniform01(seed, STREAM_TINY + 1, np.arange(5))
    X = 1 + int(u[0] * 5.0) if u[0] < 1.0 else 5
    Y = 1 + int(u[1] * 5.0) if u[1] < 1.0 else 5
    Z = 1 + int(u[2] * 12.0) if u[2] < 1.0 else 12
    delta = min(4, int(u[3] * 5.0))
    cmax = (3, 9, 255)[min(2, int(u[4] * 3.0))]
    return tiny(seed, X, Y, Z, cmax), delta


def c1_cutdown() -> np.ndarray:
    """C1 brute-force cut-down: x, y in [0,3), z in [12,20), re-based to Z=8."""
    return np.ascontiguousarray(generate("C1")[0:3, 0:3, 12:20])


def sha256_volume(c: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(c, dtype="<i4").tobytes()).hexdigest()
