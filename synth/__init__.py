"""Seeded synthetic inputs for the BASELINE.json configs.

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NONE of the method's arithmetic (no lifting, packing, cipher or hash):
only numpy PCG64 generators whose value distributions proxy the paper's
workloads:

  * uniform random bytes: compressed video / "arbitrary binary" (entropy ~8
    bits/byte);
  * smooth natural-image bitmaps: the Lenna case;
  * English-like ASCII text: the text case (entropy ~4.1-4.6 bits/byte).
"""
from __future__ import annotations

import math

import numpy as np

KEY = bytes(range(16))  # 000102...0f for every config


def iv_for(config: int, index: int = 0) -> bytes:
    """IV_i = be64(config) || be64(index)."""
    return int(config).to_bytes(8, "big") + int(index).to_bytes(8, "big")


def width_rule(n: int) -> int:
    """Matrix width used for arbitrary files (reading C18): 1024 for n >= 1 MiB,
    else the next power of two >= ceil(sqrt(n)), at least 8."""
    if n >= (1 << 20):
        return 1024
    w = 8
    while w * w < n:
        w *= 2
    return w


def random_bytes(n: int, seed: int) -> np.ndarray:
    return np.frombuffer(np.random.default_rng(seed).bytes(n), dtype=np.uint8).copy()


def bitmap(height: int, width: int, channels: int, seed: int) -> np.ndarray:
    """Natural-image proxy: 8 low-frequency 2-D sinusoids + linear gradients +
    20 filled rectangles (hard edges) + Gaussian noise sigma=2, channels
    correlated (shared luminance + per-channel offset), clipped to [0,255].
    Returned as the raw pixel array (height, width*channels) uint8 — a 24-bit
    bitmap's pixel data with no header."""
    rng = np.random.default_rng(seed)
    yy = np.linspace(0.0, 1.0, height, dtype=np.float32)[:, None]
    xx = np.linspace(0.0, 1.0, width, dtype=np.float32)[None, :]
    lum = np.full((height, width), 110.0, dtype=np.float32)
    for _ in range(8):
        fy, fx = rng.uniform(0.5, 6.0, size=2)
        ph = rng.uniform(0, 2 * math.pi)
        amp = rng.uniform(8, 30)
        lum += amp * np.sin(2 * math.pi * (fy * yy + fx * xx) + ph).astype(np.float32)
    gy, gx = rng.uniform(-40, 40, size=2)
    lum += gy * yy + gx * xx
    for _ in range(20):
        h = int(rng.integers(height // 32 + 1, height // 4 + 2))
        w = int(rng.integers(width // 32 + 1, width // 4 + 2))
        y0 = int(rng.integers(0, max(1, height - h)))
        x0 = int(rng.integers(0, max(1, width - w)))
        lum[y0:y0 + h, x0:x0 + w] = rng.uniform(0, 255)
    planes = []
    for _ in range(channels):
        off = rng.uniform(-20, 20)
        noise = rng.normal(0.0, 2.0, size=(height, width)).astype(np.float32)
        planes.append(np.clip(lum + off + noise, 0, 255))
    px = np.stack(planes, axis=-1)  # (H, W, C), BGR order by convention
    return np.rint(px).astype(np.uint8).reshape(height, width * channels)


# English letter frequencies (percent), a..z.
_EN_FREQ = [8.17, 1.49, 2.78, 4.25, 12.70, 2.23, 2.02, 6.09, 6.97, 0.15, 0.77, 4.03, 2.41,
            6.75, 7.51, 1.93, 0.10, 5.99, 6.33, 9.06, 2.76, 0.98, 2.36, 0.15, 1.97, 0.07]


def text_like(n: int, seed: int) -> np.ndarray:
    """English-like ASCII: letters at English frequencies, ~18% spaces, some
    capitals, punctuation and newlines (entropy ~4.1-4.3 bits/byte)."""
    rng = np.random.default_rng(seed)
    p = np.array(_EN_FREQ, dtype=np.float64)
    p /= p.sum()
    letters = rng.choice(26, size=n, p=p).astype(np.uint8) + ord("a")
    u = rng.random(n)
    out = letters
    out[u < 0.03] -= 32                                    # capitals
    out[(u >= 0.03) & (u < 0.21)] = ord(" ")
    punct = np.frombuffer(b".,;'-!?", dtype=np.uint8)
    m = (u >= 0.21) & (u < 0.235)
    out[m] = punct[rng.integers(0, len(punct), size=int(m.sum()))]
    out[(u >= 0.235) & (u < 0.24)] = ord("\n")
    return out


# ---- the five BASELINE.json configs ----------------------------------------

CONFIGS = {
    1: dict(name="C1-256x256-random-L1", width=256, levels=1, n_bytes=256 * 256),
    2: dict(name="C2-2048x2048x24bit-bitmap-L2", width=6144, levels=2, n_bytes=6144 * 2048),
    3: dict(name="C3-64MiB-binary-L3", width=1024, levels=3, n_bytes=1 << 26),
    4: dict(name="C4-1GiB-file-L2", width=1024, levels=2, n_bytes=1 << 30),
    5: dict(name="C5-10000-files-L2", width=None, levels=2, n_bytes=None),
}


def config_input(config: int, n_bytes: int | None = None) -> np.ndarray:
    """The seeded input of a config; ``n_bytes`` truncates (prefix) for
    reduced-size parity cases."""
    if config == 1:
        x = random_bytes(256 * 256, 1)
    elif config == 2:
        x = bitmap(2048, 2048, 3, 2).reshape(-1)
    elif config == 3:
        x = random_bytes(n_bytes or (1 << 26), 3)
    elif config == 33:
        x = text_like(n_bytes or (1 << 26), 33)
    elif config == 4:
        x = random_bytes(n_bytes or (1 << 30), 4)
    else:
        raise ValueError(config)
    return x if n_bytes is None else x[:n_bytes]


def c5_file_sizes(count: int = 10000, seed: int = 5) -> np.ndarray:
    """Sizes log-uniform on [1 KiB, 16 MiB]."""
    rng = np.random.default_rng(seed)
    s = np.exp(rng.uniform(math.log(1024), math.log(1 << 24), size=count))
    return np.rint(s).astype(np.int64)


def c5_file(i: int, size: int) -> np.ndarray:
    """Content mix 40% random / 30% bitmap-like / 30% text-like, seed (5, i)."""
    kind = i % 10
    seed = [5, i]
    if kind < 4:
        return np.frombuffer(np.random.default_rng(seed).bytes(size), dtype=np.uint8).copy()
    if kind < 7:
        w = max(8, int(math.sqrt(size / 3)))
        h = -(-size // (3 * w))
        return bitmap(h, w, 3, np.random.default_rng(seed).integers(1 << 31)).reshape(-1)[:size]
    return text_like(size, int(np.random.default_rng(seed).integers(1 << 31)))
