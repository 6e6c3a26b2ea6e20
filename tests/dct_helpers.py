"""Shared helpers of the Chapter 4 DCT tests (test infrastructure): block
reshaping in record order D7, 66-bit record unpacking (D5, D6), PSNR, and
the tie test used where floating point decides an integer."""
from __future__ import annotations

import numpy as np

SEL = [(0, 0), (0, 1), (1, 0), (2, 0), (1, 1), (0, 2)]


def psnr(a, b):
    mse = np.mean((np.asarray(a, float) - np.asarray(b, float)) ** 2)
    return float("inf") if mse == 0 else 10 * np.log10(255.0 ** 2 / mse)


def blocks(img, W, H, C):
    """(records, 8, 8) blocks in record order D7."""
    x = np.asarray(img, np.uint8).reshape(H // 8, 8, W // 8, 8, C)
    return x.transpose(0, 2, 4, 1, 3).reshape(-1, 8, 8)


def unblocks(b, W, H, C):
    return np.asarray(b).reshape(H // 8, W // 8, C, 8, 8).transpose(0, 3, 1, 4, 2).reshape(-1)


def records(a_plain, n):
    """Unpack n 66-bit records into (n, 6) signed integers (sign-magnitude, D5)."""
    bits = np.unpackbits(np.asarray(a_plain, np.uint8))[: 66 * n].reshape(n, 6, 11)
    w = (bits * (1 << np.arange(10, -1, -1))).sum(-1)
    return np.where(w >> 10, -(w & 1023), w & 1023)


def near_half(v, tau):
    """True where v lies within tau of a rounding boundary k + 1/2."""
    v = np.asarray(v, float)
    return np.abs(np.abs(v - np.floor(v)) - 0.5) <= tau
