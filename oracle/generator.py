"""numpy twin of the device input generator `td_generate` (csrc/stream.cu).

TEST INFRASTRUCTURE: used only by tests and the bench's CPU leg to recreate,
on the host, exactly the values a GPU generated for a box of a global tensor.

value(g) for global row-major linear index g:
    key = splitmix64(splitmix64(seed) ^ (tensor_id * 0xD1B54A32D192ED03))
    h   = splitmix64(key ^ g)
    mode 0: (h % 9) - 4            (integers in [-4, 4]; the reference draws the
                                    same range with random.randint(-4, 4),
                                    pkg/src/tendist/algorithms.py:54-68)
    mode 1: (h >> 11) * 2**-52 - 1 (uniform in [-1, 1))
"""

from __future__ import annotations

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def key_of(seed: int, tensor_id: int) -> np.uint64:
    with np.errstate(over="ignore"):
        mix = np.uint64(tensor_id) * np.uint64(0xD1B54A32D192ED03)
    return splitmix64(splitmix64(np.uint64(seed)) ^ mix)


def values(linear_index, seed: int, tensor_id: int, mode: int = 0) -> np.ndarray:
    h = splitmix64(key_of(seed, tensor_id) ^ np.asarray(linear_index, dtype=np.uint64))
    if mode == 0:
        return (h % np.uint64(9)).astype(np.int64).astype(np.float64) - 4.0
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 / 9007199254740992.0) - 1.0


def generate_box(gdims, origin, shape, seed: int, tensor_id: int, mode: int = 0) -> np.ndarray:
    """The box [origin, origin+shape) of the global tensor with dims gdims."""
    gdims, origin, shape = tuple(gdims), tuple(origin), tuple(shape)
    if not gdims:
        return values(np.zeros((), dtype=np.uint64), seed, tensor_id, mode).reshape(())
    strides = np.cumprod((1,) + gdims[::-1][:-1])[::-1].astype(np.uint64)
    lin = np.zeros(shape, dtype=np.uint64)
    for ax, (o, n, s) in enumerate(zip(origin, shape, strides)):
        idx = (np.arange(n, dtype=np.uint64) + np.uint64(o)) * np.uint64(s)
        lin = lin + idx.reshape([-1 if a == ax else 1 for a in range(len(shape))])
    return values(lin, seed, tensor_id, mode)


def generate(gdims, seed: int, tensor_id: int, mode: int = 0) -> np.ndarray:
    return generate_box(gdims, (0,) * len(gdims), gdims, seed, tensor_id, mode)
