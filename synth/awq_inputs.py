"""AWQ-format synthetic problems (random bits only; see synth/__init__.py for the recipe)."""
from dataclasses import dataclass

import numpy as np

from .splitmix import splitmix64, uniform01

_TENSOR_SALT = 0xD1B54A32D192ED03
T_X, T_QWEIGHT, T_ZEROS, T_SCALES = 0, 1, 2, 3


def _stream_seed(seed: int, tensor_id: int) -> int:
    return (seed ^ ((tensor_id * _TENSOR_SALT) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF


@dataclass
class AWQProblem:
    """One W4A16 problem in the AWQ "GEMM" checkpoint convention (SURVEY §8(b) conventions)."""
    x: np.ndarray        # float16 [M][K]
    qweight: np.ndarray  # uint32 [K][N/8]
    scales: np.ndarray   # float16 [K/G][N]
    zeros: np.ndarray    # uint32 [K/G][N/8]
    group_size: int

    @property
    def M(self):
        return self.x.shape[0]

    @property
    def K(self):
        return self.qweight.shape[0]

    @property
    def N(self):
        return self.scales.shape[1]


def make_x(seed: int, M: int, K: int) -> np.ndarray:
    """X ~ U[-1, 1], rounded to fp16 (BASELINE.json: inputs drawn from [-1, 1])."""
    u = uniform01(_stream_seed(seed, T_X), M * K)
    return (2.0 * u - 1.0).astype(np.float16).reshape(M, K)


def _words(seed: int, tensor_id: int, rows: int, cols: int) -> np.ndarray:
    z = splitmix64(_stream_seed(seed, tensor_id), rows * cols)
    return (z >> np.uint64(32)).astype(np.uint32).reshape(rows, cols)


def make_qweight(seed: int, K: int, N: int) -> np.ndarray:
    """Random 32-bit words: every 4-bit code uniform on [0, 15]."""
    return _words(seed, T_QWEIGHT, K, N // 8)


def make_zeros(seed: int, K: int, N: int, G: int) -> np.ndarray:
    """Random 32-bit words: every 4-bit zero point uniform on [0, 15] (harsher than real AWQ)."""
    return _words(seed, T_ZEROS, K // G, N // 8)


def make_scales(seed: int, K: int, N: int, G: int, lo: float = 0.004, hi: float = 0.012) -> np.ndarray:
    """Scales ~ U[lo, hi] rounded to fp16."""
    u = uniform01(_stream_seed(seed, T_SCALES), (K // G) * N)
    return (lo + (hi - lo) * u).astype(np.float16).reshape(K // G, N)


def make_problem(seed: int, M: int, N: int, K: int, G: int = 128) -> AWQProblem:
    return AWQProblem(make_x(seed, M, K), make_qweight(seed, K, N), make_scales(seed, K, N, G),
                      make_zeros(seed, K, N, G), G)


def make_structured(kind: str, seed: int, M: int, N: int, K: int, G: int = 128) -> AWQProblem:
    """Structured sets:

    unit         scales = 1/15 so weights span [-1, 1] (stress set)
    intexact     scales = 2^-6, X in {-1, 0, 1} with <= 128 non-zeros per row; every partial
                 sum is an integer multiple of 2^-6 below 2^11 * 2^-6, so Y is exact in fp32
                 and in fp16 whatever the summation order
    onehot       X[m][perm(m)] = 1, else 0 (M <= K): Y rows are rows of dequant(W)
    zero_weights every code equals its group's zero point: Y == 0
    """
    p = make_problem(seed, M, N, K, G)
    if kind == "unit":
        p.scales = np.full_like(p.scales, np.float16(1.0 / 15.0))
    elif kind == "intexact":
        p.scales = np.full_like(p.scales, np.float16(2.0 ** -6))
        z = splitmix64(_stream_seed(seed, T_X) ^ 0x5A5A, M * K).reshape(M, K)
        sign = np.where((z & np.uint64(1)) == 1, 1.0, -1.0)
        keep = min(K, 128)
        # keep the `keep` positions with the smallest random keys in each row
        order = np.argsort(z >> np.uint64(8), axis=1, kind="stable")[:, :keep]
        x = np.zeros((M, K), dtype=np.float64)
        rows = np.arange(M)[:, None]
        x[rows, order] = sign[rows, order]
        p.x = x.astype(np.float16)
    elif kind == "onehot":
        assert M <= K
        z = splitmix64(_stream_seed(seed, T_X) ^ 0xA5A5, K)
        perm = np.argsort(z, kind="stable")[:M]
        x = np.zeros((M, K), dtype=np.float16)
        x[np.arange(M), perm] = 1.0
        p.x = x
    elif kind == "zero_weights":
        # each qweight word of group g is the zeros word of group g: code == zero nibble-for-nibble
        p.qweight = np.repeat(p.zeros, G, axis=0).copy()
    else:
        raise ValueError(f"unknown structured set {kind!r}")
    return p


@dataclass
class GPTQProblem:
    """One problem in the AutoGPTQ checkpoint format (random bits only): qweight [K/8][N] packed along
    K, qzeros [K/G][N/8] packed along N, scales fp16 [K/G][N], g_idx [K] (act-order: a seeded random
    permutation of the rows' groups, each group holding G rows)."""
    x: np.ndarray
    qweight: np.ndarray
    qzeros: np.ndarray
    scales: np.ndarray
    g_idx: np.ndarray
    group_size: int


def make_gptq_problem(seed: int, M: int, N: int, K: int, G: int = 128, act_order: bool = True) -> GPTQProblem:
    x = make_x(seed, M, K)
    qweight = _words(seed, T_QWEIGHT, K // 8, N)
    # zeros stored as z - 1 ("v1"): keep the decoded zero in [1, 15] so it has a 4-bit form
    qzeros = _words(seed, T_ZEROS, K // G, N // 8) & np.uint32(0xEEEEEEEE)
    scales = make_scales(seed, K, N, G)
    g_idx = np.arange(K, dtype=np.int32) // G
    if act_order:
        order = np.argsort(splitmix64(_stream_seed(seed, 9), K), kind="stable")
        g_idx = g_idx[order].astype(np.int32)
    return GPTQProblem(x, qweight, qzeros, scales, g_idx, G)


def _to_bf16_bits_trunc(v: np.ndarray) -> np.ndarray:
    """bf16 bit patterns of float32 values truncated toward zero (input construction only: no rounding
    arithmetic of the method lives here)."""
    return (np.asarray(v, dtype=np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def make_problem_bf16(seed: int, M: int, N: int, K: int, G: int = 128) -> AWQProblem:
    """The bf16 variant's inputs: x and scales as bf16 BIT PATTERNS (uint16; numpy has no bf16):
    X ~ U[-1, 1] and s ~ U[0.004, 0.012] truncated to bf16; codes and zeros as make_problem."""
    u = uniform01(_stream_seed(seed, T_X), M * K)
    x = _to_bf16_bits_trunc(2.0 * u - 1.0).reshape(M, K)
    us = uniform01(_stream_seed(seed, T_SCALES), (K // G) * N)
    s = _to_bf16_bits_trunc(0.004 + 0.008 * us).reshape(K // G, N)
    return AWQProblem(x, make_qweight(seed, K, N), s, make_zeros(seed, K, N, G), G)
