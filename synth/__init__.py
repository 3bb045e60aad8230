"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no unpacking, no dequantization, no GEMM,
no layout).  It only draws random bits with a counter-based SplitMix64 generator and
formats them as the AWQ-style tensors the path consumes:

    X        fp16 [M][K]      activations, U[-1, 1]            (BASELINE.json north_star)
    qweight  uint32 [K][N/8]  random 32-bit words -> every nibble (4-bit code) uniform on [0, 15]
    zeros    uint32 [K/G][N/8] random words -> every 4-bit zero point uniform on [0, 15]
    scales   fp16 [K/G][N]    U[0.004, 0.012] (AWQ magnitude for sigma~0.02 weights at g128)

The recipe is stated in DESIGN.md §3.  Each tensor has its own stream:
seed ^ (tensor_id * 0xD1B54A32D192ED03), tensor_id 0=X, 1=qweight, 2=zeros, 3=scales.
"""
from .splitmix import splitmix64, uniform01
from .awq_inputs import (
    AWQProblem,
    make_x,
    make_qweight,
    make_zeros,
    make_scales,
    make_problem,
    make_structured,
    GPTQProblem,
    make_gptq_problem,
    make_problem_bf16,
)

__all__ = [
    "splitmix64", "uniform01", "AWQProblem", "make_x", "make_qweight", "make_zeros",
    "make_scales", "make_problem", "make_structured", "GPTQProblem", "make_gptq_problem",
    "make_problem_bf16",
]
