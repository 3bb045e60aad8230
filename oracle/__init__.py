"""CPU oracle for the QUICK W4A16 hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import or call anything under oracle/.  The product path (paper_2402_10076_b200/) never does,
and this package imports nothing from it: the two share no code, headers, tables or helpers.
Only the seeded input generators in synth/ (random bits, no method arithmetic) serve both.

Every function is pinned by `tests/test_oracle_pins.py` (marker "not gpu") against closed
forms, brute force, hand-computed golden fixtures and an independent library convention;
see DESIGN.md §2 for the list of pins.  No function here is "parity unpinned".
"""
from .quick_oracle import (  # noqa: F401
    AWQ_ORDER,
    FT_EXTRACT_ORDER,
    unpack_awq,
    pack_awq,
    dequant,
    gemm,
    w4a16_reference,
    round_fp16,
    silu_mul,
    add_bias,
    gptq_dequant,
    bf16_rne,
    bf16_bits,
    bf16_from_bits,
    dequant_bf16,
    gemm_f64,
    tol_check,
    v1_packed_bytes,
    v1_weight_pos,
    v1_meta_offset,
    pack_v1,
    unpack_v1,
)
