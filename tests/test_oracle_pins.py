"""Pins of the CPU oracle against things other than itself.

Each test names what it pins and where the expected value comes from: a closed form, a
hand-computed golden fixture (tests/golden/, each with its citation), brute force in exact
rational / integer arithmetic, or an independent library's statement of the same convention.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from _helpers import golden_lines


# ------------------------------------------------------------------ independent fp16 rounding
def _rne_fp16_bits(num: int, exp2: int, neg: bool) -> int:
    """fp16 bits of round-to-nearest-even(num * 2^exp2), num >= 0, in pure integer arithmetic."""
    sign = 0x8000 if neg else 0
    if num == 0:
        return sign
    E = num.bit_length() - 1 + exp2          # value in [2^E, 2^(E+1))
    qe = max(E - 10, -24)                     # quantum exponent of that binade (or subnormal)
    if exp2 >= qe:
        m = num << (exp2 - qe)
    else:
        sh = qe - exp2
        m = num >> sh
        rem = num - (m << sh)
        half = 1 << (sh - 1)
        if rem > half or (rem == half and (m & 1)):
            m += 1
    if m < 1024:                              # subnormal (qe == -24)
        return sign | m
    while m >= 2048:                          # carry into the next binade (exact)
        m >>= 1
        qe += 1
    e_biased = qe + 10 + 15
    if e_biased >= 31:
        return sign | 0x7C00                  # overflow -> inf
    return sign | (e_biased << 10) | (m - 1024)


def _fp16_parts(bits: int):
    """(integer significand, exponent) with value = sig * 2^exp for a finite fp16 bit pattern."""
    e = (bits >> 10) & 0x1F
    f = bits & 0x3FF
    if e == 0:
        return f, -24
    return f | 0x400, e - 25


def test_fp16_rounding_routine_self_consistency():
    # every finite fp16 value must round to itself
    for bits in range(0, 0x7C00, 7):
        sig, ex = _fp16_parts(bits)
        assert _rne_fp16_bits(sig, ex, False) == bits


# ------------------------------------------------------------------ O1 unpack / packing order
def test_awq_hand_word():
    """Codes [1..8] for columns 0..7 in AWQ order pack to 0x86427531 (hand-derived:
    nibble i holds column [0,2,4,6,1,3,5,7][i]); SPEC's natural order would give 0x87654321
    (S:L80), which the AWQ convention is not."""
    codes = np.arange(1, 9, dtype=np.uint8)[None, :]
    assert int(oracle.pack_awq(codes)[0, 0]) == 0x86427531
    assert oracle.unpack_awq(np.array([[0x86427531]], dtype=np.uint32)).tolist() == [list(range(1, 9))]
    assert int(oracle.pack_awq(codes)[0, 0]) != 0x87654321


def test_awq_order_matches_vllm_awq_pack():
    """Library pin: vLLM's awq_pack (AutoAWQ checkpoint convention) agrees with pack_awq."""
    try:
        import torch
        from vllm.model_executor.layers.quantization.utils.quant_utils import awq_pack
    except Exception as e:  # pragma: no cover - vllm absent
        pytest.skip(f"vllm not importable: {e}")
    rng = np.random.default_rng(3)
    K, N = 16, 64
    codes = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
    ref = awq_pack(torch.from_numpy(codes.astype(np.int32)), 4, K, N).numpy().view(np.uint32)
    np.testing.assert_array_equal(oracle.pack_awq(codes), ref)
    np.testing.assert_array_equal(oracle.unpack_awq(ref), codes)


def test_ft_extraction_order_emulated():
    """Fig. 5 / P:L107 'dequant-aware reorder': emulate the FasterTransformer LOP3 magic-number
    extraction bit-by-bit and check (a) it emits nibbles in FT_EXTRACT_ORDER and (b) AWQ_ORDER is
    its inverse, so AWQ-ordered words come out sequential."""
    def extract(word):
        outs = []
        for w in (word, word >> 8):
            lo = (w & 0x000F000F) | 0x64006400      # fp16 1024 + nibble
            hi = (w & 0x00F000F0) | 0x64006400      # fp16 1024 + 16*nibble
            lo_h = np.array([lo & 0xFFFF, lo >> 16], dtype=np.uint16).view(np.float16).astype(np.float64)
            hi_h = np.array([hi & 0xFFFF, hi >> 16], dtype=np.uint16).view(np.float16).astype(np.float64)
            outs.append(lo_h - 1024.0)
            outs.append(hi_h / 16.0 - 64.0)
        return [int(v) for pair in outs for v in pair]
    word = sum(i << (4 * i) for i in range(8))       # nibble i holds value i
    assert extract(word) == list(oracle.FT_EXTRACT_ORDER)
    assert [oracle.AWQ_ORDER[j] for j in oracle.FT_EXTRACT_ORDER] == list(range(8))
    codes = np.arange(8, dtype=np.uint8)[None, :] + 3
    assert extract(int(oracle.pack_awq(codes)[0, 0])) == list(range(3, 11))


def test_unpack_awq_roundtrip_random():
    rng = np.random.default_rng(0)
    w = rng.integers(0, 2**32, size=(37, 24), dtype=np.uint64).astype(np.uint32)
    np.testing.assert_array_equal(oracle.pack_awq(oracle.unpack_awq(w)), w)


# ------------------------------------------------------------------ O2 dequant
def _single_dequant(code, zero, scale_bits):
    qw = np.full((1, 1), sum(code << (4 * i) for i in range(8)), dtype=np.uint32)
    zw = np.full((1, 1), sum(zero << (4 * i) for i in range(8)), dtype=np.uint32)
    s = np.full((1, 8), scale_bits, dtype=np.uint16).view(np.float16)
    return oracle.dequant(qw, s, zw, 1).view(np.uint16)[0]


def test_dequant_golden_examples():
    """tests/golden/dequant_examples.txt: SPEC S:L71-73 and hand-derived fp16 cases."""
    rows = golden_lines("dequant_examples.txt")
    assert len(rows) >= 10
    for code, zero, sbits, ebits in rows:
        got = _single_dequant(int(code), int(zero), int(sbits, 16))
        assert all(int(g) == int(ebits, 16) for g in got), (code, zero, sbits, ebits, got)


def test_dequant_exhaustive_vs_integer_rounding():
    """Brute force: every (q, z) pair and every positive finite fp16 scale, against the
    pure-integer round-to-nearest-even above (no float arithmetic on the reference side)."""
    pos_bits = np.arange(0, 0x7C00, dtype=np.uint32)          # 31744 finite non-negative scales
    table = np.empty((16, pos_bits.size), dtype=np.uint16)
    for b in pos_bits.tolist():
        sig, ex = _fp16_parts(b)
        for d in range(16):
            table[d, b] = _rne_fp16_bits(d * sig, ex, False)
    # oracle side: K = G = 16 rows with code q = k; every column carries one (z, s) pair
    zs = np.repeat(np.arange(16, dtype=np.uint8), pos_bits.size)   # column -> z
    sb = np.tile(pos_bits, 16).astype(np.uint16)                   # column -> scale bits
    N = zs.size
    codes = np.repeat(np.arange(16, dtype=np.uint8)[:, None], N, axis=1)
    w = oracle.dequant(oracle.pack_awq(codes), sb.view(np.float16)[None, :],
                       oracle.pack_awq(zs[None, :]), 16).view(np.uint16)
    d = np.arange(16)[:, None].astype(np.int64) - zs[None, :].astype(np.int64)
    exp = table[np.abs(d), np.tile(pos_bits, 16)[None, :]]
    exp = np.where(d < 0, exp ^ 0x8000, exp)                   # sign of (q - z) * s with s > 0
    np.testing.assert_array_equal(w, exp.astype(np.uint16))


def test_dequant_negative_scales_sample():
    rng = np.random.default_rng(1)
    for b in rng.integers(0x8000, 0xFC00, size=200).tolist():
        sig, ex = _fp16_parts(b & 0x7FFF)
        for q, z in ((5, 3), (0, 15), (9, 9), (15, 0)):
            d = q - z
            # s < 0: the product is negative iff d > 0; (+0) * s = -0
            exp = _rne_fp16_bits(abs(d) * sig, ex, neg=(d > 0)) if d != 0 else 0x8000
            got = int(_single_dequant(q, z, b)[0])
            assert got == exp, (q, z, hex(b), hex(got), hex(exp))


def test_dequant_group_indexing():
    """Group g covers k in [gG, (g+1)G): a different scale per group must show up exactly there."""
    K, N, G = 8, 8, 2
    codes = np.full((K, N), 5, dtype=np.uint8)
    zeros = np.full((K // G, N), 3, dtype=np.uint8)
    scales = np.array([[0.5], [0.25], [2.0], [-1.0]], dtype=np.float16).repeat(N, axis=1)
    w = oracle.dequant(oracle.pack_awq(codes), scales, oracle.pack_awq(zeros), G).astype(np.float64)
    expect = np.repeat(np.array([1.0, 0.5, 4.0, -2.0]), G)[:, None] * np.ones((1, N))
    np.testing.assert_array_equal(w, expect)


# ------------------------------------------------------------------ O3 GEMM
def _golden_tiny():
    rows = {r[0]: r[1:] for r in golden_lines("tiny_gemm.txt")}
    qweight = np.array([int(v, 16) for v in rows["qweight"]], dtype=np.uint32)[:, None]
    zeros = np.array([int(v, 16) for v in rows["zeros"]], dtype=np.uint32)[:, None]
    scales = np.array([int(v, 16) for v in rows["scales"]], dtype=np.uint16)[:, None].repeat(8, axis=1).view(np.float16)
    x = np.array([[float(v) for v in rows["x0"]], [float(v) for v in rows["x1"]]], dtype=np.float16)
    y = np.array([[float(v) for v in rows["y0"]], [float(v) for v in rows["y1"]]])
    return x, qweight, scales, zeros, y


def test_gemm_golden_tiny():
    x, qw, s, z, y = _golden_tiny()
    np.testing.assert_array_equal(oracle.w4a16_reference(x, qw, s, z, 2), y)


def test_gemm_brute_force_fractions():
    """Exact rational dot products on a tiny random problem; fp64 must agree to ~1e-15."""
    p = synth.make_problem(11, M=3, N=8, K=16, G=8)
    w = oracle.dequant(p.qweight, p.scales, p.zeros, 8)
    y = oracle.gemm(p.x, w)
    for m in range(3):
        for n in range(8):
            exact = sum(Fraction(float(p.x[m, k])) * Fraction(float(w[k, n])) for k in range(16))
            mag = sum(abs(float(p.x[m, k]) * float(w[k, n])) for k in range(16))
            assert abs(Fraction(y[m, n]) - exact) <= Fraction(mag) * Fraction(1, 2**45)


def test_gemm_integer_exact_regime():
    """s = 2^-6, X in {-1,0,1}: Y * 2^6 is the integer matrix X . (q - z), computed in int64."""
    p = synth.make_structured("intexact", 5, M=9, N=256, K=512, G=128)
    q = oracle.unpack_awq(p.qweight).astype(np.int64)
    z = np.repeat(oracle.unpack_awq(p.zeros).astype(np.int64), 128, axis=0)
    yint = p.x.astype(np.int64) @ (q - z)
    y = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
    np.testing.assert_array_equal(y * 64.0, yint.astype(np.float64))
    assert np.abs(yint).max() < 2048
    np.testing.assert_array_equal(oracle.round_fp16(y).astype(np.float64), y)   # fp16-exact


def test_gemm_onehot_rows():
    p = synth.make_structured("onehot", 2, M=16, N=128, K=256, G=128)
    w = oracle.dequant(p.qweight, p.scales, p.zeros, 128).astype(np.float64)
    y = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
    idx = np.argmax(p.x, axis=1)
    np.testing.assert_array_equal(y, w[idx, :])


def test_gemm_zero_weights():
    p = synth.make_structured("zero_weights", 4, M=5, N=128, K=256, G=64)
    y = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 64)
    assert np.all(y == 0.0)


def test_gemm_ones_column_sums_exact():
    """X = ones: Y[m][n] = column sum of dequant(W), checked with exact Fractions."""
    p = synth.make_problem(8, M=2, N=16, K=64, G=32)
    x = np.ones((2, 64), dtype=np.float16)
    w = oracle.dequant(p.qweight, p.scales, p.zeros, 32)
    y = oracle.gemm(x, w)
    for n in range(16):
        exact = sum(Fraction(float(w[k, n])) for k in range(64))
        assert Fraction(y[0, n]) == exact      # < 2^53 dyadic: fp64 sum is exact here


def test_gemm_vs_torch_fp64():
    import torch
    p = synth.make_problem(1, M=7, N=256, K=384, G=128)
    w = oracle.dequant(p.qweight, p.scales, p.zeros, 128)
    y = oracle.gemm(p.x, w)
    yt = torch.from_numpy(p.x.astype(np.float64)) @ torch.from_numpy(w.astype(np.float64))
    np.testing.assert_allclose(y, yt.numpy(), rtol=1e-13, atol=1e-13)


# ------------------------------------------------------------------ O5 tolerance
def test_tol_check_hand_cases():
    ok = oracle.tol_check(np.array([1.0099, 0.0059, -2.0]), np.array([1.0, 0.005, -2.02]))
    assert ok["ok"], ok
    bad = oracle.tol_check(np.array([1.011]), np.array([1.0]))
    assert not bad["ok"] and bad["first_fail"] == (0,)
    assert not oracle.tol_check(np.array([0.0061]), np.array([0.005]))["ok"]
    assert not oracle.tol_check(np.array([np.nan]), np.array([0.5]))["ok"]
    assert not oracle.tol_check(np.array([np.inf]), np.array([0.5]))["ok"]
    assert oracle.tol_check(np.array([0.0109]), np.array([0.011]))["ok"]   # relative regime


# ------------------------------------------------------------------ O6 v1 layout
def test_v1_golden_positions():
    K, N, G = 64, 256, 64
    for row in golden_lines("v1_positions.txt"):
        if row[0] == "meta":
            t, g, off = map(int, row[1:])
            assert oracle.v1_meta_offset(t, g, K, N, G) == off
        else:
            k, n, byte, nib = map(int, row)
            b, i = oracle.v1_weight_pos(k, n, K, N)
            assert (int(b), int(i)) == (byte, nib), row


@pytest.mark.parametrize("K,N", [(64, 128), (128, 256), (512, 384), (4096, 128)])
def test_v1_position_bijection(K, N):
    kk, nn = np.meshgrid(np.arange(K), np.arange(N), indexing="ij")
    b, i = oracle.v1_weight_pos(kk.ravel(), nn.ravel(), K, N)
    slot = 2 * b + i
    assert slot.min() == 0 and slot.max() == K * N - 1
    assert np.unique(slot).size == K * N


def test_v1_roundtrip_and_locality():
    p = synth.make_problem(3, M=1, N=256, K=256, G=64)
    blob = oracle.pack_v1(p.qweight, p.scales, p.zeros, 64, 256, 256)
    qw, s, z = oracle.unpack_v1(blob, 64, 256, 256)
    np.testing.assert_array_equal(qw, p.qweight)
    np.testing.assert_array_equal(s.view(np.uint16), p.scales.view(np.uint16))
    np.testing.assert_array_equal(z, p.zeros)
    # flipping one input nibble changes exactly one blob nibble
    codes = oracle.unpack_awq(p.qweight)
    codes[77, 201] ^= 0x9
    blob2 = oracle.pack_v1(oracle.pack_awq(codes), p.scales, p.zeros, 64, 256, 256)
    diff = np.nonzero(blob != blob2)[0]
    b, i = oracle.v1_weight_pos(77, 201, 256, 256)
    assert diff.tolist() == [int(b)]
    assert ((blob[diff[0]] ^ blob2[diff[0]]) >> (4 * int(i))) & 0xF == 0x9


def test_v1_packed_bytes():
    assert oracle.v1_packed_bytes(4096, 4096, 128) == 4096 * 4096 // 2 + 32 * 4096 * 5 // 2
    assert oracle.v1_packed_bytes(100, 128, 4) == 0
    assert oracle.v1_packed_bytes(128, 100, 128) == 0


# ------------------------------------------------------------------ synthetic inputs
def test_splitmix64_reference_vector():
    """Published SplitMix64 outputs for seed 0 (Vigna's reference implementation)."""
    z = synth.splitmix64(0, 3)
    assert [hex(int(v)) for v in z] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x6c45d188009454f"]


def test_synth_ranges_and_determinism():
    p = synth.make_problem(0, 4, 256, 512, 128)
    q = synth.make_problem(0, 4, 256, 512, 128)
    assert np.array_equal(p.x.view(np.uint16), q.x.view(np.uint16))
    assert np.abs(p.x.astype(np.float64)).max() <= 1.0
    s = p.scales.astype(np.float64)
    assert s.min() >= 0.0039 and s.max() <= 0.0121
    assert p.qweight.dtype == np.uint32 and p.qweight.shape == (512, 32)


# ------------------------------------------------------------------ O7 silu_mul (R16)
def test_silu_mul_closed_forms():
    """SiLU(0) = 0; SiLU(1) = 1 / (1 + e^-1) (decimal value of the logistic function at 1, computed
    here with the standard-library exp, not numpy); SiLU(x) - SiLU(-x) = x for every x (since
    sigmoid(x) + sigmoid(-x) = 1); SiLU(x) -> x for large x and -> 0 for very negative x; and the
    factor u enters linearly."""
    import math
    assert oracle.silu_mul(0.0, 5.0) == 0.0
    assert abs(oracle.silu_mul(1.0, 1.0) - 1.0 / (1.0 + math.exp(-1.0))) < 1e-15
    assert abs(oracle.silu_mul(1.0, 1.0) - 0.7310585786300049) < 1e-15
    x = np.linspace(-12, 12, 97)
    np.testing.assert_allclose(oracle.silu_mul(x, 1.0) - oracle.silu_mul(-x, 1.0), x, rtol=0, atol=1e-12)
    assert abs(oracle.silu_mul(40.0, 1.0) - 40.0) < 1e-12
    assert abs(oracle.silu_mul(-40.0, 1.0)) < 1e-15
    np.testing.assert_allclose(oracle.silu_mul(x, 3.0), 3.0 * oracle.silu_mul(x, 1.0), rtol=1e-15)


def test_silu_mul_against_torch():
    """The library statement of the same activation: torch.nn.functional.silu in float64."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    g, u = rng.normal(0, 4, 1000), rng.normal(0, 1, 1000)
    ref = (torch.nn.functional.silu(torch.from_numpy(g)) * torch.from_numpy(u)).numpy()
    np.testing.assert_allclose(oracle.silu_mul(g, u), ref, rtol=1e-13, atol=1e-300)


# ------------------------------------------------------------------ O8 gptq_dequant (R17)
def test_gptq_dequant_hand_example():
    """Hand-computed: one column block, rows 0..7 hold codes 1..8 (word 0x87654321, nibble i = row i),
    stored zero 7 in a v1 checkpoint (decoded zero 8), scale 0.5: w[k] = (k + 1 - 8) * 0.5."""
    K, N, G = 8, 8, 8
    qweight = np.full((K // 8, N), 0x87654321, dtype=np.uint32)
    qzeros = np.array([[0x77777777]], dtype=np.uint32)
    scales = np.full((1, N), 0.5, dtype=np.float16)
    w = oracle.gptq_dequant(qweight, qzeros, scales, group_size=G)
    expect = np.array([-3.5, -3.0, -2.5, -2.0, -1.5, -1.0, -0.5, 0.0])
    for n in range(N):
        assert w[:, n].astype(np.float64).tolist() == expect.tolist()
    # "v2" (zeros stored as is): decoded zero 7
    w2 = oracle.gptq_dequant(qweight, qzeros, scales, group_size=G, zero_plus_one=False)
    assert w2[:, 0].astype(np.float64).tolist() == (expect + 0.5).tolist()


def test_gptq_packing_order_matches_vllm():
    """vLLM's gptq_pack (pack_rows: 8 rows per word) and pack_cols (8 columns per word, natural order)
    are the library statement of the AutoGPTQ layout: with unit scales and zero 0 (v2) the oracle
    returns the packed codes; with act-order g_idx each row takes its own group's zero and scale."""
    torch = pytest.importorskip("torch")
    qu = pytest.importorskip("vllm.model_executor.layers.quantization.utils.quant_utils")
    rng = np.random.default_rng(11)
    K, N, G = 64, 32, 16
    codes = rng.integers(0, 16, (K, N))
    qweight = qu.pack_rows(torch.from_numpy(codes), 4, K, N).numpy().view(np.uint32)
    zeros = rng.integers(0, 16, (K // G, N))
    qzeros = qu.pack_cols(torch.from_numpy(zeros), 4, K // G, N).numpy().view(np.uint32)
    ones = np.ones((K // G, N), np.float16)
    w = oracle.gptq_dequant(qweight, np.zeros_like(qzeros), ones, group_size=G, zero_plus_one=False)
    assert np.array_equal(w.astype(np.int64), codes)
    g_idx = rng.permutation(np.arange(K) // G)
    scales = (rng.integers(1, 64, (K // G, N)) / 64).astype(np.float16)
    w = oracle.gptq_dequant(qweight, qzeros, scales, g_idx=g_idx, zero_plus_one=False)
    ref = ((codes - zeros[g_idx]) * scales.astype(np.float64)[g_idx]).astype(np.float16)   # exact products
    assert np.array_equal(w.view(np.uint16), ref.view(np.uint16))


def test_gptq_v2_without_act_order_is_the_awq_dequant():
    """Same codes, zeros and scales written in the two checkpoint layouts: O8 (GPTQ, v2 zeros) equals
    O2 (AWQ), whose packing order is pinned against vLLM's awq_pack above."""
    p = synth.make_problem(17, M=1, N=64, K=128, G=32)
    codes = oracle.unpack_awq(p.qweight)
    zeros = oracle.unpack_awq(p.zeros)
    qweight = np.zeros((128 // 8, 64), np.uint32)
    for i in range(8):
        qweight |= (codes[i::8, :].astype(np.uint32) << np.uint32(4 * i))
    qzeros = np.zeros((4, 8), np.uint32)
    for i in range(8):
        qzeros |= (zeros[:, i::8].astype(np.uint32) << np.uint32(4 * i))
    w_gptq = oracle.gptq_dequant(qweight, qzeros, p.scales, group_size=32, zero_plus_one=False)
    w_awq = oracle.dequant(p.qweight, p.scales, p.zeros, 32)
    assert np.array_equal(w_gptq.view(np.uint16), w_awq.view(np.uint16))


# ------------------------------------------------------------------ O9 bf16 (R18)
def _rne_bits_exact(fr: Fraction, p: int = 8):
    """round-to-nearest-even of a positive Fraction to p significant bits, exactly (Fraction result)."""
    e = 0
    while fr >= 2:
        fr /= 2
        e += 1
    while fr < 1:
        fr *= 2
        e -= 1
    scaled = fr * (1 << (p - 1))
    n = scaled.numerator // scaled.denominator
    rem = scaled - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return Fraction(n) / (1 << (p - 1)) * (Fraction(2) ** e)


def test_bf16_rne_against_torch_and_exact_rounding():
    """bf16_rne == torch's float32 -> bfloat16 conversion (library, round-to-nearest-even) on random fp32
    values, ties included; and == exact rational RNE to 8 bits on hand-picked ties."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    bits = rng.integers(0x3000_0000, 0x4F00_0000, 20000, dtype=np.uint32)
    bits[:2000] = (bits[:2000] & np.uint32(0xFFFF0000)) | np.uint32(0x8000)   # exact ties
    vals = bits.view(np.float32)
    ref = torch.from_numpy(vals.copy()).to(torch.bfloat16).to(torch.float64).numpy()
    got = oracle.bf16_rne(vals.astype(np.float64))
    assert np.array_equal(got, ref)
    for v in (Fraction(257, 256), Fraction(259, 256), Fraction(3, 1) + Fraction(1, 64), Fraction(12345, 1024)):
        assert oracle.bf16_rne(float(v)) == float(_rne_bits_exact(v))


def test_bf16_dequant_exhaustive_codes():
    """Every (q, z) against 64 bf16 scales: bf16_rne((q - z) s) equals exact rational RNE, with the sign."""
    K, N, G = 16, 64 * 16, 16
    sbits = np.arange(64, dtype=np.uint16) * np.uint16(0x0103) + np.uint16(0x3A00)   # assorted positive scales
    cols = np.arange(N)
    z = (cols % 16).astype(np.uint8)
    s = sbits[(cols // 16) % 64]
    codes = np.tile((np.arange(K) % 16).astype(np.uint8)[:, None], (1, N))
    w = oracle.dequant_bf16(oracle.pack_awq(codes), s[None, :], oracle.pack_awq(z[None, :]), G)
    sv = oracle.bf16_from_bits(s)
    for k in range(K):
        for n in range(0, N, 7):
            d = int(codes[k, n]) - int(z[n])
            exact = Fraction(d) * Fraction(float(sv[n]))
            want = 0.0 if d == 0 else float(_rne_bits_exact(abs(exact))) * (1 if d > 0 else -1)
            assert w[k, n] == want, (k, n, d, sv[n])


def test_bf16_gemm_integer_exact_regime():
    """Small-integer X and power-of-two bf16 scales: every partial sum is exact, so O9's GEMM equals the
    int64 matmul of codes scaled once."""
    rng = np.random.default_rng(9)
    K, N, M, G = 256, 128, 4, 128
    codes = rng.integers(0, 16, (K, N))
    zeros = rng.integers(0, 16, (K // G, N))
    sb = np.full((K // G, N), 0x3C00, dtype=np.uint16)    # bf16 bits of 2^-7
    x = rng.integers(-2, 3, (M, K)).astype(np.float64)
    w = oracle.dequant_bf16(oracle.pack_awq(codes), sb, oracle.pack_awq(zeros), G)
    y = oracle.gemm_f64(x, w)
    ref = (x.astype(np.int64) @ (codes - zeros[np.arange(K) // G]).astype(np.int64)).astype(np.float64) * 2.0 ** -7
    assert np.array_equal(y, ref)


# ------------------------------------------------------------------------------------------ O10
def test_add_bias_pins():
    """O10 (R21): zero weights give Y = b exactly; in the integer-exact regime with an
    integer bias, 64 (Y + b) is the int64 matrix X . (q - z) + 64 b; each row gets the same b;
    Fraction brute force on a tiny random problem."""
    pz = synth.make_structured("zero_weights", 4, M=3, N=128, K=256, G=64)
    b = (np.arange(128) % 17 - 8).astype(np.float16) * np.float16(0.25)
    y = oracle.add_bias(oracle.w4a16_reference(pz.x, pz.qweight, pz.scales, pz.zeros, 64), b)
    np.testing.assert_array_equal(y, np.tile(b.astype(np.float64), (3, 1)))
    p = synth.make_structured("intexact", 5, M=9, N=256, K=512, G=128)
    bi = ((np.arange(256) % 9) - 4).astype(np.float16)            # integers: exact in fp16
    q = oracle.unpack_awq(p.qweight).astype(np.int64)
    z = np.repeat(oracle.unpack_awq(p.zeros).astype(np.int64), 128, axis=0)
    yint = p.x.astype(np.int64) @ (q - z) + 64 * bi.astype(np.int64)[None, :]
    y = oracle.add_bias(oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128), bi)
    np.testing.assert_array_equal(y * 64.0, yint.astype(np.float64))
    pr = synth.make_problem(13, M=2, N=8, K=16, G=8)
    br = np.array([0.5, -1.25, 3.0, 0.0, -0.0078125, 2.5, 1.0, -3.5], dtype=np.float16)
    w = oracle.dequant(pr.qweight, pr.scales, pr.zeros, 8)
    yr = oracle.add_bias(oracle.gemm(pr.x, w), br)
    for m in range(2):
        for n in range(8):
            exact = sum(Fraction(float(pr.x[m, k])) * Fraction(float(w[k, n])) for k in range(16)) + Fraction(float(br[n]))
            assert abs(Fraction(yr[m, n]) - exact) <= Fraction(1, 2**40)
