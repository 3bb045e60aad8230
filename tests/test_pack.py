"""Offline repack (quick_pack_weights / quick_unpack_weights, C++ in libquick.so) against the
oracle's independent v1 codec: bit-exact blob, exact inverse, bijection, locality."""
import numpy as np
import pytest

import oracle
import synth

quick = pytest.importorskip("paper_2402_10076_b200.quick")


@pytest.mark.parametrize("K,N,G", [(64, 128, 64), (512, 256, 128), (256, 384, 32), (1024, 128, 256),
                                   (192, 256, 96), (512, 1024, 512)])
def test_pack_matches_oracle_encoder(K, N, G):
    p = synth.make_problem(K + N + G, M=1, N=N, K=K, G=G)
    blob = quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)
    ref = oracle.pack_v1(p.qweight, p.scales, p.zeros, G, K, N)
    assert blob.size == quick.quick_packed_bytes(K, N, G) == ref.size
    np.testing.assert_array_equal(blob, ref)


@pytest.mark.parametrize("K,N,G", [(512, 256, 128), (256, 384, 32), (4096, 128, 128)])
def test_unpack_is_exact_inverse_and_matches_oracle_decoder(K, N, G):
    p = synth.make_problem(7, M=1, N=N, K=K, G=G)
    blob = quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)
    qw, s, z = quick.quick_unpack_weights(blob, G, K, N)
    np.testing.assert_array_equal(qw, p.qweight)
    np.testing.assert_array_equal(s.view(np.uint16), p.scales.view(np.uint16))
    np.testing.assert_array_equal(z, p.zeros)
    qo, so, zo = oracle.unpack_v1(blob, G, K, N)
    np.testing.assert_array_equal(qo, p.qweight)
    np.testing.assert_array_equal(so.view(np.uint16), p.scales.view(np.uint16))
    np.testing.assert_array_equal(zo, p.zeros)


def test_roundtrip_many_random_shapes():
    rng = np.random.default_rng(2024)
    for i in range(60):
        G = int(rng.choice([32, 64, 128, 256]))
        K = G * int(rng.integers(1, 6))
        K = K if K % 64 == 0 else K * 2
        N = 128 * int(rng.integers(1, 5))
        qw = rng.integers(0, 2**32, size=(K, N // 8), dtype=np.uint64).astype(np.uint32)
        z = rng.integers(0, 2**32, size=(K // G, N // 8), dtype=np.uint64).astype(np.uint32)
        s = rng.integers(0, 2**16, size=(K // G, N), dtype=np.uint32).astype(np.uint16)  # incl. NaN/Inf bits
        blob = quick.quick_pack_weights(qw, s, z, G)
        q2, s2, z2 = quick.quick_unpack_weights(blob, G, K, N)
        assert np.array_equal(q2, qw) and np.array_equal(s2.view(np.uint16), s) and np.array_equal(z2, z), (K, N, G)


def test_perturbation_locality():
    """Flip one code: exactly one blob nibble changes, at the oracle's v1 position."""
    K, N, G = 256, 256, 64
    p = synth.make_problem(1, M=1, N=N, K=K, G=G)
    blob = quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)
    codes = oracle.unpack_awq(p.qweight)
    for (k, n) in ((0, 0), (255, 255), (37, 130), (64, 127)):
        c2 = codes.copy()
        c2[k, n] ^= 0x5
        blob2 = quick.quick_pack_weights(oracle.pack_awq(c2), p.scales, p.zeros, G)
        diff = np.nonzero(blob != blob2)[0]
        b, i = oracle.v1_weight_pos(k, n, K, N)
        assert diff.tolist() == [int(b)]
        assert ((blob[b] ^ blob2[b]) >> (4 * int(i))) & 0xF == 0x5


def test_pack_is_a_permutation_of_codes():
    """Every nibble of the weights section is one input code: histogram preserved."""
    K, N, G = 512, 256, 128
    p = synth.make_problem(9, M=1, N=N, K=K, G=G)
    blob = quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)
    w = blob[: K * N // 2]
    nib = np.concatenate([w & 0xF, w >> 4])
    np.testing.assert_array_equal(np.bincount(nib, minlength=16),
                                  np.bincount(oracle.unpack_awq(p.qweight).ravel(), minlength=16))


def test_pack_rejects_bad_shapes():
    qw = np.zeros((100, 16), dtype=np.uint32)
    with pytest.raises(quick.QuickError):
        quick.quick_pack_weights(qw, np.zeros((1, 128), np.float16), np.zeros((1, 16), np.uint32), 100)


def _gate_up_columns(cg, cu, I):
    """W' of quick.h's quick_pack_gate_up, written independently: column 128t + 32q + l is gate
    column 64t + 16q + l (l < 16) or up column 64t + 16q + l - 16 (l >= 16)."""
    out = np.empty((cg.shape[0], 2 * I), dtype=cg.dtype)
    for n in range(2 * I):
        t, q, l = n // 128, (n % 128) // 32, n % 32
        src = cu if l >= 16 else cg
        out[:, n] = src[:, 64 * t + 16 * q + (l % 16)]
    return out


@pytest.mark.parametrize("K,I,G", [(256, 64, 64), (512, 192, 128), (128, 320, 32)])
def test_pack_gate_up_matches_oracle_encoder(K, I, G):
    """The fused gate||up blob is the v1 blob of the interleaved matrix W' (the oracle's independent
    v1 encoder applied to W' built column by column here), bit for bit."""
    pg = synth.make_problem(K + I, M=1, N=I, K=K, G=G)
    pu = synth.make_problem(K + I + 1, M=1, N=I, K=K, G=G)
    blob = quick.quick_pack_gate_up((pg.qweight, pg.scales, pg.zeros), (pu.qweight, pu.scales, pu.zeros), G)
    codes = _gate_up_columns(oracle.unpack_awq(pg.qweight), oracle.unpack_awq(pu.qweight), I)
    zeros = _gate_up_columns(oracle.unpack_awq(pg.zeros), oracle.unpack_awq(pu.zeros), I)
    scales = _gate_up_columns(pg.scales.view(np.uint16), pu.scales.view(np.uint16), I).view(np.float16)
    ref = oracle.pack_v1(oracle.pack_awq(codes), scales, oracle.pack_awq(zeros), G, K, 2 * I)
    assert np.array_equal(blob, ref)


def test_pack_gate_up_rejects_bad_shapes():
    pg = synth.make_problem(1, M=1, N=96, K=128, G=64)   # I = 96: not a multiple of 64
    with pytest.raises(quick.QuickError):
        quick.quick_pack_gate_up((pg.qweight, pg.scales, pg.zeros), (pg.qweight, pg.scales, pg.zeros), 64)
    pu = synth.make_problem(1, M=1, N=128, K=128, G=64)
    pg = synth.make_problem(1, M=1, N=64, K=128, G=64)
    with pytest.raises(ValueError):
        quick.quick_pack_gate_up((pg.qweight, pg.scales, pg.zeros), (pu.qweight, pu.scales, pu.zeros), 64)


# ------------------------------------------------------------------ GPTQ import (f3)
@pytest.mark.parametrize("K,N,G,act", [(256, 128, 64, True), (512, 256, 128, True), (256, 128, 32, False)])
def test_import_gptq_reorders_rows_by_group(K, N, G, act):
    """quick_import_gptq: the imported AWQ tensors dequantize (oracle O2) to the GPTQ weights (oracle O8)
    with the rows in the order perm, bit for bit; perm sorts the rows by group."""
    p = synth.make_gptq_problem(K + N, M=1, N=N, K=K, G=G, act_order=act)
    qa, sa, za, perm = quick.quick_import_gptq(p.qweight, p.qzeros, p.scales, G, g_idx=p.g_idx if act else None)
    w_gptq = oracle.gptq_dequant(p.qweight, p.qzeros, p.scales, g_idx=p.g_idx if act else None, group_size=G)
    w_imp = oracle.dequant(qa, sa, za, G)
    assert np.array_equal(w_imp.view(np.uint16), w_gptq[perm].view(np.uint16))
    assert np.array_equal(np.sort(perm), np.arange(K))
    gi = p.g_idx if act else np.arange(K) // G
    assert np.array_equal(gi[perm], np.arange(K) // G)
    if not act:
        assert np.array_equal(perm, np.arange(K))


def test_import_gptq_rejects_unrepresentable_zero_and_ragged_groups():
    p = synth.make_gptq_problem(3, M=1, N=128, K=256, G=64)
    bad = p.qzeros.copy()
    bad[0, 0] |= np.uint32(0xF)            # stored 15 -> decoded zero 16 in a v1 checkpoint
    with pytest.raises(quick.QuickError):
        quick.quick_import_gptq(p.qweight, bad, p.scales, 64, g_idx=p.g_idx)
    quick.quick_import_gptq(p.qweight, bad, p.scales, 64, g_idx=p.g_idx, zero_plus_one=False)   # v2: zero 15
    g = p.g_idx.copy()
    g[0] = (g[0] + 1) % 4                  # one group with G + 1 rows, another with G - 1
    with pytest.raises(quick.QuickError):
        quick.quick_import_gptq(p.qweight, p.qzeros, p.scales, 64, g_idx=g)
