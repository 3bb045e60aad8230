"""Plain, slow, obviously-correct CPU oracle of the QUICK W4A16 path (numpy, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

What the path computes (PAPER.md = /root/reference/PAPER.md, "P:L<n>" = its line n):

  O1 unpack   q[k][n] = 4-bit code of weight (k, n) from AWQ-packed words
              ("extract target sub-byte weights", §2.3; "128-bit weight vectors
              consisting of 32 4-bit weights").  Packing convention = AWQ "GEMM"
              checkpoint order (reading R2).
  O2 dequant  w[k][n] = fp16_rne((q[k][n] - z[g][n]) * s[g][n]), g = k // G
              ("apply zero points and scales", §2.3; fp16 result, "half-precision
              additions and multiplications"; asymmetric form = reading R1).
              (q - z) * s is exact in fp64 (<= 4 + 11 significant bits), so the single
              fp16 rounding is the only rounding.
  O3 gemm     Y[m][n] = sum_k x[m][k] * w[k][n], fp16 operands, accumulated in fp64
              ("mixed precision GEMM", §2.3; Y = X . dequant(Wq)).  Each product is
              exact in fp64; the fp64 sum is the reference the tolerance is measured from.
  O4 output   fp16_rne(Y) is the bit-exact reference where Y is exactly representable.
  O5 tol      BASELINE.json north_star: |y - ref| <= 1e-2 |ref|, or <= 1e-3 where |ref| < 1e-2.
  O6 v1 blob  the packed layout of DESIGN.md §4 (this build's offline interleave, the B200
              form of §3.2): an independent encoder/decoder written from the layout
              text, used to check the library packer bit-for-bit.

  O9 bf16     (the bf16 variant; R18): bf16 activations, scales and
              output.  bf16_rne rounds to 8 significant bits (round half to even, exponent range
              of fp32); dequant w = bf16_rne((q - z) * s) (the product is exact in fp64); the GEMM
              sums exact products in fp64 like O3; bf16 values are carried as float64 arrays and
              as uint16 bit patterns (numpy has no bf16 dtype).
  O8 gptq     (GPTQ is the P:L19 family): dequantization of an AutoGPTQ
              checkpoint, w[k][n] = fp16_rne((q[k][n] - z[g_idx[k]][n]) * s[g_idx[k]][n]),
              q packed 8 rows per word (nibble i = row 8j + i), z packed 8 columns per word
              (nibble i = column 8j + i) and stored as z - 1 in "v1" checkpoints (R17).
  O7 silu_mul (the fused gate||up epilogue; not in PAPER.md, whose MLP is
              not on its hot path -- DESIGN.md reading R16): h = SiLU(g) * u with
              SiLU(g) = g / (1 + exp(-g)) (the Llama/Mistral MLP activation), in fp64 on the
              two O3 results.
  O10 bias    (SURVEY §8(f) f2 "bias"; not in PAPER.md -- DESIGN.md reading R21):
              Y[m][n] = sum_k x[m][k] w[k][n] + b[n], the bias a 16-bit value added once to the
              exact (fp64) O3 sum, then one rounding (O4).

No blocking, fusion or reordering beyond the definitions above; numpy's fp64 matmul is the
one library primitive used (as a step: a dot product in fp64).
"""
import numpy as np

# AWQ "GEMM" packing: nibble i (bits 4i..4i+3) of a word holds column 8j + AWQ_ORDER[i].
# (R2; pinned against vLLM's awq_pack and a hand-computed word in tests.)
AWQ_ORDER = (0, 2, 4, 6, 1, 3, 5, 7)
# FasterTransformer LOP3 i4->f16 extraction emits nibbles in this order (Fig. 5):
# output slot j is nibble FT_EXTRACT_ORDER[j].  AWQ_ORDER is its inverse permutation, so
# "dequant-aware reordered" words come out in sequential order (pinned by emulation in tests).
FT_EXTRACT_ORDER = (0, 4, 1, 5, 2, 6, 3, 7)


# ----------------------------------------------------------------------------------------- O1
def unpack_awq(words: np.ndarray) -> np.ndarray:
    """O1: AWQ-packed uint32 [R][N/8] -> 4-bit codes uint8 [R][N]."""
    words = np.asarray(words, dtype=np.uint32)
    R, W = words.shape
    codes = np.empty((R, W * 8), dtype=np.uint8)
    for i in range(8):
        codes[:, AWQ_ORDER[i]::8] = ((words >> np.uint32(4 * i)) & np.uint32(0xF)).astype(np.uint8)
    return codes


def pack_awq(codes: np.ndarray) -> np.ndarray:
    """Inverse of O1: codes uint8 [R][N] (values 0..15) -> AWQ-packed uint32 [R][N/8]."""
    codes = np.asarray(codes, dtype=np.uint32)
    R, N = codes.shape
    assert N % 8 == 0
    words = np.zeros((R, N // 8), dtype=np.uint32)
    for i in range(8):
        words |= (codes[:, AWQ_ORDER[i]::8] & np.uint32(0xF)) << np.uint32(4 * i)
    return words


# ----------------------------------------------------------------------------------------- O2
def dequant(qweight: np.ndarray, scales: np.ndarray, zeros: np.ndarray, group_size: int) -> np.ndarray:
    """O2: w[k][n] = fp16_rne((q - z) * s) with g = k // G (§2.3).  Returns float16 [K][N]."""
    q = unpack_awq(qweight).astype(np.float64)               # [K][N]
    z = unpack_awq(zeros).astype(np.float64)                 # [K/G][N]
    s = np.asarray(scales, dtype=np.float16).astype(np.float64)  # [K/G][N]
    K, N = q.shape
    G = int(group_size)
    assert K % G == 0 and z.shape == (K // G, N) and s.shape == (K // G, N)
    g_of_k = np.arange(K) // G
    exact = (q - z[g_of_k, :]) * s[g_of_k, :]                # exact in fp64
    with np.errstate(over="ignore"):
        return exact.astype(np.float16)                      # one round-to-nearest-even (inf past 65504)


# ----------------------------------------------------------------------------------------- O3
def gemm(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """O3: Y = X . W with fp16 operands, fp64 accumulation.  Returns float64 [M][N]."""
    x64 = np.asarray(x, dtype=np.float16).astype(np.float64)
    w64 = np.asarray(w, dtype=np.float16).astype(np.float64)
    return x64 @ w64


def w4a16_reference(x, qweight, scales, zeros, group_size) -> np.ndarray:
    """O1 -> O2 -> O3: the fp64 reference of Y = X . dequant(Wq)."""
    return gemm(x, dequant(qweight, scales, zeros, group_size))


# ----------------------------------------------------------------------------------------- O9
def bf16_rne(x) -> np.ndarray:
    """O9: round float64 values to bf16 (8 significant bits, nearest, ties to even), returned as
    float64.  Finite inputs well inside the fp32 exponent range (the path's values) only."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                              # x = m 2^e, 0.5 <= |m| < 1
    r = np.rint(np.ldexp(m, 8))                     # 8 significant bits; np.rint ties to even
    return np.ldexp(r, e - 8)


def bf16_bits(x) -> np.ndarray:
    """uint16 bit patterns of bf16-representable float64 values (the upper half of their fp32 bits)."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bf16_from_bits(bits) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def dequant_bf16(qweight, scale_bits, zeros, group_size) -> np.ndarray:
    """O9: w[k][n] = bf16_rne((q - z) * s) with s given as bf16 bits [K/G][N]; float64 [K][N]."""
    q = unpack_awq(qweight).astype(np.int64)
    z = unpack_awq(zeros).astype(np.int64)
    s = bf16_from_bits(scale_bits)
    g = np.arange(q.shape[0]) // group_size
    return bf16_rne((q - z[g, :]).astype(np.float64) * s[g, :])


def gemm_f64(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """O9's O3: Y = X . W for operands already exact in float64 (bf16 values), fp64 accumulation."""
    return np.asarray(x, dtype=np.float64) @ np.asarray(w, dtype=np.float64)


# ----------------------------------------------------------------------------------------- O8
def gptq_dequant(qweight, qzeros, scales, g_idx=None, group_size=None, zero_plus_one=True) -> np.ndarray:
    """O8: fp16 [K][N] weights of an AutoGPTQ checkpoint (R17)."""
    qweight = np.asarray(qweight).view(np.uint32)
    qzeros = np.asarray(qzeros).view(np.uint32)
    K, N = qweight.shape[0] * 8, qweight.shape[1]
    q = np.empty((K, N), dtype=np.int64)
    for i in range(8):                                  # row 8j + i in nibble i
        q[i::8, :] = (qweight >> np.uint32(4 * i)) & np.uint32(0xF)
    NG = qzeros.shape[0]
    z = np.empty((NG, N), dtype=np.int64)
    for i in range(8):                                  # column 8j + i in nibble i
        z[:, i::8] = (qzeros >> np.uint32(4 * i)) & np.uint32(0xF)
    if zero_plus_one:
        z = z + 1
    g = np.arange(K) // group_size if g_idx is None else np.asarray(g_idx, dtype=np.int64)
    s = np.asarray(scales, dtype=np.float16).astype(np.float64)
    return ((q - z[g, :]).astype(np.float64) * s[g, :]).astype(np.float16)


# ----------------------------------------------------------------------------------------- O7
def silu_mul(g: np.ndarray, u: np.ndarray) -> np.ndarray:
    """O7: SiLU(g) * u = g / (1 + exp(-g)) * u in fp64 (R16)."""
    g = np.asarray(g, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    with np.errstate(over="ignore"):
        return g / (1.0 + np.exp(-g)) * u


# ----------------------------------------------------------------------------------------- O10
def add_bias(y: np.ndarray, bias) -> np.ndarray:
    """O10: Y + b broadcast over the rows (fp64; b given as float16 / float64 values)."""
    return np.asarray(y, dtype=np.float64) + np.asarray(bias, dtype=np.float64)[None, :]


# ----------------------------------------------------------------------------------------- O4
def round_fp16(y: np.ndarray) -> np.ndarray:
    """O4: fp16 round-to-nearest-even of the fp64 result."""
    return np.asarray(y, dtype=np.float64).astype(np.float16)


# ----------------------------------------------------------------------------------------- O5
def tol_check(y, y_ref, rel: float = 1e-2, abs_small: float = 1e-3, small: float = 1e-2) -> dict:
    """O5 (BASELINE.json north_star): pass iff for every element
    |y - ref| <= abs_small where |ref| < small, else |y - ref| <= rel * |ref|.
    A non-finite y where ref is finite fails."""
    y = np.asarray(y, dtype=np.float64)
    r = np.asarray(y_ref, dtype=np.float64)
    assert y.shape == r.shape
    err = np.abs(y - r)
    is_small = np.abs(r) < small
    bound = np.where(is_small, abs_small, rel * np.abs(r))
    bad = ~(err <= bound)                      # NaN err -> bad
    bad |= ~np.isfinite(y) & np.isfinite(r)
    rel_err = np.where(is_small, 0.0, err / np.where(is_small, 1.0, np.abs(r)))
    idx = np.argwhere(bad)
    return {
        "ok": not bool(bad.any()),
        "n_fail": int(bad.sum()),
        "n": int(y.size),
        "max_rel": float(np.max(np.where(np.isnan(rel_err), np.inf, rel_err))) if y.size else 0.0,
        "max_abs_small": float(np.nanmax(np.where(is_small, err, 0.0))) if y.size else 0.0,
        "first_fail": tuple(int(i) for i in idx[0]) if len(idx) else None,
    }


# ----------------------------------------------------------------------------------------- O6
# v1 packed layout, T = N/128 n-tiles, C = K/32 k-chunks, NG = K/G groups:
#   weights at byte ((t*C + c)*128 + r)*16 + 4*w + i//2, nibble (i % 2) of that byte,
#     for the code of (k, n) with t = n//128, r = n%128, c = k//32, w = (k%32)//8 and
#     i = the nibble slot that holds k%8, i.e. k%8 == AWQ_ORDER[i]  (dequant-aware order
#     along k, so the FT extraction yields (k, k+1) fp16 pairs in ascending k);
#   meta(t, g) at byte K*N/2 + (t*NG + g)*320: 128 fp16 scales (n = 128t + r, little-endian),
#     then 64 bytes of zero points, zero of row r in byte r//2, low nibble if r is even.
_INV_AWQ = tuple(AWQ_ORDER.index(j) for j in range(8))   # slot i holding k_off j


def v1_packed_bytes(K: int, N: int, G: int) -> int:
    if K <= 0 or N <= 0 or G <= 0 or K % G or K % 64 or N % 128:
        return 0
    return K * N // 2 + (K // G) * N * 5 // 2


def v1_weight_pos(k, n, K: int, N: int):
    """(byte offset, nibble-in-byte) of code (k, n) in the v1 weights section."""
    k = np.asarray(k, dtype=np.int64)
    n = np.asarray(n, dtype=np.int64)
    C = K // 32
    t, r = n // 128, n % 128
    c, w, j = k // 32, (k % 32) // 8, k % 8
    i = np.asarray(_INV_AWQ, dtype=np.int64)[j]
    byte = ((t * C + c) * 128 + r) * 16 + 4 * w + i // 2
    return byte, i % 2


def v1_meta_offset(t: int, g: int, K: int, N: int, G: int) -> int:
    return K * N // 2 + (t * (K // G) + g) * 320


def pack_v1(qweight, scales, zeros, G: int, K: int, N: int) -> np.ndarray:
    """Encoder written from the layout text above (independent of the library packer)."""
    nbytes = v1_packed_bytes(K, N, G)
    assert nbytes > 0
    blob = np.zeros(nbytes, dtype=np.uint8)
    q = unpack_awq(qweight)                                   # [K][N]
    kk, nn = np.meshgrid(np.arange(K), np.arange(N), indexing="ij")
    byte, nib = v1_weight_pos(kk.ravel(), nn.ravel(), K, N)
    vals = q.ravel().astype(np.uint8) << (4 * nib).astype(np.uint8)
    np.bitwise_or.at(blob, byte, vals)
    z = unpack_awq(zeros)                                     # [K/G][N]
    s_bits = np.asarray(scales, dtype=np.float16).view(np.uint16)
    for t in range(N // 128):
        for g in range(K // G):
            off = v1_meta_offset(t, g, K, N, G)
            sb = s_bits[g, 128 * t:128 * (t + 1)]
            blob[off:off + 256:2] = (sb & 0xFF).astype(np.uint8)
            blob[off + 1:off + 256:2] = (sb >> 8).astype(np.uint8)
            zr = z[g, 128 * t:128 * (t + 1)]
            blob[off + 256:off + 320] = (zr[0::2] | (zr[1::2] << 4)).astype(np.uint8)
    return blob


def unpack_v1(blob, G: int, K: int, N: int):
    """Decoder written from the layout text above: blob -> (qweight, scales, zeros) AWQ tensors."""
    blob = np.asarray(blob, dtype=np.uint8).ravel()
    assert blob.size == v1_packed_bytes(K, N, G)
    kk, nn = np.meshgrid(np.arange(K), np.arange(N), indexing="ij")
    byte, nib = v1_weight_pos(kk.ravel(), nn.ravel(), K, N)
    q = ((blob[byte] >> (4 * nib).astype(np.uint8)) & 0xF).reshape(K, N)
    s_bits = np.empty((K // G, N), dtype=np.uint16)
    z = np.empty((K // G, N), dtype=np.uint8)
    for t in range(N // 128):
        for g in range(K // G):
            off = v1_meta_offset(t, g, K, N, G)
            lo = blob[off:off + 256:2].astype(np.uint16)
            hi = blob[off + 1:off + 256:2].astype(np.uint16)
            s_bits[g, 128 * t:128 * (t + 1)] = lo | (hi << 8)
            zb = blob[off + 256:off + 320]
            z[g, 128 * t:128 * (t + 1):2] = zb & 0xF
            z[g, 128 * t + 1:128 * (t + 1):2] = zb >> 4
    return pack_awq(q), s_bits.view(np.float16), pack_awq(z)
