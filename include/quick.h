/*
 * quick.h -- C-ABI of libquick.so, a B200 (sm_100a) implementation of the QUICK W4A16 path.
 *
 * The operation (PAPER.md = arXiv 2402.10076, "P:L<n>" = its line n):
 *   Y[M][N] = X[M][K] . dequant(Wq)[K][N],   dequant(q)[k][n] = (q[k][n] - z[k/G][n]) * s[k/G][n]
 *   "mixed precision GEMM" with fp16 activations and 4-bit weights (§2.3, §4);
 *   weights are "interleaved ... offline" (abstract P:L10; §3; §3.2) so the
 *   kernel never writes dequantized weights back to shared memory (Fig. 2).
 *
 * Conventions shared by every entry point:
 *   - Plain C types only; no C++ types or exceptions cross this boundary.  All calls are
 *     thread-safe.  The library keeps no pointer after a call returns; the caller owns and
 *     frees every buffer.
 *   - Errors are returned as quick_status_t, never printed.  Device-side faults surface
 *     asynchronously, per CUDA convention, on the stream the call was issued to.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - AWQ "GEMM" checkpoint format (reading R2): qweight uint32 [K][N/8], nibble i
 *     (bits 4i..4i+3) of qweight[k][j] holds the code of column 8j + {0,2,4,6,1,3,5,7}[i];
 *     zeros uint32 [K/G][N/8] packed the same way; scales fp16 bits uint16 [K/G][N].
 *   - Supported shapes (layout v1): K % 64 == 0, N % 128 == 0, G in {32, 64, 128, 256, ...}
 *     with K % G == 0 and G % 32 == 0.  Other shapes return QUICK_ERR_UNSUPPORTED; invalid
 *     arguments (null pointers, negative sizes) return QUICK_ERR_INVALID_ARG.
 */
#ifndef QUICK_H_
#define QUICK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QUICK_OK = 0,
  QUICK_ERR_INVALID_ARG = 1, /* null pointer, M/N/K/G <= 0 (M < 0), bad ld, K % G != 0 */
  QUICK_ERR_UNSUPPORTED = 2, /* N % 128, K % 64, G % 32 != 0; misaligned pointer; bad override */
  QUICK_ERR_CUDA = 3         /* CUDA runtime/driver error; see quick_last_cuda_error()        */
} quick_status_t;

/* Version of the packed layout produced by quick_pack_weights (v1). */
uint32_t quick_layout_version(void);

/* Bytes of the packed blob for (K, N, G): K*N/2 weight bytes + (K/G)*N*2.5 metadata bytes
 * (fp16 scale + 4-bit zero per (group, column)).  Returns 0 if the shape is unsupported. */
size_t quick_packed_bytes(int K, int N, int group_size);

/* Offline repack (host; §3.2, Figs. 4-6): AWQ tensors -> v1 blob.
 *   qweight  host, uint32 [K][N/8], AWQ order
 *   scales   host, uint16 [K/G][N], fp16 bit patterns (copied verbatim, incl. NaN/Inf)
 *   zeros    host, uint32 [K/G][N/8], AWQ order
 *   packed_out host, quick_packed_bytes(K, N, G) bytes, written completely.
 * Deterministic pure function of its inputs; bit-exact and invertible (quick_unpack_weights). */
quick_status_t quick_pack_weights(const uint32_t* qweight, const uint16_t* scales,
                                  const uint32_t* zeros, int group_size, int K, int N,
                                  void* packed_out);

/* Fused gate||up repack (host, the MLP's two column-parallel projections as one GEMM
 * whose epilogue applies SiLU(gate) * up, QUICK_FLAG_SILU_MUL).  Inputs: the gate and the up
 * projection, each in the AWQ format above with I output columns (qweight [K][I/8], scales
 * [K/G][I], zeros [K/G][I/8]).  Output: the v1 blob of the N = 2I column matrix W' whose column
 * 128t + 32q + l is gate column 64t + 16q + l for l < 16 and up column 64t + 16q + l - 16 for
 * l >= 16 (a gate row and its up row sit in TMEM lanes l and l + 16 of one warp, so the epilogue
 * pairs them with one shuffle).  packed_out: quick_packed_bytes(K, 2I, G) bytes.
 * Requires I % 64 == 0 (else QUICK_ERR_UNSUPPORTED). */
quick_status_t quick_pack_gate_up(const uint32_t* qweight_gate, const uint16_t* scales_gate,
                                  const uint32_t* zeros_gate, const uint32_t* qweight_up,
                                  const uint16_t* scales_up, const uint32_t* zeros_up,
                                  int group_size, int K, int I, void* packed_out);

/* GPTQ checkpoint import (host; the GPTQ family of P:L19).  Input, the AutoGPTQ
 * format: qweight uint32 [K/8][N] with nibble i of word (j, n) = code of row 8j + i; qzeros uint32
 * [K/G][N/8] with nibble i of word (g, j) = zero of column 8j + i minus zero_plus_one (1 for the
 * classic "v1" checkpoints that store zero - 1, 0 for "v2"); scales fp16 bits [K/G][N]; g_idx
 * int32 [K] = group of row k (act-order / desc_act checkpoints permute rows across groups; NULL =
 * k / G).  Output: the same weights in the AWQ format above (qweight_awq [K][N/8], scales_out
 * [K/G][N], zeros_awq [K/G][N/8]) with the rows reordered so that group g is rows [gG, (g+1)G):
 * row k' of the output is source row perm[k'] (perm int32 [K], identity when g_idx is NULL or
 * monotone), so Y = X . W = X[:, perm] . W_out (quick_gather_k permutes X on the device).
 * QUICK_ERR_UNSUPPORTED if a group does not hold exactly G rows or a decoded zero is 16. */
quick_status_t quick_import_gptq(const uint32_t* qweight, const uint32_t* qzeros, const uint16_t* scales,
                                 const int32_t* g_idx, int zero_plus_one, int group_size, int K, int N,
                                 uint32_t* qweight_awq, uint16_t* scales_out, uint32_t* zeros_awq,
                                 int32_t* perm);

/* Exact inverse of quick_pack_weights (host). Same array shapes as above, written completely. */
quick_status_t quick_unpack_weights(const void* packed, int group_size, int K, int N,
                                    uint32_t* qweight, uint16_t* scales, uint32_t* zeros);

/* The hot path (device, asynchronous on `stream`; CUDA-graph capturable).  Y = X . dequant(Wq)
 * with fp32 accumulation (reading R4) and fp16 output.  No allocation, no synchronisation and no
 * host-visible state: the launch plan is a pure function of (M, N, K, G), identical eagerly and
 * under graph capture, and needs no workspace (split-K partials are reduced through the
 * cluster's distributed shared memory).
 *   X       device, __half [M][K] row-major, 16-byte aligned
 *   packed  device copy of the quick_pack_weights blob, 128-byte aligned
 *   Y       device, __half [M][N] row-major, 16-byte aligned
 * M == 0 is a no-op returning QUICK_OK.  The (K, N, G) given must match the blob. */
quick_status_t quick_w4a16_gemm(const void* X, const void* packed, int M, int N, int K,
                                int group_size, void* Y, void* stream);

/* Flags of quick_w4a16_gemm_ex. */
#define QUICK_FLAG_OUT_F32 1 /* Y is float: un-rounded fp32 sums (row-parallel fp32 all-reduce) */
#define QUICK_FLAG_PDL 2     /* launch with programmatic dependent launch: the kernel's prologue
                                and its (read-only) weight stream may overlap the previous
                                kernel in the stream; X is read and Y written only after that
                                kernel completes.  The weights must not be written by the
                                immediately preceding kernel.  The first weight stages are
                                also dequantized before that point.  Ignored by plans with
                                256-token tiles. */
#define QUICK_FLAG_NO_STREAMK 4 /* never use the stream-K schedule (tests / A-B timing) */
#define QUICK_FLAG_BF16 16      /* bf16 variant: X, Y and the blob's 16-bit
                                   scales are bf16 (quick_pack_weights copies the scale bits as
                                   given); dequant = bf16_rne((q - z) * s), fp32 accumulation, bf16
                                   Y (or fp32 with QUICK_FLAG_OUT_F32). */
#define QUICK_FLAG_SILU_MUL 8   /* fused gate||up epilogue for a blob made by
                                   quick_pack_gate_up: Y is __half [M][N/2] (ldy >= N/2) with
                                   Y[m][i] = fp16_rne(SiLU(G[m][i]) * U[m][i]), G = X.gate and
                                   U = X.up accumulated in fp32, SiLU(g) = g / (1 + exp(-g)) in
                                   fp32.  Not with QUICK_FLAG_OUT_F32. */

/* Bytes of caller-owned workspace the call quick_w4a16_gemm_ex(M, N, K, G, flags, tile_n,
 * split_k) can use: the small-M stream-K schedule (tiles of <= 64 tokens) keeps one fp32
 * partial tile per CTA and one arrival counter per output tile there.  0 when that call's plan
 * needs none.  Pure function of its arguments (device properties included). */
size_t quick_workspace_bytes(int M, int N, int K, int group_size, int flags, int tile_n,
                             int split_k);

/* Extended form used by tensor parallelism, layer stacks, the bench and the tests.
 *   ldy       row stride of Y in elements (>= N, multiple of 8); lets a rank write its column
 *             slice of a wider Y in place
 *   flags     QUICK_FLAG_* bits (0 = fp16 Y, ordinary stream ordering)
 *   tile_n    tokens per MMA tile (16, 32, 64, 128, 256), 0 = automatic
 *   split_k   CTAs per cluster splitting K (1..8, <= ceil(K/128)), 0 = automatic (which may
 *             choose stream-K for tiles <= 64)
 *   workspace, workspace_bytes
 *             caller-owned device memory, 256-byte aligned, ZEROED by the caller once before
 *             its first use: its first 256 KiB hold the stream-K arrival counters, which every
 *             launch leaves zeroed again (the rest is scratch for fp32 partial tiles), so one
 *             workspace may serve calls of any shapes in sequence.  The stream-K plan is used
 *             only if workspace_bytes >= quick_workspace_bytes(...) of this call; otherwise
 *             the workspace-free plan runs (so the plan never depends on anything but the
 *             arguments).  NULL / 0 = no workspace.  Two launches that may run concurrently
 *             (different streams, or graphs replayed on different streams) must not share a
 *             workspace; graphs capture the pointer, so it must outlive them.
 * With tile_n = split_k = 0 and M > 64 the automatic plan may run tiles of 128/256 tokens as CTA
 * pairs (tcgen05 cta_group::2: two n-tiles per cluster of two SMs); a forced
 * (tile_n, split_k) runs one CTA per n-tile.  Both compute the same MMAs in the same K order.
 * QUICK_FLAG_PDL is not applied to plans with 256-token tiles.
 * Deterministic: equal inputs and equal plans give bit-equal Y. */
quick_status_t quick_w4a16_gemm_ex(const void* X, const void* packed, int M, int N, int K,
                                   int group_size, void* Y, int ldy, int flags, int tile_n,
                                   int split_k, void* workspace, size_t workspace_bytes,
                                   void* stream);

/* quick_w4a16_gemm_ex with a bias epilogue (SURVEY 8(f) f2 "bias"; not in PAPER.md, whose
 * mixed-precision GEMM of §2.3 P:L58-64 has none):
 *   Y[m][n] = round16( sum_k X[m][k] . dequant(W)[k][n]  +  bias[n] )
 * bias: device pointer to N 16-bit values (fp16; bf16 with QUICK_FLAG_BF16), 8-byte aligned,
 * read-only, owned by the caller.  The bias is added in fp32 to the fp32 sum once, by the CTA
 * that writes Y (after the split-K / stream-K reduction), then the result is rounded once to 16
 * bits (or stored as fp32 with QUICK_FLAG_OUT_F32, bias included).  NULL bias -> INVALID_ARG;
 * with QUICK_FLAG_SILU_MUL -> UNSUPPORTED (the gate||up blob has no bias layout).  Every other
 * argument, rule and error as in quick_w4a16_gemm_ex. */
quick_status_t quick_w4a16_gemm_bias(const void* X, const void* packed, const void* bias, int M, int N,
                                     int K, int group_size, void* Y, int ldy, int flags, int tile_n,
                                     int split_k, void* workspace, size_t workspace_bytes,
                                     void* stream);

/* The launch plan quick_w4a16_gemm_ex(M, N, K, G, flags, tile_n = 0, split_k = 0, workspace of
 * workspace_bytes) would use: tokens per tile, cluster split-K factor (0 = stream-K schedule),
 * number of CTAs, and 1 if the tiles run as CTA pairs.  Any out pointer may be NULL. */
quick_status_t quick_gemm_plan(int M, int N, int K, int group_size, int flags,
                               size_t workspace_bytes, int* tile_n, int* split_k, int* num_ctas,
                               int* cta_pair);

/* quick_pack_weights on the device (repack of 70B-scale checkpoints at HBM speed):
 * the same AWQ tensors and the same v1 blob, bit-exact, all pointers device memory (packed_out
 * 16-byte aligned, quick_packed_bytes bytes).  Asynchronous on `stream`. */
quick_status_t quick_pack_weights_device(const uint32_t* qweight, const uint16_t* scales,
                                         const uint32_t* zeros, int group_size, int K, int N,
                                         void* packed_out, void* stream);

/* Activation side of a GPTQ act-order import: Xp[m][k'] = X[m][perm[k']] (device __half [M][K],
 * perm device int32 [K] from quick_import_gptq).  Asynchronous on `stream`. */
quick_status_t quick_gather_k(const void* X, const int32_t* perm, int M, int K, void* Xp, void* stream);

/* Device dequantization of a packed blob into W fp16 [K][N] row-major (device), computing
 * dequant(q)[k][n] bit-exactly as fp16_rne((q - z) * s) (§2.3).  Asynchronous. */
quick_status_t quick_dequant_weights(const void* packed, int K, int N, int group_size, void* W,
                                     void* stream);

/* quick_dequant_weights with flags: QUICK_FLAG_BF16 -> bf16_rne((q - z) * s), W bf16 [K][N]. */
quick_status_t quick_dequant_weights_ex(const void* packed, int K, int N, int group_size, void* W,
                                        int flags, void* stream);

/* Row-parallel epilogue: dst[i] = fp16_rne(src[i]) for i < n (device float -> device __half). */
quick_status_t quick_f32_to_f16(const void* src, void* dst, size_t n, void* stream);

/* Column-parallel epilogue: src __half [P][M][Nr] (an all-gather of per-rank Y slices) ->
 * dst __half [M][P*Nr] row-major (device, asynchronous). */
quick_status_t quick_gather_columns(const void* src, void* dst, int P, int M, int Nr,
                                    void* stream);

/* ---------------------------------------------------------------------------------------------
 * Collective-fused tensor parallelism over peer memory (BASELINE.json north_star
 * (4)).  One process per GPU.  Buffers that other ranks access are allocated with
 * quick_peer_alloc (setup time, zeroed), exported as 64-byte handles, exchanged by the caller's
 * process group, and mapped with quick_peer_import; a kernel then loads and stores peer memory
 * directly (NVLink / NVSwitch; same-device IPC when the ranks share a GPU).  Per rank the caller
 * holds arrays of world pointers, entry p = rank p's buffer as mapped in this process.
 * Barriers use a flag array of world + 1 uint32 per rank (quick_peer_alloc'd, zeroed): slot p
 * receives rank p's signals, slot `world` counts this rank's barriers on the device, so CUDA
 * graphs that capture these calls replay correctly.  Every rank must issue the same sequence of
 * TP calls on a communicator.  A barrier wait longer than 20 s traps (loud launch failure, no hang).
 * ------------------------------------------------------------------------------------------- */
#define QUICK_IPC_HANDLE_BYTES 64

quick_status_t quick_peer_alloc(size_t bytes, void** ptr);        /* device memory, zeroed */
quick_status_t quick_peer_free(void* ptr);
quick_status_t quick_peer_export(const void* ptr, void* handle_out); /* QUICK_IPC_HANDLE_BYTES */
quick_status_t quick_peer_import(const void* handle, void** ptr); /* map another rank's buffer */
quick_status_t quick_peer_close(void* ptr);                        /* unmap an imported buffer */

/* Every rank: signal every rank, wait until every rank has reached this barrier (stream-ordered). */
quick_status_t quick_tp_barrier(void* const* flag_peers, int world, int rank, void* stream);

/* Column-parallel GEMM with the all-gather fused into the epilogue: this rank's
 * Y_r = X . dequant(Wq_r) (N_local columns, packed = quick_pack_weights of the rank's column shard)
 * is stored straight into columns [rank N_local, (rank+1) N_local) of EVERY rank's Y (y_peers[p]:
 * __half [M][ldy], ldy >= world N_local, 16-byte aligned), then a barrier: when the stream passes
 * this call every rank's Y holds the full [M][world N_local] product.  Same plan, same bits as
 * quick_w4a16_gemm_ex on the shard.  flags: QUICK_FLAG_PDL / NO_STREAMK; workspace as in _ex.
 * No rank may still be reading its Y when another rank's call starts writing it (alternate two
 * Y buffers: each call's closing barrier then makes the reuse two calls later safe). */
quick_status_t quick_tp_column_gemm(const void* X, const void* packed, int M, int N_local, int K,
                                    int group_size, void* const* y_peers, int ldy,
                                    void* const* flag_peers, int world, int rank, int flags,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* Row-parallel GEMM with a peer-memory all-reduce: the fp32 partial X_local . dequant(Wq_r)
 * (K_local rows of this rank, N columns) goes to part_peers[rank] (float [M][N], every rank's
 * mapped here); barrier; this rank sums columns [rank N/P, (rank+1) N/P) over the P partials in
 * rank order 0..P-1 in fp32 and stores fp16 into every rank's Y (y_peers[p]: __half [M][ldy]);
 * barrier.  Every rank's Y is bit-identical and deterministic.  N % (8 world) == 0. */
quick_status_t quick_tp_row_gemm(const void* X_local, const void* packed, int M, int N, int K_local,
                                 int group_size, void* const* part_peers, void* const* y_peers,
                                 int ldy, void* const* flag_peers, int world, int rank, int flags,
                                 void* workspace, size_t workspace_bytes, void* stream);

const char* quick_status_string(quick_status_t status);

/* cudaError_t of the last QUICK_ERR_CUDA returned on the calling thread (0 if none). */
int quick_last_cuda_error(void);

#ifdef __cplusplus
}
#endif

#endif /* QUICK_H_ */
