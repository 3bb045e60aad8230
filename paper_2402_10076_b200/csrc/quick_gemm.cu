// QUICK W4A16 GEMM for B200 (sm_100a): Y[M][N] = X[M][K] . dequant(Wq)[K][N].
//
// PAPER.md: the mixed-precision GEMM of §2.3 with the QUICK idea of §3
// (P:L78-86): weights are interleaved offline (quick_pack.cpp) so that each thread's direct
// load, after dequantization in registers (FasterTransformer LOP3 magic), is already
// in the MMA operand layout -- no shared-memory write-back of dequantized weights and no
// ldmatrix (Fig. 2).  On Blackwell the operand a thread owns is one TMEM lane of the
// tcgen05.mma A operand, so the kernel computes the swapped product
//     D[n][m] = sum_k W^T[n][k] . X^T[k][m]        (A = dequantized weights in TMEM,
//                                                   B = X tile in SMEM via TMA, D in TMEM)
// with the weight rows n on the 128-lane MMA M dimension and the tokens m on the MMA N
// dimension (16..256), so small batches do not waste the 128-row MMA.
//
// CTA = 10 warps, warp-specialised.  The SM's warp scheduler favours the highest
// warp id, so the two latency-critical single warps take the top ids:
//   warps 0..7  dequantizers, two groups of 4 taking alternate 128-k A stages: per stage a
//               thread (one TMEM lane = one weight row) does 4 x LDS.128 of 128 codes ->
//               16 x (SHF + LOP3 x4, HSUB2/HFMA2 -> exact (q-z), HMUL2 by s) -> 2 x
//               tcgen05.st.32x32b.x32 into the TMEM A ring; then the segment epilogue
//               (tcgen05.ld -> Y, or an fp32 partial for split-K / stream-K)
//   warp 8      producer: 1-D bulk copies of the packed int4 stage + group metadata and a 3-D
//               TMA load of the X tile (SWIZZLE_128B, K-major) into a STAGES-deep mbarrier ring
//   warp 9      TMEM allocator + MMA issuer (one elected thread): 8 x tcgen05.mma.kind::f16
//               per A stage, fp32 accumulation in TMEM, tcgen05.commit -> mbarriers
// Split-K: the S CTAs of a (S,1,1) cluster share one (n-tile, m-tile) and split K (the
// "split-k" knob of §5); partial sums stay fp32 (tolerance analysis).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/quick.h"
#include "quick_ptx.cuh"

namespace quick {

// CTA shape per config: Cfg::NPAR dequant groups of 4 warps (one per TMEM lane quarter), then
// the producer warp and the MMA warp on the top warp ids
constexpr int kTileRows = 128;    // weight rows (output columns n) per tile = TMEM lanes
constexpr int kKA = 128;          // k per A stage (one TMEM A slot, 8 MMAs of K = 16)
constexpr int kAColsPerStage = kKA / 2;           // 128 fp16 of k = 64 x 32-bit TMEM columns
constexpr int kChunkBytes = kTileRows * 16;       // 32 k x 128 rows of int4 = one 2 KiB chunk
constexpr int kMetaBytes = 320;   // 128 fp16 scales + 128 4-bit zeros per (n-tile, group)
constexpr int kMaxSplit = 8;      // split-K cluster size limit (portable clusters)
constexpr int kTraceStages = 256; // debug tracing: stages recorded per traced CTA
constexpr int kTraceStride = 8 + 7 * kTraceStages;
constexpr int kDebugNoCompute = 1 << 30;   // undocumented debug flag: stream the loads only
constexpr int kDebugExitTop = 1 << 29;     // debug: return at kernel entry (launch cost probe)
constexpr int kDebugExitPrologue = 1 << 28;  // debug: return after the prologue (setup probe)
constexpr int kDebugNoMma = 1 << 27;       // debug: dequant + STTM but no MMA (commits only)
constexpr int kDebugOneCta = 1 << 26;      // debug: stream-K with one CTA per SM (smem padded)
constexpr int kDebugNoSttm = 1 << 25;      // debug: dequant into registers, no TMEM store, no MMA
constexpr int kDebugPdlEarly = 1 << 24;    // PDL trigger right after the prologue (set by the host for
                                           // stream-K grids that fill every CTA slot; forcible for tests)
constexpr int kAblationSmemA = 1 << 21;    // ablation: A stage via shared memory (Cfg AM = 1)
constexpr int kForcePair = 1 << 20;        // debug: CTA-pair (cta_group::2) plan for tiles 128/256
constexpr int kDebugNoPair = 1 << 19;      // debug: automatic plan without CTA pairs
constexpr int kDebugForceSk = 1 << 17;     // debug: stream-K whenever the tile allows it
constexpr int kDebugSkReverse = 1 << 16;   // debug: stream-K CTA c takes the unit range of CTA P-1-c
constexpr int kAblationMmaSync = 1 << 18;  // ablation: M <= 16 stream-K plans on the register-fragment
                                           // mma.sync decode kernel (QUICK's Ampere design)

// the stream-K "CTA index" that owns unit ranges (blockIdx.x, or reversed under kDebugSkReverse)
__device__ __forceinline__ int sk_cta(int flags) {
  return (flags & kDebugSkReverse) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
}

// Per tile width BN (tokens per MMA) and mode SK (stream-K):
//   KL     k per load stage: one bulk copy of KL x 64 B of weights, one bulk copy of the groups'
//          metadata, one 3-D TMA of the [KL/64][BN][64] X tile (few, large async copies: each
//          TMA/bulk issue costs ~150 SM cycles on B200, measured with tools/trace_gemm.py)
//   STAGES depth of the load ring
//   TMEM   A ring of ASTAGES x 64 columns, then NDBUF x NACC fp32 accumulators of BN columns
//          (stream-K double-buffers D so a segment's epilogue overlaps the next segment's MMAs;
//          small tiles alternate the K=16 MMAs over NACC = 2 accumulators, summed in the
//          epilogue, because a single accumulator chain makes N=16 MMAs latency-bound)
// AM (A-operand placement): 0 = the dequantized A stage in TMEM (tcgen05.st, TS MMA: the design);
// 1 = ablation of the paper's Fig. 2 baseline on B200: the dequantized A stage written back to
// shared memory (STS.128 in the UMMA SWIZZLE_128B K-major layout, conflict-free) and read by an SS
// MMA (tiles 16 and 128, cluster split-K plans only);
// 2 = CTA pair (cta_group::2): two CTAs of a cluster on the two SMs of a TPC hold the weight
// rows of two n-tiles (M = 256 across the pair, A in each CTA's TMEM) and load half of the BN
// tokens of X each; the even CTA issues one MMA for both, so each SM reads half the X bytes
// per weight row (the large-M regime is bound by the per-SM L2 -> SM input)
template <int BN, bool SK, int AM = 0>
struct Cfg {
  static constexpr bool SMEM_A = AM == 1;
  static constexpr bool PAIR = AM == 2;
  static constexpr int XN = PAIR ? BN / 2 : BN;   // token rows of X this CTA loads
  // NPAR dequant groups of 4 warps.  NPAR = 4 (one CTA per SM, 16 dequant warps, the whole TMEM
  // for a 6-7 slot A ring) was measured 1.9x slower per SM than two 2-group CTAs per SM on the
  // 70B shapes at M <= 64 (one MMA warp per SM cannot keep up), so every tile uses 2 groups; the
  // code is written for any power-of-two NPAR.
  static constexpr int NPAR = 2;
  static constexpr int THREADS = 32 * (4 * NPAR + 2);
  // warp roles: dequant warps 0..4 NPAR - 1, then the producer and the MMA warp.  The build
  // variant QUICK_ROLES_FIRST puts the producer / MMA warps at ids 0 / 1 instead: measured equal
  // on B200 over the BJ shapes x M = 1..1024 (tools/gpu_r2_experiments.sh warp_roles, profiles/r02_warp_roles_ab.txt),
  // and equally imbalanced between the two co-resident stream-K CTAs
#ifdef QUICK_ROLES_FIRST
  static constexpr int DQ_BASE = 2;
  static constexpr int PRODUCER_WARP = 0;
  static constexpr int MMA_WARP = 1;
#else
  static constexpr int DQ_BASE = 0;
  static constexpr int PRODUCER_WARP = 4 * NPAR;
  static constexpr int MMA_WARP = 4 * NPAR + 1;
#endif
  static constexpr int DQ_THREADS = 128 * NPAR;
  static constexpr int NDBUF = SK ? 2 : 1;
  static constexpr int TMEM_BUDGET = NPAR == 4 ? 512 : 256;
  static constexpr int ASTAGES_FIT = (TMEM_BUDGET - NDBUF * (BN <= 32 ? 2 : 1) * BN) / kAColsPerStage;
  static constexpr int ASTAGES =
      NPAR == 4 ? (ASTAGES_FIT > 7 ? 7 : ASTAGES_FIT)
                : (BN == 256 ? 4 : BN > 64 ? 2 : ((256 - NDBUF * BN) / kAColsPerStage >= 3 ? 3 : 2));
  static constexpr int DCOL = !SMEM_A ? ASTAGES * kAColsPerStage : 0;   // A ring columns in TMEM
  static constexpr int NACC = (BN <= 32 && DCOL + NDBUF * 2 * BN <= TMEM_BUDGET) ? 2 : 1;
  // (the 16-token stream-K tile streams 8 KiB load stages through an 8-deep ring: each slot is
  // released after one A stage instead of two, so more of the ring is in flight -- 28672x8192 and
  // 8192x28672 at M <= 16: 31.1 -> 29.5 us; the cluster split-K tile-16 plans, with few stages
  // per CTA, keep 256-k stages: 4096^2 M = 1 6.4 vs 7.1 us with 128)
  static constexpr int KL = (BN <= 16 && SK) ? 128 : BN <= 32 ? 256 : 128;
  static constexpr int APL = KL / kKA;              // A stages per load stage
  // tile 128 trades its second CTA per SM for a 4-deep ring (the MMA of a 41 KiB stage takes
  // ~512 cycles, less than the L2/HBM refill latency a 2-deep ring exposes)
  static constexpr int STAGES = NPAR == 4 ? (BN <= 16 ? 8 : BN <= 32 ? 6 : 8)
                                          : (BN <= 16 ? (KL == 128 ? 8 : 4) : BN <= 32 ? 3 : BN <= 128 ? (SMEM_A ? 3 : 4)
                                                                                   : (PAIR ? 4 : 3));
  static constexpr int X_BYTES = XN * KL * 2;       // [KL/64][XN][64] fp16, SW128 sub-tiles
  static constexpr int X_SUB = XN * 128;            // one [XN][64] sub-tile (multiple of 1 KiB)
  static constexpr int W_BYTES = KL * 64;           // KL/32 chunks of 2 KiB
  static constexpr int M_BYTES = ((KL / 32 + 1) * kMetaBytes + 15) & ~15;  // worst case G = 32
  static constexpr int X_OFF = 0;
  static constexpr int W_OFF = X_OFF + STAGES * X_BYTES;
  static constexpr int M_OFF = W_OFF + STAGES * W_BYTES;
  static constexpr int A_BYTES = kTileRows * kKA * 2;   // AM = 1: one A stage in shared memory
  static constexpr int A_OFF = (M_OFF + STAGES * M_BYTES + 1023) & ~1023;
  static constexpr int BAR_OFF = !SMEM_A ? ((M_OFF + STAGES * M_BYTES + 7) & ~7) : (A_OFF + ASTAGES * A_BYTES);
  // barriers: full[STAGES], empty[STAGES], afull[ASTAGES], aempty[ASTAGES], dfull[2], dempty[2]
  // + xfull[STAGES]: the X tile has its own barrier so that dequantization (weights + metadata
  // only) can start before X is loadable (PDL: the weights of the first stages are fetched and
  // dequantized while the previous kernel finishes)
  static constexpr int NUM_BARS = 3 * STAGES + 2 * ASTAGES + 4;
  static constexpr int HOLD_OFF = BAR_OFF + NUM_BARS * 8;   // TMEM base, then stream-K flag
  static constexpr int USED = HOLD_OFF + 16;
  static constexpr int TMEM_COLS = SMEM_A ? (NDBUF * NACC * BN <= 32 ? 32 : NDBUF * NACC * BN <= 64 ? 64
                                                : NDBUF * NACC * BN <= 128 ? 128 : 256)
                                   : ((NPAR == 2 && DCOL + NDBUF * NACC * BN <= 256) ? 256 : 512);
  // Cap co-resident CTAs per SM so that their TMEM allocations always fit (512 columns):
  // otherwise a cluster could wait on a CTA that spins in tcgen05.alloc.
  static constexpr int MAX_CTAS_PER_SM = SMEM_A ? 1 : 512 / TMEM_COLS;
  static constexpr int MIN_SMEM = (228 * 1024) / (MAX_CTAS_PER_SM + 1) + 1024;
  static constexpr int SMEM_BYTES = (USED + 1024 > MIN_SMEM ? USED + 1024 : MIN_SMEM);
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "tcgen05 M=128 needs N % 16 == 0, 16..256");
  static_assert(KL % kKA == 0 && APL <= 2, "load stage = one or two A stages");
  static_assert(!SK || BN <= 64, "stream-K is used for the small-M tiles");
  static_assert(!PAIR || (!SK && BN >= 128), "CTA pairs: large-M cluster plans only");
  static_assert(ASTAGES >= NPAR && STAGES * APL >= NPAR, "ring indices advance by NPAR per group step");
  static_assert(DCOL + NDBUF * NACC * BN <= TMEM_COLS, "TMEM budget");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  // split-K partial tile [BN][128] fp32 reuses the pipeline buffers once the mainloop is done
  static_assert(BN * kTileRows * 4 <= BAR_OFF, "split-K partial must fit in the pipeline smem");
};

// Kernel parameters (passed by value as a __grid_constant__).
constexpr int kMaxPeers = 8;   // collective-fused TP epilogue: destinations of every Y store

struct KParams {
  const uint8_t* packed;
  void* Y;
  // column-parallel TP with the all-gather fused into the epilogue: every Y
  // element is stored to each of the ndst destinations (this rank's slot of every rank's Y over
  // peer memory); ndst = 1, Ydst[0] = Y otherwise
  int ndst;
  void* Ydst[kMaxPeers];
  int M, N, K, G, g_shift, ldy, flags;
  int n_tiles, m_tiles;   // tile index = t * m_tiles + mt (n-tile major: a CTA's tiles share weights)
  // cluster grids (not stream-K): gridDim.y = m_grp m-tiles, gridDim.z = n_cl n-tile clusters (n-tiles, or
  // n-tile pairs) x m_tiles / m_grp groups -- all n-tiles of one m-tile group run before the next group, so
  // a long-K X (70B down, M = 1024: 58.7 MB) is resident in L2 one group at a time
  int m_grp, n_cl;
  int NA;                 // A stages (128 k) per tile: ceil(K / 128)
  // stream-K (gridDim = (P, 1, 1)): the U = tiles x NA (tile, A stage) units are cut into P
  // contiguous ranges, U = P q + r: CTA c owns [c q + min(c, r), ...) of q + (c < r) units
  // (32-bit, no division on the device); partial tiles go through ws and are summed by the
  // last arriver
  int U, P, sk_q, sk_r;
  // two-group stream-K (sk_h > 0): CTAs [0, sk_h) own qa units each (+1 for the first ra of them), CTAs
  // [sk_h, P) qb (+1 for the first rb) -- e.g. less work for the CTA that shares an SM second; all in
  // 32-bit arithmetic (a 64-bit-division version of this in round 2 made every launch ~4 us slower)
  int sk_h, sk_qa, sk_ra, sk_qb, sk_rb;
  float* ws;              // [P][BN][128] fp32 partial tile of each CTA's (only) non-reducer segment
  int* sems;              // [tiles] arrival counters, zero between launches (reset by the reducer)
  unsigned long long* trace;
  // optional bias: [N] fp16 (bf16 with QUICK_FLAG_BF16) added in fp32 to every token's
  // output column before the final rounding, by whichever CTA writes Y; nullptr = none
  const uint16_t* bias;
};

__device__ __forceinline__ int sk_start(int c, int q, int r) { return c * q + min(c, r); }
// first unit of stream-K CTA c (c = P: U), uniform or two-group (KParams::sk_h)
__device__ __forceinline__ int sk_begin(const KParams& p, int c) {
  if (p.sk_h == 0) return sk_start(c, p.sk_q, p.sk_r);
  if (c <= p.sk_h) return sk_start(c, p.sk_qa, p.sk_ra);
  return sk_start(p.sk_h, p.sk_qa, p.sk_ra) + sk_start(c - p.sk_h, p.sk_qb, p.sk_rb);
}
// the CTA of a uniform run (q units each, +1 for the first r) owning unit u of the run
__device__ __forceinline__ int sk_owner_run(int u, int q, int r) {
  const int b = r * (q + 1);
  return u < b ? u / (q + 1) : r + (u - b) / q;
}
// the stream-K CTA owning unit u (the largest c with sk_begin(c) <= u)
__device__ __forceinline__ int sk_owner(const KParams& p, int u) {
  if (p.sk_h == 0) return sk_owner_run(u, p.sk_q, p.sk_r);
  const int ua = sk_start(p.sk_h, p.sk_qa, p.sk_ra);
  return u < ua ? sk_owner_run(u, p.sk_qa, p.sk_ra) : p.sk_h + sk_owner_run(u - ua, p.sk_qb, p.sk_rb);
}

// One contiguous run of A stages [a_lo, a_hi) of one tile (n-tile t, m-tile mt).
struct Seg {
  int tile, t, mt, a_lo, a_hi;
};

// Enumerates this CTA's segments.  Cluster split-K: exactly one (n-tile blockIdx.z, m-tile
// blockIdx.y -- the m-tiles of one n-tile are launched next to each other, so the CTAs reading
// the same weights run in the same wave and all but the first read them from L2 -- and the
// split's A range).  Stream-K: the unit range of CTA blockIdx.x, cut at tile boundaries.
// CTA pairs: blockIdx.x = 2 x split + member, n-tile 2 blockIdx.z + member.
struct SegIter {
  int u, u1;
  int NA, m_tiles;
  bool sk, done;
  int t, mt, a_lo, a_hi;
  __device__ __forceinline__ SegIter(const KParams& p, bool sk_, bool pair = false) {
    sk = sk_;
    NA = p.NA;
    m_tiles = p.m_tiles;
    done = false;
    if (sk) {
      const int c = sk_cta(p.flags);
      u = sk_begin(p, c);
      u1 = sk_begin(p, c + 1);
    } else {
      const int S = pair ? (int)gridDim.x >> 1 : (int)gridDim.x;
      const int sp = pair ? (int)blockIdx.x >> 1 : (int)blockIdx.x;
      const int grp = (int)blockIdx.z / p.n_cl;
      const int zc = (int)blockIdx.z - grp * p.n_cl;
      t = pair ? 2 * zc + ((int)blockIdx.x & 1) : zc;
      mt = grp * p.m_grp + (int)blockIdx.y;
      a_lo = (sp * NA) / S;          // 32-bit: S <= 8 and NA = ceil(K / 128) < 2^27
      a_hi = ((sp + 1) * NA) / S;
      u = u1 = 0;
    }
  }
  __device__ __forceinline__ bool more() const { return sk ? (u < u1) : !done; }
  __device__ __forceinline__ bool next(Seg& s) {
    if (!sk) {
      if (done) return false;
      done = true;
      s.t = t;
      s.mt = mt;
      s.tile = t * m_tiles + mt;
      s.a_lo = a_lo;
      s.a_hi = a_hi;
      return a_hi > a_lo;
    }
    if (u >= u1) return false;
    const int tile = u / NA;
    const int a0 = u - tile * NA;
    const int rem = u1 - u;
    const int a1 = (rem < NA - a0) ? a0 + rem : NA;
    s.tile = tile;
    s.t = tile / m_tiles;
    s.mt = tile - s.t * m_tiles;
    s.a_lo = a0;
    s.a_hi = a1;
    u += (a1 - a0);
    return true;
  }
};


// ------------------------------------------------------------------------------------------
// Dequantization of one 32-bit word of the v1 layout (8 codes, nibble order {0,2,4,6,1,3,5,7}
// along k) into four fp16x2 registers holding (k0,k1), (k2,k3), (k4,k5), (k6,k7).
//   lo = (w & 0x000f000f) | 0x6400_6400  -> fp16 (1024 + q)          (FT "magic")
//   hi = (w & 0x00f000f0) | 0x6400_6400  -> fp16 (1024 + 16 q)
//   (q - z) = lo - (1024 + z)  and  hi * 1/16 - (64 + z): both exact for every (q, z)
//   w = (q - z) * s with one round-to-nearest-even: bit-identical to the oracle's
//   fp16_rne((q - z) * s).  Explicit .rn forbids fma contraction.
// ------------------------------------------------------------------------------------------
struct DequantConsts {
  uint32_t zlo;  // fp16x2 (1024 + z)
  uint32_t zhi;  // fp16x2 -(64 + z)
  uint32_t s2;   // fp16x2 (s, s)
};

__device__ __forceinline__ DequantConsts make_consts(uint32_t sbits, uint32_t z) {
  // both halves replicated with PRMT (ALU pipe; the FMA pipe is the dequant's bottleneck)
  DequantConsts c;
  c.zlo = __byte_perm(0x6400u + z, 0u, 0x1010);          // 1024 + z   (ulp 1 in [1024, 2048))
  c.zhi = __byte_perm(0xD400u + (z << 4), 0u, 0x1010);   // -(64 + z)  (ulp 1/16 in [64, 128))
  c.s2 = __byte_perm(sbits, 0u, 0x1010);
  return c;
}

__device__ __forceinline__ uint32_t hsub2_rn(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hmul2_rn(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hfma2_rn(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ void dequant_word(uint32_t w, const DequantConsts& c, uint32_t* out) {
  constexpr uint32_t kMagic = 0x64006400u;
  constexpr uint32_t kInv16 = 0x2C002C00u;  // fp16x2 (1/16, 1/16)
  const uint32_t lo0 = ptx::lop3<0xEA>(w, 0x000F000Fu, kMagic);  // (a & b) | c
  const uint32_t hi0 = ptx::lop3<0xEA>(w, 0x00F000F0u, kMagic);
  const uint32_t w8 = w >> 8;
  const uint32_t lo1 = ptx::lop3<0xEA>(w8, 0x000F000Fu, kMagic);
  const uint32_t hi1 = ptx::lop3<0xEA>(w8, 0x00F000F0u, kMagic);
  out[0] = hmul2_rn(hsub2_rn(lo0, c.zlo), c.s2);
  out[1] = hmul2_rn(hfma2_rn(hi0, kInv16, c.zhi), c.s2);
  out[2] = hmul2_rn(hsub2_rn(lo1, c.zlo), c.s2);
  out[3] = hmul2_rn(hfma2_rn(hi1, kInv16, c.zhi), c.s2);
}

// bf16 variant (QUICK_FLAG_BF16): X, scales and Y in bf16.  bf16 has an 8-bit
// significand, so the magic number is 128 (0x4300, ulp 1 up to 256): each nibble pair is shifted to
// bits 0-3 / 16-19 and OR-ed into 0x4300 4300 -> bf16 (128 + q); (q - z) = that - (128 + z), exact;
// one bf16 RN multiply by s -> bf16_rne((q - z) * s), bit-identical to the oracle's bf16 dequant.
// Output pairs (k0,k1), (k2,k3), (k4,k5), (k6,k7) as for fp16 (same v1 nibble order).
__device__ __forceinline__ uint32_t bsub2_rn(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t bmul2_rn(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ void dequant_word_bf16(uint32_t w, const DequantConsts& c, uint32_t* out) {
  constexpr uint32_t kMagic = 0x43004300u;   // bf16x2 (128, 128)
  out[0] = bmul2_rn(bsub2_rn(ptx::lop3<0xEA>(w, 0x000F000Fu, kMagic), c.zlo), c.s2);
  out[1] = bmul2_rn(bsub2_rn(ptx::lop3<0xEA>(w >> 4, 0x000F000Fu, kMagic), c.zlo), c.s2);
  out[2] = bmul2_rn(bsub2_rn(ptx::lop3<0xEA>(w >> 8, 0x000F000Fu, kMagic), c.zlo), c.s2);
  out[3] = bmul2_rn(bsub2_rn(ptx::lop3<0xEA>(w >> 12, 0x000F000Fu, kMagic), c.zlo), c.s2);
}
template <bool BF>
__device__ __forceinline__ void dequant_w(uint32_t w, const DequantConsts& c, uint32_t* out) {
  if constexpr (BF)
    dequant_word_bf16(w, c, out);
  else
    dequant_word(w, c, out);
}
// group constants of the bf16 variant: zlo = bf16x2 (128 + z), s2 = (s, s)
__device__ __forceinline__ DequantConsts make_consts_bf16(uint32_t sbits, uint32_t z) {
  DequantConsts c;
  c.zlo = __byte_perm(0x4300u + z, 0u, 0x1010);
  c.zhi = 0u;
  c.s2 = __byte_perm(sbits, 0u, 0x1010);
  return c;
}
// 16-bit output conversions (fp16 or bf16, round to nearest even)
template <bool BF>
__device__ __forceinline__ uint16_t cvt16(float f) {
  if constexpr (BF)
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
  else
    return __half_as_ushort(__float2half_rn(f));
}
template <bool BF>
__device__ __forceinline__ uint32_t cvt16x2(float a, float b) {
  if constexpr (BF) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

// a 16-bit bias value (fp16, or bf16 for the bf16 variant) as fp32 (exact)
template <bool BF>
__device__ __forceinline__ float bias_f(uint16_t b) {
  if constexpr (BF)
    return __uint_as_float((uint32_t)b << 16);
  else
    return __half2float(__ushort_as_half(b));
}

// SiLU(g) * u in fp32 (the fused gate||up epilogue, QUICK_FLAG_SILU_MUL)
__device__ __forceinline__ float silu_mul(float g, float u) {
  // MUFU exp2 + fast reciprocal-division (~2 ulp in fp32; the result is rounded to 16 bits)
  return __fdividef(g * u, 1.0f + __expf(-g));
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms of 1024 B (SBO), version 1
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;              // LBO (unused for swizzled K-major), 16 B
  d |= (uint64_t)(1024u >> 4) << 32;    // SBO = 1024 B between 8-row groups
  d |= (uint64_t)1u << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2u << 61;              // layout: SWIZZLE_128B
  return d;
}

// tcgen05 instruction descriptor, kind::f16: D fp32, A/B fp16, both K-major, M=128 (256 for a
// CTA pair), N=BN
template <int BN, int MM = kTileRows, bool BF = false>
__device__ __forceinline__ constexpr uint32_t instr_desc() {
  // bits 7-9 / 10-12: A / B format of kind::f16 (0 = fp16, 1 = bf16)
  return (1u << 4) | (BF ? (1u << 7) | (1u << 10) : 0u) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(MM >> 4) << 24);
}

template <int BN, bool SK, bool GBIG, bool TRACE, int AM = 0, bool BF = false>
__global__ void __launch_bounds__(Cfg<BN, SK, AM>::THREADS, Cfg<BN, SK, AM>::MAX_CTAS_PER_SM)
    quick_w4a16_tc_kernel(const __grid_constant__ CUtensorMap tmap_x,
                          const __grid_constant__ KParams p) {
  using C = Cfg<BN, SK, AM>;
  constexpr int kThreads = C::THREADS;
  constexpr int kProducerWarp = C::PRODUCER_WARP;
  constexpr int kMmaWarp = C::MMA_WARP;
  constexpr int kDqThreads = C::DQ_THREADS;
  constexpr int NPAR = C::NPAR;
  constexpr int STAGES = C::STAGES;
  constexpr int APL = C::APL;
  constexpr int kAStages = C::ASTAGES;
  constexpr int kDCol = C::DCOL;
  constexpr bool PAIR = C::PAIR;
  // afull arrivals: one per dequant warp for CTA pairs (remote arrivals are expensive); one per
  // thread otherwise (per-warp arrivals measured 0-3 % slower at small M on one CTA)
  constexpr bool kWarpArrive = PAIR;
  if (p.flags & kDebugExitTop) return;
  extern __shared__ uint8_t smem_raw[];
  // 1 KiB-aligned base, computed in the 32-bit shared window (cheap to rematerialise)
  const uint32_t sraw = ptx::smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sbase - sraw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int K = p.K, G = p.G, M = p.M;
  const int S = SK ? 1 : (PAIR ? (int)gridDim.x >> 1 : (int)gridDim.x);   // cluster split-K factor
  // CTA pair: cluster rank 2 x split + member; the even member (leader) issues the MMAs
  const uint32_t crank = PAIR ? ptx::cluster_ctarank() : 0u;
  const uint32_t member = crank & 1u;
  const uint32_t lead_rank = crank & ~1u;
  const int C32 = K / 32;
  const int NG = K / G;
  const bool out_fp32 = (p.flags & QUICK_FLAG_OUT_F32) != 0;
  // fused gate||up (quick_pack_gate_up): TMEM lanes l < 16 and l + 16 of each warp hold a gate row
  // and its up row; Y[m][n'] = SiLU(gate) * up with n' = 64 t + 16 q + l, stored by lanes l < 16
  const bool silu = (p.flags & QUICK_FLAG_SILU_MUL) != 0;
  const bool pdl = (p.flags & QUICK_FLAG_PDL) != 0;
  const bool dbg_nocompute = (p.flags & kDebugNoCompute) != 0;   // load path only (debug)
  const bool dbg_nosttm = (p.flags & kDebugNoSttm) != 0;
  const int g_shift = p.g_shift;
  // group index of k: shift when G is a power of two, division otherwise
  auto group_of = [&](int k) { return g_shift >= 0 ? (k >> g_shift) : (k / G); };

  const uint32_t bar_full = sbase + C::BAR_OFF;
  const uint32_t bar_empty = bar_full + 8 * STAGES;
  const uint32_t bar_afull = bar_empty + 8 * STAGES;
  const uint32_t bar_aempty = bar_afull + 8 * kAStages;
  const uint32_t bar_dfull = bar_aempty + 8 * kAStages;   // [2]
  const uint32_t bar_dempty = bar_dfull + 16;             // [2]
  const uint32_t bar_xfull = bar_dempty + 16;             // [STAGES]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::HOLD_OFF);

  // Prologue.  The producer initialises the barriers and starts loading at once; the other
  // warps wait on named barrier 2 (which orders the inits before them) while the MMA warp
  // allocates TMEM, so the first loads are not held up by the allocation.
  if (warp == kProducerWarp) {
    // one barrier per lane (the barriers are contiguous from BAR_OFF: full[STAGES],
    // empty[STAGES], afull[A], aempty[A], dfull[2], dempty[2], xfull[STAGES]); a serial init of
    // ~20 barriers by one thread delayed every warp's start
    for (int i = lane; i < C::NUM_BARS; i += 32) {
      uint32_t cnt = 1;   // full, aempty, dfull, xfull
      if (i >= STAGES && i < 2 * STAGES)
        cnt = 4 * 32 * APL + 1;   // empty: 128 dequant-thread arrivals per A stage (a thread reading
                                  // the only A stage of a short load stage arrives for both) + 1 commit
      else if (i >= 2 * STAGES && i < 2 * STAGES + kAStages)   // afull: one parity group (CTA pair:
        cnt = kWarpArrive ? (PAIR ? 8 : 4) : 4 * 32;          // one arrival per warp of both members)
      else if (i >= 2 * STAGES + 2 * kAStages + 2 && i < 2 * STAGES + 2 * kAStages + 4)
        cnt = kDqThreads;         // dempty
      ptx::mbar_init(bar_full + 8 * i, cnt);
    }
    ptx::fence_mbar_init();
  }
  uint32_t tmem = 0;
  if (warp == kProducerWarp) {
    if (lane == 0) ptx::prefetch_tmap(&tmap_x);
    __syncwarp();
    ptx::named_bar_arrive(2, kThreads);
  } else {
    if (warp == kMmaWarp) {
      if constexpr (PAIR)
        ptx::tmem_alloc2(ptx::smem_u32(tmem_holder), C::TMEM_COLS);
      else
        ptx::tmem_alloc(ptx::smem_u32(tmem_holder), C::TMEM_COLS);
    }
    ptx::tc_fence_before();
    ptx::named_bar_sync(2, kThreads);
    ptx::tc_fence_after();
    if constexpr (!PAIR) tmem = *tmem_holder;
  }
  // CTA pair: the peer's barriers must be initialised before any remote arrival or TMA
  // completion targets them; the pair allocation's address is read after the cluster barrier
  // (the allocation is one operation of both CTAs).  (compute-sanitizer racecheck reports 65
  // hazards in every pair launch, all between accesses inside the compiler-generated
  // tcgen05.alloc.cta_group::2 handshake -- UTCATOMSWS.2CTA, then STAS/ATOMS/SYNCS on the
  // reserved shared-memory words 0x50-0x60 of both CTAs -- none in this kernel's own code.)
  if constexpr (PAIR) {
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    tmem = *tmem_holder;
  }
  if (p.flags & kDebugExitPrologue) {
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
      ptx::tc_fence_after();
      if constexpr (PAIR)
        ptx::tmem_dealloc2(tmem, C::TMEM_COLS);
      else
        ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
    if constexpr (PAIR) ptx::cluster_sync();
    return;
  }
  // debug tracing (TRACE instantiation only, tools/trace_gemm.py): clock64 stamps per stage
  unsigned long long* tr = nullptr;
  const unsigned lin16 = SK ? blockIdx.x : blockIdx.z * gridDim.x + blockIdx.x;
  if (TRACE && blockIdx.y == 0 && lin16 < 16) tr = p.trace + (size_t)lin16 * kTraceStride;
  auto stamp = [&](int ev, int i) {
    if (TRACE && tr != nullptr && i < kTraceStages) tr[8 + ev * kTraceStages + i] = clock64();
  };
  if (TRACE && tr != nullptr && threadIdx.x == 0) tr[0] = clock64();
  unsigned long long t_start_ns = 0;
  if (TRACE && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start_ns));
  // PDL: the next kernel in the stream may launch once every CTA of this grid has triggered.
  // The trigger is placed where each warp's main loop ends (the CTA's epilogue), so the next
  // grid's CTAs land on SMs whose CTAs are finishing (its prologue, weight prefetch and first
  // dequantized stages overlap our epilogue); triggering right after the prologue let them
  // double up on SMs of grids with fewer CTAs than SMs (measured slower on 13B shapes).
  // The next grid still waits (griddepcontrol.wait) for this grid's completion before it
  // reads X or writes anything.
  const bool pdl_early = (p.flags & kDebugPdlEarly) != 0;
  if (pdl_early) ptx::griddep_launch_dependents();

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------------ producer
    // The whole warp runs the (warp-uniform) loop; one elected lane issues the copies, so the
    // addresses stay in uniform registers and no per-lane waterfall is generated.  Load
    // stages never straddle segments (the last one of a segment may be short).
    // weights: streamed once per wave of m-tiles (evict-normal for m_tiles > 1 was measured 1-2 %
    // slower on the 70B shapes at M >= 128 without fixing the M = 1024 DRAM re-reads,
    // profiles/r02_l2_policy_ab.txt)
    const uint64_t pol_w = ptx::policy_evict_first();
    const uint64_t pol_x = ptx::policy_evict_last();   // X: re-read by every n-tile
    SegIter it(p, SK, C::PAIR);
    Seg sg;
    int slot = 0, lf = 0;
    uint32_t ph = 0;
    int pre = -1;   // PDL: weight copies of the first `pre` load stages go before the X wait
    // X tile of load stage `j` into slot `xs`.  CTA pair: each member loads its half of the
    // tokens; both halves complete on the leader's xfull barrier, which expects both
    auto load_x = [&](int xs, int m0, int kc) {
      if constexpr (PAIR) {
        if (member == 0) ptx::mbar_arrive_expect_tx(bar_xfull + 8 * xs, 2 * C::X_BYTES);
        ptx::tma_load_3d_pair(sbase + C::X_OFF + xs * C::X_BYTES, &tmap_x, 0, m0 + (int)member * C::XN, kc,
                              ptx::mapa(bar_xfull + 8 * xs, lead_rank), pol_x);
      } else {
        ptx::mbar_arrive_expect_tx(bar_xfull + 8 * xs, C::X_BYTES);
        ptx::tma_load_3d_hint(sbase + C::X_OFF + xs * C::X_BYTES, &tmap_x, 0, m0, kc, bar_xfull + 8 * xs, pol_x);
      }
    };
    while (it.next(sg)) {
      const uint8_t* wbase = p.packed + (size_t)sg.t * C32 * kChunkBytes;
      const uint8_t* mbase = p.packed + (size_t)K * p.N / 2 + (size_t)sg.t * NG * kMetaBytes;
      const int m0 = sg.mt * BN;
      const int k_seg_end = min(sg.a_hi * kKA, K);
      const int nl = (sg.a_hi - sg.a_lo + APL - 1) / APL;
      if (pre < 0) pre = pdl ? (nl < STAGES ? nl : STAGES) : 0;
      // (the host never sets QUICK_FLAG_PDL for the 256-token tile)
      for (int l = 0; l < nl; ++l, ++lf) {
        const int kl0 = (sg.a_lo + l * APL) * kKA;
        const int kv = min(C::KL, k_seg_end - kl0);   // valid k in this load stage
        if (lane == 0) stamp(0, lf);
        if (lf >= pre) ptx::mbar_wait(bar_empty + 8 * slot, ph ^ 1u);
        const int g0 = group_of(kl0);
        const uint32_t meta_bytes = (uint32_t)(group_of(kl0 + kv - 1) - g0 + 1) * kMetaBytes;
        const uint32_t full = bar_full + 8 * slot;
        if (ptx::elect_one()) {
          ptx::mbar_arrive_expect_tx(full, (uint32_t)kv * 64u + meta_bytes);
          ptx::bulk_load_hint(sbase + C::W_OFF + slot * C::W_BYTES,
                              wbase + (size_t)(kl0 / 32) * kChunkBytes, (uint32_t)kv * 64u, full,
                              pol_w);
          ptx::bulk_load_hint(sbase + C::M_OFF + slot * C::M_BYTES,
                              mbase + (size_t)g0 * kMetaBytes, meta_bytes, full, pol_w);
          if (lf >= pre && !(pre == 0 && lf == 0)) {
            load_x(slot, m0, kl0 / 64);
          } else if (lf == (pre > 0 ? pre - 1 : 0)) {
            if (pdl) ptx::griddep_wait();
            if (TRACE) {   // (trace records: when the previous grid's completion released this CTA)
              unsigned long long t_gd;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_gd));
              const size_t lin = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
              p.trace[16 * (size_t)kTraceStride + 4 * lin + 3] = pdl ? t_gd : 0ull;
            }
            for (int j = 0; j <= lf; ++j)   // X of the stages issued so far (all in this segment)
              load_x(j, m0, (sg.a_lo + j * APL) * kKA / 64);
          }
        }
        __syncwarp();
        if (lane == 0) stamp(1, lf);
        if (++slot == STAGES) {
          slot = 0;
          ph ^= 1u;
        }
      }
    }
    ptx::griddep_launch_dependents();
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------------ MMA issuer
    // Warp-uniform loop; one elected lane issues the MMAs and the commits (a commit tracks
    // the async tcgen05 ops of the thread that issues it, so the same lane does both).
    constexpr uint32_t idesc = instr_desc<BN, PAIR ? 2 * kTileRows : kTileRows, BF>();
    const uint64_t desc0 = sw128_desc(sbase + C::X_OFF);
    // AM = 1: the A stage is an SW128 K-major tile in shared memory (two 64-k sub-tiles of 16 KiB)
    const uint64_t adesc0 = sw128_desc(sbase + (uint32_t)C::A_OFF);
    // one K=16 MMA of A stage `a_slot`; `a_col` is its TMEM column (AM = 0)
    auto mma_k = [&](uint32_t d, uint32_t a_col, int a_slot, int kk, uint64_t bdesc, uint32_t acc) {
      if constexpr (PAIR) {
        ptx::mma2_f16_ts(d, a_col + kk * 8, bdesc, idesc, acc);
      } else if constexpr (!C::SMEM_A) {
        ptx::mma_f16_ts(d, a_col + kk * 8, bdesc, idesc, acc);
      } else {
        ptx::mma_f16_ss(d, adesc0 + (uint64_t)((a_slot * C::A_BYTES + (kk >> 2) * (kTileRows * 128)) >> 4) +
                               (uint64_t)((kk & 3) * 2), bdesc, idesc, acc);
      }
    };
    // completion of the MMAs issued so far -> barrier (both members' copies for a pair)
    const uint16_t cmask = (uint16_t)(3u << lead_rank);
    auto commit = [&](uint32_t bar) {
      if constexpr (PAIR)
        ptx::mma2_commit(bar, cmask);
      else
        ptx::mma_commit(bar);
    };
    SegIter it(p, SK, C::PAIR);
    Seg sg;
    int slot = 0, as = 0, si = 0, ia = 0, lf_mma = 0;
    uint32_t aph = 0, xph = 0;
    // CTA pair: the odd member issues nothing; it only counts the stages for the drain below
    // (the leader's commits arrive on its barriers too)
    if (PAIR && member != 0) {
      while (it.next(sg)) {
        ia += sg.a_hi - sg.a_lo;
        lf_mma += (sg.a_hi - sg.a_lo + APL - 1) / APL;
      }
    }
    while ((!PAIR || member == 0) && it.next(sg)) {
      const int db = SK ? (si & 1) : 0;
      // stream-K: the accumulator of segment si - 2 must have been read out
      if (SK && si >= 2) ptx::mbar_wait(bar_dempty + 8 * db, (uint32_t)(((si >> 1) + 1) & 1));
      const uint32_t d_col = tmem + kDCol + (uint32_t)(db * C::NACC * BN);
      int sub = 0;
      const bool dbg_skip = dbg_nocompute || (p.flags & (kDebugNoMma | kDebugNoSttm));
      for (int a = sg.a_lo; a < sg.a_hi; ++a, ++ia) {
        // Paired fast path (2 A stages per load stage, both full, not the segment's first): one
        // iteration waits both A stages and the X tile, and issues 16 MMAs with one set of
        // bookkeeping -- the per-stage loop overhead of this warp (~470 cycles measured with
        // two CTAs per SM) was the small-M bottleneck, not the tensor pipe (~200 cycles).
        // (APL == 1: the two A stages are consecutive load stages with their own X slots)
        if (sub == 0 && a + 1 < sg.a_hi && (a + 2) * kKA <= K && a != sg.a_lo) {
          const int as1 = (as + 1 == kAStages) ? 0 : as + 1;
          const uint32_t aph1 = (as + 1 == kAStages) ? (aph ^ 1u) : aph;
          const int slot1 = APL == 2 ? slot : (slot + 1 == STAGES ? 0 : slot + 1);
          const uint32_t xph1 = (APL == 1 && slot + 1 == STAGES) ? (xph ^ 1u) : xph;
          ptx::mbar_wait(bar_afull + 8 * as, aph);
          ptx::mbar_wait(bar_xfull + 8 * slot, xph);
          ptx::tc_fence_after();
          const uint64_t dstage = desc0 + (uint64_t)((slot * C::X_BYTES) >> 4);
          if (ptx::elect_one()) {
            if (!dbg_skip) {
              const uint32_t a_col = tmem + as * kAColsPerStage;
#pragma unroll
              for (int kk = 0; kk < kKA / 16; ++kk)
                mma_k(d_col + (uint32_t)((kk % C::NACC) * BN), a_col, as, kk,
                      dstage + (uint64_t)((kk >> 2) * (C::X_SUB >> 4) + (kk & 3) * 2), 1u);
            }
            commit(bar_aempty + 8 * as);
            if (APL == 1) commit(bar_empty + 8 * slot);
          }
          __syncwarp();
          ptx::mbar_wait(bar_afull + 8 * as1, aph1);
          if (APL == 1) ptx::mbar_wait(bar_xfull + 8 * slot1, xph1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            if (!dbg_skip) {
              const uint32_t a_col = tmem + as1 * kAColsPerStage;
              const uint64_t d1 = APL == 2 ? dstage + (uint64_t)((2 * C::X_SUB) >> 4)
                                           : desc0 + (uint64_t)((slot1 * C::X_BYTES) >> 4);
#pragma unroll
              for (int kk = 0; kk < kKA / 16; ++kk)
                mma_k(d_col + (uint32_t)((kk % C::NACC) * BN), a_col, as1, kk,
                      d1 + (uint64_t)((kk >> 2) * (C::X_SUB >> 4) + (kk & 3) * 2), 1u);
            }
            commit(bar_aempty + 8 * as1);
            commit(bar_empty + 8 * slot1);
            if (a + 1 == sg.a_hi - 1) commit(bar_dfull + 8 * db);
          }
          __syncwarp();
          ++a;
          ++ia;
          lf_mma += (APL == 1) ? 2 : 1;
          slot = slot1;
          xph = xph1;
          if (++slot == STAGES) {
            slot = 0;
            xph ^= 1u;
          }
          as = (as1 + 1 == kAStages) ? 0 : as1 + 1;
          aph = (as1 + 1 == kAStages) ? (aph1 ^ 1u) : aph1;
          continue;
        }
        // A stage written by the 4 warps of its parity group (afull); the X tile of its load
        // stage has its own barrier (xfull), waited once per load stage
        ptx::mbar_wait(bar_afull + 8 * as, aph);
        if (sub == 0) ptx::mbar_wait(bar_xfull + 8 * slot, xph);   // this load stage's X tile
        if (lane == 0) stamp(5, ia);
        ptx::tc_fence_after();
        const int kv = min(kKA, K - a * kKA);   // 128, or 64 at the end of K
        const bool last_of_load = (sub == APL - 1) || (a == sg.a_hi - 1);
        if (ptx::elect_one()) {
          if (dbg_skip) {
            commit(bar_aempty + 8 * as);
            if (last_of_load) commit(bar_empty + 8 * slot);
            if (a == sg.a_hi - 1) commit(bar_dfull + 8 * db);
          } else {
          const uint32_t a_col = tmem + as * kAColsPerStage;
          // descriptor start address in 16-B units: X slot, 64-k sub-tile, then 32 B per K=16
          const uint64_t dstage = desc0 + (uint64_t)((slot * C::X_BYTES + sub * 2 * C::X_SUB) >> 4);
          const bool first = (a == sg.a_lo);
          if (kv == kKA && !first) {
            // steady state: 8 unpredicated, always-accumulating MMAs (lean issue: the A-ring
            // slot is held until these complete, so issue latency throttles the dequantizers)
#pragma unroll
            for (int kk = 0; kk < kKA / 16; ++kk)
              mma_k(d_col + (uint32_t)((kk % C::NACC) * BN), a_col, as, kk,
                    dstage + (uint64_t)((kk >> 2) * (C::X_SUB >> 4) + (kk & 3) * 2), 1u);
          } else {
#pragma unroll
            for (int kk = 0; kk < kKA / 16; ++kk) {
              if (kk * 16 < kv)
                mma_k(d_col + (uint32_t)((kk % C::NACC) * BN), a_col, as, kk,
                      dstage + (uint64_t)((kk >> 2) * (C::X_SUB >> 4) + (kk & 3) * 2),
                      (first && kk < C::NACC) ? 0u : 1u);
            }
          }
          commit(bar_aempty + 8 * as);    // A stage free once these MMAs complete
          if (last_of_load) commit(bar_empty + 8 * slot);   // X of this load stage used
          if (a == sg.a_hi - 1) commit(bar_dfull + 8 * db);  // segment accumulated
          }
        }
        __syncwarp();
        if (lane == 0) stamp(6, ia);
        if (last_of_load) {
          sub = 0;
          ++lf_mma;
          if (++slot == STAGES) {
            slot = 0;
            xph ^= 1u;
          }
        } else {
          ++sub;
        }
        if (++as == kAStages) {
          as = 0;
          aph ^= 1u;
        }
      }
      ++si;
    }
    // Drain: the mbarrier arrivals of this warp's last tcgen05.commits (A-ring and load-ring
    // slots) must have landed before the CTA exits -- a late arrival would hit the shared
    // memory of the next CTA placed on this SM (a later wave, or the next kernel under PDL).
    // Slot s of a ring of R slots received ceil((n - s) / R) commits for n stages in total.
    for (int s2 = 0; s2 < kAStages; ++s2) {
      const int n = (ia - s2 + kAStages - 1) / kAStages;
      if (n > 0) ptx::mbar_wait(bar_aempty + 8 * s2, (uint32_t)((n - 1) & 1));
    }
    for (int s2 = 0; s2 < STAGES; ++s2) {
      const int n = (lf_mma - s2 + STAGES - 1) / STAGES;
      if (n > 0) ptx::mbar_wait(bar_empty + 8 * s2, (uint32_t)((n - 1) & 1));
    }
    ptx::griddep_launch_dependents();
  } else {
    // ------------------------------------------------------------------ dequantizers
    // Warp w owns TMEM lane quarter q = w % 4 (the only lanes it may access) and takes the
    // A stages of parity p (two warps per quarter, so each SM sub-partition interleaves two
    // independent dequant streams per CTA).  Per A stage a thread (one TMEM lane = one weight
    // row) loads 4 x 16 B = 128 codes and writes 64 TMEM columns in two tcgen05.st.32x32b.x32;
    // the second half is dequantized while the first store drains.  Group constants (s,
    // 1024 + z, -(64 + z)) are rebuilt only when the group changes (G % 128 == 0), or per
    // 32-k chunk otherwise.  Every thread arrives on the barriers itself.  After each segment
    // the same warps run its epilogue (their TMEM lanes, half of the columns each).
    const int q = warp & 3;              // TMEM lane quarter this warp may access (warp id % 4)
    const int par = (warp - C::DQ_BASE) >> 2;   // group: A stages a with (a - first) % NPAR == par
    const int r = q * 32 + lane;         // tile row: output column n = 128 t + r
    const uint32_t tlane = (uint32_t)(q * 32) << 16;
    // 32-bit shared-window addresses: explicit ld.shared (a generic pointer through the
    // 1 KiB alignment cast compiles to slower generic LD.E)
    // (the base is made opaque so the compiler keeps it in a register instead of
    // re-deriving the aligned shared-window address in every iteration)
    uint32_t sb = sbase;
    asm volatile("" : "+r"(sb));
    const uint32_t wrow = sb + C::W_OFF + r * 16;
    const uint32_t mrow = sb + C::M_OFF + r * 2;           // scale of row r in a meta block
    const uint32_t zrow = sb + C::M_OFF + 256 + (r >> 1);  // zero byte of row r
    const uint32_t zsh = (uint32_t)(r & 1) * 4u;           // nibble of row r in its byte
    const uint32_t zsh_hi = 4u - zsh;
    int gsh = g_shift;                                     // kept in a register (no LDC per stage)
    asm volatile("" : "+r"(gsh));
    // group constants straight from the meta bytes (8 instructions): the zero byte is
    // replicated into both fp16 halves with one PRMT, then shifted/masked into 1024 + z and
    // -(64 + z) (bit-identical to make_consts)
    auto consts_at = [&](uint32_t mo) {
      const uint32_t zb = ptx::lds_u8(zrow + mo);
      const uint32_t sbits = ptx::lds_u16(mrow + mo);
      const uint32_t zr = __byte_perm(zb, 0u, 0x4040);   // [zb, 0, zb, 0]
      DequantConsts c;
      if constexpr (BF) {
        c.zlo = ptx::lop3<0xEA>(zr >> zsh, 0x000F000Fu, 0x43004300u);   // bf16 (128 + z)
        c.zhi = 0u;
      } else {
        c.zlo = ptx::lop3<0xEA>(zr >> zsh, 0x000F000Fu, 0x64006400u);
        c.zhi = ptx::lop3<0xEA>(zr << zsh_hi, 0x00F000F0u, 0xD400D400u);
      }
      c.s2 = __byte_perm(sbits, 0u, 0x1010);
      return c;
    };
    const bool tw = TRACE && (warp == C::DQ_BASE && lane == 0);
    // A stage written: CTA pair members both arrive on the leader's afull (its MMA reads both
    // halves of A from the two TMEMs), one arrival per warp after a warp sync (128 remote
    // per-thread arrivals per stage were measured ~750 cycles slower than local ones)
    const uint32_t afull_lead = PAIR ? ptx::mapa(bar_afull, lead_rank) : 0u;
    auto arrive_afull = [&](int as_) {
      if constexpr (kWarpArrive) {
        __syncwarp();
        if (lane == 0) {
          if (member != 0)
            ptx::mbar_arrive_remote(afull_lead + 8u * (uint32_t)as_);
          else
            ptx::mbar_arrive(bar_afull + 8 * as_);
        }
      } else {
        ptx::mbar_arrive(bar_afull + 8 * as_);
      }
    };
    // epilogue: the accumulator columns are split over the groups in chunks of >= 8
    constexpr int kColsPerWarp = BN / NPAR >= 8 ? BN / NPAR : 8;
    const int j0 = par * kColsPerWarp;   // this warp's share of the accumulator columns
    const int jend = min(j0 + kColsPerWarp, BN);
    uint32_t a_regs[32];
    SegIter it(p, SK, C::PAIR);
    Seg sg;
    int ia = 0, si = 0, lbase = 0;       // flat A-stage index, segment index, first load stage
    while (it.next(sg)) {
      int g_prev = -1;                   // group constants are per tile: reset per segment
      DequantConsts cst = make_consts(0, 0);
      const int k_seg_end = min(sg.a_hi * kKA, K);
      // This warp's A stages in the segment: every NPAR-th one, starting at the first whose
      // flat index is congruent to its group.  With APL in {1, 2} (dividing NPAR) the A stage's
      // position inside its load stage (sub) is the same for all of them, and the load stage
      // advances by NPAR / APL per step, so slot / phase / A-ring indices are kept
      // incrementally (no divisions).
      {
        const int rel0 = (par - ia) & (NPAR - 1);
        const int sub = rel0 % APL;
        int lf = lbase + rel0 / APL;
        int slot = lf % STAGES;
        uint32_t fph = (uint32_t)((lf / STAGES) & 1);
        int iw = ia + rel0;
        int as = iw % kAStages;
        uint32_t aph = (uint32_t)((iw / kAStages) & 1);
        const uint32_t sub_off = (uint32_t)(sub * 4 * kChunkBytes);
        // shared-memory addresses of this warp's slot, advanced incrementally with the slot (no
        // per-stage multiplies: the dequant is bound by the FMA pipe, where IMADs also issue)
        uint32_t wslot = wrow + (uint32_t)(slot * C::W_BYTES) + sub_off;
        uint32_t mslot = (uint32_t)(slot * C::M_BYTES);
        uint32_t acol_as = tmem + tlane + (uint32_t)(as * kAColsPerStage);
        // G == 128 (one group per A stage, the BJ value): the stage's group is block `sub` of its
        // load stage's metadata, so the constants need no group arithmetic
        const bool g128 = GBIG && gsh == 7;
        const uint32_t msub = (uint32_t)sub * kMetaBytes;
        // Lean steady-state loop (G a power of two >= 128, A in TMEM): the instruction count per
        // A stage is what bounds the small-M decode (ncu: ~300 warp instructions per warp-stage,
        // 208 of them the dequantization).  Here: one barrier register per ring (full/empty and
        // afull/aempty are constant offsets apart), waits as single asm loops, the stage's metadata
        // block folded into one running address, the arrival count and short-stage tests
        // precomputed per segment.
        // (G == 128 only: a larger power-of-two group can straddle a load stage's two A stages, which
        // the general loop below handles)
        bool lean = false;
        if constexpr (GBIG && AM == 0) lean = !dbg_nosttm && !dbg_nocompute && g128;
        if (lean) {
          const int a_end = sg.a_hi;
          // K % 128 == 64: the segment's last A stage holds one half (64 k) only
          const int a_short = (k_seg_end & (kKA - 1)) != 0 ? a_end - 1 : 0x7fffffff;
          // a load stage holding a single A stage (segment end): this thread also arrives for the
          // other parity's share
          const int a_cnt2 = (APL == 2 && sub == 0) ? a_end - 1 : 0x7fffffff;
          // ring positions are kept as (slot, phase) pairs only; the barrier, shared-memory and
          // TMEM addresses are re-derived from them each stage (LEA / one IMAD: fewer live
          // registers and no loop-carried address copies)
          const uint32_t wbase = wrow + sub_off;                    // + slot x W_BYTES
          const uint32_t mbase = mrow + msub;                       // + slot x M_BYTES
          const uint32_t zdelta = zrow - mrow;
          const uint32_t abase = tmem + tlane;                      // + as x 64 columns
          for (int a = sg.a_lo + rel0; a < a_end; a += NPAR, iw += NPAR) {
            const uint32_t fbar = bar_full + 8u * (uint32_t)slot;   // empty = fbar + 8 STAGES
            const uint32_t wp = wbase + (uint32_t)slot * (uint32_t)C::W_BYTES;
            const uint32_t maddr = mbase + (uint32_t)slot * (uint32_t)C::M_BYTES;
            ptx::mbar_wait_loop(fbar, fph);
            if (tw) stamp(2, iw);
            uint4 w[4];
            w[0] = ptx::lds128(wp);
            w[1] = ptx::lds128(wp + kChunkBytes);
            w[2] = ptx::lds128(wp + 2 * kChunkBytes);
            w[3] = ptx::lds128(wp + 3 * kChunkBytes);
            DequantConsts c;
            {
              const uint32_t zb = ptx::lds_u8(maddr + zdelta);
              const uint32_t sbits = ptx::lds_u16(maddr);
              const uint32_t zr = __byte_perm(zb, 0u, 0x4040);   // [zb, 0, zb, 0]
              if constexpr (BF) {
                c.zlo = ptx::lop3<0xEA>(zr >> zsh, 0x000F000Fu, 0x43004300u);
                c.zhi = 0u;
              } else {
                c.zlo = ptx::lop3<0xEA>(zr >> zsh, 0x000F000Fu, 0x64006400u);
                c.zhi = ptx::lop3<0xEA>(zr << zsh_hi, 0x00F000F0u, 0xD400D400u);
              }
              c.s2 = __byte_perm(sbits, 0u, 0x1010);
            }
            ptx::mbar_arrive_cnt(fbar + 8u * STAGES, a == a_cnt2 ? 2u : 1u);
            dequant_w<BF>(w[0].x, c, a_regs + 0);
            dequant_w<BF>(w[0].y, c, a_regs + 4);
            dequant_w<BF>(w[0].z, c, a_regs + 8);
            dequant_w<BF>(w[0].w, c, a_regs + 12);
            dequant_w<BF>(w[1].x, c, a_regs + 16);
            dequant_w<BF>(w[1].y, c, a_regs + 20);
            dequant_w<BF>(w[1].z, c, a_regs + 24);
            dequant_w<BF>(w[1].w, c, a_regs + 28);
            const uint32_t abar = bar_afull + 8u * (uint32_t)as;   // aempty = abar + 8 kAStages
            const uint32_t acol = abase + (uint32_t)as * (uint32_t)kAColsPerStage;
            ptx::mbar_wait_loop(abar + 8u * kAStages, aph ^ 1u);
            if (tw) stamp(3, iw);
            ptx::tc_fence_after();
            ptx::tmem_st_32x32b_x32(acol, a_regs);
            if (a != a_short) {
              uint32_t b_regs[32];
              dequant_w<BF>(w[2].x, c, b_regs + 0);
              dequant_w<BF>(w[2].y, c, b_regs + 4);
              dequant_w<BF>(w[2].z, c, b_regs + 8);
              dequant_w<BF>(w[2].w, c, b_regs + 12);
              dequant_w<BF>(w[3].x, c, b_regs + 16);
              dequant_w<BF>(w[3].y, c, b_regs + 20);
              dequant_w<BF>(w[3].z, c, b_regs + 24);
              dequant_w<BF>(w[3].w, c, b_regs + 28);
              ptx::tmem_st_32x32b_x32(acol + 32, b_regs);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            if constexpr (kWarpArrive)
              arrive_afull(as);
            else
              ptx::mbar_arrive(abar);
            if (tw) stamp(4, iw);
            // advance: the load ring by NPAR / APL slots, the A ring by NPAR slots
            slot += NPAR / APL;
            if (slot >= STAGES) {
              slot -= STAGES;
              fph ^= 1u;
            }
            as += NPAR;
            if (as >= kAStages) {
              as -= kAStages;
              aph ^= 1u;
            }
          }
        }
        for (int a = sg.a_lo + rel0; !lean && a < sg.a_hi; a += NPAR, iw += NPAR) {
          const int ka = a * kKA;
          ptx::mbar_wait(bar_full + 8 * slot, fph);
          if (tw) stamp(2, iw);
          const uint32_t wp = wslot;
          const uint32_t moff = mslot;
          const int g0 = GBIG ? ((ka - sub * kKA) >> gsh) : group_of(ka - sub * kKA);
          // all four 16-B chunks: a short last stage (K % 128 == 64) reads two stale chunks of
          // its own slot and ignores them
          uint4 w[4];
          w[0] = ptx::lds128(wp);
          w[1] = ptx::lds128(wp + kChunkBytes);
          w[2] = ptx::lds128(wp + 2 * kChunkBytes);
          w[3] = ptx::lds128(wp + 3 * kChunkBytes);
          DequantConsts cst1;
          if constexpr (GBIG) {
            if (g128) {
              cst = consts_at(moff + msub);
            } else {
              const int g = ka >> gsh;
              if (g != g_prev) {
                cst = consts_at(moff + (uint32_t)(g - g0) * kMetaBytes);
                g_prev = g;
              }
            }
          } else {
            cst = consts_at(moff + (uint32_t)(group_of(ka) - g0) * kMetaBytes);
            cst1 = consts_at(moff + (uint32_t)(group_of(ka + 32) - g0) * kMetaBytes);
          }
          // one arrival per thread per A stage; a load stage holding a single A stage (end of
          // a segment) gets the other parity's share from the same thread
          const uint32_t cnt = (APL == 2 && sub == 0 && a + 1 >= sg.a_hi) ? 2u : 1u;
          ptx::mbar_arrive_cnt(bar_empty + 8 * slot, cnt);
          if (dbg_nocompute) {
            ptx::mbar_wait(bar_aempty + 8 * as, aph ^ 1u);
            arrive_afull(as);
          } else {
            dequant_w<BF>(w[0].x, cst, a_regs + 0);
            dequant_w<BF>(w[0].y, cst, a_regs + 4);
            dequant_w<BF>(w[0].z, cst, a_regs + 8);
            dequant_w<BF>(w[0].w, cst, a_regs + 12);
            const DequantConsts& c1 = GBIG ? cst : cst1;
            dequant_w<BF>(w[1].x, c1, a_regs + 16);
            dequant_w<BF>(w[1].y, c1, a_regs + 20);
            dequant_w<BF>(w[1].z, c1, a_regs + 24);
            dequant_w<BF>(w[1].w, c1, a_regs + 28);
            ptx::mbar_wait(bar_aempty + 8 * as, aph ^ 1u);
            if (tw) stamp(3, iw);
            ptx::tc_fence_after();
            const uint32_t acol = acol_as;
            if (dbg_nosttm) {   // keep the dequant live without storing it
              uint32_t x = 0;
#pragma unroll
              for (int i = 0; i < 32; ++i) x ^= a_regs[i];
              if (x == 0x12345679u) ptx::tmem_st_32x32b_x32(acol, a_regs);
            } else if constexpr (AM == 1) {
              // ablation: write the stage back to shared memory (SW128 K-major: row r at r x 128 B,
              // 16-B chunk c at c ^ (r & 7); 8 rows of a quarter-warp hit 8 distinct chunks)
              const uint32_t arow = sbase + (uint32_t)(C::A_OFF + as * C::A_BYTES) + (uint32_t)r * 128u;
#pragma unroll
              for (int c = 0; c < 8; ++c)
                ptx::sts128(arow + (uint32_t)((c ^ (r & 7)) << 4), a_regs[4 * c], a_regs[4 * c + 1],
                            a_regs[4 * c + 2], a_regs[4 * c + 3]);
            } else {
              ptx::tmem_st_32x32b_x32(acol, a_regs);
            }
            if ((ka + kKA) <= k_seg_end) {   // second half (all but a short last stage)
              DequantConsts cst2, cst3;
              if constexpr (!GBIG) {
                cst2 = consts_at(moff + (uint32_t)(group_of(ka + 64) - g0) * kMetaBytes);
                cst3 = consts_at(moff + (uint32_t)(group_of(ka + 96) - g0) * kMetaBytes);
              }
              const DequantConsts& c2 = GBIG ? cst : cst2;
              const DequantConsts& c3 = GBIG ? cst : cst3;
              uint32_t b_regs[32];
              dequant_w<BF>(w[2].x, c2, b_regs + 0);
              dequant_w<BF>(w[2].y, c2, b_regs + 4);
              dequant_w<BF>(w[2].z, c2, b_regs + 8);
              dequant_w<BF>(w[2].w, c2, b_regs + 12);
              dequant_w<BF>(w[3].x, c3, b_regs + 16);
              dequant_w<BF>(w[3].y, c3, b_regs + 20);
              dequant_w<BF>(w[3].z, c3, b_regs + 24);
              dequant_w<BF>(w[3].w, c3, b_regs + 28);
              if (dbg_nosttm) {
                uint32_t x = 0;
#pragma unroll
                for (int i = 0; i < 32; ++i) x ^= b_regs[i];
                if (x == 0x12345679u) ptx::tmem_st_32x32b_x32(acol + 32, b_regs);
              } else if constexpr (AM == 1) {
                const uint32_t arow =
                    sbase + (uint32_t)(C::A_OFF + as * C::A_BYTES + kTileRows * 128) + (uint32_t)r * 128u;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                  ptx::sts128(arow + (uint32_t)((c ^ (r & 7)) << 4), b_regs[4 * c], b_regs[4 * c + 1],
                              b_regs[4 * c + 2], b_regs[4 * c + 3]);
              } else {
                ptx::tmem_st_32x32b_x32(acol + 32, b_regs);
              }
            }
            if constexpr (AM == 1) {
              ptx::fence_proxy_async_smem();   // generic-proxy stores -> visible to the tensor core
            } else {
              ptx::tmem_wait_st();
              ptx::tc_fence_before();
            }
            arrive_afull(as);
            if (tw) stamp(4, iw);
          }
          slot += NPAR / APL;
          wslot += (uint32_t)((NPAR / APL) * C::W_BYTES);
          mslot += (uint32_t)((NPAR / APL) * C::M_BYTES);
          if (slot >= STAGES) {
            slot -= STAGES;
            wslot -= (uint32_t)(STAGES * C::W_BYTES);
            mslot -= (uint32_t)(STAGES * C::M_BYTES);
            fph ^= 1u;
          }
          as += NPAR;
          acol_as += (uint32_t)(NPAR * kAColsPerStage);
          if (as >= kAStages) {
            as -= kAStages;
            acol_as -= (uint32_t)(kAStages * kAColsPerStage);
            aph ^= 1u;
          }
        }
      }
      ia += sg.a_hi - sg.a_lo;
      lbase += (sg.a_hi - sg.a_lo + APL - 1) / APL;

      // ---------------------------------------------------------------- segment epilogue
      if (!it.more()) ptx::griddep_launch_dependents();   // our last segment: CTA finishing
      const int db = SK ? (si & 1) : 0;
      const int m0 = sg.mt * BN;
      const int n = silu ? sg.t * (kTileRows / 2) + q * 16 + (lane & 15) : sg.t * kTileRows + r;
      const bool silu_store = (lane & 16) == 0;
      // this thread's output column n gets bias[n] (plain outputs only: the host rejects bias + SiLU)
      const float bv = p.bias != nullptr ? bias_f<BF>(p.bias[n]) : 0.0f;
      ptx::mbar_wait(bar_dfull + 8 * db, (uint32_t)((si >> 1) & 1));
      ptx::tc_fence_after();
      if (TRACE && tr != nullptr && warp == C::DQ_BASE && lane == 0) tr[1] = clock64();
      const uint32_t dcol = tmem + tlane + kDCol + (uint32_t)(db * C::NACC * BN);
      // 8 accumulator columns of this thread's row; with NACC = 2 the two partial sums are
      // added here (fixed order: even K=16 steps + odd K=16 steps)
      auto load_d = [&](int jc, uint32_t (&v)[8]) {
        ptx::tmem_ld_32x32b_x8(dcol + jc, v);
        if constexpr (C::NACC == 2) {
          uint32_t v2[8];
          ptx::tmem_ld_32x32b_x8(dcol + BN + jc, v2);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i)
            v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(v2[i]));
        } else {
          ptx::tmem_wait_ld();
        }
      };
      // 32 accumulator columns with one tcgen05.wait::ld (4 loads in flight: the epilogue was a
      // chain of load -> wait round trips, ~9000 cycles per CTA for the 256-token tile)
      constexpr bool kLd32 = C::NACC == 1 && kColsPerWarp % 32 == 0;
      auto load_d32 = [&](int jc, uint32_t (&v)[32]) {
        uint32_t a0[8], a1[8], a2[8], a3[8];
        ptx::tmem_ld_32x32b_x8(dcol + jc, a0);
        ptx::tmem_ld_32x32b_x8(dcol + jc + 8, a1);
        ptx::tmem_ld_32x32b_x8(dcol + jc + 16, a2);
        ptx::tmem_ld_32x32b_x8(dcol + jc + 24, a3);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[i] = a0[i];
          v[8 + i] = a1[i];
          v[16 + i] = a2[i];
          v[24 + i] = a3[i];
        }
      };
      // 8 tokens (columns jc .. jc + 7, the first `cnt` valid) of this thread's output column n
      auto store_y8 = [&](int jc, const float (&f)[8], int cnt) {
#pragma unroll 1
       for (int d = 0; d < p.ndst; ++d) {
        void* Yb = p.Ydst[d];
        if (silu) {   // warp-uniform: every lane shuffles; gate lanes store even tokens, up lanes odd
          float x[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = __shfl_xor_sync(0xffffffffu, f[i], 16);
          uint16_t* yp = reinterpret_cast<uint16_t*>(Yb) + (size_t)(m0 + jc + (silu_store ? 0 : 1)) * p.ldy + n;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float g = silu_store ? f[2 * j] : x[2 * j + 1];
            const float u = silu_store ? x[2 * j] : f[2 * j + 1];
            if (2 * j + (silu_store ? 0 : 1) < cnt) *yp = cvt16<BF>(silu_mul(g, u));
            yp += 2 * p.ldy;
            asm volatile("" : "+l"(yp));
          }
        } else if (out_fp32) {
          float* yp = reinterpret_cast<float*>(Yb) + (size_t)(m0 + jc) * p.ldy + n;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i < cnt) *yp = f[i] + bv;
            yp += p.ldy;
            asm volatile("" : "+l"(yp));
          }
        } else {
          uint16_t* yp = reinterpret_cast<uint16_t*>(Yb) + (size_t)(m0 + jc) * p.ldy + n;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i < cnt) *yp = cvt16<BF>(f[i] + bv);
            yp += p.ldy;
            asm volatile("" : "+l"(yp));
          }
        }
       }
      };
      const bool whole = SK ? (sg.a_lo == 0 && sg.a_hi == p.NA) : (S == 1);
      const int jmax = min(jend, M - m0);   // valid tokens (columns)
      if (whole && kLd32) {
        // column i of the chunk is token m0 + jc + i: one store per token at a running pointer
        // (row stride ldy), the output type and the full-chunk test hoisted out of the loop (the
        // per-element 64-bit index math and branches made this epilogue instruction-bound)
#pragma unroll 1
        for (int jc = j0; jc < jmax; jc += 32) {
          uint32_t v[32];
          load_d32(jc, v);
          const int cnt = jmax - jc;   // valid tokens in this chunk (>= 32: all)
          // (the pointer is made opaque after each bump so that the compiler does not keep 32
          // precomputed 64-bit addresses live)
#pragma unroll 1
         for (int d = 0; d < p.ndst; ++d) {
          void* Yb = p.Ydst[d];
          if (silu) {
            // the partner lane's values, then gate lanes take the even tokens and up lanes the odd
            // ones (each lane computes and stores half of the 32 SiLU*mul results)
            uint32_t x[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = __shfl_xor_sync(0xffffffffu, v[i], 16);
            uint16_t* yp = reinterpret_cast<uint16_t*>(Yb) + (size_t)(m0 + jc + (silu_store ? 0 : 1)) * p.ldy + n;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float g = __uint_as_float(silu_store ? v[2 * j] : x[2 * j + 1]);
              const float u = __uint_as_float(silu_store ? x[2 * j] : v[2 * j + 1]);
              if (2 * j + (silu_store ? 0 : 1) < cnt) *yp = cvt16<BF>(silu_mul(g, u));
              yp += 2 * p.ldy;
              asm volatile("" : "+l"(yp));
            }
          } else if (out_fp32) {
            float* yp = reinterpret_cast<float*>(Yb) + (size_t)(m0 + jc) * p.ldy + n;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (i < cnt) *yp = __uint_as_float(v[i]) + bv;
              yp += p.ldy;
              asm volatile("" : "+l"(yp));
            }
          } else {
            uint16_t* yp = reinterpret_cast<uint16_t*>(Yb) + (size_t)(m0 + jc) * p.ldy + n;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (i < cnt) *yp = cvt16<BF>(__uint_as_float(v[i]) + bv);
              yp += p.ldy;
              asm volatile("" : "+l"(yp));
            }
          }
         }
        }
      } else if (whole) {
        // the full K range of this tile is in our accumulator: straight to Y
#pragma unroll 1
        for (int jc = j0; jc < jmax; jc += 8) {
          uint32_t v[8];
          load_d(jc, v);
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(v[i]);
          store_y8(jc, f, jmax - jc);
        }
      } else if (!SK && kLd32) {
        // cluster split-K: fp32 partial tile [BN][128] into our shared memory (as below)
#pragma unroll 1
        for (int jc = j0; jc < jend; jc += 32) {
          uint32_t v[32];
          load_d32(jc, v);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            ptx::sts_u32(sbase + (uint32_t)(((jc + i) * kTileRows + r) * 4), v[i]);
        }
      } else if (!SK) {
        // cluster split-K: fp32 partial tile [BN][128] into our shared memory (pipeline buffers
        // are free: every stage has been consumed); reduced through DSMEM below
#pragma unroll 1
        for (int jc = j0; jc < jend; jc += 8) {
          uint32_t v[8];
          load_d(jc, v);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            ptx::sts_u32(sbase + (uint32_t)(((jc + i) * kTileRows + r) * 4), v[i]);
        }
      } else {
        // stream-K partial tile.  The tile's units are owned by CTAs c_first..c_last in k
        // order; c_first reaches them at the END of its range (its last segment), the others
        // at the start of theirs, so c_first is the fixed reducer: the others store an fp32
        // partial [BN][128] into their workspace slot and post a release increment without
        // waiting; c_first waits (rarely for long) for all of them, adds their partials in CTA
        // order to its own accumulator (straight from TMEM) and writes Y.  Deterministic.
        const int u_first = sg.tile * p.NA;
        const int c_first = sk_owner(p, u_first);
        const int c_last = sk_owner(p, u_first + p.NA - 1);
        int* sem = p.sems + sg.tile;
        if (sk_cta(p.flags) != c_first) {
          float* slot_ws = p.ws + (size_t)sk_cta(p.flags) * (BN * kTileRows);
#pragma unroll 1
          for (int jc = j0; jc < jmax; jc += 8) {
            uint32_t v[8];
            load_d(jc, v);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (jc + i < jmax) __stcg(slot_ws + (jc + i) * kTileRows + r, __uint_as_float(v[i]));
          }
          ptx::tc_fence_before();
          ptx::mbar_arrive(bar_dempty + 8 * db);   // the accumulator has been read
          // the named barrier orders every partial store of the CTA before one thread's gpu-scope
          // release (cumulativity); nobody waits for the increment itself
          ptx::named_bar_sync(1, kDqThreads);
          if (threadIdx.x == 32 * C::DQ_BASE) ptx::red_release_gpu_add(sem, 1);   // first dequant thread
        } else {
          if (threadIdx.x == 32 * C::DQ_BASE) {
            const int want = c_last - c_first;
            while (ptx::ld_acquire_gpu(sem) < want) {
            }
            *sem = 0;   // self-reset for the next launch (no one else touches it until then)
          }
          ptx::named_bar_sync(1, kDqThreads);   // acquire -> every reader thread
#pragma unroll 1
          for (int jc = j0; jc < jmax; jc += 8) {
            uint32_t v[8];
            load_d(jc, v);
            float acc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = __uint_as_float(v[i]);
            for (int c = c_first + 1; c <= c_last; ++c) {
              const float* pw = p.ws + (size_t)c * (BN * kTileRows) + (size_t)jc * kTileRows + r;
              float pv[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) pv[i] = (jc + i < jmax) ? __ldcg(pw + i * kTileRows) : 0.f;
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[i] += pv[i];
            }
            store_y8(jc, acc, jmax - jc);
          }
          ptx::tc_fence_before();
          ptx::mbar_arrive(bar_dempty + 8 * db);
        }
      }
      if (SK && whole) {
        ptx::tc_fence_before();
        ptx::mbar_arrive(bar_dempty + 8 * db);
      }
      ++si;
      if (TRACE && tr != nullptr && warp == C::DQ_BASE && lane == 0 && whole && !SK) tr[5] = clock64();
    }
  }

  if (!SK && S > 1) {
    // ---------------------------------------------------------------- cluster split-K reduce
    // fixed order p = 0..S-1 over the cluster's fp32 partials: deterministic (reading R12).
    // All S DSMEM loads of an element are issued before the first add (latency ~200 cycles).
    if (TRACE && tr != nullptr && threadIdx.x == 0) tr[5] = clock64();
    ptx::cluster_sync();
    if (TRACE && tr != nullptr && threadIdx.x == 0) tr[6] = clock64();
    const int grp = (int)blockIdx.z / p.n_cl;
    const int zc = (int)blockIdx.z - grp * p.n_cl;
    const int m0 = (grp * p.m_grp + (int)blockIdx.y) * BN;
    const uint32_t my = PAIR ? (crank >> 1) : ptx::cluster_ctarank();   // split index
    constexpr int E4 = BN * kTileRows / 4;   // the tile in float4 units, split evenly over S
    const int eb = (int)(((int)my * E4) / S) * 4;
    const int ee = (int)((((int)my + 1) * E4) / S) * 4;
    const int e_lim = min(ee, max(0, (M - m0)) * kTileRows);   // skip padded tokens
    uint32_t peer[kMaxSplit];
#pragma unroll
    for (int q = 0; q < kMaxSplit; ++q)   // (pair: the same member of each split's pair)
      peer[q] = ptx::mapa(sbase, PAIR ? (uint32_t)(2 * (q < S ? q : 0)) + member : (uint32_t)(q < S ? q : 0));
    const int tt = PAIR ? 2 * zc + (int)member : zc;
    // partial q of element e (float4 index): our own through ld.shared, the others' through DSMEM
    auto load_part = [&](int q, int e) {
      if (q == (int)my) {
        const uint4 u = ptx::lds128(sbase + (uint32_t)e * 4u);
        return make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z),
                           __uint_as_float(u.w));
      }
      return ptx::ld_dsmem_f32x4(peer[q] + (uint32_t)e * 4u);
    };
    auto store_sum = [&](int e, const float4& acc_in) {
      const int j = e / kTileRows;
      const int rr = e % kTileRows;
      const size_t o = (size_t)(m0 + j) * p.ldy + (size_t)tt * kTileRows + rr;
      float4 acc = acc_in;
      if (p.bias != nullptr) {   // output columns tt x 128 + rr .. rr + 3
        const uint2 b4 = *reinterpret_cast<const uint2*>(p.bias + (size_t)tt * kTileRows + rr);
        acc.x += bias_f<BF>((uint16_t)(b4.x & 0xFFFFu));
        acc.y += bias_f<BF>((uint16_t)(b4.x >> 16));
        acc.z += bias_f<BF>((uint16_t)(b4.y & 0xFFFFu));
        acc.w += bias_f<BF>((uint16_t)(b4.y >> 16));
      }
      if (out_fp32) {
#pragma unroll 1
        for (int d = 0; d < p.ndst; ++d)
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.Ydst[d]) + o) = acc;
      } else {
        uint2 pk;
        pk.x = cvt16x2<BF>(acc.x, acc.y);
        pk.y = cvt16x2<BF>(acc.z, acc.w);
#pragma unroll 1
        for (int d = 0; d < p.ndst; ++d)
          *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.Ydst[d]) + o) = pk;
      }
    };
    // The reduce is latency-bound (a DSMEM load takes ~500 cycles): for S <= 4 each thread keeps
    // UNR elements x S loads in flight before the first add.  Sum order q = 0..S-1 throughout.
    auto reduce_unrolled = [&](auto s_const) {
      constexpr int SS = decltype(s_const)::value;
      constexpr int UNR = SS <= 2 ? 4 : 2;
      constexpr int kStride = kThreads * 4;
      for (int e0 = eb + (int)threadIdx.x * 4; e0 < e_lim; e0 += kStride * UNR) {
        float4 v[UNR][SS];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          if (e0 + u * kStride < e_lim) {
#pragma unroll
            for (int q = 0; q < SS; ++q) v[u][q] = load_part(q, e0 + u * kStride);
          }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          if (e0 + u * kStride < e_lim) {
            float4 acc = v[u][0];
#pragma unroll
            for (int q = 1; q < SS; ++q) {
              acc.x += v[u][q].x;
              acc.y += v[u][q].y;
              acc.z += v[u][q].z;
              acc.w += v[u][q].w;
            }
            store_sum(e0 + u * kStride, acc);
          }
      }
    };
    if (silu) {
      // fused gate||up: whole tokens per CTA (token-aligned split) so that each gate float4 (rows
      // rr..rr+3, rr % 32 < 16) and its up float4 (rows rr+16..) are reduced by the same CTA; sum
      // order q = 0..S-1 as below
      const int tb = ((int)my * BN) / S;
      const int te = min((((int)my + 1) * BN) / S, max(0, M - m0));
      for (int i = (int)threadIdx.x; i < (te - tb) * 16; i += kThreads) {
        const int j = tb + (i >> 4);
        const int rr = ((i >> 2) & 3) * 32 + (i & 3) * 4;
        const int eg = j * kTileRows + rr;
        float4 g = load_part(0, eg), u = load_part(0, eg + 16);
        for (int qq = 1; qq < S; ++qq) {
          const float4 g2 = load_part(qq, eg), u2 = load_part(qq, eg + 16);
          g.x += g2.x; g.y += g2.y; g.z += g2.z; g.w += g2.w;
          u.x += u2.x; u.y += u2.y; u.z += u2.z; u.w += u2.w;
        }
        uint2 pk;
        pk.x = cvt16x2<BF>(silu_mul(g.x, u.x), silu_mul(g.y, u.y));
        pk.y = cvt16x2<BF>(silu_mul(g.z, u.z), silu_mul(g.w, u.w));
        const size_t o = (size_t)(m0 + j) * p.ldy + (size_t)tt * (kTileRows / 2) + (rr >> 5) * 16 + (rr & 15);
#pragma unroll 1
        for (int d = 0; d < p.ndst; ++d)
          *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.Ydst[d]) + o) = pk;
      }
    } else if (S == 2) {
      reduce_unrolled(std::integral_constant<int, 2>{});
    } else if (S == 3) {
      reduce_unrolled(std::integral_constant<int, 3>{});
    } else if (S == 4) {
      reduce_unrolled(std::integral_constant<int, 4>{});
    } else {
      for (int e = eb + (int)threadIdx.x * 4; e < e_lim; e += kThreads * 4) {
        float4 v[kMaxSplit];
#pragma unroll
        for (int q = 0; q < kMaxSplit; ++q)
          if (q < S) v[q] = load_part(q, e);
        float4 acc = v[0];
#pragma unroll
        for (int q = 1; q < kMaxSplit; ++q)
          if (q < S) {
            acc.x += v[q].x;
            acc.y += v[q].y;
            acc.z += v[q].z;
            acc.w += v[q].w;
          }
        store_sum(e, acc);
      }
    }
    if (TRACE && tr != nullptr && threadIdx.x == 0) tr[7] = clock64();
    // peers may still be reading our partials: arrive now (our own DSMEM reads are done), wait
    // only at the very end, so the barrier latency overlaps the teardown.  Relaxed: the barrier only
    // keeps our shared memory alive for the peers' reads (every value we loaded from theirs has been
    // consumed by the sums above); nothing written before it must become visible to them (4096^2:
    // M = 16 6.80 -> 6.54 us, M = 128 10.74 -> 10.23 us, profiles/r02c_relaxed_arrive_ab.txt).
    // (A push variant -- each CTA cp.async.bulk-copies the other owners' token chunks of its partial
    // into their shared memory, completing on an mbarrier, then sums locally -- was slower at every
    // cluster-split point, e.g. 4096^2 M = 128 11.69 vs 10.36 us: profiles/r02c_push_reduce_negative.txt)
    ptx::cluster_arrive_relaxed();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (TRACE && tr != nullptr && threadIdx.x == 0 && S == 1 && !SK) tr[6] = clock64();
  if (TRACE && threadIdx.x == 0) {
    // all CTAs: (smid, start ns, end ns, griddep release ns) after the 16 detailed records
    unsigned long long t_end_ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end_ns));
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const size_t lin = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    unsigned long long* rec = p.trace + 16 * (size_t)kTraceStride + 4 * lin;
    rec[0] = smid;
    rec[1] = t_start_ns;
    rec[2] = t_end_ns;
  }
  if (TRACE && tr != nullptr && threadIdx.x == 0) {
    tr[2] = clock64();
    int na_total = 0;
    SegIter it(p, SK, C::PAIR);
    Seg sg;
    while (it.next(sg)) na_total += sg.a_hi - sg.a_lo;
    tr[3] = (unsigned long long)na_total;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[4] = smid;
  }
  if constexpr (PAIR) {
    // both members' MMAs are complete (each waited its dfull); release the pair allocation
    // together
    if (S == 1) ptx::cluster_arrive();
    ptx::cluster_wait();
    if (warp == kMmaWarp) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc2(tmem, C::TMEM_COLS);
    }
  } else {
    if (warp == kMmaWarp) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
    if (!SK && S > 1) ptx::cluster_wait();   // (arrived after the split-K reduce)
  }
}

// ------------------------------------------------------------------------------------------
// Decode kernel (ablation, opt-in with kAblationMmaSync; M <= 16, stream-K plans): QUICK's
// register-fragment design, the paper's own (§3, Fig. 4-6), on the warp-level tensor
// path.  At M <= 16 the tcgen05 kernel spends a quarter of its time storing the dequantized A stage
// into TMEM (tcgen05.st; without those stores it runs at its loads-only time,
// profiles/r02b_small_m_tmem_store_probes.txt).  Here the dequantized registers ARE the
// mma.sync.m16n8k16 A fragment: no TMEM, no MMA warp, no afull/aempty round trip.  Same v1 blob, same
// stream-K units / workspace / fix-up as the tcgen05 kernel (a 128-row tile, 128-k stages).
// Measured on B200 (profiles/r02b_decode_mmasync_ab.txt): ~20 % slower than the tcgen05 kernel at
// 70B M <= 16 -- each thread now issues the HMMAs, its two rows' group constants and the X fragment
// loads itself (ncu: 25 vs 22 warp instructions per code word, issue slots 63 % busy either way),
// so the TMEM stores it saves are paid back in issue slots.  The automatic plan keeps tcgen05.
//
// Swap-AB: D[n][m] = sum_k W^T[n][k] X^T[k][m], A = 16 weight rows x 16 k (registers), B = 16 k x 8
// tokens (X from shared memory), D = 16 x 8 fp32 (registers).  Warp w owns rows 16w .. 16w + 15 of
// the tile; lane = 4g + t holds rows r0 = 16w + g and r1 = r0 + 8.  In the v1 layout word t of a
// row's 32-k chunk holds k = 32c + 8t + 0..7, and the FT extraction gives the pairs (k0,k1), (k2,k3),
// (k4,k5), (k6,k7) of that word; the MMA's k index is a free permutation (applied to A and B alike),
// so MMA step 0 of chunk c takes fragment columns {2t, 2t+1} = k {0, 1} and {2t+8, 2t+9} = k {2, 3},
// step 1 takes k {4, 5} and {6, 7} -- exactly the thread's own word: one LDS.32 per row and chunk is
// the A fragment after dequantization, and one LDS.128 of X[token g][32c + 8t .. + 7] (a 16-byte
// chunk of the same SW128 X tile the tcgen05 kernel uses: conflict-free) is the B fragment of both
// steps.  NT = 16 tokens adds the second 8-token half (row g + 8 of the X tile).
template <int NT>
struct DCfg {
  static constexpr int WARPS = 8;                    // compute warps (16 rows each)
  static constexpr int PRODUCER_WARP = WARPS;
  static constexpr int THREADS = 32 * (WARPS + 1);
  static constexpr int KL = 128;                     // k per stage (one stream-K unit)
  static constexpr int CTAS_PER_SM = 2;   // the 16-token stream-K plan's residency (3 per SM measured equal)
  static constexpr int STAGES = 8;
  static constexpr int XR = 16;                      // token rows of the X tile (the host's TMA box)
  static constexpr int X_BYTES = XR * KL * 2;        // [KL/64][16][64] fp16, SWIZZLE_128B
  static constexpr int X_SUB = XR * 128;
  static constexpr int W_BYTES = KL * 64;
  static constexpr int M_BYTES = kMetaBytes;         // one metadata block per stage (G a power of two >= 128)
  static constexpr int X_OFF = 0;
  static constexpr int W_OFF = X_OFF + STAGES * X_BYTES;
  static constexpr int M_OFF = W_OFF + STAGES * W_BYTES;
  static constexpr int BAR_OFF = (M_OFF + STAGES * M_BYTES + 7) & ~7;
  static constexpr int NUM_BARS = 3 * STAGES;        // full[STAGES], empty[STAGES], xfull[STAGES]
  static constexpr int USED = BAR_OFF + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = USED + 1024;
  static_assert((SMEM_BYTES + 1024) * CTAS_PER_SM <= 228 * 1024, "decode CTAs per SM");
  static_assert(NT == 8 || NT == 16, "8 or 16 tokens");
};

template <bool BF>
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  if constexpr (BF)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
                 "{%8, %9}, {%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
                 "{%8, %9}, {%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NT, bool BF>
__global__ void __launch_bounds__(DCfg<NT>::THREADS, DCfg<NT>::CTAS_PER_SM)
    quick_decode_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ KParams p) {
  using C = DCfg<NT>;
  constexpr int STAGES = C::STAGES;
  constexpr int NH = NT / 8;   // 8-token halves
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = ptx::smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int K = p.K, M = p.M;
  const int C32 = K / 32;
  const int NG = K / p.G;
  const int gsh = p.g_shift;   // G a power of two >= 128 (host-checked): one metadata block per stage
  const bool pdl = (p.flags & QUICK_FLAG_PDL) != 0;
  const uint32_t bar_full = sbase + C::BAR_OFF;
  const uint32_t bar_empty = bar_full + 8 * STAGES;
  const uint32_t bar_xfull = bar_empty + 8 * STAGES;
  if (warp == C::PRODUCER_WARP) {
    for (int i = lane; i < C::NUM_BARS; i += 32)
      ptx::mbar_init(bar_full + 8 * i, (i >= STAGES && i < 2 * STAGES) ? (uint32_t)C::WARPS : 1u);
    ptx::fence_mbar_init();
    if (lane == 0) ptx::prefetch_tmap(&tmap_x);
  }
  __syncthreads();
  if (p.flags & kDebugPdlEarly) ptx::griddep_launch_dependents();

  if (warp == C::PRODUCER_WARP) {
    // ------------------------------------------------------------------ producer (one lane issues)
    const uint64_t pol_w = ptx::policy_evict_first();
    const uint64_t pol_x = ptx::policy_evict_last();
    SegIter it(p, true);
    Seg sg;
    int slot = 0, lf = 0, pre = -1;
    uint32_t ph = 0;
    auto load_x = [&](int xs, int m0, int kc) {
      ptx::mbar_arrive_expect_tx(bar_xfull + 8 * xs, C::X_BYTES);
      ptx::tma_load_3d_hint(sbase + C::X_OFF + xs * C::X_BYTES, &tmap_x, 0, m0, kc, bar_xfull + 8 * xs, pol_x);
    };
    while (it.next(sg)) {
      const uint8_t* wbase = p.packed + (size_t)sg.t * C32 * kChunkBytes;
      const uint8_t* mbase = p.packed + (size_t)K * p.N / 2 + (size_t)sg.t * NG * kMetaBytes;
      const int m0 = sg.mt * 16;
      const int k_seg_end = min(sg.a_hi * kKA, K);
      const int nl = sg.a_hi - sg.a_lo;
      if (pre < 0) pre = pdl ? (nl < STAGES ? nl : STAGES) : 0;
      for (int l = 0; l < nl; ++l, ++lf) {
        const int kl0 = (sg.a_lo + l) * kKA;
        const int kv = min(kKA, k_seg_end - kl0);
        if (lf >= pre) ptx::mbar_wait_loop(bar_empty + 8 * slot, ph ^ 1u);
        const uint32_t full = bar_full + 8 * slot;
        if (ptx::elect_one()) {
          ptx::mbar_arrive_expect_tx(full, (uint32_t)kv * 64u + kMetaBytes);
          ptx::bulk_load_hint(sbase + C::W_OFF + slot * C::W_BYTES, wbase + (size_t)(kl0 / 32) * kChunkBytes,
                              (uint32_t)kv * 64u, full, pol_w);
          ptx::bulk_load_hint(sbase + C::M_OFF + slot * C::M_BYTES, mbase + (size_t)(kl0 >> gsh) * kMetaBytes,
                              kMetaBytes, full, pol_w);
          if (lf >= pre && !(pre == 0 && lf == 0)) {
            load_x(slot, m0, kl0 / 64);
          } else if (lf == (pre > 0 ? pre - 1 : 0)) {
            if (pdl) ptx::griddep_wait();
            for (int j = 0; j <= lf; ++j) load_x(j, m0, (sg.a_lo + j) * kKA / 64);
          }
        }
        __syncwarp();
        if (++slot == STAGES) {
          slot = 0;
          ph ^= 1u;
        }
      }
    }
    ptx::griddep_launch_dependents();
  } else {
    // ------------------------------------------------------------------ compute warps
    const int g = lane >> 2, t = lane & 3;
    const int r0 = 16 * warp + g, r1 = r0 + 8;
    const uint32_t woff0 = (uint32_t)(r0 * 16 + 4 * t), woff1 = (uint32_t)(r1 * 16 + 4 * t);
    const uint32_t soff0 = (uint32_t)(2 * r0), soff1 = (uint32_t)(2 * r1);
    const uint32_t zoff0 = (uint32_t)(256 + (r0 >> 1)), zoff1 = (uint32_t)(256 + (r1 >> 1));
    const uint32_t zs0 = (uint32_t)(r0 & 1) * 4u, zs1 = (uint32_t)(r1 & 1) * 4u;
    // X tile: [KL/64][16 rows][64 k], row = 128 B, 16-B chunk j of row g at (j ^ g): chunk c's 16 bytes
    // for this thread are j = (c & 1) * 4 + t of sub-tile c >> 1 (row g; row g + 8 for the second half)
    uint32_t xoff[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      xoff[c] = (uint32_t)((c >> 1) * C::X_SUB + g * 128 + ((((c & 1) * 4 + t) ^ g) << 4));
    auto consts = [&](uint32_t mb, uint32_t soff, uint32_t zoff, uint32_t zs) {
      const uint32_t zb = ptx::lds_u8(mb + zoff);
      const uint32_t sbits = ptx::lds_u16(mb + soff);
      const uint32_t zr = __byte_perm(zb, 0u, 0x4040);
      DequantConsts c;
      if constexpr (BF) {
        c.zlo = ptx::lop3<0xEA>(zr >> zs, 0x000F000Fu, 0x43004300u);
        c.zhi = 0u;
      } else {
        c.zlo = ptx::lop3<0xEA>(zr >> zs, 0x000F000Fu, 0x64006400u);
        c.zhi = ptx::lop3<0xEA>(zr << (4u - zs), 0x00F000F0u, 0xD400D400u);
      }
      c.s2 = __byte_perm(sbits, 0u, 0x1010);
      return c;
    };
    SegIter it(p, true);
    Seg sg;
    int slot = 0;
    uint32_t fph = 0;
    while (it.next(sg)) {
      const int k_seg_end = min(sg.a_hi * kKA, K);
      constexpr int NCH = 2;   // independent accumulation chains (chunk c -> chain c % NCH; 4 measured equal)
      float acc[NCH][NH][4];
#pragma unroll
      for (int i = 0; i < NCH; ++i)
#pragma unroll
        for (int h = 0; h < NH; ++h)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][h][j] = 0.0f;
      for (int a = sg.a_lo; a < sg.a_hi; ++a) {
        const uint32_t fbar = bar_full + 8u * (uint32_t)slot;
        const uint32_t wb = sbase + C::W_OFF + (uint32_t)slot * C::W_BYTES;
        const uint32_t mb = sbase + C::M_OFF + (uint32_t)slot * C::M_BYTES;
        const uint32_t xb = sbase + C::X_OFF + (uint32_t)slot * C::X_BYTES;
        ptx::mbar_wait_loop(fbar, fph);
        const DequantConsts c0 = consts(mb, soff0, zoff0, zs0);
        const DequantConsts c1 = consts(mb, soff1, zoff1, zs1);
        // K % 128 == 64 leaves a half last stage (chunks 0, 1); with G a power of two >= 128 (the only
        // groups this kernel takes) K is a multiple of 128, so this never fires -- kept for safety
        const bool half = (a * kKA + kKA) > k_seg_end;
        ptx::mbar_wait_loop(bar_xfull + 8u * (uint32_t)slot, fph);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= 2 && half) break;
          const uint32_t w0 = ptx::lds_u32(wb + (uint32_t)(c * kChunkBytes) + woff0);
          const uint32_t w1 = ptx::lds_u32(wb + (uint32_t)(c * kChunkBytes) + woff1);
          const uint4 x0 = ptx::lds128(xb + xoff[c]);
          uint32_t d0[4], d1[4];
          dequant_w<BF>(w0, c0, d0);
          dequant_w<BF>(w1, c1, d1);
          mma16816<BF>(acc[c % NCH][0], d0[0], d1[0], d0[1], d1[1], x0.x, x0.y);
          mma16816<BF>(acc[c % NCH][0], d0[2], d1[2], d0[3], d1[3], x0.z, x0.w);
          if constexpr (NH == 2) {
            const uint4 x1 = ptx::lds128(xb + xoff[c] + 8u * 128u);   // tokens 8 .. 15 (row g + 8)
            mma16816<BF>(acc[c % NCH][1], d0[0], d1[0], d0[1], d1[1], x1.x, x1.y);
            mma16816<BF>(acc[c % NCH][1], d0[2], d1[2], d0[3], d1[3], x1.z, x1.w);
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(fbar + 8u * STAGES);   // W, metadata and X of this slot consumed
        if (++slot == STAGES) {
          slot = 0;
          fph ^= 1u;
        }
      }
      if (!it.more()) ptx::griddep_launch_dependents();
      // ---------------------------------------------------------------- segment epilogue
      // thread (g, t) holds D[row r0 / r1][token 8h + 2t (+1)] = acc[.][h][0..3]
      float v[NH][4];
#pragma unroll
      for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float sum = acc[0][h][j];
#pragma unroll
          for (int i = 1; i < NCH; ++i) sum += acc[i][h][j];
          v[h][j] = sum;
        }
      const int n0 = sg.t * kTileRows + r0, n1 = n0 + 8;
      auto store = [&]() {
        float b0 = 0.0f, b1 = 0.0f;
        if (p.bias != nullptr) {
          b0 = bias_f<BF>(p.bias[n0]);
          b1 = bias_f<BF>(p.bias[n1]);
        }
#pragma unroll 1
        for (int d = 0; d < p.ndst; ++d) {
#pragma unroll
          for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int m = 8 * h + 2 * t + j;
              if (m < M) {
                if (p.flags & QUICK_FLAG_OUT_F32) {
                  float* y = reinterpret_cast<float*>(p.Ydst[d]) + (size_t)m * p.ldy;
                  y[n0] = v[h][j] + b0;
                  y[n1] = v[h][2 + j] + b1;
                } else {
                  uint16_t* y = reinterpret_cast<uint16_t*>(p.Ydst[d]) + (size_t)m * p.ldy;
                  y[n0] = cvt16<BF>(v[h][j] + b0);
                  y[n1] = cvt16<BF>(v[h][2 + j] + b1);
                }
              }
            }
        }
      };
      if (sg.a_lo == 0 && sg.a_hi == p.NA) {
        store();
      } else {
        // stream-K partial tile: the tile's first CTA (c_first, which reaches it at the end of its
        // range) sums the others' fp32 partials in CTA order; deterministic (as the tcgen05 kernel)
        const int u_first = sg.tile * p.NA;
        const int c_first = sk_owner(p, u_first);
        const int c_last = sk_owner(p, u_first + p.NA - 1);
        int* sem = p.sems + sg.tile;
        const int me = sk_cta(p.flags);
        if (me != c_first) {
          float* ws = p.ws + (size_t)me * (16 * kTileRows);
#pragma unroll
          for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int m = 8 * h + 2 * t + j;
              if (m < M) {
                __stcg(ws + m * kTileRows + r0, v[h][j]);
                __stcg(ws + m * kTileRows + r1, v[h][2 + j]);
              }
            }
          ptx::named_bar_sync(1, 32 * C::WARPS);
          if (threadIdx.x == 0) ptx::red_release_gpu_add(sem, 1);
        } else {
          if (threadIdx.x == 0) {
            const int want = c_last - c_first;
            while (ptx::ld_acquire_gpu(sem) < want) {
            }
            *sem = 0;
          }
          ptx::named_bar_sync(1, 32 * C::WARPS);
          for (int cc = c_first + 1; cc <= c_last; ++cc) {
            const float* ws = p.ws + (size_t)cc * (16 * kTileRows);
#pragma unroll
            for (int h = 0; h < NH; ++h)
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int m = 8 * h + 2 * t + j;
                if (m < M) {
                  v[h][j] += __ldcg(ws + m * kTileRows + r0);
                  v[h][2 + j] += __ldcg(ws + m * kTileRows + r1);
                }
              }
          }
          store();
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// Utility kernels on the same layout.
// ------------------------------------------------------------------------------------------
// One thread per 16-byte chunk (t, c, r): 32 codes of column n = 128t + r, k = 32c..32c+31.
template <bool BF>
__global__ void quick_dequant_kernel(const uint8_t* __restrict__ packed, uint16_t* __restrict__ W,
                                     int K, int N, int G) {
  const int C32 = K / 32;
  const long long total = (long long)(N / kTileRows) * C32 * kTileRows;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int r = (int)(idx % kTileRows);
  const int c = (int)((idx / kTileRows) % C32);
  const int t = (int)(idx / ((long long)kTileRows * C32));
  const uint4 wv = *reinterpret_cast<const uint4*>(packed + idx * 16);
  const int g = (32 * c) / G;
  const uint8_t* meta = packed + (size_t)K * N / 2 + ((size_t)t * (K / G) + g) * kMetaBytes;
  const uint32_t sbits = reinterpret_cast<const uint16_t*>(meta)[r];
  const uint32_t z = (meta[256 + (r >> 1)] >> ((r & 1) * 4)) & 0xFu;
  const DequantConsts dc = BF ? make_consts_bf16(sbits, z) : make_consts(sbits, z);
  uint32_t a[16];
  dequant_w<BF>(wv.x, dc, a + 0);
  dequant_w<BF>(wv.y, dc, a + 4);
  dequant_w<BF>(wv.z, dc, a + 8);
  dequant_w<BF>(wv.w, dc, a + 12);
  const int n = t * kTileRows + r;
  uint16_t* Wb = W;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const size_t k = (size_t)32 * c + 2 * i;
    Wb[k * N + n] = (uint16_t)(a[i] & 0xFFFFu);
    Wb[(k + 1) * N + n] = (uint16_t)(a[i] >> 16);
  }
}

__global__ void quick_f32_to_f16_kernel(const float* __restrict__ src, __half* __restrict__ dst,
                                        size_t n) {
  size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x * 4;
  for (; i + 3 < n; i += stride) {
    const float4 v = *reinterpret_cast<const float4*>(src + i);
    *reinterpret_cast<__half2*>(dst + i) = __floats2half2_rn(v.x, v.y);
    *reinterpret_cast<__half2*>(dst + i + 2) = __floats2half2_rn(v.z, v.w);
  }
  for (; i < n; ++i) dst[i] = __float2half_rn(src[i]);
}

// src [P][M][Nr] -> dst [M][P*Nr], 8 halves (16 B) per thread (Nr % 8 == 0)
__global__ void quick_gather_columns_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                            int P, int M, int Nr8) {
  const long long total = (long long)P * M * Nr8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % Nr8);
    const int m = (int)((i / Nr8) % M);
    const int p = (int)(i / ((long long)Nr8 * M));
    dst[((long long)m * P + p) * Nr8 + c] = src[i];
  }
}

}  // namespace quick

// ============================================================================================
// Host side: validation, launch plan, stream-K workspace, tensor map, launch.
// ============================================================================================
namespace {

thread_local int g_last_cuda_error = 0;
unsigned long long* g_trace = nullptr;   // debug tracing buffer (quick_debug_set_trace)

quick_status_t cuda_fail(cudaError_t e) {
  g_last_cuda_error = (int)e;
  return QUICK_ERR_CUDA;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

constexpr int kMaxDev = 64;
constexpr int kTiles[5] = {16, 32, 64, 128, 256};

int tile_index(int bn) {
  for (int i = 0; i < 5; ++i)
    if (kTiles[i] == bn) return i;
  return -1;
}

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 0;
  return dev;
}

int sm_count() {
  static int counts[kMaxDev] = {0};
  const int dev = current_device();
  if (counts[dev] == 0) {
    int c = 0;
    if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c <= 0)
      c = 148;
    counts[dev] = c;
  }
  return counts[dev];
}

quick_status_t check_gemm_shape(int M, int N, int K, int G) {
  if (M < 0 || N <= 0 || K <= 0 || G <= 0) return QUICK_ERR_INVALID_ARG;
  if (K % G != 0 || N % 8 != 0) return QUICK_ERR_INVALID_ARG;
  if (N % 128 != 0 || K % 64 != 0 || G % 32 != 0) return QUICK_ERR_UNSUPPORTED;
  return QUICK_OK;
}

// tile widths with a stream-K variant
inline bool sk_capable(int bn) { return bn <= 64; }

template <int BN, bool SK, bool TRACE>
void* kernel_ptr2(bool gbig) {
  return gbig ? reinterpret_cast<void*>(quick::quick_w4a16_tc_kernel<BN, SK, true, TRACE>)
              : reinterpret_cast<void*>(quick::quick_w4a16_tc_kernel<BN, SK, false, TRACE>);
}
template <bool TRACE>
void* kernel_for_t(int bn, bool sk, bool gbig) {
  switch (bn) {
    case 16: return sk ? kernel_ptr2<16, true, TRACE>(gbig) : kernel_ptr2<16, false, TRACE>(gbig);
    case 32: return sk ? kernel_ptr2<32, true, TRACE>(gbig) : kernel_ptr2<32, false, TRACE>(gbig);
    case 64: return sk ? kernel_ptr2<64, true, TRACE>(gbig) : kernel_ptr2<64, false, TRACE>(gbig);
    case 128: return kernel_ptr2<128, false, TRACE>(gbig);
    default: return kernel_ptr2<256, false, TRACE>(gbig);
  }
}
void* kernel_for(int bn, bool sk, bool gbig = true) { return kernel_for_t<false>(bn, sk, gbig); }
// the bf16 variant (QUICK_FLAG_BF16): no trace instantiation
template <int BN, bool SK>
void* bf16_ptr2(bool gbig) {
  return gbig ? reinterpret_cast<void*>(quick::quick_w4a16_tc_kernel<BN, SK, true, false, 0, true>)
              : reinterpret_cast<void*>(quick::quick_w4a16_tc_kernel<BN, SK, false, false, 0, true>);
}
void* bf16_kernel_for(int bn, bool sk, bool gbig) {
  switch (bn) {
    case 16: return sk ? bf16_ptr2<16, true>(gbig) : bf16_ptr2<16, false>(gbig);
    case 32: return sk ? bf16_ptr2<32, true>(gbig) : bf16_ptr2<32, false>(gbig);
    case 64: return sk ? bf16_ptr2<64, true>(gbig) : bf16_ptr2<64, false>(gbig);
    case 128: return bf16_ptr2<128, false>(gbig);
    default: return bf16_ptr2<256, false>(gbig);
  }
}
void* trace_kernel_for(int bn, bool sk, bool gbig = true) { return kernel_for_t<true>(bn, sk, gbig); }

#define QUICK_CFG_FIELD(FN, FIELD)                                                        \
  int FN(int bn, bool sk) {                                                               \
    switch (bn) {                                                                         \
      case 16: return sk ? quick::Cfg<16, true>::FIELD : quick::Cfg<16, false>::FIELD;   \
      case 32: return sk ? quick::Cfg<32, true>::FIELD : quick::Cfg<32, false>::FIELD;   \
      case 64: return sk ? quick::Cfg<64, true>::FIELD : quick::Cfg<64, false>::FIELD;   \
      case 128: return quick::Cfg<128, false>::FIELD;                                    \
      default: return quick::Cfg<256, false>::FIELD;                                     \
    }                                                                                     \
  }
QUICK_CFG_FIELD(tmem_cols_for, TMEM_COLS)
QUICK_CFG_FIELD(kl_for, KL)
QUICK_CFG_FIELD(smem_for, SMEM_BYTES)
QUICK_CFG_FIELD(threads_for, THREADS)
#undef QUICK_CFG_FIELD

// one-time per (device, tile, mode): opt into the dynamic shared memory the config needs
cudaError_t configure_kernel(int bn, bool sk) {
  static std::mutex mu;
  static bool done[kMaxDev][5][2] = {};
  const int dev = current_device(), ti = tile_index(bn);
  std::lock_guard<std::mutex> lock(mu);
  if (done[dev][ti][sk]) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  // every (group-size specialisation, trace) variant; the whole unified L1/shared array as
  // shared memory: two 80-110 KiB CTAs per SM
  for (int v = 0; v < 6 && e == cudaSuccess; ++v) {
    void* k = v >= 4 ? bf16_kernel_for(bn, sk, v & 1) : (v & 2) ? trace_kernel_for(bn, sk, v & 1) : kernel_for(bn, sk, v & 1);
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             std::max(smem_for(bn, sk), 120 * 1024));   // 120 KiB: kDebugOneCta
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
  }
  if (e == cudaSuccess) done[dev][ti][sk] = true;
  return e;
}

// How many clusters of S CTAs (or, for S == 1, CTAs) can be resident at once on this device.
// Cluster placement is GPC-constrained, so this is not simply SMs * CTAs-per-SM / S.
int max_resident(int bn, bool sk, int S) {
  static std::mutex mu;
  static int cache[kMaxDev][5][2][quick::kMaxSplit + 1] = {};
  const int dev = current_device(), ti = tile_index(bn);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (cache[dev][ti][sk][S]) return cache[dev][ti][sk][S];
  }
  int n = 0;
  if (configure_kernel(bn, sk) == cudaSuccess) {
    if (S == 1) {
      // per-SM limits computed directly: TMEM columns, shared memory (228 KiB per SM, 1 KiB
      // reserved per CTA), registers (64 K).  (cudaOccupancyMaxActiveBlocksPerMultiprocessor
      // reports 1 here although the hardware co-schedules 2 -- observed with %smid traces.)
      cudaFuncAttributes fa;
      int regs = 96;
      if (cudaFuncGetAttributes(&fa, kernel_for(bn, sk)) == cudaSuccess) regs = fa.numRegs;
      const int by_tmem = 512 / tmem_cols_for(bn, sk);
      const int by_smem = (228 * 1024) / (smem_for(bn, sk) + 1024);
      const int by_regs = 65536 / (((regs * 32 + 255) / 256) * 256 * (threads_for(bn, sk) / 32));
      n = std::max(1, std::min(by_tmem, std::min(by_smem, by_regs))) * sm_count();
    } else {
      cudaLaunchConfig_t cfg;
      std::memset(&cfg, 0, sizeof(cfg));
      cfg.gridDim = dim3((unsigned)S, 1, 1);
      cfg.blockDim = dim3((unsigned)threads_for(bn, sk), 1, 1);
      cfg.dynamicSmemBytes = smem_for(bn, sk);
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = (unsigned)S;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, kernel_for(bn, sk), &cfg) != cudaSuccess) n = 0;
      // like the per-CTA occupancy query, the cluster query assumes one CTA per SM for these
      // kernels although two co-reside (TMEM <= 256 columns, <= 113 KiB shared memory): take
      // the per-SM capacity computed above, less 10 % for GPC fragmentation of the clusters
      // (overestimating only costs a partial second wave: clusters never wait on each other)
      const int per_sm = max_resident(bn, sk, 1) / std::max(1, sm_count());
      if (per_sm >= 2) n = std::max(n, (per_sm * sm_count() * 9) / (10 * S));
    }
  }
  cudaGetLastError();  // occupancy queries must not leave a sticky error behind
  if (n <= 0) n = (S == 1 ? sm_count() : sm_count() / (2 * S));
  if (n <= 0) n = 1;
  std::lock_guard<std::mutex> lock(mu);
  cache[dev][ti][sk][S] = n;
  return n;
}

// CTA pairs (tiles 128 / 256, no stream-K): the kernel, and how many clusters of 2 S CTAs
// (S splits of a pair) can be resident at once
template <int BN>
void* pair_kernel(bool gbig) {
  return gbig ? reinterpret_cast<void*>(quick::quick_w4a16_tc_kernel<BN, false, true, false, 2>)
              : reinterpret_cast<void*>(quick::quick_w4a16_tc_kernel<BN, false, false, false, 2>);
}
int max_resident_pair(int bn, int S) {
  static std::mutex mu;
  static int cache[kMaxDev][2][quick::kMaxSplit + 1] = {};
  const int dev = current_device(), ti = bn == 256 ? 1 : 0;
  if (S < 1 || 2 * S > quick::kMaxSplit) return 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (cache[dev][ti][S]) return cache[dev][ti][S];
  }
  const int smem = bn == 256 ? quick::Cfg<256, false, 2>::SMEM_BYTES : quick::Cfg<128, false, 2>::SMEM_BYTES;
  const int threads = quick::Cfg<128, false, 2>::THREADS;
  const int per_sm_tmem = bn == 256 ? quick::Cfg<256, false, 2>::MAX_CTAS_PER_SM
                                    : quick::Cfg<128, false, 2>::MAX_CTAS_PER_SM;
  int n = 0;
  void* k = bn == 256 ? pair_kernel<256>(true) : pair_kernel<128>(true);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess) {
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)(2 * S), 1, 1);
    cfg.blockDim = dim3((unsigned)threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = (unsigned)(2 * S);
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) n = 0;
    // the query assumes one CTA per SM (see max_resident)
    const int per_sm = std::min(per_sm_tmem, (228 * 1024) / (smem + 1024));
    if (per_sm >= 2) n = std::max(n, (per_sm * sm_count() * 9) / (10 * 2 * S));
  }
  cudaGetLastError();
  if (n <= 0) n = std::max(1, sm_count() / (4 * S));
  std::lock_guard<std::mutex> lock(mu);
  cache[dev][ti][S] = n;
  return n;
}

// ---------------------------------------------------------------------------------------
// Stream-K workspace: CALLER-OWNED (quick_workspace_bytes / the workspace arguments of
// quick_w4a16_gemm_ex).  Layout: 65536 int32 arrival counters (256 KiB, zero between launches: the
// caller zeroes the buffer once, every launch leaves them zero), then the [P][BN][128] fp32 partial
// tiles (scratch).  The library never allocates, frees or synchronises.
constexpr size_t kSemAlign = 256;
// The counter region has a FIXED size (kMaxSkTiles counters, 256 KiB), so that calls of different
// shapes sharing one workspace never see another call's fp32 partials where their counters live
// (round 2 sized it by the call's own tile count: a call with fewer tiles wrote partials over the
// counters of a later call with more tiles).
constexpr long long kMaxSkTiles = 65536;
size_t sk_sem_bytes(long long /*tiles*/) { return (size_t)kMaxSkTiles * sizeof(int); }
size_t sk_ws_bytes(long long tiles, int P, int bn) {
  return sk_sem_bytes(tiles) + (size_t)P * bn * quick::kTileRows * sizeof(float);
}

struct Plan {
  int tile_n, split, ctas;
  bool sk;
  int P;   // stream-K CTAs
  bool pair = false;   // CTA pairs (cta_group::2), tiles 128 / 256 (split = splits per pair)
};

constexpr int kMaxAccumK = 8192;

// the smallest tile covering M (at most 128; M > 64 goes through the cost model below, which
// also considers 256-token tiles and CTA pairs)
int cover_tile(int M) { return M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128; }

// Launch plan (tuned with tools/tune_plan.py on B200):
//  - tokens per tile: the smallest MMA N covering M, at most 128 (weights are dequantized once
//    per m-tile; M > 128 tiles the tokens by 128);
//  - tiles <= 64 (the HBM-bound regime): stream-K over (tile, 128-k stage) units with one wave
//    of 2 CTAs per SM, each CTA a contiguous range of >= 4 units;
//  - M > 64 (tensor-bound): the fitted cost model over tile {128, 256}, split S and CTA pairs;
//  - otherwise split-K over a cluster: the largest S <= 6 such that all tiles x S CTAs are
//    resident in one wave (clusters are GPC-placed, so residency is queried) and every CTA
//    keeps >= 2 A stages;
//  - always S >= ceil(K / 8192) for accuracy (a TMEM accumulator sums at most 8192 of K,
//    DESIGN.md R15).
Plan choose_plan(int M, int N, int K, int G, int force_tile, int force_split, bool allow_sk,
                 bool allow_pair = true, bool force_sk = false) {
  (void)G;
  const int NA = (K + quick::kKA - 1) / quick::kKA;
  const int tn = force_tile > 0 ? force_tile : cover_tile(M);
  const int tiles = (N / quick::kTileRows) * ((M + tn - 1) / tn);
  if (allow_sk && force_split == 0 && sk_capable(tn) && (long long)tiles * NA < (1LL << 30) &&
      tiles <= kMaxSkTiles) {
    const long long U = (long long)tiles * NA;
    const long long resident = (long long)max_resident(tn, true, 1);
    long long P = std::min(resident, std::max(1LL, U / 4));
    // accuracy: a CTA's segment of one tile spans at most kMaxAccumK of K
    const long long p_min = (U * quick::kKA + kMaxAccumK - 1) / kMaxAccumK;
    if (P < p_min) P = std::min(resident, p_min);
    // stream-K pays when a CTA's range covers at least half a tile (each tile then has <= ~3
    // contributors and the fix-up is short); when K is cut finer, the DSMEM cluster split-K
    // reduce is cheaper than the workspace fix-up (measured on B200: 4096^2 and both 13B
    // shapes favour the cluster, 28672x8192 stream-K)
    // (a segment never spans more than one tile, so the accuracy cap only binds when NA > cap)
    // (tiles <= 32: up to ~5 contributors per tile still pay -- measured on B200 with the debug
    // flag kDebugForceSk: 13824x5120 M <= 16 13.2 vs 13.8 us, 8192x28672 M <= 32 31.1 vs 32.9;
    // 7-8 contributors lose: 5120x13824, 4096^2; tile 64 keeps the half-tile rule)
    const long long reach = tn <= 32 ? 5 : 2;
    if ((force_sk || reach * (U / P) >= NA) &&
        (NA <= kMaxAccumK / quick::kKA || (U + P - 1) / P <= kMaxAccumK / quick::kKA))
      return Plan{tn, 1, (int)P, true, (int)P};
  }
  const int s_min = (K + kMaxAccumK - 1) / kMaxAccumK;
  if (force_tile == 0 && force_split == 0 && M > 64) {
    // Tensor-bound regime: cost model over tile {128, 256} tokens x split S x CTA pairs
    // (cta_group::2), fitted on B200 to 280 forced-plan timings (tools/sweep.py modes
    // t<tile>s<S>[p], 5 shapes x M = 128..1024, PDL chains; rms error 10 %):
    //   time = waves x (A stages per CTA x st + fixed + [S > 1] 1.93 + 0.355 (cluster - 1)
    //          + [cluster == 8] 1.21)   (microseconds)
    // with waves = ceil(clusters / resident clusters) (queried: GPC placement).  Per-stage
    // costs: tile 128 0.486 us (pair 0.648 for twice the rows per cluster), tile 256 0.752
    // (pair 0.665): the pair halves each SM's X traffic, which bounds the large tiles.
    static const double st[2][2] = {{0.486, 0.648}, {0.752, 0.665}};
    static const double fixed[2][2] = {{3.226, 2.733}, {4.748, 4.455}};
    const int n_tiles = N / quick::kTileRows;
    double best = 1e300;
    Plan bp{128, std::max(1, s_min), 0, false, 0};
    for (int tc : {128, 256}) {
      if (tc == 256 && M <= 128) continue;
      const int mt = (M + tc - 1) / tc;
      for (int pr = 0; pr < 2; ++pr) {
        if (pr && (n_tiles % 2 != 0 || !allow_pair)) continue;
        for (int s2 = 1; s2 <= (pr ? quick::kMaxSplit / 2 : quick::kMaxSplit); ++s2) {
          if (s2 < s_min) continue;
          if (s2 > 1 && s2 > NA / 2) break;
          const long long units = (long long)(n_tiles / (pr ? 2 : 1)) * mt;
          const int res = pr ? max_resident_pair(tc, s2) : max_resident(tc, false, s2);
          const long long waves = (units + res - 1) / res;
          const int csz = s2 * (pr ? 2 : 1);
          // a tile-128 pair grid that fits one CTA per SM runs each CTA alone on its SM (the
          // fitted 0.648 us is for two co-resident pairs): 0.426 us per stage, measured at 4096^2
          // M = 192/256, S = 2 (12.5 us vs 13.2 for one CTA per n-tile)
          const bool alone = pr && tc == 128 && units * 2 * s2 <= sm_count();
          const double t = (double)waves * (((NA + s2 - 1) / s2) * (alone ? 0.426 : st[tc == 256][pr]) +
                                            fixed[tc == 256][pr] +
                                            (s2 > 1 ? 1.933 : 0.0) + 0.355 * (csz - 1) + (csz == 8 ? 1.209 : 0.0));
          if (t < best) {
            best = t;
            bp = Plan{tc, s2, n_tiles * mt * s2, false, 0, pr != 0};
          }
        }
      }
    }
    return bp;
  }
  int S = 1;
  if (force_split > 0) {
    S = force_split;
  } else {
    // the largest S <= 6 whose clusters are all resident in one wave, preferring an S that
    // divides the A stages evenly (the cluster waits for its slowest member: a 5-vs-6-stage
    // split costs a stage); measured on B200: 4096^2 S=4 (6.0 us) beats S=8 (6.6), 13824x5120
    // S=2 (13.1) beats S=1 (15.6), 5120x13824 S=6 (13.6) beats S=3 (16.0)
    const int cap = max_resident(tn, false, 1);   // CTAs/SM from TMEM, smem and registers
    int s_any = 1, s_div = 1;
    for (int s2 = 2; s2 <= 6 && s2 <= NA / 2; ++s2) {
      if (tiles * s2 > cap) break;
      if (tiles > max_resident(tn, false, s2)) continue;
      s_any = s2;
      if (NA % s2 == 0) s_div = s2;
    }
    S = (2 * s_div >= s_any) ? s_div : s_any;
    if (S < s_min) S = std::min(s_min, quick::kMaxSplit);
  }
  return Plan{tn, S, tiles * S, false, 0};
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel), not per launch
cudaError_t set_smem_once(const void* k, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<int, const void*>> done;
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == dev && d.second == k) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(dev, k);
  return e;
}

// The decode kernel (M <= 16 stream-K plans, quick_decode_kernel): same grid (P CTAs, two per
// SM), same workspace and units as the 16-token tcgen05 stream-K plan it replaces.
template <int NT, bool BF>
quick_status_t launch_decode_t(const CUtensorMap& tmap, quick::KParams& kp, int P, cudaStream_t stream) {
  using C = quick::DCfg<NT>;
  auto* k = quick::quick_decode_kernel<NT, BF>;
  cudaError_t e = set_smem_once(reinterpret_cast<const void*>(k), C::SMEM_BYTES);
  if (e != cudaSuccess) return cuda_fail(e);
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)P, 1, 1);
  cfg.blockDim = dim3((unsigned)C::THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (kp.flags & QUICK_FLAG_PDL) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  kp.trace = nullptr;
  e = cudaLaunchKernelEx(&cfg, k, tmap, kp);
  return e == cudaSuccess ? QUICK_OK : cuda_fail(e);
}
quick_status_t launch_decode(const CUtensorMap& tmap, quick::KParams& kp, int P, cudaStream_t stream) {
  const bool bf = (kp.flags & QUICK_FLAG_BF16) != 0;
  if (kp.M <= 8)
    return bf ? launch_decode_t<8, true>(tmap, kp, P, stream) : launch_decode_t<8, false>(tmap, kp, P, stream);
  return bf ? launch_decode_t<16, true>(tmap, kp, P, stream) : launch_decode_t<16, false>(tmap, kp, P, stream);
}

template <int BN, bool SK>
quick_status_t launch_bn(const CUtensorMap& tmap, quick::KParams& kp, int S, int P,
                         cudaStream_t stream, bool pair = false) {
  using C = quick::Cfg<BN, SK>;
  cudaError_t e = configure_kernel(BN, SK);
  if (e != cudaSuccess) return cuda_fail(e);
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  if (SK)
    cfg.gridDim = dim3((unsigned)P, 1, 1);
  else
    cfg.gridDim = dim3((unsigned)S, (unsigned)kp.m_grp,   // m-tiles of a group adjacent, groups outermost
                       (unsigned)(kp.n_tiles * (kp.m_tiles / kp.m_grp)));
  cfg.blockDim = dim3((unsigned)C::THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  if (kp.flags & quick::kDebugOneCta) cfg.dynamicSmemBytes = std::max<size_t>(C::SMEM_BYTES, 120 * 1024);
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (!SK && S > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = (unsigned)S;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (kp.flags & QUICK_FLAG_PDL) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  kp.trace = g_trace;
  // group-size specialisation: a power of two >= 128 (the group index is a shift and an A
  // stage never straddles groups); any other G takes the per-32-k general path
  const bool gbig = kp.G >= quick::kKA && (kp.G & (kp.G - 1)) == 0;
  const bool bf = (kp.flags & QUICK_FLAG_BF16) != 0;
  if constexpr (!SK && BN >= 128) {
    if (pair) {   // CTA pairs (cta_group::2): grid (2 S, n_tiles / 2, m_tiles), clusters of 2 S
      using CP = quick::Cfg<BN, false, 2>;
      auto* kq = bf ? (gbig ? quick::quick_w4a16_tc_kernel<BN, false, true, false, 2, true>
                            : quick::quick_w4a16_tc_kernel<BN, false, false, false, 2, true>)
               : g_trace != nullptr ? (gbig ? quick::quick_w4a16_tc_kernel<BN, false, true, true, 2>
                                            : quick::quick_w4a16_tc_kernel<BN, false, false, true, 2>)
                                    : (gbig ? quick::quick_w4a16_tc_kernel<BN, false, true, false, 2>
                                            : quick::quick_w4a16_tc_kernel<BN, false, false, false, 2>);
      e = set_smem_once(reinterpret_cast<const void*>(kq), CP::SMEM_BYTES);
      if (e != cudaSuccess) return cuda_fail(e);
      cfg.gridDim = dim3((unsigned)(2 * S), (unsigned)kp.m_grp, (unsigned)(kp.n_tiles / 2 * (kp.m_tiles / kp.m_grp)));
      cfg.dynamicSmemBytes = CP::SMEM_BYTES;
      cfg.blockDim = dim3((unsigned)CP::THREADS, 1, 1);
      na = 0;
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = (unsigned)(2 * S);
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
      if (kp.flags & QUICK_FLAG_PDL) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
      }
      cfg.numAttrs = na;
      e = cudaLaunchKernelEx(&cfg, kq, tmap, kp);
      if (e != cudaSuccess) return cuda_fail(e);
      return QUICK_OK;
    }
  }
  if constexpr (!SK && (BN == 16 || BN == 128)) {
    if (kp.flags & quick::kAblationSmemA) {   // the shared-memory-A ablation
      using CA = quick::Cfg<BN, false, 1>;
      auto* ka = gbig ? quick::quick_w4a16_tc_kernel<BN, false, true, false, 1>
                      : quick::quick_w4a16_tc_kernel<BN, false, false, false, 1>;
      e = set_smem_once(reinterpret_cast<const void*>(ka), CA::SMEM_BYTES);
      if (e != cudaSuccess) return cuda_fail(e);
      cfg.dynamicSmemBytes = CA::SMEM_BYTES;
      cfg.blockDim = dim3((unsigned)CA::THREADS, 1, 1);
      e = cudaLaunchKernelEx(&cfg, ka, tmap, kp);
      if (e != cudaSuccess) return cuda_fail(e);
      return QUICK_OK;
    }
  }
  if (bf)
    e = gbig ? cudaLaunchKernelEx(&cfg, quick::quick_w4a16_tc_kernel<BN, SK, true, false, 0, true>, tmap, kp)
             : cudaLaunchKernelEx(&cfg, quick::quick_w4a16_tc_kernel<BN, SK, false, false, 0, true>, tmap, kp);
  else if (g_trace != nullptr)
    e = gbig ? cudaLaunchKernelEx(&cfg, quick::quick_w4a16_tc_kernel<BN, SK, true, true>, tmap, kp)
             : cudaLaunchKernelEx(&cfg, quick::quick_w4a16_tc_kernel<BN, SK, false, true>, tmap, kp);
  else
    e = gbig ? cudaLaunchKernelEx(&cfg, quick::quick_w4a16_tc_kernel<BN, SK, true, false>, tmap, kp)
             : cudaLaunchKernelEx(&cfg, quick::quick_w4a16_tc_kernel<BN, SK, false, false>, tmap, kp);
  if (e != cudaSuccess) return cuda_fail(e);
  return QUICK_OK;
}

constexpr int kKnownFlags = QUICK_FLAG_OUT_F32 | QUICK_FLAG_PDL | QUICK_FLAG_NO_STREAMK | QUICK_FLAG_SILU_MUL |
                            QUICK_FLAG_BF16 |
                            quick::kDebugNoCompute |
                            quick::kDebugExitTop | quick::kDebugExitPrologue | quick::kDebugNoMma |
                            quick::kDebugOneCta | quick::kDebugNoSttm | quick::kDebugPdlEarly |
                            quick::kAblationSmemA | quick::kForcePair | quick::kDebugNoPair | quick::kDebugForceSk |
                            quick::kDebugSkReverse | quick::kAblationMmaSync;

// The launch plan of a call: a pure function of the shape, flags and overrides, and of whether
// a stream-K workspace may be used (`allow_ws`).
Plan plan_for(int M, int N, int K, int G, int flags, int tile_n, int split_k, bool allow_ws) {
  Plan plan = choose_plan(M, N, K, G, tile_n, split_k,
                          allow_ws && (flags & (QUICK_FLAG_NO_STREAMK | quick::kAblationSmemA)) == 0,
                          (flags & quick::kDebugNoPair) == 0, (flags & quick::kDebugForceSk) != 0);
  if ((flags & quick::kDebugOneCta) && plan.sk) plan.P = plan.ctas = std::min(plan.P, sm_count());
  if ((flags & quick::kForcePair) && !plan.sk && plan.tile_n >= 128 && (N / quick::kTileRows) % 2 == 0 &&
      2 * plan.split <= quick::kMaxSplit)
    plan.pair = true;
  return plan;
}

// TMA descriptor of X viewed as [K/64][M][64], box {64, rows, kc}.  Encoding costs host
// microseconds, so descriptors are cached per thread, keyed by everything they encode (the
// pointer, M, K and the box): a hit is always the same descriptor the encoder would produce.
bool x_tensor_map(const void* X, int M, int K, int rows, int kc, bool bf, CUtensorMap* out) {
  struct Entry {
    const void* x;
    int M, K, rows, kc;
    bool bf;
    CUtensorMap map;
  };
  constexpr int kEntries = 32;
  thread_local Entry cache[kEntries];
  thread_local int used = 0, next = 0;
  for (int i = 0; i < used; ++i) {
    const Entry& e = cache[i];
    if (e.x == X && e.M == M && e.K == K && e.rows == rows && e.kc == kc && e.bf == bf) {
      *out = e.map;
      return true;
    }
  }
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)M, (cuuint64_t)(K / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)rows, (cuuint32_t)kc};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(out, bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                    const_cast<void*>(X), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return false;
  Entry& e = cache[next];
  e = Entry{X, M, K, rows, kc, bf, *out};
  next = (next + 1) % kEntries;
  if (used < kEntries) ++used;
  return true;
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

}  // namespace

namespace quick {
void set_last_cuda_error(int e) { g_last_cuda_error = e; }
}  // namespace quick

extern "C" {

int quick_last_cuda_error(void) { return g_last_cuda_error; }

// Debug only (not part of quick.h): device buffer of 16 * (8 + 7 * 256) + 3 * CTAs uint64 stamps
// written by the next launches (detailed per-stage stamps for 16 CTAs, start/end for all CTAs);
// NULL disables.
void quick_debug_set_trace(void* device_buffer) {
  g_trace = static_cast<unsigned long long*>(device_buffer);
}

// Debug only: resident CTAs (S == 1) or clusters (S > 1) of the (tile, stream-K) kernel, and
// its dynamic shared memory bytes.
int quick_debug_resident(int bn, int sk, int S, int* smem_bytes, int* regs) {
  if (sk == 2) return (bn == 128 || bn == 256) ? max_resident_pair(bn, S) : -1;   // CTA pairs
  if (tile_index(bn) < 0 || S < 1 || S > quick::kMaxSplit || (sk && !sk_capable(bn))) return -1;
  if (smem_bytes) *smem_bytes = smem_for(bn, sk != 0);
  if (regs) {
    cudaFuncAttributes fa;
    *regs = cudaFuncGetAttributes(&fa, kernel_for(bn, sk != 0)) == cudaSuccess ? fa.numRegs : -1;
  }
  return max_resident(bn, sk != 0, S);
}

quick_status_t quick_gemm_plan(int M, int N, int K, int G, int flags, size_t workspace_bytes, int* tile_n,
                               int* split_k, int* num_ctas, int* cta_pair) {
  quick_status_t st = check_gemm_shape(M, N, K, G);
  if (st != QUICK_OK) return st;
  if ((flags & ~kKnownFlags) != 0) return QUICK_ERR_UNSUPPORTED;
  const int Mp = M > 0 ? M : 1;
  Plan p = plan_for(Mp, N, K, G, flags, 0, 0, true);
  if (p.sk) {
    const long long tiles = (long long)(N / quick::kTileRows) * ((Mp + p.tile_n - 1) / p.tile_n);
    if (workspace_bytes < sk_ws_bytes(tiles, p.P, p.tile_n)) p = plan_for(Mp, N, K, G, flags, 0, 0, false);
  }
  if (tile_n) *tile_n = p.tile_n;
  if (split_k) *split_k = p.sk ? 0 : p.split;   // 0 = stream-K
  if (num_ctas) *num_ctas = p.ctas;
  if (cta_pair) *cta_pair = p.pair ? 1 : 0;
  return QUICK_OK;
}

size_t quick_workspace_bytes(int M, int N, int K, int G, int flags, int tile_n, int split_k) {
  if (check_gemm_shape(M, N, K, G) != QUICK_OK || M == 0) return 0;
  if (tile_n != 0 && tile_index(tile_n) < 0) return 0;
  const Plan plan = plan_for(M, N, K, G, flags, tile_n, split_k, true);
  if (!plan.sk) return 0;
  const long long tiles = (long long)(N / quick::kTileRows) * ((M + plan.tile_n - 1) / plan.tile_n);
  return sk_ws_bytes(tiles, plan.P, plan.tile_n);
}

}  // extern "C"

namespace quick {
// The GEMM launch behind quick_w4a16_gemm_ex; `ydst` / `ndst`: every destination of the Y stores
// (quick_tp.cu's column-parallel GEMM passes one per rank, each a peer-mapped pointer to this
// rank's column slot of that rank's Y).
quick_status_t gemm_launch(const void* X, const void* packed, int M, int N, int K, int G, void* Y, int ldy,
                           int flags, int tile_n, int split_k, void* workspace, size_t workspace_bytes,
                           void* const* ydst, int ndst, void* stream, const void* bias) {
  quick_status_t st = check_gemm_shape(M, N, K, G);
  if (st != QUICK_OK) return st;
  if (M == 0) return QUICK_OK;
  if (!X || !packed || !Y) return QUICK_ERR_INVALID_ARG;
  // fused gate||up: Y has N / 2 columns (SiLU(gate) * up), fp16 only
  const bool silu = (flags & QUICK_FLAG_SILU_MUL) != 0;
  if (ldy < (silu ? N / 2 : N)) return QUICK_ERR_INVALID_ARG;
  if (ldy % 8 != 0 || (flags & ~kKnownFlags) != 0) return QUICK_ERR_UNSUPPORTED;
  if (silu && (flags & (QUICK_FLAG_OUT_F32 | quick::kAblationSmemA))) return QUICK_ERR_UNSUPPORTED;
  if (bias != nullptr && (silu || !aligned(bias, 8))) return QUICK_ERR_UNSUPPORTED;
  if ((flags & QUICK_FLAG_BF16) && (flags & quick::kAblationSmemA)) return QUICK_ERR_UNSUPPORTED;
  if (!aligned(X, 16) || !aligned(Y, 16) || !aligned(packed, 128)) return QUICK_ERR_UNSUPPORTED;
  if (workspace_bytes != 0 && (workspace == nullptr || !aligned(workspace, 256))) return QUICK_ERR_INVALID_ARG;
  if (tile_n != 0 && tile_index(tile_n) < 0) return QUICK_ERR_UNSUPPORTED;
  const int NA = (K + quick::kKA - 1) / quick::kKA;
  if (split_k < 0 || split_k > quick::kMaxSplit || split_k > NA) return QUICK_ERR_UNSUPPORTED;

  cudaStream_t strm = static_cast<cudaStream_t>(stream);
  // The plan is a pure function of the arguments: stream-K only when the caller's workspace
  // holds it (never a hidden allocation; the same plan eager and under graph capture).
  Plan plan = plan_for(M, N, K, G, flags, tile_n, split_k, true);
  quick::KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.n_tiles = N / quick::kTileRows;
  if (plan.sk) {
    const long long tiles = (long long)kp.n_tiles * ((M + plan.tile_n - 1) / plan.tile_n);
    if (workspace_bytes >= sk_ws_bytes(tiles, plan.P, plan.tile_n)) {
      kp.sems = static_cast<int*>(workspace);
      kp.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + sk_sem_bytes(tiles));
    } else {
      plan = plan_for(M, N, K, G, flags, tile_n, split_k, false);
    }
  }
  kp.m_tiles = (M + plan.tile_n - 1) / plan.tile_n;
  // m-tile groups (cluster grids): the largest divisor of m_tiles whose X rows (m_grp x tile_n x K fp16)
  // stay within 40 MB of L2 next to the streamed weights; a single group otherwise
  kp.m_grp = kp.m_tiles;
  if (!plan.sk) {
    const long long x_tile = (long long)plan.tile_n * K * 2;
    while (kp.m_grp > 1 && (long long)kp.m_grp * x_tile > (40LL << 20)) {
      int d = kp.m_grp - 1;
      while (d > 1 && kp.m_tiles % d != 0) --d;
      kp.m_grp = d;
    }
  }
  kp.n_cl = plan.pair ? kp.n_tiles / 2 : kp.n_tiles;
  const int tn = plan.tile_n, s = plan.split;

  // X viewed as [K/64][M][64] (dims innermost first: k within a 64-chunk, token, k-chunk): one
  // 3-D box {64, tile_n, KL/64} lands as KL/64 SWIZZLE_128B [tile_n][64] sub-tiles.
  CUtensorMap tmap;
  const int kl = kl_for(tn, plan.sk);
  if (!x_tensor_map(X, M, K, plan.pair ? tn / 2 : tn, kl / 64, (flags & QUICK_FLAG_BF16) != 0, &tmap))
    return cuda_fail(cudaErrorInvalidValue);

  kp.packed = static_cast<const uint8_t*>(packed);
  kp.Y = Y;
  kp.bias = static_cast<const uint16_t*>(bias);
  if (ndst < 1 || ndst > kMaxPeers) return QUICK_ERR_INVALID_ARG;
  kp.ndst = ndst;
  for (int d = 0; d < ndst; ++d) {
    if (ydst[d] == nullptr || !aligned(ydst[d], 16)) return QUICK_ERR_INVALID_ARG;
    kp.Ydst[d] = ydst[d];
  }
  kp.M = M;
  kp.N = N;
  kp.K = K;
  kp.G = G;
  kp.g_shift = -1;
  if ((G & (G - 1)) == 0) {
    kp.g_shift = 0;
    while ((1 << kp.g_shift) < G) ++kp.g_shift;
  }
  kp.ldy = ldy;
  // the 256-token tile launches without programmatic dependent launch (an
  // intermittent fault with deeper PDL prefetch whose root cause is not established)
#ifdef QUICK_PDL256
  kp.flags = flags;   // build variant for probing the tile-256 PDL fault (tools/gpu_t256.sh)
#else
  kp.flags = (tn == 256) ? (flags & ~QUICK_FLAG_PDL) : flags;
#endif
  // A stream-K grid holding every CTA slot of the machine triggers its dependents right after the
  // prologue: the next GEMM's CTAs can only land in slots our CTAs vacate, so an early trigger
  // lets each one start (prologue, weight prefetch, first dequantized stages) as soon as a slot
  // frees instead of after our slowest CTA reaches its epilogue (tools/sweep.py pdl vs pdlearly on
  // B200: 28672x8192 M = 1 31.1 -> 30.4 us).  Grids smaller than the machine keep the late trigger
  // (an early one lets the next grid double up on busy SMs).
  if (plan.sk && (kp.flags & QUICK_FLAG_PDL) && plan.P >= max_resident(tn, true, 1)) kp.flags |= quick::kDebugPdlEarly;
  // Cluster split-K plans of the 16/32-token tiles with at most one CTA per SM and short CTAs (<= 8 A
  // stages) trigger early too: the grid is mostly its ramp and split-K reduce, so the next GEMM's
  // prologue and weight prefetch gain from starting on the idle SMs and under the reduce (4096^2 M = 1
  // 6.42 -> 6.24 us, M = 32 7.56 -> 7.13).  With long CTAs the early CTAs' weight streams slow the
  // running grid (4096x14336, 28 stages per CTA: 12.2 -> 15.0 us); the 64-token tile loses as well
  // (4096^2 8.50 -> 9.16 us): profiles/r02c_pdl_early_cluster_ab.txt
#ifndef QUICK_NO_EARLY_CLUSTER
  if (!plan.sk && !plan.pair && tn <= 32 && plan.ctas <= sm_count() && (NA + plan.split - 1) / plan.split <= 8 &&
      (kp.flags & QUICK_FLAG_PDL))
    kp.flags |= quick::kDebugPdlEarly;
#endif
  kp.NA = NA;
  kp.U = kp.n_tiles * kp.m_tiles * NA;   // < 2^31: checked by choose_plan
  kp.P = plan.P;
  kp.sk_q = kp.U / max(kp.P, 1);
  kp.sk_r = kp.U - kp.sk_q * max(kp.P, 1);
#ifdef QUICK_SK_WEIGHT_PROBE
  if (plan.sk && plan.P == 2 * sm_count()) {   // probe: CTAs [0, P/2) take QUICK_SK_WEIGHT/1000 x the units
    static const int wgt = [] { const char* e = getenv("QUICK_SK_WEIGHT"); return e ? atoi(e) : 0; }();
    if (wgt > 0) {
      const int h = plan.P / 2;
      // group A: round(U * w / (w + 1000)) units over h CTAs, group B the rest over P - h
      const long long ua = ((long long)kp.U * wgt + (wgt + 1000) / 2) / (wgt + 1000);
      kp.sk_h = h;
      kp.sk_qa = (int)(ua / h);
      kp.sk_ra = (int)(ua - (long long)kp.sk_qa * h);
      kp.sk_qb = (int)((kp.U - ua) / (plan.P - h));
      kp.sk_rb = (int)((kp.U - ua) - (long long)kp.sk_qb * (plan.P - h));
      if (kp.sk_qa < 1 || kp.sk_qb < 1) kp.sk_h = 0;
    }
  }
#endif
  if (plan.sk) {
    // ablation (opt-in): the register-fragment mma.sync decode kernel for M <= 16, G a power of two
    // >= 128, plain outputs -- measured ~20 % slower than the tcgen05 kernel
    if ((flags & quick::kAblationMmaSync) && tn == 16 && M <= 16 && kp.g_shift >= 7 && !g_trace &&
        (flags & QUICK_FLAG_SILU_MUL) == 0)
      return launch_decode(tmap, kp, plan.P, strm);
    switch (tn) {
      case 16: return launch_bn<16, true>(tmap, kp, 1, plan.P, strm);
      case 32: return launch_bn<32, true>(tmap, kp, 1, plan.P, strm);
      default: return launch_bn<64, true>(tmap, kp, 1, plan.P, strm);
    }
  }
  switch (tn) {
    case 16: return launch_bn<16, false>(tmap, kp, s, 0, strm);
    case 32: return launch_bn<32, false>(tmap, kp, s, 0, strm);
    case 64: return launch_bn<64, false>(tmap, kp, s, 0, strm);
    case 128: return launch_bn<128, false>(tmap, kp, s, 0, strm, plan.pair);
    default: return launch_bn<256, false>(tmap, kp, s, 0, strm, plan.pair);
  }
}

}  // namespace quick

extern "C" {

quick_status_t quick_w4a16_gemm_ex(const void* X, const void* packed, int M, int N, int K, int G,
                                   void* Y, int ldy, int flags, int tile_n, int split_k,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  void* const dst[1] = {Y};
  return quick::gemm_launch(X, packed, M, N, K, G, Y, ldy, flags, tile_n, split_k, workspace, workspace_bytes,
                            dst, 1, stream, nullptr);
}

quick_status_t quick_w4a16_gemm_bias(const void* X, const void* packed, const void* bias, int M, int N, int K,
                                     int G, void* Y, int ldy, int flags, int tile_n, int split_k,
                                     void* workspace, size_t workspace_bytes, void* stream) {
  if (bias == nullptr) return QUICK_ERR_INVALID_ARG;
  void* const dst[1] = {Y};
  return quick::gemm_launch(X, packed, M, N, K, G, Y, ldy, flags, tile_n, split_k, workspace, workspace_bytes,
                            dst, 1, stream, bias);
}

quick_status_t quick_w4a16_gemm(const void* X, const void* packed, int M, int N, int K, int G,
                                void* Y, void* stream) {
  return quick_w4a16_gemm_ex(X, packed, M, N, K, G, Y, N, 0, 0, 0, nullptr, 0, stream);
}

quick_status_t quick_dequant_weights(const void* packed, int K, int N, int G, void* W,
                                     void* stream) {
  return quick_dequant_weights_ex(packed, K, N, G, W, 0, stream);
}

quick_status_t quick_dequant_weights_ex(const void* packed, int K, int N, int G, void* W, int flags,
                                        void* stream) {
  if ((flags & ~QUICK_FLAG_BF16) != 0) return QUICK_ERR_UNSUPPORTED;
  quick_status_t st = check_gemm_shape(0, N, K, G);
  if (st != QUICK_OK) return st;
  if (!packed || !W) return QUICK_ERR_INVALID_ARG;
  if (!aligned(packed, 16)) return QUICK_ERR_UNSUPPORTED;
  const long long total = (long long)(N / 128) * (K / 32) * 128;
  const int threads = 256;
  const unsigned blocks = (unsigned)((total + threads - 1) / threads);
  if (flags & QUICK_FLAG_BF16)
    quick::quick_dequant_kernel<true><<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(packed), static_cast<uint16_t*>(W), K, N, G);
  else
    quick::quick_dequant_kernel<false><<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(packed), static_cast<uint16_t*>(W), K, N, G);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QUICK_OK : cuda_fail(e);
}

quick_status_t quick_f32_to_f16(const void* src, void* dst, size_t n, void* stream) {
  if (n == 0) return QUICK_OK;
  if (!src || !dst) return QUICK_ERR_INVALID_ARG;
  if (!aligned(src, 16) || !aligned(dst, 8)) return QUICK_ERR_UNSUPPORTED;
  const int threads = 256;
  unsigned blocks = (unsigned)std::min<size_t>((n / 4 + threads - 1) / threads + 1, 148 * 16);
  quick::quick_f32_to_f16_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const float*>(src), static_cast<__half*>(dst), n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QUICK_OK : cuda_fail(e);
}

quick_status_t quick_gather_columns(const void* src, void* dst, int P, int M, int Nr,
                                    void* stream) {
  if (P <= 0 || M < 0 || Nr <= 0) return QUICK_ERR_INVALID_ARG;
  if (M == 0) return QUICK_OK;
  if (!src || !dst) return QUICK_ERR_INVALID_ARG;
  if (Nr % 8 != 0 || !aligned(src, 16) || !aligned(dst, 16)) return QUICK_ERR_UNSUPPORTED;
  const long long total = (long long)P * M * (Nr / 8);
  const int threads = 256;
  unsigned blocks = (unsigned)std::min<long long>((total + threads - 1) / threads, 148 * 16);
  quick::quick_gather_columns_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), P, M, Nr / 8);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QUICK_OK : cuda_fail(e);
}

}  // extern "C"
