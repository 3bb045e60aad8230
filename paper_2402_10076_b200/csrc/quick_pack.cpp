// Offline weight repack for the QUICK W4A16 path (host, C++17).
//
// PAPER.md §3: "reordering the quantized weight matrix offline" so each thread's
// direct load is already its MMA operand; §3.2 P:L97 (ldmatrix-aware interleave)
// (dequant-kernel-aware reorder, Fig. 5), P:L117 (both combined, Fig. 6).
//
// The B200 form (layout v1).  The MMA consumes the dequantized weights as the
// TMEM-resident A operand of tcgen05.mma (rows = output columns n, K-major), written by one
// thread per TMEM lane with tcgen05.st.32x32b.  So the "fragment order" is: one thread = one
// n row, 32 consecutive k per 16-byte chunk, chunks of 128 rows contiguous (a warp's LDS.128
// reads 512 contiguous bytes: conflict-free).  Within each 32-bit word the 8 k values are
// stored in nibble order {0,2,4,6,1,3,5,7} -- the inverse of the FasterTransformer LOP3
// extraction order {0,4,1,5,2,6,3,7} -- so the extraction yields fp16 pairs (k, k+1) in
// ascending k, i.e. the 32-bit TMEM columns of the A operand (Fig. 5's reorder, along K).
//
//   weights: chunk(t, c, r) at byte ((t*C + c)*128 + r)*16, t = n/128, r = n%128, c = k/32,
//            word w of the chunk covers k = 32c + 8w + {0..7}
//   meta(t, g) at byte K*N/2 + (t*NG + g)*320: scales[g][128t + 0..127] (fp16, 256 B),
//            then zeros[g][128t + 0..127] as nibbles (row r in byte r/2, low nibble if r even)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/quick.h"

namespace {

// nibble slot i of a v1 word holds k offset kNibbleK[i] (dequant-aware order, Fig. 5)
constexpr int kNibbleK[8] = {0, 2, 4, 6, 1, 3, 5, 7};
// AWQ word: column offset j (0..7) lives in nibble slot kAwqSlot[j]
constexpr int kAwqSlot[8] = {0, 4, 1, 5, 2, 6, 3, 7};

inline uint32_t awq_code(const uint32_t* words, int row, int n, int words_per_row) {
  return (words[(size_t)row * words_per_row + (n >> 3)] >> (4 * kAwqSlot[n & 7])) & 0xFu;
}

quick_status_t check_shape(int K, int N, int G) {
  if (K <= 0 || N <= 0 || G <= 0) return QUICK_ERR_INVALID_ARG;
  if (K % G != 0 || N % 8 != 0) return QUICK_ERR_INVALID_ARG;
  if (N % 128 != 0 || K % 64 != 0 || G % 32 != 0) return QUICK_ERR_UNSUPPORTED;
  return QUICK_OK;
}

template <class F>
void parallel_for(int n, F&& f) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  int nt = (int)std::min<unsigned>(hw, (unsigned)n);
  if (nt <= 1 || (size_t)n < 2) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  for (int w = 0; w < nt; ++w)
    th.emplace_back([&, w] {
      for (int i = w; i < n; i += nt) f(i);
    });
  for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

uint32_t quick_layout_version(void) { return 1u; }

size_t quick_packed_bytes(int K, int N, int group_size) {
  if (check_shape(K, N, group_size) != QUICK_OK) return 0;
  return (size_t)K * N / 2 + (size_t)(K / group_size) * N * 5 / 2;
}

quick_status_t quick_pack_weights(const uint32_t* qweight, const uint16_t* scales,
                                  const uint32_t* zeros, int G, int K, int N, void* packed_out) {
  if (!qweight || !scales || !zeros || !packed_out) return QUICK_ERR_INVALID_ARG;
  quick_status_t st = check_shape(K, N, G);
  if (st != QUICK_OK) return st;
  const int T = N / 128, C = K / 32, NG = K / G, WPR = N / 8;
  uint8_t* out = static_cast<uint8_t*>(packed_out);
  uint32_t* wout = reinterpret_cast<uint32_t*>(out);  // weights section, 4-byte words
  parallel_for(T, [&](int t) {
    for (int c = 0; c < C; ++c) {
      for (int r = 0; r < 128; ++r) {
        const int n = 128 * t + r;
        uint32_t* chunk = wout + (((size_t)t * C + c) * 128 + r) * 4;
        for (int w = 0; w < 4; ++w) {
          uint32_t word = 0;
          for (int i = 0; i < 8; ++i) {
            const int k = 32 * c + 8 * w + kNibbleK[i];
            word |= awq_code(qweight, k, n, WPR) << (4 * i);
          }
          chunk[w] = word;
        }
      }
    }
    for (int g = 0; g < NG; ++g) {
      uint8_t* meta = out + (size_t)K * N / 2 + ((size_t)t * NG + g) * 320;
      std::memcpy(meta, scales + (size_t)g * N + 128 * t, 256);
      for (int b = 0; b < 64; ++b) {
        const uint32_t z0 = awq_code(zeros, g, 128 * t + 2 * b, WPR);
        const uint32_t z1 = awq_code(zeros, g, 128 * t + 2 * b + 1, WPR);
        meta[256 + b] = (uint8_t)(z0 | (z1 << 4));
      }
    }
  });
  return QUICK_OK;
}

quick_status_t quick_pack_gate_up(const uint32_t* qw_g, const uint16_t* sc_g, const uint32_t* z_g,
                                  const uint32_t* qw_u, const uint16_t* sc_u, const uint32_t* z_u, int G,
                                  int K, int I, void* packed_out) {
  if (!qw_g || !sc_g || !z_g || !qw_u || !sc_u || !z_u || !packed_out) return QUICK_ERR_INVALID_ARG;
  if (I <= 0 || I % 8 != 0) return QUICK_ERR_INVALID_ARG;
  if (I % 64 != 0) return QUICK_ERR_UNSUPPORTED;
  const int N = 2 * I;
  quick_status_t st = check_shape(K, N, G);
  if (st != QUICK_OK) return st;
  // the interleaved AWQ tensors of W' (column map in quick.h), then the ordinary v1 repack
  const int NG = K / G, WPR = N / 8, WPR_I = I / 8;
  auto src_col = [](int n, bool* up) {   // W' column n -> (gate/up, source column)
    const int t = n / 128, q = (n % 128) / 32, l = n % 32;
    *up = l >= 16;
    return 64 * t + 16 * q + (l & 15);
  };
  std::vector<uint32_t> qw((size_t)K * WPR, 0u), zr((size_t)NG * WPR, 0u);
  std::vector<uint16_t> sc((size_t)NG * N);
  parallel_for(N / 8, [&](int j) {   // one AWQ word column of W' per task (no shared words)
    for (int o = 0; o < 8; ++o) {
      const int n = 8 * j + o;
      bool up;
      const int c = src_col(n, &up);
      const uint32_t* qsrc = up ? qw_u : qw_g;
      const uint32_t* zsrc = up ? z_u : z_g;
      const uint16_t* ssrc = up ? sc_u : sc_g;
      for (int k = 0; k < K; ++k) qw[(size_t)k * WPR + j] |= awq_code(qsrc, k, c, WPR_I) << (4 * kAwqSlot[o]);
      for (int g = 0; g < NG; ++g) {
        zr[(size_t)g * WPR + j] |= awq_code(zsrc, g, c, WPR_I) << (4 * kAwqSlot[o]);
        sc[(size_t)g * N + n] = ssrc[(size_t)g * I + c];
      }
    }
  });
  return quick_pack_weights(qw.data(), sc.data(), zr.data(), G, K, N, packed_out);
}

quick_status_t quick_import_gptq(const uint32_t* qweight, const uint32_t* qzeros, const uint16_t* scales,
                                 const int32_t* g_idx, int zero_plus_one, int G, int K, int N,
                                 uint32_t* qweight_awq, uint16_t* scales_out, uint32_t* zeros_awq, int32_t* perm) {
  if (!qweight || !qzeros || !scales || !qweight_awq || !scales_out || !zeros_awq || !perm)
    return QUICK_ERR_INVALID_ARG;
  if (K <= 0 || N <= 0 || G <= 0 || K % G != 0 || K % 8 != 0 || N % 8 != 0) return QUICK_ERR_INVALID_ARG;
  const int NG = K / G, WPR = N / 8;
  // row order of the imported matrix: rows sorted by group (stable), so every group is G
  // consecutive rows (GPTQ act-order permutes the rows of each group across K)
  std::vector<int> count(NG, 0);
  for (int k = 0; k < K; ++k) {
    const int g = g_idx ? g_idx[k] : k / G;
    if (g < 0 || g >= NG) return QUICK_ERR_INVALID_ARG;
    ++count[g];
  }
  for (int g = 0; g < NG; ++g)
    if (count[g] != G) return QUICK_ERR_UNSUPPORTED;   // not G rows per group: no v1 group structure
  std::vector<int> next(NG);
  for (int g = 0; g < NG; ++g) next[g] = g * G;
  for (int k = 0; k < K; ++k) perm[next[g_idx ? g_idx[k] : k / G]++] = k;
  // zeros: GPTQ packs (z - zero_plus_one) along N in natural nibble order; a decoded zero of 16
  // (v1 checkpoints storing 15) has no 4-bit representation
  std::memset(zeros_awq, 0, (size_t)NG * WPR * 4);
  for (int g = 0; g < NG; ++g)
    for (int n = 0; n < N; ++n) {
      const uint32_t z = ((qzeros[(size_t)g * WPR + (n >> 3)] >> (4 * (n & 7))) & 0xFu) + (zero_plus_one ? 1u : 0u);
      if (z > 15u) return QUICK_ERR_UNSUPPORTED;
      zeros_awq[(size_t)g * WPR + (n >> 3)] |= z << (4 * kAwqSlot[n & 7]);
    }
  std::memcpy(scales_out, scales, (size_t)NG * N * sizeof(uint16_t));
  // codes: GPTQ packs 8 rows per word (nibble i = row 8j + i); AWQ packs 8 columns per word
  parallel_for(K / 8, [&](int kb) {
    for (int kk = 0; kk < 8; ++kk) {
      const int k2 = 8 * kb + kk;   // row of the imported matrix
      const int k = perm[k2];       // source row
      uint32_t* dst = qweight_awq + (size_t)k2 * WPR;
      const uint32_t* src = qweight + (size_t)(k >> 3) * N;
      const int sh = 4 * (k & 7);
      for (int j = 0; j < WPR; ++j) {
        uint32_t word = 0;
        for (int o = 0; o < 8; ++o) word |= ((src[8 * j + o] >> sh) & 0xFu) << (4 * kAwqSlot[o]);
        dst[j] = word;
      }
    }
  });
  return QUICK_OK;
}

quick_status_t quick_unpack_weights(const void* packed, int G, int K, int N, uint32_t* qweight,
                                    uint16_t* scales, uint32_t* zeros) {
  if (!packed || !qweight || !scales || !zeros) return QUICK_ERR_INVALID_ARG;
  quick_status_t st = check_shape(K, N, G);
  if (st != QUICK_OK) return st;
  const int T = N / 128, C = K / 32, NG = K / G, WPR = N / 8;
  const uint8_t* in = static_cast<const uint8_t*>(packed);
  const uint32_t* win = reinterpret_cast<const uint32_t*>(in);
  std::memset(qweight, 0, (size_t)K * WPR * 4);
  std::memset(zeros, 0, (size_t)NG * WPR * 4);
  // each n-tile owns 16 whole AWQ words per row, so threads over t never share a word
  parallel_for(T, [&](int t) {
    for (int c = 0; c < C; ++c) {
      for (int r = 0; r < 128; ++r) {
        const int n = 128 * t + r;
        const uint32_t* chunk = win + (((size_t)t * C + c) * 128 + r) * 4;
        for (int w = 0; w < 4; ++w) {
          for (int i = 0; i < 8; ++i) {
            const int k = 32 * c + 8 * w + kNibbleK[i];
            const uint32_t code = (chunk[w] >> (4 * i)) & 0xFu;
            qweight[(size_t)k * WPR + (n >> 3)] |= code << (4 * kAwqSlot[n & 7]);
          }
        }
      }
    }
    for (int g = 0; g < NG; ++g) {
      const uint8_t* meta = in + (size_t)K * N / 2 + ((size_t)t * NG + g) * 320;
      std::memcpy(scales + (size_t)g * N + 128 * t, meta, 256);
      for (int r = 0; r < 128; ++r) {
        const int n = 128 * t + r;
        const uint32_t z = (meta[256 + r / 2] >> (4 * (r & 1))) & 0xFu;
        zeros[(size_t)g * WPR + (n >> 3)] |= z << (4 * kAwqSlot[n & 7]);
      }
    }
  });
  return QUICK_OK;
}

const char* quick_status_string(quick_status_t s) {
  switch (s) {
    case QUICK_OK: return "QUICK_OK";
    case QUICK_ERR_INVALID_ARG: return "QUICK_ERR_INVALID_ARG";
    case QUICK_ERR_UNSUPPORTED: return "QUICK_ERR_UNSUPPORTED";
    case QUICK_ERR_CUDA: return "QUICK_ERR_CUDA";
  }
  return "QUICK_ERR_UNKNOWN";
}

}  // extern "C"
