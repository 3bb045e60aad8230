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
