// Device-side repack and GPTQ activation-order support, sm_100a.
//
//  quick_pack_weights_device: the v1 repack of quick_pack.cpp (§3, §3.2)
//    run on the GPU for 70B-scale checkpoints (117 MiB of codes per 8192 x 28672 matrix: the host
//    packer takes seconds, this takes a few hundred microseconds).  Bit-exact with the host packer.
//  quick_gather_k: X'[m][k'] = X[m][perm[k']] -- the activation side of a GPTQ act-order import
//    (quick_import_gptq sorts the weight rows by group; the product needs the same permutation of
//    X's columns: Y = X W = X[:, perm] W[perm, :]).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/quick.h"

namespace quick_repack {

// nibble slot i of a v1 word holds k offset kNibbleK[i]; AWQ column offset j lives in slot kAwqSlot[j]
__constant__ int kNibbleK[8] = {0, 2, 4, 6, 1, 3, 5, 7};
__constant__ int kAwqSlot[8] = {0, 4, 1, 5, 2, 6, 3, 7};

// One thread per 16-byte v1 chunk (t, c, r): the 32 codes of column n = 128 t + r, k = 32 c .. 32 c + 31.
// Threads r = 0..127 of a chunk row read the same 32 AWQ rows, 16 consecutive words each: coalesced.
__global__ void pack_weights_kernel(const uint32_t* __restrict__ qweight, uint4* __restrict__ out, int K, int N) {
  const int C = K / 32, WPR = N / 8;
  const long long total = (long long)(N / 128) * C * 128;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx % 128);
    const int c = (int)((idx / 128) % C);
    const int t = (int)(idx / (128LL * C));
    const int n = 128 * t + r;
    const int shift = 4 * kAwqSlot[n & 7];
    const uint32_t* col = qweight + (n >> 3);
    uint32_t w[4];
#pragma unroll
    for (int ww = 0; ww < 4; ++ww) {
      uint32_t word = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = 32 * c + 8 * ww + kNibbleK[i];
        word |= ((__ldg(col + (size_t)k * WPR) >> shift) & 0xFu) << (4 * i);
      }
      w[ww] = word;
    }
    out[idx] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// One block of 64 threads per metadata block (t, g): 128 scales copied, 64 zero bytes built.
__global__ void pack_meta_kernel(const uint16_t* __restrict__ scales, const uint32_t* __restrict__ zeros,
                                 uint8_t* __restrict__ meta_out, int K, int N, int G) {
  const int NG = K / G, WPR = N / 8;
  const int t = blockIdx.x / NG, g = blockIdx.x % NG;
  uint8_t* meta = meta_out + ((size_t)t * NG + g) * 320;
  const int b = threadIdx.x;   // 0..63: zero byte b (rows 2b, 2b+1) and scales 2b, 2b+1
  const int n0 = 128 * t + 2 * b;
  const uint16_t* srow = scales + (size_t)g * N;
  reinterpret_cast<uint16_t*>(meta)[2 * b] = srow[n0];
  reinterpret_cast<uint16_t*>(meta)[2 * b + 1] = srow[n0 + 1];
  const uint32_t* zrow = zeros + (size_t)g * WPR;
  const uint32_t z0 = (zrow[n0 >> 3] >> (4 * kAwqSlot[n0 & 7])) & 0xFu;
  const uint32_t z1 = (zrow[(n0 + 1) >> 3] >> (4 * kAwqSlot[(n0 + 1) & 7])) & 0xFu;
  meta[256 + b] = (uint8_t)(z0 | (z1 << 4));
}

// X'[m][k'] = X[m][perm[k']], 8 output halves per thread iteration where possible (perm is arbitrary)
__global__ void gather_k_kernel(const __half* __restrict__ X, const int32_t* __restrict__ perm,
                                __half* __restrict__ Xp, int M, int K) {
  const long long total = (long long)M * K;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(i / K), k = (int)(i % K);
    Xp[i] = X[(size_t)m * K + __ldg(perm + k)];
  }
}

}  // namespace quick_repack

namespace quick {
void set_last_cuda_error(int e);   // quick_gemm.cu: the quick_last_cuda_error() state
}

extern "C" {

quick_status_t quick_pack_weights_device(const uint32_t* qweight, const uint16_t* scales, const uint32_t* zeros,
                                         int G, int K, int N, void* packed_out, void* stream) {
  if (!qweight || !scales || !zeros || !packed_out) return QUICK_ERR_INVALID_ARG;
  if (K <= 0 || N <= 0 || G <= 0 || K % G != 0 || N % 8 != 0) return QUICK_ERR_INVALID_ARG;
  if (N % 128 != 0 || K % 64 != 0 || G % 32 != 0) return QUICK_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(packed_out) & 15) != 0) return QUICK_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long chunks = (long long)(N / 128) * (K / 32) * 128;
  const int threads = 256;
  const unsigned blocks = (unsigned)((chunks + threads - 1) / threads < 148 * 64 ? (chunks + threads - 1) / threads
                                                                                 : 148 * 64);
  quick_repack::pack_weights_kernel<<<blocks, threads, 0, s>>>(qweight, static_cast<uint4*>(packed_out), K, N);
  quick_repack::pack_meta_kernel<<<(unsigned)((N / 128) * (K / G)), 64, 0, s>>>(
      scales, zeros, static_cast<uint8_t*>(packed_out) + (size_t)K * N / 2, K, N, G);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    quick::set_last_cuda_error((int)e);
    return QUICK_ERR_CUDA;
  }
  return QUICK_OK;
}

quick_status_t quick_gather_k(const void* X, const int32_t* perm, int M, int K, void* Xp, void* stream) {
  if (M < 0 || K <= 0) return QUICK_ERR_INVALID_ARG;
  if (M == 0) return QUICK_OK;
  if (!X || !perm || !Xp) return QUICK_ERR_INVALID_ARG;
  const long long total = (long long)M * K;
  const int threads = 256;
  const unsigned blocks = (unsigned)((total + threads - 1) / threads < 148 * 32 ? (total + threads - 1) / threads
                                                                                : 148 * 32);
  quick_repack::gather_k_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __half*>(X), perm, static_cast<__half*>(Xp), M, K);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    quick::set_last_cuda_error((int)e);
    return QUICK_ERR_CUDA;
  }
  return QUICK_OK;
}

}  // extern "C"
