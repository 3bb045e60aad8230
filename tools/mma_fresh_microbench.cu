// Microbenchmark: steady-state cycles per tcgen05.mma.kind::f16 (M=128, A in TMEM, B in SMEM
// SW128) when every MMA reads FRESH operands, as in the QUICK kernel (A: the 8 K=16 column
// groups of a 64-column A slot rotating over 3 slots; B: 8 K=16 steps of an X tile rotating
// over 4 stages), versus re-reading the same few operands.  One CTA per SM, all SMs, one
// issuing thread, accumulators alternating over 2 TMEM buffers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_fresh_mb tools/mma_fresh_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2402_10076_b200/csrc/quick_ptx.cuh"

using namespace quick;

__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

template <int N>
__global__ void kern(int fresh_a, int fresh_b, int n_stages, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
  }
  constexpr int XSUB = N * 128;            // one [N][64] fp16 SW128 sub-tile
  constexpr int XSTAGE = 2 * XSUB;         // 128 k per stage
  for (int i = threadIdx.x; i < 4 * XSTAGE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&holder), 512);
  ptx::tc_fence_before();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t b0 = sw128_desc(ptx::smem_u32(sm));
    const unsigned long long t0 = clock64();
    int as = 0, xs = 0;
    for (int s = 0; s < n_stages; ++s) {
      if (ptx::elect_one()) {
        const uint32_t a_col = tmem + (fresh_a ? as * 64 : 0);
        const uint64_t bst = b0 + (uint64_t)(fresh_b ? ((xs * XSTAGE) >> 4) : 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_f16_ts_acc(tmem + 256 + (kk & 1) * N, a_col + (fresh_a ? kk * 8 : (kk & 3) * 8),
                              bst + (uint64_t)(fresh_b ? ((kk >> 2) * (XSUB >> 4) + (kk & 3) * 2) : (kk & 3) * 2),
                              idesc);
      }
      __syncwarp();
      if (++as == 3) as = 0;
      if (++xs == 4) xs = 0;
    }
    if (ptx::elect_one()) ptx::mma_commit(ptx::smem_u32(&bar));
    __syncwarp();
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

template <int N>
void run(unsigned long long* d) {
  const int n_stages = 512;
  cudaFuncSetAttribute(kern<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int mode = 0; mode < 4; ++mode) {
    const int fa = mode & 1, fb = mode >> 1;
    kern<N><<<148, 128, 160 * 1024>>>(fa, fb, n_stages, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return;
    }
    static unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int b = 0; b < 148; ++b) avg += (double)h[b] / 148;
    printf("N=%3d fresh A %d fresh B %d : %6.1f cycles per MMA (128x%dx16), %7.1f per 8-MMA A stage\n", N, fa, fb,
           avg / (n_stages * 8), N, avg / n_stages);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run<16>(d);
  run<32>(d);
  run<64>(d);
  run<128>(d);
  return 0;
}
