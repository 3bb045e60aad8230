// Microbenchmark: does a warp issuing tcgen05.mma (kind::f16, A in TMEM, N=16) slow the FP16/ALU
// dequant mix of the other warps, and on which SM sub-partition?  One CTA per SM, 8 mix warps
// (2 per SMSP) + optionally one MMA warp on SMSP `mma_smsp`.  Prints cycles per mix iteration
// per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mix_mb tools/mix_mma_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2402_10076_b200/csrc/quick_ptx.cuh"

using namespace quick;

constexpr int kIters = 2048;

__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm volatile("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm volatile("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// blockDim = 320: warps 0..7 mix, warp 8 or 9 (or none) MMA, the other idle
__global__ void kern(int mma_warp, int n_mma_per_iter, int sleep, unsigned long long* cyc, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
    stop = 0;
  }
  for (int i = threadIdx.x; i < 16 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 9) ptx::tmem_alloc(ptx::smem_u32(&holder), 256);
  ptx::tc_fence_before();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  if (warp < 8) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (threadIdx.x * 7919u + i * 104729u) | 0x3c003c00u;
    const uint32_t c1 = 0x64086408u, c2 = 0x3c003c00u, kInv16 = 0x2C002C00u;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t w = v[i];
        const uint32_t lo0 = lop3(w, 0x000F000Fu, 0x64006400u);
        const uint32_t hi0 = lop3(w, 0x00F000F0u, 0x64006400u);
        const uint32_t w8 = w >> 8;
        const uint32_t lo1 = lop3(w8, 0x000F000Fu, 0x64006400u);
        const uint32_t hi1 = lop3(w8, 0x00F000F0u, 0x64006400u);
        const uint32_t a = hmul2(hsub2(lo0, c1), c2);
        const uint32_t b = hmul2(hfma2(hi0, kInv16, c1), c2);
        const uint32_t c = hmul2(hsub2(lo1, c1), c2);
        const uint32_t d = hmul2(hfma2(hi1, kInv16, c1), c2);
        v[i] = (a ^ b) + (c ^ d);
      }
    }
    const unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= v[i];
    if (acc == 0x12345678u) out[0] = acc;
    if ((threadIdx.x & 31) == 0) {
      cyc[blockIdx.x * 8 + warp] = t1 - t0;
      atomicAdd((int*)&stop, 1);   // the MMA warp stops once all 8 mix warps are done
    }
  } else {
    uint32_t phase = 0;
    if (warp == mma_warp) {
      constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t bdesc = sw128_desc(ptx::smem_u32(sm));
      // issue MMAs until the mix warps are done (checked every batch)
      for (int batch = 0; batch < 1000000; ++batch) {
        if (ptx::elect_one()) {
          for (int k = 0; k < n_mma_per_iter; ++k)
            ptx::mma_f16_ts(tmem + 128 + (k & 1) * 16, tmem + (k & 3) * 8, bdesc + (uint64_t)(k & 3) * 2, idesc, 1u);
          ptx::mma_commit(ptx::smem_u32(&bar));
        }
        __syncwarp();
        if (sleep)
          ptx::mbar_wait_sleep(ptx::smem_u32(&bar), phase);
        else
          ptx::mbar_wait(ptx::smem_u32(&bar), phase);
        phase ^= 1u;
        if (stop >= 8) break;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

int main() {
  unsigned long long* c;
  uint32_t* d;
  cudaMalloc(&c, 148 * 8 * 8);
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int mw : {-1, 9}) {
    for (int n : {8, 32}) for (int sl : {0, 1}) {
      if (mw < 0 && (n == 32 || sl)) continue;
      kern<<<148, 320, 48 * 1024>>>(mw, n, sl, c, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h[148 * 8];
      cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
      double per[4] = {0, 0, 0, 0};
      for (int b = 0; b < 148; ++b)
        for (int w = 0; w < 8; ++w) per[w % 4] += (double)h[b * 8 + w] / (148 * 2);
      printf("sleep %d mma warp %2d (SMSP %d) mmas/batch %2d : cycles per 8-word iteration by SMSP: %.1f %.1f %.1f %.1f\n",
             sl, mw, mw < 0 ? -1 : mw % 4, mw < 0 ? 0 : n, per[0] / kIters, per[1] / kIters, per[2] / kIters,
             per[3] / kIters);
    }
  }
  return 0;
}
