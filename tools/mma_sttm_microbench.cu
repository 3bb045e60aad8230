// Microbenchmark: latency of an 8-MMA batch (tcgen05.mma kind::f16, M=128, N=16, A from TMEM)
// + commit + mbarrier wait, as the QUICK MMA warp issues it, alone and while the 8 other warps
// of the CTA (a) write TMEM with tcgen05.st.32x32b.x32 (the dequantizers' A-stage stores) or
// (b) run the fp16/ALU dequant mix.  One or two CTAs per SM, all SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mst_mb tools/mma_sttm_microbench.cu
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

// mode 0: MMA alone; 1: + STTM warps; 2: + ALU warps; 3: STTM alone (no MMA)
template <int N>
__global__ void kern(int mode, int batches, unsigned long long* out) {
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
    if (mode == 1 || mode == 3) {
      uint32_t v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0x3c003c00u + i;
      const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32);
      const unsigned long long t0 = clock64();
      int n = 0;
      while (stop == 0 && n < (mode == 3 ? 4096 : 1 << 30)) {
        ptx::tmem_st_32x32b_x32(taddr, v);
        ptx::tmem_wait_st();
        ++n;
      }
      const unsigned long long t1 = clock64();
      if ((threadIdx.x & 31) == 0 && warp == 0) {
        out[blockIdx.x * 4 + 2] = t1 - t0;
        out[blockIdx.x * 4 + 3] = n;
      }
    } else if (mode == 2) {
      uint32_t v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = (threadIdx.x * 7919u + i * 104729u) | 0x3c003c00u;
      while (stop == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint32_t w = v[i], d;
          asm volatile("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(w), "r"(0x2C002C00u), "r"(w));
          asm volatile("mul.rn.f16x2 %0, %1, %2;" : "=r"(w) : "r"(d), "r"(0x3c003c00u));
          v[i] = ptx::lop3<0xEA>(w, 0x000F000Fu, 0x64006400u) + (w >> 8);
        }
      }
      if (v[0] == 0x12345u) out[0] = v[1];
    }
  } else if (warp == 9 && mode != 3) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bdesc = sw128_desc(ptx::smem_u32(sm));
    uint32_t phase = 0;
    unsigned long long tot = 0;
    for (int b = 0; b < batches; ++b) {
      const unsigned long long t0 = clock64();
      if (ptx::elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          ptx::mma_f16_ts_acc(tmem + 128 + (k & 1) * N, tmem + 64 + k * 8, bdesc + (uint64_t)(k & 3) * 2, idesc);
        ptx::mma_commit(ptx::smem_u32(&bar));
      }
      __syncwarp();
      ptx::mbar_wait(ptx::smem_u32(&bar), phase);
      phase ^= 1u;
      tot += clock64() - t0;
    }
    if ((threadIdx.x & 31) == 0) {
      out[blockIdx.x * 4 + 0] = tot;
      out[blockIdx.x * 4 + 1] = batches;
    }
    stop = 1;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

template <int N>
void run(unsigned long long* d, int ctas_per_sm) {
  const int grid = 148 * ctas_per_sm;
  cudaFuncSetAttribute(kern<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(d, 0, 148 * 2 * 4 * 8);
    kern<N><<<grid, 320, 48 * 1024>>>(mode, 2000, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return;
    }
    static unsigned long long h[148 * 2 * 4];
    cudaMemcpy(h, d, sizeof(unsigned long long) * grid * 4, cudaMemcpyDeviceToHost);
    double mma = 0, st = 0, stn = 0;
    for (int b = 0; b < grid; ++b) {
      if (h[b * 4 + 1]) mma += (double)h[b * 4] / h[b * 4 + 1];
      if (h[b * 4 + 3]) {
        st += (double)h[b * 4 + 2];
        stn += (double)h[b * 4 + 3];
      }
    }
    const char* names[4] = {"MMA alone", "MMA + 8 STTM warps", "MMA + 8 ALU warps", "STTM alone"};
    printf("N=%3d ctas/SM %d %-20s : cycles per 8-MMA batch (issue+commit+wait) %7.1f ; STTM.x32 (4 KiB/warp) cycles each %6.1f\n",
           N, ctas_per_sm, names[mode], mode == 3 ? 0.0 : mma / grid, stn > 0 ? st / stn : 0.0);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 2 * 4 * 8);
  run<16>(d, 1);
  run<16>(d, 2);
  run<64>(d, 2);
  run<128>(d, 1);
  return 0;
}
