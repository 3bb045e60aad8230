// Microbenchmark: cycles per tcgen05.mma.kind::f16 (A in TMEM "TS", or A in SMEM "SS"; B in SMEM)
// as a function of the MMA N and of the number of independent accumulators the MMAs rotate
// over, issued the way the QUICK kernel issues them (warp-uniform loop, elect.sync lane).
// Also: latency of one MMA + tcgen05.commit until the mbarrier phase flips.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_mb tools/mma_microbench.cu
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

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(1)
      : "memory");
}

template <int N, int NACC, bool SS>
__global__ void mb_kernel(int n_iter, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&holder), 512);
  ptx::tc_fence_before();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bdesc = sw128_desc(ptx::smem_u32(sm + 16384));   // B: N rows x 128 B
    const uint64_t adesc = sw128_desc(ptx::smem_u32(sm));           // A (SS): 128 rows x 128 B
    uint32_t phase = 0;
    // latency of a single MMA + commit
    unsigned long long lat = 0;
    for (int rep = 0; rep < 4; ++rep) {
      const unsigned long long t0 = clock64();
      if (ptx::elect_one()) {
        if (SS) mma_ss(tmem + 128, adesc, bdesc, idesc);
        else ptx::mma_f16_ts(tmem + 128, tmem, bdesc, idesc, 1u);
        ptx::mma_commit(ptx::smem_u32(&bar));
      }
      __syncwarp();
      ptx::mbar_wait(ptx::smem_u32(&bar), phase);
      phase ^= 1u;
      lat = clock64() - t0;
    }
    // throughput: n_iter x NACC MMAs, rotating accumulators
    const unsigned long long t0 = clock64();
    for (int i = 0; i < n_iter; ++i) {
      if (ptx::elect_one()) {
#pragma unroll
        for (int a = 0; a < NACC; ++a) {
          if (SS) mma_ss(tmem + 128 + a * N, adesc, bdesc + (uint64_t)(a & 3) * 2, idesc);
          else ptx::mma_f16_ts(tmem + 128 + a * N, tmem + (a & 3) * 8, bdesc + (uint64_t)(a & 3) * 2, idesc, 1u);
        }
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::mma_commit(ptx::smem_u32(&bar));
    __syncwarp();
    const unsigned long long t1 = clock64();
    ptx::mbar_wait(ptx::smem_u32(&bar), phase);
    const unsigned long long t2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = t2 - t0;
      out[1] = t1 - t0;
      out[2] = lat;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

template <int N, int NACC, bool SS>
void run(unsigned long long* d) {
  constexpr int n_iter = 512 / NACC;
  cudaFuncSetAttribute(mb_kernel<N, NACC, SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  mb_kernel<N, NACC, SS><<<1, 128, 64 * 1024>>>(n_iter, d);
  unsigned long long c[3] = {0, 0, 0};
  cudaError_t e = cudaMemcpy(c, d, 24, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  printf("%s N=%3d acc=%d  cycles/mma=%6.1f  issue/mma=%5.1f  single mma+commit latency=%llu\n",
         SS ? "SS" : "TS", N, NACC, (double)c[0] / (n_iter * NACC), (double)c[1] / (n_iter * NACC), c[2]);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<16, 1, false>(d); run<16, 2, false>(d); run<16, 4, false>(d); run<16, 8, false>(d);
  run<32, 1, false>(d); run<32, 4, false>(d);
  run<64, 1, false>(d); run<64, 4, false>(d);
  run<128, 1, false>(d); run<128, 2, false>(d);
  run<256, 1, false>(d);
  run<16, 1, true>(d); run<16, 4, true>(d); run<64, 1, true>(d); run<128, 1, true>(d); run<256, 1, true>(d);
  return 0;
}
