// Microbenchmark: throughput of tcgen05.st by shape on B200, 4 KiB per warp per store (32 registers
// per thread), W warps per CTA storing into their own lane quarter, 1 or 2 CTAs per SM, all SMs.
// Modes: store + wait::st per iteration, or 4 stores then one wait.  Question it answers: is the
// 32x32b shape (thread = TMEM lane, the QUICK dequant layout) slower per byte than 16x256b /
// 16x128b / 16x64b, i.e. would a different register-fragment layout of the A stage pay?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sttm_shape_mb tools/sttm_shape_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2402_10076_b200/csrc/quick_ptx.cuh"

using namespace quick;

#define REGS32(v) \
  "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), \
  "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), \
  "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), \
  "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
#define OPS32 "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, " \
              "%21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32}"

template <int SHAPE>
__device__ __forceinline__ void st(uint32_t taddr, const uint32_t (&v)[32]) {
  if constexpr (SHAPE == 0)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " OPS32 ";" ::"r"(taddr), REGS32(v) : "memory");
  else if constexpr (SHAPE == 1)
    asm volatile("tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], " OPS32 ";" ::"r"(taddr), REGS32(v) : "memory");
  else if constexpr (SHAPE == 2)
    asm volatile("tcgen05.st.sync.aligned.16x128b.x16.b32 [%0], " OPS32 ";" ::"r"(taddr), REGS32(v) : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.16x64b.x32.b32 [%0], " OPS32 ";" ::"r"(taddr), REGS32(v) : "memory");
}

template <int SHAPE, int BATCH>
__global__ void kern(int iters, unsigned long long* out) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&holder), 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  uint32_t v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = 0x3c003c00u + i + threadIdx.x;
  // lane quarter of this warp; 32 (or 16-lane: 2 x 16) rows; column offset by warp group
  const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(((warp >> 2) & 3) * 64);
  const unsigned long long t0 = clock64();
  for (int n = 0; n < iters; n += BATCH) {
#pragma unroll
    for (int b = 0; b < BATCH; ++b) st<SHAPE>(taddr + (uint32_t)((b & 1) * 32), v);
    ptx::tmem_wait_st();
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += 1u;
  }
  const unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) atomicMax(out, t1 - t0);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
  (void)nw;
}

template <int SHAPE, int BATCH>
void run(const char* name, int warps, int ctas_per_sm) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  const int iters = 2048;
  // pad shared memory so exactly ctas_per_sm CTAs fit on an SM
  const int smem = ctas_per_sm == 1 ? 150 * 1024 : 100 * 1024;
  cudaFuncSetAttribute(kern<SHAPE, BATCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<SHAPE, BATCH><<<148 * ctas_per_sm, 32 * warps, smem>>>(iters, d);
  cudaMemset(d, 0, 8);
  kern<SHAPE, BATCH><<<148 * ctas_per_sm, 32 * warps, smem>>>(iters, d);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double bytes_per_sm = (double)iters * warps * ctas_per_sm * 4096.0;
  printf("%-16s batch %d warps/CTA %2d CTAs/SM %d : %7.1f cycles per store per warp, %6.1f B/clk/SM  (%s)\n", name,
         BATCH, warps, ctas_per_sm, (double)cyc / iters, bytes_per_sm / (double)cyc,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int cps : {1, 2})
    for (int w : {4, 8}) {
      run<0, 1>("32x32b.x32", w, cps);
      run<1, 1>("16x256b.x8", w, cps);
      run<2, 1>("16x128b.x16", w, cps);
      run<3, 1>("16x64b.x32", w, cps);
      run<0, 2>("32x32b.x32", w, cps);
      run<1, 2>("16x256b.x8", w, cps);
    }
  return 0;
}
