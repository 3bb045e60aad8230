// Microbenchmark: can a register-fragment decode path (QUICK's original design: each thread
// dequantizes the 8 codes of its m16n8k16 A fragment and feeds mma.sync directly, no TMEM, no
// MMA warp, no barriers) sustain the per-SM weight rate HBM needs on B200 (~43 weights/clk/SM)?
// Each warp streams 16 x 64 weight blocks from shared memory (one LDS.128 per thread = 4
// fragments), dequantizes (LOP3 magic, exact (q-z), fp16 scale) and issues 1 (M <= 8) or 2
// (M <= 16) mma.sync.m16n8k16 f32 per 16 x 16 block.  Prints weights/clk/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mmasync_mb tools/mmasync_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t lop3ea(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// a fragment: reg0 = rows g (k pair 0), reg1 = row g+8, reg2 = row g (k+8), reg3 = row g+8 (k+8)
__device__ __forceinline__ void dq(uint32_t w, uint32_t zlo_g, uint32_t zlo_h, uint32_t zhi_g,
                                   uint32_t zhi_h, uint32_t s_g, uint32_t s_h, uint32_t (&a)[4]) {
  const uint32_t lo0 = lop3ea(w, 0x000F000Fu, 0x64006400u);
  const uint32_t hi0 = lop3ea(w, 0x00F000F0u, 0x64006400u);
  const uint32_t w8 = w >> 8;
  const uint32_t lo1 = lop3ea(w8, 0x000F000Fu, 0x64006400u);
  const uint32_t hi1 = lop3ea(w8, 0x00F000F0u, 0x64006400u);
  a[0] = hmul2(hsub2(lo0, zlo_g), s_g);
  a[1] = hmul2(hfma2(hi0, 0x2C002C00u, zhi_h), s_h);
  a[2] = hmul2(hsub2(lo1, zlo_g), s_g);
  a[3] = hmul2(hfma2(hi1, 0x2C002C00u, zhi_h), s_h);
  (void)zlo_h;
  (void)zhi_g;
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NT>   // token tiles of 8
__global__ void kern(int iters, unsigned long long* cyc, float* sink) {
  extern __shared__ __align__(16) uint4 wsm[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16 * 1024 / 16; i += blockDim.x)
    wsm[i] = make_uint4(0x12345678u * (i + 1), 0x9abcdef0u ^ i, 0x0f1e2d3cu + i, 0x4b5a6978u * i);
  __syncthreads();
  float c[NT][4] = {};
  const uint32_t zlo = 0x64086408u, zhi = 0xD480D480u, s = 0x20002000u;
  uint32_t bx[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    bx[t][0] = 0x3c003c00u + lane + t;
    bx[t][1] = 0x3c003c00u ^ lane;
  }
  const unsigned long long t0 = clock64();
  int idx = (warp * 32 + lane) & 1023;
  for (int it = 0; it < iters; ++it) {
    const uint4 w = wsm[idx];          // 4 fragments (16 x 64 weights per warp)
    idx = (idx + blockDim.x) & 1023;
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      uint32_t a[4];
      dq(ws[f], zlo, zlo, zhi, zhi, s, s, a);
#pragma unroll
      for (int t = 0; t < NT; ++t) mma16816(c[t], a, bx[t][0], bx[t][1]);
    }
  }
  const unsigned long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int t = 0; t < NT; ++t) acc += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (acc == 1234.5f) sink[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NT>
void run(int warps, int ctas_per_sm) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 4 * 8);
  cudaMalloc(&sink, 4);
  const int iters = 4096;
  cudaFuncSetAttribute(kern<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024);
  kern<NT><<<148 * ctas_per_sm, warps * 32, 16 * 1024>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  static unsigned long long h[148 * 4];
  cudaMemcpy(h, d, sizeof(unsigned long long) * 148 * ctas_per_sm, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int b = 0; b < 148 * ctas_per_sm; ++b) avg += (double)h[b] / (148 * ctas_per_sm);
  // weights per CTA: warps x iters x (16 rows x 64 k)
  const double w_per_sm = (double)warps * iters * 16 * 64 * ctas_per_sm;
  printf("tokens<=%2d warps/CTA %2d CTAs/SM %d : %.1f weights/clk/SM (%.0f cycles)\n", NT * 8, warps, ctas_per_sm,
         w_per_sm / avg, avg);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {8, 16, 32}) run<1>(w, 1);
  for (int w : {8, 16, 32}) run<2>(w, 1);
  run<1>(16, 2);
  run<2>(16, 2);
  return 0;
}
