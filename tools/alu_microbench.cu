// Microbenchmark: per-SM issue throughput of the instruction forms the dequant uses
// (fp16x2 sub / fma-with-immediates / mul, LOP3, SHF) and of their mixes, with enough warps
// and independent chains to saturate the pipes.  Prints warp-instructions per cycle per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/alu_mb tools/alu_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 4096;

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
__device__ __forceinline__ uint32_t shr8(uint32_t a) {
  uint32_t d;
  asm volatile("shr.b32 %0, %1, 8;" : "=r"(d) : "r"(a));
  return d;
}

// MODE: 0 hsub2 (reg), 1 hfma2 x*imm + reg, 2 hmul2 reg, 3 hfma2 reg*reg+reg, 4 lop3, 5 shr,
//       6 the dequant word mix (1 shr + 4 lop3 + 2 sub + 2 fma(imm) + 4 mul)
template <int MODE>
__global__ void kern(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t v[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) v[i] = seed * (threadIdx.x + 17 * i) | 0x3c003c00u;
  const uint32_t c1 = seed ^ 0x64086408u, c2 = seed ^ 0x3c003c00u;
  const uint32_t kInv16 = 0x2C002C00u;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      if (MODE == 0) v[i] = hsub2(v[i], c1);
      if (MODE == 1) v[i] = hfma2(v[i], kInv16, c1);
      if (MODE == 2) v[i] = hmul2(v[i], c2);
      if (MODE == 3) v[i] = hfma2(v[i], c2, c1);
      if (MODE == 4) v[i] = lop3(v[i], 0x000F000Fu, c1);
      if (MODE == 5) v[i] = shr8(v[i]) ^ i;
      if (MODE == 6) {
        const uint32_t w = v[i];
        const uint32_t lo0 = lop3(w, 0x000F000Fu, 0x64006400u);
        const uint32_t hi0 = lop3(w, 0x00F000F0u, 0x64006400u);
        const uint32_t w8 = shr8(w);
        const uint32_t lo1 = lop3(w8, 0x000F000Fu, 0x64006400u);
        const uint32_t hi1 = lop3(w8, 0x00F000F0u, 0x64006400u);
        const uint32_t a = hmul2(hsub2(lo0, c1), c2);
        const uint32_t b = hmul2(hfma2(hi0, kInv16, c1), c2);
        const uint32_t c = hmul2(hsub2(lo1, c1), c2);
        const uint32_t d = hmul2(hfma2(hi1, kInv16, c1), c2);
        v[i] = (a ^ b) + (c ^ d);   // 3 more ALU ops keep the chain alive (counted below)
      }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc ^= v[i];
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int inst_per_chain_iter, int threads, uint32_t* d, unsigned long long* c) {
  kern<MODE><<<148, threads>>>(0x1234567u, d, c);
  cudaDeviceSynchronize();
  kern<MODE><<<148, threads>>>(0x1234567u, d, c);
  unsigned long long h[148];
  cudaError_t e = cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = mx > h[i] ? mx : (double)h[i];
  const double warp_inst = (double)(threads / 32) * kIters * kChains * inst_per_chain_iter;
  printf("%-34s warps/SM %2d  warp-inst/clk/SM %.2f\n", name, threads / 32, warp_inst / mx);
}

int main() {
  uint32_t* d;
  unsigned long long* c;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 148 * 8);
  for (int t : {256, 512, 1024}) {
    run<0>("sub.rn.f16x2 (HADD2 reg)", 1, t, d, c);
    run<1>("fma.rn.f16x2 x*imm+reg", 1, t, d, c);
    run<2>("mul.rn.f16x2 (HMUL2 reg)", 1, t, d, c);
    run<3>("fma.rn.f16x2 reg*reg+reg", 1, t, d, c);
    run<4>("lop3", 1, t, d, c);
    run<5>("shr + xor", 2, t, d, c);
    run<6>("dequant word (13 + 3 glue)", 16, t, d, c);
  }
  return 0;
}
