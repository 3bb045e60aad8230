// Collective-fused tensor-parallel epilogues over peer memory (BASELINE.json
// north_star (4)), sm_100a.  One process per GPU; every rank maps the other ranks' buffers
// (CUDA IPC: quick_peer_export / quick_peer_import, the handles exchanged by the caller's process
// group), so a kernel reads and writes peer memory directly over NVLink / NVSwitch.
//
//  column-parallel  quick_tp_column_gemm: the GEMM of this rank's N/P columns stores each Y element
//                   into this rank's column slot of EVERY rank's Y (the all-gather and the column
//                   permutation fused into the GEMM epilogue: no separate collective, no gather
//                   kernel), then a barrier so every rank's Y is complete when the stream proceeds.
//  row-parallel     quick_tp_row_gemm: the GEMM writes this rank's un-rounded fp32 partial into its
//                   own peer-visible buffer; barrier; each rank sums its 1/P slice of the columns
//                   over all P partials in rank order (deterministic, fp32) and stores the fp16
//                   result into every rank's Y (reduce-scatter + all-gather in one kernel);
//                   barrier.  fp32 on the wire (fp16 partials fail the tolerance).
//
// Barriers are flag arrays in peer memory, world + 1 uint32 per rank: slot p receives rank p's
// epochs, slot `world` is this rank's own barrier counter.  A barrier increments the counter on the
// device (so captured CUDA graphs replay correctly: nothing host-side is baked in), writes the new
// epoch e into slot r of every rank's array (release, system scope) and waits until its own slots
// all hold >= e (acquire).  Every rank runs the same sequence of barriers, so the counters move in
// lockstep.  A wait that exceeds kBarrierTimeoutNs traps (a loud launch failure, not a hung GPU).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/quick.h"

namespace quick {
quick_status_t gemm_launch(const void* X, const void* packed, int M, int N, int K, int G, void* Y, int ldy,
                           int flags, int tile_n, int split_k, void* workspace, size_t workspace_bytes,
                           void* const* ydst, int ndst, void* stream, const void* bias);
void set_last_cuda_error(int e);
}  // namespace quick

namespace quick_tp {

constexpr int kMaxRanks = 8;
constexpr unsigned long long kBarrierTimeoutNs = 20ull * 1000 * 1000 * 1000;

struct Ptrs {
  void* p[kMaxRanks];
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// one warp: lane 0 advances this rank's barrier counter; lane p < world signals rank p, then waits
// for rank p's signal
__global__ void barrier_kernel(Ptrs flags, int world, int rank) {
  const int p = threadIdx.x;
  asm volatile("fence.acq_rel.sys;" ::: "memory");   // this stream's prior writes (peer Y / partials)
  uint32_t* counter = static_cast<uint32_t*>(flags.p[rank]) + world;
  uint32_t epoch = 0;
  if (p == 0) epoch = *counter + 1u, *counter = epoch;
  epoch = __shfl_sync(0xffffffffu, epoch, 0);
  if (p < world) {
    uint32_t* slot = static_cast<uint32_t*>(flags.p[p]) + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch) : "memory");
    const uint32_t* mine = static_cast<const uint32_t*>(flags.p[rank]) + p;
    const unsigned long long t0 = globaltimer();
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      if (globaltimer() - t0 > kBarrierTimeoutNs) __trap();
      __nanosleep(256);
    }
  }
  __syncwarp();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// this rank's column slice [c0, c1) of every row: Y = fp16(sum_p part_p) in rank order, stored to
// every rank's Y; 8 columns (2 x float4 loads per rank, one 16-byte store per rank) per thread step
__global__ void row_reduce_kernel(Ptrs parts, Ptrs ys, int world, int M, int N, int ldy, int c0, int c1) {
  const int w8 = (c1 - c0) / 8;
  const long long total = (long long)M * w8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(i / w8);
    const int n = c0 + 8 * (int)(i % w8);
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int p = 0; p < world; ++p) {   // fixed order: bit-identical on every rank, run to run
      const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(parts.p[p]) + (size_t)m * N + n);
      const float4 a = __ldcv(src), b = __ldcv(src + 1);
      if (p == 0) {
        acc[0] = a.x; acc[1] = a.y; acc[2] = a.z; acc[3] = a.w;
        acc[4] = b.x; acc[5] = b.y; acc[6] = b.z; acc[7] = b.w;
      } else {
        acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
        acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
      }
    }
    uint4 out;
    __half2 h;
    h = __floats2half2_rn(acc[0], acc[1]); out.x = *reinterpret_cast<uint32_t*>(&h);
    h = __floats2half2_rn(acc[2], acc[3]); out.y = *reinterpret_cast<uint32_t*>(&h);
    h = __floats2half2_rn(acc[4], acc[5]); out.z = *reinterpret_cast<uint32_t*>(&h);
    h = __floats2half2_rn(acc[6], acc[7]); out.w = *reinterpret_cast<uint32_t*>(&h);
    for (int q = 0; q < world; ++q)
      *reinterpret_cast<uint4*>(static_cast<__half*>(ys.p[q]) + (size_t)m * ldy + n) = out;
  }
}

quick_status_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return QUICK_OK;
  quick::set_last_cuda_error((int)e);
  return QUICK_ERR_CUDA;
}

quick_status_t barrier(void* const* flag_peers, int world, int rank, cudaStream_t s) {
  Ptrs f;
  std::memset(&f, 0, sizeof(f));
  for (int p = 0; p < world; ++p) {
    if (!flag_peers[p]) return QUICK_ERR_INVALID_ARG;
    f.p[p] = flag_peers[p];
  }
  barrier_kernel<<<1, 32, 0, s>>>(f, world, rank);
  return cuda_status(cudaGetLastError());
}

bool valid_group(int world, int rank) { return world >= 1 && world <= kMaxRanks && rank >= 0 && rank < world; }

}  // namespace quick_tp

extern "C" {

quick_status_t quick_peer_alloc(size_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return QUICK_ERR_INVALID_ARG;
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, bytes);
  return quick_tp::cuda_status(e);
}

quick_status_t quick_peer_free(void* ptr) { return quick_tp::cuda_status(cudaFree(ptr)); }

quick_status_t quick_peer_export(const void* ptr, void* handle_out) {
  if (!ptr || !handle_out) return QUICK_ERR_INVALID_ARG;
  static_assert(sizeof(cudaIpcMemHandle_t) == QUICK_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(ptr));
  if (e == cudaSuccess) std::memcpy(handle_out, &h, sizeof(h));
  return quick_tp::cuda_status(e);
}

quick_status_t quick_peer_import(const void* handle, void** ptr) {
  if (!handle || !ptr) return QUICK_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return quick_tp::cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
}

quick_status_t quick_peer_close(void* ptr) { return quick_tp::cuda_status(cudaIpcCloseMemHandle(ptr)); }

quick_status_t quick_tp_barrier(void* const* flag_peers, int world, int rank, void* stream) {
  if (!flag_peers || !quick_tp::valid_group(world, rank)) return QUICK_ERR_INVALID_ARG;
  return quick_tp::barrier(flag_peers, world, rank, static_cast<cudaStream_t>(stream));
}

quick_status_t quick_tp_column_gemm(const void* X, const void* packed, int M, int N_local, int K, int G,
                                    void* const* y_peers, int ldy, void* const* flag_peers, int world, int rank,
                                    int flags, void* workspace, size_t workspace_bytes, void* stream) {
  if (!y_peers || !flag_peers || !quick_tp::valid_group(world, rank)) return QUICK_ERR_INVALID_ARG;
  if (ldy < world * N_local) return QUICK_ERR_INVALID_ARG;
  if (flags & (QUICK_FLAG_OUT_F32 | QUICK_FLAG_SILU_MUL)) return QUICK_ERR_UNSUPPORTED;
  if (M == 0) return QUICK_OK;
  void* dst[quick_tp::kMaxRanks];
  for (int p = 0; p < world; ++p) {
    if (!y_peers[p]) return QUICK_ERR_INVALID_ARG;
    dst[p] = static_cast<__half*>(y_peers[p]) + (size_t)rank * N_local;   // this rank's column slot
  }
  quick_status_t st = quick::gemm_launch(X, packed, M, N_local, K, G, dst[rank], ldy, flags, 0, 0, workspace,
                                         workspace_bytes, dst, world, stream, nullptr);
  if (st != QUICK_OK) return st;
  return quick_tp::barrier(flag_peers, world, rank, static_cast<cudaStream_t>(stream));
}

quick_status_t quick_tp_row_gemm(const void* X_local, const void* packed, int M, int N, int K_local, int G,
                                 void* const* part_peers, void* const* y_peers, int ldy, void* const* flag_peers,
                                 int world, int rank, int flags, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  if (!part_peers || !y_peers || !flag_peers || !quick_tp::valid_group(world, rank)) return QUICK_ERR_INVALID_ARG;
  if (ldy < N || ldy % 8 != 0 || N % (8 * world) != 0) return QUICK_ERR_UNSUPPORTED;
  if (flags & (QUICK_FLAG_OUT_F32 | QUICK_FLAG_SILU_MUL)) return QUICK_ERR_UNSUPPORTED;
  if (M == 0) return QUICK_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  quick_status_t st = quick::gemm_launch(X_local, packed, M, N, K_local, G, part_peers[rank], N,
                                         flags | QUICK_FLAG_OUT_F32, 0, 0, workspace, workspace_bytes,
                                         &part_peers[rank], 1, stream, nullptr);
  if (st != QUICK_OK) return st;
  // 2 barriers per call: partials ready, then results delivered (partials reusable)
  st = quick_tp::barrier(flag_peers, world, rank, s);
  if (st != QUICK_OK) return st;
  quick_tp::Ptrs parts, ys;
  std::memset(&parts, 0, sizeof(parts));
  std::memset(&ys, 0, sizeof(ys));
  for (int p = 0; p < world; ++p) {
    if (!part_peers[p] || !y_peers[p]) return QUICK_ERR_INVALID_ARG;
    parts.p[p] = part_peers[p];
    ys.p[p] = y_peers[p];
  }
  const int c0 = (N / world) * rank, c1 = c0 + N / world;
  const long long work = (long long)M * ((c1 - c0) / 8);
  const int threads = 256;
  const unsigned blocks = (unsigned)((work + threads - 1) / threads < 148 * 4 ? (work + threads - 1) / threads : 148 * 4);
  quick_tp::row_reduce_kernel<<<blocks, threads, 0, s>>>(parts, ys, world, M, N, ldy, c0, c1);
  st = quick_tp::cuda_status(cudaGetLastError());
  if (st != QUICK_OK) return st;
  return quick_tp::barrier(flag_peers, world, rank, s);
}

}  // extern "C"
