// Fused tensor-parallel reduction of a row-parallel linear over peer memory (NVLink / NVSwitch).
//
// The reference simulates the row-parallel all-reduce by summing the shard products in shard
// order (inference.py:216-223, tp_forward). Here each rank's k_sbmm leaves its fp32 partial
// planes (base K-splits + delta) in its workspace, exactly as for one GPU, and this kernel
// replaces both k_finalize and a separate NCCL all-reduce:
//
//   1. sum the local planes (fixed order) into this rank's reduce buffer R_rank[epoch & 1];
//   2. grid barrier; one thread publishes `epoch` into every peer's ready-flag slot for this
//      rank (release, system scope) and advances the local epoch;
//   3. every CTA waits until all peers' flags reached `epoch` (acquire, system scope);
//   4. Y = act(R_0 + R_1 + ... + R_{world-1}) read over NVLink in rank order: identical and
//      deterministic on every rank (the reference's shard-order sum, in fp32).
//
// R is double-buffered by epoch parity: a rank can only be writing epoch e after it saw every
// peer's ready flag for e-1, which each peer published after it finished reading epoch e-2 (the
// same buffer) in stream order. The epoch lives in device memory, so a captured CUDA graph
// replays correctly. All CTAs must be co-resident (grid <= SMs), which the launcher guarantees.
#include <cuda_runtime.h>

#include <cstdint>

#include "dz_common.cuh"

namespace dz {
namespace tp {

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sense-reversal grid barrier (count + generation words); all CTAs are resident.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire_gpu(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0;
      st_release_gpu(gen, g + 1);
    } else {
      long long spins = 0;
      while (ld_acquire_gpu(gen) == g) {
        __nanosleep(64);
        if (++spins > (1ll << 27)) __trap();
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_tp_finalize(const float* __restrict__ part, int nsplit, int T, int out,
                                                     dz_tp_ctx tp, void* __restrict__ Y, int64_t ldy, int y_dtype,
                                                     int act) {
  const int e = static_cast<int>(tp.sync[0]) + 1;  // read by every CTA before the first barrier
  const int64_t buf = (e & 1) * tp.max_elems;
  const int64_t plane = static_cast<int64_t>(T) * out;
  const int64_t n4 = plane / 4;  // out % 4 == 0 (checked by the launcher)
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  float* mine = tp.peer_R[tp.rank] + buf;

  // 1. local planes -> this rank's reduce buffer
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 v = __ldcs(reinterpret_cast<const float4*>(part) + i);
    for (int sp = 1; sp <= nsplit; sp++) {
      const float4 w = __ldcs(reinterpret_cast<const float4*>(part + sp * plane) + i);
      v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
    }
    reinterpret_cast<float4*>(mine)[i] = v;
  }
  // 2. all local writes done -> publish readiness to every peer, advance the epoch
  grid_barrier(tp.sync + 1, tp.sync + 2);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < tp.world; p++) st_release_sys(tp.peer_flags[p] + tp.rank, e);
    tp.sync[0] = static_cast<unsigned>(e);
  }
  // 3. wait for every peer's buffer of this epoch (bounded: a peer that never arrives aborts the
  //    kernel after ~10 s instead of hanging the GPU)
  if (threadIdx.x < tp.world) {
    const int* f = tp.peer_flags[tp.rank] + threadIdx.x;
    long long spins = 0;
    while (ld_acquire_sys(f) < e) {
      __nanosleep(128);
      if (++spins > (1ll << 26)) __trap();
    }
  }
  __syncthreads();
  // 4. rank-order sum over peer memory -> Y
  const bool vec = (ldy % 4) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 v = __ldcv(reinterpret_cast<const float4*>(tp.peer_R[0] + buf) + i);
    for (int p = 1; p < tp.world; p++) {
      const float4 w = __ldcv(reinterpret_cast<const float4*>(tp.peer_R[p] + buf) + i);
      v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
    }
    if (act == DZ_ACT_TANH) { v.x = tanhf(v.x); v.y = tanhf(v.y); v.z = tanhf(v.z); v.w = tanhf(v.w); }
    const int t = static_cast<int>((4 * i) / out), r = static_cast<int>((4 * i) % out);
    const int64_t yo = static_cast<int64_t>(t) * ldy + r;
    const float f[4] = {v.x, v.y, v.z, v.w};
    if (y_dtype == DZ_F32) {
      if (vec) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(Y) + yo) = v;
      } else {
        for (int c = 0; c < 4; c++) reinterpret_cast<float*>(Y)[yo + c] = f[c];
      }
    } else {
      if (vec) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 w;
        w.x = *reinterpret_cast<const uint32_t*>(&lo);
        w.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(Y) + yo) = w;
      } else {
        for (int c = 0; c < 4; c++) reinterpret_cast<__nv_bfloat16*>(Y)[yo + c] = __float2bfloat16_rn(f[c]);
      }
    }
  }
}

}  // namespace tp
}  // namespace dz

using namespace dz;

// Launched by dz_sbmm (after k_sbmm) for a decode plan with args->tp set.
extern "C" int dz_tp_finalize_launch(const float* part, int nsplit, int T, int out, const dz_tp_ctx* ctx, void* Y,
                                     int64_t ldy, int y_dtype, int act, void* stream) {
  if (!ctx || ctx->world < 1 || ctx->rank < 0 || ctx->rank >= ctx->world || ctx->world > 64) return DZ_E_VALUE;
  if (out % 4 != 0) return DZ_E_SHAPE;
  if (static_cast<int64_t>(T) * out > ctx->max_elems) return DZ_E_SHAPE;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DZ_E_CUDA;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return DZ_E_CUDA;
  const int64_t n4 = static_cast<int64_t>(T) * out / 4;
  int grid = static_cast<int>((n4 + 255) / 256);
  if (grid > sms) grid = sms;  // co-resident CTAs: the grid barrier spins
  if (grid < 1) grid = 1;
  tp::k_tp_finalize<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(part, nsplit, T, out, *ctx, Y, ldy, y_dtype,
                                                                           act);
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}

extern "C" int dz_peer_alloc(size_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return DZ_E_VALUE;
  if (cudaMalloc(ptr, bytes) != cudaSuccess) return DZ_E_CUDA;
  return cudaMemset(*ptr, 0, bytes) == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}

extern "C" int dz_peer_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? DZ_OK : DZ_E_CUDA; }

extern "C" int dz_ipc_handle(void* ptr, uint8_t* handle64) {
  if (!ptr || !handle64) return DZ_E_VALUE;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return DZ_E_CUDA;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  for (int i = 0; i < 64; i++) handle64[i] = reinterpret_cast<const uint8_t*>(&h)[i];
  return DZ_OK;
}

extern "C" int dz_ipc_open(const uint8_t* handle64, void** ptr) {
  if (!ptr || !handle64) return DZ_E_VALUE;
  cudaIpcMemHandle_t h;
  for (int i = 0; i < 64; i++) reinterpret_cast<uint8_t*>(&h)[i] = handle64[i];
  return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}

extern "C" int dz_ipc_close(void* ptr) { return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? DZ_OK : DZ_E_CUDA; }
