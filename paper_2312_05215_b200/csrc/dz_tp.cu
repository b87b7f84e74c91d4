// Fused tensor-parallel reduction of a row-parallel linear over peer memory (NVLink / NVSwitch).
//
// The reference simulates the row-parallel all-reduce by summing the shard products in shard
// order (inference.py:216-223, tp_forward). Here each rank's k_sbmm leaves its fp32 partial
// planes (base K-splits + delta) in its workspace, exactly as for one GPU, and this kernel
// replaces both k_finalize and a separate NCCL all-reduce with a two-shot reduction:
//
//   1. sum the local planes (fixed order) into this rank's buffer R_rank[epoch & 1] (fp32);
//   2. grid barrier; publish `epoch` into every peer's phase-A flag slot for this rank
//      (release, system scope); wait for every peer's phase-A flag;
//   3. reduce-scatter: rank r owns the r-th contiguous chunk of the T x out output; it reads that
//      chunk of every peer's R in rank order (fp32 over NVLink), applies the activation, and
//      stores the chunk in G_r[epoch & 1] already in Y's dtype;
//   4. grid barrier; publish the phase-B flag; wait for every peer's phase-B flag;
//   5. all-gather: Y = the concatenation of every rank's G chunk (bf16 over NVLink for a bf16 Y).
// Every element is summed once, by its owner, in rank order: Y is identical on every rank and
// deterministic. NVLink bytes read per rank per reduction: (w-1)/w * T*out * (4 + sizeof(Y)),
// i.e. 6 * T*out * (w-1)/w for a bf16 Y (the one-shot version read (w-1) * T*out * 4).
//
// R and G are double-buffered by epoch parity: a rank writes epoch e only after it saw every
// peer's phase-A flag for e, which each peer published after finishing epoch e-1 (and so e-2)
// in stream order. The epoch lives in device memory, so a captured CUDA graph replays correctly.
// All CTAs must be co-resident (grid <= SMs), which the launcher guarantees.
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

__device__ __forceinline__ void publish_and_wait(const dz_tp_ctx& tp, int slot_off, int e) {
  grid_barrier(tp.sync + 1, tp.sync + 2);  // every CTA's writes of this phase are done
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < tp.world; p++) st_release_sys(tp.peer_flags[p] + slot_off + tp.rank, e);
  }
  // bounded wait: a peer that never arrives aborts the kernel after ~10 s instead of hanging
  if (threadIdx.x < tp.world) {
    const int* f = tp.peer_flags[tp.rank] + slot_off + threadIdx.x;
    long long spins = 0;
    while (ld_acquire_sys(f) < e) {
      __nanosleep(128);
      if (++spins > (1ll << 26)) __trap();
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void store4(void* base, int y_dtype, int64_t idx4, float4 v) {
  if (y_dtype == DZ_F32) {
    reinterpret_cast<float4*>(base)[idx4] = v;
  } else {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 w;
    w.x = *reinterpret_cast<const uint32_t*>(&lo);
    w.y = *reinterpret_cast<const uint32_t*>(&hi);
    reinterpret_cast<uint2*>(base)[idx4] = w;
  }
}

__global__ void __launch_bounds__(256) k_tp_finalize(const float* __restrict__ part, int nsplit, int T, int out,
                                                     dz_tp_ctx tp, void* __restrict__ Y, int64_t ldy, int y_dtype,
                                                     int act) {
  const int e = static_cast<int>(tp.sync[0]) + 1;  // read by every CTA before the first barrier
  const int64_t buf = (e & 1) * tp.max_elems;
  const int64_t plane = static_cast<int64_t>(T) * out;
  const int64_t n4 = plane / 4;  // out % 4 == 0 (checked by the launcher)
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t first = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  float* mine = tp.peer_R[tp.rank] + buf;

  // 1. local planes -> this rank's reduce buffer
  for (int64_t i = first; i < n4; i += stride) {
    float4 v = __ldcs(reinterpret_cast<const float4*>(part) + i);
    for (int sp = 1; sp <= nsplit; sp++) {
      const float4 w = __ldcs(reinterpret_cast<const float4*>(part + sp * plane) + i);
      v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
    }
    reinterpret_cast<float4*>(mine)[i] = v;
  }
  publish_and_wait(tp, 0, e);  // phase A: every rank's R is complete
  // 3. reduce-scatter: this rank's chunk, rank-order sum over peer memory -> G (Y's dtype)
  const int64_t c0 = n4 * tp.rank / tp.world, c1 = n4 * (tp.rank + 1) / tp.world;
  void* g_mine = tp.peer_R[tp.rank] + 2 * tp.max_elems + buf;
  for (int64_t i = c0 + first; i < c1; i += stride) {
    float4 v = __ldcv(reinterpret_cast<const float4*>(tp.peer_R[0] + buf) + i);
    for (int p = 1; p < tp.world; p++) {
      const float4 w = __ldcv(reinterpret_cast<const float4*>(tp.peer_R[p] + buf) + i);
      v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
    }
    if (act == DZ_ACT_TANH) { v.x = tanhf(v.x); v.y = tanhf(v.y); v.z = tanhf(v.z); v.w = tanhf(v.w); }
    store4(g_mine, y_dtype, i, v);
  }
  publish_and_wait(tp, 64, e);  // phase B: every rank's G chunk is complete
  if (blockIdx.x == 0 && threadIdx.x == 0) tp.sync[0] = static_cast<unsigned>(e);
  // 5. all-gather: copy every owner's chunk into Y
  const bool vec = (ldy % 4) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  for (int64_t i = first; i < n4; i += stride) {
    int p = static_cast<int>((i * tp.world) / n4);  // owner of float4 i (chunks are floor-split)
    while (p + 1 < tp.world && n4 * (p + 1) / tp.world <= i) p++;
    while (p > 0 && n4 * p / tp.world > i) p--;
    const void* g = tp.peer_R[p] + 2 * tp.max_elems + buf;
    const int t = static_cast<int>((4 * i) / out), r = static_cast<int>((4 * i) % out);
    const int64_t yo = static_cast<int64_t>(t) * ldy + r;
    if (y_dtype == DZ_F32) {
      const float4 v = __ldcv(reinterpret_cast<const float4*>(g) + i);
      if (vec) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(Y) + yo) = v;
      } else {
        const float f[4] = {v.x, v.y, v.z, v.w};
        for (int c = 0; c < 4; c++) reinterpret_cast<float*>(Y)[yo + c] = f[c];
      }
    } else {
      const uint2 w = __ldcv(reinterpret_cast<const uint2*>(g) + i);
      if (vec) {
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(Y) + yo) = w;
      } else {
        const uint16_t* h = reinterpret_cast<const uint16_t*>(&w);
        for (int c = 0; c < 4; c++) reinterpret_cast<uint16_t*>(Y)[yo + c] = h[c];
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
