// On-device plan (dz_plan_device) — group_by_delta (inference.py:106-123) and the dz_plan job cut
// computed on the GPU from device-resident slots, so a decode loop needs no host round trip.
#include <mutex>
#include <cuda_runtime.h>

#include <cstdint>

#include "dz_common.cuh"

// Stable counting sort of tokens by slot + the dz_plan job cut, by one CTA. Stability comes from
// a single warp scattering the tokens in index order, 32 at a time (__match_any_sync ranks equal
// slots inside a chunk).
namespace dz {
namespace plan {

__global__ void __launch_bounds__(1024) k_plan(const int32_t* __restrict__ slots, int T,
                                               const int32_t* __restrict__ kinds, int n_slots, int with_base,
                                               int32_t* __restrict__ order, dz_job* __restrict__ jobs, int max_jobs,
                                               int32_t* __restrict__ n_jobs_out, int32_t* __restrict__ err) {
  extern __shared__ int sh[];
  int* count = sh;              // [n_slots]
  int* fill = sh + n_slots;     // [n_slots] running position (stable scatter)
  int* jstart = fill + n_slots; // [n_slots] first job of the slot
  __shared__ int bad, total_jobs;
  const int tid = threadIdx.x;
  for (int s = tid; s < n_slots; s += blockDim.x) count[s] = 0;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int t = tid; t < T; t += blockDim.x) {
    const int s = slots[t];
    if (s < 0 || s >= n_slots) bad = 1;
    else atomicAdd(&count[s], 1);
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) { *err = DZ_E_UNKNOWN; *n_jobs_out = 0; }
    return;
  }
  const int n_base = with_base ? (T + DZ_BASE_JOB_TOKENS - 1) / DZ_BASE_JOB_TOKENS : 0;
  if (tid == 0) {  // exclusive scans over slots (n_slots <= 4096: a serial pass is ~µs)
    int pos = 0, jb = n_base;
    for (int s = 0; s < n_slots; s++) {
      const int c = count[s], chunk = kinds[s] == DZ_KIND_DENSE ? 32 : 8;
      fill[s] = pos;
      jstart[s] = jb;
      pos += c;
      jb += (c + chunk - 1) / chunk;
    }
    total_jobs = jb;
    *err = jb > max_jobs ? DZ_E_VALUE : DZ_OK;
    *n_jobs_out = jb > max_jobs ? 0 : jb;
  }
  __syncthreads();
  if (total_jobs > max_jobs) return;
  // delta jobs (slot order) and base jobs, before fill[] is consumed by the scatter
  for (int s = tid; s < n_slots; s += blockDim.x) {
    const int c = count[s], chunk = kinds[s] == DZ_KIND_DENSE ? 32 : 8;
    for (int k = 0; k * chunk < c; k++) {
      const int n = c - k * chunk < chunk ? c - k * chunk : chunk;
      jobs[jstart[s] + k] = dz_job{s, fill[s] + k * chunk, n, kinds[s]};
    }
  }
  for (int b = tid; b < n_base; b += blockDim.x) {
    const int b0 = b * DZ_BASE_JOB_TOKENS;
    jobs[b] = dz_job{-1, b0, T - b0 < DZ_BASE_JOB_TOKENS ? T - b0 : DZ_BASE_JOB_TOKENS, 0};
  }
  __syncthreads();
  if (tid < 32) {  // stable scatter, one warp, tokens in index order
    const unsigned lt = (1u << tid) - 1u;
    for (int base = 0; base < T; base += 32) {
      const int t = base + tid;
      const unsigned active = __ballot_sync(0xffffffffu, t < T);
      if (t < T) {
        const int s = slots[t];
        const unsigned same = __match_any_sync(active, s);
        const int pos = fill[s] + __popc(same & lt);
        order[pos] = t;
        __syncwarp(active);
        if ((same & lt) == 0) fill[s] += __popc(same);  // the group's lowest lane advances the slot
      }
      __syncwarp();
    }
  }
}

}  // namespace plan
}  // namespace dz

using namespace dz;

extern "C" int dz_plan_device(const int32_t* slots_dev, int32_t T, const int32_t* kinds_dev, int32_t n_slots,
                              int32_t with_base, int32_t* order_dev, dz_job* jobs_dev, int32_t max_jobs,
                              int32_t* n_jobs_dev, int32_t* err_dev, void* stream) {
  if (T < 0 || n_slots < 1 || n_slots > 4096 || !n_jobs_dev || !err_dev || max_jobs < 0) return DZ_E_VALUE;
  if (T > 0 && (!slots_dev || !order_dev || !jobs_dev || !kinds_dev)) return DZ_E_VALUE;
  const size_t smem = static_cast<size_t>(3) * n_slots * sizeof(int);
  static std::once_flag once;  // one-time, idempotent kernel attribute setup
  std::call_once(once, [] {
    cudaFuncSetAttribute(plan::k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 4096 * 4);
  });
  plan::k_plan<<<1, 1024, smem, static_cast<cudaStream_t>(stream)>>>(slots_dev, T, kinds_dev, n_slots, with_base,
                                                                   order_dev, jobs_dev, max_jobs, n_jobs_dev, err_dev);
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}
