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
                                               int32_t* __restrict__ n_jobs_out, int32_t* __restrict__ err,
                                               int sp_chunk) {
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
      const int c = count[s], chunk = kinds[s] == DZ_KIND_DENSE ? DZ_DENSE_JOB_TOKENS : sp_chunk;
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
    const int c = count[s], chunk = kinds[s] == DZ_KIND_DENSE ? DZ_DENSE_JOB_TOKENS : sp_chunk;
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
                              int32_t* n_jobs_dev, int32_t* err_dev, int32_t sparse_job_tokens, void* stream) {
  const int sp_chunk = sparse_job_tokens == 0 ? 8 : sparse_job_tokens;
  if (T < 0 || n_slots < 1 || n_slots > 4096 || !n_jobs_dev || !err_dev || max_jobs < 0) return DZ_E_VALUE;
  if (sp_chunk != 8 && sp_chunk != 16) return DZ_E_VALUE;
  if (T > 0 && (!slots_dev || !order_dev || !jobs_dev || !kinds_dev)) return DZ_E_VALUE;
  const size_t smem = static_cast<size_t>(3) * n_slots * sizeof(int);
  static std::once_flag once;  // one-time, idempotent kernel attribute setup
  std::call_once(once, [] {
    cudaFuncSetAttribute(plan::k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 4096 * 4);
  });
  plan::k_plan<<<1, 1024, smem, static_cast<cudaStream_t>(stream)>>>(slots_dev, T, kinds_dev, n_slots, with_base,
                                                                   order_dev, jobs_dev, max_jobs, n_jobs_dev, err_dev, sp_chunk);
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}

// ------------------------------------------------------------------------------------------
// On-device MIXED plan (dz_plan_mixed_device): the same staging and job cut as the host
// dz_plan_mixed (dz_host.cpp): groups of >= pf_min tokens of a 2:4 kind go whole to prefill jobs
// (K3) of DZ_PREFILL_JOB_SIZE tokens, staged first grouped by slot; every other token follows in
// its original order and is planned for K2 like dz_plan over the staged rows. Prefill jobs go to
// jobs[0, T) and decode jobs to jobs[T, ...) so the launches can use fixed offsets; the counts
// are written to counts[0] = prefill jobs, counts[1] = decode jobs, counts[2] = t_pf.
namespace dz {
namespace plan {

__global__ void __launch_bounds__(1024) k_plan_mixed(const int32_t* __restrict__ slots, int T,
                                                     const int32_t* __restrict__ kinds, int n_slots, int with_base,
                                                     int pf_min, int32_t* __restrict__ perm, int32_t* __restrict__ order,
                                                     dz_job* __restrict__ jobs, int32_t* __restrict__ counts,
                                                     int32_t* __restrict__ err, int sp_chunk) {
  extern __shared__ int sh[];
  int* count = sh;               // [n_slots]
  int* npf = sh + n_slots;       // [n_slots] prefill tokens of the slot
  int* pstart = npf + n_slots;   // [n_slots] first staged prefill row of the slot
  int* dstart = pstart + n_slots;  // [n_slots] first decode `order` position of the slot
  int* rank = dstart + n_slots;  // [n_slots] running occurrence counter (stable pass)
  __shared__ int bad, t_pf, n_pf, n_dec;
  const int tid = threadIdx.x;
  for (int s = tid; s < n_slots; s += blockDim.x) { count[s] = 0; rank[s] = 0; }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int t = tid; t < T; t += blockDim.x) {
    const int s = slots[t];
    if (s < 0 || s >= n_slots) bad = 1;
    else atomicAdd(&count[s], 1);
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) { *err = DZ_E_UNKNOWN; counts[0] = counts[1] = counts[2] = 0; }
    return;
  }
  if (tid == 0) {  // per-slot split and exclusive scans (n_slots <= 4096: a serial pass is ~µs)
    int ps = 0, pj = 0;
    for (int s = 0; s < n_slots; s++) {
      const int c = count[s], k = kinds[s];
      const int np = (pf_min > 0 && c >= pf_min && k != DZ_KIND_DENSE) ? DZ_PREFILL_TOKENS(c) : 0;
      npf[s] = np;
      pstart[s] = ps;
      ps += np;
      const int step = DZ_PREFILL_JOB_SIZE(np);
      pj += (np + step - 1) / step;
    }
    t_pf = ps;
    n_pf = pj;
    const int n_base = with_base ? (T - ps + DZ_BASE_JOB_TOKENS - 1) / DZ_BASE_JOB_TOKENS : 0;
    int ds = 0, dj = n_base;
    for (int s = 0; s < n_slots; s++) {
      const int c = count[s] - npf[s], chunk = kinds[s] == DZ_KIND_DENSE ? DZ_DENSE_JOB_TOKENS : sp_chunk;
      dstart[s] = ds;
      ds += c;
      dj += (c + chunk - 1) / chunk;
    }
    n_dec = dj;
    counts[0] = pj;
    counts[1] = dj;
    counts[2] = ps;
    *err = DZ_OK;
  }
  __syncthreads();
  // prefill jobs [0, n_pf) in slot order, decode jobs from T: base jobs, then delta jobs per slot
  if (tid == 32) {  // (warp 0 runs the stable pass below)
    int pj = 0, dj = 0;
    for (int s = 0; s < n_slots; s++) {
      const int step = DZ_PREFILL_JOB_SIZE(npf[s]);
      for (int off = 0; off < npf[s]; off += step) jobs[pj++] = dz_job{s, pstart[s] + off, min(step, npf[s] - off), kinds[s]};
    }
    const int n_base = with_base ? (T - t_pf + DZ_BASE_JOB_TOKENS - 1) / DZ_BASE_JOB_TOKENS : 0;
    for (int b = 0; b < n_base; b++) {
      const int b0 = t_pf + b * DZ_BASE_JOB_TOKENS;
      jobs[T + dj++] = dz_job{-1, b0, min(DZ_BASE_JOB_TOKENS, T - b0), 0};
    }
    for (int s = 0; s < n_slots; s++) {
      const int c = count[s] - npf[s], chunk = kinds[s] == DZ_KIND_DENSE ? DZ_DENSE_JOB_TOKENS : sp_chunk;
      for (int off = 0; off < c; off += chunk) jobs[T + dj++] = dz_job{s, dstart[s] + off, min(chunk, c - off), kinds[s]};
    }
  }
  // stable pass, one warp, tokens in original order: the occurrence rank of each token inside its
  // slot decides prefill (rank < npf) or decode; decode tokens keep their original order after t_pf
  if (tid < 32) {
    const unsigned lt = (1u << tid) - 1u;
    int ndec = 0;  // decode tokens seen so far (warp-uniform)
    for (int b = 0; b < T; b += 32) {
      const int t = b + tid;
      const unsigned active = __ballot_sync(0xffffffffu, t < T);
      int s = 0, r = 0;
      bool pre = false;
      if (t < T) {
        s = slots[t];
        const unsigned same = __match_any_sync(active, s);
        r = rank[s] + __popc(same & lt);
        __syncwarp(active);
        if ((same & lt) == 0) rank[s] += __popc(same);
        pre = r < npf[s];
      }
      const unsigned dec = __ballot_sync(0xffffffffu, t < T && !pre);
      if (t < T) {
        if (pre) {
          perm[pstart[s] + r] = t;
        } else {
          const int row = t_pf + ndec + __popc(dec & lt);  // staged row of this decode token
          perm[row] = t;
          order[dstart[s] + (r - npf[s])] = row;
        }
      }
      ndec += __popc(dec);
      __syncwarp();
    }
  }
}

}  // namespace plan
}  // namespace dz

extern "C" int dz_plan_mixed_device(const int32_t* slots_dev, int32_t T, const int32_t* kinds_dev, int32_t n_slots,
                                    int32_t with_base, int32_t pf_min, int32_t* perm_dev, int32_t* order_dev,
                                    dz_job* jobs_dev, int32_t* counts_dev, int32_t* err_dev,
                                    int32_t sparse_job_tokens, void* stream) {
  const int sp_chunk = sparse_job_tokens == 0 ? 8 : sparse_job_tokens;
  if (T < 0 || n_slots < 1 || n_slots > 4096 || !counts_dev || !err_dev) return DZ_E_VALUE;
  if (sp_chunk != 8 && sp_chunk != 16) return DZ_E_VALUE;
  if (T > 0 && (!slots_dev || !perm_dev || !order_dev || !jobs_dev || !kinds_dev)) return DZ_E_VALUE;
  const size_t smem = static_cast<size_t>(5) * n_slots * sizeof(int);
  static std::once_flag once;  // one-time, idempotent kernel attribute setup
  std::call_once(once, [] {
    cudaFuncSetAttribute(plan::k_plan_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 4096 * 4);
  });
  plan::k_plan_mixed<<<1, 1024, smem, static_cast<cudaStream_t>(stream)>>>(
      slots_dev, T, kinds_dev, n_slots, with_base, pf_min, perm_dev, order_dev, jobs_dev, counts_dev, err_dev, sp_chunk);
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}
