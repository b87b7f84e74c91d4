// On-device admission (dz_admit_device) — the decision of scheduler.select_batch
// (scheduler.py:73-123) computed by one CTA from device-resident request metadata, so a serving
// loop can go admission -> slots -> dz_plan_device -> dz_sbmm without a host round trip.
//
// select_batch scans the arrival-ordered queue once: a request joins while the batch has room
// (< K including the running requests) and its delta is already selected or fewer than N deltas
// are; an admission that bypasses a rejected request is a line skip, linked to the earliest
// batch member of its delta. The scan is sequential, but its outcome has a closed form:
//   * let S0 be the running requests' deltas; a new delta d (not in S0) is selected at its FIRST
//     queue occurrence iff fewer than N deltas are selected then, i.e. iff its rank among new
//     deltas in first-occurrence order is <= N - |S0|; every occurrence of d shares that
//     eligibility;
//   * the admitted requests are the eligible ones in queue order, cut after K - R of them (the
//     loop stops as soon as the batch is full, so nothing later is scanned);
//   * a request is a line skip iff a scanned, ineligible request precedes it; its parent is the
//     earlier of the delta's earliest running request and its first queue occurrence (queue order
//     is key order).
// Each quantity is a block-wide scan or a per-delta min, so the kernel is O(Q / threads).
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include <cub/block/block_scan.cuh>

#include "dz_common.cuh"

namespace dz {
namespace sched {

constexpr int THREADS = 1024;
constexpr int ITEMS = 8;  // queue entries per thread: Q <= 8192
constexpr int BIG = 0x7fffffff;

__global__ void __launch_bounds__(THREADS) k_admit(const int32_t* __restrict__ q_model, const int32_t* __restrict__ q_id,
                                                   const int32_t* __restrict__ q_rank, int Q,
                                                   const int32_t* __restrict__ r_model, const int32_t* __restrict__ r_id,
                                                   const int32_t* __restrict__ r_rank, int R, int n_models, int K, int N,
                                                   uint8_t* __restrict__ admitted, uint8_t* __restrict__ skipped,
                                                   int32_t* __restrict__ parent, uint8_t* __restrict__ selected,
                                                   int32_t* __restrict__ counts, int32_t* __restrict__ err) {
  using Scan = cub::BlockScan<int, THREADS>;
  __shared__ typename Scan::TempStorage scan_tmp;
  extern __shared__ int sh[];
  int* first_pos = sh;                // [n_models] first queue position of the delta
  int* run_rank = sh + n_models;      // [n_models] smallest key rank among its running requests
  int* run_who = sh + 2 * n_models;   // [n_models] that request's id
  int* new_rank = sh + 3 * n_models;  // [n_models] rank of the delta among new deltas (1-based), 0 = none
  __shared__ int n_s0, bad, cut;
  const int tid = threadIdx.x;
  for (int m = tid; m < n_models; m += THREADS) {
    first_pos[m] = BIG;
    run_rank[m] = BIG;
    run_who[m] = -1;
    new_rank[m] = 0;
  }
  if (tid == 0) { n_s0 = 0; bad = 0; cut = Q; }
  __syncthreads();
  for (int i = tid; i < R; i += THREADS) {
    const int m = r_model[i];
    if (m < 0 || m >= n_models) { bad = 1; continue; }
    atomicMin(&run_rank[m], r_rank[i]);
  }
  for (int i = tid; i < Q; i += THREADS) {
    const int m = q_model[i];
    if (m < 0 || m >= n_models) { bad = 1; continue; }
    atomicMin(&first_pos[m], i);
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) { *err = DZ_E_VALUE; counts[0] = counts[1] = 0; }
    return;
  }
  for (int i = tid; i < R; i += THREADS)
    if (r_rank[i] == run_rank[r_model[i]]) run_who[r_model[i]] = r_id[i];  // ranks are unique
  for (int m = tid; m < n_models; m += THREADS)
    if (run_rank[m] != BIG) atomicAdd(&n_s0, 1);
  __syncthreads();
  // rank of each new delta in first-occurrence order: exclusive scan of first-occurrence flags
  int flag[ITEMS], pre[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    const int i = tid * ITEMS + k;
    const int m = i < Q ? q_model[i] : 0;
    flag[k] = (i < Q && first_pos[m] == i && run_rank[m] == BIG) ? 1 : 0;
  }
  Scan(scan_tmp).ExclusiveSum(flag, pre);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ITEMS; k++)
    if (flag[k]) new_rank[q_model[tid * ITEMS + k]] = pre[k] + 1;
  __syncthreads();
  // eligibility, then the K cut: admitted = the first K - R eligible requests in queue order
  const int room = K - R, free_deltas = N - n_s0;
  int elig[ITEMS], epre[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    const int i = tid * ITEMS + k;
    const int m = i < Q ? q_model[i] : 0;
    elig[k] = (i < Q && (run_rank[m] != BIG || new_rank[m] <= free_deltas)) ? 1 : 0;
  }
  int n_elig = 0;
  Scan(scan_tmp).ExclusiveSum(elig, epre, n_elig);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ITEMS; k++)  // the room-th eligible request ends the scan
    if (room > 0 && elig[k] && epre[k] == room - 1) cut = tid * ITEMS + k;
  if (room <= 0 && tid == 0) cut = -1;  // the batch is full before the first queued request
  __syncthreads();
  // line skips: an ineligible request scanned before an admitted one
  int inel[ITEMS], ipre[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    const int i = tid * ITEMS + k;
    inel[k] = (i < Q && i <= cut && !elig[k]) ? 1 : 0;
  }
  Scan(scan_tmp).ExclusiveSum(inel, ipre);
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    const int i = tid * ITEMS + k;
    if (i >= Q) continue;
    const int m = q_model[i];
    const bool adm = elig[k] && i <= cut;
    const bool skip = adm && ipre[k] > 0;
    admitted[i] = adm ? 1 : 0;
    skipped[i] = skip ? 1 : 0;
    int par = -1;
    if (skip) {  // earliest batch member of the delta before this request (scheduler.py:101-104)
      const int fp = first_pos[m];
      const bool q_first = fp < i;  // the delta's first queue occurrence, already admitted
      if (q_first && (run_rank[m] == BIG || q_rank[fp] < run_rank[m]))
        par = q_id[fp];
      else
        par = run_who[m];
    }
    parent[i] = par;
  }
  // selected deltas: S0 and the new deltas whose first occurrence was admitted
  for (int m = tid; m < n_models; m += THREADS)
    selected[m] = (run_rank[m] != BIG || (new_rank[m] > 0 && new_rank[m] <= free_deltas && first_pos[m] <= cut)) ? 1 : 0;
  if (tid == 0) {
    const int n_adm = cut < 0 ? 0 : (n_elig < room ? n_elig : room);
    counts[0] = n_adm;
    counts[1] = 0;
    *err = DZ_OK;
  }
}

}  // namespace sched
}  // namespace dz

using namespace dz;

extern "C" int dz_admit_device(const int32_t* q_model, const int32_t* q_id, const int32_t* q_rank, int32_t Q,
                               const int32_t* r_model, const int32_t* r_id, const int32_t* r_rank, int32_t R,
                               int32_t n_models, int32_t K, int32_t N, uint8_t* admitted, uint8_t* skipped,
                               int32_t* parent, uint8_t* selected, int32_t* counts, int32_t* err, void* stream) {
  if (Q < 0 || R < 0 || K < 1 || N < 1 || n_models < 1 || n_models > 4096) return DZ_E_VALUE;
  if (Q > sched::THREADS * sched::ITEMS) return DZ_E_VALUE;
  if (!admitted || !skipped || !parent || !selected || !counts || !err) return DZ_E_VALUE;
  if ((Q > 0 && (!q_model || !q_id || !q_rank)) || (R > 0 && (!r_model || !r_id || !r_rank))) return DZ_E_VALUE;
  const size_t smem = static_cast<size_t>(4) * n_models * sizeof(int);
  static std::once_flag once;  // one-time, idempotent kernel attribute setup
  std::call_once(once, [] {
    cudaFuncSetAttribute(sched::k_admit, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4096 * 4);
  });
  sched::k_admit<<<1, sched::THREADS, smem, static_cast<cudaStream_t>(stream)>>>(
      q_model, q_id, q_rank, Q, r_model, r_id, r_rank, R, n_models, K, N, admitted, skipped, parent, selected, counts,
      err);
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}
