// Host-side parts of the C ABI: status strings and the batch plan (group_by_delta).
#include <cstdint>
#include <vector>

#include "../../include/dz_b200.h"

extern "C" const char* dz_version(void) { return "dz_b200 0.1.0 sm_100a"; }

extern "C" const char* dz_strerror(int status) {
  switch (status) {
    case DZ_OK: return "ok";
    case DZ_E_SHAPE: return "ShapeError: operands have incompatible or invalid dimensions";
    case DZ_E_ENCODING: return "EncodingError: packed payload too short for the requested codes";
    case DZ_E_FORMAT: return "FormatError: corrupt index stream (length, or kept positions not increasing)";
    case DZ_E_PARTITION: return "PartitionError: invalid tensor-parallel partition";
    case DZ_E_UNKNOWN: return "UnknownDeltaError: a row references an unknown delta";
    case DZ_E_VALUE: return "ValueError: invalid argument (e.g. scales length)";
    case DZ_E_UNSUPPORTED: return "unsupported layout for this kernel";
    case DZ_E_CUDA: return "CUDA runtime error";
    default: return "unknown status";
  }
}

extern "C" int32_t dz_plan_max_jobs(int32_t T) { return T < 0 ? 0 : 2 * T + 2; }

// Stable sort of token rows by slot (inference.py:106-123: `sorted` is stable), then cut into
// jobs: base token chunks of 64, sparse delta chunks of 8, dense delta chunks of 32.
extern "C" int dz_plan(const int32_t* slots, int32_t T, const int32_t* kinds, int32_t n_slots,
                       int32_t with_base, int32_t* order_out, dz_job* jobs_out, int32_t max_jobs,
                       int32_t* n_jobs_out) {
  if (T < 0 || n_slots < 0 || !n_jobs_out) return DZ_E_VALUE;
  *n_jobs_out = 0;
  for (int32_t t = 0; t < T; t++)
    if (slots[t] < 0 || slots[t] >= n_slots) return DZ_E_UNKNOWN;  // inference.py:135-137
  std::vector<int32_t> count(static_cast<size_t>(n_slots) + 1, 0);
  for (int32_t t = 0; t < T; t++) count[slots[t] + 1]++;
  for (int32_t s = 0; s < n_slots; s++) count[s + 1] += count[s];
  std::vector<int32_t> start(count.begin(), count.end() - 1), fill(start);
  for (int32_t t = 0; t < T; t++) order_out[fill[slots[t]]++] = t;
  int32_t nj = 0;
  auto push = [&](int32_t slot, int32_t b, int32_t c, int32_t kind) -> bool {
    if (nj >= max_jobs) return false;
    jobs_out[nj++] = dz_job{slot, b, c, kind};
    return true;
  };
  if (with_base)
    for (int32_t b = 0; b < T; b += 64)
      if (!push(-1, b, (T - b) < 64 ? (T - b) : 64, 0)) return DZ_E_VALUE;
  for (int32_t s = 0; s < n_slots; s++) {
    const int32_t c = count[s + 1] - count[s];
    if (c == 0) continue;
    const int32_t kind = kinds[s];
    if (kind != DZ_KIND_SPARSE4 && kind != DZ_KIND_SPARSE2 && kind != DZ_KIND_SPARSE3 && kind != DZ_KIND_DENSE)
      return DZ_E_VALUE;
    const int32_t chunk = kind == DZ_KIND_DENSE ? 32 : 8;
    for (int32_t off = 0; off < c; off += chunk)
      if (!push(s, start[s] + off, (c - off) < chunk ? (c - off) : chunk, kind)) return DZ_E_VALUE;
  }
  *n_jobs_out = nj;
  return DZ_OK;
}
