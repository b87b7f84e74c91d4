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

extern "C" int32_t dz_plan_max_jobs(int32_t T) { return T < 0 ? 0 : 2 * T + 2; }  // >= base + delta + prefill jobs

static int32_t sparse_chunk(int32_t sparse_job_tokens) {
  return sparse_job_tokens == 16 ? 16 : sparse_job_tokens == 0 || sparse_job_tokens == 8 ? 8 : -1;
}

// Stable sort of token rows by slot (inference.py:106-123: `sorted` is stable), then cut into
// jobs: base token chunks of DZ_BASE_JOB_TOKENS, sparse delta chunks of 8, dense delta chunks of 32.
extern "C" int dz_plan(const int32_t* slots, int32_t T, const int32_t* kinds, int32_t n_slots,
                       int32_t with_base, int32_t* order_out, dz_job* jobs_out, int32_t max_jobs,
                       int32_t* n_jobs_out, int32_t sparse_job_tokens) {
  const int32_t sp_chunk = sparse_chunk(sparse_job_tokens);
  if (T < 0 || n_slots < 0 || !n_jobs_out || sp_chunk < 0) return DZ_E_VALUE;
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
    for (int32_t b = 0; b < T; b += DZ_BASE_JOB_TOKENS)
      if (!push(-1, b, (T - b) < DZ_BASE_JOB_TOKENS ? (T - b) : DZ_BASE_JOB_TOKENS, 0)) return DZ_E_VALUE;
  for (int32_t s = 0; s < n_slots; s++) {
    const int32_t c = count[s + 1] - count[s];
    if (c == 0) continue;
    const int32_t kind = kinds[s];
    if (kind != DZ_KIND_SPARSE4 && kind != DZ_KIND_SPARSE2 && kind != DZ_KIND_SPARSE3 && kind != DZ_KIND_DENSE)
      return DZ_E_VALUE;
    const int32_t chunk = kind == DZ_KIND_DENSE ? DZ_DENSE_JOB_TOKENS : sp_chunk;
    for (int32_t off = 0; off < c; off += chunk)
      if (!push(s, start[s] + off, (c - off) < chunk ? (c - off) : chunk, kind)) return DZ_E_VALUE;
  }
  *n_jobs_out = nj;
  return DZ_OK;
}

// Mixed plan (prefill + decode). A group of c >= pf_min tokens with a 2:4 sparse kind goes to the
// prefill kernel whole: ceil(c / J) jobs (J = DZ_PREFILL_JOB_TOKENS) of equal 16-aligned size, the
// last one shorter (a 256-token request becomes 2 x 128 instead of 240 + a 16-token remainder that
// would re-stream the delta twice on the decode kernel). Prefill tokens are staged first (grouped
// by slot in slot order); every other token follows in its original order and is planned exactly
// like dz_plan over the staged rows.
extern "C" int dz_plan_mixed(const int32_t* slots, int32_t T, const int32_t* kinds, int32_t n_slots,
                             int32_t with_base, int32_t pf_min, int32_t* perm_out, int32_t* order_out,
                             dz_job* jobs_out, int32_t max_jobs, int32_t* n_jobs_out, int32_t* n_pf_jobs_out,
                             int32_t* t_pf_out, int32_t sparse_job_tokens) {
  const int32_t sp_chunk = sparse_chunk(sparse_job_tokens);
  if (T < 0 || n_slots < 0 || !n_jobs_out || !n_pf_jobs_out || !t_pf_out || sp_chunk < 0) return DZ_E_VALUE;
  *n_jobs_out = *n_pf_jobs_out = *t_pf_out = 0;
  for (int32_t t = 0; t < T; t++)
    if (slots[t] < 0 || slots[t] >= n_slots) return DZ_E_UNKNOWN;  // inference.py:135-137
  for (int32_t s = 0; s < n_slots; s++)
    if (kinds[s] != DZ_KIND_SPARSE4 && kinds[s] != DZ_KIND_SPARSE2 && kinds[s] != DZ_KIND_SPARSE3 &&
        kinds[s] != DZ_KIND_DENSE)
      return DZ_E_VALUE;
  std::vector<int32_t> count(static_cast<size_t>(n_slots), 0);
  for (int32_t t = 0; t < T; t++) count[slots[t]]++;
  std::vector<int32_t> npf(static_cast<size_t>(n_slots), 0);  // prefill tokens per slot
  for (int32_t s = 0; s < n_slots; s++)
    if (pf_min > 0 && count[s] >= pf_min && kinds[s] != DZ_KIND_DENSE) npf[s] = DZ_PREFILL_TOKENS(count[s]);
  // staged order: prefill groups by slot, then the decode tokens in original order
  std::vector<int32_t> pstart(static_cast<size_t>(n_slots) + 1, 0);
  for (int32_t s = 0; s < n_slots; s++) pstart[s + 1] = pstart[s] + npf[s];
  const int32_t t_pf = pstart[n_slots];
  std::vector<int32_t> fill(pstart.begin(), pstart.end() - 1);
  int32_t nd = t_pf;
  std::vector<int32_t> dslot;  // slot of each decode staged row
  dslot.reserve(static_cast<size_t>(T - t_pf));
  for (int32_t t = 0; t < T; t++) {
    const int32_t s = slots[t];
    if (fill[s] < pstart[s] + npf[s]) {
      perm_out[fill[s]++] = t;
    } else {
      perm_out[nd++] = t;
      dslot.push_back(slots[t]);
    }
  }
  int32_t nj = 0;
  auto push = [&](int32_t slot, int32_t b, int32_t c, int32_t kind) -> bool {
    if (nj >= max_jobs) return false;
    jobs_out[nj++] = dz_job{slot, b, c, kind};
    return true;
  };
  for (int32_t s = 0; s < n_slots; s++) {
    const int32_t step = DZ_PREFILL_JOB_SIZE(npf[s]);
    for (int32_t off = 0; off < npf[s]; off += step)
      if (!push(s, pstart[s] + off, (npf[s] - off) < step ? (npf[s] - off) : step, kinds[s])) return DZ_E_VALUE;
  }
  const int32_t n_pf = nj;
  // decode part over staged rows [t_pf, T): base jobs, then delta jobs (dz_plan's rules)
  const int32_t Td = T - t_pf;
  std::vector<int32_t> dcount(static_cast<size_t>(n_slots) + 1, 0);
  for (int32_t i = 0; i < Td; i++) dcount[dslot[i] + 1]++;
  for (int32_t s = 0; s < n_slots; s++) dcount[s + 1] += dcount[s];
  std::vector<int32_t> dstart(dcount.begin(), dcount.end() - 1), dfill(dstart);
  for (int32_t i = 0; i < Td; i++) order_out[dfill[dslot[i]]++] = t_pf + i;
  if (with_base)
    for (int32_t b = t_pf; b < T; b += DZ_BASE_JOB_TOKENS)
      if (!push(-1, b, (T - b) < DZ_BASE_JOB_TOKENS ? (T - b) : DZ_BASE_JOB_TOKENS, 0)) return DZ_E_VALUE;
  for (int32_t s = 0; s < n_slots; s++) {
    const int32_t c = dcount[s + 1] - dcount[s];
    if (c == 0) continue;
    const int32_t chunk = kinds[s] == DZ_KIND_DENSE ? DZ_DENSE_JOB_TOKENS : sp_chunk;
    for (int32_t off = 0; off < c; off += chunk)
      if (!push(s, dstart[s] + off, (c - off) < chunk ? (c - off) : chunk, kinds[s])) return DZ_E_VALUE;
  }
  *n_jobs_out = nj;
  *n_pf_jobs_out = n_pf;
  *t_pf_out = t_pf;
  return DZ_OK;
}
