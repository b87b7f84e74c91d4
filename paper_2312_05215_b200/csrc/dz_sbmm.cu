// K2 — fused base GEMM + selective batched (2:4, low-bit) delta matmul for sm_100a.
//
// Replaces inference.sbmm (inference.py:126-154): y_t = W_base x_t + ΔW_{slot(t)} x_t.
//
// Work decomposition. An item is (row tile of RT=128 output rows, job); a job is either the
// base GEMM for up to 64 tokens or one delta group for up to 16 (sparse) / 64 (dense) of its
// tokens (dz_plan, the group_by_delta of inference.py:106-123). Persistent CTAs pull items from
// an atomic counter. Per CTA: warp NW is the producer — it TMA-bulk-copies the native blocks of
// its item (one contiguous copy per 16-row group per chunk) and the X rows of the job's tokens
// into a 4-stage shared-memory ring; warps 0..NW-1 each own 16 rows, decode codes in registers
// (LOP3 magic-number bf16 conversion, deferred per-(row,128-col) scaling) and issue mma.sp
// m16n8k32 (2:4 deltas, the index nibble IS the sparse metadata) or mma m16n8k16 (base, dense
// deltas), fp32 accumulation. At the end of an item each warp writes its fp32 partial
// (base -> Pb, delta -> Pd; tokens are disjoint across delta jobs) and the LAST item of a row
// tile (per-tile counter) writes Y = Pb + Pd — no separate add kernel, no atomics on data,
// deterministic and batch-invariant (a token's K order never depends on the batch).
#include <cstdio>
#include <mutex>

#include "dz_common.cuh"

namespace dz {

constexpr int NW = 8;                     // consumer warps (16 rows each)
constexpr int NTHREADS = (NW + 1) * 32;   // + 1 producer warp
constexpr int RT = NW * kBlkRows;         // rows per item
constexpr int NB_SP = 4;                  // sparse chunk = 4 blocks = 512 columns
constexpr int NT_SP = 2;                  // n-tiles per sparse job (16 tokens)
constexpr int NT_DN = 8;                  // n-tiles per dense job (64 tokens)
constexpr int XS_SP = NB_SP * kBlkCols * 2 + 16;  // smem bytes per staged token row (16 B pad:
constexpr int XS_DN = kBlkCols * 2 + 16;          //   ldmatrix rows hit distinct bank groups)
constexpr int A_SP = NW * NB_SP * sparse_block_bytes(4);  // 26624
constexpr int X_SP = NT_SP * 8 * XS_SP;                   // 16640
constexpr int A_DN = NW * kDenseBlockBytes;               // 32768
constexpr int X_DN = NT_DN * 8 * XS_DN;                   // 17408
constexpr int STAGE_BYTES = (A_SP + X_SP > A_DN + X_DN) ? A_SP + X_SP : A_DN + X_DN;
constexpr int NSTAGE = 4;
constexpr int JOB_DN_TOK = NT_DN * 8;
constexpr int kMaxTiles = 4096;           // row tiles per call (out <= 524288)

struct StageHdr {
  int item;   // -1: end of work
  int chunk;
  int nb;     // blocks (of 128 columns) in this chunk
  int pad;
};

struct Smem {
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  StageHdr hdr[NSTAGE];
  int last_flag;
  int pad[3];
};
constexpr int SMEM_BYTES = STAGE_BYTES * NSTAGE + 1024;

struct Geo {
  int nkb;   // 128-column blocks along K
  int n16;   // 16-row groups along out
  int nrt;   // row tiles
};

__device__ __forceinline__ bool job_dense(int kind) { return kind == 0 || kind == DZ_KIND_DENSE; }
__device__ __forceinline__ int job_nchunks(int kind, const Geo& geo) {
  return job_dense(kind) ? geo.nkb : ceil_div(geo.nkb, NB_SP);
}
__device__ __forceinline__ int blk_bytes(int kind) {
  return job_dense(kind) ? kDenseBlockBytes : sparse_block_bytes(kind == DZ_KIND_SPARSE2 ? 2 : 4);
}

// ------------------------------------------------------------------------------------------
// Consumer math
// ------------------------------------------------------------------------------------------
template <int FB>
__device__ __forceinline__ void sparse_chunk(float (&acc)[NT_SP][4], uint32_t sA, uint32_t xl, int nb, int nt,
                                             uint32_t off2, int lane) {
  constexpr int CODE = sparse_code_bytes(FB);
  constexpr int BLK = sparse_block_bytes(FB);
  const int g = lane >> 2;
#pragma unroll 1
  for (int b = 0; b < nb; b++) {
    const uint32_t blk = sA + b * BLK;
    uint32_t cw[4];
    if (FB == 4) {
      const uint4 c = lds128(blk + lane * 16);
      cw[0] = c.x; cw[1] = c.y; cw[2] = c.z; cw[3] = c.w;
    } else {
      const uint2 c = lds64(blk + lane * 8);
      cw[0] = c.x; cw[1] = c.y; cw[2] = 0; cw[3] = 0;
    }
    const uint2 m = lds64(blk + CODE + lane * 8);
    const uint2 sv = lds64(blk + CODE + kMetaBytes + g * 8);
    const float s0 = __uint_as_float(sv.x), s1 = __uint_as_float(sv.y);
    float tmp[NT_SP][4];
#pragma unroll
    for (int n = 0; n < NT_SP; n++) tmp[n][0] = tmp[n][1] = tmp[n][2] = tmp[n][3] = 0.f;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      uint32_t a[4];
      if (FB == 4) {
        const uint32_t w = cw[i];
#pragma unroll
        for (int k = 0; k < 4; k++) a[k] = bf16x2_sub(lop3_and_or(w >> (4 * k), 0x000F000Fu, 0x43004300u), off2);
      } else {
        const uint32_t w = cw[i >> 1];
        const int o = 4 * (i & 1);
#pragma unroll
        for (int k = 0; k < 4; k++)
          a[k] = bf16x2_sub(lop3_and_or(w >> (2 * (o + k)), 0x00030003u, 0x43004300u), off2);
      }
      const uint32_t e = (i < 2) ? m.x : m.y;
#pragma unroll
      for (int n = 0; n < NT_SP; n++) {
        if (n < nt) {
          uint32_t bf[4];
          ldmatrix_x4(bf, xl + n * 8 * XS_SP + (b * kBlkCols + 32 * i) * 2);
          if (i & 1)
            mma_sp_bf16_16832<1>(tmp[n], a, bf, e);
          else
            mma_sp_bf16_16832<0>(tmp[n], a, bf, e);
        }
      }
    }
#pragma unroll
    for (int n = 0; n < NT_SP; n++) {
      acc[n][0] = fmaf(s0, tmp[n][0], acc[n][0]);
      acc[n][1] = fmaf(s0, tmp[n][1], acc[n][1]);
      acc[n][2] = fmaf(s1, tmp[n][2], acc[n][2]);
      acc[n][3] = fmaf(s1, tmp[n][3], acc[n][3]);
    }
  }
}

__device__ __forceinline__ void dense_chunk(float (&acc)[NT_DN][4], uint32_t sA, uint32_t xl, int nt, int lane) {
#pragma unroll
  for (int jj = 0; jj < 4; jj++) {
    const uint4 a0v = lds128(sA + (2 * jj) * 512 + lane * 16);
    const uint4 a1v = lds128(sA + (2 * jj + 1) * 512 + lane * 16);
    const uint32_t a0[4] = {a0v.x, a0v.y, a0v.z, a0v.w};
    const uint32_t a1[4] = {a1v.x, a1v.y, a1v.z, a1v.w};
#pragma unroll
    for (int n = 0; n < NT_DN; n++) {
      if (n < nt) {
        uint32_t bf[4];
        ldmatrix_x4(bf, xl + n * 8 * XS_DN + jj * 64);
        mma_bf16_16816(acc[n], a0, bf[0], bf[1]);
        mma_bf16_16816(acc[n], a1, bf[2], bf[3]);
      }
    }
  }
}

template <int NT>
__device__ __forceinline__ void write_partial(const float (&acc)[NT][4], float* __restrict__ P, int out, int row0,
                                              int tcount, const int* __restrict__ tok_ids, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int n = 0; n < NT; n++) {
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const int tk = n * 8 + 2 * t + (v & 1);
      const int r = row0 + g + ((v & 2) ? 8 : 0);
      if (tk < tcount && r < out) P[static_cast<int64_t>(tok_ids[tk]) * out + r] = acc[n][v];
    }
  }
}

// ------------------------------------------------------------------------------------------
// The persistent kernel
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHREADS, 1) k_sbmm(dz_sbmm_args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stages = smem_raw;
  Smem* sm = reinterpret_cast<Smem*>(smem_raw + STAGE_BYTES * NSTAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  Geo geo;
  geo.nkb = ceil_div(a.in, kBlkCols);
  geo.n16 = ceil_div(a.out, kBlkRows);
  geo.nrt = ceil_div(a.out, RT);
  const int n_items = geo.nrt * a.n_jobs;

  int* ws_i = reinterpret_cast<int*>(a.workspace);
  int* sched = ws_i;              // [0] item counter, [1] finished CTAs
  int* tile_cnt = ws_i + 64;      // [nrt] (fixed-size region: layout independent of out)
  float* Pb = reinterpret_cast<float*>(ws_i + 64 + kMaxTiles);
  float* Pd = Pb + static_cast<int64_t>(a.T) * a.out;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; s++) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ===================== producer =====================
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    while (true) {
      int item = 0;
      if (lane == 0) item = atomicAdd(&sched[0], 1);
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= n_items) break;
      const int rt = item / a.n_jobs;
      const dz_job job = a.jobs[item - rt * a.n_jobs];
      const bool dense = job_dense(job.kind);
      const uint8_t* src = static_cast<const uint8_t*>(job.kind == 0 ? a.base : a.table[job.slot].blocks);
      const int bb = blk_bytes(job.kind);
      const int nch = job_nchunks(job.kind, geo);
      const int nbmax = dense ? 1 : NB_SP;
      const int xs = dense ? XS_DN : XS_SP;
      const int aoff = dense ? A_DN : A_SP;
      int nvalid = geo.n16 - rt * NW;
      nvalid = nvalid > NW ? NW : nvalid;
      for (int ch = 0; ch < nch; ch++) {
        const int kb0 = ch * nbmax;
        const int nb = (geo.nkb - kb0) < nbmax ? (geo.nkb - kb0) : nbmax;
        mbar_wait(&sm->empty[stage], phase ^ 1);
        uint8_t* sbuf = stages + static_cast<size_t>(stage) * STAGE_BYTES;
        if (lane == 0) {
          sm->hdr[stage] = StageHdr{item, ch, nb, 0};
          const uint32_t bytes = static_cast<uint32_t>(nvalid * nb * bb + job.tok_count * nb * kBlkCols * 2);
          mbar_arrive_expect_tx(&sm->full[stage], bytes);
        }
        __syncwarp();
        if (lane < nvalid) {
          const int rg = rt * NW + lane;
          const uint8_t* s = src + (static_cast<size_t>(rg) * geo.nkb + kb0) * bb;
          tma_load_1d(sbuf + lane * nbmax * bb, s, static_cast<uint32_t>(nb * bb), &sm->full[stage], pol_stream);
        }
        for (int tk = lane; tk < job.tok_count; tk += 32) {
          const int tok = job.kind == 0 ? job.tok_begin + tk : a.order[job.tok_begin + tk];
          const uint16_t* xs_src = a.X + static_cast<int64_t>(tok) * a.ldx + kb0 * kBlkCols;
          tma_load_1d(sbuf + aoff + tk * xs, xs_src, static_cast<uint32_t>(nb * kBlkCols * 2), &sm->full[stage],
                      pol_keep);
        }
        if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
      }
    }
    mbar_wait(&sm->empty[stage], phase ^ 1);
    if (lane == 0) {
      sm->hdr[stage] = StageHdr{-1, 0, 0, 0};
      mbar_arrive(&sm->full[stage]);
      __threadfence();
      const int done = atomicAdd(&sched[1], 1);
      if (done == static_cast<int>(gridDim.x) - 1) {  // last CTA out resets the scheduler
        sched[0] = 0;
        sched[1] = 0;
      }
    }
    return;
  }

  // ===================== consumers =====================
  const int g = lane >> 2;
  float acc_d[NT_DN][4];
  float acc_s[NT_SP][4];
  int stage = 0;
  uint32_t phase = 0;
  __shared__ int tok_ids_sh[JOB_DN_TOK];
  while (true) {
    mbar_wait(&sm->full[stage], phase);
    const StageHdr h = sm->hdr[stage];
    if (h.item < 0) break;
    const int rt = h.item / a.n_jobs;
    const dz_job job = a.jobs[h.item - rt * a.n_jobs];
    const bool dense = job_dense(job.kind);
    const int rg = rt * NW + warp;
    const bool valid = rg < geo.n16;
    const uint32_t sbuf = smem_u32(stages + static_cast<size_t>(stage) * STAGE_BYTES);
    if (h.chunk == 0) {
#pragma unroll
      for (int n = 0; n < NT_DN; n++) acc_d[n][0] = acc_d[n][1] = acc_d[n][2] = acc_d[n][3] = 0.f;
#pragma unroll
      for (int n = 0; n < NT_SP; n++) acc_s[n][0] = acc_s[n][1] = acc_s[n][2] = acc_s[n][3] = 0.f;
    }
    const int nt = ceil_div(job.tok_count, 8);
    if (valid) {
      if (dense) {
        const uint32_t xl = sbuf + A_DN + (lane & 7) * XS_DN + (lane >> 3) * 16;
        dense_chunk(acc_d, sbuf + warp * kDenseBlockBytes, xl, nt, lane);
      } else {
        const uint32_t xl = sbuf + A_SP + (lane & 7) * XS_SP + (lane >> 3) * 16;
        const int qmax = a.table[job.slot].qmax;
        const uint32_t off = 0x4300u + static_cast<uint32_t>(qmax);  // bf16(128 + qmax), exact
        const uint32_t off2 = off | (off << 16);
        if (job.kind == DZ_KIND_SPARSE4)
          sparse_chunk<4>(acc_s, sbuf + warp * NB_SP * sparse_block_bytes(4), xl, h.nb, nt, off2, lane);
        else
          sparse_chunk<2>(acc_s, sbuf + warp * NB_SP * sparse_block_bytes(2), xl, h.nb, nt, off2, lane);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm->empty[stage]);
    if (++stage == NSTAGE) { stage = 0; phase ^= 1; }

    if (h.chunk == job_nchunks(job.kind, geo) - 1) {
      // ---- item epilogue: partial -> workspace, then row-tile completion ----
      const int ctid = threadIdx.x;  // 0 .. NW*32-1
      named_bar_sync(1, NW * 32);    // tok_ids_sh reuse guard
      for (int tk = ctid; tk < job.tok_count; tk += NW * 32)
        tok_ids_sh[tk] = job.kind == 0 ? job.tok_begin + tk : a.order[job.tok_begin + tk];
      named_bar_sync(1, NW * 32);
      if (valid) {
        if (dense)
          write_partial<NT_DN>(acc_d, job.kind == 0 ? Pb : Pd, a.out, rg * kBlkRows, job.tok_count, tok_ids_sh, lane);
        else
          write_partial<NT_SP>(acc_s, Pd, a.out, rg * kBlkRows, job.tok_count, tok_ids_sh, lane);
      }
      __threadfence();
      named_bar_sync(1, NW * 32);
      if (ctid == 0) {
        const int old = atomicAdd(&tile_cnt[rt], 1);
        sm->last_flag = (old == a.n_jobs - 1);
      }
      named_bar_sync(1, NW * 32);
      if (sm->last_flag) {
        __threadfence();
        const int r0 = rt * RT;
        const int nr = (a.out - r0) < RT ? (a.out - r0) : RT;
        const bool has_base = a.base != nullptr;
        for (int idx = ctid; idx < a.T * nr; idx += NW * 32) {
          const int tk = idx / nr, r = r0 + idx % nr;
          const int64_t o = static_cast<int64_t>(tk) * a.out + r;
          float y = __ldcg(Pd + o);
          if (has_base) y = __ldcg(Pb + o) + y;
          if (a.act == DZ_ACT_TANH) y = tanhf(y);
          if (a.y_dtype == DZ_F32)
            reinterpret_cast<float*>(a.Y)[static_cast<int64_t>(tk) * a.ldy + r] = y;
          else
            reinterpret_cast<__nv_bfloat16*>(a.Y)[static_cast<int64_t>(tk) * a.ldy + r] = __float2bfloat16_rn(y);
        }
        if (ctid == 0) tile_cnt[rt] = 0;  // self-reset for the next launch
      }
    }
  }
  (void)g;
}

}  // namespace dz

using namespace dz;

extern "C" size_t dz_sbmm_workspace_bytes(int32_t T, int32_t out) {
  if (T < 0 || out < 1) return 0;
  if (ceil_div(out, RT) > kMaxTiles) return 0;
  return (64 + static_cast<size_t>(kMaxTiles)) * sizeof(int) + 2 * static_cast<size_t>(T) * out * sizeof(float);
}

extern "C" int dz_sbmm(const dz_sbmm_args* a, void* stream) {
  if (!a || !a->X || !a->Y || !a->workspace) return DZ_E_VALUE;
  if (a->T < 0 || a->out < 1 || a->in < 1) return DZ_E_SHAPE;
  if (a->T == 0 || a->n_jobs == 0) return DZ_OK;
  const int in_pad = ceil_div(a->in, kBlkCols) * kBlkCols;
  if (a->ldx < in_pad || (a->ldx % 8) != 0 || (reinterpret_cast<uintptr_t>(a->X) & 15) != 0) return DZ_E_SHAPE;
  if (a->ldy < a->out) return DZ_E_SHAPE;
  if (ceil_div(a->out, RT) > kMaxTiles) return DZ_E_SHAPE;
  if (a->y_dtype != DZ_F32 && a->y_dtype != DZ_BF16) return DZ_E_VALUE;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_sbmm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return DZ_E_CUDA;
  int grid = a->grid;
  if (grid <= 0) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return DZ_E_CUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return DZ_E_CUDA;
    grid = sms;
  }
  const int n_items = ceil_div(a->out, RT) * a->n_jobs;
  if (grid > n_items) grid = n_items;
  k_sbmm<<<grid, NTHREADS, SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(*a);
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}
