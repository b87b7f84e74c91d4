// K3 — prefill SBMM on the 5th-generation tensor cores (sm_100a).
//
// Replaces inference.sbmm (inference.py:126-154) for delta groups with many tokens (prefill):
// y_t = W_base x_t + ΔW_{slot(t)} x_t, where every token of a job shares one delta. The decode
// kernel (K2) re-streams a delta per 8 tokens with legacy mma.sp; for a 256-token group that is
// 32 re-reads and a CUDA-core decode per 8 tokens. Here the delta tile is decoded ONCE per
// (row tile, job) and both products run on tcgen05:
//
//   TMEM acc[128 rows][N tokens] = Σ_k  W_base[rows, k] · X[tokens, k]ᵀ        (tcgen05, A = W tile)
//                                 + Σ_k  ΔW[rows, k]    · X[tokens, k]ᵀ        (tcgen05, A = ΔW tile)
//
// with ΔW[r][c] = bf16(code · scale) written by CUDA-core warps from the native 2:4 blocks into a
// SWIZZLE_128B K-major shared-memory tile (the layout TMA gives the W tile). The base and the
// delta products accumulate into the same fp32 TMEM tile: no partial buffers, no add kernel.
// Unlike a merged weight bf16(W + ΔW), the delta keeps its own rounding (one bf16 rounding of
// code·scale, relative 2^-9), so the fine-tune signal is not swamped by the base's quantum.
//
// Item = (128-row tile, job of <= 256 consecutive staged tokens of one delta); items are taken
// row-tile-major in a static round robin, so the W tile of a row tile is shared through L2 by the
// jobs running at the same time and the staged X of every job stays L2-resident.
//
// Warp roles (15 warps, one CTA per SM, 224 KB shared memory, 512 TMEM columns):
//  * warps 0-7  dequant: per 64-column stage, one 16-row group each: native block -> bf16 ΔW tile.
//  * warps 8-11 epilogue: TMEM lane quarter (warp % 4) -> Y rows (tcgen05.ld 32x32b), activation.
//  * warp 12    TMA producer: W tile (2-D tensor map of the base, box 64 x 128) and X tiles
//               (box 64 x 64, up to 4 per stage) into a 3-stage ring.
//  * warp 13    TMEM owner + MMA issuer: 4 K=16 MMAs of W and 4 of ΔW per stage into a
//               double-buffered accumulator (2 x 256 columns), so the epilogue of an item
//               overlaps the next item's main loop.
//  * warp 14    native-block producer: per 128 columns the row tile's native blocks (one 1-D bulk
//               copy per 16-row group) into a 4-slot ring that runs ahead of the stage ring.
#include <cuda.h>

#include <cstdint>
#include <cstdlib>

#include "dz_common.cuh"
#include "dz_tmap.h"

namespace dz {
namespace pf {

constexpr int M = 128;                      // rows per UMMA M tile
constexpr int NMAX = 256;                   // X tile rows per stage (4 TMA boxes of 64 tokens)
constexpr int NJOB = DZ_PREFILL_JOB_TOKENS; // tokens per job (UMMA N <= 256; dz_plan_mixed)
constexpr int KC = 64;                      // columns per stage (one 128-B swizzle row)
constexpr int NDQ = 8;                      // dequant warps
constexpr int NEPI = 4;                     // epilogue warps
constexpr int WARP_PROD = NDQ + NEPI;
constexpr int WARP_MMA = WARP_PROD + 1;
constexpr int WARP_DPROD = WARP_MMA + 1;    // native-block producer (runs ahead of the stage ring)
constexpr int NTHREADS = (WARP_DPROD + 1) * 32;
constexpr int RGS = M / kBlkRows;           // 8 row groups (native block rows) per M tile
constexpr int W_TILE = M * KC * 2;          // 16 KB: one W (or ΔW) tile of a stage
constexpr int XBOX = 64;                    // tokens per X TMA box
constexpr int X_BYTES = NMAX * KC * 2;      // 32 KB
constexpr int ACC_COLS = NJOB;
constexpr int TMEM_COLS = 512;
// SP: the metadata columns (4 per stage) follow the accumulator(s); with jobs of <= 240 tokens two
// accumulators still fit next to them (double-buffered), with 256-token jobs only one does.
constexpr bool SP_DOUBLE = 2 * ACC_COLS + 32 <= TMEM_COLS;
constexpr int E_COL0 = SP_DOUBLE ? 2 * ACC_COLS : ACC_COLS;
constexpr uint32_t kIdescSparse = 1u << 2;       // instruction descriptor: sparse A (2:4)

// MT = UMMA M tiles per item (rows per item = 128·MT). MT = 1: 3 stages, double-buffered TMEM
// accumulator (the epilogue overlaps the next item). MT = 2: the two M tiles share every X tile
// (half the L2 traffic per flop), 2 stages, one accumulator pair (the epilogue is exposed).
// Each output element sees the same MMA sequence either way (W k-steps then ΔW k-steps per
// stage), so the choice never changes a result bit.
// SP: the delta product runs as 2:4-sparse tcgen05 MMAs (tcgen05.mma.sp, K=32 logical per
// instruction): the dequant warps write only the kept values (bf16, compressed K-major tile) and
// the index nibbles go to TMEM as the sparse metadata. The TMEM then holds one 256-column
// accumulator (single-buffered) plus the metadata columns.
template <int MT, bool SP = false>
struct Cfg {
  static constexpr int NSTAGE = MT == 1 ? 3 : 2;
  static constexpr int NDSLOT = MT == 1 ? 4 : 2;  // native-block ring: 128-column block columns in flight
  static constexpr int NBUF = MT == 1 && (!SP || SP_DOUBLE) ? 2 : 1;
  static constexpr int W_BYTES = MT * W_TILE;
  static constexpr int DW_BYTES = SP ? MT * W_TILE / 2 : MT * W_TILE;
  static constexpr int STAGE = W_BYTES + DW_BYTES + X_BYTES;
  static constexpr int DSLOT = MT * RGS * sparse_block_bytes(4);  // one 128-column block column
  static constexpr int ROWS = MT * M;
};

template <int MT, bool SP = false>
struct Smem {
  uint64_t full[Cfg<MT, SP>::NSTAGE];    // TMA: W + X of the stage landed
  uint64_t empty[Cfg<MT, SP>::NSTAGE];   // MMA: the stage (W, ΔW, X) was consumed
  uint64_t dq[Cfg<MT, SP>::NSTAGE];      // dequant warps: ΔW tiles of the stage written
  uint64_t dfull[Cfg<MT, SP>::NDSLOT];   // TMA: native blocks of a 128-column block column landed
  uint64_t dempty[Cfg<MT, SP>::NDSLOT];  // dequant warps: done with the block column
  uint64_t tfull[2];                 // MMA: accumulator complete
  uint64_t tempty[2];                // epilogue: accumulator drained
  uint32_t tmem_base;
};
template <int MT, bool SP = false>
constexpr int smem_bytes() {
  return 1024 + Cfg<MT, SP>::NSTAGE * Cfg<MT, SP>::STAGE + Cfg<MT, SP>::NDSLOT * Cfg<MT, SP>::DSLOT +
         static_cast<int>(sizeof(Smem<MT, SP>));
}

__device__ __forceinline__ void sts64(uint32_t addr, uint32_t lo, uint32_t hi) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(lo), "r"(hi) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// byte offset of element (row, col) in a [rows][64] bf16 SWIZZLE_128B K-major tile (1024-B aligned)
__device__ __forceinline__ uint32_t sw128(int row, int col) {
  return static_cast<uint32_t>(row * 128 + ((((col >> 3) ^ row) & 7) << 4) + (col & 7) * 2);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

struct Item {
  int rt, tok_begin, tok_count, npad, slot, kind;
};

// Static round-robin schedule with a split tail: when the last round of (row tile, job) items would
// leave most CTAs idle, its items are cut into `split` (2 or 4) token slices, so the tail round
// streams the same weights with fewer tokens per CTA. Each output column's MMA sequence is the
// same whatever the slice width, so this never changes a result bit.
struct Sched {
  int tail0, split, n_items;
};
__device__ __forceinline__ Sched make_sched(int n_full, int grid) {
  Sched sc;
  const int tail = n_full % grid;
  int split = 1;
  if (tail)
    while (split < 4 && tail * split * 2 <= grid) split *= 2;
  sc.split = split;
  sc.tail0 = split > 1 ? n_full - tail : n_full;
  sc.n_items = sc.tail0 + (n_full - sc.tail0) * split;
  return sc;
}

__device__ __forceinline__ Item item_at(const dz_sbmm_args& a, int item, int n_jobs, const Sched& sc) {
  int base = item, part = 0;
  if (item >= sc.tail0) {
    const int j = item - sc.tail0;
    base = sc.tail0 + j / sc.split;
    part = j - (j / sc.split) * sc.split;
  }
  Item it;
  it.rt = base / n_jobs;
  const dz_job jb = a.jobs[base - it.rt * n_jobs];
  int b0 = 0, cnt = jb.tok_count;
  if (item >= sc.tail0) {
    const int ps = ((jb.tok_count + sc.split - 1) / sc.split + 15) & ~15;
    b0 = part * ps;
    cnt = max(0, min(jb.tok_count, b0 + ps) - b0);
  }
  it.tok_begin = jb.tok_begin + b0;
  it.tok_count = cnt;
  it.npad = (cnt + 15) & ~15;
  it.slot = jb.slot;
  it.kind = jb.kind;
  return it;
}

// Dequantise the 64-column half `h` of the current block column for row groups rg0, rg0+1 of the
// item into the stage's ΔW tile. Native block layout: dz_codec.cu (k_repack_sparse).
template <int FB, int NRG>
__device__ __forceinline__ void dequant_half(uint32_t dw, uint32_t dslot, int rg0, int n_valid, int h, int qmax,
                                             int lane) {
  constexpr int CODE = sparse_code_bytes(FB);
  constexpr int BB = sparse_block_bytes(FB);
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int m = 0; m < NRG; m++) {
    const int rgl = rg0 + m;
    const bool valid = rgl < n_valid;  // warp-uniform
    const uint32_t blk = dslot + rgl * BB;
    uint2 meta = make_uint2(0x44444444u, 0x44444444u);
    float sA = 0.f, sB = 0.f;
    if (valid) {
      meta = lds64(blk + CODE + lane * 8);
      const uint2 sv = lds64(blk + CODE + kMetaBytes + g * 8);
      sA = __uint_as_float(sv.x);
      sB = __uint_as_float(sv.y);
    }
    const uint32_t mw = h ? meta.y : meta.x;  // word i>>1 == h for MMAs i = 2h, 2h+1
#pragma unroll
    for (int ii = 0; ii < 2; ii++) {
      const int i = 2 * h + ii;
      // E(MMA i, half hh) lives in lane 4g + 2(i&1) + hh (see k_repack_sparse)
      const uint32_t e0 = __shfl_sync(0xffffffffu, mw, 4 * g + 2 * ii + 0);
      const uint32_t e1 = __shfl_sync(0xffffffffu, mw, 4 * g + 2 * ii + 1);
      uint32_t u[8];
      if (FB == 4) {
        const uint32_t w = valid ? lds32(blk + lane * 16 + i * 4) : 0x77777777u;
#pragma unroll
        for (int k = 0; k < 8; k++) u[k] = (w >> (4 * k)) & 0xFu;
      } else {
        const uint32_t w = valid ? lds32(blk + lane * 8 + h * 4) : 0x55555555u;
        const int o = 4 * ii;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          u[k] = (w >> (2 * (o + k))) & 3u;
          u[k + 4] = (w >> (2 * (o + k + 8))) & 3u;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int r = g + ((k & 1) ? 8 : 0);
        const int slot = t + ((k & 2) ? 4 : 0);
        const uint32_t e = (slot >> 2) ? e1 : e0;
        const uint32_t nib = (e >> (((k & 1) ? 16 : 0) + 4 * (slot & 3))) & 0xFu;
        const float s = (k & 1) ? sB : sA;
        const float v0 = static_cast<float>(static_cast<int>(u[k]) - qmax) * s;
        const float v1 = static_cast<float>(static_cast<int>(u[k + 4]) - qmax) * s;
        const int p0 = nib & 3, p1 = nib >> 2;
        const float c0 = p0 == 0 ? v0 : 0.f, c1 = p0 == 1 ? v0 : (p1 == 1 ? v1 : 0.f);
        const float c2 = p0 == 2 ? v0 : (p1 == 2 ? v1 : 0.f), c3 = p1 == 3 ? v1 : 0.f;
        const int row = kBlkRows * rgl + r;
        const int col = 32 * ii + 4 * slot;
        sts64(dw + sw128(row, col), pack_bf16(c0, c1), pack_bf16(c2, c3));
      }
    }
  }
}

// SP: kept values only. Row group rg (16 rows) of the 64-column half `h` of the block column into the
// compressed K-major tile (32 bf16 per row; element (r, c) at (r/8)*512 + (c/8)*128 + (r%8)*16 +
// (c%8)*2). Group j of a row keeps (first, second) at compressed columns (2j, 2j+1), the order of
// the index nibble (p0 < p1), which the metadata in TMEM describes.
template <int FB>
__device__ __forceinline__ void dequant_half_sp(uint32_t dw, uint32_t dslot, int rg, int n_valid, int h, int qmax,
                                                int lane) {
  constexpr int BB = sparse_block_bytes(FB);
  constexpr int CODE = sparse_code_bytes(FB);
  const int g = lane >> 2, t = lane & 3;
  const bool valid = rg < n_valid;  // warp-uniform
  const uint32_t blk = dslot + rg * BB;
  float sA = 0.f, sB = 0.f;
  if (valid) {
    const uint2 sv = lds64(blk + CODE + kMetaBytes + g * 8);
    sA = __uint_as_float(sv.x);
    sB = __uint_as_float(sv.y);
  }
#pragma unroll
  for (int ii = 0; ii < 2; ii++) {
    const int i = 2 * h + ii;
    uint32_t u[8];
    if (FB == 4) {
      const uint32_t w = valid ? lds32(blk + lane * 16 + i * 4) : 0x77777777u;
#pragma unroll
      for (int k = 0; k < 8; k++) u[k] = (w >> (4 * k)) & 0xFu;
    } else {
      const uint32_t w = valid ? lds32(blk + lane * 8 + h * 4) : 0x55555555u;
      const int o = 4 * ii;
#pragma unroll
      for (int k = 0; k < 4; k++) {
        u[k] = (w >> (2 * (o + k))) & 3u;
        u[k + 4] = (w >> (2 * (o + k + 8))) & 3u;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int row = kBlkRows * rg + g + ((k & 1) ? 8 : 0);
      const int slot = t + ((k & 2) ? 4 : 0);
      const float sc = (k & 1) ? sB : sA;
      const float v0 = static_cast<float>(static_cast<int>(u[k]) - qmax) * sc;
      const float v1 = static_cast<float>(static_cast<int>(u[k + 4]) - qmax) * sc;
      const int c = 16 * ii + 2 * slot;  // compressed column
      const uint32_t addr = dw + (row >> 3) * 512 + (c >> 3) * 128 + (row & 7) * 16 + (c & 7) * 2;
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(pack_bf16(v0, v1)) : "memory");
    }
  }
}

template <int MT, bool SP>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_prefill(const __grid_constant__ dz_sbmm_args a, const __grid_constant__ CUtensorMap xmap) {
  using C = Cfg<MT, SP>;
  constexpr int NSTAGE = C::NSTAGE, STAGE = C::STAGE, DSLOT = C::DSLOT, W_BYTES = C::W_BYTES;
  constexpr int DW_BYTES = C::DW_BYTES, NBUF = C::NBUF, IRG = MT * RGS;  // row groups per item
  constexpr int NDSLOT = C::NDSLOT;
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* stages = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
  uint8_t* dslots = stages + NSTAGE * STAGE;
  Smem<MT, SP>* sm = reinterpret_cast<Smem<MT, SP>*>(dslots + NDSLOT * DSLOT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int n_jobs = a.n_pf_jobs;
  if (a.pf_counts_dev != nullptr) {  // device mixed plan: the count is the planner's output
    griddep_wait();
    n_jobs = a.pf_counts_dev[0];
  }
  const int nrt = ceil_div(a.out, C::ROWS);
  const Sched sc = make_sched(nrt * n_jobs, static_cast<int>(gridDim.x));
  const int n_items = sc.n_items;
  const int nch = ceil_div(a.in, KC);
  const int nkb = ceil_div(a.in, kBlkCols);
  const int n16 = ceil_div(a.out, kBlkRows);
  const bool has_base = a.base != nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; s++) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->empty[s], 1);
      mbar_init(&sm->dq[s], NDQ);
    }
    for (int s = 0; s < NDSLOT; s++) {
      mbar_init(&sm->dfull[s], 1);
      mbar_init(&sm->dempty[s], NDQ);
    }
    for (int b = 0; b < NBUF; b++) {
      mbar_init(&sm->tfull[b], 1);
      mbar_init(&sm->tempty[b], NEPI);
    }
    fence_mbar_init();
  }
  if (warp == WARP_MMA) {
    tmem_alloc(&sm->tmem_base, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = sm->tmem_base;

  if (warp == WARP_PROD) {
    // ===================== TMA producer (W and X tiles) =====================
    const uint64_t pol_keep = policy_evict_last();
    if (lane == 0) prefetch_tmap(&xmap);
    griddep_wait();  // the staged X is the preceding kernel's output (programmatic dependent launch)
    griddep_launch_dependents();
    int s = 0;
    uint32_t ph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const Item it = item_at(a, item, n_jobs, sc);
      if (it.tok_count == 0) continue;  // empty tail slice (same decision in every role)
      const int nxb = ceil_div(it.npad, XBOX);
      const int ntile = min(MT, ceil_div(a.out - it.rt * C::ROWS, M));  // W tiles inside `out`
      for (int ch = 0; ch < nch; ch++) {
        mbar_wait(&sm->empty[s], ph ^ 1);
        if (lane == 0) {
          uint8_t* sb = stages + s * STAGE;
          mbar_arrive_expect_tx(&sm->full[s], (has_base ? ntile * W_TILE : 0) + nxb * XBOX * KC * 2);
          if (has_base)
            for (int h = 0; h < ntile; h++)
              tma_load_2d(sb + h * W_TILE, a.base->tmap, ch * KC, it.rt * C::ROWS + h * M, &sm->full[s], pol_keep);
          for (int b = 0; b < nxb; b++)
            tma_load_2d(sb + W_BYTES + DW_BYTES + b * XBOX * KC * 2, &xmap, ch * KC, it.tok_begin + b * XBOX,
                        &sm->full[s], pol_keep);
        }
        __syncwarp();
        if (++s == NSTAGE) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == WARP_DPROD) {
    // ===================== native-block producer =====================
    // Per 128-column block column, the item's native blocks (one 1-D bulk copy per 16-row group)
    // into an NDSLOT-deep ring, independent of the W/X stage ring so the delta stream runs ahead.
    const uint64_t pol_stream = policy_evict_first();
    int ds = 0;
    uint32_t dph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const Item it = item_at(a, item, n_jobs, sc);
      if (it.tok_count == 0) continue;
      const uint8_t* blocks = static_cast<const uint8_t*>((a.table + it.slot)->blocks);
      const int bb = sparse_block_bytes(kind_fbits(it.kind));
      const int nrg = min(IRG, n16 - it.rt * IRG);
      for (int kb = 0; kb < ceil_div(nch, 2); kb++) {
        mbar_wait(&sm->dempty[ds], dph ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&sm->dfull[ds], static_cast<uint32_t>(nrg * bb));
        __syncwarp();
        if (lane < nrg)
          tma_load_1d(dslots + ds * DSLOT + lane * bb,
                      blocks + (static_cast<int64_t>(it.rt * IRG + lane) * nkb + kb) * bb, static_cast<uint32_t>(bb),
                      &sm->dfull[ds], pol_stream);
        if (++ds == NDSLOT) { ds = 0; dph ^= 1; }
      }
    }
  } else if (warp == WARP_MMA) {
    // ===================== tcgen05 issuer =====================
    int s = 0, nacc = 0;
    uint32_t ph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const Item it = item_at(a, item, n_jobs, sc);
      if (it.tok_count == 0) continue;  // empty tail slice (same decision in every role)
      const int buf = NBUF == 1 ? 0 : (nacc & 1);
      const uint32_t tph = NBUF == 1 ? (nacc & 1) : ((nacc >> 1) & 1);
      mbar_wait(&sm->tempty[buf], tph ^ 1);
      tc_fence_after();
      const uint32_t idesc = umma_idesc_bf16(M, it.npad);
      for (int ch = 0; ch < nch; ch++) {
        mbar_wait(&sm->full[s], ph);
        mbar_wait(&sm->dq[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sb = smem_u32(stages + s * STAGE);
          const uint64_t xdesc = umma_desc_sw128(sb + W_BYTES + DW_BYTES);
          if (has_base) {
#pragma unroll
            for (int h = 0; h < MT; h++) {
              const uint64_t wdesc = umma_desc_sw128(sb + h * W_TILE);
              const uint32_t tmem_d = tmem_base + (buf * MT + h) * ACC_COLS;
#pragma unroll
              for (int k = 0; k < KC / 16; k++)
                umma_bf16(tmem_d, wdesc + 2 * k, xdesc + 2 * k, idesc, (ch | k) ? 1u : 0u);
            }
          }
          if constexpr (SP) {
            // compressed ΔW tile (no swizzle, [8-row group][16-B chunk][8 x 16 B]: SBO 512, LBO 128)
            // x X: 2 sparse MMAs of K=32 logical; metadata column per MMA (E_COL0 + 4 s + ii)
            const uint32_t tmem_d = tmem_base + buf * ACC_COLS;
#pragma unroll
            for (int ii = 0; ii < KC / 32; ii++)
              // metadata address: the even column of the stage; sparse_id2 (idesc bits 0-1) = ii selects
              // the column of this MMA (CUTLASS mma_traits_sm100: id2 = tmem_e & 1)
              umma_sp_bf16(tmem_d, umma_desc_interleave(sb + W_BYTES + ii * 256, 128, 512), xdesc + 4 * ii,
                           tmem_base + E_COL0 + 4 * s, idesc | kIdescSparse | static_cast<uint32_t>(ii),
                           (has_base || (ch | ii)) ? 1u : 0u);
          } else {
#pragma unroll
            for (int h = 0; h < MT; h++) {
              const uint64_t ddesc = umma_desc_sw128(sb + W_BYTES + h * W_TILE);
              const uint32_t tmem_d = tmem_base + (buf * MT + h) * ACC_COLS;
#pragma unroll
              for (int k = 0; k < KC / 16; k++)
                umma_bf16(tmem_d, ddesc + 2 * k, xdesc + 2 * k, idesc, (has_base || (ch | k)) ? 1u : 0u);
            }
          }
          umma_commit(&sm->empty[s]);
          if (ch == nch - 1) umma_commit(&sm->tfull[buf]);
        }
        __syncwarp();
        if (++s == NSTAGE) { s = 0; ph ^= 1; }
      }
      nacc++;
    }
  } else if (warp < NDQ) {
    // ===================== dequant warps =====================
    int s = 0, ds = 0;
    uint32_t ph = 0, dph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const Item it = item_at(a, item, n_jobs, sc);
      if (it.tok_count == 0) continue;  // empty tail slice (same decision in every role)
      const int nrg = min(IRG, n16 - it.rt * IRG);
      const int qmax = kind_qmax(it.kind);
      const bool two_bit = it.kind == DZ_KIND_SPARSE2;
      const int bb = sparse_block_bytes(kind_fbits(it.kind));
      for (int ch = 0; ch < nch; ch++) {
        if ((ch & 1) == 0) mbar_wait(&sm->dfull[ds], dph);
        mbar_wait(&sm->empty[s], ph ^ 1);  // the MMAs that last read these ΔW tiles are done
        if constexpr (SP) {
          // kept values of row group `warp` -> compressed tile; warps 0-3 also write the metadata of
          // row groups 2q, 2q+1 into their TMEM lane quarter (lane = g + 8 h + 16 rg, column = MMA)
          const uint32_t dw = smem_u32(stages + s * STAGE + W_BYTES);
          const uint32_t dsl = smem_u32(dslots + ds * DSLOT);
          if (two_bit)
            dequant_half_sp<2>(dw, dsl, warp, nrg, ch & 1, qmax, lane);
          else
            dequant_half_sp<4>(dw, dsl, warp, nrg, ch & 1, qmax, lane);
          if (warp < 4) {
            const int rgm = 2 * warp + (lane >> 4), g = lane & 7, hh = (lane >> 3) & 1, h = ch & 1;
            uint32_t e0 = 0x44444444u, e1 = 0x44444444u;
            if (rgm < nrg) {
              const uint32_t mb = dsl + rgm * bb + (two_bit ? sparse_code_bytes(2) : sparse_code_bytes(4));
              e0 = lds32(mb + (4 * g + 0 + hh) * 8 + h * 4);  // MMA i = 2h     (i & 1 = 0)
              e1 = lds32(mb + (4 * g + 2 + hh) * 8 + h * 4);  // MMA i = 2h + 1 (i & 1 = 1)
            }
            tmem_st2(tmem_base + (static_cast<uint32_t>(32 * warp) << 16) + E_COL0 + 4 * s, e0, e1);
            tmem_st_wait();
          }
          tc_fence_before();
        } else {
          // warp w covers RPW consecutive row groups of the item (within one M tile)
          constexpr int RPW = IRG / NDQ;
          const int rg = RPW * warp, tile = rg / RGS;
          const uint32_t dw = smem_u32(stages + s * STAGE + W_BYTES + tile * W_TILE);
          const uint32_t dsl = smem_u32(dslots + ds * DSLOT) + tile * RGS * bb;
          if (two_bit)
            dequant_half<2, RPW>(dw, dsl, rg - tile * RGS, nrg - tile * RGS, ch & 1, qmax, lane);
          else
            dequant_half<4, RPW>(dw, dsl, rg - tile * RGS, nrg - tile * RGS, ch & 1, qmax, lane);
        }
        fence_proxy_async();  // generic-proxy st.shared -> visible to the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm->dq[s]);
        if ((ch & 1) == 1 || ch == nch - 1) {
          if (lane == 0) mbar_arrive(&sm->dempty[ds]);
          if (++ds == NDSLOT) { ds = 0; dph ^= 1; }
        }
        if (++s == NSTAGE) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ===================== epilogue warps =====================
    const int q = warp & 3;
    griddep_wait();  // Y rows may still be written by the preceding kernel
    int nacc = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const Item it = item_at(a, item, n_jobs, sc);
      if (it.tok_count == 0) continue;  // empty tail slice (same decision in every role)
      const int buf = NBUF == 1 ? 0 : (nacc & 1);
      mbar_wait(&sm->tfull[buf], NBUF == 1 ? (nacc & 1) : ((nacc >> 1) & 1));
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < MT * (it.npad / 16); cc++) {
        const int h = cc / (it.npad / 16), c = cc - h * (it.npad / 16);
        const int row = it.rt * C::ROWS + h * M + 32 * q + lane;
        const uint32_t taddr = tmem_base + (buf * MT + h) * ACC_COLS + (static_cast<uint32_t>(32 * q) << 16);
        uint32_t v[16];
        tmem_ld16(taddr + c * 16, v);
        const int i0 = it.tok_begin + c * 16;
        int yr = i0 + (lane & 15);
        if (a.perm != nullptr && c * 16 + (lane & 15) < it.tok_count) yr = a.perm[yr];
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int yrow = __shfl_sync(0xffffffffu, yr, j);
          if (c * 16 + j < it.tok_count && row < a.out) {
            float y = __uint_as_float(v[j]);
            if (a.act == DZ_ACT_TANH) y = tanhf(y);
            const int64_t yo = static_cast<int64_t>(yrow) * a.ldy + row;
            if (a.y_dtype == DZ_F32)
              reinterpret_cast<float*>(a.Y)[yo] = y;
            else
              reinterpret_cast<__nv_bfloat16*>(a.Y)[yo] = __float2bfloat16_rn(y);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm->tempty[buf]);
      nacc++;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// Staging gather: Xs[i] = X[perm[i]], 16 B per thread.
__global__ void k_gather_rows(const uint16_t* __restrict__ X, int64_t ldx, const int32_t* __restrict__ perm, int T,
                              int in8, uint16_t* __restrict__ Xs, int64_t ldxs) {
  const int64_t n = static_cast<int64_t>(T) * in8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / in8), c = static_cast<int>(i - static_cast<int64_t>(r) * in8);
    const int src = __ldg(perm + r);
    reinterpret_cast<uint4*>(Xs + r * ldxs)[c] = __ldg(reinterpret_cast<const uint4*>(X + src * ldx) + c);
  }
}

}  // namespace pf
}  // namespace dz

using namespace dz;

static_assert(pf::smem_bytes<1>() <= 232448 && pf::smem_bytes<2>() <= 232448 && pf::smem_bytes<1, true>() <= 232448,
              "prefill kernel shared memory");
static_assert(pf::Cfg<1>::STAGE % 1024 == 0 && pf::Cfg<2>::STAGE % 1024 == 0 && pf::W_TILE % 1024 == 0,
              "SW128 tile alignment");

extern "C" int dz_gather_rows(const uint16_t* X, int64_t ldx, const int32_t* perm, int32_t T, int32_t in,
                              uint16_t* Xs, int64_t ldxs, void* stream) {
  if (T < 0 || in < 1) return DZ_E_SHAPE;
  if (!X || !perm || !Xs) return DZ_E_VALUE;
  if ((ldx % 8) || (ldxs % 8) || (reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(Xs) & 15))
    return DZ_E_SHAPE;
  if (T == 0) return DZ_OK;
  if (ldx < in || ldxs < in) return DZ_E_SHAPE;
  const int in8 = ceil_div(in, 8);  // callers pass in = the padded width (zero tail kept)
  const int64_t n = static_cast<int64_t>(T) * in8;
  const int blocks = static_cast<int>((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
  pf::k_gather_rows<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(X, ldx, perm, T, in8, Xs, ldxs);
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}

template <int MT, bool SP>
static int launch_prefill(const dz_sbmm_args& k, const CUtensorMap& xmap, int grid, void* stream) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(pf::k_prefill<MT, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    pf::smem_bytes<MT, SP>());
  });
  if (attr_err != cudaSuccess) return DZ_E_CUDA;
  return launch_pdl(1, pf::k_prefill<MT, SP>, grid, pf::NTHREADS, pf::smem_bytes<MT, SP>(), stream, k, xmap);
}

// Launch K3 over jobs[0:n_pf_jobs]; X is the staged buffer (dz_sbmm passes it as X).
// Items of 128 or 256 rows: the one with fewer item rounds per SM, weighted by the measured
// per-item efficiency (MT=2 shares each X tile between two M tiles). Results are identical.
extern "C" int dz_sbmm_prefill(const dz_sbmm_args* a, void* stream) {
  if (!a) return DZ_E_VALUE;
  if (a->T < 0 || a->out < 1 || a->in < 1) return DZ_E_SHAPE;
  if (a->n_pf_jobs <= 0 || a->T == 0) return DZ_OK;  // nothing to compute
  if (!a->Y || !a->table || !a->jobs) return DZ_E_VALUE;
  const uint16_t* X = a->X;  // the staged buffer (dz_sbmm passes it as X with its row stride)
  if (!X) return DZ_E_VALUE;
  if ((a->ldx % 8) != 0 || (reinterpret_cast<uintptr_t>(X) & 15) != 0 || a->ldx < a->in) return DZ_E_SHAPE;
  if (a->y_dtype != DZ_F32 && a->y_dtype != DZ_BF16) return DZ_E_VALUE;
  CUtensorMap xmap;  // staged X [T][in] bf16, 64-column x 64-token SWIZZLE_128B boxes (UMMA B operand)
  const int st = encode_2d(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, X, static_cast<uint64_t>(a->in),
                           static_cast<uint64_t>(a->T), static_cast<uint64_t>(a->ldx) * 2, pf::KC, pf::XBOX,
                           CU_TENSOR_MAP_SWIZZLE_128B);
  if (st) return st;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DZ_E_CUDA;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return DZ_E_CUDA;
  const int g = a->grid > 0 ? a->grid : sms;
  const int items1 = ceil_div(a->out, pf::M) * a->n_pf_jobs;
  const int items2 = ceil_div(a->out, 2 * pf::M) * a->n_pf_jobs;
  // time ~ rounds x rows per item / per-item efficiency. Measured (profiles/r01_pf_mt.txt): MT=2 is
  // 7-33% slower at every 13B shape (2-stage ring, exposed epilogue), so MT=1 unless overridden.
  const double t1 = ceil_div(items1, g) * 1.0 / 0.75, t2 = ceil_div(items2, g) * 2.0 / 0.62;
  // 2:4-sparse tcgen05 delta product by default (8-23% faster than the dense-dequantised one at the
  // 13B shapes, profiles/r01_pf_sparse.txt); args.prefill_variant selects the dense-dequantised
  // delta product with 128-row (1) or 256-row (2) items for A/B runs and the equivalence tests.
  if (a->prefill_variant < 0 || a->prefill_variant > 2) return DZ_E_VALUE;
  int mt = t2 < t1 ? 2 : 1;
  if (a->prefill_variant > 0) mt = a->prefill_variant;
  const int n_items = mt == 2 ? items2 : items1;
  const int grid = g > n_items ? n_items : g;
  if (a->prefill_variant == 0 && mt == 1) return launch_prefill<1, true>(*a, xmap, grid, stream);
  return mt == 2 ? launch_prefill<2, false>(*a, xmap, grid, stream) : launch_prefill<1, false>(*a, xmap, grid, stream);
}
