// K2 — fused base GEMM + selective batched (2:4, low-bit) delta matmul for sm_100a (decode regime).
//
// Replaces inference.sbmm (inference.py:126-154): y_t = W_base x_t + ΔW_{slot(t)} x_t.
//
// Work decomposition. An item is (row tile, job); a job is either the base GEMM for up to 128
// tokens (row tile = 128 rows, one UMMA M tile) or one delta group for up to 8 or 16 (2:4 sparse:
// the plan's job width, one kernel instantiation each) / 32 (dense) of its tokens (row tile = 256
// rows; dz_plan = group_by_delta, inference.py:106-123).
// Base items come first, then delta items row-tile-major; one persistent CTA per SM pulls items
// from a self-resetting atomic counter with one item of lookahead.
//
// Warp roles per CTA (11 warps):
//  * TMA producer (1 warp): per stage ONE tensor copy of the A operand — two (three when the
//    launch has <= 32 tokens) 64-col x 128-row SWIZZLE_128B tiles of the base W in its natural
//    layout, or a 3-D box of 4 native blocks x 16 row groups of a delta (53 KB) — plus, for base
//    stages, the swizzled X tile (bn = 128 or 32 contiguous token rows, OOB rows zero-filled). 3-deep ring with full/empty mbarriers; the next item's id, descriptor
//    and token ids are prefetched while the current item streams.
//  * X producer (1 warp): one 1-D bulk copy per routed token row of a delta stage.
//  * MMA issuer (1 warp, one elected thread): base stages become tcgen05.mma kind::f16 (M=128,
//    N=bn tokens, K=16 per MMA) into a double-buffered TMEM accumulator; tcgen05.commit
//    frees the stage and, on the last chunk, signals the accumulator full.
//  * consumers (8 warps, two 16-row groups each): 2:4 delta stages — decode codes in registers
//    (LOP3 magic-number bf16 conversion; deferred per-(row,128-col) scaling) and mma.sp m16n8k32
//    (the reference's index nibble IS the sparse-MMA metadata), fp32 accumulation; dense-delta
//    stages use mma m16n8k16. They also drain the base accumulator from TMEM (tcgen05.ld).
//
// Merge: every contributor of y[t][r] — the base job's K-split s, the token's delta job — stores its
// fp32 partial with a plain store into its own plane of the workspace (exactly one writer per
// element, no atomics on data). Two ways to finish (dz_sbmm_args.fused_merge):
//  * default: k_finalize (one short launch) sums the planes in a fixed order and writes Y;
//  * fused (k_sbmm<true>): a 12th "combiner" warp per CTA writes Y for each delta item's tokens
//    once the base partials of its rows are published (per-32-row-slice counters), so no second
//    launch. Measured 1-3% slower on the 7B step and 5-20% slower at cfg5 points than the
//    k_finalize path on the same box (profiles/r02_ab_fused_merge.txt, r02_ab_chain.txt), hence
//    opt-in. The same body also runs a whole decode step as one chained launch (k_sbmm_chain).
// Both are deterministic and batch-invariant: the summation order is fixed per element.
//
// Mixed batches: groups large enough for the tensor-core prefill kernel (K3, dz_prefill.cu) are
// staged first in a permuted copy of X; this kernel then covers the remaining (decode) rows and
// writes row i of the staged X to Y row perm[i].
#include <cuda.h>

#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "dz_common.cuh"
#include "dz_tmap.h"

#ifdef DZ_TRACE
// Per-warp private event slots of the traced CTA (the one that took item 0): plain stores, no
// atomics, so tracing does not perturb the pipeline. Slot [warp][i] = {globaltimer, ev|a0|a1}.
__device__ unsigned long long dz_trace_buf[12][1024][2];
__device__ int dz_trace_cnt[12];
__device__ volatile int dz_trace_cta = -1;
__device__ unsigned long long dz_item_trace[65536][3];  // per item: start, end, (cta << 32 | kind)
#define ITEM_TRACE(slot, item, val) do { if ((item) < 65536) dz_item_trace[(item)][(slot)] = (val); } while (0)
#define TRACE(ev, a0, a1) do { if (blockIdx.x == 0 && trace_i < 1024) { \
  dz_trace_buf[threadIdx.x >> 5][trace_i][0] = clock64(); \
  dz_trace_buf[threadIdx.x >> 5][trace_i][1] = (static_cast<unsigned long long>(ev) << 56) | \
      (static_cast<unsigned long long>(static_cast<uint32_t>(a0)) << 16) | static_cast<uint16_t>(a1); \
  trace_i++; dz_trace_cnt[threadIdx.x >> 5] = trace_i; } } while (0)
#else
#define TRACE(ev, a0, a1) do {} while (0)
#define ITEM_TRACE(slot, item, val) do {} while (0)
#endif

namespace dz {

constexpr int NW = 8;                     // consumer warps per CTA (one CTA per SM); 16 measured -1.5%
constexpr int MR = 16 / NW;               // 16-row groups per consumer warp (RG = 16 per item)
constexpr int WARP_PROD = NW;             // TMA producer warp
constexpr int WARP_MMA = NW + 1;          // tcgen05 issuer / TMEM owner warp
constexpr int WARP_XPROD = NW + 2;        // per-token X copies of delta stages
constexpr int WARP_COMB = NW + 3;         // fused-merge instantiation only: combines delta items into Y
constexpr int NTHREADS = (NW + 3) * 32;   // k_sbmm<false>; k_sbmm<true> has one more warp
template <bool FUSED>
constexpr int nthreads() { return FUSED ? NTHREADS + 32 : NTHREADS; }
constexpr int RG = NW * MR;               // row groups per item
constexpr int RT = RG * kBlkRows;         // rows per item (256) == 2 x UMMA M
constexpr int UMMA_M = 128;
#ifndef DZ_SHIFT_FMA
#define DZ_SHIFT_FMA 0  // 1: code-field shifts on the FMA pipe (IMAD.HI); measured 15% slower (ab_shift)
#endif
#ifndef DZ_NB_SP
#define DZ_NB_SP 4
#endif
#ifndef DZ_DRAIN_BATCH
#define DZ_DRAIN_BATCH 1  // base drain: two TMEM loads per wait (+0.5-1.4%, profiles/r01_ab_drain.txt)
#endif
#ifndef DZ_PAIR_UNROLL
#define DZ_PAIR_UNROLL 1  // unroll the block-pair loop of a full sparse chunk (+2.6-3.0%, profiles/r01_ab_pair.txt)
#endif
#ifndef DZ_NSTAGE
#define DZ_NSTAGE 3
#endif
constexpr int NB_SP = DZ_NB_SP;           // sparse chunk = 4 blocks = 512 columns (one 3-D TMA box)
constexpr int NT_SP = DZ_SPARSE_JOB_TOKENS / 8;  // most n-tiles per 2:4 job (dz_plan): the codes of a
                                                 // chunk are decoded once for all of the job's tokens
constexpr int NT_DN = 4;                  // n-tiles per dense-delta job (32 tokens, dz_plan)
constexpr int KC_DN = 64;                 // dense / base chunk = 64 columns
constexpr int BASE_N = DZ_BASE_JOB_TOKENS; // most tokens per base job (dz_plan's cut) = TMEM buffer stride
constexpr int XS_SP = NB_SP * kBlkCols * 2 + 16;  // smem bytes per staged token row; +16 B so the
constexpr int XS_DN = KC_DN * 2 + 16;             //   8 rows of an ldmatrix hit distinct banks
constexpr int A_SP = RG * NB_SP * sparse_block_bytes(4);  // 53248
template <int NTS>
constexpr int x_sp() { return NTS * 8 * XS_SP; }          // 8320 per 8 tokens
constexpr int DN_HALF = kDenseBlockBytes / 2;             // 2048
constexpr int A_DN = RG * DN_HALF;                        // 32768 == 256 rows x 128 B (base W tile)
constexpr int X_DN = 64 * XS_DN;                          // 9216 (>= 64 x 128 B swizzled X tile)
__host__ __device__ constexpr int cmax(int x, int y) { return x > y ? x : y; }
__host__ __device__ constexpr int cmin(int x, int y) { return x < y ? x : y; }
constexpr int NSTAGE = DZ_NSTAGE;
constexpr int JOB_DN_TOK = BASE_N;        // largest token count of a job
constexpr int BASE_RT = UMMA_M;           // rows per base item: one UMMA M tile (half a delta row tile)
constexpr int SPLIT_CH = 2;               // base K-splits fall on 2-chunk (128-column) boundaries
constexpr int TMEM_COLS = 2 * BASE_N;     // double-buffered fp32 accumulator, 128 lanes x 128 tokens
// Base stage shape of a launch, from its token count T only (so never from the batch's composition):
// UMMA N = bn (the X tile holds bn token rows) and bch 64-column K-chunks per stage. A narrow X tile
// (T <= 32) leaves room for 3 W chunks, 48 KB of W in flight per stage instead of 32 KB. The
// accumulation order of a token is the same for every (bn, bch): K-chunks in order, splits on
// SPLIT_CH-chunk boundaries (profiles/r02_ab_base_n.txt).
#ifndef DZ_BASE_BN64
#define DZ_BASE_BN64 0  // bn = 64 for 32 < T <= 64: measured -1% on the 7B step (T = 64), off
#endif
__host__ __device__ constexpr int base_bn(int T) {
  return T <= 32 ? cmin(32, BASE_N) : (DZ_BASE_BN64 && T <= 64) ? cmin(64, BASE_N) : BASE_N;
}
__host__ __device__ constexpr int base_bch(int bn) { return bn <= 32 ? 3 : 2; }
__host__ __device__ constexpr int base_xoff(int bch) { return cmax(A_DN, bch * UMMA_M * KC_DN * 2); }
__host__ __device__ constexpr int base_stage_bytes(int bn) {
  return base_xoff(base_bch(bn)) + base_bch(bn) * KC_DN * bn * 2;
}
// Stage size of the instantiation for 2:4 jobs of up to NTS n-tiles (X rows staged per stage).
template <int NTS>
constexpr int stage_bytes() {
  return (cmax(cmax(cmax(A_SP + x_sp<NTS>(), A_DN + X_DN), base_stage_bytes(BASE_N)),
               cmax(base_stage_bytes(32), base_stage_bytes(64))) + 1023) / 1024 * 1024;
}
constexpr int PF_CHUNKS = 4;              // stages of the first item prefetched into L2 before the PDL wait
// Workspace: [0, 256) scheduler words; [256, +4*MAX_SLICES) per-32-row-slice arrival counters;
// then the fp32 partial planes [base K-splits + delta K-splits][T][out].
constexpr int MAX_SLICES = 8192;          // out <= 262144 rows per launch
constexpr int MAX_CHAIN = 256;            // linears per chained launch
constexpr int DZ_WS_CNT_OFF = 256;
constexpr int DZ_WS_CHAIN_OFF = DZ_WS_CNT_OFF + 4 * MAX_SLICES;  // [exit count][item counters][done counts]
constexpr int DZ_WS_PART_OFF = DZ_WS_CHAIN_OFF + 4 * (1 + 2 * MAX_CHAIN) + 252;

struct StageHdr {
  int item;       // -1: end of work
  int rt;         // row tile
  int kind;       // 0 base, DZ_KIND_*
  int tok_begin;
  int tok_count;
  int nb;         // sparse: blocks in chunk; dense: 1
  int flags;      // bit0: first chunk, bit1: last chunk
  int pad;        // K-split of the item
  int lin;        // linear of a chained launch (0 otherwise)
};

struct Smem {
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  uint64_t xreq[NSTAGE];   // producer -> X producer: header + token ids of the stage are written
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  StageHdr hdr[NSTAGE];
  uint64_t mfull[8];       // consumer warps -> combiner: the item's partial planes are stored (MREC <= 8)
  uint64_t mempty[8];      // combiner -> consumers: the record slot may be reused
  uint32_t tmem_base;
  int tok_ids[NSTAGE][JOB_DN_TOK];  // token ids of the item, staged with its last chunk
  int recs[8][36];                  // MergeRec ring (fused merge), MREC <= 8
  int comb_tok[32];                 // the combiner's current token list
};
template <int NTS>
constexpr int smem_bytes() { return 1024 + stage_bytes<NTS>() * NSTAGE + static_cast<int>(sizeof(Smem)); }
constexpr int SMEM_BYTES = smem_bytes<1>();

__device__ __forceinline__ bool kind_dense(int kind) { return kind == 0 || kind == DZ_KIND_DENSE; }

// Item order: all base items first (row tile order; the big ones start early), then the delta
// items row-tile-major, so row tiles complete (and are combined) progressively through the launch
// instead of all at the end. dz_plan puts the n_base base jobs first in the job list. Base items
// cover BASE_RT = 128 rows (nbt tiles), delta items RT = 256 rows (nrt tiles): a base item streams
// 2 bytes per weight against a 4-bit delta's ~0.8, so halving it keeps the long base items off the
// launch's critical path. Each output element still gets exactly one base and one delta partial.
__device__ __forceinline__ void item_coords(int item, int nrt, int nbt, int nsplit, int dsplit, int n_jobs, int n_base,
                                            int& rt, int& j, int& sp) {
  const int nb_items = nbt * nsplit * n_base;
  if (item < nb_items) {
    j = item / (nbt * nsplit);
    const int r = item - j * (nbt * nsplit);
    sp = r / nbt;
    rt = r - sp * nbt;
  } else {
    const int k = item - nb_items, per = (n_jobs - n_base) * dsplit;
    rt = k / per;
    const int r = k - rt * per;
    j = n_base + r / dsplit;
    sp = r - (r / dsplit) * dsplit;
  }
}

// Default base K-splits when the caller passes 0 (DZ_SPLIT_RULE 2): two for layers of <= 4096 output
// rows (o / down at 7B: 32 base tiles of 1 MB each; two K-halves bring a base item near a delta
// item's size and give a low batch twice the base items), one otherwise. Same box
// (profiles/r02_ab_split_rule2.txt): cfg5 batch 1-8 +16-19%, the headline step -0.4%. Rule 1 (up
// to 4 splits for every shape) gave +3..39% at low batch but -2.5% on the headline
// (profiles/r02_ab_split_rule.txt). A deployment can still pass dz_sbmm_args.base_splits. The split
// count is never derived from the batch, so a token's result does not depend on the other tokens.
#ifndef DZ_DEFAULT_BASE_SPLITS
#define DZ_DEFAULT_BASE_SPLITS 1
#endif
#ifndef DZ_SPLIT_RULE
#define DZ_SPLIT_RULE 2  // 0: DZ_DEFAULT_BASE_SPLITS everywhere; 1: enough items for 148 SMs; 2: see above
#endif
__host__ __device__ inline int base_splits(int out, int /*in*/) {
  if (DZ_SPLIT_RULE == 1) {  // enough base items for every SM of a B200 (148): shape-keyed, never batch-keyed
    const int nbt = (out + 127) / 128, s = (148 + nbt - 1) / nbt;
    return s > 4 ? 4 : s;
  }
  if (DZ_SPLIT_RULE == 2) return out <= 4096 ? 2 : 1;  // base items of the narrow layers ~ delta-item size
  return DZ_DEFAULT_BASE_SPLITS;
}
// Default K-splits of each decode delta job: 1. Splitting the delta items of the out <= 4096 layers
// in two measured neutral at the BASELINE batch and mixed at low batch (profiles/r01_ab_dsplit.txt),
// so it stays an explicit knob (dz_sbmm_args.delta_splits). Never derived from the batch.
__host__ __device__ inline int delta_splits(int /*out*/, int /*in*/) { return 1; }
// The K-split counts a launch actually uses: the requested (or shape-default) counts, capped so that
// every split owns at least one K-chunk (a split without chunks would never publish its partial).
__host__ __device__ inline void resolve_splits(int out, int in, bool has_base, int& bs, int& ds) {
  if (bs <= 0) bs = base_splits(out, in);
  if (ds <= 0) ds = delta_splits(out, in);
  const int nch_base = ceil_div(in, SPLIT_CH * KC_DN), nch_sp = ceil_div(ceil_div(in, kBlkCols), NB_SP);
  bs = bs > 4 ? 4 : bs;
  bs = bs > nch_base ? nch_base : bs;
  ds = ds > 2 ? 2 : ds;
  ds = ds > nch_sp ? nch_sp : ds;
  if (!has_base) ds = 1;  // single contributor: the delta writes Y directly
}

// K-chunk range [k0, k1) of base split sp of ns: splits cut whole SPLIT_CH-chunk units, whatever the
// stage size, so a token's partial sums the same chunks in the same order for every bn / bch.
__host__ __device__ inline void base_chunks(int in, int sp, int ns, int& k0, int& k1) {
  const int nck = ceil_div(in, KC_DN), nsu = ceil_div(nck, SPLIT_CH);
  k0 = SPLIT_CH * (sp * nsu / ns);
  k1 = cmin(nck, SPLIT_CH * ((sp + 1) * nsu / ns));
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ------------------------------------------------------------------------------------------
// Consumer math (CUDA-core decode + legacy mma.sp / mma)
// ------------------------------------------------------------------------------------------
// Codes -> bf16 A fragments. RAW: leave the value as 128 + u (the offset 128 + qmax is removed
// later with a ones-MMA, see sparse_pair); else subtract it here (one HADD2 per register).
template <int FB, bool RAW>
__device__ __forceinline__ void conv_codes(uint32_t (&a)[4], const uint32_t (&cw)[4], int i, uint32_t off2) {
  if (FB == 4) {
    const uint32_t w = cw[i];
    // shifts on the FMA pipe (IMAD.HI): the ALU pipe carries the LOP3s (DZ_SHIFT_FMA=0: SHF on ALU)
    const uint32_t sh[4] = {w, DZ_SHIFT_FMA ? mulhi_shr<4>(w) : w >> 4, DZ_SHIFT_FMA ? mulhi_shr<8>(w) : w >> 8,
                            DZ_SHIFT_FMA ? mulhi_shr<12>(w) : w >> 12};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      a[k] = lop3_and_or(sh[k], 0x000F000Fu, 0x43004300u);
      if (!RAW) a[k] = bf16x2_sub(a[k], off2);
    }
  } else {
    const uint32_t w = cw[i >> 1];
    const int o = 4 * (i & 1);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      a[k] = lop3_and_or(w >> (2 * (o + k)), 0x00030003u, 0x43004300u);
      if (!RAW) a[k] = bf16x2_sub(a[k], off2);
    }
  }
}

// The offset trick (kOnesMma): the tensor core computes S1 = sum (128+u) x and, with an all-ones A
// and the same metadata, S0 = sum_kept x; then sum code*x = S1 - (128+qmax) S0 in fp32. It moves
// 16 HADD2 per 16x128 block-row from the FMA pipe to the tensor pipe. Off by default: it measured
// ~8% slower on B200 (kept for the record; build a variant with -DDZ_ONES_MMA=1 to retry).
#ifndef DZ_ONES_MMA
#define DZ_ONES_MMA 0
#endif
constexpr bool kOnesMma = DZ_ONES_MMA != 0;

// Two consecutive blocks (b0, b0+1 < nb) of a sparse chunk for this warp's nrv <= MR row groups
// and NT token tiles: loads, decodes and issues 4 independent mma.sp chains.
#ifndef DZ_PAIR
#define DZ_PAIR 2
#endif
constexpr int PAIR1 = DZ_PAIR;  // blocks per sparse_pair call at one n-tile
// FULL: both blocks and all MR row groups valid -> no guards, straight-line code the compiler can
// interleave (the common case); otherwise guarded (tail chunk / tail row tile).
template <int FB, int NT, bool FULL, int PAIR>
__device__ __forceinline__ void sparse_pair(float (&acc)[MR][NT_DN][4], uint32_t sA, uint32_t xl, int b0, int nb,
                                            int nrv, uint32_t off2, int lane) {
  const float offf = __uint_as_float((off2 & 0xFFFFu) << 16);  // 128 + qmax
  constexpr int CODE = sparse_code_bytes(FB);
  constexpr int BLK = sparse_block_bytes(FB);
  const int g = lane >> 2;
  uint32_t cw[PAIR][MR][4];
  uint2 meta[PAIR][MR];
  float2 sc[PAIR][MR];
#pragma unroll
  for (int p = 0; p < PAIR; p++) {
#pragma unroll
    for (int r = 0; r < MR; r++) {
      // the TMA box lands row group by row group: rg r of this warp holds NB_SP contiguous blocks
      const uint32_t blk = sA + (r * NB_SP + b0 + p) * BLK;
      if (FULL || (b0 + p < nb && r < nrv)) {
        if (FB == 4) {
          const uint4 c = lds128(blk + lane * 16);
          cw[p][r][0] = c.x; cw[p][r][1] = c.y; cw[p][r][2] = c.z; cw[p][r][3] = c.w;
        } else {
          const uint2 c = lds64(blk + lane * 8);
          cw[p][r][0] = c.x; cw[p][r][1] = c.y; cw[p][r][2] = 0; cw[p][r][3] = 0;
        }
        meta[p][r] = lds64(blk + CODE + lane * 8);
        const uint2 sv = lds64(blk + CODE + kMetaBytes + g * 8);
        sc[p][r] = make_float2(__uint_as_float(sv.x), __uint_as_float(sv.y));
      } else {
        cw[p][r][0] = cw[p][r][1] = cw[p][r][2] = cw[p][r][3] = 0;
        meta[p][r] = make_uint2(0x44444444u, 0x44444444u);
        sc[p][r] = make_float2(0.f, 0.f);
      }
    }
  }
  float tmp[PAIR][MR][NT][4];
  float sx[PAIR][MR][NT][4];  // S0 = sum of the kept x (kOnesMma)
#pragma unroll
  for (int p = 0; p < PAIR; p++)
#pragma unroll
    for (int r = 0; r < MR; r++)
#pragma unroll
      for (int n = 0; n < NT; n++) {
        tmp[p][r][n][0] = tmp[p][r][n][1] = tmp[p][r][n][2] = tmp[p][r][n][3] = 0.f;
        sx[p][r][n][0] = sx[p][r][n][1] = sx[p][r][n][2] = sx[p][r][n][3] = 0.f;
      }
  const uint32_t ones[4] = {0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u};
#pragma unroll
  for (int i = 0; i < 4; i++) {
#pragma unroll
    for (int p = 0; p < PAIR; p++) {
      if (!FULL && b0 + p >= nb) continue;  // partial last chunk
      uint32_t bf[NT][4];
#pragma unroll
      for (int n = 0; n < NT; n++) ldmatrix_x4(bf[n], xl + n * 8 * XS_SP + ((b0 + p) * kBlkCols + 32 * i) * 2);
#pragma unroll
      for (int r = 0; r < MR; r++) {
        if (!FULL && r >= nrv) continue;  // padding row group (zero-filled by TMA, never stored)
        uint32_t a[4];
        conv_codes<FB, kOnesMma>(a, cw[p][r], i, off2);
        const uint32_t e = (i < 2) ? meta[p][r].x : meta[p][r].y;
#pragma unroll
        for (int n = 0; n < NT; n++) {
          if (i & 1) {
            mma_sp_bf16_16832<1>(tmp[p][r][n], a, bf[n], e);
            if (kOnesMma) mma_sp_bf16_16832<1>(sx[p][r][n], ones, bf[n], e);
          } else {
            mma_sp_bf16_16832<0>(tmp[p][r][n], a, bf[n], e);
            if (kOnesMma) mma_sp_bf16_16832<0>(sx[p][r][n], ones, bf[n], e);
          }
        }
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PAIR; p++)
#pragma unroll
    for (int r = 0; r < MR; r++)
#pragma unroll
      for (int n = 0; n < NT; n++) {
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const float t = kOnesMma ? fmaf(-offf, sx[p][r][n][v], tmp[p][r][n][v]) : tmp[p][r][n][v];
          acc[r][n][v] = fmaf((v & 2) ? sc[p][r].y : sc[p][r].x, t, acc[r][n][v]);
        }
      }
}

template <int FB, int NT>
__device__ __forceinline__ void sparse_chunk(float (&acc)[MR][NT_DN][4], uint32_t sA, uint32_t xl, int nb,
                                             int nrv, uint32_t off2, int lane) {
  // blocks per call: 2 at one n-tile (8 independent mma.sp chains per warp), 1 at more n-tiles
  // (the same chain count from the extra n-tiles' accumulators)
  constexpr int PAIR = NT == 1 ? PAIR1 : 1;
  if (nb == NB_SP && nrv == MR) {
#if DZ_PAIR_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int b0 = 0; b0 < NB_SP; b0 += PAIR) sparse_pair<FB, NT, true, PAIR>(acc, sA, xl, b0, nb, nrv, off2, lane);
  } else {
#pragma unroll 1
    for (int b0 = 0; b0 < nb; b0 += PAIR) sparse_pair<FB, NT, false, PAIR>(acc, sA, xl, b0, nb, nrv, off2, lane);
  }
}

// One dense-delta half-block chunk (64 columns = 4 k16 MMAs); X rows are per-token (XS_DN).
template <int NT>
__device__ __forceinline__ void dense_chunk(float (&acc)[MR][NT_DN][4], uint32_t sA, uint32_t sX, int nrv,
                                            int lane) {
#pragma unroll
  for (int jj = 0; jj < 2; jj++) {
    uint32_t a[MR][2][4];
#pragma unroll
    for (int r = 0; r < MR; r++) {
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const uint4 v = lds128(sA + r * DN_HALF + (2 * jj + s) * 512 + lane * 16);
        a[r][s][0] = v.x; a[r][s][1] = v.y; a[r][s][2] = v.z; a[r][s][3] = v.w;
      }
    }
#pragma unroll
    for (int n = 0; n < NT; n++) {
      uint32_t bf[4];
      ldmatrix_x4(bf, sX + (n * 8 + (lane & 7)) * XS_DN + ((jj * 4 + (lane >> 3)) << 4));
#pragma unroll
      for (int r = 0; r < MR; r++) {
        if (r >= nrv) continue;
        mma_bf16_16816(acc[r][n], a[r][0], bf[0], bf[1]);
        mma_bf16_16816(acc[r][n], a[r][1], bf[2], bf[3]);
      }
    }
  }
}

__device__ __forceinline__ void dense_dispatch(int nt, float (&acc)[MR][NT_DN][4], uint32_t sA, uint32_t sX,
                                               int nrv, int lane) {
  switch (nt) {
    case 1: dense_chunk<1>(acc, sA, sX, nrv, lane); break;
    case 2: dense_chunk<2>(acc, sA, sX, nrv, lane); break;
    case 3: dense_chunk<3>(acc, sA, sX, nrv, lane); break;
    case 4: dense_chunk<4>(acc, sA, sX, nrv, lane); break;
    default: dense_chunk<4>(acc, sA, sX, nrv, lane); break;
  }
}

struct MergeCtx {
  float* part;                // [planes][T][out] fp32 partials (workspace)
  int* slice_cnt;             // [ceil(out / 32)] arrival counters (workspace, zero between launches)
  const int32_t* perm;        // staged row -> Y row (mixed plans), or NULL
  void* Y;
  int64_t ldy;
  int out, y_dtype, act, debug, T, nsplit;
  int base_target;            // base-plane publications per 32-row slice (2 warps x base jobs x K-splits)
  int readers;                // delta items combining per slice (the decode delta jobs)
  bool has_base;
  bool fused;                 // delta items combine base planes + their product into Y (else: planes only)
};

__device__ __forceinline__ void store_y(const MergeCtx& m, int tok, int row, float v) {
  if (m.act == DZ_ACT_TANH) v = tanhf(v);
  const int yrow = m.perm != nullptr ? __ldg(m.perm + tok) : tok;
  const int64_t yo = static_cast<int64_t>(yrow) * m.ldy + row;
  if (m.y_dtype == DZ_F32)
    reinterpret_cast<float*>(m.Y)[yo] = v;
  else
    reinterpret_cast<__nv_bfloat16*>(m.Y)[yo] = __float2bfloat16_rn(v);
}

// Publish N fp32 partials v[i] of y[tok[i]][row[i]] (valid[i]) into partial slot `slot` of the
// workspace: [planes][T][out] fp32, slot s < nsplit = base K-split s, slots nsplit.. = the
// token's delta job (per delta K-split). Plain stores — every (slot, token, row) has exactly one
// producer. With the fused merge the CTA's combiner warp sums the planes of each delta item's
// tokens into Y (see combine_tokens). Without a base there is a single contributor and Y is
// written directly.
template <int N>
__device__ __forceinline__ void merge_batch(const MergeCtx& m, int slot, const int (&tok)[N], const int (&row)[N],
                                            const float (&v)[N], const bool (&valid)[N]) {
  if (m.debug & 4) return;  // debug bit 2: drop the merge (probe of its cost; Y is not written)
  if (!m.has_base) {
#pragma unroll
    for (int i = 0; i < N; i++)
      if (valid[i]) store_y(m, tok[i], row[i], v[i]);
    return;
  }
  float* part = m.part + static_cast<int64_t>(slot) * m.T * m.out;
#pragma unroll
  for (int i = 0; i < N; i++)
    if (valid[i]) part[static_cast<int64_t>(tok[i]) * m.out + row[i]] = v[i];
}

__device__ __forceinline__ void merge_contribution(const MergeCtx& m, int slot, int tok, int row, float v) {
  const int t[1] = {tok}, r[1] = {row};
  const float x[1] = {v};
  const bool ok[1] = {true};
  merge_batch<1>(m, slot, t, r, x, ok);
}

// Base accumulators (TMEM, lane = output row, column = token) -> merge. Warp w drains half w/4
// (rows 128*(w/4)..) of the tile, TMEM lanes 32*(w%4)..+31 (the lanes warp w may access).
template <int BN>
__device__ __forceinline__ void drain_base_accumulator(uint32_t tmem_acc, int warp, int lane, const MergeCtx& m,
                                                       int split, int row0, int tok_begin, int tcount) {
  // TMEM lane quarter q = warp % 4 (the hardware's warp -> lane restriction); the NW/4 warps of a
  // quarter split the BN token columns.
  constexpr int PER = BN / 16 / (NW / 4);  // 16-column chunks per warp
  const int q = warp & 3, part = warp >> 2;
  const int row = row0 + 32 * q + lane;
  const uint32_t taddr = tmem_acc + (static_cast<uint32_t>(32 * q) << 16);
#if DZ_DRAIN_BATCH
  // both TMEM loads of a chunk pair in flight before one wait (half the load latencies)
#pragma unroll 1
  for (int c0 = part * PER; c0 < (part + 1) * PER; c0 += 2) {
    if (c0 * 16 >= tcount) break;
    uint32_t vv[2][16];
    tmem_ld16(taddr + c0 * 16, vv[0]);
    if (c0 + 1 < (part + 1) * PER && (c0 + 1) * 16 < tcount) tmem_ld16(taddr + (c0 + 1) * 16, vv[1]);
    tmem_ld_wait();
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int c = c0 + h;
      if (c >= (part + 1) * PER || c * 16 >= tcount) break;
      int tk[16], rw[16];
      float x[16];
      bool ok[16];
#pragma unroll
      for (int j = 0; j < 16; j++) {
        tk[j] = tok_begin + c * 16 + j;
        rw[j] = row;
        x[j] = __uint_as_float(vv[h][j]);
        ok[j] = row < m.out && c * 16 + j < tcount;
      }
      merge_batch<16>(m, split, tk, rw, x, ok);
    }
  }
#else
#pragma unroll 1
  for (int c = part * PER; c < (part + 1) * PER; c++) {
    if (c * 16 >= tcount) break;
    uint32_t v[16];
    tmem_ld16(taddr + c * 16, v);
    tmem_ld_wait();
    int tk[16], rw[16];
    float x[16];
    bool ok[16];
#pragma unroll
    for (int j = 0; j < 16; j++) {
      tk[j] = tok_begin + c * 16 + j;
      rw[j] = row;
      x[j] = __uint_as_float(v[j]);
      ok[j] = row < m.out && c * 16 + j < tcount;
    }
    merge_batch<16>(m, split, tk, rw, x, ok);
  }
#endif
}

// The narrow-tile drain (T <= 32). Inline: out of line (__noinline__) measured ~1% slower on the
// 7B step and at cfg5 points (the MergeCtx goes through the stack).
__device__ __forceinline__ void drain_narrow(uint32_t tmem_acc, int warp, int lane, const MergeCtx& m, int split,
                                          int row0, int tok_begin, int tcount) {
  drain_base_accumulator<DZ_BASE_BN64 ? 64 : 32>(tmem_acc, warp, lane, m, split, row0, tok_begin, tcount);
}

// Dense-delta job partial (mma.sync fragments) -> merge.
__device__ __forceinline__ void merge_fragments(const float (&acc)[MR][NT_DN][4], int nt, const MergeCtx& m,
                                                int plane, int rg0, int tcount, const int* tok_ids, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int r = 0; r < MR; r++) {
    const int row0 = (rg0 + r) * kBlkRows;
#pragma unroll
    for (int n = 0; n < NT_DN; n++) {
      if (n < nt) {
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const int tk = n * 8 + 2 * t + (v & 1);
          const int row = row0 + g + ((v & 2) ? 8 : 0);
          if (tk < tcount && row < m.out) merge_contribution(m, plane, tok_ids[tk], row, acc[r][n][v]);
        }
      }
    }
  }
}

__device__ __forceinline__ void finalize_rows(const float* __restrict__ part, int nsplit, int t0, int T, int out,
                                              const int32_t* __restrict__ perm, void* __restrict__ Y, int64_t ldy,
                                              int y_dtype, int act, int64_t first, int64_t stride) {
  const int64_t plane = static_cast<int64_t>(T) * out;
  const bool vec = (out % 4) == 0 && (ldy % 4) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  if (vec) {
    const int o4 = out / 4;
    const int64_t n = static_cast<int64_t>(T - t0) * o4;
    for (int64_t i = first; i < n; i += stride) {
      const int t = t0 + static_cast<int>(i / o4), r = 4 * static_cast<int>(i % o4);
      const float* p = part + static_cast<int64_t>(t) * out + r;
      float4 v = __ldcg(reinterpret_cast<const float4*>(p));
      for (int sp = 1; sp <= nsplit; sp++) {
        const float4 w = __ldcg(reinterpret_cast<const float4*>(p + sp * plane));
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
      if (act == DZ_ACT_TANH) { v.x = tanhf(v.x); v.y = tanhf(v.y); v.z = tanhf(v.z); v.w = tanhf(v.w); }
      const int yr = perm != nullptr ? __ldg(perm + t) : t;
      const int64_t yo = static_cast<int64_t>(yr) * ldy + r;
      if (y_dtype == DZ_F32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(Y) + yo) = v;
      } else {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 w;
        w.x = *reinterpret_cast<const uint32_t*>(&lo);
        w.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(Y) + yo) = w;
      }
    }
  } else {
    const int64_t n = static_cast<int64_t>(T - t0) * out;
    for (int64_t i = first; i < n; i += stride) {
      const int t = t0 + static_cast<int>(i / out), r = static_cast<int>(i % out);
      const float* p = part + static_cast<int64_t>(t) * out + r;
      float v = __ldcg(p);
      for (int sp = 1; sp <= nsplit; sp++) v += __ldcg(p + sp * plane);
      if (act == DZ_ACT_TANH) v = tanhf(v);
      const int yr = perm != nullptr ? __ldg(perm + t) : t;
      const int64_t yo = static_cast<int64_t>(yr) * ldy + r;
      if (y_dtype == DZ_F32)
        reinterpret_cast<float*>(Y)[yo] = v;
      else
        reinterpret_cast<__nv_bfloat16*>(Y)[yo] = __float2bfloat16_rn(v);
    }
  }
}

// Finalize the merged decode rows [t0, T): Y[perm[t]][r] = act(((P_0 + P_1) + ... + P_{S-1}) + P_S)
// with P_s the base K-split partials and the delta partials after them — a fixed summation order,
// so the result is deterministic and independent of the batch. Only for launches that keep every
// partial in planes: the default decode launch (k_sbmm<false>), delta K-splits, probes.
__global__ void __launch_bounds__(256) k_finalize(const float* __restrict__ part, int nsplit, int t0, int T, int out,
                                                  const int32_t* __restrict__ perm, void* __restrict__ Y, int64_t ldy,
                                                  int y_dtype, int act, const int32_t* __restrict__ t0_dev) {
  griddep_wait();
  griddep_launch_dependents();
  if (t0_dev != nullptr) t0 = *t0_dev;  // device mixed plan: t_pf
  finalize_rows(part, nsplit, t0, T, out, perm, Y, ldy, y_dtype, act,
                blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x, static_cast<int64_t>(gridDim.x) * blockDim.x);
}

// Tail prefetch: a CTA with no more items warms L2 with the first weight stages of the item its
// blockIdx takes first in the next linear of the step (items [0, grid) are static there), so the
// launch boundary keeps HBM busy with bytes the next launch reads anyway.
#ifndef DZ_TAIL_PF
#define DZ_TAIL_PF 6
#endif
constexpr int TAIL_PF_CHUNKS = DZ_TAIL_PF;
__device__ __forceinline__ void tail_prefetch(const dz_sbmm_args& nx) {
  if (nx.perm != nullptr || nx.T <= 0) return;  // decode plans only
  const int nrt = ceil_div(nx.out, RT), nbt = ceil_div(nx.out, BASE_RT), nkb = ceil_div(nx.in, kBlkCols);
  const int n_base = nx.base != nullptr ? ceil_div(nx.T, BASE_N) : 0;
  const int n_jobs = nx.n_jobs_dev != nullptr ? *nx.n_jobs_dev : nx.n_jobs;
  int nsplit = nx.base_splits, dsplit = nx.delta_splits;
  resolve_splits(nx.out, nx.in, nx.base != nullptr, nsplit, dsplit);
  const int n_items = n_jobs < n_base ? 0 : nbt * nsplit * n_base + nrt * (n_jobs - n_base) * dsplit;
  const int item = blockIdx.x;
  if (item >= n_items) return;
  int rt = 0, jj = 0, sp = 0;
  item_coords(item, nrt, nbt, nsplit, dsplit, n_jobs, n_base, rt, jj, sp);
  const dz_job job = nx.jobs[jj];
  const dz_native_delta* e = job.kind == 0 ? nx.base : nx.table + job.slot;
  const void* m = e->tmap;
  if (job.kind == 0) {
    int k0, k1;
    base_chunks(nx.in, sp, nsplit, k0, k1);
    for (int c = k0; c < k0 + TAIL_PF_CHUNKS * base_bch(base_bn(nx.T)) && c < k1; c++)
      tma_prefetch_2d(m, c * KC_DN, rt * BASE_RT);
  } else if (kind_dense(job.kind)) {
    const int d0 = sp * (2 * nkb) / dsplit;
    for (int c = d0; c < d0 + TAIL_PF_CHUNKS && c < 2 * nkb; c++) tma_prefetch_2d(m, c * (DN_HALF / 8), rt * RG);
  } else {
    const int d0 = sp * ceil_div(nkb, NB_SP) / dsplit;
    for (int c = d0; c < d0 + TAIL_PF_CHUNKS && c * NB_SP < nkb; c++) tma_prefetch_3d(m, 0, c * NB_SP, rt * RG);
  }
}

// ---- fused merge (combiner warp) ---------------------------------------------------------------
// Every work item's contributions go to fp32 planes with plain stores (base K-split s -> plane s,
// the token's delta -> plane nsplit), as in the unfused layout. After an item, the consumer warps
// arrive on a shared-memory record ring; the CTA's combiner warp then
//   * base item: publishes the item's four 32-row slices on their counters (fence + relaxed add);
//   * delta item: waits until every base contribution of its eight slices is published (acquire),
//     writes y = act(((P_0 + P_1) + ...) + P_delta) for the item's tokens and rows, and counts
//     itself as a reader in the counters' high bits; the last reader re-arms the counter.
// Every output element is written exactly once, by the delta item of its token, with a fixed
// summation order (deterministic, batch-invariant). A combiner only ever waits on base items,
// which are first in the item order and never wait, so the persistent grid cannot deadlock; the
// consumers never wait on a round trip.
#ifndef DZ_MREC
#define DZ_MREC 4
#endif
#ifndef DZ_COMB_SLEEP
#define DZ_COMB_SLEEP 32  // ns between polls of the record ring (the combiner shares an SMSP with consumers)
#endif
constexpr int MREC = DZ_MREC;             // records in flight (consumer warps -> combiner)
struct MergeRec {
  int rt;        // row tile (base: 128-row tile, delta: 256-row tile); -1 = end of work
  int is_base;
  int ntok;      // delta: tokens of the job (<= 32)
  int lin;       // linear of a chained launch
  int tok[32];   // delta: the job's token (staged row) ids
};

__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_s32(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Y rows [r0, r0 + 256) of the `ntok` tokens `tok[]`: planes 0..nsplit (base splits, then the delta)
// summed in that order. Lanes own row quads (two per lane); the loads of a group of CT tokens are all
// in flight before any add, so a group costs about one L2 round trip per plane pass.
constexpr int CT = 4;
__device__ __forceinline__ void store_y4(const MergeCtx& m, int t, int r, float4 y) {
  if (m.act == DZ_ACT_TANH) { y.x = tanhf(y.x); y.y = tanhf(y.y); y.z = tanhf(y.z); y.w = tanhf(y.w); }
  const int yr = m.perm != nullptr ? __ldg(m.perm + t) : t;
  const int64_t yo = static_cast<int64_t>(yr) * m.ldy + r;
  if (m.y_dtype == DZ_F32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(m.Y) + yo) = y;
  } else {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(y.x, y.y), hi = __floats2bfloat162_rn(y.z, y.w);
    uint2 w;
    w.x = *reinterpret_cast<const uint32_t*>(&lo);
    w.y = *reinterpret_cast<const uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(m.Y) + yo) = w;
  }
}

__device__ __noinline__ void combine_tokens(const MergeCtx m, int r0, int ntok, const int* tok, int lane) {
  const int64_t plane = static_cast<int64_t>(m.T) * m.out;
  const bool vec = (m.out % 4) == 0 && (m.ldy % 4) == 0 && (reinterpret_cast<uintptr_t>(m.Y) & 15) == 0;
  if (vec) {
    const int ra = r0 + 4 * lane, rb = ra + 128;
    const bool oka = ra < m.out, okb = rb < m.out;
#pragma unroll 1
    for (int i0 = 0; i0 < ntok; i0 += CT) {
      float4 va[CT], vb[CT], da[CT], db[CT];
      int t[CT];
#pragma unroll
      for (int c = 0; c < CT; c++) {
        t[c] = i0 + c < ntok ? tok[i0 + c] : -1;
        const float* p = m.part + static_cast<int64_t>(t[c] < 0 ? 0 : t[c]) * m.out;
        if (t[c] >= 0 && oka) {
          va[c] = __ldcg(reinterpret_cast<const float4*>(p + ra));
          da[c] = __ldcg(reinterpret_cast<const float4*>(p + m.nsplit * plane + ra));
        }
        if (t[c] >= 0 && okb) {
          vb[c] = __ldcg(reinterpret_cast<const float4*>(p + rb));
          db[c] = __ldcg(reinterpret_cast<const float4*>(p + m.nsplit * plane + rb));
        }
      }
      for (int sp = 1; sp < m.nsplit; sp++) {  // further base K-splits, in order
#pragma unroll
        for (int c = 0; c < CT; c++) {
          const float* p = m.part + sp * plane + static_cast<int64_t>(t[c] < 0 ? 0 : t[c]) * m.out;
          if (t[c] >= 0 && oka) {
            const float4 w = __ldcg(reinterpret_cast<const float4*>(p + ra));
            va[c].x += w.x; va[c].y += w.y; va[c].z += w.z; va[c].w += w.w;
          }
          if (t[c] >= 0 && okb) {
            const float4 w = __ldcg(reinterpret_cast<const float4*>(p + rb));
            vb[c].x += w.x; vb[c].y += w.y; vb[c].z += w.z; vb[c].w += w.w;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < CT; c++) {
        if (t[c] < 0) continue;
        if (oka) store_y4(m, t[c], ra, make_float4(va[c].x + da[c].x, va[c].y + da[c].y, va[c].z + da[c].z, va[c].w + da[c].w));
        if (okb) store_y4(m, t[c], rb, make_float4(vb[c].x + db[c].x, vb[c].y + db[c].y, vb[c].z + db[c].z, vb[c].w + db[c].w));
      }
    }
  } else {
#pragma unroll 1
    for (int i = 0; i < ntok; i++) {
      const int t = tok[i];
      for (int r = r0 + lane; r < r0 + RT && r < m.out; r += 32) {
        const float* p = m.part + static_cast<int64_t>(t) * m.out + r;
        float v = __ldcg(p);
        for (int sp = 1; sp <= m.nsplit; sp++) v += __ldcg(p + sp * plane);
        if (m.act == DZ_ACT_TANH) v = tanhf(v);
        const int yr = m.perm != nullptr ? __ldg(m.perm + t) : t;
        const int64_t yo = static_cast<int64_t>(yr) * m.ldy + r;
        if (m.y_dtype == DZ_F32)
          reinterpret_cast<float*>(m.Y)[yo] = v;
        else
          reinterpret_cast<__nv_bfloat16*>(m.Y)[yo] = __float2bfloat16_rn(v);
      }
    }
  }
}

// Consumer warp `warp` finished its plane stores of merged item #k: warp 0 fills the record, every
// warp arrives (its lanes' stores, ordered by the warp barrier, precede the arrive's release).
__device__ __forceinline__ void publish_item(MergeRec* recs, uint64_t* mfull, uint64_t* mempty, int k, int warp,
                                             int lane, int rt, int is_base, int ntok, int rtok, int lin = 0) {
  const int slot = k % MREC;
  mbar_wait(&mempty[slot], ((k / MREC) & 1) ^ 1);
  if (warp == 0) {
    if (lane == 0) {
      recs[slot].rt = rt;
      recs[slot].is_base = is_base;
      recs[slot].ntok = ntok;
      recs[slot].lin = lin;
    }
    if (lane < ntok) recs[slot].tok[lane] = rtok;
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&mfull[slot]);
}

// The combiner's work for merged item #k (its record is complete): returns false at end of work.
__device__ __forceinline__ bool service_record(Smem* sm, const MergeCtx& mctx, int k, int lane) {
  const MergeRec* recs = reinterpret_cast<const MergeRec*>(sm->recs);
  const int slot = k % MREC;
  const int n_slices = ceil_div(mctx.out, 32);
  const int rt = recs[slot].rt, is_base = recs[slot].is_base, ntok = recs[slot].ntok;
  const int mytok = lane < ntok ? recs[slot].tok[lane] : 0;
  __syncwarp();
  if (lane == 0) mbar_arrive(&sm->mempty[slot]);
  if (rt < 0) return false;
  if (is_base) {
    fence_acq_rel_gpu();  // release: the consumers' plane stores (CTA-synchronized) -> GPU scope
    const int slice = rt * (BASE_RT / 32) + lane;
    if (lane < BASE_RT / 32 && slice < n_slices) red_add_s32(mctx.slice_cnt + slice, 1);
    return true;
  }
  const int slice = rt * (RT / 32) + lane;
  const bool mine = lane < RT / 32 && slice < n_slices;
  if (mine)
    while ((ld_relaxed_s32(mctx.slice_cnt + slice) & 0xFFFF) < mctx.base_target) __nanosleep(32);
  __syncwarp();
  fence_acq_rel_gpu();  // acquire: the base planes of these slices (and this CTA's delta plane)
  // count this reader now (every reader has passed its wait once the count completes); the result
  // is only needed after the combine, so its round trip overlaps the plane loads
  const int old = mine ? atomicAdd(mctx.slice_cnt + slice, 1 << 16) : 0;
  if (lane < ntok) sm->comb_tok[lane] = mytok;
  __syncwarp();
  combine_tokens(mctx, rt * RT, ntok, sm->comb_tok, lane);
  if (mine && (old >> 16) == mctx.readers - 1) mctx.slice_cnt[slice] = 0;  // last reader re-arms
  return true;
}

// Per-linear constants of a launch, or of one linear of a chained launch.
struct LinGeo {
  int n16, nrt, nkb, nbt, n_base, nsplit, dsplit, bn, bch;
};
__device__ __forceinline__ LinGeo lin_geo(const dz_sbmm_args& a) {
  LinGeo g;
  g.n16 = ceil_div(a.out, kBlkRows);
  g.nrt = ceil_div(a.out, RT);
  g.nkb = ceil_div(a.in, kBlkCols);
  g.bn = base_bn(a.T);
  g.bch = base_bch(g.bn);
  g.nbt = ceil_div(a.out, BASE_RT);
  int t_pf = a.t_pf;
  if (a.pf_counts_dev != nullptr) {  // device mixed plan: the staged prefill rows come from the planner
    griddep_wait();
    t_pf = a.pf_counts_dev[2];
  }
  g.n_base = a.base != nullptr ? ceil_div(a.T - t_pf, BASE_N) : 0;  // dz_plan: base jobs first
  g.nsplit = a.base_splits;   // resolved by the host (launch_decode / dz_sbmm_chain_encode)
  g.dsplit = a.delta_splits;
  return g;
}

template <bool FUSED>
__device__ __forceinline__ MergeCtx make_mctx(const dz_sbmm_args& a, const LinGeo& g) {
  MergeCtx m;
  m.slice_cnt = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(a.workspace) + DZ_WS_CNT_OFF);
  m.part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(a.workspace) + DZ_WS_PART_OFF);
  m.fused = FUSED && a.base != nullptr && !a.keep_planes && g.dsplit == 1 && !(a.debug & 6);
  m.base_target = g.n_base * g.nsplit;  // base items publishing each slice
  m.readers = 0;
  m.T = a.T;
  m.nsplit = g.nsplit;
  m.perm = a.perm;
  m.Y = a.Y;
  m.ldy = a.ldy;
  m.out = a.out;
  m.y_dtype = a.y_dtype;
  m.act = a.act;
  m.has_base = a.base != nullptr;
  m.debug = a.debug;
  return m;
}

// One linear of a chained launch (dz_sbmm_chain): its arguments (splits resolved by the host) and
// the tensor map of its X. Host-encoded by dz_sbmm_chain_encode, copied to the device by the caller.
struct ChainLin {
  dz_sbmm_args a;
  alignas(64) CUtensorMap xmap;
};

// Delta items of a linear: what its combiners count in the chain's done counter.
__device__ __forceinline__ int delta_items(const dz_sbmm_args& a) {
  const LinGeo g = lin_geo(a);
  const int n_jobs = a.n_jobs_dev != nullptr ? *a.n_jobs_dev : a.n_jobs;
  return g.nrt * (n_jobs - g.n_base) * g.dsplit;
}

__device__ __forceinline__ int ld_acquire_gpu_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Chained launch: wait until linear l-1 wrote all of Y (its X), then let the async proxy (TMA) see it.
__device__ __forceinline__ void wait_linear(const int* done, int target) {
  while (ld_acquire_gpu_s32(done) < target) __nanosleep(64);
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Work items of a launch (debug bit 1: base items only, a probe of the base stream).
__device__ __forceinline__ int job_items(const dz_sbmm_args& a, int n_jobs, int n_base, int nrt, int nbt, int nsplit,
                                         int dsplit) {
  return n_jobs < n_base ? 0 : nbt * nsplit * n_base + ((a.debug & 2) ? 0 : nrt * (n_jobs - n_base) * dsplit);
}

// ------------------------------------------------------------------------------------------
// The persistent kernel
// ------------------------------------------------------------------------------------------
// The body of one launch. CHAIN: a chained launch over L linears (lins, device), each linear's items
// after the previous linear's, one global pipeline; a linear's X loads wait for the previous linear's
// last combined Y row (the weights stream ahead). Otherwise one linear (a0 / xmap0, kernel params).
template <bool FUSED, int NTS, bool CHAIN>
__device__ __forceinline__ void sbmm_body(const dz_sbmm_args& a0, const CUtensorMap* xmap0, const ChainLin* lins,
                                          int L) {
  auto lin = [&](int l) -> const dz_sbmm_args& { return CHAIN ? lins[l].a : a0; };
  const dz_sbmm_args& a = a0;  // launch-wide fields (workspace) and the single-linear case
  extern __shared__ uint8_t smem_dyn[];
  constexpr int STAGE_BYTES = stage_bytes<NTS>();
  // 1024-B alignment for the SWIZZLE_128B tiles
  uint8_t* stages = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
  Smem* sm = reinterpret_cast<Smem*>(stages + STAGE_BYTES * NSTAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int* sched = reinterpret_cast<int*>(a.workspace);  // [0] item counter, [1] finished CTAs
  int* chain = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(a.workspace) + DZ_WS_CHAIN_OFF);
  int* chain_cnt = chain + 1;               // per-linear item counters (chained launch)
  int* chain_done = chain + 1 + MAX_CHAIN;  // per-linear combined delta items (chained launch)

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; s++) {
      mbar_init(&sm->full[s], 1);
      mbar_init(&sm->empty[s], NW + 1);  // consumer warps + the MMA warp (commit or arrive)
      mbar_init(&sm->xreq[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&sm->tmem_full[b], 1);
      mbar_init(&sm->tmem_empty[b], NW);
    }
    for (int r = 0; r < MREC; r++) {
      mbar_init(&sm->mfull[r], NW);
      mbar_init(&sm->mempty[r], 1);
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
    // ===================== TMA producer =====================
    int trace_i = 0;
    (void)trace_i;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int l = 0; l < L; l++) {
    // chained launch: the linear's arguments live in global memory, whose L1 lines every acquire
    // poll invalidates; a register copy keeps them off the per-stage path (kernel params otherwise)
    std::conditional_t<CHAIN, const dz_sbmm_args, const dz_sbmm_args&> a = lin(l);
    const CUtensorMap* xmap = CHAIN ? &lins[l].xmap : xmap0;
    if (lane == 0) prefetch_tmap(xmap);
    const LinGeo geo = lin_geo(a);
    const int nrt = geo.nrt, nkb = geo.nkb, nbt = geo.nbt, n_base = geo.n_base, bn = geo.bn, bch = geo.bch;
    const int nsplit = geo.nsplit, dsplit = geo.dsplit;
    int* item_cnt = CHAIN ? chain_cnt + l : &sched[0];
    bool dep_ready = !CHAIN || l == 0;  // X of this linear = Y of the previous one
    // First item static (blockIdx.x), later ones from the counter. Before waiting for the preceding
    // kernel (programmatic dependent launch), prefetch the first chunks of this item's weight
    // stream into L2: it depends only on resident weights, not on the predecessor's output.
    // A device plan (n_jobs_dev) is the predecessor's output: nothing of it is read before the wait.
    int item = blockIdx.x;
    int rt = 0, jj = 0, sp = 0;
    int n_jobs = a.n_jobs;
    int n_items = job_items(a, n_jobs, n_base, nrt, nbt, nsplit, dsplit);
    dz_job job = dz_job{0, 0, 0, 0};
    if (a.n_jobs_dev == nullptr && item < n_items) {
      item_coords(item, nrt, nbt, nsplit, dsplit, n_jobs, n_base, rt, jj, sp);
      job = a.jobs[jj];
    }
    if (a.n_jobs_dev == nullptr && item < n_items && lane == 0) {
      const bool dn = kind_dense(job.kind);
      const dz_native_delta* e0 = job.kind == 0 ? a.base : a.table + job.slot;
      const void* m0 = e0->tmap;
      if (job.kind == 0) {
        int k0, k1;
        base_chunks(a.in, sp, nsplit, k0, k1);
        for (int c = k0; c < k0 + PF_CHUNKS * bch && c < k1; c++) tma_prefetch_2d(m0, c * KC_DN, rt * BASE_RT);
      } else if (dn) {
        const int d0 = sp * (2 * nkb) / dsplit;
        for (int c = d0; c < d0 + PF_CHUNKS && c < 2 * nkb; c++) tma_prefetch_2d(m0, c * (DN_HALF / 8), rt * RG);
      } else {
        const int d0 = sp * ceil_div(nkb, NB_SP) / dsplit;
        for (int c = d0; c < d0 + PF_CHUNKS && c * NB_SP < nkb; c++) tma_prefetch_3d(m0, 0, c * NB_SP, rt * RG);
      }
    }
    if (l == 0) {
      griddep_wait();
      griddep_launch_dependents();
    }
    if (a.n_jobs_dev != nullptr) {  // dz_plan_device wrote the count and the jobs
      n_jobs = *a.n_jobs_dev;
      n_items = job_items(a, n_jobs, n_base, nrt, nbt, nsplit, dsplit);
      if (item < n_items) {
        item_coords(item, nrt, nbt, nsplit, dsplit, n_jobs, n_base, rt, jj, sp);
        job = a.jobs[jj];
      }
    }
    int tok = 0, tok2 = 0;
    if (item < n_items) {
      if (lane < job.tok_count) tok = job.kind == 0 ? job.tok_begin + lane : a.order[job.tok_begin + lane];
      if (lane + 32 < job.tok_count)
        tok2 = job.kind == 0 ? job.tok_begin + lane + 32 : a.order[job.tok_begin + lane + 32];
    }
    while (item < n_items) {
      const bool is_base = job.kind == 0;
      const bool dense = kind_dense(job.kind);
      const dz_native_delta* ent = is_base ? a.base : a.table + job.slot;
      const void* amap = ent->tmap;  // address only: the descriptor stays in global memory
      const int bb = dense ? kDenseBlockBytes : sparse_block_bytes(kind_fbits(job.kind));
      // base items stream the K-chunks [kb0, kb1) of split sp, bch per stage; delta items stages
      // [c0, c0 + nch) of split sp
      int kb0 = 0, kb1 = 0;
      if (is_base) base_chunks(a.in, sp, nsplit, kb0, kb1);
      const int nch_all = dense ? 2 * nkb : ceil_div(nkb, NB_SP);
      const int c0 = is_base ? 0 : sp * nch_all / dsplit;
      const int nch = is_base ? ceil_div(kb1 - kb0, bch) : (sp + 1) * nch_all / dsplit - c0;
      const uint32_t abytes = is_base ? static_cast<uint32_t>(BASE_RT * KC_DN * 2)
                              : dense ? static_cast<uint32_t>(A_DN) : static_cast<uint32_t>(RG * NB_SP * bb);
      // Next item: its id is fetched after chunk 0 goes out (one item of lookahead per CTA keeps
      // the dynamic schedule balanced), its descriptor and token ids after chunks 1 and 2, so the
      // dependent global loads overlap this item's stream instead of stalling the ring.
      int id_nxt_raw = 0, item_nxt = n_items, tok_n = 0, tok2_n = 0, rt_n = 0, sp_n = 0;
      dz_job job_n{0, 0, 0, 0};
      for (int ch = 0; ch < nch; ch++) {
        if (lane == 0) TRACE(1, item, ch);
        if (lane == 0 && ch == 0)
          ITEM_TRACE(2, item, (static_cast<unsigned long long>(blockIdx.x) << 32) | static_cast<uint32_t>(job.kind));
        mbar_wait(&sm->empty[stage], phase ^ 1);
        if (lane == 0 && ch == 0) ITEM_TRACE(0, item, globaltimer());
        if (lane == 0) TRACE(2, item, ch);
        uint8_t* sbuf = stages + static_cast<size_t>(stage) * STAGE_BYTES;
        int nb, col0, xbytes, ax, ay;
        if (is_base) {
          col0 = (kb0 + ch * bch) * KC_DN;
          nb = cmin(bch, kb1 - (kb0 + ch * bch));  // K-chunks in this stage (none fully out of bounds)
          xbytes = 0;
          ax = col0;
          ay = rt * BASE_RT;
        } else if (dense) {
          nb = 1;
          col0 = (c0 + ch) * KC_DN;
          xbytes = KC_DN * 2;
          ax = (c0 + ch) * (DN_HALF / 8);
          ay = rt * RG;
        } else {
          const int kb0 = (c0 + ch) * NB_SP;
          nb = (nkb - kb0) < NB_SP ? (nkb - kb0) : NB_SP;
          col0 = kb0 * kBlkCols;
          xbytes = nb * kBlkCols * 2;
          ax = kb0;  // 3-D box {block bytes, NB_SP blocks, RG row groups}: coords (0, kb0, rg0)
          ay = rt * RG;
        }
        const bool last = ch == nch - 1;
        if (!is_base || last) {  // token ids: the X producer's gather list / the epilogue's scatter list
          if (lane < job.tok_count) sm->tok_ids[stage][lane] = tok;
          if (lane + 32 < job.tok_count) sm->tok_ids[stage][lane + 32] = tok2;
          __syncwarp();
        }
        if (lane == 0) {
          StageHdr h;
          h.item = item; h.rt = rt; h.kind = job.kind;
          h.tok_begin = job.tok_begin; h.tok_count = job.tok_count; h.nb = nb;
          // bits 2-4: bn / 32 of a base stage (the MMA's N and X layout); bits 8+: absolute chunk (X producer)
          h.flags = (ch == 0 ? 1 : 0) | (last ? 2 : 0) | (is_base ? (bn >> 5) << 2 : 0) | ((c0 + ch) << 8);
          h.pad = sp;  // K-split of the item: selects the partial plane its epilogue writes
          h.lin = CHAIN ? l : 0;
          sm->hdr[stage] = h;
          const uint32_t xb = is_base ? static_cast<uint32_t>(nb * KC_DN * bn * 2)
                                      : static_cast<uint32_t>(job.tok_count * xbytes);
          TRACE(6, item, ch);
          mbar_arrive_expect_tx(&sm->full[stage], (is_base ? nb : 1) * abytes + xb);  // release: orders the smem writes above
          TRACE(7, item, ch);
          if (is_base) {
            for (int c = 0; c < nb; c++)
              tma_load_2d(sbuf + c * (BASE_RT * KC_DN * 2), amap, ax + c * KC_DN, ay, &sm->full[stage], pol_stream);
            if (CHAIN && !dep_ready) {  // the weights are in flight; X waits for the previous linear
              wait_linear(chain_done + l - 1, delta_items(lin(l - 1)));
              dep_ready = true;
            }
            for (int c = 0; c < nb; c++)
              tma_load_2d(sbuf + base_xoff(bch) + c * (KC_DN * bn * 2), xmap, col0 + c * KC_DN, job.tok_begin,
                          &sm->full[stage], pol_keep);
          } else if (dense) {
            tma_load_2d(sbuf, amap, ax, ay, &sm->full[stage], pol_stream);
          } else {
            tma_load_3d(sbuf, amap, 0, ax, ay, &sm->full[stage], pol_stream);
          }
          TRACE(8, item, ch);
          mbar_arrive(&sm->xreq[stage]);  // release: header + token ids are visible to the X producer
        }
        if (lane == 0) TRACE(9, item, ch);
        if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
        // ---- next-item prefetch, spread over the first chunks ----
        if (ch == 0 && lane == 0) id_nxt_raw = static_cast<int>(gridDim.x) + atomicAdd(item_cnt, 1);
        if (ch == (nch > 1 ? 1 : 0)) {
          item_nxt = __shfl_sync(0xffffffffu, id_nxt_raw, 0);
          if (item_nxt < n_items) {
            int j_n = 0;
            item_coords(item_nxt, nrt, nbt, nsplit, dsplit, n_jobs, n_base, rt_n, j_n, sp_n);
            job_n = a.jobs[j_n];
            if (lane == 0) prefetch_tmap((job_n.kind == 0 ? a.base : a.table + job_n.slot)->tmap);
          }
        }
        if (ch == (nch > 2 ? 2 : nch - 1) && item_nxt < n_items) {
          if (lane < job_n.tok_count)
            tok_n = job_n.kind == 0 ? job_n.tok_begin + lane : a.order[job_n.tok_begin + lane];
          if (lane + 32 < job_n.tok_count)
            tok2_n = job_n.kind == 0 ? job_n.tok_begin + lane + 32 : a.order[job_n.tok_begin + lane + 32];
        }
      }
      item = item_nxt;
      rt = rt_n;
      sp = sp_n;
      job = job_n;
      tok = tok_n;
      tok2 = tok2_n;
    }
    }  // linears
    if (!CHAIN && a.next != nullptr && lane == 0) tail_prefetch(*a.next);
    mbar_wait(&sm->empty[stage], phase ^ 1);
    if (lane == 0) {
      sm->hdr[stage].item = -1;
      mbar_arrive(&sm->xreq[stage]);
      mbar_arrive(&sm->full[stage]);
      if (!CHAIN) {
        const int done = atomicAdd(&sched[1], 1);
        if (done == static_cast<int>(gridDim.x) - 1) {  // last CTA out resets the scheduler
          sched[0] = 0;
          sched[1] = 0;
        }
      }
    }
  } else if (warp == WARP_XPROD) {
    // ===================== X producer (delta stages) =====================
    // One 1-D bulk copy per routed token row of the chunk, completing on the stage's full barrier
    // (whose expect_tx the producer already armed with these bytes).
    const uint64_t pol_keep = policy_evict_last();
    griddep_wait();  // X is the preceding kernel's output
    int stage = 0;
    uint32_t phase = 0;
    int dep_l = 0;  // chained launch: the X of linears <= dep_l is known to be complete
    int x_l = 0;    // linear of xg / ldx
    const uint16_t* xg = lin(0).X;
    int64_t ldx = lin(0).ldx;
    while (true) {
      mbar_wait(&sm->xreq[stage], phase);
      const StageHdr h = sm->hdr[stage];
      if (h.item < 0) break;
      if (h.kind != 0) {
        if (CHAIN && h.lin != x_l) {
          x_l = h.lin;
          xg = lin(x_l).X;
          ldx = lin(x_l).ldx;
        }
        if (CHAIN && h.lin > dep_l) {
          wait_linear(chain_done + h.lin - 1, delta_items(lin(h.lin - 1)));
          dep_l = h.lin;
        }
        const bool dense = h.kind == DZ_KIND_DENSE;
        const int col0 = dense ? (h.flags >> 8) * KC_DN : (h.flags >> 8) * NB_SP * kBlkCols;
        const int xbytes = dense ? KC_DN * 2 : h.nb * kBlkCols * 2;
        const int aoff = dense ? A_DN : A_SP;
        const int xs = dense ? XS_DN : XS_SP;
        uint8_t* sbuf = stages + static_cast<size_t>(stage) * STAGE_BYTES;
        for (int tk = lane; tk < h.tok_count; tk += 32)
          tma_load_1d(sbuf + aoff + tk * xs, xg + static_cast<int64_t>(sm->tok_ids[stage][tk]) * ldx + col0,
                      static_cast<uint32_t>(xbytes), &sm->full[stage], pol_keep);
      }
      if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
    }
  } else if (warp == WARP_MMA) {
    // ===================== tcgen05 issuer =====================
    int stage = 0;
    uint32_t phase = 0;
    int nbase = 0;  // base items seen (selects the TMEM accumulator buffer and its phase)
    while (true) {
      mbar_wait(&sm->full[stage], phase);
      const StageHdr h = sm->hdr[stage];
      if (h.item < 0) break;
      if (h.kind == 0) {
        const int buf = nbase & 1;
        const uint32_t acc_phase = (nbase >> 1) & 1;
        if (h.flags & 1) mbar_wait(&sm->tmem_empty[buf], acc_phase ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sbuf = smem_u32(stages + static_cast<size_t>(stage) * STAGE_BYTES);
          const uint32_t tmem_d = tmem_base + buf * BASE_N;
          const int bn = ((h.flags >> 2) & 7) << 5;
          const int xoff = base_xoff(base_bch(bn));
          const uint32_t idesc = umma_idesc_bf16(UMMA_M, bn);
          for (int c = 0; c < h.nb; c++) {
            const uint64_t adesc = umma_desc_sw128(sbuf + c * (BASE_RT * KC_DN * 2));
            const uint64_t bdesc = umma_desc_sw128(sbuf + xoff + c * (KC_DN * bn * 2));
#pragma unroll
            for (int k = 0; k < KC_DN / 16; k++)  // K=16 per MMA: +32 B inside the 128-B swizzle atom
              umma_bf16(tmem_d, adesc + 2 * k, bdesc + 2 * k, idesc, (h.flags & 1) && c == 0 && k == 0 ? 0u : 1u);
          }
          umma_commit(&sm->empty[stage]);
          if (h.flags & 2) umma_commit(&sm->tmem_full[buf]);
        }
        __syncwarp();
        if (h.flags & 2) nbase++;
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm->empty[stage]);
      }
      if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
    }
  } else if (FUSED && warp == WARP_COMB) {
    // ===================== combiner (fused merge) =====================
    griddep_wait();
    int cur_l = 0;
    const LinGeo g0 = lin_geo(lin(0));
    MergeCtx mctx = make_mctx<FUSED>(lin(0), g0);
    mctx.readers = (lin(0).n_jobs_dev != nullptr ? *lin(0).n_jobs_dev : lin(0).n_jobs) - g0.n_base;  // delta jobs
    if (mctx.fused) {
      const MergeRec* recs = reinterpret_cast<const MergeRec*>(sm->recs);
      for (int k = 0;; k++) {
        while (!mbar_test(&sm->mfull[k % MREC], (k / MREC) & 1)) __nanosleep(DZ_COMB_SLEEP);
        const int rl = recs[k % MREC].lin, rbase = recs[k % MREC].is_base;
        if (CHAIN && rl != cur_l && recs[k % MREC].rt >= 0) {
          cur_l = rl;
          const LinGeo g = lin_geo(lin(rl));
          mctx = make_mctx<FUSED>(lin(rl), g);
          mctx.readers = (lin(rl).n_jobs_dev != nullptr ? *lin(rl).n_jobs_dev : lin(rl).n_jobs) - g.n_base;
        }
        if (!service_record(sm, mctx, k, lane)) break;
        // chained launch: count the delta item's Y rows as written (release: its stores first)
        if (CHAIN && !rbase && lane == 0)
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(chain_done + rl) : "memory");
      }
    }
  } else {
    // ===================== consumers =====================
    griddep_wait();  // Y / merge slots may still be in use by the preceding kernel
    int trace_i = 0;
    (void)trace_i;
    float acc[MR][NT_DN][4];  // dense deltas use all NT_DN tiles, sparse deltas the first NTS
    int stage = 0;
    uint32_t phase = 0;
    int nbase = 0;
    int cur_l = 0;
    LinGeo geo = lin_geo(lin(0));
    MergeCtx mctx = make_mctx<FUSED>(lin(0), geo);
    int c_debug = lin(0).debug, c_out = lin(0).out;  // register copies (chained launch: global memory)
    int nmerge = 0;  // items merged so far (record ring position)
    MergeRec* recs = reinterpret_cast<MergeRec*>(sm->recs);
    while (true) {
      mbar_wait(&sm->full[stage], phase);
      const StageHdr h = sm->hdr[stage];
      if (lane == 0 && warp == 0) TRACE(3, h.item, stage);
      if (h.item < 0) {
        if (mctx.fused) publish_item(recs, sm->mfull, sm->mempty, nmerge, warp, lane, -1, 0, 0, 0);
        break;
      }
      if (CHAIN && h.lin != cur_l) {  // the next linear of a chained launch
        cur_l = h.lin;
        geo = lin_geo(lin(cur_l));
        mctx = make_mctx<FUSED>(lin(cur_l), geo);
        c_debug = lin(cur_l).debug;
        c_out = lin(cur_l).out;
      }
      const int n16 = geo.n16, nsplit = geo.nsplit;
      const bool is_base = h.kind == 0;
      const int rg0 = h.rt * RG + warp * MR;
      const int nrv = (n16 - rg0) < MR ? (n16 - rg0) : MR;  // row groups of this warp inside `out`
      const uint32_t sbuf = smem_u32(stages + static_cast<size_t>(stage) * STAGE_BYTES);
      const int nt = ceil_div(h.tok_count, 8);
      if (!is_base && !(c_debug & 1)) {
        if (h.flags & 1) {
#pragma unroll
          for (int r = 0; r < MR; r++)
#pragma unroll
            for (int n = 0; n < NT_DN; n++) acc[r][n][0] = acc[r][n][1] = acc[r][n][2] = acc[r][n][3] = 0.f;
        }
        if (nrv > 0) {
          if (h.kind == DZ_KIND_DENSE) {
            dense_dispatch(nt, acc, sbuf + warp * MR * DN_HALF, sbuf + A_DN, nrv, lane);
          } else {
            const uint32_t xl = sbuf + A_SP + (lane & 7) * XS_SP + (lane >> 3) * 16;
            const uint32_t off = 0x4300u + static_cast<uint32_t>(kind_qmax(h.kind));  // bf16(128 + qmax)
            const uint32_t off2 = off | (off << 16);
            if (h.kind != DZ_KIND_SPARSE2) {
              const uint32_t sA = sbuf + warp * MR * NB_SP * sparse_block_bytes(4);
              if (NTS == 1 || nt <= 1)
                sparse_chunk<4, 1>(acc, sA, xl, h.nb, nrv, off2, lane);
              else
                sparse_chunk<4, NTS>(acc, sA, xl, h.nb, nrv, off2, lane);
            } else {
              const uint32_t sA = sbuf + warp * MR * NB_SP * sparse_block_bytes(2);
              if (NTS == 1 || nt <= 1)
                sparse_chunk<2, 1>(acc, sA, xl, h.nb, nrv, off2, lane);
              else
                sparse_chunk<2, NTS>(acc, sA, xl, h.nb, nrv, off2, lane);
            }
          }
        }
      }
      int tkn[NTS][2] = {};  // this lane's token ids per n-tile (sparse epilogue), read before release
      if ((h.flags & 2) && !is_base) {
        const int t2 = 2 * (lane & 3);
#pragma unroll
        for (int n = 0; n < NTS; n++) {
          if (8 * n + t2 < h.tok_count) tkn[n][0] = sm->tok_ids[stage][8 * n + t2];
          if (8 * n + t2 + 1 < h.tok_count) tkn[n][1] = sm->tok_ids[stage][8 * n + t2 + 1];
        }
      }
      if ((h.flags & 2) && h.kind == DZ_KIND_DENSE && nrv > 0)  // rare path: needs the stage's token list
        merge_fragments(acc, nt, mctx, nsplit + h.pad, rg0, h.tok_count, sm->tok_ids[stage], lane);
      const int rtok = ((h.flags & 2) && !is_base && lane < h.tok_count && lane < 32) ? sm->tok_ids[stage][lane] : 0;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm->empty[stage]);  // the stage is free before the epilogue
      if (lane == 0 && warp == 0) TRACE(4, h.item, stage);
      if (++stage == NSTAGE) { stage = 0; phase ^= 1; }

      if (h.flags & 2) {
        // ---- item epilogue: this warp's contributions -> merged into Y ----
        if (is_base) {
          const int buf = nbase & 1;
          mbar_wait(&sm->tmem_full[buf], (nbase >> 1) & 1);
          tc_fence_after();
          if (geo.bn == BASE_N)
            drain_base_accumulator<BASE_N>(tmem_base + buf * BASE_N, warp, lane, mctx, h.pad, h.rt * BASE_RT,
                                           h.tok_begin, h.tok_count);
          else  // bn = 32 (or 64 with DZ_BASE_BN64; columns at or past tcount are skipped)
            drain_narrow(tmem_base + buf * BASE_N, warp, lane, mctx, h.pad, h.rt * BASE_RT, h.tok_begin, h.tok_count);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm->tmem_empty[buf]);
          nbase++;
        } else if (nrv > 0 && h.kind != DZ_KIND_DENSE) {
          const int g = lane >> 2, t2 = 2 * (lane & 3);
#pragma unroll
          for (int n = 0; n < NTS; n++) {
            if (8 * n >= h.tok_count) break;
            int tk[4 * MR], rw[4 * MR];
            float x[4 * MR];
            bool ok[4 * MR];
#pragma unroll
            for (int r = 0; r < MR; r++) {
              const int row = (rg0 + r) * kBlkRows + g;
#pragma unroll
              for (int v = 0; v < 4; v++) {  // fragment: v&1 -> token t2 / t2+1, v&2 -> row +8
                const int i = 4 * r + v;
                tk[i] = tkn[n][v & 1];
                rw[i] = row + ((v & 2) ? 8 : 0);
                x[i] = acc[r][n][v];
                ok[i] = r < nrv && 8 * n + t2 + (v & 1) < h.tok_count && rw[i] < c_out;
              }
            }
            merge_batch<4 * MR>(mctx, nsplit + h.pad, tk, rw, x, ok);
          }
        }
        if (mctx.fused) {  // hand the item to the combiner warp (no wait on any round trip)
          publish_item(recs, sm->mfull, sm->mempty, nmerge, warp, lane, h.rt, is_base ? 1 : 0, is_base ? 0 : h.tok_count,
                       rtok, h.lin);
          nmerge++;
        }
        if (lane == 0 && warp == 0) TRACE(5, h.item, 0);
        if (lane == 0 && warp == 0) ITEM_TRACE(1, h.item, globaltimer());
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
  if (CHAIN && threadIdx.x == 0) {  // every role of this CTA is done: the last CTA re-arms the chain
    __threadfence();
    if (atomicAdd(chain, 1) == static_cast<int>(gridDim.x) - 1) {
      for (int l = 0; l < L; l++) {
        chain_cnt[l] = 0;
        chain_done[l] = 0;
      }
      chain[0] = 0;
    }
  }
}

template <bool FUSED, int NTS>
__global__ void __launch_bounds__(nthreads<FUSED>(), 1)
    k_sbmm(const __grid_constant__ dz_sbmm_args a, const __grid_constant__ CUtensorMap xmap) {
  sbmm_body<FUSED, NTS, false>(a, &xmap, nullptr, 1);
}

// Chained launch: L linears of a decode step in one persistent kernel (fused merge).
template <int NTS>
__global__ void __launch_bounds__(nthreads<true>(), 1) k_sbmm_chain(const ChainLin* __restrict__ lins, int L) {
  sbmm_body<true, NTS, true>(lins[0].a, &lins[0].xmap, lins, L);
}

}  // namespace dz

using namespace dz;

static_assert(base_stage_bytes(32) <= stage_bytes<1>() && base_stage_bytes(64) <= stage_bytes<1>() &&
                  base_stage_bytes(BASE_N) <= stage_bytes<1>() && BASE_N % 32 == 0,
              "base stage layout");
static_assert(NB_SP % PAIR1 == 0, "sparse stages hold whole block pairs");
static_assert(DZ_SPARSE_JOB_TOKENS % 8 == 0 && NT_SP >= 1 && NT_SP <= NT_DN, "2:4 job = whole n-tiles");
static_assert(smem_bytes<NT_SP>() <= 232448, "shared memory per CTA");
static_assert(sizeof(MergeRec) == 36 * sizeof(int) && MREC <= 8, "MergeRec ring layout in Smem");
static_assert(NW == 8 && MR == 2, "8 consumer warps of 32 rows (one 32-row output slice each)");
static_assert(sizeof(dz_native_delta) == 192, "dz_native_delta must be 192 bytes");
static_assert(offsetof(dz_native_delta, tmap) == 64, "tensor map must be 64-byte aligned in the entry");
static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");

extern "C" int dz_native_delta_init(dz_native_delta* e, const void* blocks, int32_t kind, int32_t rows, int32_t cols) {
  if (!e || !blocks) return DZ_E_VALUE;
  if (rows < 1 || cols < 1) return DZ_E_SHAPE;
  if (kind != DZ_KIND_SPARSE4 && kind != DZ_KIND_SPARSE2 && kind != DZ_KIND_SPARSE3 && kind != DZ_KIND_DENSE)
    return DZ_E_VALUE;
  if (reinterpret_cast<uintptr_t>(blocks) & 15) return DZ_E_VALUE;
  std::memset(e, 0, sizeof(*e));
  e->blocks = blocks;
  e->kind = kind;
  e->qmax = kind == DZ_KIND_DENSE ? 0 : kind_qmax(kind);
  e->rows = rows;
  e->cols = cols;
  const int nkb = ceil_div(cols, kBlkCols), n16 = ceil_div(rows, kBlkRows);
  if (kind == DZ_KIND_DENSE)
    return encode_2d(reinterpret_cast<CUtensorMap*>(e->tmap), CU_TENSOR_MAP_DATA_TYPE_UINT64, blocks,
                     static_cast<uint64_t>(nkb) * kDenseBlockBytes / 8, static_cast<uint64_t>(n16),
                     static_cast<uint64_t>(nkb) * kDenseBlockBytes, DN_HALF / 8, RG, CU_TENSOR_MAP_SWIZZLE_NONE);
  // sparse: 3-D view {block bytes / 8, blocks along K, row groups}; one box = NB_SP blocks x RG groups
  const int bb = sparse_block_bytes(kind_fbits(kind));
  EncodeTiledFn fn = encode_fn();
  if (!fn) return DZ_E_CUDA;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(bb / 8), static_cast<cuuint64_t>(nkb),
                              static_cast<cuuint64_t>(n16)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(bb), static_cast<cuuint64_t>(nkb) * bb};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(bb / 8), NB_SP, RG};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(reinterpret_cast<CUtensorMap*>(e->tmap), CU_TENSOR_MAP_DATA_TYPE_UINT64, 3,
                        const_cast<void*>(blocks), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? DZ_OK : DZ_E_CUDA;
}

extern "C" int dz_base_init(dz_native_delta* e, const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols) {
  if (!e || !W) return DZ_E_VALUE;
  if (rows < 1 || cols < 1 || ldw < cols) return DZ_E_SHAPE;
  if ((reinterpret_cast<uintptr_t>(W) & 15) || (ldw % 8)) return DZ_E_SHAPE;  // TMA: 16-B rows
  std::memset(e, 0, sizeof(*e));
  e->blocks = W;
  e->kind = 0;
  e->rows = rows;
  e->cols = cols;
  return encode_2d(reinterpret_cast<CUtensorMap*>(e->tmap), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, W,
                   static_cast<uint64_t>(cols), static_cast<uint64_t>(rows), static_cast<uint64_t>(ldw) * 2, KC_DN,
                   BASE_RT, CU_TENSOR_MAP_SWIZZLE_128B);  // one box = 64 columns x 128 rows (one UMMA M tile)
}

extern "C" size_t dz_sbmm_workspace_bytes(int32_t T, int32_t out) {
  if (T < 0 || out < 1 || out > 32 * MAX_SLICES) return 0;
  return DZ_WS_PART_OFF + static_cast<size_t>(T) * out * sizeof(float) * 6;  // <= 4 base + 2 delta K-split planes
}

extern "C" int dz_sbmm_diag(int* v) {  // numRegs, static smem, dynamic smem, max threads, localBytes
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_sbmm<false, 1>) != cudaSuccess) return -1;
  v[0] = fa.numRegs; v[1] = static_cast<int>(fa.sharedSizeBytes); v[2] = SMEM_BYTES;
  v[3] = fa.maxThreadsPerBlock; v[4] = static_cast<int>(fa.localSizeBytes);
  size_t avail = 0;
  cudaFuncSetAttribute(k_sbmm<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  cudaOccupancyAvailableDynamicSMemPerBlock(&avail, k_sbmm<false, 1>, 2, NTHREADS);
  v[5] = static_cast<int>(avail);
  cudaFuncSetAttribute(k_sbmm<false, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_sbmm<false, 1>, NTHREADS, SMEM_BYTES);
  v[6] = n;
  return 0;
}

extern "C" int dz_sbmm_ctas_per_sm(void) {
  int n = 0;
  if (cudaFuncSetAttribute(k_sbmm<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess) return -1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_sbmm<false, 1>, NTHREADS, SMEM_BYTES) != cudaSuccess) return -1;
  return n;
}

extern "C" int dz_tp_finalize_launch(const float* part, int nsplit, int T, int out, const dz_tp_ctx* ctx, void* Y,
                                     int64_t ldy, int y_dtype, int act, void* stream);

// Host side of one K2 launch. The K-split counts come from the caller or from the shape alone
// (never from the batch, so a token's result does not depend on the other tokens of the call).
static int launch_decode(const dz_sbmm_args* a_in, void* stream) {
  dz_sbmm_args kargs = *a_in;
  const dz_sbmm_args* a = &kargs;
  resolve_splits(kargs.out, kargs.in, kargs.base != nullptr, kargs.base_splits, kargs.delta_splits);
  const bool tp = a->tp != nullptr && a->tp->world > 1;
  kargs.keep_planes = tp ? 1 : 0;  // row-parallel shard: the peer-memory reduction reads the planes
  // must match MergeCtx::fused in the kernel: the combiner warp writes Y (no k_finalize launch)
  const bool fused = a->fused_merge != 0 && a->base != nullptr && !tp && kargs.delta_splits == 1 && !(a->debug & 6);
  // One-time, idempotent kernel attribute setup (the only process-wide state; no per-call state).
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  static int ctas_per_sm = 1;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_sbmm<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<1>());
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(k_sbmm<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<1>());
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(k_sbmm<false, NT_SP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      smem_bytes<NT_SP>());
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(k_sbmm<true, NT_SP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      smem_bytes<NT_SP>());
    if (attr_err == cudaSuccess)
      attr_err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, k_sbmm<false, 1>, NTHREADS, SMEM_BYTES);
    if (ctas_per_sm < 1) ctas_per_sm = 1;
  });
  if (attr_err != cudaSuccess) return DZ_E_CUDA;
  CUtensorMap xmap;  // X [T][in] bf16, 64-column x 128-token SWIZZLE_128B tiles (base UMMA B operand)
  int st = encode_2d(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a->X, static_cast<uint64_t>(a->in),
                     static_cast<uint64_t>(a->T), static_cast<uint64_t>(a->ldx) * 2, KC_DN, base_bn(a->T),
                     CU_TENSOR_MAP_SWIZZLE_128B);
  if (st) return st;
  int grid = a->grid;
  if (grid <= 0) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return DZ_E_CUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return DZ_E_CUDA;
    grid = sms * ctas_per_sm;
  }
  const int n_items = ceil_div(a->out, RT) * a->n_jobs * a->delta_splits +
                      ceil_div(a->out, BASE_RT) * a->base_splits * ceil_div(a->T, BASE_N);
  if (grid > n_items) grid = n_items;
  // the narrow instantiation when the plan's 2:4 jobs have <= 8 tokens (a smaller X stage)
  const bool narrow = a->sparse_job_tokens == 8;
  if (fused)
    st = narrow ? launch_pdl(1, k_sbmm<true, 1>, grid, nthreads<true>(), smem_bytes<1>(), stream, *a, xmap)
                : launch_pdl(1, k_sbmm<true, NT_SP>, grid, nthreads<true>(), smem_bytes<NT_SP>(), stream, *a, xmap);
  else
    st = narrow ? launch_pdl(1, k_sbmm<false, 1>, grid, NTHREADS, smem_bytes<1>(), stream, *a, xmap)
                : launch_pdl(1, k_sbmm<false, NT_SP>, grid, NTHREADS, smem_bytes<NT_SP>(), stream, *a, xmap);
  if (st || fused || a->base == nullptr || (a->debug & 4)) return st;
  const float* part = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(a->workspace) + DZ_WS_PART_OFF);
  if (tp)  // row-parallel shard: fused reduction over peer memory
    return dz_tp_finalize_launch(part, a->base_splits + a->delta_splits - 1, a->T, a->out, a->tp, a->Y, a->ldy,
                                 a->y_dtype, a->act, stream);
  // every partial in planes, summed by k_finalize in a fixed order (base splits, then delta splits)
  const int64_t work = static_cast<int64_t>(a->T - a->t_pf) * a->out / 4;
  int fgrid = static_cast<int>((work + 255) / 256);
  fgrid = fgrid > 4 * 148 ? 4 * 148 : fgrid < 1 ? 1 : fgrid;
  return launch_pdl(2, k_finalize, fgrid, 256, 0, stream, part, a->base_splits + a->delta_splits - 1, a->t_pf, a->T,
                    a->out, a->perm, a->Y, a->ldy, a->y_dtype, a->act,
                    a->pf_counts_dev != nullptr ? a->pf_counts_dev + 2 : static_cast<const int32_t*>(nullptr));
}

extern "C" int dz_sbmm(const dz_sbmm_args* a, void* stream) {
  if (!a) return DZ_E_VALUE;
  if (a->T < 0 || a->out < 1 || a->in < 1 || a->out > 32 * MAX_SLICES) return DZ_E_SHAPE;
  if (a->T == 0 || a->n_jobs == 0) return DZ_OK;  // nothing to compute (empty X / Y may be null)
  if (!a->X || !a->Y || !a->workspace) return DZ_E_VALUE;
  if (a->tp != nullptr && a->tp->world > 1 && (a->perm != nullptr || a->base == nullptr))
    return DZ_E_UNSUPPORTED;  // the fused reduction takes decode plans with a base
  const int in_pad = ceil_div(a->in, kBlkCols) * kBlkCols;
  if (a->ldx < in_pad || (a->ldx % 8) != 0 || (reinterpret_cast<uintptr_t>(a->X) & 15) != 0) return DZ_E_SHAPE;
  if (a->ldy < a->out) return DZ_E_SHAPE;
  if (a->y_dtype != DZ_F32 && a->y_dtype != DZ_BF16) return DZ_E_VALUE;
  if (a->perm == nullptr) {
    if (a->n_pf_jobs != 0 || a->t_pf != 0 || a->pf_counts_dev != nullptr) return DZ_E_VALUE;
    return launch_decode(a, stream);
  }
  // mixed plan: stage X in plan order, prefill jobs on K3, the rest on K2 (a device mixed plan
  // passes capacities on the host and the counts in pf_counts_dev)
  if (!a->xs || a->n_pf_jobs < 0 || a->n_pf_jobs > a->n_jobs || a->t_pf < 0 || a->t_pf > a->T) return DZ_E_VALUE;
  const int64_t ldxs = a->ldxs > 0 ? a->ldxs : a->ldx;
  if (ldxs < in_pad || (ldxs % 8) != 0 || (reinterpret_cast<uintptr_t>(a->xs) & 15) != 0) return DZ_E_SHAPE;
  const int parts = a->mixed_parts != 0 ? a->mixed_parts : 7;
  if (parts & ~7) return DZ_E_VALUE;
  int st = DZ_OK;
  if (parts & 1) {
    st = dz_gather_rows(a->X, a->ldx, a->perm, a->T, in_pad, static_cast<uint16_t*>(a->xs), ldxs, stream);
    if (st) return st;
  }
  dz_sbmm_args s = *a;  // the staged buffer replaces X for both kernels
  s.X = static_cast<const uint16_t*>(a->xs);
  s.ldx = ldxs;
  if ((parts & 2) && a->n_pf_jobs > 0) {
    st = dz_sbmm_prefill(&s, stream);
    if (st) return st;
  }
  if ((parts & 4) && a->n_jobs > a->n_pf_jobs) {
    dz_sbmm_args k = s;
    k.jobs = a->jobs + a->n_pf_jobs;
    k.n_jobs = a->n_jobs - a->n_pf_jobs;
    k.n_pf_jobs = 0;
    if (a->pf_counts_dev != nullptr) k.n_jobs_dev = a->pf_counts_dev + 1;  // decode job count
    return launch_decode(&k, stream);
  }
  return DZ_OK;
}


// ------------------------------------------------------------------------------------------
// Chained launch: the linears of a decode step in ONE persistent kernel (see sbmm_body, CHAIN).
// ------------------------------------------------------------------------------------------
extern "C" size_t dz_sbmm_chain_desc_bytes(int32_t L) {
  return L < 1 || L > MAX_CHAIN ? 0 : static_cast<size_t>(L) * sizeof(ChainLin);
}

extern "C" int dz_sbmm_chain_encode(const dz_sbmm_args* args, int32_t L, void* desc_host, size_t desc_bytes,
                                    int32_t* narrow_out) {
  if (!args || !desc_host || !narrow_out || L < 1 || L > MAX_CHAIN) return DZ_E_VALUE;
  if (desc_bytes < dz_sbmm_chain_desc_bytes(L) || (reinterpret_cast<uintptr_t>(desc_host) & 63)) return DZ_E_VALUE;
  ChainLin* lins = static_cast<ChainLin*>(desc_host);
  int narrow = 1;
  for (int l = 0; l < L; l++) {
    const dz_sbmm_args& a = args[l];
    if (!a.X || !a.Y || !a.workspace || !a.base || !a.table || !a.jobs || !a.order) return DZ_E_VALUE;
    if (a.workspace != args[0].workspace) return DZ_E_VALUE;  // one scheduler / plane region for the chain
    if (a.perm != nullptr || a.pf_counts_dev != nullptr || (a.tp != nullptr && a.tp->world > 1) || a.debug)
      return DZ_E_UNSUPPORTED;  // decode plans of single-GPU linears only
    if (a.T < 1 || a.out < 1 || a.in < 1 || a.out > 32 * MAX_SLICES) return DZ_E_SHAPE;
    const int in_pad = ceil_div(a.in, kBlkCols) * kBlkCols;
    if (a.ldx < in_pad || (a.ldx % 8) != 0 || (reinterpret_cast<uintptr_t>(a.X) & 15) != 0 || a.ldy < a.out)
      return DZ_E_SHAPE;
    if (a.y_dtype != DZ_F32 && a.y_dtype != DZ_BF16) return DZ_E_VALUE;
    ChainLin& c = lins[l];
    std::memset(&c, 0, sizeof(c));
    c.a = a;
    resolve_splits(c.a.out, c.a.in, true, c.a.base_splits, c.a.delta_splits);
    if (c.a.delta_splits != 1) return DZ_E_UNSUPPORTED;
    c.a.keep_planes = 0;
    c.a.fused_merge = 1;
    c.a.next = nullptr;
    if (a.sparse_job_tokens != 8) narrow = 0;
    const int st = encode_2d(&c.xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.X, static_cast<uint64_t>(a.in),
                             static_cast<uint64_t>(a.T), static_cast<uint64_t>(a.ldx) * 2, KC_DN, base_bn(a.T),
                             CU_TENSOR_MAP_SWIZZLE_128B);
    if (st) return st;
  }
  *narrow_out = narrow;
  return DZ_OK;
}

extern "C" int dz_sbmm_chain(const void* desc_dev, int32_t L, int32_t narrow, int32_t grid, void* stream) {
  if (!desc_dev || L < 1 || L > MAX_CHAIN || (reinterpret_cast<uintptr_t>(desc_dev) & 63)) return DZ_E_VALUE;
  static std::once_flag once;  // one-time, idempotent kernel attribute setup
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_sbmm_chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<1>());
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(k_sbmm_chain<NT_SP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      smem_bytes<NT_SP>());
  });
  if (attr_err != cudaSuccess) return DZ_E_CUDA;
  if (grid <= 0) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return DZ_E_CUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return DZ_E_CUDA;
    grid = sms;  // one CTA per SM: every CTA must be resident (the chain's waits span CTAs)
  }
  const ChainLin* lins = static_cast<const ChainLin*>(desc_dev);
  return narrow ? launch_pdl(1, k_sbmm_chain<1>, grid, nthreads<true>(), smem_bytes<1>(), stream, lins, L)
                : launch_pdl(1, k_sbmm_chain<NT_SP>, grid, nthreads<true>(), smem_bytes<NT_SP>(), stream, lins, L);
}

#ifdef DZ_TRACE
extern "C" int dz_item_trace_read(unsigned long long* host, int n_items) {
  if (n_items > 65536) n_items = 65536;
  cudaMemcpyFromSymbol(host, dz_item_trace, sizeof(unsigned long long) * 3 * n_items);
  return n_items;
}
// host: copy out {warp, t, ev, a0, a1} tuples of the traced CTA, then reset
extern "C" int dz_trace_read(unsigned long long* host, int max_events) {
  static unsigned long long buf[12][1024][2];
  int cnt[12];
  cudaMemcpyFromSymbol(cnt, dz_trace_cnt, sizeof(cnt));
  cudaMemcpyFromSymbol(buf, dz_trace_buf, sizeof(buf));
  int n = 0;
  for (int w = 0; w < 12; w++)
    for (int i = 0; i < cnt[w] && i < 1024 && n < max_events; i++, n++) {
      host[4 * n + 0] = buf[w][i][0];
      host[4 * n + 1] = (buf[w][i][1] >> 56) | (static_cast<unsigned long long>(w) << 8);
      host[4 * n + 2] = (buf[w][i][1] >> 16) & 0xFFFFFFFFull;
      host[4 * n + 3] = buf[w][i][1] & 0xFFFFull;
    }
  int zero[12] = {0};
  cudaMemcpyToSymbol(dz_trace_cnt, zero, sizeof(zero));
  int neg = -1;
  cudaMemcpyToSymbol(dz_trace_cta, &neg, sizeof(int));
  return n;
}
#endif
