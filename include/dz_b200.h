/*
 * dz_b200.h — C ABI of the B200-native DeltaZip serving hot path.
 *
 * The reference (DeltaZip, arXiv 2312.05215; /root/reference/pkg) is a pure
 * Python/numpy package with no FFI. Each entry point below replaces one
 * reference function on the serving hot path; the citation names it.
 * Plain pointers and sizes only: device pointers are CUDA global memory,
 * `stream` is a cudaStream_t passed as void*. Every call is stream-ordered,
 * never synchronises the host, allocates nothing and keeps no global mutable
 * state, so a whole decode step can be captured in a CUDA graph.
 *
 * Status codes mirror the reference exception contract (errors.py:8-43).
 */
#ifndef DZ_B200_H
#define DZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py) ---------------------------------------------------- */
#define DZ_OK 0
#define DZ_E_SHAPE 1       /* ShapeError      errors.py:8   */
#define DZ_E_ENCODING 2    /* EncodingError   errors.py:12  */
#define DZ_E_FORMAT 3      /* FormatError     errors.py:24  */
#define DZ_E_PARTITION 4   /* PartitionError  errors.py:35  */
#define DZ_E_UNKNOWN 5     /* UnknownDeltaError errors.py:43 */
#define DZ_E_VALUE 6       /* plain ValueError (e.g. scales reshape, compress.py:484) */
#define DZ_E_UNSUPPORTED 7 /* layout the called kernel does not take (caller routes elsewhere) */
#define DZ_E_CUDA 8        /* CUDA runtime error */

/* ---- plan granularity ---------------------------------------------------------------- */
#ifndef DZ_BASE_JOB_TOKENS
#define DZ_BASE_JOB_TOKENS 128 /* tokens per base-GEMM job of the decode kernel (its largest UMMA N; a
                                   launch of <= 32 tokens runs its base stages at N = 32) */
#endif
#define DZ_SPARSE_JOB_TOKENS 16  /* most tokens per 2:4 delta job of the decode kernel (2 mma.sp n-tiles);
                                    the planners take the job width (8 or 16; 0 = 8) as an argument */
#define DZ_DENSE_JOB_TOKENS 32   /* tokens per dense-delta job of the decode kernel */
#ifndef DZ_PREFILL_JOB_TOKENS
#define DZ_PREFILL_JOB_TOKENS 256 /* most tokens per prefill job of K3 (its UMMA N), multiple of 16;
                                    a group is cut into ceil(c / 256) jobs of equal 16-aligned size
                                    (256: one job per 256-token request, single-buffered TMEM
                                    accumulator; profiles/r02_ab_prefill_jobs.txt) */
#endif
/* ---- element types --------------------------------------------------------------- */
#define DZ_F32 0
#define DZ_BF16 1
#define DZ_F64 2   /* K1 only: exact f64 product, bit-identical to dequantize_layer */

/* ---- fused epilogue activations (dz_sbmm) ------------------------------------------ */
#define DZ_ACT_NONE 0
#define DZ_ACT_TANH 1   /* forward_model's tanh between layers (inference.py:288-289) */

/* ---- delta kinds held in a device delta table ------------------------------------ */
#define DZ_KIND_SPARSE4 1  /* 2:4, 4-bit codes (qmax 7) in native blocks                */
#define DZ_KIND_SPARSE2 2  /* 2:4, 2-bit codes (qmax 1) in native blocks                */
#define DZ_KIND_DENSE 3    /* bf16 matrix in the dense native block layout (base weight, or
                              a delta variant the sparse path does not take, dequantised) */
#define DZ_KIND_SPARSE3 4  /* 2:4, 3-bit codes (qmax 3) held in 4-bit fields           */

/* One layer delta in the REFERENCE packed layout (LayerDelta, compress.py:101-143),
 * all pointers device-resident, bytes exactly as the reference stores them. */
typedef struct dz_ref_delta {
  const uint32_t* packed;   /* packed_values, <u4                                  */
  int64_t n_words;
  const uint8_t* index;     /* index_stream (NULL / 0 bytes when sparsity="none")  */
  int64_t index_bytes;
  const float* scales;      /* scales <f4, (rows, n_groups) row-major; may be empty */
  int64_t n_scales;
  int32_t rows, cols, bits, sparse, group_size, _pad;
} dz_ref_delta;

/* One entry of a device delta table consumed by dz_sbmm (192 bytes; arrays of entries must be
 * 64-byte aligned). Fill it on the host with dz_native_delta_init, then copy it to the device. */
typedef struct dz_native_delta {
  const void* blocks;       /* native blocks (dz_repack_sparse / dz_pack_dense_bf16) */
  int32_t kind;             /* DZ_KIND_*                                             */
  int32_t qmax;             /* code offset: u - qmax = code (compress.py:265-277)     */
  int32_t rows, cols;
  uint8_t _reserved[40];
  uint64_t tmap[16];        /* TMA descriptor (CUtensorMap) of `blocks` as a 2-D array */
} dz_native_delta;

/* One unit of SBMM work over a row tile (built by dz_plan). */
typedef struct dz_job {
  int32_t slot;             /* delta-table index; -1 = base GEMM over all tokens     */
  int32_t tok_begin;        /* first position in `order` (delta) or token (base)     */
  int32_t tok_count;        /* <= DZ_BASE_JOB_TOKENS (base), <= DZ_DENSE_JOB_TOKENS (dense delta),
                               <= DZ_SPARSE_JOB_TOKENS (2:4 delta), <= DZ_PREFILL_JOB_TOKENS (prefill) */
  int32_t kind;             /* 0 = base, else DZ_KIND_* of the slot                  */
} dz_job;

typedef struct dz_sbmm_args {
  const uint16_t* X;        /* bf16 [T][ldx]; columns in..ceil128(in) must be zero  */
  int64_t ldx;
  void* Y;                  /* [T][ldy] of y_dtype                                   */
  int64_t ldy;
  int32_t y_dtype;          /* DZ_F32 or DZ_BF16                                     */
  int32_t act;              /* DZ_ACT_*, applied to y = base + delta in the epilogue */
  int32_t T, out, in;
  const dz_native_delta* base; /* device entry (dz_base_init) of W_base [out][in], or NULL */
  const dz_native_delta* table; /* device array [n_slots]                            */
  int32_t n_slots;
  const int32_t* order;     /* device [T]: token indices stably sorted by slot       */
  const dz_job* jobs;       /* device [n_jobs]                                       */
  int32_t n_jobs;
  void* workspace;          /* dz_sbmm_workspace_bytes(T, out) bytes, zeroed once at
                               allocation; the kernel re-zeroes its counters after every call
                               (one workspace per stream: launches on it must not overlap) */
  int32_t grid;             /* persistent CTAs; 0 = one per SM                       */
  int32_t debug;            /* 0; bit 0 = skip consumer math (pipeline bandwidth probe) */
  /* Mixed prefill + decode batches (dz_plan_mixed). perm == NULL: pure decode plan, X is used
   * as is. Otherwise X is first staged into xs with xs[i] = X[perm[i]]; jobs[0:n_pf_jobs] are
   * prefill jobs over staged rows [0, t_pf) (K3: tcgen05 base + dequantised-delta MMAs in one
   * TMEM accumulator), the remaining jobs cover staged rows [t_pf, T) (K2), and staged row i
   * is written to Y row perm[i]. */
  const int32_t* perm;      /* device [T] or NULL                                     */
  void* xs;                 /* device bf16 [T][ldxs] staging buffer (perm != NULL)     */
  int32_t n_pf_jobs;
  int32_t t_pf;
  int64_t ldxs;             /* row stride of xs (elements, >= ceil128(in), % 8 == 0)  */
  int32_t base_splits;      /* K-splits of the base GEMM (1..4); 0 = chosen from (out, in) only,
                               so results never depend on the batch                     */
  int32_t delta_splits;     /* K-splits of each decode delta job (1..2); 0 = from (out, in) only */
  const struct dz_tp_ctx* tp; /* host pointer or NULL: fused tensor-parallel reduction of a
                               row-parallel linear (decode plans only, see dz_tp_ctx)    */
  const int32_t* n_jobs_dev; /* device job count written by dz_plan_device, or NULL; when set,
                               n_jobs is only the capacity of `jobs` (grid sizing)       */
  int32_t keep_planes;      /* set by dz_sbmm (callers leave 0): 1 = leave the fp32 partial planes
                               for the TP peer reduction instead of writing Y in the kernel */
  int32_t prefill_variant;  /* K3 delta product: 0 = 2:4-sparse tcgen05 (default); 1 / 2 =
                               dense-dequantised with 128- / 256-row items (A/B and tests) */
  int32_t fused_merge;      /* 1: Y written inside k_sbmm by a combiner warp per CTA (one launch per
                               linear, no k_finalize); 0 (default): k_finalize sums the partial
                               planes (measured faster, profiles/r02_ab_fused_merge.txt) */
  int32_t mixed_parts;      /* mixed plans: which parts this call runs, bit 0 = stage X into xs,
                               bit 1 = prefill jobs (K3), bit 2 = decode jobs (K2 + merge); 0 = all.
                               Lets a caller run K3 and K2 concurrently on two streams with a
                               split of the SMs (args.grid per call) after staging once. */
  const struct dz_sbmm_args* next; /* device copy of the NEXT linear's args in the step, or NULL:
                               CTAs that run out of items warm L2 with the first weight stages
                               their blockIdx gets in that launch (decode plans only)      */
  const int32_t* pf_counts_dev; /* mixed plan made on the device (dz_plan_mixed_device), or NULL:
                               device [3] = {prefill jobs, decode jobs, t_pf}; then n_pf_jobs is
                               the prefill-region capacity (T: decode jobs start at jobs[T]),
                               n_jobs = n_pf_jobs + decode capacity, and t_pf is ignored     */
  int32_t sparse_job_tokens; /* the plan's 2:4 job width (the planners' argument): 8 selects the
                               kernel instantiation with the smaller X stage; 0 / 16 the wide one */
  int32_t _pad6;
} dz_sbmm_args;

/* Fused tensor-parallel reduction over peer memory (NVLink / NVSwitch), replacing the
 * reference's simulated all-reduce of row-parallel shards (inference.py:216-223) and a separate
 * NCCL all-reduce. Every rank's k_sbmm leaves fp32 partial planes; the finalize kernel sums them
 * into this rank's reduce buffer R, then runs a two-shot reduction over the peers' memory:
 * reduce-scatter (rank r sums chunk r of every peer's R in rank order, applies the activation,
 * stores it in its gather buffer G in Y's dtype) and all-gather (every rank copies every owner's
 * chunk of G into Y). Identical, deterministic Y on every rank; NVLink bytes read per rank
 * (w-1)/w * T*out * (4 + sizeof(Y)). Buffers are double-buffered by a device-resident epoch, so
 * the step stays CUDA-graph capturable. */
typedef struct dz_tp_ctx {
  float* const* peer_R;     /* device array [world]: rank p's two reduce buffers R (fp32,
                               2 x max_elems) followed by its two gather buffers G (2 x
                               max_elems x 4 bytes), peer-mapped (dz_ipc_open)             */
  int* const* peer_flags;   /* device array [world]: rank p's ready flags [2 phases][64]  */
  unsigned int* sync;       /* this rank's device words: [0] epoch, [1] barrier count,
                               [2] barrier generation (zeroed once)                        */
  int64_t max_elems;        /* capacity of one reduce buffer: >= T * out                   */
  int32_t rank, world;
} dz_tp_ctx;
/* Peer-shareable device memory (cudaMalloc, zeroed) and its IPC handle exchange (64-byte
 * cudaIpcMemHandle_t): rank r allocates, all-gathers the handles, opens every peer's. */
int dz_peer_alloc(size_t bytes, void** ptr);
int dz_peer_free(void* ptr);
int dz_ipc_handle(void* ptr, uint8_t* handle64);
int dz_ipc_open(const uint8_t* handle64, void** ptr);
int dz_ipc_close(void* ptr);

const char* dz_version(void);
const char* dz_strerror(int status);

/* K1 — bit-exact unpack. Replaces compress.dequantize_layer (compress.py:467-497),
 * with unpack_codes (:265-277), decode_mask_indices (:295-314) and
 * _float64_unpayload (:343-345). out = [rows][ld_out] of out_dtype; fp32 output is
 * bit-identical to np.float32(dequantize_layer(ld)), bf16 to torch .to(bfloat16).
 * A corrupt nibble (p0 >= p1) sets *err_flag (device int) to DZ_E_FORMAT. */
int dz_unpack(const dz_ref_delta* d, int out_dtype, void* out, int64_t ld_out,
              int* err_flag, void* stream);

/* Pieces of K1 exposed for the codec API: unpack_codes (compress.py:265-277) into
 * int32 codes, and decode_mask_indices (compress.py:295-314) into a uint8 keep mask
 * [rows][cols]. Same error contract (host-checked lengths, *err_flag on bad nibble). */
int dz_unpack_codes(const uint32_t* words, int64_t n_words, int32_t bits, int64_t count,
                    int32_t* out, void* stream);
int dz_decode_index(const uint8_t* index, int64_t index_bytes, int32_t rows, int32_t cols,
                    uint8_t* keep, int* err_flag, void* stream);

/* Upload-time re-layout of a 2:4 delta (bits 2/3/4, group_size % 128 == 0 or one
 * group per row) into 16x128 native blocks: the same codes, index nibbles and
 * scales, arranged as mma.sp fragments. Lossless (dz_unpack_native inverts it);
 * validates every index nibble like decode_mask_indices (compress.py:307-309). */
int64_t dz_native_sparse_bytes(int32_t rows, int32_t cols, int32_t bits);
int dz_repack_sparse(const dz_ref_delta* d, void* native_out, int* err_flag, void* stream);
/* Inverse view of a native sparse delta, for parity checks of the re-layout. */
int dz_unpack_native(const void* native, int32_t rows, int32_t cols, int32_t bits,
                     int32_t qmax, float* out, int64_t ld_out, void* stream);

/* Dense bf16 [rows][ldw] -> dense native blocks (base weight, or a dequantised delta
 * that the sparse kernel does not take). */
int64_t dz_native_dense_bytes(int32_t rows, int32_t cols);
int dz_pack_dense_bf16(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols,
                       void* native_out, void* stream);

/* Host: fill the entry of a base weight W [rows][cols] bf16 (row stride ldw elements, 16-byte
 * aligned rows). The fused kernel streams W in its natural layout with 128B-swizzled TMA tiles
 * straight into tcgen05 MMAs — no re-layout of the base model. */
int dz_base_init(dz_native_delta* entry, const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols);

/* Host: fill a table entry, encoding the TMA descriptor the fused kernel streams `blocks`
 * with (kind DZ_KIND_*; rows/cols of the layer). */
int dz_native_delta_init(dz_native_delta* entry, const void* blocks, int32_t kind, int32_t rows,
                         int32_t cols);

/* Copy X [T][in] (ldx) into a zero-padded [T][ldp] buffer, ldp = ceil128(in). */
int dz_pad_x(const uint16_t* X, int64_t ldx, int32_t T, int32_t in, uint16_t* Xp,
             int64_t ldp, void* stream);

/* Host-side plan. Replaces inference.group_by_delta (inference.py:106-123): stable
 * sort of token rows by slot, then cut into dz_jobs. kinds[n_slots] gives each
 * slot's DZ_KIND_*. Returns DZ_E_UNKNOWN when a slot is out of range
 * (inference.py:135-137). max_jobs >= dz_plan_max_jobs(T). sparse_job_tokens (8 or 16,
 * 0 = 8; the same argument on every planner) is the width of a 2:4 delta job: a token's result
 * does not depend on it (the n-tiles of a job are independent MMA columns), 16 decodes each
 * delta chunk once for twice the tokens (pass dz_sbmm_args.sparse_job_tokens the same value). */
int32_t dz_plan_max_jobs(int32_t T);
int dz_plan(const int32_t* slots, int32_t T, const int32_t* kinds, int32_t n_slots,
            int32_t with_base, int32_t* order_out, dz_job* jobs_out, int32_t max_jobs,
            int32_t* n_jobs_out, int32_t sparse_job_tokens);
/* Tokens per prefill job of a c-token group: ceil(c / ceil(c / DZ_PREFILL_JOB_TOKENS)) rounded up
 * to 16 (the last job of the group takes the rest). */
/* Prefill tokens of a c-token group (c >= pf_min): all of them, except that a remainder of fewer
 * than DZ_PREFILL_REM_MIN tokens beyond whole jobs stays on the decode kernel (a few decode tokens
 * of the request's delta would otherwise double its prefill jobs). 0 disables the rule. */
#ifndef DZ_PREFILL_REM_MIN
#define DZ_PREFILL_REM_MIN 32
#endif
#define DZ_PREFILL_TOKENS(c)                                                                      \
  ((c) >= DZ_PREFILL_JOB_TOKENS && (c) % DZ_PREFILL_JOB_TOKENS < DZ_PREFILL_REM_MIN               \
       ? (c) - (c) % DZ_PREFILL_JOB_TOKENS                                                        \
       : (c))
#ifdef DZ_PREFILL_GREEDY_CUT  /* A/B variant: full 240-token jobs, the remainder as one more job */
#define DZ_PREFILL_JOB_SIZE(c) DZ_PREFILL_JOB_TOKENS
#else
#define DZ_PREFILL_JOB_SIZE(c)                                                                   \
  ((c) < 1 ? DZ_PREFILL_JOB_TOKENS                                                                \
           : ((((c) + ((c) + DZ_PREFILL_JOB_TOKENS - 1) / DZ_PREFILL_JOB_TOKENS - 1) /            \
               (((c) + DZ_PREFILL_JOB_TOKENS - 1) / DZ_PREFILL_JOB_TOKENS) + 15) / 16) * 16)
#endif
/* Mixed plan: delta groups of >= pf_min tokens (2:4 sparse kinds) go to K3 whole, cut into
 * ceil(c / DZ_PREFILL_JOB_TOKENS) jobs of DZ_PREFILL_JOB_SIZE(c) tokens (a 256-token request: 2 x 128),
 * staged first in perm (grouped by slot, stable); the remaining tokens
 * keep their original order after them and are planned for K2 exactly as dz_plan does, with
 * order_out indexing staged rows. *t_pf_out = staged prefill rows; when it is 0 the plan is
 * the pure decode plan and perm is the identity (pass perm = NULL to dz_sbmm). */
int dz_plan_mixed(const int32_t* slots, int32_t T, const int32_t* kinds, int32_t n_slots,
                  int32_t with_base, int32_t pf_min, int32_t* perm_out, int32_t* order_out,
                  dz_job* jobs_out, int32_t max_jobs, int32_t* n_jobs_out, int32_t* n_pf_jobs_out,
                  int32_t* t_pf_out, int32_t sparse_job_tokens);

/* On-device plan (decode plans): the same stable group_by_delta and job cut as dz_plan, computed
 * by one CTA from device-resident slots, so a decode loop never round-trips to the host (SURVEY
 * §8(f)-3). Writes order[T], jobs[<= max_jobs] and *n_jobs_dev; *err_dev = DZ_E_UNKNOWN when a
 * slot is out of range (inference.py:135-137; *n_jobs_dev = 0 then), DZ_E_VALUE when max_jobs
 * is too small. n_slots <= 4096. Stream-ordered, graph-capturable. */
int dz_plan_device(const int32_t* slots_dev, int32_t T, const int32_t* kinds_dev, int32_t n_slots,
                   int32_t with_base, int32_t* order_dev, dz_job* jobs_dev, int32_t max_jobs,
                   int32_t* n_jobs_dev, int32_t* err_dev, int32_t sparse_job_tokens, void* stream);
/* On-device admission: the decision of scheduler.select_batch (scheduler.py:73-123) — up to K
 * requests spanning at most N deltas, first come first served, line skips linked to the earliest
 * batch member of their delta — for an arrival-ordered queue q_*[Q] (Q <= 8192) and the running
 * requests r_*[R]. *_model: delta id in [0, n_models) (n_models <= 4096); *_id: request id;
 * *_rank: the request's rank in (arrival, id) order over queue and running requests together.
 * Writes admitted[Q], skipped[Q] (0/1), parent[Q] (request id, -1 = none), selected[n_models]
 * (0/1: the batch's delta set) and counts[0] = admitted requests; *err = DZ_E_VALUE for a delta
 * id out of range. One CTA, stream-ordered, graph-capturable: the admitted requests' slots can
 * feed dz_plan_device without a host round trip. Queue removal, request states and the lazy
 * delta eviction (scheduler.py:106-123) stay with the caller's bookkeeping. */
int dz_admit_device(const int32_t* q_model, const int32_t* q_id, const int32_t* q_rank, int32_t Q,
                    const int32_t* r_model, const int32_t* r_id, const int32_t* r_rank, int32_t R,
                    int32_t n_models, int32_t K, int32_t N, uint8_t* admitted, uint8_t* skipped,
                    int32_t* parent, uint8_t* selected, int32_t* counts, int32_t* err, void* stream);

/* On-device mixed plan: dz_plan_mixed (prefill staging for K3 + the decode plan over the staged
 * rows) computed by one CTA from device-resident slots. Writes perm[T], order[T], prefill jobs to
 * jobs[0, T) and decode jobs to jobs[T, T + dz_plan_max_jobs(T)), counts_dev[3] = {prefill jobs,
 * decode jobs, t_pf}; *err_dev as dz_plan_device. Pass counts_dev as dz_sbmm_args.pf_counts_dev. */
int dz_plan_mixed_device(const int32_t* slots_dev, int32_t T, const int32_t* kinds_dev, int32_t n_slots,
                         int32_t with_base, int32_t pf_min, int32_t* perm_dev, int32_t* order_dev,
                         dz_job* jobs_dev, int32_t* counts_dev, int32_t* err_dev,
                         int32_t sparse_job_tokens, void* stream);

/* K2 — fused decode SBMM. Replaces inference.sbmm (inference.py:126-154):
 * Y[t] = W_base x_t + ΔW_{slot(t)} x_t for every token in ONE persistent launch:
 * TMA stages W tiles (tcgen05.mma into TMEM), native delta blocks and X through
 * shared memory, warps decode codes in registers and issue mma.sp (2:4) / mma (dense)
 * with fp32 accumulation, per-(row,128-col) scales are applied per block. The base and
 * delta partials go to fp32 planes (one writer per element) and are summed in a fixed
 * order with the activation applied: by a short k_finalize launch (default), or inside
 * k_sbmm by a combiner warp (args.fused_merge = 1). Deterministic and batch-invariant:
 * a token's result does not depend on the other tokens in the call. */
size_t dz_sbmm_workspace_bytes(int32_t T, int32_t out);
/* Chained launch: the linears of a decode step (L <= 256, e.g. 4 per decoder layer) in ONE
 * persistent kernel — the launches of dz_sbmm, back to back, without the launch boundaries: the
 * items of linear l follow those of linear l-1 in one scheduler, each delta item's rows are
 * merged and written by the CTA's combiner warp (the fused merge), and linear l's X loads wait
 * until every Y row of linear l-1 is written (its weights stream ahead meanwhile). Linear l's
 * input may be any earlier linear's output. Decode plans of single-GPU linears with a base, one
 * shared workspace (sized for the widest linear), results bit-identical to fused_merge launches.
 * dz_sbmm_chain_encode fills a host buffer (64-byte aligned, dz_sbmm_chain_desc_bytes) that the
 * caller copies to device memory once; *narrow_out selects the kernel instantiation for
 * dz_sbmm_chain (1 when every linear's plan has 8-token 2:4 jobs). All CTAs must be resident:
 * grid <= SMs (0 = one per SM). */
size_t dz_sbmm_chain_desc_bytes(int32_t L);
int dz_sbmm_chain_encode(const dz_sbmm_args* args, int32_t L, void* desc_host, size_t desc_bytes,
                         int32_t* narrow_out);
int dz_sbmm_chain(const void* desc_dev, int32_t L, int32_t narrow, int32_t grid, void* stream);
/* K3 — prefill SBMM (dz_prefill.cu), launched by dz_sbmm for the prefill jobs of a mixed plan:
 * per (128-row tile, <= 256-token group) one TMEM accumulator receives tcgen05 MMAs of the base
 * W tile and of the group's delta tile, dequantised (code * scale -> bf16) from native blocks
 * into shared memory by CUDA-core warps. Exposed for diagnostics / the kernel bench. */
int dz_sbmm_prefill(const dz_sbmm_args* args, void* stream);
/* Gather rows: Xs[i] = X[perm[i]] (bf16, row strides in elements, 16-byte aligned rows). */
int dz_gather_rows(const uint16_t* X, int64_t ldx, const int32_t* perm, int32_t T, int32_t in,
                   uint16_t* Xs, int64_t ldxs, void* stream);
/* Resident CTAs per SM of the fused kernel (diagnostics; < 0 on error). */
int dz_sbmm_ctas_per_sm(void);
int dz_sbmm(const dz_sbmm_args* args, void* stream);

/* ---- DZDL container (formats.py:60-169): the delta swap-in path ------------------- */
typedef struct dz_dzdl_info {
  int32_t version, flags;   /* flags bit 0 = deflate payloads (FLAG_LOSSLESS)          */
  int32_t lossless, _pad;
  int64_t header_off, header_len; /* JSON header bytes (configuration; parsed by the caller) */
  int64_t layers_off;       /* first layer record                                     */
} dz_dzdl_info;
typedef struct dz_dzdl_layer {
  int64_t name_off;         /* byte ranges inside the container buffer                 */
  int32_t name_len, rows, cols, _pad;
  int64_t scales_off, scales_len;
  int64_t index_off, index_len;
  int64_t payload_off, payload_len; /* stored payload (deflate stream when lossless)   */
} dz_dzdl_layer;
/* Replaces the magic/version/header part of formats.read_delta (formats.py:102-130):
 * DZ_E_FORMAT (bad magic / truncated, *err_offset = byte offset), DZ_E_UNSUPPORTED (version). */
int dz_dzdl_parse_header(const uint8_t* buf, int64_t len, dz_dzdl_info* info, int64_t* err_offset);
/* Replaces the per-layer loop of formats.read_delta (formats.py:132-162): byte ranges of
 * layer_count records starting at layers_off. DZ_E_FORMAT on truncation (*err_offset = the
 * offset where reading failed), DZ_E_VALUE on trailing bytes (*err_offset = end of the last layer). */
int dz_dzdl_parse_layers(const uint8_t* buf, int64_t len, int64_t layers_off, int32_t layer_count,
                         dz_dzdl_layer* layers, int64_t* err_offset);
/* Replaces compress.lossless_decode (compress.py:560-564, zlib): inflate src into dst[cap].
 * *out_len = inflated bytes; DZ_E_FORMAT = corrupt stream; DZ_E_ENCODING = dst too small
 * (*out_len = the size needed; call again). dst may be NULL to size the output. */
int dz_inflate(const uint8_t* src, int64_t n, uint8_t* dst, int64_t cap, int64_t* out_len);
/* ---- GPU ΔCompress ---------------------------------------------------
 * obs_compress_layer (compress.py:348-464): greedy OBS column solver over a layer delta with
 * 2:4 keep masks (_keep_mask_groups compress.py:204-215) and per-(row, group) symmetric RTN.
 * W     [rows, cols] f64 device, the delta; overwritten with the quantized delta (the solver's
 *       final `w`, i.e. dequantize_layer of the result) — the caller's propagation input.
 * U     [cols, cols] f64 device, upper Cholesky factor of H^-1 (_inverse_cholesky_factor,
 *       compress.py:321-336; computed by the caller, e.g. cuSOLVER).
 * packed  n_words u32 (bits < 16: ceil(n / (32/bits)), n = rows*cols/2 under 2:4 else rows*cols;
 *         bits 16: 2 words per stored f64 value)
 * index   rows*cols/8 bytes (2:4 only), scales rows*ceil(cols/gs) f32 (bits < 16 only),
 * proxy_loss one f64. Stream-ordered; workspace from dz_obs_workspace_bytes. */
typedef struct dz_obs_cfg {
  int32_t bits;       /* 2, 3, 4, 8, or 16 (identity quantizer: values stored raw) */
  int32_t sparse;     /* 1 = two_of_four */
  int32_t group_size;
  int32_t block_size; /* <= 256; multiple of 4 under 2:4 */
} dz_obs_cfg;
size_t dz_obs_workspace_bytes(int32_t rows, int32_t cols, const dz_obs_cfg* cfg);
int dz_obs_compress(double* W, const double* U, int32_t rows, int32_t cols, const dz_obs_cfg* cfg,
                    uint32_t* packed, uint8_t* index, float* scales, double* proxy_loss, void* ws,
                    size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DZ_B200_H */
