// GPU ΔCompress: the OBS column solver that produces a packed layer delta.
//
// Reference: obs_compress_layer (compress.py:348-464) with _keep_mask_groups (compress.py:204-215)
// and the symmetric per-(row, group) RTN grid (compress.py:403-428). The solver is sequential
// over columns but independent over rows given the shared inverse-Hessian Cholesky factor U:
//
//   for each block [i1, i2) of `block_size` columns:
//     k_obs_block   each row walks the block's columns in order (4 lanes per row): group scale at
//                   col % gs == 0 (from the block-start W, as the reference reads `w`, not `w1`),
//                   2:4 keep mask at col % 4 == 0 (stable argsort of w^2 / u_ii^2), RTN code,
//                   err = (w - q) / u_col,col, and the in-block update w1[:, j] -= err * u[col, j]
//                   held in shared memory; writes the quantized block back into W and err into E;
//     k_obs_update  W[:, i2:] -= E @ U[i1:i2, i2:] (rank-block_size update, f64 tiles), applied
//                   eagerly inside a window of columns (one scale group) and, for the columns
//                   beyond it, once per window with every block's product rounded in order.
//   k_obs_loss / k_obs_pack_* then reduce the proxy loss and emit the reference's packed layout
//   (pack_codes compress.py:243-262, encode_mask_indices compress.py:280-292).
//
// Floating-point order follows the reference: the in-block update is a rounded product then a
// rounded subtraction (numpy's `w1 -= np.outer(err, u)`), so it uses __dmul_rn / __dsub_rn
// (never contracted to FMA); the trailing product accumulates k in order with FMA from zero,
// the order OpenBLAS's dgemm kernels use for `err1 @ u`, and is subtracted after rounding.
// Codes, masks and scales are therefore bit-identical to the reference on the same U whenever
// the reference's BLAS follows that order (tests/test_gpu_obs.py).
#include <cuda_runtime.h>

#include <cstdint>

#include "dz_b200.h"

namespace dz {
namespace obs {

#ifndef DZ_OBS_LPR
#define DZ_OBS_LPR 8
#endif
constexpr int ROWS_PER_CTA = 32;  // rows per CTA
constexpr int LPR = DZ_OBS_LPR;   // lanes per row: a row's in-block update is split LPR ways
constexpr int OBS_THREADS = ROWS_PER_CTA * LPR;
constexpr int RS = ROWS_PER_CTA + 1;  // shared row stride of the [column][row] tiles
constexpr int MAX_BLOCK = 256;    // block_size limit (row segments in shared memory)

struct Cfg {
  int bits, sparse, gs, bs, qmax, passthrough, n_groups;
};

// One block of columns [i1, i2) for all rows: 32 rows per CTA, 4 lanes per row (8 rows per warp).
// Column i is quantised by its owner lane (i % 4) of each row; err is broadcast to the row's 4
// lanes by a shuffle, and lane q applies the update to the block columns j > i with j % 4 == q.
// That cuts the serial update per column 4x and puts 4 warps on each SM instead of 1 (the walk
// is latency-bound). Shared memory: row segments w1[B][33], squared residuals sq[B][33], and,
// when it fits (B <= 128), U's diagonal block su[B][B] (broadcast reads). The column loop is
// not unrolled: a fully unrolled block thrashes the instruction cache (ncu: no_instructions).
__global__ void __launch_bounds__(OBS_THREADS) k_obs_block(double* __restrict__ W, const double* __restrict__ U,
                                                           int rows, int cols, int i1, int i2, Cfg cfg,
                                                           int32_t* __restrict__ codes, uint8_t* __restrict__ nib,
                                                           double* __restrict__ kept_vals, float* __restrict__ scales,
                                                           double* __restrict__ E, int ldE, int e_off,
                                                           double* __restrict__ loss_part, int stage_u) {
  extern __shared__ double smem[];
  const int nb = i2 - i1;
  double* w1s = smem;                 // [nb][RS]
  double* sq = smem + nb * RS;        // [nb][RS]
  double* su = smem + 2 * nb * RS;    // [nb][nb] when stage_u
  const int tid = threadIdx.x, q = tid & (LPR - 1), rl = tid / LPR;
  const int gbase = (tid & 31) & ~(LPR - 1);  // this row's lane 0 within the warp
  const int row = blockIdx.x * ROWS_PER_CTA + rl;
  const bool live = row < rows;
  double* wrow = W + static_cast<int64_t>(row) * cols;
  auto w1 = [&](int j) -> double& { return w1s[j * RS + rl]; };
  auto ublk = [&](int i, int j) -> double {
    return stage_u ? su[i * nb + j] : __ldg(U + static_cast<int64_t>(i1 + i) * cols + i1 + j);
  };
  if (stage_u)
    for (int e = tid; e < nb * nb; e += OBS_THREADS) su[e] = U[static_cast<int64_t>(i1 + e / nb) * cols + i1 + e % nb];
  for (int j = q; j < nb; j += LPR) w1(j) = live ? wrow[i1 + j] : 0.0;
  __syncthreads();

  // the scale of a group that started in an earlier block (stored f32 = the snapped value)
  double scale = (!cfg.passthrough && live && i1 % cfg.gs != 0)
                     ? static_cast<double>(scales[static_cast<int64_t>(row) * cfg.n_groups + i1 / cfg.gs])
                     : 0.0;
  unsigned keep4 = 0xF;  // blocks start at multiples of 4 under 2:4: the mask is set at i = 0
#pragma unroll 1
  for (int i = 0; i < nb; i++) {
    const int col = i1 + i;
    const int own = i & (LPR - 1);
    if (!cfg.passthrough && col % cfg.gs == 0) {
      // scales[:, g] = f32(max|w[:, col:col+gs]| / qmax), w = the block-start matrix; the row's
      // 4 lanes take every 4th column and combine (max is order-free, so this is exact)
      const int end = min(col + cfg.gs, cols);
      double m = 0.0;
      if (live)
        for (int j = col + q; j < end; j += LPR) m = fmax(m, fabs(wrow[j]));
#pragma unroll
      for (int o = 1; o < LPR; o <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      scale = static_cast<double>(__double2float_rn(__ddiv_rn(m, static_cast<double>(cfg.qmax))));
      if (live && q == 0) scales[static_cast<int64_t>(row) * cfg.n_groups + col / cfg.gs] = static_cast<float>(scale);
    }
    if (cfg.sparse && (col & 3) == 0) {
      // saliency w^2 / hd over the 4-group, stable argsort: prune the two smallest (every lane
      // of the row computes the same mask)
      double s4[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const double uk = ublk(i + k, i + k);
        const double w = w1(i + k);
        s4[k] = __ddiv_rn(__dmul_rn(w, w), __dmul_rn(uk, uk));
      }
      keep4 = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        int rank = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) rank += (s4[k] < s4[j]) || (s4[k] == s4[j] && k < j);
        if (rank >= 2) keep4 |= 1u << j;
      }
      if (live && q == 0) {
        const int p0 = __ffs(keep4) - 1, p1 = 31 - __clz(keep4);
        nib[(static_cast<int64_t>(row) * cols + col) >> 2] = static_cast<uint8_t>(p0 | (p1 << 2));
      }
    }
    double err = 0.0;
    if (q == own) {
      const bool kc = !cfg.sparse || ((keep4 >> (col & 3)) & 1u);
      const double wc = w1(i);
      double qc;
      int32_t code = 0;
      if (cfg.passthrough) {
        qc = kc ? wc : 0.0;
      } else {
        if (scale > 0.0 && kc) {
          double r = rint(__ddiv_rn(wc, scale));
          r = fmin(fmax(r, -static_cast<double>(cfg.qmax)), static_cast<double>(cfg.qmax));
          code = static_cast<int32_t>(r);
        }
        qc = __dmul_rn(static_cast<double>(code), scale);
      }
      const double diff = __dsub_rn(wc, qc);
      err = __ddiv_rn(diff, ublk(i, i));
      w1(i) = qc;  // w[:, i1:i2] = quantized[:, i1:i2] after the block
      sq[i * RS + rl] = live ? __dmul_rn(diff, diff) : 0.0;
      if (live) {
        if (cfg.sparse) {
          if (kc) {
            // kept index: two per 4-group, row-major, in column order (codes[keep])
            const int slot = __popc(keep4 & ((1u << (col & 3)) - 1u));
            const int64_t kk = (static_cast<int64_t>(row) * cols + (col & ~3)) / 2 + slot;
            if (cfg.passthrough) kept_vals[kk] = qc;
            else codes[kk] = code;
          }
        } else if (!cfg.passthrough) {
          codes[static_cast<int64_t>(row) * cols + col] = code;
        }
        E[static_cast<int64_t>(row) * ldE + e_off + i] = err;
      }
    }
    err = __shfl_sync(0xffffffffu, err, gbase + own);
    // w1[:, j] -= err * u[col, j] for this lane's columns of the rest of the block (rounded
    // product, rounded difference)
    for (int j = i + 1 + ((q - i - 1) & (LPR - 1)); j < nb; j += LPR)
      w1(j) = __dsub_rn(w1(j), __dmul_rn(err, ublk(i, j)));
    __syncwarp();
  }
  __syncthreads();
  // proxy loss partials: per column, the sum over this CTA's rows in row order
  for (int j = tid; j < nb; j += OBS_THREADS) {
    double t = 0.0;
    for (int k = 0; k < ROWS_PER_CTA; k++) t = __dadd_rn(t, sq[j * RS + k]);
    loss_part[static_cast<int64_t>(blockIdx.x) * cols + i1 + j] = t;
  }
  if (live)
    for (int j = q; j < nb; j += LPR) wrow[i1 + j] = w1(j);
}

// W[:, i2:] -= E[:, :B] @ U[i1:i2, i2:] on the FP64 tensor cores (mma.sync m8n8k4 f64, DMMA).
// DMMA is bit-identical to the k-ordered FMA chain fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c))))
// (tools/dmma_probe.cu, 2.56M cases), so chaining k-steps from a zero accumulator reproduces the
// in-order FMA accumulation of the reference's BLAS exactly; one rounded subtraction per element.
//
// Windowed schedule: W[:, c_begin:c_end] receives the updates of `nch` consecutive blocks
// (chunks of `bs` columns of E / rows of U) in block order, each chunk's product rounded and
// subtracted before the next (the reference's per-block `w[:, i2:] -= err1 @ u`). The W tile
// stays in registers across the chunks, so W is read and written once per window instead of
// once per block.
// 64x64 output tile per CTA, 8 warps as 2 (rows) x 4 (cols), 32x16 per warp = 4x2 DMMA tiles.
// Shared tiles are [k][64 + 4]: the +4 pad spreads a half-warp's 4 k-rows over all 32 banks.
constexpr int UTM = 64, UTN = 64, UK = 32, EPAD = UTM + 4, UPAD = UTN + 4;
constexpr size_t UPD_SMEM = static_cast<size_t>(UK) * (EPAD + UPAD) * 8;
__global__ void __launch_bounds__(256, 2) k_obs_update(double* __restrict__ W, const double* __restrict__ E, int ldE, int e_base,
                                                       const double* __restrict__ U, int rows, int cols, int u0,
                                                       int c_begin, int c_end, int nch, int bs, int last_len) {
  extern __shared__ double sm[];
  double* sE = sm;              // [UK][EPAD]: E[r0 + row][ch * bs + k0 + k]
  double* sU = sm + UK * EPAD;  // [UK][UPAD]: U[u0 + ch * bs + k0 + k][c0 + col]
  const int c0 = c_begin + blockIdx.x * UTN, r0 = blockIdx.y * UTM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int fr = lane >> 2, fk = lane & 3;
  // this thread's W elements: rows wm + 8m + fr, cols wn + 8n + 2fk + {0, 1}
  double w[4][2][2];
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const int r = r0 + wm + m * 8 + fr;
#pragma unroll
    for (int n = 0; n < 2; n++) {
      const int c = c0 + wn + n * 8 + 2 * fk;
      const double* wr = W + static_cast<int64_t>(r) * cols;
      w[m][n][0] = (r < rows && c < c_end) ? wr[c] : 0.0;
      w[m][n][1] = (r < rows && c + 1 < c_end) ? wr[c + 1] : 0.0;
    }
  }
  for (int ch = 0; ch < nch; ch++) {
    const int B = ch == nch - 1 ? last_len : bs;
    const int e0 = e_base + ch * bs, ur = u0 + ch * bs;
    double acc[4][2][2];
#pragma unroll
    for (int m = 0; m < 4; m++)
#pragma unroll
      for (int n = 0; n < 2; n++) acc[m][n][0] = acc[m][n][1] = 0.0;
    for (int k0 = 0; k0 < B; k0 += UK) {
      const int kn = min(UK, B - k0);
      // all global loads of the tile in flight before any shared store
      constexpr int PE = UK * UTM / 256, PU = UK * UTN / 256;
      double ve[PE], vu[PU];
#pragma unroll
      for (int t = 0; t < PE; t++) {
        const int e = threadIdx.x + 256 * t;
        const int kr = e % UK, r = r0 + e / UK;
        ve[t] = (kr < kn && r < rows) ? E[static_cast<int64_t>(r) * ldE + e0 + k0 + kr] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < PU; t++) {
        const int e = threadIdx.x + 256 * t;
        const int kc = e / UTN, c = c0 + e % UTN;
        vu[t] = (kc < kn && c < c_end) ? U[static_cast<int64_t>(ur + k0 + kc) * cols + c] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < PE; t++) {
        const int e = threadIdx.x + 256 * t;
        sE[(e % UK) * EPAD + e / UK] = ve[t];
      }
#pragma unroll
      for (int t = 0; t < PU; t++) {
        const int e = threadIdx.x + 256 * t;
        sU[(e / UTN) * UPAD + e % UTN] = vu[t];
      }
      __syncthreads();
      const int ksteps = (kn + 3) >> 2;
      for (int ks = 0; ks < ksteps; ks++) {
        const int kk = ks * 4 + fk;
        double a[4], b[2];
#pragma unroll
        for (int m = 0; m < 4; m++) a[m] = sE[kk * EPAD + wm + m * 8 + fr];
#pragma unroll
        for (int n = 0; n < 2; n++) b[n] = sU[kk * UPAD + wn + n * 8 + fr];
#pragma unroll
        for (int m = 0; m < 4; m++)
#pragma unroll
          for (int n = 0; n < 2; n++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
                         : "d"(a[m]), "d"(b[n]));
      }
      __syncthreads();
    }
    // this block's product is complete: one rounded subtraction per element
#pragma unroll
    for (int m = 0; m < 4; m++)
#pragma unroll
      for (int n = 0; n < 2; n++) {
        w[m][n][0] = __dsub_rn(w[m][n][0], acc[m][n][0]);
        w[m][n][1] = __dsub_rn(w[m][n][1], acc[m][n][1]);
      }
  }
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const int r = r0 + wm + m * 8 + fr;
    if (r >= rows) continue;
    double* wr = W + static_cast<int64_t>(r) * cols;
#pragma unroll
    for (int n = 0; n < 2; n++) {
      const int c = c0 + wn + n * 8 + 2 * fk;
      if (c < c_end) wr[c] = w[m][n][0];
      if (c + 1 < c_end) wr[c + 1] = w[m][n][1];
    }
  }
}

// proxy_loss = sum_col (sum_rows sq) / u_col,col^2: one thread per column folds the per-CTA
// partials in CTA order into part[0][col], then one CTA sums the columns (fixed order).
__global__ void __launch_bounds__(256) k_obs_loss_cols(double* __restrict__ part, int n_cta, int cols,
                                                       const double* __restrict__ U) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= cols) return;
  double s = 0.0;
  for (int b = 0; b < n_cta; b++) s = __dadd_rn(s, part[static_cast<int64_t>(b) * cols + c]);
  const double d = U[static_cast<int64_t>(c) * cols + c];
  part[c] = __ddiv_rn(s, __dmul_rn(d, d));
}

__global__ void __launch_bounds__(256) k_obs_loss(const double* __restrict__ part, int cols,
                                                  double* __restrict__ loss) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int c = threadIdx.x; c < cols; c += 256) acc = __dadd_rn(acc, part[c]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = red[0];
}

// pack_codes: word w holds codes [w*per, w*per+per) as (code + qmax) << (bits * j)
__global__ void k_obs_pack_codes(const int32_t* __restrict__ codes, int64_t n, int bits, int qmax,
                                 uint32_t* __restrict__ words, int64_t n_words) {
  const int per = 32 / bits;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < n_words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t v = 0;
    for (int j = 0; j < per; j++) {
      const int64_t k = w * per + j;
      if (k < n) v |= static_cast<uint32_t>(codes[k] + qmax) << (bits * j);
    }
    words[w] = v;
  }
}

// encode_mask_indices: byte b = nib[2b] | nib[2b+1] << 4 (zero nibble pads an odd count)
__global__ void k_obs_pack_index(const uint8_t* __restrict__ nib, int64_t n_groups, uint8_t* __restrict__ index,
                                 int64_t n_bytes) {
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < n_bytes;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint8_t lo = nib[2 * b];
    const uint8_t hi = (2 * b + 1 < n_groups) ? nib[2 * b + 1] : 0;
    index[b] = static_cast<uint8_t>(lo | (hi << 4));
  }
}

struct WsLayout {
  size_t E, codes, nib, part, total;
};

// Columns a window defers: the trailing update of every column beyond the window waits until the
// window's last block. A window must cover each scale group whole (the group scale at its first
// column reads the group's current values), so it is the group when block_size divides it;
// without scales (identity quantizer) any multiple of the block works.
static int window_cols(const dz_obs_cfg& c) {
  if (c.bits == 16) return c.block_size * (c.block_size >= 128 ? 1 : 128 / c.block_size);
  if (c.group_size % c.block_size == 0 && c.group_size <= 512) return c.group_size;
  return c.block_size;
}

static WsLayout ws_layout(int rows, int cols, const dz_obs_cfg& c) {
  auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  const int n_cta = (rows + ROWS_PER_CTA - 1) / ROWS_PER_CTA;
  const int64_t rc = static_cast<int64_t>(rows) * cols;
  WsLayout L{};
  size_t off = 0;
  L.E = off;
  off += al(static_cast<size_t>(rows) * window_cols(c) * 8);
  L.codes = off;
  off += al(static_cast<size_t>(c.sparse ? rc / 2 : rc) * 4);
  L.nib = off;
  off += al(static_cast<size_t>(c.sparse ? rc / 4 : 1));
  L.part = off;
  off += al(static_cast<size_t>(n_cta) * cols * 8);
  L.total = off;
  return L;
}

static int check_cfg(int rows, int cols, const dz_obs_cfg* c) {
  if (!c || rows < 1 || cols < 1) return DZ_E_VALUE;
  if (!(c->bits == 2 || c->bits == 3 || c->bits == 4 || c->bits == 8 || c->bits == 16)) return DZ_E_VALUE;
  if (c->group_size < 1 || c->block_size < 1 || c->block_size > MAX_BLOCK) return DZ_E_VALUE;
  if (c->sparse && (c->block_size % 4 != 0)) return DZ_E_VALUE;
  if (c->sparse && (cols % 4 != 0)) return DZ_E_SHAPE;
  return DZ_OK;
}

}  // namespace obs
}  // namespace dz

using namespace dz;

extern "C" size_t dz_obs_workspace_bytes(int32_t rows, int32_t cols, const dz_obs_cfg* cfg) {
  if (obs::check_cfg(rows, cols, cfg) != DZ_OK) return 0;
  return obs::ws_layout(rows, cols, *cfg).total;
}

extern "C" int dz_obs_compress(double* W, const double* U, int32_t rows, int32_t cols, const dz_obs_cfg* cfg,
                               uint32_t* packed, uint8_t* index, float* scales, double* proxy_loss, void* ws,
                               size_t ws_bytes, void* stream) {
  const int st = obs::check_cfg(rows, cols, cfg);
  if (st != DZ_OK) return st;
  if (!W || !U || !packed || !proxy_loss) return DZ_E_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t rc = static_cast<int64_t>(rows) * cols;
  const bool passthrough = cfg->bits == 16;
  if (passthrough && !cfg->sparse) {
    // identity quantizer, no pruning: the raw f64 values are the payload (compress.py:372-385)
    if (cudaMemcpyAsync(packed, W, rc * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return DZ_E_CUDA;
    return cudaMemsetAsync(proxy_loss, 0, 8, s) == cudaSuccess ? DZ_OK : DZ_E_CUDA;
  }
  if (cfg->sparse && !index) return DZ_E_VALUE;
  if (!passthrough && !scales) return DZ_E_VALUE;
  const obs::WsLayout L = obs::ws_layout(rows, cols, *cfg);
  if (!ws || ws_bytes < L.total) return DZ_E_VALUE;
  char* base = static_cast<char*>(ws);
  double* E = reinterpret_cast<double*>(base + L.E);
  int32_t* codes = reinterpret_cast<int32_t*>(base + L.codes);
  uint8_t* nib = reinterpret_cast<uint8_t*>(base + L.nib);
  double* part = reinterpret_cast<double*>(base + L.part);

  obs::Cfg c{cfg->bits, cfg->sparse, cfg->group_size, cfg->block_size, (1 << (cfg->bits - 1)) - 1,
             passthrough ? 1 : 0, (cols + cfg->group_size - 1) / cfg->group_size};
  const int n_cta = (rows + obs::ROWS_PER_CTA - 1) / obs::ROWS_PER_CTA;
  const int bs = cfg->block_size;
  const int stage_u = bs <= 128;
  const size_t smem = 2 * static_cast<size_t>(bs) * obs::RS * 8 + (stage_u ? static_cast<size_t>(bs) * bs * 8 : 0);
  if (smem > 48 * 1024 && cudaFuncSetAttribute(obs::k_obs_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem)) != cudaSuccess)
    return DZ_E_CUDA;
  if (cudaFuncSetAttribute(obs::k_obs_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(obs::UPD_SMEM)) != cudaSuccess)
    return DZ_E_CUDA;
  double* kept_vals = reinterpret_cast<double*>(packed);  // passthrough 2:4: f64 payload of kept values
  const int win = obs::window_cols(*cfg);
  auto update = [&](int u0, int e_base, int c_begin, int c_end, int nch, int last_len) {
    dim3 grid((c_end - c_begin + obs::UTN - 1) / obs::UTN, (rows + obs::UTM - 1) / obs::UTM);
    obs::k_obs_update<<<grid, 256, obs::UPD_SMEM, s>>>(W, E, win, e_base, U, rows, cols, u0, c_begin, c_end, nch, bs,
                                                       last_len);
  };
  for (int g0 = 0; g0 < cols; g0 += win) {
    const int g1 = g0 + win < cols ? g0 + win : cols;
    for (int i1 = g0; i1 < g1; i1 += bs) {
      const int i2 = i1 + bs < g1 ? i1 + bs : g1;
      obs::k_obs_block<<<n_cta, obs::OBS_THREADS, smem, s>>>(W, U, rows, cols, i1, i2, c, codes, nib, kept_vals,
                                                               scales, E, win, i1 - g0, part, stage_u);
      if (i2 < g1) update(i1, i1 - g0, i2, g1, 1, i2 - i1);  // eager inside the window
    }
    if (g1 < cols) update(g0, 0, g1, cols, (g1 - g0 + bs - 1) / bs, (g1 - g0) - ((g1 - g0 - 1) / bs) * bs);
  }
  obs::k_obs_loss_cols<<<(cols + 255) / 256, 256, 0, s>>>(part, n_cta, cols, U);
  obs::k_obs_loss<<<1, 256, 0, s>>>(part, cols, proxy_loss);
  if (cfg->sparse) {
    const int64_t n_groups = rc / 4, n_bytes = (n_groups + 1) / 2;
    obs::k_obs_pack_index<<<static_cast<int>((n_bytes + 255) / 256 < 4096 ? (n_bytes + 255) / 256 : 4096), 256, 0,
                            s>>>(nib, n_groups, index, n_bytes);
  }
  if (!passthrough) {
    const int64_t n = cfg->sparse ? rc / 2 : rc;
    const int per = 32 / cfg->bits;
    const int64_t n_words = (n + per - 1) / per;
    obs::k_obs_pack_codes<<<static_cast<int>((n_words + 255) / 256 < 4096 ? (n_words + 255) / 256 : 4096), 256, 0,
                            s>>>(codes, n, cfg->bits, c.qmax, packed, n_words);
  }
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}
