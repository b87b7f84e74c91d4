// K1 (bit-exact unpack) and the upload-time native re-layout kernels.
//
// Reference layout (LayerDelta, compress.py:101-143):
//   packed_values: offset-unsigned codes u = code + qmax, `bits` each, LSB first, 32//bits per
//                  word, kept-only under 2:4 in row-major kept order (compress.py:243-262, 439-447)
//   index_stream : one nibble p0 | p1<<2 per 4-column group, row-major, low nibble first
//                  (compress.py:280-292)
//   scales       : f32 [rows][ceil(cols/gs)] (compress.py:450-452)
//   bits == 16 with no scales: packed_values holds raw f64 values (compress.py:339-345, 479-480)
#include <cstdio>

#include "dz_common.cuh"

namespace dz {

__device__ __forceinline__ uint32_t ref_code_u(const uint32_t* __restrict__ packed, int64_t k, int bits) {
  const int per = 32 / bits;
  const uint32_t w = __ldg(packed + k / per);
  return (w >> ((k % per) * bits)) & ((1u << bits) - 1u);
}

__device__ __forceinline__ uint32_t ref_nibble(const uint8_t* __restrict__ index, int64_t j) {
  const uint32_t byte = __ldg(index + (j >> 1));
  return (j & 1) ? (byte >> 4) : (byte & 0xFu);
}

__device__ __forceinline__ void store_out(void* out, int64_t off, double v, int dtype) {
  if (dtype == DZ_F64) {
    reinterpret_cast<double*>(out)[off] = v;
    return;
  }
  const float f = __double2float_rn(v);  // v is the exact product: one rounding == np.float32(ref)
  if (dtype == DZ_F32)
    reinterpret_cast<float*>(out)[off] = f;
  else
    reinterpret_cast<__nv_bfloat16*>(out)[off] = __float2bfloat16_rn(f);  // == torch f64->bf16
}

__device__ __forceinline__ double ref_f64(const uint32_t* __restrict__ packed, int64_t k) {
  const uint32_t lo = __ldg(packed + 2 * k), hi = __ldg(packed + 2 * k + 1);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

// value of kept/dense element number k at column `col` of row r (dequantize_layer, compress.py:482-490):
// f64(code) * f64(scale) is exact (<= 16-bit code x 24-bit mantissa), as in the reference.
__device__ __forceinline__ double ref_value(const dz_ref_delta& d, int64_t k, int r, int col) {
  if (d.bits == 16 && d.n_scales == 0) return ref_f64(d.packed, k);
  const int qmax = (1 << (d.bits - 1)) - 1;
  const int code = static_cast<int>(ref_code_u(d.packed, k, d.bits)) - qmax;  // no clamp (:277)
  const int ng = ceil_div(d.cols, d.group_size);
  const float s = __ldg(d.scales + static_cast<int64_t>(r) * ng + col / d.group_size);
  return static_cast<double>(code) * static_cast<double>(s);
}

// One thread per (row, 4-column group) for 2:4, per element for dense.
__global__ void k_unpack(dz_ref_delta d, int dtype, void* out, int64_t ld, int* err) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d.sparse) {
    const int ncg = d.cols / 4;
    const int64_t n = static_cast<int64_t>(d.rows) * ncg;
    if (i >= n) return;
    const int r = static_cast<int>(i / ncg), c = static_cast<int>(i % ncg);
    const uint32_t nib = ref_nibble(d.index, i);
    const int p0 = nib & 3, p1 = nib >> 2;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (p0 >= p1) {
      atomicExch(err, DZ_E_FORMAT);  // decode_mask_indices, compress.py:307-309
    } else {
      const int64_t k = static_cast<int64_t>(r) * (d.cols / 2) + 2 * c;
      v[p0] = ref_value(d, k, r, 4 * c + p0);
      v[p1] = ref_value(d, k + 1, r, 4 * c + p1);
    }
    const int64_t o = static_cast<int64_t>(r) * ld + 4 * c;
#pragma unroll
    for (int q = 0; q < 4; q++) store_out(out, o + q, v[q], dtype);
  } else {
    const int64_t n = static_cast<int64_t>(d.rows) * d.cols;
    if (i >= n) return;
    const int r = static_cast<int>(i / d.cols), c = static_cast<int>(i % d.cols);
    store_out(out, static_cast<int64_t>(r) * ld + c, ref_value(d, i, r, c), dtype);
  }
}

// ------------------------------------------------------------------------------------------
// Native sparse blocks. Block (rb, kb) covers rows 16rb..16rb+15, cols 128kb..128kb+127 and
// drives 4 mma.sp m16n8k32 (MMA i covers cols 32i..32i+31 of the block). Lane l = 4g+t:
//   codes, fbits=4: word i = MMA i, nibbles n0..n7 = (rA,sA,1st) (rB,sA,1st) (rA,sB,1st)
//                   (rB,sB,1st) then the same four 2nd-kept; rA=g, rB=g+8, sA=slot t, sB=t+4.
//                   a_k = (n_k, n_{k+4}) = lop3(w >> 4k, 0x000F000F, 0x43004300) - (128+qmax).
//   codes, fbits=2: word j holds MMAs 2j (fields 0-3 / 8-11) and 2j+1 (fields 4-7 / 12-15);
//                   a_k = fields (o+k, o+k+8), o = 4*(i&1).
//   meta:  word 0 = E of MMA (t<2 ? 0 : 1), word 1 = E of MMA (t<2 ? 2 : 3), half h = t&1:
//          E = nibbles(row g, groups 4h..4h+3) | nibbles(row g+8, same) << 16; MMA i uses
//          sparsity selector i&1 (measured layout, profiles/r01_probe_mma_layout.txt).
//   scales: float2 (scale[g], scale[g+8]) at position g.
// ------------------------------------------------------------------------------------------
struct KeptPair {
  uint32_t u0, u1;  // unsigned codes of the 1st / 2nd kept element
  uint32_t nib;     // index nibble
};

__device__ __forceinline__ KeptPair ref_pair(const dz_ref_delta& d, int r, int cg, int qmax, int* err) {
  KeptPair p{static_cast<uint32_t>(qmax), static_cast<uint32_t>(qmax), 0x4u};
  if (r >= d.rows || 4 * cg >= d.cols) return p;  // padding: code 0, any valid nibble
  const int64_t j = static_cast<int64_t>(r) * (d.cols / 4) + cg;
  p.nib = ref_nibble(d.index, j);
  if ((p.nib & 3) >= (p.nib >> 2)) {
    atomicExch(err, DZ_E_FORMAT);
    p.nib = 0x4u;
  }
  const int64_t k = static_cast<int64_t>(r) * (d.cols / 2) + 2 * cg;
  p.u0 = ref_code_u(d.packed, k, d.bits);
  p.u1 = ref_code_u(d.packed, k + 1, d.bits);
  return p;
}

__global__ void k_repack_sparse(dz_ref_delta d, uint8_t* __restrict__ out, int fbits, int* err) {
  const int nkb = ceil_div(d.cols, kBlkCols);
  const int blk = blockIdx.x;  // rb * nkb + kb
  const int rb = blk / nkb, kb = blk % nkb;
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  const int qmax = (1 << (d.bits - 1)) - 1;
  const int rA = rb * 16 + g, rB = rA + 8;
  const int bbytes = sparse_block_bytes(fbits);
  uint8_t* base = out + static_cast<int64_t>(blk) * bbytes;

  uint32_t cw[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4; i++) {
    const int cgA = kb * 32 + 8 * i + t, cgB = cgA + 4;
    const KeptPair pAA = ref_pair(d, rA, cgA, qmax, err), pBA = ref_pair(d, rB, cgA, qmax, err);
    const KeptPair pAB = ref_pair(d, rA, cgB, qmax, err), pBB = ref_pair(d, rB, cgB, qmax, err);
    const uint32_t first[4] = {pAA.u0, pBA.u0, pAB.u0, pBB.u0};
    const uint32_t second[4] = {pAA.u1, pBA.u1, pAB.u1, pBB.u1};
    if (fbits == 4) {
      uint32_t w = 0;
      for (int k = 0; k < 4; k++) w |= (first[k] << (4 * k)) | (second[k] << (4 * (k + 4)));
      cw[i] = w;
    } else {
      const int o = 4 * (i & 1);
      for (int k = 0; k < 4; k++)
        cw[i >> 1] |= (first[k] << (2 * (o + k))) | (second[k] << (2 * (o + k + 8)));
    }
  }
  if (fbits == 4)
    reinterpret_cast<uint4*>(base)[lane] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
  else
    reinterpret_cast<uint2*>(base)[lane] = make_uint2(cw[0], cw[1]);

  uint32_t mw[2];
  const int h = t & 1;
  for (int m = 0; m < 2; m++) {
    const int i = (t < 2 ? 0 : 1) + 2 * m;
    uint32_t e = 0;
    for (int q = 0; q < 4; q++) {
      const int cg = kb * 32 + 8 * i + 4 * h + q;
      e |= ref_pair(d, rA, cg, qmax, err).nib << (4 * q);
      e |= ref_pair(d, rB, cg, qmax, err).nib << (16 + 4 * q);
    }
    mw[m] = e;
  }
  reinterpret_cast<uint2*>(base + sparse_code_bytes(fbits))[lane] = make_uint2(mw[0], mw[1]);

  if (t == 0) {
    const int ng = ceil_div(d.cols, d.group_size);
    const int grp = (kb * kBlkCols) / d.group_size;
    float sA = 0.f, sB = 0.f;
    if (rA < d.rows) sA = __ldg(d.scales + static_cast<int64_t>(rA) * ng + grp);
    if (rB < d.rows) sB = __ldg(d.scales + static_cast<int64_t>(rB) * ng + grp);
    reinterpret_cast<float2*>(base + sparse_code_bytes(fbits) + kMetaBytes)[g] = make_float2(sA, sB);
  }
}

// Inverse of k_repack_sparse (parity check of the re-layout): dense fp32 code*scale.
__global__ void k_unpack_native(const uint8_t* __restrict__ nat, int rows, int cols, int fbits, int qmax,
                                float* __restrict__ out, int64_t ld) {
  const int nkb = ceil_div(cols, kBlkCols);
  const int blk = blockIdx.x;
  const int rb = blk / nkb, kb = blk % nkb;
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  const uint8_t* base = nat + static_cast<int64_t>(blk) * sparse_block_bytes(fbits);
  const float2 sc = reinterpret_cast<const float2*>(base + sparse_code_bytes(fbits) + kMetaBytes)[g];
  // metadata: gather E words of all four MMAs for rows g and g+8 from the quad
  const uint2 m = reinterpret_cast<const uint2*>(base + sparse_code_bytes(fbits))[lane];
  for (int i = 0; i < 4; i++) {
    // E(MMA i, half h) lives in lane 4g + (i&1)*2 + h, word i>>1
    uint32_t e[2];
    for (int h = 0; h < 2; h++) {
      const int src = 4 * g + (i & 1) * 2 + h;
      const uint32_t w0 = __shfl_sync(0xffffffffu, m.x, src), w1 = __shfl_sync(0xffffffffu, m.y, src);
      e[h] = (i >> 1) ? w1 : w0;
    }
    uint32_t u[8];
    if (fbits == 4) {
      const uint4 c4 = reinterpret_cast<const uint4*>(base)[lane];
      const uint32_t wi = i == 0 ? c4.x : i == 1 ? c4.y : i == 2 ? c4.z : c4.w;
      for (int k = 0; k < 8; k++) u[k] = (wi >> (4 * k)) & 0xF;
    } else {
      const uint2 c2 = reinterpret_cast<const uint2*>(base)[lane];
      const uint32_t wj = (i >> 1) ? c2.y : c2.x;
      const int o = 4 * (i & 1);
      for (int k = 0; k < 4; k++) {
        u[k] = (wj >> (2 * (o + k))) & 3;
        u[k + 4] = (wj >> (2 * (o + k + 8))) & 3;
      }
    }
    // u[k]: first kept of pair k, u[k+4]: second; pair k -> (row, slot): 0:(g,t) 1:(g+8,t) 2:(g,t+4) 3:(g+8,t+4)
    for (int k = 0; k < 4; k++) {
      const int r = rb * 16 + g + ((k & 1) ? 8 : 0);
      const int slot = t + ((k & 2) ? 4 : 0);
      const int h = slot >> 2, q = slot & 3;
      const uint32_t nib = (e[h] >> ((k & 1) ? 16 + 4 * q : 4 * q)) & 0xF;
      const int col0 = kb * kBlkCols + 32 * i + 4 * slot;
      if (r >= rows || col0 >= cols) continue;
      const float s = (k & 1) ? sc.y : sc.x;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      v[nib & 3] = static_cast<float>(static_cast<int>(u[k]) - qmax) * s;
      v[nib >> 2] = static_cast<float>(static_cast<int>(u[k + 4]) - qmax) * s;
      for (int c = 0; c < 4; c++) out[static_cast<int64_t>(r) * ld + col0 + c] = v[c];
    }
  }
}

// Dense native blocks: block (rb, kb) = 8 k16 MMAs; lane l=4g+t, MMA j, k = 128kb + 16j:
//   a0 = W[g][k+2t..+1], a1 = W[g+8][k+2t..], a2 = W[g][k+8+2t..], a3 = W[g+8][k+8+2t..]
__global__ void k_pack_dense(const uint16_t* __restrict__ W, int64_t ldw, int rows, int cols,
                             uint8_t* __restrict__ out) {
  const int nkb = ceil_div(cols, kBlkCols);
  const int blk = blockIdx.x;
  const int rb = blk / nkb, kb = blk % nkb;
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  auto ld2 = [&](int r, int c) -> uint32_t {
    uint32_t lo = 0, hi = 0;
    if (r < rows && c < cols) lo = W[static_cast<int64_t>(r) * ldw + c];
    if (r < rows && c + 1 < cols) hi = W[static_cast<int64_t>(r) * ldw + c + 1];
    return lo | (hi << 16);
  };
  const int k = kb * kBlkCols + 16 * j;
  const int rA = rb * 16 + g, rB = rA + 8;
  uint4 v;
  v.x = ld2(rA, k + 2 * t);
  v.y = ld2(rB, k + 2 * t);
  v.z = ld2(rA, k + 8 + 2 * t);
  v.w = ld2(rB, k + 8 + 2 * t);
  reinterpret_cast<uint4*>(out + static_cast<int64_t>(blk) * kDenseBlockBytes)[j * 32 + lane] = v;
}

__global__ void k_unpack_codes(const uint32_t* __restrict__ w, int bits, int64_t count, int32_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  out[i] = static_cast<int32_t>(ref_code_u(w, i, bits)) - ((1 << (bits - 1)) - 1);
}

__global__ void k_decode_index(const uint8_t* __restrict__ index, int64_t ngroups, uint8_t* __restrict__ keep,
                               int* err) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= ngroups) return;
  const uint32_t nib = ref_nibble(index, j);
  const int p0 = nib & 3, p1 = nib >> 2;
  if (p0 >= p1) atomicExch(err, DZ_E_FORMAT);
  uchar4 k = make_uchar4(0, 0, 0, 0);
  if (p0 < p1) {
    reinterpret_cast<uint8_t*>(&k)[p0] = 1;
    reinterpret_cast<uint8_t*>(&k)[p1] = 1;
  }
  reinterpret_cast<uchar4*>(keep)[j] = k;
}

__global__ void k_pad_x(const uint16_t* __restrict__ X, int64_t ldx, int T, int in, uint16_t* __restrict__ Xp,
                        int64_t ldp) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(T) * ldp) return;
  const int64_t t = i / ldp, c = i % ldp;
  Xp[i] = c < in ? X[t * ldx + c] : static_cast<uint16_t>(0);
}

}  // namespace dz

using namespace dz;

static inline int launch_status() {
  return cudaGetLastError() == cudaSuccess ? DZ_OK : DZ_E_CUDA;
}

static int check_ref(const dz_ref_delta* d) {
  if (!d || d->rows < 1 || d->cols < 1) return DZ_E_SHAPE;
  if (d->bits != 2 && d->bits != 3 && d->bits != 4 && d->bits != 8 && d->bits != 16) return DZ_E_VALUE;
  if (d->group_size < 1) return DZ_E_VALUE;
  const int64_t n = d->sparse ? static_cast<int64_t>(d->rows) * d->cols / 2 : static_cast<int64_t>(d->rows) * d->cols;
  if (d->sparse) {
    if (d->cols % 4) return DZ_E_SHAPE;
    const int64_t ng = static_cast<int64_t>(d->rows) * (d->cols / 4);
    if (d->index_bytes != (ng + 1) / 2) return DZ_E_FORMAT;  // compress.py:298-302
  }
  if (d->bits == 16 && d->n_scales == 0) {
    if (d->n_words < 2 * n) return DZ_E_ENCODING;
    return DZ_OK;
  }
  const int per = 32 / d->bits;
  if (n > d->n_words * per) return DZ_E_ENCODING;  // compress.py:271-272
  const int64_t ng = (d->cols + d->group_size - 1) / d->group_size;
  if (d->n_scales != static_cast<int64_t>(d->rows) * ng) return DZ_E_VALUE;  // reshape, :484
  return DZ_OK;
}

extern "C" int dz_unpack(const dz_ref_delta* d, int out_dtype, void* out, int64_t ld_out, int* err_flag,
                         void* stream) {
  int st = check_ref(d);
  if (st) return st;
  if (out_dtype != DZ_F32 && out_dtype != DZ_BF16 && out_dtype != DZ_F64) return DZ_E_VALUE;
  if (ld_out < d->cols) return DZ_E_SHAPE;
  const int64_t n = d->sparse ? static_cast<int64_t>(d->rows) * (d->cols / 4) : static_cast<int64_t>(d->rows) * d->cols;
  if (n == 0) return DZ_OK;
  const int tpb = 256;
  k_unpack<<<static_cast<unsigned>((n + tpb - 1) / tpb), tpb, 0, static_cast<cudaStream_t>(stream)>>>(
      *d, out_dtype, out, ld_out, err_flag);
  return launch_status();
}

static int sparse_fbits(int bits) { return bits == 2 ? 2 : 4; }

extern "C" int64_t dz_native_sparse_bytes(int32_t rows, int32_t cols, int32_t bits) {
  if (rows < 1 || cols < 1 || (bits != 2 && bits != 3 && bits != 4)) return -1;
  return static_cast<int64_t>(ceil_div(rows, kBlkRows)) * ceil_div(cols, kBlkCols) *
         sparse_block_bytes(sparse_fbits(bits));
}

extern "C" int dz_repack_sparse(const dz_ref_delta* d, void* native_out, int* err_flag, void* stream) {
  int st = check_ref(d);
  if (st) return st;
  if (!d->sparse || (d->bits != 2 && d->bits != 3 && d->bits != 4)) return DZ_E_UNSUPPORTED;
  const int ng = ceil_div(d->cols, d->group_size);
  if (!(d->group_size % kBlkCols == 0 || ng == 1)) return DZ_E_UNSUPPORTED;
  const int nblk = ceil_div(d->rows, kBlkRows) * ceil_div(d->cols, kBlkCols);
  k_repack_sparse<<<nblk, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      *d, static_cast<uint8_t*>(native_out), sparse_fbits(d->bits), err_flag);
  return launch_status();
}

extern "C" int dz_unpack_native(const void* native, int32_t rows, int32_t cols, int32_t bits, int32_t qmax,
                                float* out, int64_t ld_out, void* stream) {
  if (rows < 1 || cols < 1 || ld_out < cols) return DZ_E_SHAPE;
  if (bits != 2 && bits != 3 && bits != 4) return DZ_E_UNSUPPORTED;
  const int nblk = ceil_div(rows, kBlkRows) * ceil_div(cols, kBlkCols);
  k_unpack_native<<<nblk, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(native), rows, cols, sparse_fbits(bits), qmax, out, ld_out);
  return launch_status();
}

extern "C" int64_t dz_native_dense_bytes(int32_t rows, int32_t cols) {
  if (rows < 1 || cols < 1) return -1;
  return static_cast<int64_t>(ceil_div(rows, kBlkRows)) * ceil_div(cols, kBlkCols) * kDenseBlockBytes;
}

extern "C" int dz_pack_dense_bf16(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols, void* native_out,
                                  void* stream) {
  if (rows < 1 || cols < 1 || ldw < cols) return DZ_E_SHAPE;
  const int nblk = ceil_div(rows, kBlkRows) * ceil_div(cols, kBlkCols);
  k_pack_dense<<<nblk, 256, 0, static_cast<cudaStream_t>(stream)>>>(W, ldw, rows, cols,
                                                                   static_cast<uint8_t*>(native_out));
  return launch_status();
}

extern "C" int dz_pad_x(const uint16_t* X, int64_t ldx, int32_t T, int32_t in, uint16_t* Xp, int64_t ldp,
                        void* stream) {
  if (T < 0 || in < 1 || ldx < in || ldp < in) return DZ_E_SHAPE;
  const int64_t n = static_cast<int64_t>(T) * ldp;
  if (n == 0) return DZ_OK;
  k_pad_x<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(X, ldx, T, in,
                                                                                                 Xp, ldp);
  return launch_status();
}

extern "C" int dz_unpack_codes(const uint32_t* words, int64_t n_words, int32_t bits, int64_t count, int32_t* out,
                               void* stream) {
  if (bits < 2 || bits > 16) return DZ_E_VALUE;
  if (count < 0) return DZ_E_VALUE;
  if (count > n_words * (32 / bits)) return DZ_E_ENCODING;  // compress.py:271-272
  if (count == 0) return DZ_OK;
  k_unpack_codes<<<static_cast<unsigned>((count + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      words, bits, count, out);
  return launch_status();
}

extern "C" int dz_decode_index(const uint8_t* index, int64_t index_bytes, int32_t rows, int32_t cols, uint8_t* keep,
                               int* err_flag, void* stream) {
  if (rows < 0 || cols < 0 || cols % 4) return DZ_E_SHAPE;
  const int64_t ng = static_cast<int64_t>(rows) * (cols / 4);
  if (index_bytes != (ng + 1) / 2) return DZ_E_FORMAT;  // compress.py:298-302
  if (ng == 0) return DZ_OK;
  k_decode_index<<<static_cast<unsigned>((ng + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      index, ng, keep, err_flag);
  return launch_status();
}
