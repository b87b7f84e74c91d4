// TMA streaming probe: how fast can a persistent producer/consumer ring of 1-D bulk copies
// stream HBM into shared memory on B200, as a function of stage bytes, ring depth, CTAs/SM?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_stream(const uint8_t* src, size_t chunks, int chunk_bytes, int nstage, int split, int work, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  uint8_t* ring = sm + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstage; s++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(ncons));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == ncons) {
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
        asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su32(&empty[stage])), "r"(phase ^ 1) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[stage])), "r"(chunk_bytes) : "memory");
        const int piece = chunk_bytes / split;
        for (int p = 0; p < split; p++)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(ring + (size_t)stage * chunk_bytes + p * piece)),
                       "l"(src + c * chunk_bytes + p * piece), "r"(piece), "r"(su32(&full[stage])) : "memory");
        if (++stage == nstage) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    int stage = 0; uint32_t phase = 0; uint32_t x = 0;
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
      asm volatile("{\n.reg .pred P;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2;\n}" ::"r"(su32(&full[stage])), "r"(phase) : "memory");
      x ^= reinterpret_cast<const uint32_t*>(ring + (size_t)stage * chunk_bytes)[threadIdx.x];
      if (work > 0) {  // emulated per-stage consumer processing time (clock cycles)
        const long long t0 = clock64();
        while (clock64() - t0 < work) x += 1;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[stage])) : "memory");
      if (++stage == nstage) { stage = 0; phase ^= 1; }
    }
    if (x == 0x12345u) out[0] = x;
  }
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const size_t bytes = (size_t)8 << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  uint32_t* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  struct Cfg { int chunk, nstage, cpsm, threads, split, work; };
  Cfg cfgs[] = {
      {61440, 3, 1, 352, 1, 0},    {61440, 3, 1, 352, 1, 500},  {61440, 3, 1, 352, 1, 1000},
      {61440, 3, 1, 352, 1, 1500}, {61440, 3, 1, 352, 1, 2000}, {61440, 3, 1, 352, 1, 2500},
      {40960, 5, 1, 352, 1, 0},    {40960, 5, 1, 352, 1, 1000}, {40960, 5, 1, 352, 1, 1600},
      {30720, 7, 1, 352, 1, 0},    {30720, 7, 1, 352, 1, 800},  {30720, 7, 1, 352, 1, 1200},
      {102400, 2, 1, 352, 1, 0},   {102400, 2, 1, 352, 1, 2000},
  };
  for (const Cfg& c : cfgs) {
    const int smem = 256 + c.chunk * c.nstage;
    if (smem > 227 * 1024) continue;
    const size_t chunks = bytes / c.chunk;
    const int grid = prop.multiProcessorCount * c.cpsm;
    k_stream<<<grid, c.threads, smem>>>(buf, chunks, c.chunk, c.nstage, c.split, c.work, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_stream<<<grid, c.threads, smem>>>(buf, chunks, c.chunk, c.nstage, c.split, c.work, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream, c.threads, smem);
    printf("chunk=%6d stages=%2d ctas/sm=%d (occ %d) split=%d work=%5d cyc inflight/SM=%4d KB : %7.1f GB/s\n", c.chunk,
           c.nstage, c.cpsm, occ, c.split, c.work, c.chunk * c.nstage * c.cpsm / 1024, bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
