// Probe: is mma.sync m8n8k4 f64 (DMMA) bit-identical to a k-ordered FMA chain
// acc = fma(a3, b3, fma(a2, b2, fma(a1, b1, fma(a0, b0, c))))?  Prints mismatch counts.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, const double* C, double* D, double* R, int trials) {
  const int lane = threadIdx.x;
  for (int t = blockIdx.x; t < trials; t += gridDim.x) {
    const double* a = A + t * 32;  // 8x4 row-major
    const double* b = B + t * 32;  // 4x8 row-major
    const double* c = C + t * 64;  // 8x8
    // fragments (PTX ISA m8n8k4 f64): A: row = lane/4, col = lane%4; B: row(k) = lane%4, col = lane/4;
    // C/D: row = lane/4, cols 2*(lane%4) + {0,1}
    double fa = a[(lane >> 2) * 4 + (lane & 3)];
    double fb = b[(lane & 3) * 8 + (lane >> 2)];
    double c0 = c[(lane >> 2) * 8 + 2 * (lane & 3)], c1 = c[(lane >> 2) * 8 + 2 * (lane & 3) + 1];
    double d0, d1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d0), "=d"(d1) : "d"(fa), "d"(fb), "d"(c0), "d"(c1));
    D[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = d0;
    D[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = d1;
    // sequential FMA reference
    for (int e = lane; e < 64; e += 32) {
      const int r = e / 8, cc = e % 8;
      double acc = c[e];
      for (int kk = 0; kk < 4; kk++) acc = fma(a[r * 4 + kk], b[kk * 8 + cc], acc);
      R[t * 64 + e] = acc;
    }
  }
}

int main() {
  const int trials = 20000;
  size_t na = trials * 32, nc = trials * 64;
  double *A, *B, *C, *D, *R;
  cudaMallocManaged(&A, na * 8); cudaMallocManaged(&B, na * 8); cudaMallocManaged(&C, nc * 8);
  cudaMallocManaged(&D, nc * 8); cudaMallocManaged(&R, nc * 8);
  srand(1);
  auto rnd = []() { return (rand() / (double)RAND_MAX - 0.5) * pow(2.0, (rand() % 40) - 20); };
  for (size_t i = 0; i < na; i++) { A[i] = rnd(); B[i] = rnd(); }
  for (int mode = 0; mode < 2; mode++) {
    for (size_t i = 0; i < nc; i++) C[i] = mode ? rnd() : 0.0;
    k<<<256, 32>>>(A, B, C, D, R, trials);
    cudaDeviceSynchronize();
    long mism = 0, mism_rev = 0;
    for (size_t i = 0; i < nc; i++) {
      if (D[i] != R[i]) mism++;
    }
    (void)mism_rev;
    printf("C=%s: DMMA vs k-ordered FMA chain: %ld / %zu mismatches\n", mode ? "rand" : "zero", mism, nc);
  }
  return 0;
}
