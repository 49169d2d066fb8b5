// FP64 tensor-core (mma.sync.m8n8k4.f64) throughput on sm_100a: (a) register-resident
// operands, (b) a 40 x 40 x 36 complex block product from shared memory (A ld 36, B ld 38:
// conflict-free LDS.128 fragments), against the DFMA 4 x 4 register-tiled product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_dmma tools/bench_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void k_peak(double* out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// complex C (40x40) = A (40x36, ld 36) * B (36x40, ld 38), double2 interleaved in smem;
// warp w of NW handles output tiles t = w, w + NW, ... of the 5 x 5 tile grid
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_cmm(double2* out, int reps, long long* cyc) {
  extern __shared__ double2 smx[];
  double2* A = smx; double2* B = A + 40 * 36; double2* C = B + 36 * 42;
  for (int e = threadIdx.x; e < 40 * 36; e += blockDim.x) A[e] = make_double2(1e-3 * (e % 7), 1e-3 * (e % 5));
  for (int e = threadIdx.x; e < 36 * 42; e += blockDim.x) B[e] = make_double2(1e-3 * (e % 3), 1e-3 * (e % 11));
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int t = warp; t < 25; t += NW) {
      const int i0 = (t / 5) * 8, j0 = (t % 5) * 8;
      double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0;
#pragma unroll
      for (int k0 = 0; k0 < 36; k0 += 4) {
        const double2 a = A[(i0 + (lane >> 2)) * 36 + k0 + (lane & 3)];
        const double2 b = B[(k0 + (lane & 3)) * 42 + j0 + (lane >> 2)];
        dmma(cr0, cr1, a.x, b.x);
        dmma(cr0, cr1, -a.y, b.y);
        dmma(ci0, ci1, a.x, b.y);
        dmma(ci0, ci1, a.y, b.x);
      }
      C[(i0 + (lane >> 2)) * 42 + j0 + 2 * (lane & 3)] = make_double2(cr0, ci0);
      C[(i0 + (lane >> 2)) * 42 + j0 + 2 * (lane & 3) + 1] = make_double2(cr1, ci1);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = C[threadIdx.x];
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 16);
  long long* cyc;
  cudaMallocManaged(&cyc, 4096 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    k_peak<<<148 * 4, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    k_peak<<<148 * 4, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 148.0 * 4 * warps * iters * 8 * 512.0;
    printf("DMMA register-resident, %2d warps/CTA x 4 CTAs/SM: %.1f TFLOP/s\n", warps, flop / ms * 1e-9);
  }
  const int SMB = (40 * 36 + 36 * 42 + 40 * 42) * 16;
  cudaFuncSetAttribute(k_cmm<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMB);
  cudaFuncSetAttribute(k_cmm<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMB);
  for (int ctas : {1, 2, 3}) {
    const int reps = 2000;
    k_cmm<4><<<148 * ctas, 128, SMB>>>((double2*)out, 10, cyc);
    k_cmm<4><<<148 * ctas, 128, SMB>>>((double2*)out, reps, cyc);
    cudaDeviceSynchronize();
    double m = 0; for (int i = 0; i < 148 * ctas; ++i) m += cyc[i]; m /= 148 * ctas;
    printf("complex 40x40x36 product from smem, 4 warps, %d CTAs/SM: %.0f cycles per product per CTA, %.0f SM-cycles per product\n",
           ctas, m / reps, m / reps / ctas);
    k_cmm<8><<<148 * ctas, 256, SMB>>>((double2*)out, reps, cyc);
    cudaDeviceSynchronize();
    m = 0; for (int i = 0; i < 148 * ctas; ++i) m += cyc[i]; m /= 148 * ctas;
    printf("   8 warps, %d CTAs/SM: %.0f cycles per product per CTA, %.0f SM-cycles per product\n", ctas, m / reps, m / reps / ctas);
  }
  printf("err=%s (DFMA peak: a 35^3 complex product is 171.5k DFMA = 2.9k SM-cycles at 58.7 DFMA/clk)\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
