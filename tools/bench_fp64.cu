// Microbenchmarks: (1) FP64 FMA throughput / latency per SM on this GPU,
// (2) the isolated 35x35 complex shared-memory mat-vec step (8 lanes per row).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_fp64 tools/bench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma_tput(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dfma_lat(double* out, int iters, long long* cyc) {
  double a = threadIdx.x;
  const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_ffma_tput(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = 1.0000001f, c = 1e-9f;
  for (int i = 0; i < iters; ++i) {
    a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
    a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// isolated mat-vec step: y = S v, S 35x35 complex in smem, 8 lanes per row, 3-level shuffle, 1 barrier
__global__ void k_step(int steps, double2* out, long long* cyc) {
  __shared__ double2 S[35 * 35];
  __shared__ double2 v[2][40];
  const int w = 35;
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) S[e] = make_double2(1e-3 * (e % 17), 1e-3 * (e % 13));
  for (int e = threadIdx.x; e < 40; e += blockDim.x) v[0][e] = v[1][e] = make_double2(1.0, 0.5);
  __syncthreads();
  const int ri = threadIdx.x >> 3, q = threadIdx.x & 7;
  long long t0 = clock64();
  int cur = 0;
  for (int s = 0; s < steps; ++s) {
    double ax = 0, ay = 0, bx = 0, by = 0;
    if (ri < w) {
      for (int k = q; k < w; k += 16) {
        double2 m = S[ri * w + k], x = v[cur][k];
        ax = fma(m.x, x.x, ax); ax = fma(-m.y, x.y, ax); ay = fma(m.x, x.y, ay); ay = fma(m.y, x.x, ay);
        if (k + 8 < w) {
          double2 m2 = S[ri * w + k + 8], x2 = v[cur][k + 8];
          bx = fma(m2.x, x2.x, bx); bx = fma(-m2.y, x2.y, bx); by = fma(m2.x, x2.y, by); by = fma(m2.y, x2.x, by);
        }
      }
    }
    ax += bx; ay += by;
    for (int off = 4; off > 0; off >>= 1) {
      ax += __shfl_xor_sync(0xffffffffu, ax, off);
      ay += __shfl_xor_sync(0xffffffffu, ay, off);
    }
    if (q == 0 && ri < w) v[cur ^ 1][ri] = make_double2(ax * 1e-2, ay * 1e-2);
    __syncthreads();
    cur ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = v[cur][0]; }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  float* f;
  double2* o2;
  long long* cyc;
  cudaMalloc(&d, 1 << 26);
  cudaMalloc(&f, 1 << 26);
  cudaMalloc(&o2, 1 << 16);
  cudaMalloc(&cyc, 1 << 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 1 << 14;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_dfma_tput<<<nsm * 4, 256>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * iters * (double)nsm * 4 * 256;
    if (rep) printf("FP64 FMA: %.1f TFLOP/s  (%.1f FMA/clk/SM at 1.965 GHz)\n", flops / ms / 1e9,
                    flops / 2 / (ms * 1e-3) / nsm / 1.965e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_ffma_tput<<<nsm * 4, 256>>>(f, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * iters * (double)nsm * 4 * 256;
    if (rep) printf("FP32 FMA: %.1f TFLOP/s\n", flops / ms / 1e9);
  }
  k_dfma_lat<<<1, 32>>>(d, 4096, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", c / 4096.0);
  for (int th : {288, 320, 576}) {
    k_step<<<1, th>>>(10000, o2, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("isolated 35x35 complex mat-vec step (%d threads, 1 CTA): %.0f cycles/step\n", th, c / 10000.0);
  }
  k_step<<<nsm, 288>>>(10000, o2, cyc);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("isolated step, %d CTAs: %.0f cycles/step\n", nsm, c / 10000.0);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
