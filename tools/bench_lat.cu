// Latency decomposition of one dependent mat-vec step (S in registers, resident).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_lat tools/bench_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W = 35, L = 8, NK = 5;

__device__ __forceinline__ void cfma(double2& a, double2 m, double2 x) {
  a.x = fma(m.x, x.x, a.x); a.x = fma(-m.y, x.y, a.x);
  a.y = fma(m.x, x.y, a.y); a.y = fma(m.y, x.x, a.y);
}

// FLAGS: 1 = tA+tB input (else single v), 2 = writer does cmul next-input (else plain store),
//        4 = barrier, 8 = butterfly, 16 = named barrier instead of __syncthreads
template <int FLAGS>
__global__ void __launch_bounds__(288) k_lat(const double2* __restrict__ src, int steps, double2* out, long long* cyc) {
  __shared__ double2 tA[2][64], tB[2][64], co[192];
  for (int e = threadIdx.x; e < 128; e += blockDim.x) { (&tA[0][0])[e] = make_double2(1, .5); (&tB[0][0])[e] = make_double2(0, 0); }
  for (int e = threadIdx.x; e < 192; e += blockDim.x) co[e] = make_double2(0.1, 0.01);
  __syncthreads();
  const int ri = threadIdx.x / L, q = threadIdx.x % L;
  double2 m[NK];
#pragma unroll
  for (int c = 0; c < NK; ++c) {
    int k = q + c * L;
    m[c] = (ri < W && k < W) ? src[ri * W + k] : make_double2(0, 0);
  }
  double2 cr = co[ri], ne = co[64 + ri], bn = co[128 + ri];
  long long t0 = clock64();
  int cur = 0;
  for (int s = 0; s < steps; ++s) {
    double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
#pragma unroll
    for (int c = 0; c < NK; ++c) {
      int k = q + c * L;
      if (k < W) {
        double2 v = tA[cur][k];
        if (FLAGS & 1) { double2 vb = tB[cur][k]; v.x += vb.x; v.y += vb.y; }
        if (c & 1) cfma(a1, m[c], v); else cfma(a0, m[c], v);
      }
    }
    double2 acc = make_double2(a0.x + a1.x, a0.y + a1.y);
    if (FLAGS & 8) {
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      }
    }
    if (q == 0 && ri < W) {
      if (FLAGS & 2) {
        tA[cur ^ 1][ri] = make_double2(bn.x - (cr.x * acc.x - cr.y * acc.y) * 1e-2, bn.y - (cr.x * acc.y + cr.y * acc.x) * 1e-2);
        if (ri + 1 < W) tB[cur ^ 1][ri + 1] = make_double2(-(ne.x * acc.x) * 1e-2, -(ne.y * acc.y) * 1e-2);
      } else {
        tA[cur ^ 1][ri] = make_double2(acc.x * 1e-2, acc.y * 1e-2);
      }
    }
    if (FLAGS & 4) {
      if (FLAGS & 16) asm volatile("bar.sync 1, 288;" ::: "memory");
      else __syncthreads();
    }
    cur ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = tA[cur][0]; }
}

template <int F>
void run(const char* nm, const double2* src, double2* o, long long* cyc) {
  k_lat<F><<<1, 288>>>(src, 20000, o, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-44s %6.0f cycles/step (%s)\n", nm, c / 20000.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double2 *src, *o;
  long long* cyc;
  cudaMalloc(&src, W * W * 16);
  cudaMemset(src, 0, W * W * 16);
  cudaMalloc(&o, 64);
  cudaMalloc(&cyc, 64);
  run<1 | 2 | 4 | 8>("full (tA+tB, writer, barrier, butterfly)", src, o, cyc);
  run<1 | 2 | 4 | 8 | 16>("full, named barrier", src, o, cyc);
  run<2 | 4 | 8>("single v", src, o, cyc);
  run<1 | 4 | 8>("plain writer", src, o, cyc);
  run<4 | 8>("single v, plain writer", src, o, cyc);
  run<1 | 2 | 8>("no barrier", src, o, cyc);
  run<1 | 2 | 4>("no butterfly", src, o, cyc);
  run<4>("only FMA + barrier", src, o, cyc);
  run<0>("only FMA", src, o, cyc);
}
