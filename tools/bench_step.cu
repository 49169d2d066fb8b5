// Variants of the dependent complex mat-vec step y = S v (S w x w in smem).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_step tools/bench_step.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int L, int MODE>  // MODE 0 normal, 1 no barrier, 2 no shuffle, 3 split-v (tA+tB)
__global__ void k_step(int steps, double2* out, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* S = sm;
  double2* v = sm + W * W;  // [2][64]
  double2* v2 = v + 128;
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) S[e] = make_double2(1e-3 * (e % 17), 1e-3 * (e % 13));
  for (int e = threadIdx.x; e < 256; e += blockDim.x) v[e] = make_double2(1.0, 0.5);
  __syncthreads();
  const int ri = threadIdx.x / L, q = threadIdx.x % L;
  constexpr int NK = (W + L - 1) / L;
  long long t0 = clock64();
  int cur = 0;
  for (int s = 0; s < steps; ++s) {
    double ax0 = 0, ay0 = 0, ax1 = 0, ay1 = 0;
    if (ri < W) {
      const double2* Sr = S + ri * W;
      const double2* vv = v + cur * 64;
      const double2* vb = v2 + cur * 64;
#pragma unroll
      for (int c = 0; c < NK; ++c) {
        const int k = q + c * L;
        if (k < W) {
          double2 m = Sr[k], x = vv[k];
          if (MODE == 3) { double2 y = vb[k]; x.x += y.x; x.y += y.y; }
          if (c & 1) {
            ax1 = fma(m.x, x.x, ax1); ax1 = fma(-m.y, x.y, ax1);
            ay1 = fma(m.x, x.y, ay1); ay1 = fma(m.y, x.x, ay1);
          } else {
            ax0 = fma(m.x, x.x, ax0); ax0 = fma(-m.y, x.y, ax0);
            ay0 = fma(m.x, x.y, ay0); ay0 = fma(m.y, x.x, ay0);
          }
        }
      }
    }
    double ax = ax0 + ax1, ay = ay0 + ay1;
    if (MODE != 2) {
#pragma unroll
      for (int off = L / 2; off > 0; off >>= 1) {
        ax += __shfl_xor_sync(0xffffffffu, ax, off);
        ay += __shfl_xor_sync(0xffffffffu, ay, off);
      }
    }
    if (q == 0 && ri < W) v[(cur ^ 1) * 64 + ri] = make_double2(ax * 1e-2, ay * 1e-2);
    if (MODE != 1) __syncthreads();
    cur ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = v[cur * 64]; }
}

template <int W, int L, int MODE>
void run(const char* name, double2* o2, long long* cyc) {
  int threads = ((W * L + 31) / 32) * 32;
  if (threads > 1024) return;
  size_t smem = sizeof(double2) * (W * W + 256);
  cudaFuncSetAttribute(k_step<W, L, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_step<W, L, MODE><<<1, threads, smem>>>(20000, o2, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("w=%d %-30s threads=%4d: %6.0f cycles/step  (%s)\n", W, name, threads, c / 20000.0,
         cudaGetErrorString(cudaGetLastError()));
}

// NCH independent chains per step (separate S blocks and vectors), one barrier
template <int W, int L, int NCH>
__global__ void k_multi(int steps, double2* out, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* S = sm;                 // NCH blocks
  double2* v = sm + NCH * W * W;   // [NCH][2][64]
  for (int e = threadIdx.x; e < NCH * W * W; e += blockDim.x) S[e] = make_double2(1e-3 * (e % 17), 1e-3 * (e % 13));
  for (int e = threadIdx.x; e < NCH * 128; e += blockDim.x) v[e] = make_double2(1.0, 0.5);
  __syncthreads();
  const int ri = threadIdx.x / L, q = threadIdx.x % L;
  constexpr int NK = (W + L - 1) / L;
  long long t0 = clock64();
  int cur = 0;
  for (int s = 0; s < steps; ++s) {
    double ax[NCH], ay[NCH];
#pragma unroll
    for (int h = 0; h < NCH; ++h) {
      double a0 = 0, b0 = 0, a1 = 0, b1 = 0;
      if (ri < W) {
        const double2* Sr = S + h * W * W + ri * W;
        const double2* vv = v + h * 128 + cur * 64;
#pragma unroll
        for (int c = 0; c < NK; ++c) {
          const int k = q + c * L;
          if (k < W) {
            double2 m = Sr[k], x = vv[k];
            if (c & 1) { a1 = fma(m.x, x.x, a1); a1 = fma(-m.y, x.y, a1); b1 = fma(m.x, x.y, b1); b1 = fma(m.y, x.x, b1); }
            else { a0 = fma(m.x, x.x, a0); a0 = fma(-m.y, x.y, a0); b0 = fma(m.x, x.y, b0); b0 = fma(m.y, x.x, b0); }
          }
        }
      }
      ax[h] = a0 + a1; ay[h] = b0 + b1;
    }
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) {
#pragma unroll
      for (int h = 0; h < NCH; ++h) {
        ax[h] += __shfl_xor_sync(0xffffffffu, ax[h], off);
        ay[h] += __shfl_xor_sync(0xffffffffu, ay[h], off);
      }
    }
    if (q == 0 && ri < W)
#pragma unroll
      for (int h = 0; h < NCH; ++h) v[h * 128 + (cur ^ 1) * 64 + ri] = make_double2(ax[h] * 1e-2, ay[h] * 1e-2);
    __syncthreads();
    cur ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = v[cur * 64]; }
}

template <int W, int L, int NCH>
void runm(double2* o2, long long* cyc) {
  int threads = ((W * L + 31) / 32) * 32;
  size_t smem = sizeof(double2) * (NCH * W * W + NCH * 128);
  cudaFuncSetAttribute(k_multi<W, L, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_multi<W, L, NCH><<<1, threads, smem>>>(20000, o2, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("w=%d L=%d chains=%d threads=%4d: %6.0f cycles/step (%5.0f per chain-step) (%s)\n", W, L, NCH, threads,
         c / 20000.0, c / 20000.0 / NCH, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double2* o2;
  long long* cyc;
  cudaMalloc(&o2, 1 << 16);
  cudaMalloc(&cyc, 1 << 16);
  runm<35, 8, 1>(o2, cyc);
  runm<35, 8, 2>(o2, cyc);
  runm<35, 8, 3>(o2, cyc);
  runm<35, 8, 4>(o2, cyc);
  runm<35, 4, 2>(o2, cyc);
  runm<35, 4, 4>(o2, cyc);
  runm<35, 16, 2>(o2, cyc);
  run<35, 1, 0>("1 lane/row", o2, cyc);
  run<35, 2, 0>("2 lanes/row", o2, cyc);
  run<35, 4, 0>("4 lanes/row", o2, cyc);
  run<35, 8, 0>("8 lanes/row", o2, cyc);
  run<35, 16, 0>("16 lanes/row", o2, cyc);
  run<35, 32, 0>("32 lanes/row", o2, cyc);
  run<35, 8, 1>("8 lanes/row no barrier", o2, cyc);
  run<35, 8, 2>("8 lanes/row no shuffle", o2, cyc);
  run<35, 8, 3>("8 lanes/row v = tA + tB", o2, cyc);
  run<35, 4, 3>("4 lanes/row v = tA + tB", o2, cyc);
  run<99, 4, 0>("4 lanes/row", o2, cyc);
  run<99, 8, 0>("8 lanes/row", o2, cyc);
  run<17, 4, 0>("4 lanes/row", o2, cyc);
  run<17, 8, 0>("8 lanes/row", o2, cyc);
}
