// Shared-memory load cost per warp instruction for the access patterns of the
// sweep step (10 warps per SM): LDS.128 broadcast, 4 distinct 16-byte addresses
// (the input-vector pattern), 32 consecutive 16-byte addresses, LDS.64 variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_lds tools/bench_lds.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int PAT>
__global__ void __launch_bounds__(320, 1) k(int iters, double* out, long long* cyc) {
  __shared__ double2 buf[2048];
  for (int e = threadIdx.x; e < 2048; e += blockDim.x) buf[e] = make_double2(e, 1.0 / (e + 1));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int idx;
  if (PAT == 0) idx = 0;                       // broadcast
  else if (PAT == 1) idx = lane & 3;           // 4 distinct consecutive
  else if (PAT == 2) idx = lane;               // 32 consecutive
  else if (PAT == 3) idx = (lane >> 2) * 37 + (lane & 3);   // 8 rows x 4, stride 37 (packed-like)
  else idx = (lane >> 2) * 36 + (lane & 3);    // 8 rows x 4, stride 36
  double ax = 0, ay = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double2 v;
      const unsigned a = (unsigned)__cvta_generic_to_shared(&buf[(idx + 4 * c + (it & 1) * 64) & 2047]);
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
      ax += v.x;
      ay += v.y;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = ax + ay;
}

int main() {
  double* o;
  long long* cyc;
  cudaMalloc(&o, 1 << 22);
  cudaMalloc(&cyc, 1 << 12);
  const char* names[] = {"LDS.128 broadcast", "LDS.128 4 distinct", "LDS.128 32 consecutive",
                         "LDS.128 8 rows x 4, stride 37", "LDS.128 8 rows x 4, stride 36"};
  const int iters = 2000;
  for (int p = 0; p < 5; ++p) {
    for (int rep = 0; rep < 2; ++rep) {
      if (p == 0) k<0><<<148, 320>>>(iters, o, cyc);
      if (p == 1) k<1><<<148, 320>>>(iters, o, cyc);
      if (p == 2) k<2><<<148, 320>>>(iters, o, cyc);
      if (p == 3) k<3><<<148, 320>>>(iters, o, cyc);
      if (p == 4) k<4><<<148, 320>>>(iters, o, cyc);
    }
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    // 10 warps x 8 loads per iteration share the SM's shared-memory pipe
    printf("%-34s %6.2f cycles per warp instruction (SM-wide, 10 warps)\n", names[p], (double)h / iters / 8 / 10);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
