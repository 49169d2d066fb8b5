// Per-SM streaming bandwidth: N CTAs (one per SM, 288 threads) each read a private region
// with LDG.128 (.cg), U loads in flight per thread, several passes.  Regions larger than L2
// in total stream from HBM; small regions are L2 hits after the first pass.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_smbw tools/bench_smbw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(288, 1) k_stream(const double2* __restrict__ src, long elems_per_cta, int passes,
                                                   double2* sink, long long* cyc) {
  const double2* base = src + (long)blockIdx.x * elems_per_cta;
  double2 acc = make_double2(0, 0);
  __syncthreads();
  long long t0 = clock64();
  for (int p = 0; p < passes; ++p) {
    for (long e = threadIdx.x; e < elems_per_cta; e += 288L * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long i = e + 288L * u;
        v[u] = i < elems_per_cta ? __ldcg(base + i) : make_double2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc.x == 12345.678) sink[0] = acc;
}

int main() {
  const long maxbytes = 6L << 30;
  double2* buf;
  cudaMalloc(&buf, maxbytes);
  cudaMemset(buf, 0, maxbytes);
  long long* cyc;
  cudaMallocManaged(&cyc, 256 * sizeof(long long));
  double2* sink;
  cudaMalloc(&sink, 64);
  const int ns[] = {1, 33, 66, 148};
  const long sizes[] = {256L << 10, 5L << 20, 32L << 20};   // per CTA
  printf("per-CTA region | CTAs | U | passes | B/clk/SM (mean) | aggregate GB/s at 1.965 GHz\n");
  for (long sz : sizes)
    for (int n : ns)
      for (int U : {8, 16, 32}) {
        const long elems = sz / 16;
        const int passes = sz <= (256L << 10) ? 40 : (sz <= (5L << 20) ? 4 : 1);
        for (int rep = 0; rep < 2; ++rep) {
          if (U == 8) k_stream<8><<<n, 288>>>(buf, elems, passes, sink, cyc);
          else if (U == 16) k_stream<16><<<n, 288>>>(buf, elems, passes, sink, cyc);
          else k_stream<32><<<n, 288>>>(buf, elems, passes, sink, cyc);
          cudaDeviceSynchronize();
        }
        double mean = 0;
        for (int i = 0; i < n; ++i) mean += (double)cyc[i];
        mean /= n;
        const double bpc = (double)sz * passes / mean;
        printf("%8ld KB | %3d | %2d | %2d | %6.1f | %8.0f\n", sz >> 10, n, U, passes, bpc, bpc * n * 1.965);
      }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
