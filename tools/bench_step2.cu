// Mat-vec step mappings with realistic next-input production (tA/tB).
// RPT rows per thread (rows g, g+G, ... with G = ceil(W/RPT) groups), L lanes per row group.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_step2 tools/bench_step2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cfma(double2& a, double2 m, double2 x) {
  a.x = fma(m.x, x.x, a.x); a.x = fma(-m.y, x.y, a.x);
  a.y = fma(m.x, x.y, a.y); a.y = fma(m.y, x.x, a.y);
}

template <int W, int L, int RPT, int NCH>
__global__ void k_map(int steps, double2* out, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* S = sm;                        // NCH blocks W x W
  double2* tA = S + NCH * W * W;          // [NCH][2][64]
  double2* tB = tA + NCH * 128;
  double2* co = tB + NCH * 128;           // coefficients [64] x 3
  for (int e = threadIdx.x; e < NCH * W * W; e += blockDim.x) S[e] = make_double2(1e-3 * (e % 17), 1e-3 * (e % 13));
  for (int e = threadIdx.x; e < NCH * 128; e += blockDim.x) tA[e] = tB[e] = make_double2(1.0, 0.5);
  for (int e = threadIdx.x; e < 192; e += blockDim.x) co[e] = make_double2(0.1, 0.01);
  __syncthreads();
  constexpr int G = (W + RPT - 1) / RPT;   // row groups
  const int g = threadIdx.x / L, q = threadIdx.x % L;
  constexpr int NK = (W + L - 1) / L;
  long long t0 = clock64();
  int cur = 0;
  for (int s = 0; s < steps; ++s) {
    double2 acc[NCH][RPT];
#pragma unroll
    for (int h = 0; h < NCH; ++h)
#pragma unroll
      for (int j = 0; j < RPT; ++j) acc[h][j] = make_double2(0, 0);
    if (g < G) {
#pragma unroll
      for (int h = 0; h < NCH; ++h) {
        const double2* Sb = S + h * W * W;
        const double2* a = tA + h * 128 + cur * 64;
        const double2* b = tB + h * 128 + cur * 64;
#pragma unroll
        for (int c = 0; c < NK; ++c) {
          const int k = q + c * L;
          if (k < W) {
            double2 va = a[k], vb = b[k];
            double2 v = make_double2(va.x + vb.x, va.y + vb.y);
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
              const int r = g + j * G;
              if (r < W) cfma(acc[h][j], Sb[r * W + k], v);
            }
          }
        }
      }
    }
    // butterfly over L lanes for every row value
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1)
#pragma unroll
      for (int h = 0; h < NCH; ++h)
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          acc[h][j].x += __shfl_xor_sync(0xffffffffu, acc[h][j].x, off);
          acc[h][j].y += __shfl_xor_sync(0xffffffffu, acc[h][j].y, off);
        }
    // writers: lane j of the group writes row g + j*G (spread the writer work over lanes)
#pragma unroll
    for (int h = 0; h < NCH; ++h)
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int r = g + j * G;
        if (q == (j % L) && g < G && r < W) {
          double2 o = acc[h][j];
          double2 cr = co[r], ne = co[64 + r], bn = co[128 + r];
          double2* An = tA + h * 128 + (cur ^ 1) * 64;
          double2* Bn = tB + h * 128 + (cur ^ 1) * 64;
          An[r] = make_double2(bn.x - (cr.x * o.x - cr.y * o.y) * 1e-2, bn.y - (cr.x * o.y + cr.y * o.x) * 1e-2);
          if (r + 1 < W) Bn[r + 1] = make_double2(-(ne.x * o.x - ne.y * o.y) * 1e-2, -(ne.x * o.y + ne.y * o.x) * 1e-2);
          if (r == 0) Bn[0] = make_double2(0, 0);
        }
      }
    __syncthreads();
    cur ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = tA[cur * 64]; }
}

template <int W, int L, int RPT, int NCH>
void run(double2* o2, long long* cyc) {
  constexpr int G = (W + RPT - 1) / RPT;
  int threads = ((G * L + 31) / 32) * 32;
  size_t smem = sizeof(double2) * (NCH * W * W + NCH * 256 + 192);
  cudaFuncSetAttribute(k_map<W, L, RPT, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_map<W, L, RPT, NCH><<<1, threads, smem>>>(20000, o2, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("w=%d L=%2d rows/thr=%d chains=%d threads=%4d: %6.0f cyc/step  %5.0f per chain-step (%s)\n", W, L, RPT, NCH,
         threads, c / 20000.0, c / 20000.0 / NCH, cudaGetErrorString(cudaGetLastError()));
}

template <int W, int L, int RPT, int NCH>
void run_occ(int per_sm, double2* o2, long long* cyc) {
  constexpr int G = (W + RPT - 1) / RPT;
  int threads = ((G * L + 31) / 32) * 32;
  size_t smem = sizeof(double2) * (NCH * W * W + NCH * 256 + 192);
  cudaFuncSetAttribute(k_map<W, L, RPT, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nsm = 148;
  k_map<W, L, RPT, NCH><<<nsm * per_sm, threads, smem>>>(20000, o2, cyc);
  static long long h[148 * 8];
  cudaMemcpy(h, cyc, 8 * nsm * per_sm, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm * per_sm; ++i) avg += h[i];
  avg /= nsm * per_sm;
  printf("w=%d L=%d rows/thr=%d chains=%d  CTAs/SM=%d: %6.0f cyc/step per CTA -> %5.0f cyc per chain-step per SM (%s)\n",
         W, L, RPT, NCH, per_sm, avg / 20000.0, avg / 20000.0 / NCH / per_sm, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double2* o2;
  long long* cyc;
  cudaMalloc(&o2, 1 << 16);
  cudaMalloc(&cyc, 1 << 16);
  cudaMalloc(&cyc, 1 << 20);
  run_occ<35, 8, 1, 1>(1, o2, cyc);
  run_occ<35, 8, 1, 1>(2, o2, cyc);
  run_occ<35, 8, 1, 1>(3, o2, cyc);
  run_occ<35, 8, 1, 1>(4, o2, cyc);
  run_occ<35, 8, 2, 1>(2, o2, cyc);
  run_occ<35, 8, 2, 1>(4, o2, cyc);
  run_occ<35, 4, 1, 1>(4, o2, cyc);
  run_occ<35, 8, 1, 2>(2, o2, cyc);
  return 0;
  run<35, 8, 1, 1>(o2, cyc);
  run<35, 8, 2, 1>(o2, cyc);
  run<35, 8, 3, 1>(o2, cyc);
  run<35, 8, 4, 1>(o2, cyc);
  run<35, 4, 2, 1>(o2, cyc);
  run<35, 4, 4, 1>(o2, cyc);
  run<35, 16, 2, 1>(o2, cyc);
  run<35, 16, 4, 1>(o2, cyc);
  run<35, 8, 1, 2>(o2, cyc);
  run<35, 8, 2, 2>(o2, cyc);
  run<35, 8, 4, 2>(o2, cyc);
  run<35, 4, 2, 2>(o2, cyc);
  run<35, 16, 2, 2>(o2, cyc);
  run<35, 8, 2, 4>(o2, cyc);
  run<99, 8, 4, 1>(o2, cyc);
  run<99, 16, 4, 1>(o2, cyc);
  run<99, 16, 8, 1>(o2, cyc);
}
