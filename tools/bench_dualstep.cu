// Microbenchmark of the k_sweep_dual block step in isolation (one CTA per SM,
// two groups of 5 warps, 4 lanes per row, 9 complex products per lane, named
// barrier per group).  Variants isolate the DFMA block, the shuffles and the
// barrier.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_dualstep tools/bench_dualstep.cu
#include <cstdio>
#include <cuda_runtime.h>

struct cd { double x, y; };
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

template <int VAR, int GG>
__device__ __forceinline__ void body(int steps, double2* out, long long* cyc, const double2* __restrict__ F,
                                     double2 (*vb)[2][40]) {
  const int tid = threadIdx.x, g = GG, gt = tid - g * 160, lane = tid & 31, q = lane & 3;
  for (int e = tid - g * 160; e < 80; e += 160) (&vb[g][0][0])[e] = make_double2(1e-3 * e, 2e-3);
  double2 S[9];
  for (int c = 0; c < 9; ++c) S[c] = make_double2(1e-2 * (c + tid % 7), 1e-3 * c);
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(160) : "memory");
  const int w = 35;
  int cur = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const double2* vin = vb[g][cur];
    double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
    if (VAR != 3) {
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        const int k = q + 4 * c;
        if (k < w) {
          const double2 v = vin[k];
          if ((c & 3) == 0) cfma(a0, S[c], v);
          else if ((c & 3) == 1) cfma(a1, S[c], v);
          else if ((c & 3) == 2) cfma(a2, S[c], v);
          else cfma(a3, S[c], v);
        }
      }
    } else {
      a0 = vin[q];
    }
    double2 acc = make_double2(a0.x + a1.x + a2.x + a3.x, a0.y + a1.y + a2.y + a3.y);
    if (VAR != 2) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
    }
    if (VAR == 4 || VAR == 5) {
      // refill S like k_sweep_dual: 9 x 16-byte loads per lane from a 35 x 35 block
      // row-major (8 rows x 64 bytes per warp instruction), a new block every step
      const double2* B = F + ((long)blockIdx.x * 2 + g) * 4096L * 1225 + (long)(s % 4096) * 1225;
      const int r = (gt >> 5) * 7 + (lane >> 2) - 1;
      if (r >= 0 && r < w) {
#pragma unroll
        for (int c = 0; c < 9; ++c)
          if (q + 4 * c < w) S[c] = VAR == 4 ? __ldg(B + r * w + q + 4 * c) : __ldg(F + r * w + q + 4 * c);
      }
    }
    const int row = (gt >> 5) * 7 + (lane >> 2) - 1;
    if (q == 0 && row >= 0 && row < w) vb[g][cur ^ 1][row] = make_double2(acc.x * 1e-2, acc.y * 1e-2);
    if (VAR != 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(160) : "memory");
    else __syncwarp();
    cur ^= 1;
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  if (tid == 0) out[blockIdx.x] = vb[0][cur][0];
}

template <int VAR>
__global__ void __launch_bounds__(320, 1) k(int steps, double2* out, long long* cyc, const double2* __restrict__ F) {
  __shared__ double2 vb[2][2][40];
  if (VAR == 6) {
    // the two groups execute two different copies of the loop (as in k_sweep_dual)
    if (threadIdx.x < 160) body<4, 0>(steps, out, cyc, F, vb);
    else body<4, 1>(steps, out, cyc, F, vb);
  } else {
    if (threadIdx.x < 160) body<VAR, 0>(steps, out, cyc, F, vb);
    else body<VAR, 1>(steps, out, cyc, F, vb);
  }
}

__global__ void k_tput(double* out, int iters, int nchains) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double2* o;
  long long* cyc;
  double* d;
  cudaMalloc(&o, 1 << 20);
  cudaMalloc(&cyc, 1 << 20);
  cudaMalloc(&d, 1 << 26);
  long long h[256];
  const int steps = 4000;
  const char* names[] = {"full step", "no barrier (syncwarp)", "no shuffles", "no FMAs", "+LDG refill (streaming)", "+LDG refill (same block)", "+LDG, distinct code per group"};
  double2* F;
  const long fbytes = (long)nsm * 2 * 4096L * 1225 * 16;
  if (cudaMalloc(&F, fbytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(F, 0, fbytes);
  for (int ctas : {1, nsm}) {
    for (int v = 0; v < 7; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) k<0><<<ctas, 320>>>(steps, o, cyc, F);
        if (v == 1) k<1><<<ctas, 320>>>(steps, o, cyc, F);
        if (v == 2) k<2><<<ctas, 320>>>(steps, o, cyc, F);
        if (v == 3) k<3><<<ctas, 320>>>(steps, o, cyc, F);
        if (v == 4) k<4><<<ctas, 320>>>(steps, o, cyc, F);
        if (v == 5) k<5><<<ctas, 320>>>(steps, o, cyc, F);
        if (v == 6) k<6><<<ctas, 320>>>(steps, o, cyc, F);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(long long) * 1, cudaMemcpyDeviceToHost);
      printf("ctas=%3d %-24s %7.0f cycles/step\n", ctas, names[v], (double)h[0] / steps);
    }
  }
  // FP64 throughput with 10 warps per SM and with 32 warps per SM
  for (int thr : {320, 1024}) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    k_tput<<<nsm, thr>>>(d, iters, 8);
    cudaEventRecord(e0);
    k_tput<<<nsm, thr>>>(d, iters, 8);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * nsm * thr * (double)iters * 8;
    printf("DFMA throughput, %4d threads/SM: %.1f TFLOP/s\n", thr, fl / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
