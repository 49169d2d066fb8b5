// Streaming mat-vec chain: S_j (35x35 complex, row-major, contiguous in global)
// consumed either (a) from global straight into registers with a D-step register
// prefetch (LDG path) or (b) via a TMA bulk-copy smem ring (TMA path).
// Realistic per-step vector work (tA + tB input, writer producing next tA/tB).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_ldg tools/bench_ldg.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int W = 35, L = 8, NK = 5;

__device__ __forceinline__ void cfma(double2& a, double2 m, double2 x) {
  a.x = fma(m.x, x.x, a.x); a.x = fma(-m.y, x.y, a.x);
  a.y = fma(m.x, x.y, a.y); a.y = fma(m.y, x.x, a.y);
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int D>
__global__ void __launch_bounds__(288) k_ldg(const double2* __restrict__ src, int steps, long stride_cta,
                                             double2* out, long long* cyc) {
  __shared__ double2 tA[2][64], tB[2][64], co[192];
  for (int e = threadIdx.x; e < 128; e += blockDim.x) { (&tA[0][0])[e] = make_double2(1, .5); (&tB[0][0])[e] = make_double2(0, 0); }
  for (int e = threadIdx.x; e < 192; e += blockDim.x) co[e] = make_double2(0.1, 0.01);
  __syncthreads();
  const int ri = threadIdx.x / L, q = threadIdx.x % L;
  const double2* base = src + (long)blockIdx.x * stride_cta;
  double2 pre[D][NK];
  auto load = [&](int j, double2* dst) {
    const double2* S = base + (long)j * W * W + ri * W;
#pragma unroll
    for (int c = 0; c < NK; ++c) {
      int k = q + c * L;
      dst[c] = (ri < W && k < W) ? __ldcg(S + k) : make_double2(0, 0);
    }
  };
#pragma unroll
  for (int d = 0; d < D; ++d) load(d, pre[d]);
  long long t0 = clock64();
  int cur = 0;
  for (int s = 0; s < steps; s += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double2 m[NK];
#pragma unroll
      for (int c = 0; c < NK; ++c) m[c] = pre[d][c];
      if (s + d + D < steps) load(s + d + D, pre[d]);
      double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
#pragma unroll
      for (int c = 0; c < NK; ++c) {
        int k = q + c * L;
        if (k < W) {
          double2 va = tA[cur][k], vb = tB[cur][k];
          double2 v = make_double2(va.x + vb.x, va.y + vb.y);
          if (c & 1) cfma(a1, m[c], v); else cfma(a0, m[c], v);
        }
      }
      double2 acc = make_double2(a0.x + a1.x, a0.y + a1.y);
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      }
      if (q == 0 && ri < W) {
        double2 cr = co[ri], ne = co[64 + ri], bn = co[128 + ri];
        tA[cur ^ 1][ri] = make_double2(bn.x - (cr.x * acc.x - cr.y * acc.y) * 1e-2, bn.y - (cr.x * acc.y + cr.y * acc.x) * 1e-2);
        if (ri + 1 < W) tB[cur ^ 1][ri + 1] = make_double2(-(ne.x * acc.x) * 1e-2, -(ne.y * acc.y) * 1e-2);
        if (ri == 0) tB[cur ^ 1][0] = make_double2(0, 0);
      }
      __syncthreads();
      cur ^= 1;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = tA[cur][0]; }
}

template <int NS>
__global__ void __launch_bounds__(320) k_tma(const double2* __restrict__ src, int steps, long stride_cta, double2* out,
                                             long long* cyc) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = (uint64_t*)smraw;
  uint64_t* empty = full + 16;
  double2* stage = (double2*)(smraw + 256);
  __shared__ double2 tA[2][64], tB[2][64], co[192];
  const int bytes = W * W * 16;
  const int ncons = 288;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int e = threadIdx.x; e < 128; e += blockDim.x) { (&tA[0][0])[e] = make_double2(1, .5); (&tB[0][0])[e] = make_double2(0, 0); }
  for (int e = threadIdx.x; e < 192; e += blockDim.x) co[e] = make_double2(0.1, 0.01);
  __syncthreads();
  const double2* base = src + (long)blockIdx.x * stride_cta;
  if (threadIdx.x >= ncons) {
    if (threadIdx.x == ncons) {
      for (int f = 0; f < steps; ++f) {
        int s = f % NS;
        if (f >= NS) {
          uint32_t par = ((f / NS) - 1) & 1;
          asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su32(&empty[s])), "r"(par));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + (long)s * W * W)),
                     "l"(base + (long)f * W * W), "r"(bytes), "r"(su32(&full[s])) : "memory");
      }
    }
    return;
  }
  const int ri = threadIdx.x / L, q = threadIdx.x % L;
  long long t0 = clock64();
  int cur = 0;
  for (int f = 0; f < steps; ++f) {
    int s = f % NS;
    uint32_t par = (f / NS) & 1;
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su32(&full[s])), "r"(par));
    const double2* S = stage + (long)s * W * W + ri * W;
    double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
    if (ri < W) {
#pragma unroll
      for (int c = 0; c < NK; ++c) {
        int k = q + c * L;
        if (k < W) {
          double2 va = tA[cur][k], vb = tB[cur][k];
          double2 v = make_double2(va.x + vb.x, va.y + vb.y);
          if (c & 1) cfma(a1, S[k], v); else cfma(a0, S[k], v);
        }
      }
    }
    double2 acc = make_double2(a0.x + a1.x, a0.y + a1.y);
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (q == 0 && ri < W) {
      double2 cr = co[ri], ne = co[64 + ri], bn = co[128 + ri];
      tA[cur ^ 1][ri] = make_double2(bn.x - (cr.x * acc.x - cr.y * acc.y) * 1e-2, bn.y - (cr.x * acc.y + cr.y * acc.x) * 1e-2);
      if (ri + 1 < W) tB[cur ^ 1][ri + 1] = make_double2(-(ne.x * acc.x) * 1e-2, -(ne.y * acc.y) * 1e-2);
      if (ri == 0) tB[cur ^ 1][0] = make_double2(0, 0);
    }
    asm volatile("bar.sync 1, 288;" ::: "memory");
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    cur ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = tA[cur][0]; }
}

int main() {
  const int steps = 2000;
  const long stride = (long)steps * W * W;
  const int maxctas = 148 * 4;
  double2* src;
  double2* o2;
  long long* cyc;
  size_t bytes = sizeof(double2) * stride * maxctas;   // 2.9 GB: HBM streaming
  if (cudaMalloc(&src, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(src, 0x3f, bytes);
  cudaMalloc(&o2, 1 << 16);
  cudaMalloc(&cyc, 1 << 16);
  static long long h[maxctas];
  auto rep = [&](const char* nm, int ctas, int per_sm) {
    cudaMemcpy(h, cyc, 8 * ctas, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < ctas; ++i) avg += h[i];
    avg /= ctas;
    printf("%-16s CTAs/SM=%d: %6.0f cyc/step per CTA -> %5.0f cyc per block-step per SM  (%s)\n", nm, per_sm,
           avg / steps, avg / steps / per_sm, cudaGetErrorString(cudaGetLastError()));
  };
  for (int per : {1, 2, 3, 4}) {
    int ctas = 148 * per;
    k_ldg<2><<<ctas, 288>>>(src, steps, stride, o2, cyc);
    cudaDeviceSynchronize();
    rep("LDG D=2", ctas, per);
    k_ldg<3><<<ctas, 288>>>(src, steps, stride, o2, cyc);
    cudaDeviceSynchronize();
    rep("LDG D=3", ctas, per);
  }
  int smem4 = 256 + 4 * W * W * 16;
  cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4);
  for (int per : {1, 2}) {
    int ctas = 148 * per;
    k_tma<4><<<ctas, 320, smem4>>>(src, steps, stride, o2, cyc);
    cudaDeviceSynchronize();
    rep("TMA NS=4", ctas, per);
  }
}
