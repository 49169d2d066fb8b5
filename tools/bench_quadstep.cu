// Microbenchmark: the k_sweep_dual block step with ONE vs TWO independent
// recurrence chains per warp (lockstep sub-segments), each chain fed by a TMA
// ring of padded packed 35 x 35 complex-symmetric blocks streamed from HBM.
// Question it answers: how much longer is a step that carries two chains than
// one that carries one (the two-sub-segment design halves the chain length).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bench_quadstep tools/bench_quadstep.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef double2 cplx;
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                   smem_u32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ cplx lds128(uint32_t a) {
  cplx v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__host__ __device__ inline int pk_start(int r, int w) {
  const int c = ((2 - w) % 8 + 8) % 8;
  int pad = 28 * (r >> 3);
  for (int i = r & ~7; i < r; ++i) pad += (i + c) & 7;
  return r * w - r * (r - 1) / 2 + pad;
}
__host__ __device__ inline int pk_size(int w) { return ((pk_start(w - 1, w) + 1) + 7) / 8 * 8; }

constexpr int W = 35, KPL = 9, WM = 40, NW = 5;
constexpr int NBLK = 256;   // blocks per chain stream (cycled): 256 x 12 KB x chains >> L2

// NCH chains per warp; NST ring stages per group; each stage holds NCH blocks.
// MODE 0: next blocks' entries read between the FMAs (k_sweep_dual), MODE 1: just in time.
template <int NCH, int NST, int MODE, int NG = 2>
__global__ void __launch_bounds__(NG * NW * 32 + 32 * NG, 1) k_step(int steps, const cplx* __restrict__ F, int pks,
                                                              long long* cyc, cplx* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int stage_elems = NCH * (pks + 8);
  cplx* ring = (cplx*)sm;                                 // [2][NST][NCH][pks+8]
  uint64_t* full = (uint64_t*)(ring + 2 * NST * stage_elems);
  uint64_t* empty = full + 2 * NST;
  cplx* vbuf = (cplx*)(empty + 2 * NST);                  // [2 groups][NCH][2][WM]
  int* pkst = (int*)(vbuf + 2 * NCH * 2 * WM);
  const int tid = threadIdx.x, gsz = NW * 32, ncons = NG * gsz;
  for (int r = tid; r < W; r += blockDim.x) pkst[r] = pk_start(r, W);
  for (int e = tid; e < 2 * NCH * 2 * WM; e += blockDim.x) vbuf[e] = make_double2(1e-3 * (e % 37), 1e-4);
  for (int e = tid; e < 2 * NST * NCH; e += blockDim.x) ring[(long)e * (pks + 8) + pks + 7] = make_double2(0, 0);
  if (tid == 0) {
    for (int e = 0; e < 2 * NST; ++e) { mbar_init(&full[e], 1); mbar_init(&empty[e], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= ncons) {
    const int pg = (tid - ncons) >> 5;
    if ((tid & 31) == 0) {
      const uint32_t bytes = pks * sizeof(cplx);
      for (int f = 0; f < steps; ++f) {
        const int st = f % NST;
        if (f >= NST) mbar_wait(&empty[pg * NST + st], ((f / NST) - 1) & 1);
        mbar_expect_tx(&full[pg * NST + st], bytes * NCH);
        for (int ch = 0; ch < NCH; ++ch) {
          const cplx* src = F + (((long)blockIdx.x * 2 + pg) * NCH + ch) * NBLK * pks + (long)(f % NBLK) * pks;
          bulk_g2s(ring + ((long)pg * NST + st) * stage_elems + ch * (pks + 8), src, bytes, &full[pg * NST + st]);
        }
      }
    }
    return;
  }
  const int g = tid >= gsz ? 1 : 0, gtid = tid - g * gsz, wi = gtid >> 5, lane = tid & 31;
  const int slot = lane & 7, q = lane >> 3;
  const int row = 7 * wi + slot - 1;   // low-halo mapping
  const bool act = row >= 0 && row < W;
  const bool owned = q == 0 && act && slot >= 1;
  uint32_t off[KPL];
  const int zero = pks + 7;
#pragma unroll
  for (int c = 0; c < KPL; ++c) {
    const int k = q + 4 * c;
    int idx = zero;
    if (act && k < W) idx = k >= row ? pkst[row] + (k - row) : pkst[k] + (row - k);
    off[c] = idx * 16u;
  }
  const uint32_t rb = smem_u32(ring + (long)g * NST * stage_elems);
  const uint32_t sbytes = stage_elems * 16u;
  cplx* myv = vbuf + g * NCH * 2 * WM;
  int cur = 0;
  long long t0 = clock64();
  cplx acc_out = make_double2(0, 0);
  if (MODE == 0) {
    cplx S[NCH][2][KPL];
    mbar_wait(&full[g * NST], 0);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
      for (int c = 0; c < KPL; ++c) S[ch][0][c] = lds128(rb + ch * (pks + 8) * 16u + off[c]);
    for (int s = 0; s < steps; s += 2) {
#pragma unroll
      for (int hb = 0; hb < 2; ++hb) {
        const int ss = s + hb;
        const int st = ss % NST;
        const bool last = ss + 1 >= steps;
        uint32_t sbn = 0;
        if (!last) {
          mbar_wait(&full[g * NST + (ss + 1) % NST], ((ss + 1) / NST) & 1);
          sbn = rb + ((ss + 1) % NST) * sbytes;
        }
        cplx o[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const cplx* vin = myv + (ch * 2 + cur) * WM;
          cplx a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
          for (int c = 0; c < KPL; ++c) {
            const cplx v = vin[q + 4 * c];
            if ((c & 3) == 0) cfma(a0, S[ch][hb][c], v);
            else if ((c & 3) == 1) cfma(a1, S[ch][hb][c], v);
            else if ((c & 3) == 2) cfma(a2, S[ch][hb][c], v);
            else cfma(a3, S[ch][hb][c], v);
            if (!last) S[ch][hb ^ 1][c] = lds128(sbn + ch * (pks + 8) * 16u + off[c]);
          }
          cplx a = make_double2(a0.x + a1.x + a2.x + a3.x, a0.y + a1.y + a2.y + a3.y);
          a.x += __shfl_xor_sync(0xffffffffu, a.x, 16);
          a.y += __shfl_xor_sync(0xffffffffu, a.y, 16);
          a.x += __shfl_xor_sync(0xffffffffu, a.x, 8);
          a.y += __shfl_xor_sync(0xffffffffu, a.y, 8);
          o[ch] = a;
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          cplx nb;
          nb.x = __shfl_up_sync(0xffffffffu, o[ch].x, 1, 8);
          nb.y = __shfl_up_sync(0xffffffffu, o[ch].y, 1, 8);
          if (owned) {
            cplx t = make_double2(1e-2 * o[ch].x - 1e-3 * nb.x, 1e-2 * o[ch].y + 1e-3 * nb.y);
            myv[(ch * 2 + (cur ^ 1)) * WM + row] = t;
          }
          acc_out.x += o[ch].x;
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(gsz) : "memory");
        if (gtid == 0) mbar_arrive(&empty[g * NST + st]);
        cur ^= 1;
      }
    }
  } else {
    for (int s = 0; s < steps; ++s) {
      const int st = s % NST;
      mbar_wait(&full[g * NST + st], (s / NST) & 1);
      const uint32_t sb = rb + st * sbytes;
      cplx a[NCH][2];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) a[ch][0] = a[ch][1] = make_double2(0, 0);
#pragma unroll
      for (int c = 0; c < KPL; ++c)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const cplx sv = lds128(sb + ch * (pks + 8) * 16u + off[c]);
          const cplx v = myv[(ch * 2 + cur) * WM + q + 4 * c];
          cfma(a[ch][c & 1], sv, v);
        }
      cplx o[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        cplx x = make_double2(a[ch][0].x + a[ch][1].x, a[ch][0].y + a[ch][1].y);
        x.x += __shfl_xor_sync(0xffffffffu, x.x, 16);
        x.y += __shfl_xor_sync(0xffffffffu, x.y, 16);
        x.x += __shfl_xor_sync(0xffffffffu, x.x, 8);
        x.y += __shfl_xor_sync(0xffffffffu, x.y, 8);
        o[ch] = x;
      }
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        cplx nb;
        nb.x = __shfl_up_sync(0xffffffffu, o[ch].x, 1, 8);
        nb.y = __shfl_up_sync(0xffffffffu, o[ch].y, 1, 8);
        if (owned) {
          cplx t = make_double2(1e-2 * o[ch].x - 1e-3 * nb.x, 1e-2 * o[ch].y + 1e-3 * nb.y);
          myv[(ch * 2 + (cur ^ 1)) * WM + row] = t;
        }
        acc_out.x += o[ch].x;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(gsz) : "memory");
      if (gtid == 0) mbar_arrive(&empty[g * NST + st]);
      cur ^= 1;
    }
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  if (owned) out[(long)blockIdx.x * 512 + tid] = acc_out;
}

template <int NCH, int NST, int MODE, int NG = 2>
void run(const char* name, int ctas, const cplx* F, int pks, long long* dcyc, cplx* dout) {
  const int steps = 2048;
  const int stage_elems = NCH * (pks + 8);
  size_t smem = 16ul * 2 * NST * stage_elems + 8 * 4 * NST + 16ul * 2 * NCH * 2 * WM + 4 * 64 + 256;
  cudaFuncSetAttribute(k_step<NCH, NST, MODE, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_step<NCH, NST, MODE, NG><<<ctas, NG * NW * 32 + 32 * NG, smem>>>(steps, F, pks, dcyc, dout);
  cudaEventRecord(e0);
  k_step<NCH, NST, MODE, NG><<<ctas, NG * NW * 32 + 32 * NG, smem>>>(steps, F, pks, dcyc, dout);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[160];
  cudaMemcpy(h, dcyc, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < ctas; ++i) avg += h[i];
  avg /= ctas;
  const double bytes = (double)ctas * NG * NCH * steps * pks * 16.0;
  printf("%-34s ctas=%3d  %6.0f cycles/step  %5.0f cycles/(chain-step per group)  %6.3f ms  %6.0f GB/s  err=%s\n", name,
         ctas, avg / steps, avg / steps / NCH, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}


// FP32 data path: factor blocks float2 (8 B per entry), input vector float2, FP32 FMAs
__device__ __forceinline__ void cfmaf(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
template <int NST, int CONV>
__global__ void __launch_bounds__(2 * NW * 32 + 64, 1) k_step32(int steps, const float2* __restrict__ F, int pks,
                                                                long long* cyc, float2* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int stage_elems = pks + 8;
  float2* ring = (float2*)sm;
  uint64_t* full = (uint64_t*)(ring + 2 * NST * stage_elems);
  uint64_t* empty = full + 2 * NST;
  float2* vbuf = (float2*)(empty + 2 * NST);
  double2* vbufd = (double2*)(vbuf + 2 * 2 * WM);
  int* pkst = (int*)(vbufd + 2 * 2 * WM);
  const int tid = threadIdx.x, gsz = NW * 32, ncons = 2 * gsz;
  for (int r = tid; r < W; r += blockDim.x) pkst[r] = pk_start(r, W);
  for (int e = tid; e < 2 * 2 * WM; e += blockDim.x) { vbuf[e] = make_float2(1e-3f * (e % 37), 1e-4f); vbufd[e] = make_double2(1e-3 * (e % 37), 1e-4); }
  for (int e = tid; e < 2 * NST; e += blockDim.x) ring[(long)e * stage_elems + pks + 7] = make_float2(0, 0);
  if (tid == 0) {
    for (int e = 0; e < 2 * NST; ++e) { mbar_init(&full[e], 1); mbar_init(&empty[e], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= ncons) {
    const int pg = (tid - ncons) >> 5;
    if ((tid & 31) == 0) {
      const uint32_t bytes = pks * sizeof(float2);
      for (int f = 0; f < steps; ++f) {
        const int st = f % NST;
        if (f >= NST) mbar_wait(&empty[pg * NST + st], ((f / NST) - 1) & 1);
        mbar_expect_tx(&full[pg * NST + st], bytes);
        const float2* src = F + ((long)blockIdx.x * 2 + pg) * NBLK * pks + (long)(f % NBLK) * pks;
        bulk_g2s(ring + ((long)pg * NST + st) * stage_elems, src, bytes, &full[pg * NST + st]);
      }
    }
    return;
  }
  const int g = tid >= gsz ? 1 : 0, gtid = tid - g * gsz, wi = gtid >> 5, lane = tid & 31;
  const int slot = lane & 7, q = lane >> 3;
  const int row = 7 * wi + slot - 1;
  const bool act = row >= 0 && row < W;
  const bool owned = q == 0 && act && slot >= 1;
  uint32_t off[KPL];
#pragma unroll
  for (int c = 0; c < KPL; ++c) {
    const int k = q + 4 * c;
    int idx = pks + 7;
    if (act && k < W) idx = k >= row ? pkst[row] + (k - row) : pkst[k] + (row - k);
    off[c] = idx * 8u;
  }
  const uint32_t rb = smem_u32(ring + (long)g * NST * stage_elems);
  const uint32_t sbytes = stage_elems * 8u;
  float2* myv = vbuf + g * 2 * WM;
  double2* myvd = vbufd + g * 2 * WM;
  int cur = 0;
  long long t0 = clock64();
  float accout = 0.f;
  double accoutd = 0.0;
  float2 S[2][KPL];
  mbar_wait(&full[g * NST], 0);
#pragma unroll
  for (int c = 0; c < KPL; ++c) S[0][c] = lds64(rb + off[c]);
  for (int s = 0; s < steps; s += 2) {
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const int ss = s + hb;
      const int st = ss % NST;
      const bool last = ss + 1 >= steps;
      uint32_t sbn = 0;
      if (!last) {
        mbar_wait(&full[g * NST + (ss + 1) % NST], ((ss + 1) / NST) & 1);
        sbn = rb + ((ss + 1) % NST) * sbytes;
      }
      if (CONV == 0) {
        const float2* vin = myv + cur * WM;
        float2 a0 = make_float2(0, 0), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
        for (int c = 0; c < KPL; ++c) {
          const float2 v = vin[q + 4 * c];
          if ((c & 3) == 0) cfmaf(a0, S[hb][c], v);
          else if ((c & 3) == 1) cfmaf(a1, S[hb][c], v);
          else if ((c & 3) == 2) cfmaf(a2, S[hb][c], v);
          else cfmaf(a3, S[hb][c], v);
          if (!last) S[hb ^ 1][c] = lds64(sbn + off[c]);
        }
        float2 a = make_float2(a0.x + a1.x + a2.x + a3.x, a0.y + a1.y + a2.y + a3.y);
        a.x += __shfl_xor_sync(0xffffffffu, a.x, 16);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, 16);
        a.x += __shfl_xor_sync(0xffffffffu, a.x, 8);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, 8);
        float2 nb;
        nb.x = __shfl_up_sync(0xffffffffu, a.x, 1, 8);
        nb.y = __shfl_up_sync(0xffffffffu, a.y, 1, 8);
        if (owned) myv[(cur ^ 1) * WM + row] = make_float2(1e-2f * a.x - 1e-3f * nb.x, 1e-2f * a.y + 1e-3f * nb.y);
        accout += a.x;
      } else {
        // fp32 factors, fp64 vector and accumulation (convert each entry)
        const double2* vin = myvd + cur * WM;
        double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
        for (int c = 0; c < KPL; ++c) {
          const double2 v = vin[q + 4 * c];
          const double2 sv = make_double2((double)S[hb][c].x, (double)S[hb][c].y);
          if ((c & 3) == 0) cfma(a0, sv, v);
          else if ((c & 3) == 1) cfma(a1, sv, v);
          else if ((c & 3) == 2) cfma(a2, sv, v);
          else cfma(a3, sv, v);
          if (!last) S[hb ^ 1][c] = lds64(sbn + off[c]);
        }
        double2 a = make_double2(a0.x + a1.x + a2.x + a3.x, a0.y + a1.y + a2.y + a3.y);
        a.x += __shfl_xor_sync(0xffffffffu, a.x, 16);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, 16);
        a.x += __shfl_xor_sync(0xffffffffu, a.x, 8);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, 8);
        double2 nb;
        nb.x = __shfl_up_sync(0xffffffffu, a.x, 1, 8);
        nb.y = __shfl_up_sync(0xffffffffu, a.y, 1, 8);
        if (owned) myvd[(cur ^ 1) * WM + row] = make_double2(1e-2 * a.x - 1e-3 * nb.x, 1e-2 * a.y + 1e-3 * nb.y);
        accoutd += a.x;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(gsz) : "memory");
      if (gtid == 0) mbar_arrive(&empty[g * NST + st]);
      cur ^= 1;
    }
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  if (owned) out[(long)blockIdx.x * 512 + tid] = make_float2(accout, (float)accoutd);
}

template <int NST, int CONV>
void run32(const char* name, int ctas, const float2* F, int pks, long long* dcyc, float2* dout) {
  const int steps = 2048;
  size_t smem = 8ul * 2 * NST * (pks + 8) + 8 * 4 * NST + 8ul * 4 * WM + 16ul * 4 * WM + 4 * 64 + 256;
  cudaFuncSetAttribute(k_step32<NST, CONV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_step32<NST, CONV><<<ctas, 2 * NW * 32 + 64, smem>>>(steps, F, pks, dcyc, dout);
  cudaEventRecord(e0);
  k_step32<NST, CONV><<<ctas, 2 * NW * 32 + 64, smem>>>(steps, F, pks, dcyc, dout);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[160];
  cudaMemcpy(h, dcyc, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < ctas; ++i) avg += h[i];
  avg /= ctas;
  printf("%-40s ctas=%3d  %6.0f cycles/step  %6.3f ms  err=%s\n", name, ctas, avg / steps, ms,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int pks = pk_size(W);
  const long n = (long)nsm * 2 * 2 * NBLK * pks;
  cplx* F;
  if (cudaMalloc(&F, n * sizeof(cplx)) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(F, 0, n * sizeof(cplx));
  long long* dcyc;
  cplx* dout;
  cudaMalloc(&dcyc, 8 * 1024);
  cudaMalloc(&dout, 16L * 160 * 512);
  printf("pk_size(35) = %d entries (%d bytes)\n", pks, pks * 16);
  for (int ctas : {1, 132}) {
    run<1, 4, 0>("fp64: 2 groups x 1 chain NST4 prefetch", ctas, F, pks, dcyc, dout);
    run32<4, 0>("fp32 data path: 2 groups x 1 chain NST4", ctas, (const float2*)F, pks, dcyc, (float2*)dout);
    run32<6, 0>("fp32 data path: 2 groups x 1 chain NST6", ctas, (const float2*)F, pks, dcyc, (float2*)dout);
    run32<4, 1>("fp32 factors, fp64 vector+FMA NST4", ctas, (const float2*)F, pks, dcyc, (float2*)dout);
    run32<6, 1>("fp32 factors, fp64 vector+FMA NST6", ctas, (const float2*)F, pks, dcyc, (float2*)dout);
  }
  for (int ctas : {1, 136, nsm}) {
    run<1, 4, 0>("2 groups x 1 chain NST4 prefetch", ctas, F, pks, dcyc, dout);
    run<1, 4, 0, 1>("1 group x 1 chain NST4 prefetch", ctas, F, pks, dcyc, dout);
    run<1, 6, 0, 1>("1 group x 1 chain NST6 prefetch", ctas, F, pks, dcyc, dout);
    run<1, 4, 1, 1>("1 group x 1 chain NST4 just-in-time", ctas, F, pks, dcyc, dout);
    run<2, 4, 1, 1>("1 group x 2 chains NST4 just-in-time", ctas, F, pks, dcyc, dout);
  }
  return 0;
}
