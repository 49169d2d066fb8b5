// bench_gj.cu -- the register-row Gauss-Jordan (row_gj.cuh) in isolation: cycles
// per 35 x 35 complex inversion, one CTA alone (latency) and a full GPU of CTAs
// (throughput), for row_invert (2 threads per row, normalised pivot row) and
// row_invert_g<LPR> (raw pivot row, multipliers through shared memory).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2408_11929_b200/csrc -I include tools/bench_gj.cu -o tools/bench_gj
#include <cstdio>
#include <cstring>
#include <cmath>
#include "row_gj.cuh"
#include "../tools/warp_gj.cuh"

constexpr int W = 35, NMAT = 64;

__device__ __noinline__ cplx hash_entry(int m, int i, int j) {
  unsigned x = (unsigned)(m * 1315423911u) ^ (unsigned)(i * 2654435761u) ^ (unsigned)(j * 97531u);
  x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
  const double r = (double)(x & 0xffff) / 65536.0 - 0.5, q = (double)((x >> 16) & 0xffff) / 65536.0 - 0.5;
  return cmk(r + (i == j ? 4.0 : 0.0), q);
}

template <int MODE>   // 0: row_invert, k > 0: row_invert_g<k>, -1: row_invert_p
__global__ void k_bench(long long* out, double* sink, cplx* inv0) {
  __shared__ RowSmem sm;
  if (threadIdx.x == 0) sm.gjp[0] = sm.gjp[1] = sm.gjp[2] = 0;
  __syncthreads();
  constexpr int LPR = MODE <= 0 ? kLPR : MODE;
  constexpr int HW = kRowW / LPR;
  const int i = threadIdx.x / LPR, h = threadIdx.x % LPR;
  double acc = 0;
  long long t0 = clock64();
  for (int m = 0; m < NMAT; ++m) {
    cplx a[HW];
#pragma unroll
    for (int jj = 0; jj < HW; ++jj) {
      const int col = LPR * jj + h;
      a[jj] = (i < W && col < W) ? hash_entry(m + blockIdx.x, i, col) : cmk(0, 0);
    }
    int bad;
    if constexpr (MODE == 0) bad = row_invert(a, W, sm);
    else if constexpr (MODE == -2) bad = row_invert_r<HELM_ROW_UP>(a, W, sm);
    else bad = row_invert_g<LPR>(a, W, sm);
    if (m == 0) {   // the first inverse, for the comparison of the variants
      __syncthreads();
      for (int e = threadIdx.x; e < W * W; e += blockDim.x) inv0[(long)blockIdx.x * W * W + e] = sm.mat[(e / W) * kRowW + e % W];
      __syncthreads();
    }
    acc += bad + sm.mat[(threadIdx.x % W) * kRowW].x;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = t1 - t0;
    if (blockIdx.x == 0) { out[gridDim.x] = sm.gjp[0]; out[gridDim.x + 1] = sm.gjp[1]; out[gridDim.x + 2] = sm.gjp[2]; }
  }
  if (acc == 12345.0) sink[0] = acc;
}


// one warp per inversion (warp_gj.cuh): WPC warps per CTA, each with its own
// WarpGJ + 36 x 36 output block in dynamic shared memory (the factorisation's layout)
constexpr int NPOOL = 256;   // the warp variant reads its blocks from a pool (no calls next to 144 live registers)
__global__ void k_fill_pool(cplx* pool) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < NPOOL * kWW * kWW; e += gridDim.x * blockDim.x) {
    const int m = e / (kWW * kWW), i = (e / kWW) % kWW, j = e % kWW;
    pool[e] = (i < W && j < W) ? hash_entry(m, i, j) : cmk(0, 0);
  }
}
template <int U>
__global__ void k_bench_warp(long long* out, double* sink, cplx* inv0, int wpc, const cplx* __restrict__ pool) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * wpc + warp;
  const size_t per = sizeof(WarpGJ) + sizeof(cplx) * kWW * kWW;
  WarpGJ& g = *reinterpret_cast<WarpGJ*>(smraw + warp * per);
  cplx* mat = reinterpret_cast<cplx*>(smraw + warp * per + sizeof(WarpGJ));
  warp_gj_init(g);
  double acc = 0;
  long long t0 = clock64();
  for (int m = 0; m < NMAT; ++m) {
    cplx a[kWW];
    const cplx* src = pool + (long)((m + gw) % NPOOL) * kWW * kWW;
#pragma unroll
    for (int s = 0; s < kWW; ++s) a[s] = __ldg(src + lane * kWW + s);
    for (int e = lane; e < kWX * kWW; e += 32) g.ext[e / kWW][e % kWW] = __ldg(src + 32 * kWW + e);
    __syncwarp();
    int ks = 0, kx[kWX] = {0, 0, 0, 0};
    const int bad = warp_invert<U>(a, W, g, ks, kx);
    warp_gj_store(a, W, g, ks, kx, mat);
    if (m == 0)
      for (int e = lane; e < W * W; e += 32) inv0[(long)gw * W * W + e] = mat[(e / W) * kWW + e % W];
    acc += bad + mat[(lane % W) * kWW].x;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) out[gw] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}

static cplx* g_ref = nullptr;
template <int MODE>
void run(const char* name, int threads, int ctas) {
  long long* d;
  double* s;
  cudaMalloc(&d, sizeof(long long) * (ctas + 3));
  cudaMalloc(&s, 8);
  cplx* inv;
  cudaMalloc(&inv, sizeof(cplx) * W * W * ctas);
  k_bench<MODE><<<ctas, threads>>>(d, s, inv);
  cudaDeviceSynchronize();
  k_bench<MODE><<<ctas, threads>>>(d, s, inv);
  cudaDeviceSynchronize();
  long long* h = new long long[ctas + 3];
  cudaMemcpy(h, d, sizeof(long long) * (ctas + 3), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int c = 0; c < ctas; ++c) mean += h[c];
  mean /= ctas;
  printf("%-22s threads %3d ctas %4d: %8.0f cycles per inversion per CTA (%.0f per pivot)%s", name, threads, ctas,
         mean / NMAT, mean / NMAT / W, cudaGetLastError() == cudaSuccess ? "" : "  [error]");
  if (h[ctas] + h[ctas + 1] + h[ctas + 2] > 0)   // (-DHELM_GJ_PROF, row_invert_g only; thread 0 of CTA 0)
    printf("  | per pivot: search %.0f publish %.0f update %.0f", h[ctas] / (2.0 * NMAT * W), h[ctas + 1] / (2.0 * NMAT * W),
           h[ctas + 2] / (2.0 * NMAT * W));
  printf("\n");
  static cplx* ref = nullptr;
  cplx* hi = new cplx[W * W];
  cudaMemcpy(hi, inv, sizeof(cplx) * W * W, cudaMemcpyDeviceToHost);
  if (!ref) { ref = new cplx[W * W]; memcpy(ref, hi, sizeof(cplx) * W * W); g_ref = ref; }
  double md = 0;
  for (int e = 0; e < W * W; ++e) md = fmax(md, fabs(hi[e].x - ref[e].x) + fabs(hi[e].y - ref[e].y));
  printf("    max |inv - inv(row_invert)| = %.3e\n", md);
  delete[] hi;
  cudaFree(inv);
  delete[] h;
  cudaFree(d);
  cudaFree(s);
}


template <int U>
void runw(const char* name, int wpc, int ctas) {
  const int nw = wpc * ctas;
  long long* d;
  double* s;
  cudaMalloc(&d, sizeof(long long) * nw);
  cudaMalloc(&s, 8);
  cplx* inv;
  cudaMalloc(&inv, sizeof(cplx) * W * W * nw);
  const size_t smem = wpc * (sizeof(WarpGJ) + sizeof(cplx) * kWW * kWW);
  cudaFuncSetAttribute(k_bench_warp<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  static cplx* pool = nullptr;
  if (!pool) {
    cudaMalloc(&pool, sizeof(cplx) * NPOOL * kWW * kWW);
    k_fill_pool<<<256, 256>>>(pool);
  }
  k_bench_warp<U><<<ctas, 32 * wpc, smem>>>(d, s, inv, wpc, pool);
  cudaDeviceSynchronize();
  k_bench_warp<U><<<ctas, 32 * wpc, smem>>>(d, s, inv, wpc, pool);
  cudaError_t err = cudaDeviceSynchronize();
  long long* h = new long long[nw];
  cudaMemcpy(h, d, sizeof(long long) * nw, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int c = 0; c < nw; ++c) mean += h[c];
  mean /= nw;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bench_warp<U>, 32 * wpc, smem);
  printf("%-22s warps %4d (%d per CTA, %d CTAs/SM): %8.0f cycles per inversion per warp (%.0f per pivot) -> %.0f SM-cycles per inversion%s\n",
         name, nw, wpc, occ, mean / NMAT, mean / NMAT / W, mean / NMAT / (nw < 148 ? 1.0 : (double)nw / 148.0),
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  cplx* hi = new cplx[W * W];
  cudaMemcpy(hi, inv, sizeof(cplx) * W * W, cudaMemcpyDeviceToHost);
  double md = 0;
  for (int e = 0; e < W * W; ++e) md = fmax(md, fabs(hi[e].x - g_ref[e].x) + fabs(hi[e].y - g_ref[e].y));
  printf("    max |inv - inv(row_invert)| = %.3e\n", md);
  delete[] hi;
  cudaFree(inv);
  delete[] h;
  cudaFree(d);
  cudaFree(s);
}

int main() {
  for (int ctas : {1, 148 * 5}) {
    run<0>("row_invert (LPR 2)", 96, ctas);
    run<-2>("row_invert_r (rotating)", 96, ctas);
    run<2>("row_invert_g<2>", 96, ctas);
    run<4>("row_invert_g<4>", 160, ctas);
    run<9>("row_invert_g<9>", 352, ctas);
  }
  runw<2>("warp_invert<2>", 1, 1);
  runw<4>("warp_invert<4>", 1, 1);
  runw<6>("warp_invert<6>", 1, 1);
  for (int wps : {6, 8, 9}) {
    runw<2>("warp_invert<2>", 1, 148 * wps);
    runw<4>("warp_invert<4>", 1, 148 * wps);
    runw<6>("warp_invert<6>", 1, 148 * wps);
  }
  runw<4>("warp_invert<4>", 4, 148 * 2);
  return 0;
}
