// Microbenchmark: streaming w x w complex blocks (19.6 KB) into shared memory
// per CTA with (a) one cp.async.bulk per block, (b) cp.async.bulk split into
// row-sized chunks, (c) 16-byte cp.async (LDGSTS), (d) LDG.128 -> STS.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_tma tools/bench_tma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS>
__global__ void k_bulk(const char* src, long blocks_per_cta, int bytes, int chunks, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  char* stage = (char*)(sm + 256);
  const char* base = src + (long)blockIdx.x * blocks_per_cta * bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](long f) {
    int s = f % NS;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes));
    int cb = bytes / chunks;
    for (int c = 0; c < chunks; ++c)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(stage + (long)s * bytes + (long)c * cb)),
                   "l"(base + f * bytes + (long)c * cb), "r"(cb), "r"(su32(&full[s]))
                   : "memory");
  };
  if (threadIdx.x == 0)
    for (int f = 0; f < NS && f < blocks_per_cta; ++f) issue(f);
  double acc = 0;
  for (long k = 0; k < blocks_per_cta; ++k) {
    int s = k % NS;
    uint32_t par = (k / NS) & 1;
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                     su32(&full[s])),
                 "r"(par));
    acc += ((double*)(stage + (long)s * bytes))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && k + NS < blocks_per_cta) issue(k + NS);
  }
  if (acc == 12345.0) sink[0] = 1;
}

__global__ void k_ldg(const char* src, long blocks_per_cta, int bytes, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int4* base = (const int4*)(src + (long)blockIdx.x * blocks_per_cta * bytes);
  int4* st = (int4*)sm;
  const int n16 = bytes / 16;
  double acc = 0;
  for (long k = 0; k < blocks_per_cta; ++k) {
    const int4* b = base + k * n16;
    for (int i = threadIdx.x; i < n16; i += blockDim.x) st[i] = __ldg(b + i);
    __syncthreads();
    acc += ((double*)sm)[threadIdx.x];
    __syncthreads();
  }
  if (acc == 12345.0) sink[0] = 1;
}

int main() {
  const int bytes = 35 * 35 * 16;  // 19600
  const int ctas = 132;
  const long per = 2000;
  size_t total = (size_t)ctas * per * bytes;
  char* src;
  unsigned long long* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 0, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto report = [&](const char* name, float ms) {
    printf("%-40s %8.3f ms  %8.1f GB/s total  %6.2f GB/s/CTA  %6.1f ns/block\n", name, ms, total / ms / 1e6,
           total / ms / 1e6 / ctas, ms * 1e6 / per);
  };
  int smem = 256 + 8 * bytes;
  cudaFuncSetAttribute(k_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  for (int chunks : {1, 5, 35, 245}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_bulk<8><<<ctas, 288, smem>>>(src, per, bytes, chunks, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      char nm[64];
      snprintf(nm, 64, "bulk NS=8 chunks=%d", chunks);
      if (rep) report(nm, ms);
    }
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_bulk<4><<<ctas, 288, smem>>>(src, per, bytes, 1, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) report("bulk NS=4 chunks=1", ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_ldg<<<ctas, 288, bytes>>>(src, per, bytes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) report("ldg.128 -> sts (no prefetch)", ms);
  }
  // small total: L2-resident re-reads (per CTA the same 8 blocks)
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
