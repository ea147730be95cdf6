// Microbenchmark (measurement tool, not part of the library): cycles per tcgen05.mma issued
// back to back by one thread on one SM, M=128, kind::i8 / kind::f16, operands SS (no swizzle /
// 128-byte swizzle) or TS (A in tensor memory).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/mma_microbench tools/mma_microbench.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t a, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((a >> 4) & 0x3FFF); d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  uint64_t d = 0; d |= (uint64_t)((a >> 4) & 0x3FFF); d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61; return d; }
template <int KIND, int MODE, int N>   // KIND 0 = i8, 1 = f16 ; MODE 0 = SS none, 1 = TS, 2 = SS sw128
__global__ void bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot; __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 131072; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  constexpr uint32_t idesc = KIND == 0 ? ((2 << 4) | ((N >> 3) << 17) | ((128 >> 4) << 24))
                                       : ((1 << 4) | (1 << 7) | (1 << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24));
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 65536);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t ka = (it & 7);
      uint64_t da = MODE == 2 ? desc_sw128(a + (ka & 3) * 32) : desc_none(a + ka * 256, 2048);
      uint64_t db = MODE == 2 || MODE == 1 ? desc_sw128(b + (ka & 3) * 32) : desc_none(b + ka * 256, 2048);
      if (MODE == 1) {
        if (KIND == 0) asm volatile("{\n .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}\n" ::"r"(tm), "r"(tm + 256 + 8 * ka), "l"(db), "r"(idesc), "r"(it));
        else asm volatile("{\n .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}\n" ::"r"(tm), "r"(tm + 256 + 8 * ka), "l"(db), "r"(idesc), "r"(it));
      } else {
        if (KIND == 0) asm volatile("{\n .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}\n" ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(it));
        else asm volatile("{\n .reg .pred p; setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}\n" ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(it));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}
template <int K, int M, int N> void run(const char* name) {
  long long* d; cudaMalloc(&d, 8); long long h;
  cudaFuncSetAttribute(bench<K, M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int w = 0; w < 2; ++w) bench<K, M, N><<<1, 128, 131072>>>(d, 4000);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("%-28s N=%3d  %.1f cycles/MMA  %s\n", name, N, h / 4000.0, cudaGetErrorString(e));
}
int main() {
  run<0, 0, 32>("i8 SS (no swizzle)"); run<0, 0, 64>("i8 SS (no swizzle)"); run<0, 0, 128>("i8 SS (no swizzle)"); run<0, 0, 256>("i8 SS (no swizzle)");
  run<0, 2, 64>("i8 SS (sw128)"); run<0, 2, 128>("i8 SS (sw128)");
  run<0, 1, 32>("i8 TS"); run<0, 1, 64>("i8 TS"); run<0, 1, 128>("i8 TS"); run<0, 1, 256>("i8 TS");
  run<1, 0, 64>("f16 SS (no swizzle)"); run<1, 2, 64>("f16 SS (sw128)"); run<1, 1, 64>("f16 TS"); run<1, 2, 256>("f16 SS (sw128)");
  return 0;
}
