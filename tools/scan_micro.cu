// Micro-benchmark of the 8-bit PQ scan's inner loop (k_pq_scan_rq), to split its time between
// the lookups themselves, the per-chunk LUT staging + barriers, and the code loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/scan_micro tools/scan_micro.cu
// Variants (argv[1]):
//   0  PRMT + LDS + FADD on register-held code words, no barriers, no staging
//   1  0 + the per-chunk staging of the replicated LUT (128 KB) between two barriers
//   2  1 + the code words loaded from global memory (buffer of argv[2] MB, 2 loads in flight)
//   3  2 without the staging (barriers only)
//   4  2 with two waves of accumulators per CTA (the second wave parked in tensor memory), so
//      that one staging of a LUT chunk serves twice the objects
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NT = 1024, GPL = 8, MC = 4, P = 12;
constexpr unsigned kBase = 1024;

template <int IMM>
__device__ __forceinline__ float lds_imm(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(IMM));
  return v;
}
__device__ __forceinline__ float look4(float a, uint32_t w, uint32_t lane4) {
  a = __fadd_rn(a, lds_imm<kBase + 0>(__byte_perm(w, lane4, 0x7604)));
  a = __fadd_rn(a, lds_imm<kBase + 128>(__byte_perm(w, lane4, 0x7614)));
  a = __fadd_rn(a, lds_imm<kBase + 65536>(__byte_perm(w, lane4, 0x7624)));
  a = __fadd_rn(a, lds_imm<kBase + 65536 + 128>(__byte_perm(w, lane4, 0x7634)));
  return a;
}

#define TM_REGS32(v) "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), \
  "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), \
  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), \
  "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
#define TM_IREGS32(v) "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), \
  "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), \
  "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), \
  "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
#define TM_LIST32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
__device__ __forceinline__ void tm_ld32(uint32_t taddr, float* a) {
  uint32_t v[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " TM_LIST32 ", [%32];" : TM_REGS32(v) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int e = 0; e < 32; ++e) a[e] = __uint_as_float(v[e]);
}
__device__ __forceinline__ void tm_st32(uint32_t taddr, const float* a) {
  uint32_t v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(a[e]);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               :: "r"(taddr), TM_IREGS32(v));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

template <int V>
__global__ void __launch_bounds__(NT, 1) k_micro(const uint4* __restrict__ codes, unsigned nwords16, int items,
                                                 float* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  float* lut = reinterpret_cast<float*>(sm);
  if ((unsigned)__cvta_generic_to_shared(sm) != kBase) __trap();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t lane4 = lane * 4u;
  float acc[4 * GPL];
#pragma unroll
  for (int e = 0; e < 4 * GPL; ++e) acc[e] = 0.f;
  uint32_t seed = (blockIdx.x * NT + threadIdx.x) * 2654435761u;
  constexpr int W = V == 4 ? 2 : 1;                  // waves of accumulators per LUT staging
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(sm + 131072);
  uint32_t tm = 0;
  if (V == 4) {
    if (wid == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&tslot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tm = tslot + ((uint32_t)((wid & 3) * 32) << 16) + (uint32_t)((wid >> 2) * 64);
  }
  for (int it = 0; it < items; ++it) {
    // group base (in 16-byte units) of this warp: contiguous 8 KB per chunk-group
    const unsigned gb = ((unsigned)(blockIdx.x + it * gridDim.x) * (NT / 32) + wid) * (GPL * 4 * 8 * P) % nwords16;
    uint4 cw[2];
    auto ldc = [&](int i, int p, int w = 0) -> uint4 {
      const unsigned idx = (gb * W + (unsigned)(((p * W + w) * GPL + i) * 32 + lane)) % nwords16;
      uint4 r;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(codes + idx));
      return r;
    };
    if (V >= 2) { cw[0] = ldc(0, 0); cw[1] = ldc(1, 0); }
#pragma unroll 1
    for (int p = 0; p < P; ++p) {
      if (V >= 1) {
        __syncthreads();
        if (V != 3) {
          const float v = (float)(threadIdx.x + p);
          const float4 a4 = make_float4(v, v, v, v);
          const int ea = threadIdx.x;
          float4* ra = reinterpret_cast<float4*>(lut + (size_t)((ea >> 9) * 256 + (ea & 255)) * 64 + ((ea >> 8) & 1) * 32);
#pragma unroll
          for (int r = 0; r < 8; ++r) ra[(r + lane) & 7] = a4;
        }
        __syncthreads();
      }
      const int pn = p + 1 < P ? p + 1 : p;
#pragma unroll 1
      for (int w = 0; w < W; ++w) {
      if (V == 4 && p > 0) tm_ld32(tm + 32 * w, acc);
      const int wn = w + 1 < W ? w + 1 : 0;
      const int pw = w + 1 < W ? p : pn;
#pragma unroll
      for (int i = 0; i < GPL; ++i) {
        uint4 c;
        if (V >= 2) {
          c = cw[i & 1];
          cw[i & 1] = i + 2 < GPL ? ldc(i + 2, p, w) : ldc(i + 2 - GPL, pw, wn);
        } else {
          seed = seed * 1664525u + 1013904223u;
          c = make_uint4(seed, seed ^ 0x5bd1e995u, seed * 3u, seed ^ 0x9e3779b9u);
        }
        acc[4 * i + 0] = look4(acc[4 * i + 0], c.x, lane4);
        acc[4 * i + 1] = look4(acc[4 * i + 1], c.y, lane4);
        acc[4 * i + 2] = look4(acc[4 * i + 2], c.z, lane4);
        acc[4 * i + 3] = look4(acc[4 * i + 3], c.w, lane4);
      }
      if (V == 4) {
        if (p + 1 < P) tm_st32(tm + 32 * w, acc);
        else if (w == 0) {                         // wave 0 done: fold into the checksum
          float s0 = 0.f;
#pragma unroll
          for (int e = 0; e < 4 * GPL; ++e) { s0 += acc[e]; acc[e] = 0.f; }
          out[blockIdx.x * NT + threadIdx.x] = s0;
        }
      }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < 4 * GPL; ++e) s += acc[e];
  out[blockIdx.x * NT + threadIdx.x] += s;
  if (V == 4) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(512));
  }
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  const size_t mb = argc > 2 ? atol(argv[2]) : 4096;
  const int items = argc > 3 ? atoi(argv[3]) : 64;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = mb << 20;
  uint4* codes;
  float* out;
  cudaMalloc(&codes, bytes);
  cudaMemset(codes, 0x5a, bytes);
  cudaMalloc(&out, (size_t)nsm * NT * 4);
  const int smem = 131072 + 8192;
  auto run = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<nsm, NT, smem>>>(codes, (unsigned)(bytes / 16), items, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<nsm, NT, smem>>>(codes, (unsigned)(bytes / 16), items, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double lookups = (double)nsm * NT * items * P * GPL * 16 * (v == 4 ? 2 : 1);
    printf("{\"variant\": %d, \"mb\": %zu, \"ms\": %.3f, \"Tlookups_s\": %.3f, \"err\": \"%s\"}\n", v, mb,
           ms, lookups / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  if (v == 0) run(k_micro<0>);
  if (v == 1) run(k_micro<1>);
  if (v == 2) run(k_micro<2>);
  if (v == 3) run(k_micro<3>);
  if (v == 4) run(k_micro<4>);
  return 0;
}
