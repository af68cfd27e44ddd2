// Micro-benchmark: tcgen05.ld (LDTM) throughput per SM, alone and while one
// thread keeps the tensor core busy with TS MMAs (A read from TMEM) or SS MMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldtm_rate ldtm_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (bmn ? (1u << 16) : 0u) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
}

// MMA: 0 none, 1 TS (A = TMEM cols [0,64) as 128x128 fp16), 2 SS; the loading
// warps read TMEM columns [128, 256)
template <int MMA>
__global__ void k(int iters, int mma_iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5;
  const int nld = (blockDim.x >> 5) - 1;  // the last warp issues MMAs
  if (warp == nld) {
    if (MMA && (threadIdx.x & 31) == 0) {
      const uint64_t da = desc(su32(s), 16, 1024), db = desc(su32(s + 32768), 16, 1024);
      const uint32_t id = idesc(128, MMA == 1);
      long long t0 = clock64();
      for (int it = 0; it < mma_iters; ++it)
        for (int kk = 0; kk < 8; ++kk) {
          if (MMA == 1)
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 384),
                "r"(tmem + kk * 8), "l"(db), "r"(id));
          else
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 384),
                "l"(da + (uint64_t)((kk * 32) >> 4)), "l"(db), "r"(id));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
          su32(&bar)));
      out[blockIdx.x * 64 + 63] = clock64() - t0;
    }
  } else {
    const uint32_t base = tmem + 128 + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
          "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(base + (uint32_t)((it & 1) * 64)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int e = 0; e < 32; ++e) acc ^= r[e];
    }
    const long long t = clock64() - t0;
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 64 + warp] = t;
    if (acc == 0x12345678u) out[0] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int MMA>
void run(int warps, int iters, int mma_iters) {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8 * 148);
  cudaMemset(d, 0, 64 * 8 * 148);
  cudaFuncSetAttribute(k<MMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<MMA><<<1, (warps + 1) * 32, 70000>>>(iters, mma_iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[64];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
  const double bytes = (double)warps * iters * 32 * 128;
  printf("MMA=%d warps=%2d: ldtm %.1f B/clk (%llu clk)  mma %llu clk (%d x 8 MMAs: %.1f clk/MMA) %s\n", MMA, warps,
         bytes / mx, mx, h[63], mma_iters, mma_iters ? (double)h[63] / (8.0 * mma_iters) : 0.0,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int w : {1, 4, 8, 16}) run<0>(w, 2000, 0);
  run<1>(8, 2000, 400);
  run<1>(4, 1, 400);
  run<2>(8, 2000, 400);
  run<2>(4, 1, 400);
  return 0;
}
