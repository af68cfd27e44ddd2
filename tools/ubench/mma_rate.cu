// Micro-benchmark: tcgen05.mma issue/execute rate for the shapes K4 uses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (bmn ? (1u << 16) : 0u) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
}

template <int MODE, int RANDOM>  // 0: SS N=64, 1: SS N=128, 2: TS N=128, 3: SS N=256, 4: SS N=64 desc per mma
__global__ void k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2[6];
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    uint32_t x = (i * 2654435761u) ^ (blockIdx.x * 40503u);
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    ((uint32_t*)s)[i] = RANDOM ? (x & 0xbfffbfffu) : 0u;  // random bf16 pairs, |v| < 2
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int i = 0; i < 6; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2[i])));
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
  uint32_t tmem = slot;
  if (MODE == 8 && threadIdx.x >= 32) {  // spinning waiters on a barrier that completes at the end
    asm volatile("{\n.reg .pred P1;\nW2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W2;\n}\n" ::"r"(su32(&bar)));
  }
  if (threadIdx.x == 0) {
    const uint32_t a0 = su32(s), b0 = su32(s + 32768);
    const uint64_t da = desc(a0, 16, 1024), db = desc(b0, 16, 1024);
    constexpr int N = (MODE == 0 || MODE == 4) ? 64 : MODE == 3 ? 256 : 128;
    const uint32_t id = idesc(N, MODE == 2);
    long long t0 = clock64();
    if (MODE >= 5) {  // 8: mix+commits with 3 spinning warps
      const uint64_t dv = desc(b0, 8192, 1024);
      for (int it = 0; it < iters / 4; ++it) {
        for (int i = 0; i < 2; ++i) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem + i * 128 + (it & 1) * 64), "l"(da + ks * 2), "l"(db + ks * 2), "r"(idesc(64, false)), "r"(ks));
          if (MODE == 5 || MODE == 7 || MODE == 8) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[i])));
          if (MODE == 7) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (MODE == 5 || MODE == 8) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[2])));
        for (int i = 0; i < 2; ++i) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(tmem + 256 + i * 128), "r"(tmem + i * 128 + (it & 1) * 64 + ks * 4), "l"(dv + (ks & 3) * 128), "r"(idesc(128, true)), "r"(1));
          if (MODE == 5) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[3 + i])));
        }
        if (MODE == 5) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[5])));
      }
    }
    for (int it = 0; it < (MODE >= 5 ? 0 : iters); ++it) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (MODE == 2) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tmem + 256), "r"(tmem + ks * 8), "l"(db + ks * 2), "r"(id), "r"(ks));
        } else if (MODE == 4) {
          const uint32_t sa = su32(s) + (ks >> 2) * 16384 + (ks & 3) * 32 + (it & 1) * 64 * 0;
          const uint32_t sb = su32(s + 32768) + ((it & 3) * 16384) % 32768 + (ks >> 2) * 8192 + (ks & 3) * 32;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem + (it & 1) * 64), "l"(desc(sa, 16, 1024)), "l"(desc(sb, 16, 1024)), "r"(id), "r"(ks));
        } else {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(da + ks * 2), "l"(db + ks * 2), "r"(id), "r"(ks));
        }
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar)));
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int MODE, int RANDOM>
void run(const char* name) {
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<MODE, RANDOM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  const int iters = 2000;
  k<MODE, RANDOM><<<148, (MODE == 8 ? 320 : 128), 100000>>>(iters, d);
  k<MODE, RANDOM><<<148, (MODE == 8 ? 320 : 128), 100000>>>(iters, d);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("%-12s issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", name, (double)h[0] / (iters * 8),
         (double)h[1] / (iters * 8), cudaGetErrorString(e));
}

int main() {
  run<0, 0>("SS N=64");
  run<1, 0>("SS N=128");
  run<2, 0>("TS N=128");
  run<3, 0>("SS N=256");
  run<4, 0>("SS N=64 dyn");
  run<0, 1>("SS N=64 rnd");
  run<1, 1>("SS N=128 rnd");
  run<2, 1>("TS N=128 rnd");
  run<4, 1>("SS64 dyn rnd");
  run<5, 1>("mix+commits");
  run<6, 1>("mix nocommit");
  run<7, 1>("mix+fence");
  run<8, 1>("mix+spinners");
  return 0;
}
