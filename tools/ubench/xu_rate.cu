// Micro-benchmark: per-SM throughput of the softmax's instruction classes on
// sm_100a (MUFU.EX2, F2FP f32x2->f16x2 pack, an integer f32->f16 pack, FFMA2),
// with W warps per SM each running independent chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu_rate xu_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int iters, float seed, uint32_t* out, unsigned long long* cyc) {
  float x[8];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i + 1) * 1e-3f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // MUFU.EX2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      } else if (MODE == 1) {  // F2FP pack (x[i], x[i^1])
        uint32_t h;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        acc += h;
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (h & 1));
      } else if (MODE == 2) {  // integer pack: round-half-up to f16 bits of two normal floats
        const uint32_t b0 = __float_as_uint(x[i]) + 0x1000u - 0x38000000u;
        const uint32_t b1 = __float_as_uint(x[(i + 1) & 7]) + 0x1000u - 0x38000000u;
        const uint32_t h = __funnelshift_r(b0, b1 >> 13, 13) ;
        acc += h;
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (h & 1));
      } else {  // FFMA2
        float2 v = make_float2(x[i], x[(i + 1) & 7]);
        v = __ffma2_rn(v, make_float2(1.0001f, 0.9999f), make_float2(1e-7f, -1e-7f));
        x[i] = v.x;
        x[(i + 1) & 7] = v.y;
      }
    }
  }
  const unsigned long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(s) + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  unsigned long long* cyc;
  cudaMalloc(&out, sms * warps * 32 * 4);
  cudaMalloc(&cyc, sms * 8);
  const int iters = 4096;
  k<MODE><<<sms, warps * 32>>>(iters, 1.f, out, cyc);
  cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)iters * 8 * warps * 32;  // per SM (lane-ops; MODE 3 counts pairs)
  printf("%-12s warps/SM %2d: %8.2f lane-ops/clk/SM, %6.2f cycles per warp-instr per SMSP\n", name, warps,
         ops / c, (double)c / ((double)iters * 8 * warps / 4));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<0>("MUFU.EX2", w);
    run<1>("F2FP pack", w);
    run<2>("int pack", w);
    run<3>("FFMA2", w);
  }
  return 0;
}
