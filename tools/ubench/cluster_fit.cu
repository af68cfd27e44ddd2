// Co-resident cluster count per cluster size and per-CTA shared memory
// (cudaOccupancyMaxActiveClusters), plus the SM ids the CTAs of one launch
// land on (two CTAs per SM or spread?).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* sm) {
  extern __shared__ char s[];
  unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  if (threadIdx.x == 0) { sm[blockIdx.x] = r; s[0] = 1; }
  __nanosleep(200000);
}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int kb[] = {60, 100, 110, 120, 200};
  for (int b : kb) {
    printf("smem %3d KB:", b);
    for (int cs = 1; cs <= 16; ++cs) {
      cudaLaunchConfig_t c{}; c.gridDim = dim3(cs * 8); c.blockDim = dim3(352); c.dynamicSmemBytes = b * 1024;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim = {(unsigned)cs, 1, 1};
      c.attrs = at; c.numAttrs = 1;
      int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &c);
      printf(" %d:%d", cs, e == cudaSuccess ? n : -1);
    }
    printf("\n");
  }
  // placement: 8 clusters of 14 at 110 KB
  int* d; cudaMalloc(&d, 4096 * 4);
  for (int b : {110, 200}) for (int cs : {14, 7}) {
    int nclu = cs == 14 ? 8 : 16;
    cudaLaunchConfig_t c{}; c.gridDim = dim3(cs * nclu); c.blockDim = dim3(352); c.dynamicSmemBytes = b * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim = {(unsigned)cs, 1, 1};
    c.attrs = at; c.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&c, k, d);
    cudaDeviceSynchronize();
    int h[4096]; cudaMemcpy(h, d, cs * nclu * 4, cudaMemcpyDeviceToHost);
    int cnt[256] = {0}; int distinct = 0, dbl = 0;
    for (int i = 0; i < cs * nclu; ++i) { if (cnt[h[i]]++ == 0) distinct++; else if (cnt[h[i]] == 2) dbl++; }
    printf("launch %d clusters of %d at %d KB: %s, distinct SMs %d, doubled %d\n", nclu, cs, b, cudaGetErrorString(e), distinct, dbl);
  }
  return 0;
}
