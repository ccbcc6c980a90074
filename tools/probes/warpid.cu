#include <cstdio>
__global__ void k(int* out) {
  unsigned w, sm; asm volatile("mov.u32 %0, %%warpid;" : "=r"(w)); asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if ((threadIdx.x & 31) == 0) { int i = blockIdx.x * 4 + threadIdx.x / 32; out[3*i] = sm; out[3*i+1] = w; out[3*i+2] = threadIdx.x/32; }
  // keep blocks resident together
  long long t0 = clock64(); while (clock64() - t0 < 2000000) {}
}
int main() {
  int nb = 148 * 3; int* d; cudaMalloc(&d, nb * 4 * 3 * sizeof(int));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<<<nb, 128, 70000>>>(d); cudaDeviceSynchronize();
  int* h = new int[nb * 12]; cudaMemcpy(h, d, nb * 12 * sizeof(int), cudaMemcpyDeviceToHost);
  for (int i = 0; i < nb * 4; i++) if (h[3*i] == 0 || h[3*i] == 1) printf("sm %d warpid %d (warp %d of block %d) -> smsp %d\n", h[3*i], h[3*i+1], h[3*i+2], i/4, h[3*i+1] % 4);
  return 0;
}
