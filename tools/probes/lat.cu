// Latency probes: dependent FMNMX3->FADD chains (1, 2, 4 interleaved), SHFL round trip.
#include <cstdio>
__global__ void chains(float* out, long long* cyc, int n, float l, float l2) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  const float c = 0.5f;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) a0 = __fadd_rn(fminf(fminf(l, a1 * 0 + l), a0), c);
  }
  long long t1 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      a0 = __fadd_rn(fminf(fminf(l, l2), a0), c);
      a1 = __fadd_rn(fminf(fminf(l, l2), a1), c);
    }
  }
  long long t2 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      a0 = __fadd_rn(fminf(fminf(l, l2), a0), c);
      a1 = __fadd_rn(fminf(fminf(l, l2), a1), c);
      a2 = __fadd_rn(fminf(fminf(l, l2), a2), c);
      a3 = __fadd_rn(fminf(fminf(l, l2), a3), c);
    }
  }
  long long t3 = clock64();
  float s = a0;
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) s = __shfl_sync(0xffffffffu, s, (threadIdx.x + 31) & 31);
  }
  long long t4 = clock64();
  float q = a0;
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) { q = __shfl_sync(0xffffffffu, q, (threadIdx.x + 31) & 31); q = threadIdx.x == 0 ? c : q; q = __fadd_rn(fminf(q, l), c); }
  }
  long long t5 = clock64();
  out[threadIdx.x] = a0 + a1 + a2 + a3 + s + q;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  const int n = 10000;
  chains<<<1, 32>>>(o, c, n, 1e30f, 2e30f); cudaDeviceSynchronize();
  chains<<<1, 32>>>(o, c, n, 1e30f, 2e30f); cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  const double k = 8.0 * n;
  printf("1 chain  FMNMX3->FADD: %.2f cyc/link\n", h[0] / k);
  printf("2 chains FMNMX3->FADD: %.2f cyc/link-pair\n", h[1] / k);
  printf("4 chains FMNMX3->FADD: %.2f cyc/link-quad\n", h[2] / k);
  printf("SHFL dependent chain : %.2f cyc/shfl\n", h[3] / k);
  printf("SHFL->SEL->FMNMX->FADD chain: %.2f cyc\n", h[4] / k);
  return 0;
}
