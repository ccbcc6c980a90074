// FP32 lane-op throughput per SMSP for mixes of packed FFMA2 and scalar FFMA
// (independent chains, 4 warps per SMSP): does fma-lite add capacity next to
// packed ops on fma-heavy?
#include <cstdio>
typedef unsigned long long u64;
template <int NP2, int NS>  // per iteration: NP2 packed, NS scalar instructions
__global__ void k(float* out, int iters, long long* cyc) {
  u64 p[8];
  float f[8];
#pragma unroll
  for (int q = 0; q < 8; q++) { p[q] = 0x3f8000003f800000ull + threadIdx.x + q; f[q] = 1.0f + threadIdx.x + q; }
  const u64 pm = 0x3f7fffff3f7fffffull; const float fm = 0.999999f;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int q = 0; q < NP2; q++) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[q & 7]) : "l"(pm));
#pragma unroll
    for (int q = 0; q < NS; q++) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[q & 7]) : "f"(fm));
  }
  long long t1 = clock64();
  float s = 0; for (int q = 0; q < 8; q++) s += f[q] + __uint_as_float((unsigned)p[q]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int NP2, int NS> void run(float* o, long long* c) {
  const int iters = 4000;
  k<NP2, NS><<<148, 512>>>(o, iters, c);  // 16 warps per SM = 4 per SMSP
  cudaDeviceSynchronize();
  k<NP2, NS><<<148, 512>>>(o, iters, c);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double laneops = 4.0 * iters * (64.0 * NP2 + 32.0 * NS);  // per SMSP (4 warps)
  printf("packed %d scalar %d per iter: %.2f lane-ops/clk/SMSP, %.2f instr/clk/SMSP\n", NP2, NS, laneops / h,
         4.0 * iters * (NP2 + NS) / h);
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 8);
  run<8, 0>(o, c); run<0, 8>(o, c); run<8, 4>(o, c); run<8, 8>(o, c); run<4, 8>(o, c); run<8, 2>(o, c);
  return 0;
}
