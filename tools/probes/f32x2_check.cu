// Checks packed f32x2 PTX ops against scalar _rn intrinsics, bit for bit,
// and measures their issue throughput.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void upk2(u64 v, float& lo, float& hi) { asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ u64 sub2b(u64 a, float y) { u64 yy = pk2(y, y), r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(yy)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }

__global__ void check(const float* a, const float* b, const float* y, const float* s, int n, int* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u64 A = pk2(a[i], b[i]);
  u64 D = sub2b(A, y[i]);
  u64 Q = mul2(D, D);
  u64 S = add2(pk2(s[i], s[(i + 1) % n]), Q);
  float d0, d1, q0, q1, s0, s1;
  upk2(D, d0, d1); upk2(Q, q0, q1); upk2(S, s0, s1);
  float e0 = __fsub_rn(a[i], y[i]), e1 = __fsub_rn(b[i], y[i]);
  float f0 = __fmul_rn(e0, e0), f1 = __fmul_rn(e1, e1);
  float g0 = __fadd_rn(s[i], f0), g1 = __fadd_rn(s[(i + 1) % n], f1);
  if (__float_as_uint(d0) != __float_as_uint(e0) || __float_as_uint(d1) != __float_as_uint(e1)) atomicAdd(bad, 1);
  if (__float_as_uint(q0) != __float_as_uint(f0) || __float_as_uint(q1) != __float_as_uint(f1)) atomicAdd(bad + 1, 1);
  if (__float_as_uint(s0) != __float_as_uint(g0) || __float_as_uint(s1) != __float_as_uint(g1)) atomicAdd(bad + 2, 1);
}

template <int MODE>
__global__ void tput(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  u64 p0 = pk2(a0, a1), p1 = pk2(a2, a3), p2 = pk2(a4, a5), p3 = pk2(a6, a7), p4 = pk2(a1, a0), p5 = pk2(a3, a2), p6 = pk2(a5, a4), p7 = pk2(a7, a6);
  const u64 k = pk2(1.0000001f, 0.9999999f);
  for (int it = 0; it < iters; it++) {
    if (MODE == 0) {  // scalar FADD chains, 8 independent
      a0 = __fadd_rn(a0, 1e-7f); a1 = __fadd_rn(a1, 1e-7f); a2 = __fadd_rn(a2, 1e-7f); a3 = __fadd_rn(a3, 1e-7f);
      a4 = __fadd_rn(a4, 1e-7f); a5 = __fadd_rn(a5, 1e-7f); a6 = __fadd_rn(a6, 1e-7f); a7 = __fadd_rn(a7, 1e-7f);
    } else if (MODE == 1) {  // FADD2, 8 independent
      p0 = add2(p0, k); p1 = add2(p1, k); p2 = add2(p2, k); p3 = add2(p3, k);
      p4 = add2(p4, k); p5 = add2(p5, k); p6 = add2(p6, k); p7 = add2(p7, k);
    } else if (MODE == 2) {  // FMUL2
      p0 = mul2(p0, k); p1 = mul2(p1, k); p2 = mul2(p2, k); p3 = mul2(p3, k);
      p4 = mul2(p4, k); p5 = mul2(p5, k); p6 = mul2(p6, k); p7 = mul2(p7, k);
    } else {  // scalar FMUL
      a0 = __fmul_rn(a0, 1.0000001f); a1 = __fmul_rn(a1, 1.0000001f); a2 = __fmul_rn(a2, 1.0000001f); a3 = __fmul_rn(a3, 1.0000001f);
      a4 = __fmul_rn(a4, 1.0000001f); a5 = __fmul_rn(a5, 1.0000001f); a6 = __fmul_rn(a6, 1.0000001f); a7 = __fmul_rn(a7, 1.0000001f);
    }
  }
  float r0, r1;
  upk2(p0 ^ p1 ^ p2 ^ p3 ^ p4 ^ p5 ^ p6 ^ p7, r0, r1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + r0 + r1;
}

int main() {
  const int n = 1 << 22;
  float *h = (float*)malloc(4 * n * sizeof(float));
  unsigned s = 12345;
  for (int i = 0; i < 4 * n; i++) {
    s = s * 1664525u + 1013904223u;
    unsigned bits = s;
    if (i % 7 == 0) bits &= 0x807fffff;  // some denormals
    float f; memcpy(&f, &bits, 4);
    if (!(f == f) || f > 1e30f || f < -1e30f) f = 1.5f;
    h[i] = f;
  }
  float* d; cudaMalloc(&d, 4 * n * sizeof(float));
  cudaMemcpy(d, h, 4 * n * sizeof(float), cudaMemcpyHostToDevice);
  int* bad; cudaMalloc(&bad, 3 * sizeof(int)); cudaMemset(bad, 0, 3 * sizeof(int));
  check<<<n / 256, 256>>>(d, d + n, d + 2 * n, d + 3 * n, n, bad);
  int hb[3]; cudaMemcpy(hb, bad, sizeof hb, cudaMemcpyDeviceToHost);
  printf("f32x2 mismatches vs scalar _rn: sub %d mul %d add %d (of %d)\n", hb[0], hb[1], hb[2], n);
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[4] = {"FADD x8", "FADD2 x8", "FMUL2 x8", "FMUL x8"};
  for (int mode = 0; mode < 4; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      const int iters = 4096, grid = 148 * 8, block = 256;
      cudaEventRecord(e0);
      if (mode == 0) tput<0><<<grid, block>>>(out, iters);
      if (mode == 1) tput<1><<<grid, block>>>(out, iters);
      if (mode == 2) tput<2><<<grid, block>>>(out, iters);
      if (mode == 3) tput<3><<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double instr = (double)grid * block / 32 * iters * 8;  // warp instructions
      double lanes = instr * 32 * (mode == 1 || mode == 2 ? 2 : 1);
      if (rep) printf("%-9s %.3f ms  %.1f warp-instr/clk/SM  %.1f fp32 lane-ops/clk/SM (at 1.965 GHz)\n", names[mode], ms,
                      instr / (ms * 1e-3) / 1.965e9 / 148, lanes / (ms * 1e-3) / 1.965e9 / 148);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
