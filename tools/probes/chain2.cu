// DP step chain variants on one warp (cycles per step, and per column).
#include <cstdio>
__device__ __forceinline__ float mn2(float a, float b) { float r; asm("min.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__global__ void k(const float* __restrict__ cin, float* out, int steps, int mode, long long* cyc) {
  const int lane = threadIdx.x;
  float L[4] = {1e30f, 1e30f, 1e30f, 1e30f}, L2[4] = {1e30f, 1e30f, 1e30f, 1e30f};
  float bottom = 1e30f, bottom2 = 1e30f, prevtop = 0.f;
  float feedv = 0.5f + lane;
  long long t0 = clock64();
#pragma unroll 4
  for (int s = 0; s < steps; s++) {
    const float4 c = reinterpret_cast<const float4*>(cin)[(s & 63) * 32 + lane];
    if (mode <= 1) {
      const float feed = __shfl_sync(0xffffffffu, feedv, s & 31);
      float top = __shfl_sync(0xffffffffu, bottom, (lane + 31) & 31);
      top = lane == 0 ? feed : top;
      const float cc[4] = {c.x, c.y, c.z, c.w};
      float up = top, dg = prevtop;
      if (mode == 0) {
#pragma unroll
        for (int r = 0; r < 4; r++) { float m = fminf(fminf(L[r], dg), up); dg = L[r]; L[r] = __fadd_rn(m, cc[r]); up = L[r]; }
      } else {
        float t[4];
        t[0] = mn2(L[0], prevtop);
#pragma unroll
        for (int r = 1; r < 4; r++) t[r] = mn2(L[r], L[r - 1]);
#pragma unroll
        for (int r = 0; r < 4; r++) { float m = mn2(t[r], up); L[r] = __fadd_rn(m, cc[r]); up = L[r]; }
      }
      bottom = L[3]; prevtop = top;
    } else {
      // two columns per step, hoisted min(left, diag)
      const float4 c2 = reinterpret_cast<const float4*>(cin)[((s + 7) & 63) * 32 + lane];
      const float fa = __shfl_sync(0xffffffffu, feedv, s & 31);
      const float fb = __shfl_sync(0xffffffffu, feedv, (s + 1) & 31);
      float ta = __shfl_sync(0xffffffffu, bottom, (lane + 31) & 31);
      float tb = __shfl_sync(0xffffffffu, bottom2, (lane + 31) & 31);
      ta = lane == 0 ? fa : ta; tb = lane == 0 ? fb : tb;
      const float ca[4] = {c.x, c.y, c.z, c.w}, cb[4] = {c2.x, c2.y, c2.z, c2.w};
      float t[4];
      t[0] = mn2(L[0], prevtop);
#pragma unroll
      for (int r = 1; r < 4; r++) t[r] = mn2(L[r], L[r - 1]);
      float A[4];
      float up = ta;
#pragma unroll
      for (int r = 0; r < 4; r++) { A[r] = __fadd_rn(mn2(t[r], up), ca[r]); up = A[r]; }
      // column j+1: left = A[r], diag = A[r-1] (or ta for r=0), up from above
      up = tb;
      float dgb = ta;
#pragma unroll
      for (int r = 0; r < 4; r++) { float m = mn2(mn2(A[r], dgb), up); dgb = A[r]; L[r] = __fadd_rn(m, cb[r]); up = L[r]; }
      bottom = A[3]; bottom2 = L[3]; prevtop = tb;
    }
  }
  long long t1 = clock64();
  out[lane] = bottom + bottom2;
  if (lane == 0) cyc[mode] = t1 - t0;
}
int main() {
  float* c; cudaMalloc(&c, 64 * 32 * 16); cudaMemset(c, 0, 64 * 32 * 16);
  float* o; cudaMalloc(&o, 128); long long* cy; cudaMalloc(&cy, 64);
  const int steps = 100000;
  const char* nm[3] = {"FMNMX3 chain, 1 col", "hoisted 2-input min, 1 col", "hoisted, 2 cols/step"};
  for (int mode = 0; mode < 3; mode++) {
    k<<<1, 32>>>(c, o, steps, mode, cy); cudaDeviceSynchronize();
    long long h[3]; cudaMemcpy(h, cy, 24, cudaMemcpyDeviceToHost);
    double per = (double)h[mode] / steps;
    printf("mode %d (%s): %.1f cycles/step, %.1f cycles/column\n", mode, nm[mode], per, mode == 2 ? per / 2 : per);
  }
  return 0;
}
