// Latency floor of the DP step chain on one warp.
#include <cstdio>
__global__ void k(const float* __restrict__ cin, float* out, int steps, int mode, long long* cyc) {
  const int lane = threadIdx.x;
  float left0 = 1e30f, left1 = 1e30f, left2 = 1e30f, left3 = 1e30f, bottom = 1e30f, prevtop = 0.f;
  float feedv = 0.5f + lane;
  long long t0 = clock64();
  for (int s = 0; s < steps; s++) {
    const float4 c = reinterpret_cast<const float4*>(cin)[(s & 63) * 32 + lane];
    float top;
    if (mode == 0) {       // shfl + sel
      const float feed = __shfl_sync(0xffffffffu, feedv, s & 31);
      top = __shfl_sync(0xffffffffu, bottom, (lane + 31) & 31);
      top = lane == 0 ? feed : top;
    } else if (mode == 1) { // shfl only
      top = __shfl_sync(0xffffffffu, bottom, (lane + 31) & 31);
    } else {                // no shuffle (chain within a lane)
      top = bottom;
    }
    float up = top, dg = prevtop, m;
    m = fminf(fminf(left0, dg), up); dg = left0; left0 = __fadd_rn(m, c.x); up = left0;
    m = fminf(fminf(left1, dg), up); dg = left1; left1 = __fadd_rn(m, c.y); up = left1;
    m = fminf(fminf(left2, dg), up); dg = left2; left2 = __fadd_rn(m, c.z); up = left2;
    m = fminf(fminf(left3, dg), up); dg = left3; left3 = __fadd_rn(m, c.w); up = left3;
    bottom = left3; prevtop = top;
  }
  long long t1 = clock64();
  out[lane] = bottom;
  if (lane == 0) cyc[mode] = t1 - t0;
}
int main() {
  float* c; cudaMalloc(&c, 64 * 32 * 16); cudaMemset(c, 0, 64 * 32 * 16);
  float* o; cudaMalloc(&o, 128); long long* cy; cudaMalloc(&cy, 64);
  const int steps = 100000;
  for (int mode = 0; mode < 3; mode++) {
    k<<<1, 32>>>(c, o, steps, mode, cy); cudaDeviceSynchronize();
    long long h[3]; cudaMemcpy(h, cy, 24, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.1f cycles/step\n", mode, mode == 0 ? "2 shfl + sel" : mode == 1 ? "1 shfl" : "no shfl", (double)h[mode] / steps);
  }
  return 0;
}
