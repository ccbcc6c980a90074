// DP-warp step microbenchmark: cycles per step of the min-plus systolic chain
// for lane skews 1 and 2 (shuffle on / off the critical path) and R rows per
// lane, alone and next to FFMA2-streaming "cost" warps on the same SMSPs.
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ float mn(float a, float b) { return fminf(a, b); }

template <int R, int SKEW>
__device__ void dp(const float* __restrict__ cin, float* out, int steps, long long* cyc) {
  const int lane = threadIdx.x & 31;
  float L[R];
#pragma unroll
  for (int r = 0; r < R; r++) L[r] = 1e30f;
  float bottom = 1e30f, prevtop = 0.f, topn = 1e30f, topo = 1e30f;
  const float feedv = 0.5f + lane;
  long long t0 = clock64();
  float cn[R];
#pragma unroll
  for (int q = 0; q < R / 4; q++) {
    const float4 c = reinterpret_cast<const float4*>(cin)[(lane) * (R / 4) + q];
    cn[4 * q] = c.x; cn[4 * q + 1] = c.y; cn[4 * q + 2] = c.z; cn[4 * q + 3] = c.w;
  }
#pragma unroll 4
  for (int s = 0; s < steps; s++) {
    float cc[R];
#pragma unroll
    for (int r = 0; r < R; r++) cc[r] = cn[r];
    // prefetch the next step's costs (register double buffer)
#pragma unroll
    for (int q = 0; q < R / 4; q++) {
      const float4 c = reinterpret_cast<const float4*>(cin)[(((s + 1) & 63) * 32 + lane) * (R / 4) + q];
      cn[4 * q] = c.x; cn[4 * q + 1] = c.y; cn[4 * q + 2] = c.z; cn[4 * q + 3] = c.w;
    }
    const float feed = __shfl_sync(0xffffffffu, feedv, s & 31);
    float top;
    if (SKEW == 1) {
      top = __shfl_sync(0xffffffffu, bottom, (lane + 31) & 31);
    } else {
      top = topo;  // shuffled two steps ago (end of step s-2)
    }
    top = lane == 0 ? feed : top;
    float up = top, dg = prevtop;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const float m = mn(mn(L[r], dg), up);
      dg = L[r];
      L[r] = __fadd_rn(m, cc[r]);
      up = L[r];
    }
    if (SKEW == 2) {
      topo = topn;
      topn = __shfl_sync(0xffffffffu, L[R - 1], (lane + 31) & 31);
    }
    bottom = L[R - 1];
    prevtop = top;
  }
  long long t1 = clock64();
  out[threadIdx.x] = bottom;
  if (lane == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}

__device__ void burn(float* out, int iters) {
  u64 a[8];
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = (u64)threadIdx.x * 0x3f8000003f800000ull + k;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < 8; k++) asm volatile("fma.rn.f32x2 %0, %0, %0, %1;" : "+l"(a[k]) : "l"(a[(k + 1) & 7]));
  }
  u64 s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s ^= a[k];
  out[threadIdx.x] = (float)s;
}

template <int R, int SKEW>
__global__ void k(const float* cin, float* out, int steps, long long* cyc, int burners) {
  const int w = threadIdx.x >> 5;
  // DP warps are the top 4 warp slots (one per SMSP); burners below
  if (w >= burners) dp<R, SKEW>(cin, out, steps, cyc);
  else burn(out, steps * R / 2);
}


// Two 4-row chains per lane (virtual lanes v = l and 32 + l, skew 2): chain B's
// lane 0 takes chain A's lane-31 bottom from the same rotated shuffle.
__device__ void dp2(const float* __restrict__ cin, float* out, int steps, long long* cyc) {
  const int lane = threadIdx.x & 31;
  float La[4], Lb[4];
#pragma unroll
  for (int r = 0; r < 4; r++) { La[r] = 1e30f; Lb[r] = 1e30f; }
  float pa = 0.f, pb = 0.f, tna = 1e30f, toa = 1e30f, tnb = 1e30f, tob = 1e30f;
  const float feedv = 0.5f + lane;
  float4 na = reinterpret_cast<const float4*>(cin)[lane * 2], nb = reinterpret_cast<const float4*>(cin)[lane * 2 + 1];
  long long t0 = clock64();
#pragma unroll 4
  for (int s = 0; s < steps; s++) {
    const float4 ca = na, cb = nb;
    na = reinterpret_cast<const float4*>(cin)[(((s + 1) & 63) * 32 + lane) * 2];
    nb = reinterpret_cast<const float4*>(cin)[(((s + 1) & 63) * 32 + lane) * 2 + 1];
    const float feed = __shfl_sync(0xffffffffu, feedv, s & 31);
    const float ta = lane == 0 ? feed : toa;
    const float tb = lane == 0 ? toa : tob;  // lane 0 of B: lane 31 of A (rotated shuffle)
    const float cca[4] = {ca.x, ca.y, ca.z, ca.w}, ccb[4] = {cb.x, cb.y, cb.z, cb.w};
    float ua = ta, da = pa, ub = tb, db = pb;
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const float ma = mn(mn(La[r], da), ua);
      const float mb = mn(mn(Lb[r], db), ub);
      da = La[r]; db = Lb[r];
      La[r] = __fadd_rn(ma, cca[r]); Lb[r] = __fadd_rn(mb, ccb[r]);
      ua = La[r]; ub = Lb[r];
    }
    toa = tna; tob = tnb;
    tna = __shfl_sync(0xffffffffu, La[3], (lane + 31) & 31);
    tnb = __shfl_sync(0xffffffffu, Lb[3], (lane + 31) & 31);
    pa = ta; pb = tb;
  }
  long long t1 = clock64();
  out[threadIdx.x] = La[3] + Lb[3];
  if (lane == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}
__global__ void k2(const float* cin, float* out, int steps, long long* cyc, int burners) {
  const int w = threadIdx.x >> 5;
  if (w >= burners) dp2(cin, out, steps, cyc);
  else burn(out, steps * 4);
}


// Two R-row chains per lane, skew SK (virtual lanes l and 32+l), costs prefetched.
template <int R, int SK>
__device__ void dpc(const float* __restrict__ cin, float* out, int steps, long long* cyc) {
  const int lane = threadIdx.x & 31;
  float La[R], Lb[R], na[R], nb[R];
#pragma unroll
  for (int r = 0; r < R; r++) { La[r] = 1e30f; Lb[r] = 1e30f; na[r] = 0.f; nb[r] = 0.f; }
  float pa = 0.f, pb = 0.f, tna = 1e30f, toa = 1e30f, tnb = 1e30f, tob = 1e30f;
  const float feedv = 0.5f + lane;
  long long t0 = clock64();
#pragma unroll 4
  for (int s = 0; s < steps; s++) {
    float ca[R], cb[R];
#pragma unroll
    for (int r = 0; r < R; r++) { ca[r] = na[r]; cb[r] = nb[r]; }
    const float* p = cin + (((s + 1) & 63) * 32 + lane) * 2 * R;
    if (R == 2) { float4 v = *reinterpret_cast<const float4*>(p); na[0] = v.x; na[1] = v.y; nb[0] = v.z; nb[1] = v.w; }
    else {
#pragma unroll
      for (int r = 0; r < R; r++) { na[r] = p[r]; nb[r] = p[R + r]; }
    }
    const float feed = __shfl_sync(0xffffffffu, feedv, s & 31);
    const float sa = SK == 1 ? tna : toa, sb = SK == 1 ? tnb : tob;
    const float ta = lane == 0 ? feed : sa;
    const float tb = lane == 0 ? sa : sb;
    float ua = ta, da = pa, ub = tb, db = pb;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const float ma = mn(mn(La[r], da), ua);
      const float mb = mn(mn(Lb[r], db), ub);
      da = La[r]; db = Lb[r];
      La[r] = __fadd_rn(ma, ca[r]); Lb[r] = __fadd_rn(mb, cb[r]);
      ua = La[r]; ub = Lb[r];
    }
    toa = tna; tob = tnb;
    tna = __shfl_sync(0xffffffffu, La[R - 1], (lane + 31) & 31);
    tnb = __shfl_sync(0xffffffffu, Lb[R - 1], (lane + 31) & 31);
    pa = ta; pb = tb;
  }
  long long t1 = clock64();
  out[threadIdx.x] = La[R - 1] + Lb[R - 1];
  if (lane == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}
template <int R, int SK>
__global__ void kc(const float* cin, float* out, int steps, long long* cyc, int burners) {
  const int w = threadIdx.x >> 5;
  if (w >= burners) dpc<R, SK>(cin, out, steps, cyc);
  else burn(out, steps * R);
}
template <int R, int SK> void runc(const float* c, float* o, long long* cy, int b) {
    const int steps = 20000;
    kc<R, SK><<<1, 32 * (b + 4)>>>(c, o, steps, cy, b);
    cudaDeviceSynchronize();
    long long h[32];
    cudaMemcpy(h, cy, sizeof(h), cudaMemcpyDeviceToHost);
    printf("2 chains x R=%d skew=%d burners/SMSP=%d: %.1f cyc/step  %.3f cells/cyc/warp\n", R, SK, b / 4, (double)h[b] / steps, 64.0 * R * steps / h[b]);
}

template <int R, int SKEW> void run(const float* c, float* o, long long* cy, int burners) {
  const int steps = 20000;
  k<R, SKEW><<<1, 32 * (burners + 4)>>>(c, o, steps, cy, burners);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cy, sizeof(h), cudaMemcpyDeviceToHost);
  const double per = (double)h[burners] / steps;
  printf("R=%d skew=%d burners/SMSP=%d: %.1f cyc/step  %.3f cells/cyc/warp\n", R, SKEW, burners / 4, per,
         32.0 * R / per);
}

// "Split" step: the lane's top-independent part X_r (its rows' values if the
// row above contributed +inf) is computed from the previous step's values
// while the shuffle is in flight; the chain from the arriving top is only
// t_r = (((top + c0) + c1) ...) and D_r = min(X_r, t_r) -- exact because
// rounding is monotone: fl(min(a, b) + c) = min(fl(a + c), fl(b + c)).
template <int R>
__device__ void dps(const float* __restrict__ cin, float* out, int steps, long long* cyc) {
  const int lane = threadIdx.x & 31;
  float L[R];
#pragma unroll
  for (int r = 0; r < R; r++) L[r] = 1e30f;
  float bottom = 1e30f, prevtop = 0.f;
  const float feedv = 0.5f + lane;
  float cn[R];
#pragma unroll
  for (int q = 0; q < R / 4; q++) {
    const float4 c = reinterpret_cast<const float4*>(cin)[(lane) * (R / 4) + q];
    cn[4 * q] = c.x; cn[4 * q + 1] = c.y; cn[4 * q + 2] = c.z; cn[4 * q + 3] = c.w;
  }
  long long t0 = clock64();
#pragma unroll 4
  for (int s = 0; s < steps; s++) {
    float cc[R];
#pragma unroll
    for (int r = 0; r < R; r++) cc[r] = cn[r];
#pragma unroll
    for (int q = 0; q < R / 4; q++) {
      const float4 c = reinterpret_cast<const float4*>(cin)[(((s + 1) & 63) * 32 + lane) * (R / 4) + q];
      cn[4 * q] = c.x; cn[4 * q + 1] = c.y; cn[4 * q + 2] = c.z; cn[4 * q + 3] = c.w;
    }
    const float feed = __shfl_sync(0xffffffffu, feedv, s & 31);
    float top = __shfl_sync(0xffffffffu, bottom, (lane + 31) & 31);
    // off the cross-lane chain
    float X[R];
    float dg = prevtop;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const float a = __fadd_rn(mn(L[r], dg), cc[r]);
      X[r] = r == 0 ? a : mn(a, __fadd_rn(X[r - 1], cc[r]));
      dg = L[r];
    }
    top = lane == 0 ? feed : top;
    float t = top;
#pragma unroll
    for (int r = 0; r < R; r++) {
      t = __fadd_rn(t, cc[r]);
      L[r] = mn(X[r], t);
    }
    bottom = L[R - 1];
    prevtop = top;
  }
  long long t1 = clock64();
  out[threadIdx.x] = bottom;
  if (lane == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}
template <int R>
__global__ void ks(const float* cin, float* out, int steps, long long* cyc, int burners) {
  const int w = threadIdx.x >> 5;
  if (w >= burners) dps<R>(cin, out, steps, cyc);
  else burn(out, steps * R / 2);
}
template <int R> void runs(const float* c, float* o, long long* cy, int burners) {
  const int steps = 20000;
  ks<R><<<1, 32 * (burners + 4)>>>(c, o, steps, cy, burners);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cy, sizeof(h), cudaMemcpyDeviceToHost);
  const double per = (double)h[burners] / steps;
  printf("SPLIT R=%d burners/SMSP=%d: %.1f cyc/step  %.3f cells/cyc/warp\n", R, burners / 4, per, 32.0 * R / per);
}
int main() {
  float* c; cudaMalloc(&c, 64 * 32 * 8 * 4); cudaMemset(c, 0, 64 * 32 * 8 * 4);
  float* o; cudaMalloc(&o, 4096); long long* cy; cudaMalloc(&cy, 256);
  for (int b : {0, 4, 8, 12}) {
    run<4, 1>(c, o, cy, b); run<4, 2>(c, o, cy, b);
    run<8, 1>(c, o, cy, b); run<8, 2>(c, o, cy, b);
    runs<4>(c, o, cy, b); runs<8>(c, o, cy, b);
    runc<2, 1>(c, o, cy, b); runc<2, 2>(c, o, cy, b); runc<4, 1>(c, o, cy, b); runc<4, 2>(c, o, cy, b);
    const int steps = 20000;
    k2<<<1, 32 * (b + 4)>>>(c, o, steps, cy, b);
    cudaDeviceSynchronize();
    long long h[32];
    cudaMemcpy(h, cy, sizeof(h), cudaMemcpyDeviceToHost);
    printf("2 chains x R=4 skew=2 burners/SMSP=%d: %.1f cyc/step  %.3f cells/cyc/warp\n", b / 4, (double)h[b] / steps, 256.0 * steps / h[b]);
  }
  return 0;
}
