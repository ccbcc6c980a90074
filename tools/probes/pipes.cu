// Issue/pipe throughput of the instruction forms the exact cost computation can
// use (independent chains, W warps per SMSP), in warp-instructions per clock
// per SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes tools/probes/pipes.cu
#include <cstdio>
typedef unsigned long long u64;

#define BODY_P2(ASM)                                                              \
    _Pragma("unroll") for (int q = 0; q < 8; q++) asm volatile(ASM : "+l"(p[q]) : "l"(pm), "l"(p[(q + 1) & 7]));
#define BODY_F(ASM)                                                               \
    _Pragma("unroll") for (int q = 0; q < 8; q++) asm volatile(ASM : "+f"(f[q]) : "f"(fm), "f"(f[(q + 1) & 7]));

template <int V>
__global__ void k(float* out, int iters, long long* cyc, const u64* pmv, const float* fmv) {
    const u64 pm = pmv[threadIdx.x];
    const float fm = fmv[threadIdx.x];
    u64 p[8];
    float f[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
        p[q] = 0x3f8000003f800000ull + threadIdx.x + q;
        f[q] = 1.0f + threadIdx.x + q;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        if (V == 0) { BODY_P2("fma.rn.f32x2 %0, %0, %1, %2;") }           // FFMA2 3 regs
        if (V == 1) { _Pragma("unroll") for (int q = 0; q < 8; q++) asm volatile("fma.rn.f32x2 %0, %0, %0, %1;" : "+l"(p[q]) : "l"(0ull)); }  // FFMA2 a*a + 0
        if (V == 2) { BODY_P2("add.rn.f32x2 %0, %0, %1;") }               // FADD2
        if (V == 3) { BODY_P2("mul.rn.f32x2 %0, %0, %1;") }               // FMUL2
        if (V == 4) { BODY_F("fma.rn.f32 %0, %0, %1, %2;") }              // FFMA
        if (V == 5) { BODY_F("add.rn.f32 %0, %0, %1;") }                  // FADD
        if (V == 6) { BODY_F("mul.rn.f32 %0, %0, %1;") }                  // FMUL
        if (V == 7) { BODY_F("min.f32 %0, %0, %1;") }                     // FMNMX
        if (V == 8) { BODY_F("rsqrt.approx.ftz.f32 %0, %0;") }            // MUFU.RSQ
        if (V == 9) {  // the cost pattern: sub2, square, add2 (3 instr per 2 cells per dim)
#pragma unroll
            for (int q = 0; q < 4; q++) {
                u64 d;
                asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(p[q]), "l"(pm));
                asm volatile("fma.rn.f32x2 %0, %0, %0, %1;" : "+l"(d) : "l"(0ull));
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[q + 4]) : "l"(d));
            }
        }
        if (V == 10) { BODY_P2("sub.rn.f32x2 %0, %0, %1;") }              // FADD2 (sub)
        if (V == 11) { BODY_F("fma.rn.f32 %0, %0, %0, 0f00000000;") }    // FFMA a*a + 0 scalar
    }
    long long t1 = clock64();
    float s = 0;
    for (int q = 0; q < 8; q++) s += f[q] + __uint_as_float((unsigned)p[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

static u64* g_pm;
static float* g_fm;
template <int V>
void run(const char* name, float* o, long long* c, int wps) {
    const int iters = 4000;
    k<V><<<148, 128 * wps>>>(o, iters, c, g_pm, g_fm);
    cudaDeviceSynchronize();
    k<V><<<148, 128 * wps>>>(o, iters, c, g_pm, g_fm);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const int per_iter = (V == 9) ? 12 : 8;
    printf("%-34s warps/SMSP %2d: %.3f warp-instr/clk/SMSP\n", name, wps, (double)wps * iters * per_iter / h);
}

int main() {
    float* o;
    long long* c;
    cudaMalloc(&o, 148 * 2048 * 4);
    cudaMalloc(&c, 8);
    {
        u64 hp[1024];
        float hf[1024];
        for (int q = 0; q < 1024; q++) { hp[q] = 0x3f7fffff3f7fffffull; hf[q] = 0.999999f; }
        cudaMalloc(&g_pm, sizeof hp);
        cudaMalloc(&g_fm, sizeof hf);
        cudaMemcpy(g_pm, hp, sizeof hp, cudaMemcpyHostToDevice);
        cudaMemcpy(g_fm, hf, sizeof hf, cudaMemcpyHostToDevice);
    }
    for (int w : {1, 2, 4, 8}) {
        run<0>("FFMA2 a*b+c", o, c, w);
        run<1>("FFMA2 a*a+0", o, c, w);
        run<2>("FADD2", o, c, w);
        run<10>("FADD2 (sub)", o, c, w);
        run<3>("FMUL2", o, c, w);
        run<4>("FFMA a*b+c", o, c, w);
        run<11>("FFMA a*a+0", o, c, w);
        run<5>("FADD", o, c, w);
        run<6>("FMUL", o, c, w);
        run<7>("FMNMX", o, c, w);
        run<8>("MUFU.RSQ", o, c, w);
        run<9>("cost pattern sub2,sq2,add2", o, c, w);
    }
    return 0;
}
