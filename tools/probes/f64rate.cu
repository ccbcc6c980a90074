// fp64 DADD/DMUL issue rate on one GPU: 8 independent chains per thread.
#include <cstdio>
__global__ void k(double* out, int iters, double a) {
    double s[8];
    for (int i = 0; i < 8; i++) s[i] = threadIdx.x + i;
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) s[i] = __dmul_rn(__dsub_rn(s[i], a), a);
    double t = 0;
    for (int i = 0; i < 8; i++) t += s[i];
    if (t == 1.2345) out[0] = t;
}
int main() {
    double* o; cudaMalloc(&o, 8);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int th : {256, 512, 1024}) {
        const int iters = 4096;
        k<<<nsm, th>>>(o, iters, 0.999);
        cudaEventRecord(e0);
        k<<<nsm * 2, th>>>(o, iters, 0.999);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = 2.0 * nsm * 2 * th * iters * 8;
        printf("threads/CTA %d: %.2f Tops/s fp64 (%.1f lane-ops/clk/SM at 1.965 GHz)\n", th, ops / ms / 1e9,
               ops / (ms * 1e-3) / nsm / 1.965e9);
    }
}
