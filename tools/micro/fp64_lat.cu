// Dependent-chain latency of FP64 / FP32 / conversion instructions on one warp (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, float* outf, long long* t, double a, float af) {
    double x = a, y = 1.0000001;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) x = fma(x, y, a);
    long long t1 = clock64();
    double z = a;
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) z = z + y;
    long long t2 = clock64();
    float f = af, g = 1.0000001f;
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) f = fmaf(f, g, af);
    long long t3 = clock64();
    double c = a;
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) c = (double)(float)c + a;   // F2F x2 + DADD
    long long t4 = clock64();
    int p = 0;
    double w = a;
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) { if (w > 0.5) p++; w = w * y; }  // DSETP + DMUL
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        out[0] = x + z + c + w + p; outf[0] = f;
        t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4;
    }
}
int main() {
    double* o; float* of; long long* t;
    cudaMalloc(&o, 8); cudaMalloc(&of, 4); cudaMalloc(&t, 64);
    for (int threads : {32, 128, 512}) {
        k<<<1, threads>>>(o, of, t, 0.3, 0.3f);
        long long h[5];
        cudaMemcpy(h, t, 40, cudaMemcpyDeviceToHost);
        printf("threads %d: DFMA %.1f  DADD %.1f  FFMA %.1f  F2F+F2F+DADD %.1f  DSETP/DMUL loop %.1f cycles per iteration\n",
               threads, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0);
    }
    return 0;
}
