// Dependent-chain latency of DADD (and FADD for reference) on one thread: clock64 per op.
#include <cstdio>
__global__ void k(double *out, float *outf, long long *cyc, int n, double x, float xf)
{
    double a = x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; i++) a = a + x;
    long long t1 = clock64();
    float b = xf;
#pragma unroll 16
    for (int i = 0; i < n; i++) b = b + xf;
    long long t2 = clock64();
    out[0] = a;
    outf[0] = b;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
}
int main()
{
    double *o; float *of; long long *c, h[2];
    cudaMalloc(&o, 8); cudaMalloc(&of, 4); cudaMalloc(&c, 16);
    const int n = 1 << 20;
    k<<<1, 1>>>(o, of, c, n, 1e-300, 1e-30f);
    k<<<1, 1>>>(o, of, c, n, 1e-300, 1e-30f);
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency %.2f cycles, FADD %.2f cycles\n", (double)h[0] / n, (double)h[1] / n);
    return 0;
}
