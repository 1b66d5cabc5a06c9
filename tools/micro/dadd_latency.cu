// Dependent float64 add chain latency (cycles per DADD), one thread.
#include <cstdio>
__global__ void chain(double *out, double x, int n, long long *cyc) {
    double c = x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) c = __dadd_rn(c, x);
    long long t1 = clock64();
    out[0] = c;
    cyc[0] = t1 - t0;
}
__global__ void chain_f2f(const float *in, double *out, int n, long long *cyc) {
    double c = 0.0;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) c = __dadd_rn(c, (double)in[i & 31]);
    long long t1 = clock64();
    out[0] = c;
    cyc[0] = t1 - t0;
}
int main() {
    double *o; long long *c; float *f;
    cudaMalloc(&o, 8); cudaMalloc(&c, 8); cudaMalloc(&f, 128); cudaMemset(f, 0, 128);
    long long h;
    for (int rep = 0; rep < 2; ++rep) {
        chain<<<1, 1>>>(o, 1.5, 4096, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("dadd chain: %.2f cycles/add\n", h / 4096.0);
        chain_f2f<<<1, 1>>>(f, o, 4096, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("dadd(+ld+f2f) chain: %.2f cycles/add\n", h / 4096.0);
    }
    return 0;
}
