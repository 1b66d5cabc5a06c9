// Shared-memory float -> double widening of a 32 x 64 block by 64 threads
// (the fold kernel's widen step), cycles per block.  Diagnostic.
#include <cstdio>
template <int MODE>
__global__ void k(int reps, long long *cyc, double *sink) {
    __shared__ float xs[32 * 64];
    __shared__ double xw[32 * 64];
    const int t = threadIdx.x;
    for (int e = t; e < 2048; e += 64) xs[e] = e * 0.5f;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0) {
#pragma unroll 8
            for (int e = t; e < 2048; e += 64) xw[e] = (double)xs[e];
        } else {
            double v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = (double)xs[t + 64 * i];
#pragma unroll
            for (int i = 0; i < 32; ++i) xw[t + 64 * i] = v[i];
        }
        asm volatile("bar.sync 1, 64;");
    }
    long long t1 = clock64();
    if (t == 0) { cyc[0] = t1 - t0; sink[0] = xw[5]; }
}
int main() {
    long long *c, h; double *s;
    cudaMalloc(&c, 8); cudaMalloc(&s, 8);
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 64>>>(100, c, s); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("widen unroll8: %.0f cycles per block\n", h / 100.0);
        k<1><<<1, 64>>>(100, c, s); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("widen all-loads-first: %.0f cycles per block\n", h / 100.0);
    }
}
