// Dependent-chain latency of F2F.F64.F32 + F2F.F32.F64 (float -> double ->
// float round trip) and of DADD, one thread.  Diagnostic micro-benchmark.
#include <cstdio>
__global__ void rt(float *out, float f, int n, long long *cyc) {
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) f = __double2float_rn((double)f);
    long long t1 = clock64();
    out[0] = f;
    cyc[0] = t1 - t0;
}
__global__ void rt_int(float *out, float f, int n, long long *cyc) {  // float -> int -> float (I2F/F2I)
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) f = (float)__float2int_rz(f);
    long long t1 = clock64();
    out[0] = f;
    cyc[0] = t1 - t0;
}
__global__ void dchain(double *out, double x, int n, long long *cyc) {
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, 1.0);
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}
int main() {
    float *o; double *od; long long *c, h;
    cudaMalloc(&o, 8); cudaMalloc(&od, 8); cudaMalloc(&c, 8);
    for (int rep = 0; rep < 2; ++rep) {
        rt<<<1, 1>>>(o, 1.5f, 4096, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("F2F.F64.F32 + F2F.F32.F64 round trip: %.1f cycles\n", h / 4096.0);
        rt_int<<<1, 1>>>(o, 1.5f, 4096, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("F2I + I2F round trip: %.1f cycles\n", h / 4096.0);
        dchain<<<1, 1>>>(od, 1.5, 4096, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("DADD: %.1f cycles\n", h / 4096.0);
    }
    return 0;
}
