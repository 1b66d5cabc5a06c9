// Throughput of float64 adds and float<->double / int->double conversions on
// one SM (1 CTA of 1024 threads, 8 independent chains per thread), cycles per
// warp instruction per SM.  Diagnostic micro-benchmark.
#include <cstdio>
#define N 1024
template <int OP>
__global__ void k(const float *fin, double *dout, float *fout, long long *cyc) {
    float f[8];
    double d[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { f[j] = fin[(threadIdx.x + j) & 31]; d[j] = (double)f[j]; }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) d[j] = __dadd_rn(d[j], 1.5);                     // DADD
            if (OP == 1) { d[j] = __dadd_rn(d[j], (double)f[j]); f[j] += 1.0f; }  // F2F.F64.F32 + DADD
            if (OP == 2) { f[j] = __double2float_rn(d[j]); d[j] = __dadd_rn(d[j], 0.25); }  // F2F.F32.F64 + DADD
            if (OP == 3) { d[j] = __dadd_rn(d[j], (double)(int)i); }  // I2F.F64 + DADD
            if (OP == 4) { f[j] = __fadd_rn(f[j], 1.5f); }  // FADD
        }
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0; float g = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { s += d[j]; g += f[j]; }
    dout[threadIdx.x] = s; fout[threadIdx.x] = g;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float *fi, *fo; double *d; long long *c, h;
    cudaMalloc(&fi, 128); cudaMalloc(&fo, 4096); cudaMalloc(&d, 8192); cudaMalloc(&c, 8);
    cudaMemset(fi, 0, 128);
    const char *names[] = {"DADD", "F2F.F64.F32+DADD", "F2F.F32.F64+DADD", "I2F.F64+DADD", "FADD"};
    for (int rep = 0; rep < 2; ++rep)
        for (int op = 0; op < 5; ++op) {
            if (op == 0) k<0><<<1, 1024>>>(fi, d, fo, c);
            if (op == 1) k<1><<<1, 1024>>>(fi, d, fo, c);
            if (op == 2) k<2><<<1, 1024>>>(fi, d, fo, c);
            if (op == 3) k<3><<<1, 1024>>>(fi, d, fo, c);
            if (op == 4) k<4><<<1, 1024>>>(fi, d, fo, c);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            // warp instructions of the op per SM: 32 warps * N * 8
            printf("%-20s %.3f cycles per warp-op per SM (%.1f ops/clk/SM)\n", names[op],
                   h / (32.0 * N * 8), 32.0 * 32 * N * 8 / h);
        }
    return 0;
}
