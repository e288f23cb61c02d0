// FP64 dependent-chain latency probe (one warp): cycles per dependent
// DADD / DMUL / DFMA / IEEE division / rsqrt seed, and an LDS round trip.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/lat_probe.cu -o expt/lat_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[64];
    sm[threadIdx.x] = a;
    __syncwarp();
    double x = a + threadIdx.x * 1e-300;
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (OP == 0) x = x + b;
            if (OP == 1) x = x * b;
            if (OP == 2) x = __fma_rn(x, b, a);
            if (OP == 3) x = a / x;
            if (OP == 4) asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(x) : "d"(x));
            if (OP == 5) x = sm[(__double2loint(x) & 1) + (int)(x == 12345.0)];
        }
    }
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 64 * sizeof(double));
    cudaMalloc(&c, sizeof(long long));
    const char* names[] = {"DADD", "DMUL", "DFMA", "DDIV(IEEE)", "MUFU.RSQ64", "LDS(dep)"};
    const int n = 4096;
    for (int op = 0; op < 6; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: chain<0><<<1, 32>>>(d, c, 1.0, 1e-17, n); break;
                case 1: chain<1><<<1, 32>>>(d, c, 1.0, 1.0000000001, n); break;
                case 2: chain<2><<<1, 32>>>(d, c, 0.5, 0.5, n); break;
                case 3: chain<3><<<1, 32>>>(d, c, 1.5, 1.0, n); break;
                case 4: chain<4><<<1, 32>>>(d, c, 1.5, 1.0, n); break;
                case 5: chain<5><<<1, 32>>>(d, c, 1.5, 1.0, n); break;
            }
            long long h;
            cudaMemcpy(&h, c, sizeof h, cudaMemcpyDeviceToHost);
            if (rep) printf("%-12s %6.2f cycles/op\n", names[op], (double)h / (16.0 * n));
        }
    }
    return 0;
}
