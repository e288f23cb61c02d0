// FP64 pipe cost versus active lanes: does a DADD/DFMA warp instruction with
// only `act` lanes enabled occupy the FP64 pipe for fewer cycles?
// W warps per SMSP run ILP independent dependent chains each; the figure is
// SMSP cycles per warp-instruction (pipe-bound when W * ILP covers latency).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mask_probe.cu -o expt/mask_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void probe(double* out, long long* cyc, double b, int n, int act) {
    const int lane = threadIdx.x & 31;
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = 1.0 + j + threadIdx.x * 1e-9;
    __syncthreads();
    const long long t0 = clock64();
    if (lane < act) {
#pragma unroll 1
        for (int i = 0; i < n; ++i) {
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int j = 0; j < ILP; ++j) x[j] = x[j] + b;
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 148 * 1024 * sizeof(double));
    cudaMalloc(&c, sizeof(long long));
    const int n = 2048;
    const int acts[] = {32, 17, 16, 8, 1};
    for (int wps = 1; wps <= 4; wps *= 2) {      // warps per SMSP
        for (int a = 0; a < 5; ++a) {
            long long h = 0;
            for (int rep = 0; rep < 2; ++rep) {
                probe<4><<<148, 128 * wps>>>(d, c, 1e-17, n, acts[a]);
                cudaMemcpy(&h, c, sizeof h, cudaMemcpyDeviceToHost);
            }
            const double instr = (double)n * 8 * 4 * wps;  // warp-instructions per SMSP
            printf("warps/SMSP %d  ILP 4  active lanes %2d : %6.3f SMSP cycles per FP64 warp-instruction\n", wps,
                   acts[a], (double)h / instr);
        }
    }
    return 0;
}
