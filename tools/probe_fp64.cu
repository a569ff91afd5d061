// probe_fp64.cu — single-warp latency of dependent fp64 chains on this GPU
// (DFMA, division, sqrt, atan2), in SM clocks per operation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/probe_fp64 tools/probe_fp64.cu
#include <cstdio>

__global__ void chains(double seed, long long* out, double* sink) {
    double x = seed;
    long long t0 = clock64();
    for (int i = 0; i < 1000; ++i) x = fma(x, 0.999999, 1e-7);
    long long t1 = clock64();
    for (int i = 0; i < 200; ++i) x = 1.0 + 1.0 / (x + 1.0);
    long long t2 = clock64();
    for (int i = 0; i < 200; ++i) x = sqrt(x + 1.0);
    long long t3 = clock64();
    for (int i = 0; i < 200; ++i) x = atan2(x, 0.75) + 1.0;
    long long t4 = clock64();
    for (int i = 0; i < 200; ++i) x = __shfl_sync(0xffffffffu, x, (i + threadIdx.x) & 31) + 1e-9;
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t1;
        out[2] = t3 - t2;
        out[3] = t4 - t3;
        out[4] = t5 - t4;
    }
    sink[threadIdx.x] = x;
}

int main() {
    long long* d;
    double* s;
    cudaMalloc(&d, 64);
    cudaMalloc(&s, 32 * 8);
    for (int rep = 0; rep < 3; ++rep) {
        chains<<<1, 32>>>(1.5, d, s);
        long long h[5];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        printf("clocks/op: dfma %.1f  div %.1f  sqrt %.1f  atan2 %.1f  shfl %.1f\n", h[0] / 1000.0,
               h[1] / 200.0, h[2] / 200.0, h[3] / 200.0, h[4] / 200.0);
    }
    return 0;
}
