// DMMA (mma.sync m8n8k4 f64) issue/latency probe: W warps per CTA, one CTA per SM, each warp
// running ILP independent accumulator chains of N dependent DMMAs.  Prints cycles per DMMA per
// warp and the SM-level DMMA rate.      nvcc -arch=sm_100a -O3 -o build/dmma_lat tools/dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int ILP>
__global__ void probe(double* out, long long* cyc, int n) {
    double acc[ILP][2];
    for (int i = 0; i < ILP; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) dmma(acc[i][0], acc[i][1], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
void run(int warps, double* out, long long* cyc) {
    const int n = 4096;
    probe<ILP><<<148, 32 * warps>>>(out, cyc, n);
    probe<ILP><<<148, 32 * warps>>>(out, cyc, n);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double per = (double)h / ((double)n * ILP);
    printf("warps=%2d ILP=%d: %.1f cyc per DMMA per warp, SM rate one DMMA per %.2f cyc\n", warps, ILP, per, per / warps);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * 148 * 1024);
    cudaMalloc(&cyc, sizeof(long long));
    for (int w : {1, 2, 4, 8, 16}) {
        run<1>(w, out, cyc);
        run<2>(w, out, cyc);
        run<4>(w, out, cyc);
        run<8>(w, out, cyc);
    }
    return 0;
}
