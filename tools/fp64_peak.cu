// FP64 peak microbenchmark: DFMA vs DMMA (mma.sync m8n8k4 f64) on sm_100a.
// Used once to pick the FP64 GEMM micro-kernel style and as the FP64 roofline
// denominator (MEASURED_PEAKS.json carries no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double d[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { d[t][0] = 0; d[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(d[t][0]), "+d"(d[t][1]) : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16_kernel(double* out, int iters) {
  double a[4], b[2];
  for (int q = 0; q < 4; ++q) a[q] = threadIdx.x * 1e-9 + q;
  for (int q = 0; q < 2; ++q) b[q] = 1.0 - threadIdx.x * 1e-9 - q;
  double d[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) d[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(d[t][0]), "+d"(d[t][1]), "+d"(d[t][2]), "+d"(d[t][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      }
    }
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) s += d[t][q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  for (int threads : {256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = p.multiProcessorCount * bps;
      dfma_kernel<<<blocks, threads>>>(out, 10);
      cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * 16 * (double)iters * blocks * threads;
      printf("DFMA  threads=%d blocks=%d : %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
      dmma_kernel<<<blocks, threads>>>(out, 10);
      cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * 16 * (double)iters * blocks * (threads / 32);
      printf("DMMA m8n8k4 threads=%d blocks=%d : %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
      dmma16_kernel<<<blocks, threads>>>(out, 10);
      cudaEventRecord(e0); dmma16_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 16 * 8 * 8 * 4 * 16 * (double)iters * blocks * (threads / 32);
      printf("DMMA m16n8k8 threads=%d blocks=%d : %.2f TFLOP/s (%s)\n", threads, blocks, fl / ms / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
