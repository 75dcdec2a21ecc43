// Verifies the fragment layout assumed for mma.sync.aligned.m16n8k8.row.col.f64:
//   a0=(g,t) a1=(g+8,t) a2=(g,t+4) a3=(g+8,t+4); b0=(t,g) b1=(t+4,g);
//   c0=(g,2t) c1=(g,2t+1) c2=(g+8,2t) c3=(g+8,2t+1)
#include <cstdio>
#include <cmath>

__global__ void k(const double* A, const double* B, double* C) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    double a0 = A[g * 8 + t], a1 = A[(g + 8) * 8 + t], a2 = A[g * 8 + t + 4], a3 = A[(g + 8) * 8 + t + 4];
    double b0 = B[t * 8 + g], b1 = B[(t + 4) * 8 + g];
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
                 : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
    C[g * 8 + 2 * t] = c0;
    C[g * 8 + 2 * t + 1] = c1;
    C[(g + 8) * 8 + 2 * t] = c2;
    C[(g + 8) * 8 + 2 * t + 1] = c3;
}

int main() {
    double hA[128], hB[64], hC[128], ref[128];
    for (int i = 0; i < 128; ++i) hA[i] = 1.0 + i * 0.01 + (i % 7) * 0.3;
    for (int i = 0; i < 64; ++i) hB[i] = 0.5 - i * 0.02 + (i % 5) * 0.1;
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int q = 0; q < 8; ++q) s += hA[r * 8 + q] * hB[q * 8 + c];
            ref[r * 8 + c] = s;
        }
    double *A, *B, *C;
    cudaMalloc(&A, sizeof(hA));
    cudaMalloc(&B, sizeof(hB));
    cudaMalloc(&C, sizeof(hC));
    cudaMemcpy(A, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, sizeof(hB), cudaMemcpyHostToDevice);
    k<<<1, 32>>>(A, B, C);
    cudaMemcpy(hC, C, sizeof(hC), cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 128; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
    printf("m16n8k8 f64 layout max abs err %.3e (%s)\n", err, err < 1e-12 ? "OK" : "MISMATCH");
    return 0;
}
