// Standalone timing of the block-tridiagonal solve kernel (K3) on a C5-shaped
// batch: B chains, n = 2048, W (64 or 32), c = 200, z = 2, optional row
// permutation.  Random factor slabs (the timing does not depend on the values).
//   solve_bench [B] [c] [reps] [W] [perm]        Build: make tools
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1810_02719_b200/csrc/solve.cu"

namespace smg {
int count_launch() { return 0; }
void ensure_smem(const void* f, int bytes) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); }
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 32;
    const int c = argc > 2 ? atoi(argv[2]) : 200;
    const int reps = argc > 3 ? atoi(argv[3]) : 20;
    const int W = argc > 4 ? atoi(argv[4]) : 64;
    const int use_perm = argc > 5 ? atoi(argv[5]) : 0;
    const int n = 2048, Kb = n / W, ld = (c + 31) / 32 * 32;
    const int64_t strideF = (int64_t)Kb * 2 * W * smg::factor_row(W);
    double *Ff, *Fb, *in, *tmp, *out;
    cudaMalloc(&Ff, sizeof(double) * strideF * B);
    cudaMalloc(&Fb, sizeof(double) * strideF * B);
    cudaMalloc(&in, sizeof(double) * (int64_t)n * ld * B);
    cudaMalloc(&tmp, sizeof(double) * (int64_t)n * ld * B);
    cudaMalloc(&out, sizeof(double) * (int64_t)n * ld * B);
    std::vector<double> h(strideF);
    for (auto& v : h) v = (rand() / (double)RAND_MAX - 0.5) * 1e-2;
    for (int b = 0; b < B; ++b) {
        cudaMemcpy(Ff + b * strideF, h.data(), sizeof(double) * strideF, cudaMemcpyHostToDevice);
        cudaMemcpy(Fb + b * strideF, h.data(), sizeof(double) * strideF, cudaMemcpyHostToDevice);
    }
    cudaMemset(in, 0, sizeof(double) * (int64_t)n * ld * B);
    smg::SolveParams p;
    p.n = n; p.Kb = Kb; p.z = 2; p.c_cap = c; p.batch = B;
    p.Ffwd = Ff; p.Fbwd = Fb; p.strideF = strideF;
    p.in = in; p.ldin = ld; p.strideIn = (int64_t)n * ld;
    p.tmp = tmp; p.ldt = ld; p.strideT = (int64_t)n * ld;
    p.out = out; p.ldout = ld; p.strideOut = (int64_t)n * ld;
    int32_t* perm = nullptr;
    if (use_perm) {
        std::vector<int32_t> ph((size_t)n * B);
        for (int b = 0; b < B; ++b)
            for (int i = 0; i < n; ++i) ph[(size_t)b * n + i] = (i * 37 + 11) % n;  // a fixed scatter
        cudaMalloc(&perm, sizeof(int32_t) * ph.size());
        cudaMemcpy(perm, ph.data(), sizeof(int32_t) * ph.size(), cudaMemcpyHostToDevice);
        p.perm = perm;
        p.stridePerm = n;
    }
    for (int i = 0; i < 3; ++i) smg::solve_block_tridiag(p, W, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) smg::solve_block_tridiag(p, W, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = 1e3 * ms / reps;
    const double algo = (double)B * 2 * 4.0 * n * 65 * c;  // z*4*n*b*c
    printf("W=%d perm=%d ", W, use_perm);
    printf("B=%d c=%d: %.1f us/launch, algorithmic %.2f TFLOP/s (%.1f%% of 37.18) err=%s\n", B, c, us,
           algo / (us * 1e-6) / 1e12, 100 * algo / (us * 1e-6) / 1e12 / 37.18, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
