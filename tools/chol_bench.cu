// Standalone timing of the CholeskyQR factor kernel (K6) for a batch of c x c
// Gram matrices G = V^T V (V: n x c Gaussian, graded columns), with per-phase
// clock64 probes of CTA 0 (-DSMG_CHOL_TIMING).  Build: make tools
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_1810_02719_b200/csrc/cholqr.cu"

namespace smg {
int count_launch() { return 0; }
void ensure_smem(const void* f, int bytes) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); }
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 4;
    const int c = argc > 2 ? atoi(argv[2]) : 200;
    const int reps = argc > 3 ? atoi(argv[3]) : 20;
    const int ld = (c + 31) / 32 * 32, n = 2048;
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    std::vector<double> V((size_t)n * c), G((size_t)ld * ld, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < c; ++j) V[(size_t)i * c + j] = nd(rng) * (1.0 + j);
    for (int a = 0; a < c; ++a)
        for (int b2 = 0; b2 < c; ++b2) {
            double s = 0;
            for (int i = 0; i < n; ++i) s += V[(size_t)i * c + a] * V[(size_t)i * c + b2];
            G[(size_t)a * ld + b2] = s;
        }
    double *dG, *dA, *dB, *dD, *dv;
    int *st, *ep;
    int64_t* det;
    const size_t mat = (size_t)ld * ld;
    cudaMalloc(&dG, 8 * mat * B);
    cudaMalloc(&dA, 8 * mat * B);
    cudaMalloc(&dB, 8 * mat * B);
    cudaMalloc(&dD, 8 * (size_t)ld * B);
    cudaMalloc(&dv, 8 * (size_t)B);
    cudaMalloc(&st, 4 * B);
    cudaMalloc(&ep, 4 * B);
    cudaMalloc(&det, 8 * B);
    for (int b = 0; b < B; ++b) cudaMemcpy(dG + b * mat, G.data(), 8 * mat, cudaMemcpyHostToDevice);
    smg::CholParams p;
    p.batch = B; p.c_cap = c; p.G = dG; p.ldg = ld; p.strideG = mat; p.A = dA; p.lda = ld; p.strideA = mat;
    p.Binv = dB; p.ldb = ld; p.strideB = mat; p.dscale = dD; p.strideD = ld; p.status = st;
    p.status_detail = det; p.errpos = ep; p.vnorm = dv; p.rank_test = 1; p.column_scale = 1;
    cudaMemset(st, 0, 4 * B);
    for (int i = 0; i < 3; ++i) smg::chol_factor(p, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) smg::chol_factor(p, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int hst = 0;
    cudaMemcpy(&hst, st, 4, cudaMemcpyDeviceToHost);
    printf("B=%d c=%d: %.1f us/launch status=%d err=%s\n", B, c, 1e3 * ms / reps, hst,
           cudaGetErrorString(cudaGetLastError()));
#ifdef SMG_CHOL_TIMING
    long long t[128];
    cudaMemcpyFromSymbol(t, smg::g_chol_t, sizeof(t));
    const int P = (c + 31) / 32;
    const double f = 1.0 / 1.965e3;  // cycles -> us at 1965 MHz
    printf("init %.1f us\n", (t[1] - t[0]) * f);
    double sa = 0, si = 0, sb = 0, sc = 0, sl = 0;
    for (int pb = 0; pb < P; ++pb) {
        const long long* q = t + 2 + pb * 5;
        const long long prev = pb == 0 ? t[1] : t[2 + (pb - 1) * 5 + 4];
        sl += (q[0] - prev) * f; sa += (q[1] - q[0]) * f; si += (q[2] - q[1]) * f;
        sb += (q[3] - q[2]) * f; sc += (q[4] - q[3]) * f;
    }
    printf("panel load %.1f  factor %.1f  diag-inverse %.1f  panel-row+B %.1f  trailing %.1f  back-subst %.1f  total %.1f us\n",
           sl, sa, si, sb, sc, (t[127] - t[2 + (P - 1) * 5 + 4]) * f, (t[127] - t[0]) * f);
#endif
    return 0;
}
