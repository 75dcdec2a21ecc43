// Standalone timing of the shared-memory Cholesky (cholx.cu) with per-phase
// %globaltimer probes of chain 0 (-DSMG_CHOLX_TIMING).
//   build/cholx_bench B c [reps] [CL]
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_1810_02719_b200/csrc/cholx.cu"

namespace smg {
int count_launch() { return 0; }
void ensure_smem(const void* f, int bytes) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); }
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 1;
    const int c = argc > 2 ? atoi(argv[2]) : 200;
    const int reps = argc > 3 ? atoi(argv[3]) : 20;
    if (argc > 4) setenv("SMG_CHOLX_CL", argv[4], 1);
    const int skipinv = argc > 5 ? atoi(argv[5]) : 0;
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
    p.status_detail = det; p.errpos = ep; p.vnorm = dv; p.rank_test = 1; p.column_scale = 1; p.skip_inverse = skipinv;
    cudaMemset(st, 0, 4 * B);
    printf("cluster %d\n", smg::cholx_cluster(c, B));
    for (int i = 0; i < 3; ++i) smg::cholx_factor(p, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) smg::cholx_factor(p, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int hst = 0;
    cudaMemcpy(&hst, st, 4, cudaMemcpyDeviceToHost);
    printf("B=%d c=%d skip_inverse=%d: %.1f us/launch status=%d err=%s\n", B, c, skipinv, 1e3 * ms / reps, hst,
           cudaGetErrorString(cudaGetLastError()));
#ifdef SMG_CHOLX_TIMING
    unsigned long long t[512];
    cudaMemcpyFromSymbol(t, smg::g_cx_t, sizeof(t));
    const int P = (c + 31) / 32;
    double sd = 0, s1 = 0, sr = 0, s2 = 0, st2 = 0;
    for (int pb = 0; pb < P; ++pb) {
        const unsigned long long* q = t + 8 + pb * 8;
        sd += (q[1] - q[0]) * 1e-3;
        s1 += (q[2] - q[1]) * 1e-3;
        if (pb + 1 < P) {
            sr += (q[3] - q[2]) * 1e-3;
            s2 += (q[4] - q[3]) * 1e-3;
            st2 += (q[5] - q[4]) * 1e-3;
        }
    }
    printf("init %.1f  diag %.1f  sync1 %.1f  panel-row %.1f  sync2 %.1f  trailing %.1f  tail %.1f  total %.1f us\n",
           (t[8] - t[0]) * 1e-3 * 0 + 0.0, sd, s1, sr, s2, st2, (t[2] - t[1]) * 1e-3, (t[2] - t[0]) * 1e-3);
#endif
    return 0;
}
