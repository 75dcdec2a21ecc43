// Orthonormality probe for the adaptive CholeskyQR2 (K6/K7): decides per chain whether
// the pass-1 factor Q1 is already orthonormal WITHOUT forming the second Gram.
//
// With P = 8 fixed +-1 probe vectors X (c x 8, a hash of the column index),
//   Z = Q1^T (Q1 X) - X = (Q1^T Q1 - I) X,      E[ |Z|_F^2 / P ] = |Q1^T Q1 - I|_F^2
// (Hutchinson; E[x x^T] = I).  One pass over Q1 (n x c, read once: 8 n c bytes per chain
// instead of the Gram's n c^2 flops): a CTA takes 128 rows, stages 32 at a time in shared
// memory (rows padded to 4 mod 16 doubles: conflict-free DMMA fragments), forms y = Q_rows X
// (32 x 8) and accumulates z += Q_rows^T y (c x 8) on the FP64 tensor pipe (m8n8k4; the probe
// signs are generated in registers); the per-CTA partials are summed in chunk order by one
// CTA per chain, which sets skip[b] = (sqrt(|Z|_F^2 / P) <= tol).  Fixed order throughout.
// Chains that fail take the exact path (second Gram, near-identity or full second Cholesky).
// Replaces nothing in the reference: HouseholderQR (spectral.hpp:125-129) needs no second
// pass; this is the check that lets CholeskyQR2 stop after one.
#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int PROBES = 8, ROWS_PER_CTA = 128, PNT_ = 256, PWARPS = PNT_ / 32;
// SUB rows are staged at a time: 32, or 16 when two 32-row stages of a wide block (c > 432) would not fit
constexpr int MAX_MT = 8;  // column tiles (of 8) per warp: c <= 8 * 8 * 8 = 512

SMG_DEV unsigned probe_bits(int k) {
    unsigned h = (unsigned)k * 0x9E3779B9u + 0x7F4A7C15u;
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h & 0xFFu;
}

__host__ __device__ inline int probe_lds(int c) { return ((c + 15) / 16) * 16 + 4; }  // staged row stride, 4 mod 16

template <int SUB>
__global__ void __launch_bounds__(PNT_) orth_probe_partial_kernel(const double* __restrict__ Q, int64_t ldq,
                                                                  int64_t strideQ, int n, const int* dimC, int c_cap,
                                                                  double* __restrict__ part, int chunks) {
    extern __shared__ __align__(16) double psm[];
    const int b = blockIdx.y, chunk = blockIdx.x;
    const int c = dimC ? dimC[b] : c_cap;
    const int lds = probe_lds(c_cap);
    const int c8 = (c + 7) & ~7;          // columns staged (zero past c): whole 8-wide tiles
    double* Sbuf[2] = {psm, psm + SUB * lds};   // two SUB x lds stages (cp.async double buffer)
    constexpr int MTILES = SUB / 8, KPARTS = PWARPS / MTILES;  // y = S X: row tiles x k-range parts over the warps
    double* ysm = psm + 2 * SUB * lds;    // KPARTS partial (SUB x PROBES) blocks; block 0 receives the sum
    const double* q = Q + (int64_t)b * strideQ;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int r0 = chunk * ROWS_PER_CTA;
    const int ntile = c8 / 8;
    const int nsub = min(ROWS_PER_CTA / SUB, (n - r0 + SUB - 1) / SUB);
    double z[MAX_MT][2];
#pragma unroll
    for (int i = 0; i < MAX_MT; ++i) z[i][0] = z[i][1] = 0.0;
    // the padding (columns c..c8, rows past n) is zeroed once; the copies never touch it
    for (int e = tid; e < 2 * SUB * lds; e += PNT_) psm[e] = 0.0;
    __syncthreads();
    // stage sub-chunk `sub` into buffer sub & 1: whole double2 chunks + the odd last column
    auto stage = [&](int sub) {
        double* S = Sbuf[sub & 1];
        const int rs = r0 + sub * SUB, pairs = c / 2;
        for (int e = tid; e < SUB * pairs; e += PNT_) {
            const int r = e / pairs, kk = 2 * (e % pairs);
            if (rs + r < n) cp_async16(S + r * lds + kk, q + (int64_t)(rs + r) * ldq + kk);
        }
        if ((c & 1) && tid < SUB && rs + tid < n) {
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(S + tid * lds + c - 1));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(q + (int64_t)(rs + tid) * ldq + c - 1));
        }
        cp_async_commit();
    };
    if (nsub > 0) stage(0);
    for (int sub = 0; sub < nsub; ++sub) {
        if (sub + 1 < nsub) {
            // a partial last sub-chunk reuses a buffer that held full rows: clear the rows past n
            // (the buffer's previous reader finished at the barrier that ended sub - 1)
            const int nextrows = n - (r0 + (sub + 1) * SUB);
            if (nextrows < SUB) {
                double* Sn = Sbuf[(sub + 1) & 1];
                for (int e = tid; e < (SUB - nextrows) * lds; e += PNT_) Sn[nextrows * lds + e] = 0.0;
            }
            stage(sub + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* S = Sbuf[sub & 1];
        // y = S X: row tile warp % MTILES, the k range split in KPARTS parts
        {
            const int mt = warp % MTILES, part = warp / MTILES;
            const int ksteps = c8 / 4, per = (ksteps + KPARTS - 1) / KPARTS;
            const int kb = min(ksteps, part * per), ke = min(ksteps, kb + per);
            double y0[2] = {0.0, 0.0}, y1[2] = {0.0, 0.0};
            const double* srow = S + (8 * mt + g) * lds + t;
            int ks = kb;
            for (; ks + 1 < ke; ks += 2) {
                const double a0 = srow[4 * ks], a1 = srow[4 * ks + 4];
                const double b0 = ((probe_bits(4 * ks + t) >> g) & 1u) ? 1.0 : -1.0;
                const double b1 = ((probe_bits(4 * ks + 4 + t) >> g) & 1u) ? 1.0 : -1.0;
                dmma884(y0[0], y0[1], a0, b0);
                dmma884(y1[0], y1[1], a1, b1);
            }
            if (ks < ke) {
                const double a0 = srow[4 * ks];
                const double b0 = ((probe_bits(4 * ks + t) >> g) & 1u) ? 1.0 : -1.0;
                dmma884(y0[0], y0[1], a0, b0);
            }
            y0[0] += y1[0];
            y0[1] += y1[1];
            double* dst = ysm + part * (SUB * PROBES) + (8 * mt + g) * PROBES + 2 * t;
            *reinterpret_cast<double2*>(dst) = make_double2(y0[0], y0[1]);
        }
        __syncthreads();
        if (tid < SUB * PROBES) {
            double v = ysm[tid];
#pragma unroll
            for (int part = 1; part < KPARTS; ++part) v += ysm[part * (SUB * PROBES) + tid];
            ysm[tid] = v;
        }
        __syncthreads();
        // z += S^T y: column tiles warp, warp + 8, ...; k = the SUB rows
        {
            double bf[SUB / 4];
#pragma unroll
            for (int k4 = 0; k4 < SUB / 4; ++k4) bf[k4] = ysm[(4 * k4 + t) * PROBES + g];
#pragma unroll
            for (int i = 0; i < MAX_MT; ++i) {
                const int mt = warp + PWARPS * i;
                if (mt < ntile) {
#pragma unroll
                    for (int k4 = 0; k4 < SUB / 4; ++k4)
                        dmma884(z[i][0], z[i][1], S[(4 * k4 + t) * lds + 8 * mt + g], bf[k4]);
                }
            }
        }
        __syncthreads();
    }
    double* out = part + ((int64_t)b * chunks + chunk) * (int64_t)c_cap * PROBES;
#pragma unroll
    for (int i = 0; i < MAX_MT; ++i) {
        const int k = 8 * (warp + PWARPS * i) + g;
        if (k < c) *reinterpret_cast<double2*>(out + (int64_t)k * PROBES + 2 * t) = make_double2(z[i][0], z[i][1]);
    }
}

// Z = sum over chunks (in order) - X; est = sqrt(|Z|_F^2 / P).  A thread per (column, probe
// pair): the chunk loads are independent, the adds ordered.
constexpr int FNT_ = 1024;  // one item per thread at c = 200: two rounds of 8 independent loads
__global__ void __launch_bounds__(FNT_) orth_probe_finish_kernel(const double* __restrict__ part, int chunks, int n,
                                                                 const int* dimC, int c_cap, double tol, int* skip,
                                                                 double* est_out) {
    __shared__ double red[FNT_];
    const int b = blockIdx.x, tid = threadIdx.x;
    const int c = dimC ? dimC[b] : c_cap;
    const int live = min(chunks, (n + ROWS_PER_CTA - 1) / ROWS_PER_CTA);
    double ss = 0.0;
    for (int item = tid; item < c * (PROBES / 2); item += FNT_) {
        const int k = item / (PROBES / 2), pp = 2 * (item % (PROBES / 2));
        const double* src = part + ((int64_t)b * chunks * c_cap + k) * PROBES + pp;
        double2 zs = make_double2(0.0, 0.0);
        for (int ch0 = 0; ch0 < live; ch0 += 8) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = ch0 + u < live ? __ldcg(reinterpret_cast<const double2*>(src + (int64_t)(ch0 + u) * c_cap * PROBES))
                                      : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                zs.x += v[u].x;
                zs.y += v[u].y;
            }
        }
        const unsigned bits = probe_bits(k);
        zs.x -= ((bits >> pp) & 1u) ? 1.0 : -1.0;
        zs.y -= ((bits >> (pp + 1)) & 1u) ? 1.0 : -1.0;
        ss += zs.x * zs.x + zs.y * zs.y;
    }
    red[tid] = ss;
    __syncthreads();
    for (int o = FNT_ / 2; o > 0; o >>= 1) {
        if (tid < o) red[tid] += red[tid + o];
        __syncthreads();
    }
    if (tid == 0) {
        const double est = sqrt(red[0] / PROBES);
        skip[b] = (est <= tol) ? 1 : 0;  // NaN -> no skip
        if (est_out) est_out[b] = est;
    }
}

}  // namespace

int orth_probe_chunks(int n) { return (n + ROWS_PER_CTA - 1) / ROWS_PER_CTA; }

void orth_probe(const double* Q, int64_t ldq, int64_t strideQ, int n, const int* dimC, int c_cap, int batch, double tol,
                double* part, int* skip, double* est_out, cudaStream_t st) {
    const int chunks = orth_probe_chunks(n);
    const int lds = probe_lds(c_cap);
    const int bytes32 = (2 * 32 * lds + PWARPS * 8 * PROBES) * (int)sizeof(double);
    const int bytes16 = (2 * 16 * lds + PWARPS * 8 * PROBES) * (int)sizeof(double);
    if (bytes32 <= 220 * 1024) {
        ensure_smem((const void*)orth_probe_partial_kernel<32>, bytes32);
        ::smg::count_launch(), orth_probe_partial_kernel<32><<<dim3(chunks, batch), PNT_, bytes32, st>>>(
            Q, ldq, strideQ, n, dimC, c_cap, part, chunks);
    } else {
        ensure_smem((const void*)orth_probe_partial_kernel<16>, bytes16);
        ::smg::count_launch(), orth_probe_partial_kernel<16><<<dim3(chunks, batch), PNT_, bytes16, st>>>(
            Q, ldq, strideQ, n, dimC, c_cap, part, chunks);
    }
    ::smg::count_launch(), orth_probe_finish_kernel<<<batch, FNT_, 0, st>>>(part, chunks, n, dimC, c_cap, tol, skip,
                                                                            est_out);
}

}  // namespace smg
