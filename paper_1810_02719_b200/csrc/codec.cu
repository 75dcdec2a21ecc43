// F2: the spectral codec's per-block stages (compress.hpp:33-89, :378-474).
//
//  * encode_block (compress.hpp:33-62): per axis [lo, hi] of the c
//    coefficients, step = (hi - lo) / 2^q, value = clamp(long((x - lo) / step),
//    0, 2^q - 1); an axis with !(hi > lo) is flagged constant and sends no values.
//  * serialize_encoded_mesh's payload (compress.hpp:415-423): the values of the
//    non-constant axes, axis-major, q bits each, MSB first, padded to a byte per
//    block.  One thread per output byte gathers its 8 bits, so the packed stream
//    is written in one coalesced pass with no serial bit cursor.
//  * dequantize_block (compress.hpp:64-80): lo + (q + 0.5) * step, or lo on a
//    constant axis; the values are unpacked straight from the payload.
// Every floating-point step uses explicitly rounded intrinsics so no FMA
// contraction changes a quantisation decision or a decoded coefficient: the
// results are bit-identical to the reference's double arithmetic.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace smg {

namespace {

constexpr int CNT = 256;

// coefficients of position p: c x 3 column-major at coef[p] (signed, as gft returns)
__global__ void __launch_bounds__(CNT) encode_kernel(CodecParams p) {
    const int pos = blockIdx.x;
    const int c = p.c[pos];
    const double* x = p.coef[pos];
    const uint32_t levels = 1u << p.quant_bits;
    __shared__ double red_lo[CNT / 32], red_hi[CNT / 32];
    __shared__ double s_lo[3], s_hi[3];
    for (int a = 0; a < 3; ++a) {
        double lo = INFINITY, hi = -INFINITY;
        for (int i = threadIdx.x; i < c; i += CNT) {
            const double v = x[(int64_t)a * c + i];
            lo = fmin(lo, v);
            hi = fmax(hi, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if ((threadIdx.x & 31) == 0) {
            red_lo[threadIdx.x >> 5] = lo;
            red_hi[threadIdx.x >> 5] = hi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < CNT / 32; ++w) {
                lo = fmin(lo, red_lo[w]);
                hi = fmax(hi, red_hi[w]);
            }
            s_lo[a] = lo;
            s_hi[a] = hi;
        }
        __syncthreads();
    }
    uint16_t* vals = p.values + p.value_off[pos];
    int nconst_bits = 0;
    for (int a = 0; a < 3; ++a) {
        const double lo = s_lo[a], hi = s_hi[a];
        const bool constant = !(hi > lo);
        nconst_bits |= constant ? (1 << a) : 0;
        const double step = __ddiv_rn(__dsub_rn(hi, lo), (double)levels);
        for (int i = threadIdx.x; i < c; i += CNT) {
            uint16_t q = 0;
            if (!constant) {
                long v = (long)__ddiv_rn(__dsub_rn(x[(int64_t)a * c + i], lo), step);
                v = v < 0 ? 0 : (v > (long)levels - 1 ? (long)levels - 1 : v);
                q = (uint16_t)v;
            }
            vals[(int64_t)a * c + i] = q;
        }
    }
    if (threadIdx.x == 0) {
        for (int a = 0; a < 3; ++a) {
            p.lo[3 * pos + a] = s_lo[a];
            p.hi[3 * pos + a] = s_hi[a];
        }
        p.flags[pos] = (uint8_t)nconst_bits;
        const int axes = 3 - __popc(nconst_bits);
        p.payload_bytes[pos] = ((int64_t)axes * c * p.quant_bits + 7) / 8;
    }
}

// the a_rank-th non-constant axis
SMG_DEV int live_axis(int flags, int rank) {
    for (int a = 0; a < 3; ++a)
        if (!((flags >> a) & 1)) {
            if (rank == 0) return a;
            --rank;
        }
    return 2;
}

__global__ void __launch_bounds__(CNT) pack_kernel(CodecParams p) {
    const int pos = blockIdx.x;
    const int c = p.c[pos], q = p.quant_bits, flags = p.flags[pos];
    const int64_t nbits = (int64_t)(3 - __popc(flags)) * c * q;
    const int64_t nbytes = (nbits + 7) / 8;
    const uint16_t* vals = p.values + p.value_off[pos];
    uint8_t* out = p.payload + p.payload_off[pos];
    for (int64_t b = threadIdx.x; b < nbytes; b += CNT) {
        unsigned byte = 0;
        for (int j = 0; j < 8; ++j) {
            const int64_t bit = 8 * b + j;
            unsigned v = 0;
            if (bit < nbits) {
                const int64_t vi = bit / q;
                const int r = (int)(bit % q);
                const int a = live_axis(flags, (int)(vi / c));
                v = (vals[(int64_t)a * c + vi % c] >> (q - 1 - r)) & 1u;
            }
            byte = (byte << 1) | v;
        }
        out[b] = (uint8_t)byte;
    }
}

// dequantize straight from the payload into C (c x ldc row-major per position)
__global__ void __launch_bounds__(CNT) unpack_kernel(CodecParams p) {
    const int pos = blockIdx.x;
    const int c = p.c[pos], q = p.quant_bits, flags = p.flags[pos];
    const uint8_t* in = p.payload + p.payload_off[pos];
    const uint32_t levels = 1u << q;
    double* C = p.C + (int64_t)p.dest[pos] * p.strideC;  // by submesh id
    int rank = 0;
    for (int a = 0; a < 3; ++a) {
        const double lo = p.lo[3 * pos + a];
        const bool constant = (flags >> a) & 1;
        const double step = __ddiv_rn(__dsub_rn(p.hi[3 * pos + a], lo), (double)levels);
        for (int i = threadIdx.x; i < c; i += CNT) {
            double v = lo;
            if (!constant) {
                const int64_t bit0 = ((int64_t)rank * c + i) * q;
                unsigned val = 0;
                for (int r = 0; r < q; ++r) {
                    const int64_t bit = bit0 + r;
                    val = (val << 1) | ((in[bit >> 3] >> (7 - (bit & 7))) & 1u);
                }
                if (p.values) p.values[p.value_off[pos] + (int64_t)a * c + i] = (uint16_t)val;
                v = __dadd_rn(lo, __dmul_rn((double)val + 0.5, step));
            }
            C[(int64_t)i * p.ldc + a] = v;
        }
        rank += constant ? 0 : 1;
    }
}

}  // namespace

void codec_encode(const CodecParams& p, cudaStream_t st) {
    if (p.blocks <= 0) return;
    ::smg::count_launch(), encode_kernel<<<p.blocks, CNT, 0, st>>>(p);
}

void codec_pack(const CodecParams& p, cudaStream_t st) {
    if (p.blocks <= 0) return;
    ::smg::count_launch(), pack_kernel<<<p.blocks, CNT, 0, st>>>(p);
}

void codec_unpack(const CodecParams& p, cudaStream_t st) {
    if (p.blocks <= 0) return;
    ::smg::count_launch(), unpack_kernel<<<p.blocks, CNT, 0, st>>>(p);
}

}  // namespace smg
